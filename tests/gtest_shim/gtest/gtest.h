// Minimal GoogleTest-compatible shim (TEST INFRASTRUCTURE).
//
// GoogleTest is not installed in this image; this header implements the subset
// of its API the reference suites use (TEST, TEST_F, ::testing::Test,
// EXPECT_/ASSERT_ EQ NE LT LE GT GE TRUE FALSE NEAR DOUBLE_EQ THROW NO_THROW,
// with `<< message` streaming) so /root/reference/proj/tests/*_test.cpp compile
// unchanged against the drop-in headers and run on the GPU backend.  main() is
// provided here (gtest_main equivalent); exit code = number of failed tests.
#pragma once

#include <cmath>
#include <cstring>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

class Test {
 public:
  virtual ~Test() = default;
  virtual void SetUp() {}
  virtual void TearDown() {}
  virtual void TestBody() = 0;
};

namespace internal {

struct Registry {
  struct Entry {
    std::string name;
    std::function<Test*()> make;
  };
  std::vector<Entry> tests;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

inline bool& current_failed() {
  static bool f = false;
  return f;
}

struct AssertFatal {};

// Collects the optional streamed message of a failed assertion and reports on
// destruction (fatal assertions throw AssertFatal after reporting).
class Reporter {
 public:
  Reporter(bool ok, const char* file, int line, std::string what, bool fatal)
      : ok_(ok), file_(file), line_(line), what_(std::move(what)), fatal_(fatal) {}
  Reporter(const Reporter&) = delete;
  ~Reporter() noexcept(false) {
    if (ok_) return;
    current_failed() = true;
    std::cerr << file_ << ":" << line_ << ": Failure\n" << what_;
    const std::string m = msg_.str();
    if (!m.empty()) std::cerr << "\n  " << m;
    std::cerr << std::endl;
    if (fatal_ && std::uncaught_exceptions() == 0) throw AssertFatal{};
  }
  template <class T>
  Reporter& operator<<(const T& v) {
    if (!ok_) msg_ << v;
    return *this;
  }

 private:
  bool ok_;
  const char* file_;
  int line_;
  std::string what_;
  bool fatal_;
  std::ostringstream msg_;
};

template <class T>
std::string show(const T& v) {
  std::ostringstream o;
  if constexpr (requires(std::ostream& os, const T& x) { os << x; }) {
    o.precision(17);
    o << v;
  } else if constexpr (requires(const T& x) { x.begin(); x.end(); }) {
    o << "{";
    bool first = true;
    for (const auto& e : v) {
      o << (first ? "" : ", ") << show(e);
      first = false;
    }
    o << "}";
  } else {
    o << "<value>";
  }
  return o.str();
}

template <class A, class B>
std::string binmsg(const char* op, const char* ea, const char* eb, const A& a, const B& b) {
  return std::string("Expected: (") + ea + ") " + op + " (" + eb + "), actual: " + show(a) + " vs " + show(b);
}

inline bool near(double a, double b, double tol) { return std::fabs(a - b) <= tol; }

// 4-ULP equality, as GoogleTest's EXPECT_DOUBLE_EQ
inline bool double_eq(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return false;
  auto biased = [](double x) {
    int64_t i;
    std::memcpy(&i, &x, sizeof i);
    return i < 0 ? static_cast<uint64_t>(~i) + 1 : static_cast<uint64_t>(i) | (uint64_t{1} << 63);
  };
  const uint64_t ua = biased(a), ub = biased(b);
  return (ua > ub ? ua - ub : ub - ua) <= 4;
}

struct Registrar {
  Registrar(const char* suite, const char* name, std::function<Test*()> make) {
    Registry::get().tests.push_back({std::string(suite) + "." + name, std::move(make)});
  }
};

}  // namespace internal
}  // namespace testing

#include <cstring>

#define GTEST_SHIM_CLASS(suite, name) suite##_##name##_Test

#define TEST_F(fixture, name)                                                                  \
  class GTEST_SHIM_CLASS(fixture, name) : public fixture {                                     \
   public:                                                                                     \
    void TestBody() override;                                                                  \
  };                                                                                           \
  static ::testing::internal::Registrar GTEST_SHIM_CLASS(fixture, name##_reg)(                 \
      #fixture, #name, [] { return static_cast<::testing::Test*>(new GTEST_SHIM_CLASS(fixture, name)); }); \
  void GTEST_SHIM_CLASS(fixture, name)::TestBody()

#define TEST(suite, name) TEST_F_PLAIN(suite, name)
#define TEST_F_PLAIN(suite, name)                                                              \
  class GTEST_SHIM_CLASS(suite, name) : public ::testing::Test {                               \
   public:                                                                                     \
    void TestBody() override;                                                                  \
  };                                                                                           \
  static ::testing::internal::Registrar GTEST_SHIM_CLASS(suite, name##_reg)(                   \
      #suite, #name, [] { return static_cast<::testing::Test*>(new GTEST_SHIM_CLASS(suite, name)); }); \
  void GTEST_SHIM_CLASS(suite, name)::TestBody()

#define GTEST_SHIM_REPORT(ok, what, fatal) ::testing::internal::Reporter((ok), __FILE__, __LINE__, (what), (fatal))

#define GTEST_SHIM_BIN(a, b, op, fatal)                                                         \
  for (bool gtest_shim_once = true; gtest_shim_once; gtest_shim_once = false)                   \
    for (const auto gtest_a = (a); gtest_shim_once; gtest_shim_once = false)                    \
      for (const auto gtest_b = (b); gtest_shim_once; gtest_shim_once = false)                  \
  GTEST_SHIM_REPORT(gtest_a op gtest_b, ::testing::internal::binmsg(#op, #a, #b, gtest_a, gtest_b), fatal)

#define EXPECT_EQ(a, b) GTEST_SHIM_BIN(a, b, ==, false)
#define EXPECT_NE(a, b) GTEST_SHIM_BIN(a, b, !=, false)
#define EXPECT_LT(a, b) GTEST_SHIM_BIN(a, b, <, false)
#define EXPECT_LE(a, b) GTEST_SHIM_BIN(a, b, <=, false)
#define EXPECT_GT(a, b) GTEST_SHIM_BIN(a, b, >, false)
#define EXPECT_GE(a, b) GTEST_SHIM_BIN(a, b, >=, false)
#define ASSERT_EQ(a, b) GTEST_SHIM_BIN(a, b, ==, true)
#define ASSERT_NE(a, b) GTEST_SHIM_BIN(a, b, !=, true)
#define ASSERT_LE(a, b) GTEST_SHIM_BIN(a, b, <=, true)
#define ASSERT_GE(a, b) GTEST_SHIM_BIN(a, b, >=, true)

#define FAIL() GTEST_SHIM_REPORT(false, std::string("Failed"), true)
#define ADD_FAILURE() GTEST_SHIM_REPORT(false, std::string("Failure"), false)
#define EXPECT_TRUE(c) GTEST_SHIM_REPORT(static_cast<bool>(c), std::string("Expected true: ") + #c, false)
#define EXPECT_FALSE(c) GTEST_SHIM_REPORT(!static_cast<bool>(c), std::string("Expected false: ") + #c, false)
#define ASSERT_TRUE(c) GTEST_SHIM_REPORT(static_cast<bool>(c), std::string("Expected true: ") + #c, true)
#define ASSERT_FALSE(c) GTEST_SHIM_REPORT(!static_cast<bool>(c), std::string("Expected false: ") + #c, true)

#define EXPECT_NEAR(a, b, tol)                                                                   \
  for (bool gtest_shim_once = true; gtest_shim_once; gtest_shim_once = false)                     \
    for (const double gtest_a = (a), gtest_b = (b), gtest_t = (tol); gtest_shim_once; gtest_shim_once = false) \
  GTEST_SHIM_REPORT(::testing::internal::near(gtest_a, gtest_b, gtest_t),                         \
                    ::testing::internal::binmsg("~=", #a, #b, gtest_a, gtest_b) + " tol " +      \
                        ::testing::internal::show(gtest_t),                                      \
                    false)

#define EXPECT_DOUBLE_EQ(a, b)                                                                   \
  for (bool gtest_shim_once = true; gtest_shim_once; gtest_shim_once = false)                     \
    for (const double gtest_a = (a), gtest_b = (b); gtest_shim_once; gtest_shim_once = false)     \
  GTEST_SHIM_REPORT(::testing::internal::double_eq(gtest_a, gtest_b),                             \
                    ::testing::internal::binmsg("==", #a, #b, gtest_a, gtest_b), false)

#define EXPECT_THROW(stmt, exc)                                                                  \
  for (bool gtest_shim_once = true; gtest_shim_once; gtest_shim_once = false)                     \
    for (int gtest_r = [&] {                                                                     \
           try {                                                                                 \
             stmt;                                                                               \
           } catch (const exc&) {                                                                \
             return 0;                                                                           \
           } catch (...) {                                                                       \
             return 2;                                                                           \
           }                                                                                     \
           return 1;                                                                             \
         }();                                                                                    \
         gtest_shim_once; gtest_shim_once = false)                                               \
  GTEST_SHIM_REPORT(gtest_r == 0,                                                                \
                    std::string("Expected: ") + #stmt + " throws " + #exc +                      \
                        (gtest_r == 1 ? " (nothing thrown)" : " (other exception)"),             \
                    false)

#define EXPECT_NO_THROW(stmt)                                                                    \
  for (bool gtest_shim_once = true; gtest_shim_once; gtest_shim_once = false)                     \
    for (int gtest_r = [&] {                                                                     \
           try {                                                                                 \
             stmt;                                                                               \
           } catch (...) {                                                                       \
             return 1;                                                                           \
           }                                                                                     \
           return 0;                                                                             \
         }();                                                                                    \
         gtest_shim_once; gtest_shim_once = false)                                               \
  GTEST_SHIM_REPORT(gtest_r == 0, std::string("Expected no throw: ") + #stmt, false)

#ifndef GTEST_SHIM_NO_MAIN
int main() {
  int failed = 0, run = 0;
  for (auto& e : ::testing::internal::Registry::get().tests) {
    ::testing::internal::current_failed() = false;
    std::cout << "[ RUN      ] " << e.name << std::endl;
    ::testing::Test* t = e.make();
    try {
      t->SetUp();
      t->TestBody();
    } catch (const ::testing::internal::AssertFatal&) {
    } catch (const std::exception& ex) {
      ::testing::internal::current_failed() = true;
      std::cerr << "uncaught exception: " << ex.what() << std::endl;
    }
    try {
      t->TearDown();
    } catch (...) {
    }
    delete t;
    ++run;
    const bool f = ::testing::internal::current_failed();
    failed += f ? 1 : 0;
    std::cout << (f ? "[  FAILED  ] " : "[       OK ] ") << e.name << std::endl;
  }
  std::cout << "[==========] " << run << " tests ran, " << failed << " failed" << std::endl;
  return failed;
}
#endif
