// Minimal CLI11-compatible shim (TEST INFRASTRUCTURE).
//
// CLI11 is not installed in this image.  This header implements the subset of its
// API that the reference's command-line driver uses (/root/reference/proj/tools/
// hestat_cli.cpp: App, add_subcommand, add_option, add_flag, Option::required /
// count, App::callback / require_subcommand / parsed, ValidationError,
// CLI11_PARSE), so that driver compiles unchanged: once against the drop-in
// headers and libhestat_gpu.so (tests/dropin/Makefile -> build/hestat_cli_gpu), and
// once against the reference headers (oracle/Makefile -> oracle/_ref/hestat_cli_ref)
// to produce the golden reports in tests/golden/cli/.
#pragma once

#include <cstdint>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct Error : std::runtime_error {
  int code;
  Error(const std::string& msg, int c) : std::runtime_error(msg), code(c) {}
};
struct ParseError : Error {
  explicit ParseError(const std::string& msg, int c = 109) : Error(msg, c) {}
};
struct ValidationError : ParseError {
  ValidationError(const std::string& name, const std::string& msg) : ParseError(name + ": " + msg, 105) {}
};

class Option {
 public:
  Option(std::string name, bool flag, std::function<void(const std::string&)> set)
      : name_(std::move(name)), flag_(flag), set_(std::move(set)) {}
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  std::size_t count() const { return count_; }

 private:
  friend class App;
  std::string name_;
  bool flag_;
  bool required_ = false;
  std::size_t count_ = 0;
  std::function<void(const std::string&)> set_;
};

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}

  App* add_subcommand(const std::string& name, const std::string& desc = "") {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }
  void require_subcommand(int n) { require_sub_ = n; }
  void callback(std::function<void()> f) { callback_ = std::move(f); }
  bool parsed() const { return parsed_; }

  template <class T>
  Option* add_option(const std::string& name, T& var, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(name, false, [&var, name](const std::string& v) { assign(var, v, name); }));
    return opts_.back().get();
  }
  Option* add_flag(const std::string& name, bool& var, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(name, true, [&var](const std::string&) { var = true; }));
    return opts_.back().get();
  }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    std::size_t i = 0;
    parse_args(args, i);
  }
  int exit(const Error& e) const {
    std::cerr << e.what() << '\n';
    return e.code == 0 ? 1 : e.code;
  }

 private:
  template <class T>
  static void assign(T& var, const std::string& v, const std::string& name) {
    try {
      std::size_t used = 0;
      if constexpr (std::is_same_v<T, std::string>) {
        var = v;
        used = v.size();
      } else if constexpr (std::is_floating_point_v<T>) {
        var = static_cast<T>(std::stod(v, &used));
      } else if constexpr (std::is_unsigned_v<T>) {
        if (!v.empty() && v[0] == '-') throw std::invalid_argument(v);
        var = static_cast<T>(std::stoull(v, &used));
      } else {
        var = static_cast<T>(std::stoll(v, &used));
      }
      if (used != v.size()) throw std::invalid_argument(v);
    } catch (const std::exception&) {
      throw ParseError(name + ": cannot parse '" + v + "'", 106);
    }
  }

  Option* find(const std::string& name) {
    for (auto& o : opts_)
      if (o->name_ == name) return o.get();
    return nullptr;
  }

  void parse_args(const std::vector<std::string>& args, std::size_t& i) {
    parsed_ = true;
    while (i < args.size()) {
      const std::string& a = args[i];
      if (a.rfind("--", 0) == 0) {
        std::string name = a, value;
        bool inline_value = false;
        const auto eq = a.find('=');
        if (eq != std::string::npos) {
          name = a.substr(0, eq);
          value = a.substr(eq + 1);
          inline_value = true;
        }
        Option* o = find(name);
        if (!o) throw ParseError("unknown option " + name, 109);
        if (!o->flag_ && !inline_value) {
          if (i + 1 >= args.size()) throw ParseError(name + " needs a value", 109);
          value = args[++i];
        }
        o->set_(value);
        ++o->count_;
        ++i;
        continue;
      }
      App* sub = nullptr;
      for (auto& s : subs_)
        if (s->name_ == a) sub = s.get();
      if (!sub) throw ParseError("unexpected argument " + a, 109);
      ++i;
      sub->parse_args(args, i);
    }
    for (auto& o : opts_)
      if (o->required_ && o->count_ == 0) throw ParseError(o->name_ + " is required", 106);
    if (require_sub_ > 0) {
      int n = 0;
      for (auto& s : subs_) n += s->parsed_ ? 1 : 0;
      if (n < require_sub_) throw ParseError("a subcommand is required", 106);
    }
    if (callback_) callback_();
  }

  std::string desc_, name_;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
  std::function<void()> callback_;
  int require_sub_ = 0;
  bool parsed_ = false;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv) \
  try {                              \
    (app).parse((argc), (argv));     \
  } catch (const CLI::Error& e) {    \
    return (app).exit(e);            \
  }
