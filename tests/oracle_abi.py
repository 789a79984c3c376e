"""ctypes harness over the CPU oracles (TEST INFRASTRUCTURE ONLY).

Two libraries share one C ABI (oracle/hestat_oracle.h):
  * ``oracle/liboracle.so``          -- the C restatement (prefix ``ora_``),
  * ``oracle/_ref/libhestat_ref.so`` -- the unmodified reference headers behind
    oracle/ref_shim.cpp (prefix ``ref_``), present where the reference compiled.

Every call returns an ``OResult(rc, out, levels, meter)`` so tests can compare
status codes, slot bit patterns, levels and meters in one assertion.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import NamedTuple, Optional, Sequence

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libhestat_ref.so")

OP_ADD, OP_SUB, OP_ADD_PT, OP_MUL_CT, OP_MUL_PT, OP_MUL_PT_VEC, OP_ROTATE, OP_BOOTSTRAP, OP_SUM_ALL = range(9)
FIT_INVSQRT_SHIFTED, FIT_SQRT_SHIFTED, FIT_IDENT, FIT_SQUARE, FIT_EXP, FIT_RECIP2, FIT_COS2, FIT_COS3, FIT_ONE, FIT_SQRT = range(10)
INV_SQRT, INV, BASELINE_INVSQRT, SQRT = range(4)
ST_MEAN, ST_VAR, ST_VAR_TO_SCALE, ST_MOMENTS, ST_ZNORM, ST_KURT, ST_SKEW, ST_CV, ST_PEARSON = range(9)
ALL_SLOTS = (1 << 64) - 1


class _Params(C.Structure):
    _fields_ = [("slot_count", C.c_uint64), ("max_level", C.c_int32), ("scale_bits", C.c_int32),
                ("quantize", C.c_int32), ("auto_bootstrap", C.c_int32), ("debug_checks", C.c_int32),
                ("_pad", C.c_int32)]


class _Meter(C.Structure):
    _fields_ = [("mul_ct", C.c_uint64), ("mul_pt", C.c_uint64), ("add", C.c_uint64),
                ("rotate", C.c_uint64), ("bootstrap", C.c_uint64)]


class _Cfg(C.Structure):
    _fields_ = [("n", C.c_int32), ("cheb_degree", C.c_int32), ("newton_iters", C.c_int32),
                ("baseline_mode", C.c_int32), ("baseline_iters", C.c_int32), ("_pad", C.c_int32)]


@dataclass
class Params:
    slot_count: int = 32768
    max_level: int = 11
    scale_bits: int = 40
    quantize: bool = True
    auto_bootstrap: bool = True
    debug_checks: bool = False

    def c(self) -> _Params:
        return _Params(self.slot_count, self.max_level, self.scale_bits, int(self.quantize),
                       int(self.auto_bootstrap), int(self.debug_checks), 0)


@dataclass
class Cfg:
    n: int = 2
    cheb_degree: int = 511
    newton_iters: int = 6
    baseline_mode: bool = False
    baseline_iters: int = 0

    def c(self) -> _Cfg:
        return _Cfg(self.n, self.cheb_degree, self.newton_iters, int(self.baseline_mode),
                    self.baseline_iters, 0)


class OResult(NamedTuple):
    rc: int
    out: np.ndarray
    levels: tuple
    meter: tuple


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _arr(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.float64))


class OracleLib:
    """One of the two oracle libraries, selected by path + symbol prefix."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        self._f = lambda name: getattr(self.lib, prefix + name)
        self._f("last_error").restype = C.c_char_p
        self._f("eval_plain").restype = C.c_double
        self._f("eval_plain").argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_double, C.c_double,
                                          C.c_double, C.POINTER(C.c_int32)]

    def last_error(self) -> str:
        return self._f("last_error")().decode()

    # -- ckks.hpp ---------------------------------------------------------
    def encrypt(self, p: Params, v) -> OResult:
        v = _arr(v)
        out = np.zeros(p.slot_count)
        lvl = C.c_int32(0)
        rc = self._f("encrypt")(C.byref(p.c()), _dp(v), C.c_uint64(len(v)), _dp(out), C.byref(lvl))
        return OResult(rc, out, (lvl.value,), (0,) * 5)

    def op(self, p: Params, op: int, a, la: int, b=None, lb: int = 0, c: float = 0.0, vec=None,
           k: int = 0, n_valid: int = 0) -> OResult:
        a = _arr(a)
        b = None if b is None else _arr(b)
        vec = None if vec is None else _arr(vec)
        out = np.zeros(p.slot_count)
        lvl = C.c_int32(0)
        m = _Meter()
        rc = self._f("op")(C.byref(p.c()), C.c_int(op), _dp(a), C.c_uint64(len(a)), C.c_int32(la),
                           _dp(b), C.c_uint64(0 if b is None else len(b)), C.c_int32(lb),
                           C.c_double(c), _dp(vec), C.c_uint64(0 if vec is None else len(vec)),
                           C.c_int64(k), C.c_uint64(n_valid), _dp(out), C.byref(lvl), C.byref(m))
        return OResult(rc, out, (lvl.value,), _mt(m))

    # -- chebyshev.hpp ----------------------------------------------------
    def fit(self, kind: int, S: float, degree: int, lo: float = -1.0, hi: float = 1.0):
        out = np.zeros(max(degree + 1, 1))
        rc = self._f("fit")(C.c_int(kind), C.c_double(S), C.c_int32(degree), C.c_double(lo),
                            C.c_double(hi), _dp(out))
        return rc, out

    def eval_plain(self, coeffs, lo: float, hi: float, x: float):
        cf = _arr(coeffs)
        ex = C.c_int32(0)
        r = self._f("eval_plain")(_dp(cf), C.c_uint64(len(cf)), C.c_double(lo), C.c_double(hi),
                                  C.c_double(x), C.byref(ex))
        return r, bool(ex.value)

    def eval_encrypted(self, p: Params, coeffs, lo: float, hi: float, x, lx: int) -> OResult:
        cf = _arr(coeffs)
        x = _arr(x)
        out = np.zeros(p.slot_count)
        lvl = C.c_int32(0)
        m = _Meter()
        rc = self._f("eval_encrypted")(C.byref(p.c()), _dp(cf), C.c_uint64(len(cf)), C.c_double(lo),
                                       C.c_double(hi), _dp(x), C.c_int32(lx), _dp(out), C.byref(lvl),
                                       C.byref(m))
        return OResult(rc, out, (lvl.value,), _mt(m))

    # -- primitives.hpp ---------------------------------------------------
    def newton_refine(self, p: Params, x, lx: int, y0, ly: int, n: int, iters: int,
                      n_valid: int = ALL_SLOTS) -> OResult:
        x, y0 = _arr(x), _arr(y0)
        out = np.zeros(p.slot_count)
        lvl = C.c_int32(0)
        m = _Meter()
        rc = self._f("newton_refine")(C.byref(p.c()), _dp(x), C.c_int32(lx), _dp(y0), C.c_int32(ly),
                                      C.c_int32(n), C.c_int32(iters), C.c_uint64(n_valid), _dp(out),
                                      C.byref(lvl), C.byref(m))
        return OResult(rc, out, (lvl.value,), _mt(m))

    def invroot(self, p: Params, which: int, x, lx: int, S: float, cfg: Optional[Cfg] = None,
                n_valid: int = ALL_SLOTS) -> OResult:
        x = _arr(x)
        out = np.zeros(p.slot_count)
        lvl = C.c_int32(0)
        m = _Meter()
        cc = (cfg or Cfg()).c()
        rc = self._f("invroot")(C.byref(p.c()), C.c_int(which), _dp(x), C.c_int32(lx), C.c_double(S),
                                C.byref(cc), C.c_uint64(n_valid), _dp(out), C.byref(lvl), C.byref(m))
        return OResult(rc, out, (lvl.value,), _mt(m))

    def crypto_sign(self, p: Params, x, lx: int, mode: int = 0, folds: int = 7,
                    polys: Sequence[Sequence[float]] = ()) -> OResult:
        x = _arr(x)
        flat = _arr([v for pl in polys for v in pl]) if polys else _arr([0.0])
        lens = (C.c_uint64 * max(len(polys), 1))(*[len(pl) for pl in polys])
        out = np.zeros(p.slot_count)
        lvl = C.c_int32(0)
        m = _Meter()
        rc = self._f("crypto_sign")(C.byref(p.c()), _dp(x), C.c_int32(lx), C.c_int32(mode),
                                    C.c_int32(folds), _dp(flat), lens, C.c_uint64(len(polys)),
                                    _dp(out), C.byref(lvl), C.byref(m))
        return OResult(rc, out, (lvl.value,), _mt(m))

    # -- column.hpp / stats.hpp -------------------------------------------
    def stat(self, p: Params, which: int, x, B: float, y=None, cfg: Optional[Cfg] = None) -> OResult:
        x = _arr(x)
        y = None if y is None else _arr(y)
        n_out = len(x) if which == ST_ZNORM else (2 * p.slot_count if which == ST_MOMENTS else p.slot_count)
        out = np.zeros(max(n_out, 1))
        lv = (C.c_int32 * 2)()
        m = _Meter()
        cc = (cfg or Cfg()).c()
        rc = self._f("stat")(C.byref(p.c()), C.c_int(which), _dp(x), C.c_uint64(len(x)), _dp(y),
                             C.c_uint64(0 if y is None else len(y)), C.c_double(B), C.byref(cc),
                             _dp(out), lv, C.byref(m))
        return OResult(rc, out[:n_out], (lv[0], lv[1]), _mt(m))

    def znorm_reps(self, p: Params, x, B: float, reps: int):
        x = _arr(x)
        out = np.zeros(len(x))
        m = _Meter()
        rc = self._f("znorm_reps")(C.byref(p.c()), _dp(x), C.c_uint64(len(x)), C.c_double(B),
                                   C.c_int32(reps), _dp(out), C.byref(m))
        return rc, out, _mt(m)

    # -- data.hpp / plain.hpp ---------------------------------------------
    def synthetic_uniform(self, seed: int, n: int, lo: float, hi: float) -> np.ndarray:
        out = np.zeros(n)
        rc = self._f("synthetic_uniform")(C.c_uint64(seed), C.c_uint64(n), C.c_double(lo),
                                          C.c_double(hi), _dp(out))
        assert rc == 0, self.last_error()
        return out

    def synthetic_grid(self, n: int, lo: float, hi: float) -> np.ndarray:
        out = np.zeros(n)
        rc = self._f("synthetic_grid")(C.c_uint64(n), C.c_double(lo), C.c_double(hi), _dp(out))
        assert rc == 0, self.last_error()
        return out

    def two_subrange_grid(self, n: int, lo: float, hi: float) -> np.ndarray:
        out = np.zeros(n)
        rc = self._f("two_subrange_grid")(C.c_uint64(n), C.c_double(lo), C.c_double(hi), _dp(out))
        assert rc == 0, self.last_error()
        return out

    def plain(self, which: int, x, y=None):
        x = _arr(x)
        y = None if y is None else _arr(y)
        out = np.zeros(max(len(x), 1))
        rc = self._f("plain")(C.c_int(which), _dp(x), C.c_uint64(len(x)), _dp(y), _dp(out))
        return rc, (out if which == 6 else out[0])


def _mt(m: _Meter) -> tuple:
    return (m.mul_ct, m.mul_pt, m.add, m.rotate, m.bootstrap)


_cache = {}


def oracle() -> OracleLib:
    """The C restatement (always available once oracle/Makefile ran)."""
    if "ora" not in _cache:
        _cache["ora"] = OracleLib(ORACLE_SO, "ora_")
    return _cache["ora"]


def reference() -> Optional[OracleLib]:
    """The compiled reference, or None where it was not built."""
    if "ref" not in _cache:
        _cache["ref"] = OracleLib(REF_SO, "ref_") if os.path.exists(REF_SO) else None
    return _cache["ref"]


def bits(a: np.ndarray) -> np.ndarray:
    """IEEE bit patterns: bitwise comparisons distinguish -0.0 from +0.0."""
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)
