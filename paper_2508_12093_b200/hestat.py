"""Python mirror of the reference's ``hestat`` operator surface over the B200 C ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/hestat/{ckks,chebyshev,primitives,column,stats,
plain,data}.hpp) so tests read like the reference's own suites:

    ctx = EvalContext(CkksParams(slot_count=4096))
    col = encode_column(ctx, values)
    z = decode_column(ctx, znorm(ctx, col, 100.0))

Every homomorphic op runs as CUDA kernels in libhestat_gpu.so; ciphertext
slots stay in HBM and are copied back only by ``slots()`` / ``decrypt``.
Exceptions are the reference's taxonomy (errors.hpp:11-38), mapped from the ABI
status codes.  ``ctx.meter()`` returns a snapshot (the reference returns a
mutable reference; use ``ctx.set_meter`` to overwrite).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import hs_column, hs_invroot_cfg, hs_meter, hs_params, hs_sign_cfg

ALL_SLOTS = (1 << 64) - 1  # primitives.hpp:20


# ---- errors.hpp:11-38 ---------------------------------------------------------------
class error(RuntimeError):
    pass


class too_many_values(error): pass
class level_exhausted(error): pass
class length_mismatch(error): pass
class dirty_padding(error): pass
class non_finite_target(error): pass
class domain_violation(error): pass
class divergence(error): pass
class empty_column(error): pass
class degenerate_variance(error): pass
class near_zero_mean(error): pass
class io_error(error): pass
class missing_column(error): pass
class unparsable_cell(error): pass
class non_finite_value(error): pass
class zero_reference(error): pass
class cuda_error(error): pass


_ERRORS = {1: error, 2: too_many_values, 3: level_exhausted, 4: length_mismatch, 5: dirty_padding,
           6: non_finite_target, 7: domain_violation, 8: divergence, 9: empty_column,
           10: degenerate_variance, 11: near_zero_mean, 12: io_error, 13: missing_column,
           14: unparsable_cell, 15: non_finite_value, 16: zero_reference, 100: cuda_error, 101: error}


def _check(rc: int) -> None:
    if rc:
        msg = _abi.lib().hs_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, error)(msg)


def _dp(a: np.ndarray):
    # byref(c_double.from_buffer(a)) costs ~1 us; ndarray.ctypes.data_as ~4.5 us (per call,
    # on the e2e path).  Read-only or empty arrays take the generic route.
    try:
        return C.byref(C.c_double.from_buffer(a))
    except (TypeError, ValueError, BufferError):
        return a.ctypes.data_as(C.POINTER(C.c_double))


def _arr(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))


# ---- ckks.hpp ---------------------------------------------------------------------------------
@dataclass
class CkksParams:  # ckks.hpp:19-42
    slot_count: int = 32768
    max_level: int = 11
    scale_bits: int = 40
    quantize: bool = True
    auto_bootstrap: bool = True
    debug_checks: bool = False

    def _c(self) -> hs_params:
        return hs_params(self.slot_count, self.max_level, self.scale_bits, int(self.quantize),
                         int(self.auto_bootstrap), int(self.debug_checks), 0)

    def validate(self) -> None:
        _check(_abi.lib().hs_params_validate(C.byref(self._c())))

    def quantum(self) -> float:
        return math.ldexp(1.0, -self.scale_bits)


@dataclass
class CostMeter:  # ckks.hpp:46-60
    mul_ct: int = 0
    mul_pt: int = 0
    add: int = 0
    rotate: int = 0
    bootstrap: int = 0

    def merge(self, o: "CostMeter") -> None:
        self.mul_ct += o.mul_ct
        self.mul_pt += o.mul_pt
        self.add += o.add
        self.rotate += o.rotate
        self.bootstrap += o.bootstrap

    def as_tuple(self) -> tuple:
        return (self.mul_ct, self.mul_pt, self.add, self.rotate, self.bootstrap)


class Ciphertext:  # ckks.hpp:64-78
    """Immutable handle: device slot vector + level.  ``Ciphertext(slots, level)``
    builds a host-side ciphertext (no quantisation), uploaded on first use."""

    __slots__ = ("_h",)

    def __init__(self, slots=None, level: int = 0, *, _handle=None):
        if _handle is not None:
            self._h = _handle
            return
        v = _arr([] if slots is None else slots)
        h = C.c_void_p()
        _check(_abi.lib().hs_ct_new(_dp(v), len(v), int(level), C.byref(h)))
        self._h = h

    @classmethod
    def _own(cls, h: C.c_void_p) -> "Ciphertext":
        o = object.__new__(cls)
        o._h = h
        return o

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and h.value and _abi._lib is not None:
                _abi._lib.hs_ct_release(h)
        except Exception:  # interpreter teardown
            pass
        self._h = None

    def slots(self) -> np.ndarray:
        n = self.size()
        out = np.empty(n)
        _check(_abi.lib().hs_ct_read(self._h, _dp(out), n))
        return out

    def level(self) -> int:
        return int(_abi.lib().hs_ct_level(self._h))

    def size(self) -> int:
        return int(_abi.lib().hs_ct_size(self._h))

    def __repr__(self) -> str:
        return f"Ciphertext(size={self.size()}, level={self.level()})"


def _out(fn, *args) -> Ciphertext:
    h = C.c_void_p()
    _check(fn(*args, C.byref(h)))
    return Ciphertext._own(h)


BOOT_REFRESH, BOOT_LOGICAL = 0, 1  # hestat_rns.h HS_RNS_BOOT_*


class EvalContext:  # ckks.hpp:83-257
    """backend=None: the emulator-semantics GPU backend (Tier E; RNS when the process has
    HESTAT_BACKEND=rns); backend="rns": every op on RNS-CKKS ciphertexts (Tier R), with
    `boot` BOOT_REFRESH (secret-key refresh at the reference's bootstraps, chain max_level + 1)
    or BOOT_LOGICAL (deep chain), and `rns_spec` an explicit RnsSpec (rns.py) or None."""

    def __init__(self, params: Optional[CkksParams] = None, rng_seed: int = 0, backend: Optional[str] = None,
                 boot: int = BOOT_REFRESH, rns_spec=None):
        self._p = CkksParams(**vars(params)) if params is not None else CkksParams()
        h = C.c_void_p()
        if backend == "rns":
            sp = C.byref(rns_spec.c()) if rns_spec is not None else None
            _check(_abi.lib().hs_ctx_create_rns(C.byref(self._p._c()), int(rng_seed), sp, int(boot), C.byref(h)))
        elif backend is None:
            _check(_abi.lib().hs_ctx_create(C.byref(self._p._c()), int(rng_seed), C.byref(h)))
        else:
            raise ValueError(f"unknown backend {backend!r}")
        self._h = h

    def rns_backed(self) -> bool:
        return _abi.lib().hs_ctx_backend(self._h) == 1

    def rns_spec(self):
        """(hs_rns_spec, boot mode) of an RNS-backed context."""
        s, b = _abi.hs_rns_spec(), C.c_int()
        _check(_abi.lib().hs_ctx_rns_spec(self._h, C.byref(s), C.byref(b)))
        return s, b.value

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and h.value and _abi._lib is not None:
                _abi._lib.hs_ctx_destroy(h)
        except Exception:  # interpreter teardown
            pass
        self._h = None

    def params(self) -> CkksParams:
        return self._p

    def meter(self) -> CostMeter:
        m = hs_meter()
        _check(_abi.lib().hs_ctx_meter(self._h, C.byref(m)))
        return CostMeter(m.mul_ct, m.mul_pt, m.add, m.rotate, m.bootstrap)

    def set_meter(self, m: CostMeter) -> None:
        _check(_abi.lib().hs_ctx_set_meter(self._h, C.byref(hs_meter(*m.as_tuple()))))

    def rng_seed(self) -> int:
        return int(_abi.lib().hs_ctx_rng_seed(self._h))

    def encrypt(self, values) -> Ciphertext:  # ckks.hpp:97-104
        v = _arr(values)
        return _out(_abi.lib().hs_encrypt, self._h, _dp(v), len(v))

    def decrypt(self, ct: Ciphertext, n: int) -> np.ndarray:  # ckks.hpp:107-111
        out = np.empty(max(int(n), 0))
        _check(_abi.lib().hs_decrypt(self._h, ct._h, int(n), _dp(out)))
        return out

    def add_ct(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        return _out(_abi.lib().hs_add_ct, self._h, a._h, b._h)

    def sub_ct(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        return _out(_abi.lib().hs_sub_ct, self._h, a._h, b._h)

    def add_pt(self, a: Ciphertext, c: float) -> Ciphertext:
        return _out(_abi.lib().hs_add_pt, self._h, a._h, float(c))

    def mul_ct(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        return _out(_abi.lib().hs_mul_ct, self._h, a._h, b._h)

    def mul_pt(self, a: Ciphertext, c) -> Ciphertext:
        if np.ndim(c) == 0:
            return _out(_abi.lib().hs_mul_pt, self._h, a._h, float(c))
        v = _arr(c)
        return _out(_abi.lib().hs_mul_pt_vec, self._h, a._h, _dp(v), len(v))

    def rotate(self, a: Ciphertext, k: int) -> Ciphertext:
        return _out(_abi.lib().hs_rotate, self._h, a._h, int(k))

    def bootstrap(self, a: Ciphertext) -> Ciphertext:
        return _out(_abi.lib().hs_bootstrap, self._h, a._h)

    def sum_all_slots(self, a: Ciphertext, n_valid: int) -> Ciphertext:
        return _out(_abi.lib().hs_sum_all_slots, self._h, a._h, int(n_valid))

    # ---- batched forms (C5): the single op's semantics per element, one launch per 64 ----
    def _batch(self, fn, a, *rest):
        n = len(a)
        arr = (C.c_void_p * max(n, 1))(*[x._h.value for x in a])
        outs = (C.c_void_p * max(n, 1))()
        if rest and isinstance(rest[0], (list, tuple)):
            b = rest[0]
            if len(b) != n:
                raise length_mismatch("batch: operand counts differ")
            barr = (C.c_void_p * max(n, 1))(*[x._h.value for x in b])
            _check(fn(self._h, arr, barr, n, outs))
        else:
            _check(fn(self._h, arr, *rest, n, outs))
        return [Ciphertext._own(C.c_void_p(outs[i])) for i in range(n)]

    def add_ct_batch(self, a, b):
        return self._batch(_abi.lib().hs_add_ct_batch, a, list(b))

    def sub_ct_batch(self, a, b):
        return self._batch(_abi.lib().hs_sub_ct_batch, a, list(b))

    def mul_ct_batch(self, a, b):
        return self._batch(_abi.lib().hs_mul_ct_batch, a, list(b))

    def add_pt_batch(self, a, c: float):
        return self._batch(_abi.lib().hs_add_pt_batch, a, float(c))

    def mul_pt_batch(self, a, c: float):
        return self._batch(_abi.lib().hs_mul_pt_batch, a, float(c))

    def rotate_batch(self, a, k: int):
        return self._batch(_abi.lib().hs_rotate_batch, a, int(k))


# ---- chebyshev.hpp ------------------------------------------------------------------------------
@dataclass
class ChebyshevSeries:  # chebyshev.hpp:24-31
    coeffs: List[float] = field(default_factory=list)
    domain_lo: float = -1.0
    domain_hi: float = 1.0

    def degree(self) -> int:
        return len(self.coeffs) - 1

    def native_domain(self) -> bool:
        return self.domain_lo == -1.0 and self.domain_hi == 1.0


class ScaledTargetKind(enum.IntEnum):  # chebyshev.hpp:37
    InvSqrtShifted = 0
    SqrtShifted = 1


def scaled_target(kind: ScaledTargetKind, S: float, t: float) -> float:
    return float(_abi.lib().hs_scaled_target(int(kind), float(S), float(t)))


def cheb_eval_depth(degree: int) -> int:
    return int(_abi.lib().hs_cheb_eval_depth(int(degree)))


def fit(target: Callable[[float], float], degree: int, domain_lo: float = -1.0,
        domain_hi: float = 1.0) -> ChebyshevSeries:  # chebyshev.hpp:59-85 (host)
    out = np.zeros(max(int(degree) + 1, 1))
    err = []

    def cb(x, _u):
        try:
            return float(target(x))
        except Exception as e:  # surfaced after the call
            err.append(e)
            return float("nan")

    fn = _abi.TARGET_FN(cb)
    rc = _abi.lib().hs_fit(fn, None, int(degree), float(domain_lo), float(domain_hi), _dp(out))
    if err:
        raise err[0]
    _check(rc)
    return ChebyshevSeries(list(out[: int(degree) + 1]), float(domain_lo), float(domain_hi))


def fit_scaled(kind: ScaledTargetKind, S: float, degree: int) -> ChebyshevSeries:
    """fit() of a ScaledTarget on [-1, 1] without a Python callback (cached on the host)."""
    out = np.zeros(max(int(degree) + 1, 1))
    _check(_abi.lib().hs_fit_target(int(kind), float(S), int(degree), -1.0, 1.0, _dp(out)))
    return ChebyshevSeries(list(out[: int(degree) + 1]))


def eval_plain(s: ChebyshevSeries, x: float, extrapolated: Optional[list] = None) -> float:
    """Clenshaw (chebyshev.hpp:90-105).  Pass a list to receive the extrapolation flag."""
    cf = _arr(s.coeffs)
    ex = C.c_int32(0)
    r = _abi.lib().hs_eval_plain(_dp(cf), len(cf), float(s.domain_lo), float(s.domain_hi), float(x), C.byref(ex))
    if extrapolated is not None:
        extrapolated[:] = [bool(ex.value)]
    return float(r)


def eval_encrypted(ctx: EvalContext, s: ChebyshevSeries, ct: Ciphertext) -> Ciphertext:  # :171-189
    cf = _arr(s.coeffs)
    return _out(_abi.lib().hs_eval_encrypted, ctx._h, _dp(cf), len(cf), float(s.domain_lo),
                float(s.domain_hi), ct._h)


# ---- primitives.hpp ---------------------------------------------------------------------------------
@dataclass
class InvRootConfig:  # primitives.hpp:23-40
    n: int = 2
    cheb_degree: int = 511
    newton_iters: int = 6
    baseline_mode: bool = False
    baseline_iters: int = 0

    def effective_baseline_iters(self) -> int:
        if self.baseline_iters > 0:
            return self.baseline_iters
        return 25 if self.n == 1 else 21

    def validate(self) -> None:
        if self.n not in (1, 2):
            raise error("InvRootConfig: n must be 1 or 2")
        if self.newton_iters < 0:
            raise error("InvRootConfig: newton_iters < 0")
        if self.cheb_degree < 0:
            raise error("InvRootConfig: cheb_degree < 0")

    def _c(self) -> hs_invroot_cfg:
        return hs_invroot_cfg(self.n, self.cheb_degree, self.newton_iters, int(self.baseline_mode),
                              self.baseline_iters, 0)


class SignMode(enum.IntEnum):
    G3Composition = 0
    CustomComposite = 1


@dataclass
class SignConfig:  # primitives.hpp:59-70
    mode: SignMode = SignMode.G3Composition
    folds: int = 7
    custom_polys: List[List[float]] = field(default_factory=list)

    def mode_name(self) -> str:
        return "g3_composition" if self.mode == SignMode.G3Composition else "custom_composite"

    def _c(self):
        flat = _arr([v for p in self.custom_polys for v in p] or [0.0])
        lens = (C.c_uint64 * max(len(self.custom_polys), 1))(*[len(p) for p in self.custom_polys])
        cfg = hs_sign_cfg(int(self.mode), int(self.folds), flat.ctypes.data_as(C.POINTER(C.c_double)), lens,
                          len(self.custom_polys))
        return cfg, (flat, lens)  # keep buffers alive


_DEFAULT_CFG = None


def _cfg(cfg: Optional[InvRootConfig]):
    global _DEFAULT_CFG
    if cfg is None:
        if _DEFAULT_CFG is None:
            _DEFAULT_CFG = InvRootConfig()._c()
        return C.byref(_DEFAULT_CFG)
    return C.byref(cfg._c())


class detail:
    @staticmethod
    def newton_loop(ctx: EvalContext, x_op: Ciphertext, y: Ciphertext, n: int, iters: int,
                    n_valid: int = ALL_SLOTS) -> Ciphertext:  # primitives.hpp:105-132
        return _out(_abi.lib().hs_newton_loop, ctx._h, x_op._h, y._h, int(n), int(iters), int(n_valid))


def newton_refine(ctx: EvalContext, ct_x: Ciphertext, ct_y0: Ciphertext, n: int, iters: int,
                  n_valid: int = ALL_SLOTS) -> Ciphertext:  # primitives.hpp:152-158
    return _out(_abi.lib().hs_newton_refine, ctx._h, ct_x._h, ct_y0._h, int(n), int(iters), int(n_valid))


def crypto_invsqrt(ctx: EvalContext, ct: Ciphertext, S: float, cfg: Optional[InvRootConfig] = None,
                   n_valid: int = ALL_SLOTS) -> Ciphertext:  # primitives.hpp:186-208
    return _out(_abi.lib().hs_crypto_invsqrt, ctx._h, ct._h, float(S), _cfg(cfg), int(n_valid))


def baseline_invsqrt(ctx: EvalContext, ct: Ciphertext, S: float, iters: int = 21,
                     n_valid: int = ALL_SLOTS) -> Ciphertext:  # primitives.hpp:173-184
    return _out(_abi.lib().hs_baseline_invsqrt, ctx._h, ct._h, float(S), int(iters), int(n_valid))


def crypto_inv(ctx: EvalContext, ct: Ciphertext, S: float, cfg: Optional[InvRootConfig] = None,
               n_valid: int = ALL_SLOTS) -> Ciphertext:  # primitives.hpp:211-217
    return _out(_abi.lib().hs_crypto_inv, ctx._h, ct._h, float(S), _cfg(cfg), int(n_valid))


def crypto_sqrt(ctx: EvalContext, ct: Ciphertext, S: float, degree: int = 511,
                n_valid: int = ALL_SLOTS) -> Ciphertext:  # primitives.hpp:222-238
    return _out(_abi.lib().hs_crypto_sqrt, ctx._h, ct._h, float(S), int(degree), int(n_valid))


def crypto_sign(ctx: EvalContext, ct: Ciphertext, cfg: Optional[SignConfig] = None) -> Ciphertext:  # :279-300
    c, keep = (cfg or SignConfig())._c()
    r = _out(_abi.lib().hs_crypto_sign, ctx._h, ct._h, C.byref(c))
    del keep
    return r


# ---- column.hpp ------------------------------------------------------------------------------------
@dataclass
class EncryptedColumn:  # column.hpp:19-23
    chunks: List[Ciphertext] = field(default_factory=list)
    n_valid: int = 0
    name: str = ""

    def _c(self):
        # the ctypes view is cached while the chunk list and n_valid are unchanged (columns made
        # by encode_column / znorm are born with it: the handle array the C call filled)
        key = (tuple(map(id, self.chunks)), int(self.n_valid))
        cache = self.__dict__.get("_cview")
        if cache is not None and cache[0] == key:
            return cache[1], cache[2]
        arr = _ptr_array(len(self.chunks))(*[c._h.value for c in self.chunks])
        col = hs_column(arr, len(self.chunks), int(self.n_valid))
        self.__dict__["_cview"] = (key, col, arr)
        return col, arr

    @classmethod
    def _from_handles(cls, arr, n: int, n_valid: int, name: str) -> "EncryptedColumn":
        """Wrap n handles a C call wrote into arr (owned from here on), view cached."""
        own = Ciphertext._own
        chunks = [own(C.c_void_p(arr[i])) for i in range(n)]
        col = cls(chunks, n_valid, name)
        col.__dict__["_cview"] = ((tuple(map(id, chunks)), int(n_valid)), hs_column(arr, n, int(n_valid)), arr)
        return col


_PTR_ARRAYS = {}


def _ptr_array(n: int):
    """ctypes array type c_void_p * max(n, 1), cached."""
    t = _PTR_ARRAYS.get(n)
    if t is None:
        t = _PTR_ARRAYS[n] = C.c_void_p * max(n, 1)
    return t


def encode_column(ctx: EvalContext, values, name: str = "") -> EncryptedColumn:  # column.hpp:25-39
    v = values if (isinstance(values, np.ndarray) and values.dtype == np.float64 and values.ndim == 1
                   and values.flags.c_contiguous) else _arr(values)
    S = ctx._p.slot_count
    nch = (len(v) + S - 1) // S
    arr = _ptr_array(nch)()
    got = C.c_uint64(0)
    _check(_abi.lib().hs_encode_column(ctx._h, _dp(v), len(v), arr, C.byref(got)))
    return EncryptedColumn._from_handles(arr, got.value, len(v), name)


def decode_column(ctx: EvalContext, col: EncryptedColumn, out: Optional[np.ndarray] = None) -> np.ndarray:
    """column.hpp:41-56.  Pass a (pinned) float64 `out` of n_valid elements to
    receive the slots by direct DMA."""
    c, keep = col._c()
    if out is None:
        out = np.empty(max(int(col.n_valid), 0))
    elif out.dtype != np.float64 or not out.flags.c_contiguous or out.size < col.n_valid:
        raise length_mismatch("decode_column: out must be a contiguous float64 array of n_valid elements")
    _check(_abi.lib().hs_decode_column(ctx._h, C.byref(c), _dp(out) if len(out) else None))
    del keep
    return out


class Pending:
    """An asynchronous transfer in flight (hs_pending).  ``wait()`` blocks until it has completed
    and raises the call's deferred error (non_finite_value for an encode whose input held a NaN or
    infinity).  The host buffer handed to the call must not be touched until then."""

    __slots__ = ("_h", "_keep")

    def __init__(self, h: C.c_void_p, keep=None):
        self._h = h
        self._keep = keep  # host arrays and ctypes views the transfer still uses

    def wait(self) -> None:
        _check(_abi.lib().hs_pending_wait(self._h))
        self._keep = None

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and h.value and _abi._lib is not None:
                _abi._lib.hs_pending_release(h)
        except Exception:  # interpreter teardown
            pass
        self._h = None


def encode_column_async(ctx: EvalContext, values, name: str = ""):
    """encode_column without the wait: returns (column, Pending).  The column can be passed to
    any op at once (the library orders its streams behind the upload); ``Pending.wait()`` delivers
    the finiteness verdict.  ``values`` (pinned for a DMA at PCIe rate) must stay untouched until
    then."""
    v = values if (isinstance(values, np.ndarray) and values.dtype == np.float64 and values.ndim == 1
                   and values.flags.c_contiguous) else _arr(values)
    S = ctx._p.slot_count
    nch = (len(v) + S - 1) // S
    arr = _ptr_array(nch)()
    got = C.c_uint64(0)
    h = C.c_void_p()
    _check(_abi.lib().hs_encode_column_async(ctx._h, _dp(v), len(v), arr, C.byref(got), C.byref(h)))
    return EncryptedColumn._from_handles(arr, got.value, len(v), name), Pending(h, v)


def decode_column_async(ctx: EvalContext, col: EncryptedColumn, out: np.ndarray) -> Pending:
    """decode_column without the wait: ``out`` (a contiguous float64 array of n_valid elements,
    pinned for direct DMA) holds the slots once ``Pending.wait()`` returns."""
    if out.dtype != np.float64 or not out.flags.c_contiguous or out.size < col.n_valid:
        raise length_mismatch("decode_column: out must be a contiguous float64 array of n_valid elements")
    c, keep = col._c()
    h = C.c_void_p()
    _check(_abi.lib().hs_decode_column_async(ctx._h, C.byref(c), _dp(out) if len(out) else None, C.byref(h)))
    return Pending(h, (out, col, keep))


# ---- stats.hpp ------------------------------------------------------------------------------------
@dataclass
class MomentSet:  # stats.hpp:18-22
    ct_mu: Ciphertext
    ct_var: Ciphertext
    n_valid: int = 0


def _col_call(fn, ctx: EvalContext, col: EncryptedColumn, *args) -> Ciphertext:
    c, keep = col._c()
    r = _out(fn, ctx._h, C.byref(c), *args)
    del keep
    return r


def mean_scaled(ctx: EvalContext, col: EncryptedColumn, B: float) -> Ciphertext:  # :97-103
    return _col_call(_abi.lib().hs_mean_scaled, ctx, col, float(B))


def variance_to_scale(ctx: EvalContext, col: EncryptedColumn, S: float) -> Ciphertext:  # :110-126
    return _col_call(_abi.lib().hs_variance_to_scale, ctx, col, float(S))


def variance_scaled(ctx: EvalContext, col: EncryptedColumn, B: float) -> Ciphertext:  # :130-134
    return _col_call(_abi.lib().hs_variance_scaled, ctx, col, float(B))


def moments(ctx: EvalContext, col: EncryptedColumn, B: float) -> MomentSet:  # :138-148
    c, keep = col._c()
    mu, var = C.c_void_p(), C.c_void_p()
    _check(_abi.lib().hs_moments(ctx._h, C.byref(c), float(B), C.byref(mu), C.byref(var)))
    del keep
    return MomentSet(Ciphertext._own(mu), Ciphertext._own(var), col.n_valid)


def znorm(ctx: EvalContext, col: EncryptedColumn, B: float,
          cfg: Optional[InvRootConfig] = None) -> EncryptedColumn:  # :153-166
    c, keep = col._c()
    n = len(col.chunks)
    arr = _ptr_array(n)()
    _check(_abi.lib().hs_znorm(ctx._h, C.byref(c), float(B), _cfg(cfg), arr))
    del keep
    return EncryptedColumn._from_handles(arr, n, col.n_valid, col.name)


def kurtosis(ctx: EvalContext, col: EncryptedColumn, B: float,
             cfg: Optional[InvRootConfig] = None) -> Ciphertext:  # :170-188
    return _col_call(_abi.lib().hs_kurtosis, ctx, col, float(B), _cfg(cfg))


def skewness(ctx: EvalContext, col: EncryptedColumn, B: float,
             cfg: Optional[InvRootConfig] = None) -> Ciphertext:  # :192-210
    return _col_call(_abi.lib().hs_skewness, ctx, col, float(B), _cfg(cfg))


def coeff_variation(ctx: EvalContext, col: EncryptedColumn, B: float, sign_cfg: Optional[SignConfig] = None,
                    cfg: Optional[InvRootConfig] = None) -> Ciphertext:  # :216-233
    sc, keep2 = (sign_cfg or SignConfig())._c()
    r = _col_call(_abi.lib().hs_coeff_variation, ctx, col, float(B), C.byref(sc), _cfg(cfg))
    del keep2
    return r


def pearson(ctx: EvalContext, col_x: EncryptedColumn, col_y: EncryptedColumn, B: float,
            cfg: Optional[InvRootConfig] = None) -> Ciphertext:  # :239-265
    cx, k1 = col_x._c()
    cy, k2 = col_y._c()
    r = _out(_abi.lib().hs_pearson, ctx._h, C.byref(cx), C.byref(cy), float(B), _cfg(cfg))
    del k1, k2
    return r


def znorm_batch(ctx: EvalContext, cols: Sequence[EncryptedColumn], B: float,
                cfg: Optional[InvRootConfig] = None) -> List[EncryptedColumn]:
    """znorm(col) for every column, in order (hs_znorm_batch: one launch per 64 single-chunk
    columns; same slots, levels and meter as the calls)."""
    cs, keep = [], []
    for col in cols:
        c, k = col._c()
        cs.append(c)
        keep.append(k)
    arr = (C.POINTER(_abi.hs_column) * max(len(cs), 1))(*[C.pointer(c) for c in cs])
    total = sum(len(c.chunks) for c in cols)
    out = _ptr_array(max(total, 1))()
    _check(_abi.lib().hs_znorm_batch(ctx._h, arr, len(cs), float(B), _cfg(cfg), out))
    del keep
    res, off = [], 0
    for col in cols:
        n = len(col.chunks)
        chunks = [Ciphertext._own(C.c_void_p(out[off + i])) for i in range(n)]
        res.append(EncryptedColumn(chunks, col.n_valid, col.name))
        off += n
    return res


def pearson_table(ctx: EvalContext, cols: Sequence[EncryptedColumn], B: float,
                  cfg: Optional[InvRootConfig] = None) -> List[Ciphertext]:
    """pearson(cols[i], cols[j]) for every pair i < j, in that order (hs_pearson_table: one
    launch for up to 8 single-chunk columns; same slots, levels and meter as the calls)."""
    cs, keep = [], []
    for col in cols:
        c, k = col._c()
        cs.append(c)
        keep.append(k)
    arr = (C.POINTER(_abi.hs_column) * max(len(cs), 1))(*[C.pointer(c) for c in cs])
    npairs = len(cs) * (len(cs) - 1) // 2
    hs = (C.c_void_p * max(npairs, 1))()
    _check(_abi.lib().hs_pearson_table(ctx._h, arr, len(cs), float(B), _cfg(cfg),
                                       C.cast(hs, C.POINTER(C.c_void_p))))
    del keep
    return [Ciphertext._own(C.c_void_p(hs[k])) for k in range(npairs)]


# ---- data.hpp / plain.hpp (host) --------------------------------------------------------------------
def synthetic_uniform(seed: int, n: int, lo: float, hi: float) -> np.ndarray:  # data.hpp:148-160
    out = np.empty(max(int(n), 1))
    _check(_abi.lib().hs_synthetic_uniform(int(seed), int(n), float(lo), float(hi), _dp(out)))
    return out[: int(n)]


def synthetic_grid(n: int, lo: float, hi: float) -> np.ndarray:  # data.hpp:163-173
    out = np.empty(max(int(n), 1))
    _check(_abi.lib().hs_synthetic_grid(int(n), float(lo), float(hi), _dp(out)))
    return out[: int(n)]


def two_subrange_grid(n: int, lo: float, hi: float) -> np.ndarray:  # data.hpp:178-186
    out = np.empty(max(int(n), 1))
    _check(_abi.lib().hs_two_subrange_grid(int(n), float(lo), float(hi), _dp(out)))
    return out[: int(n)]


def mre(approx, exact) -> float:  # data.hpp:190-203
    a, e = _arr(approx), _arr(exact)
    if len(a) != len(e):
        raise length_mismatch("mre: length mismatch")
    r = C.c_double(0.0)
    _check(_abi.lib().hs_mre(_dp(a), _dp(e), len(a), C.byref(r)))
    return r.value


def relative_error(approx: float, exact: float) -> float:  # data.hpp:205-208
    r = C.c_double(0.0)
    _check(_abi.lib().hs_relative_error(float(approx), float(exact), C.byref(r)))
    return r.value


class plain:  # plain.hpp:16-92
    @staticmethod
    def _one(which: int, x, y=None) -> float:
        xv = _arr(x)
        yv = None if y is None else _arr(y)
        if yv is not None and len(yv) != len(xv):
            raise length_mismatch("plain::pearson: length mismatch")
        out = np.zeros(1)
        _check(_abi.lib().hs_plain(which, _dp(xv), len(xv), None if yv is None else _dp(yv), _dp(out)))
        return float(out[0])

    mean = staticmethod(lambda x: plain._one(0, x))
    variance = staticmethod(lambda x: plain._one(1, x))
    skewness = staticmethod(lambda x: plain._one(2, x))
    kurtosis_ratio = staticmethod(lambda x: plain._one(3, x))
    coeff_variation = staticmethod(lambda x: plain._one(4, x))
    pearson = staticmethod(lambda x, y: plain._one(5, x, y))
    stddev = staticmethod(lambda x: plain._one(7, x))

    @staticmethod
    def znorm(x) -> np.ndarray:
        xv = _arr(x)
        out = np.zeros(max(len(xv), 1))
        _check(_abi.lib().hs_plain(6, _dp(xv), len(xv), None, _dp(out)))
        return out[: len(xv)]


# ---- runtime ------------------------------------------------------------------------------------------
def init(device: int = -1) -> None:
    _check(_abi.lib().hs_init(int(device)))


def sync() -> None:
    _check(_abi.lib().hs_sync())


def stream_handle() -> int:
    return int(_abi.lib().hs_stream() or 0)


def set_fused(enabled: bool) -> None:
    _check(_abi.lib().hs_set_fused(int(bool(enabled))))


def kernel_launches() -> int:
    return int(_abi.lib().hs_kernel_launches())


class Graph:
    """CUDA graph of captured library calls (``with Graph() as g: ...; g.launch()``).

    Capture only warm calls (same shapes already executed once) and release the
    captured calls' outputs inside the ``with`` block."""

    def __init__(self):
        self._h = None

    def __enter__(self):
        _check(_abi.lib().hs_graph_begin())
        return self

    def __exit__(self, et, ev, tb):
        h = C.c_void_p()
        rc = _abi.lib().hs_graph_end(C.byref(h))
        if et is None:
            _check(rc)
            self._h = h
        return False

    def launch(self) -> None:
        _check(_abi.lib().hs_graph_launch(self._h))

    def __del__(self):
        try:
            if self._h is not None and self._h.value and _abi._lib is not None:
                _abi._lib.hs_graph_destroy(self._h)
        except Exception:
            pass
        self._h = None
