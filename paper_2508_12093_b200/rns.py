"""Python mirror of include/hestat_rns.h (Tier-R RNS-CKKS kernels).

Thin ctypes layer: device buffers are `DeviceBuffer`s of u64 words owned by the
library's stream-ordered pool; every op runs on the library stream.  There is
no CPU path: the oracle lives under oracle/ and is used by tests only.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from .hestat import _check


@dataclass
class RnsSpec:
    logN: int = 16
    L: int = 24
    K: int = 9
    dnum: int = 3
    logq0: int = 60
    logq: int = 40
    logp: int = 61
    seed: int = 0
    h: int = 0  # secret Hamming weight: 0 dense ternary, else sparse

    @property
    def N(self) -> int:
        return 1 << self.logN

    def c(self) -> _abi.hs_rns_spec:
        return _abi.hs_rns_spec(self.logN, self.L, self.K, self.dnum, self.logq0, self.logq, self.logp, self.h,
                                self.seed)

    def ct_words(self, level: int) -> int:
        return 2 * (level + 1) * self.N


def encode(logN: int, z, scale: float) -> np.ndarray:
    """CKKS canonical-embedding encoding (host): <= N/2 reals -> N int64 coefficients."""
    z = np.ascontiguousarray(np.asarray(z, dtype=np.float64).reshape(-1))
    out = np.zeros(1 << logN, dtype=np.int64)
    _check(_abi.lib().hs_rns_encode(logN, z.ctypes.data_as(C.POINTER(C.c_double)), z.size, scale,
                                    out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out


def decode(logN: int, coeffs: np.ndarray, scale: float, n: int | None = None) -> np.ndarray:
    co = np.ascontiguousarray(coeffs, dtype=np.int64)
    n = (1 << logN) // 2 if n is None else n
    out = np.zeros(n, dtype=np.float64)
    _check(_abi.lib().hs_rns_decode(logN, co.ctypes.data_as(C.POINTER(C.c_int64)), scale,
                                    out.ctypes.data_as(C.POINTER(C.c_double)), n))
    return out


def encode_gpu(logN: int, z, scale: float) -> np.ndarray:
    """The device codec (what RNS-backed contexts use): N integer-valued float64 coefficients."""
    z = np.ascontiguousarray(np.asarray(z, dtype=np.float64).reshape(-1))
    out = np.zeros(1 << logN, dtype=np.float64)
    _check(_abi.lib().hs_rns_encode_gpu(logN, z.ctypes.data_as(C.POINTER(C.c_double)), z.size, scale,
                                        out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def decode_gpu(logN: int, coeffs: np.ndarray, scale: float, n: int | None = None) -> np.ndarray:
    co = np.ascontiguousarray(coeffs, dtype=np.float64)
    n = (1 << logN) // 2 if n is None else n
    out = np.zeros(n, dtype=np.float64)
    _check(_abi.lib().hs_rns_decode_gpu(logN, co.ctypes.data_as(C.POINTER(C.c_double)), scale,
                                        out.ctypes.data_as(C.POINTER(C.c_double)), n))
    return out


class DeviceBuffer:
    """`words` u64 words of device memory (freed stream-ordered on release)."""

    def __init__(self, words: int):
        p = C.c_void_p()
        _check(_abi.lib().hs_rns_alloc(words, C.byref(p)))
        self.ptr, self.words = p.value, words

    def upload(self, a: np.ndarray) -> "DeviceBuffer":
        a = np.ascontiguousarray(a, dtype=np.uint64)
        if a.size > self.words:
            raise ValueError("upload larger than the buffer")
        _check(_abi.lib().hs_rns_upload(self.ptr, a.ctypes.data_as(_abi.U64P), a.size))
        return self

    def download(self, words: int | None = None) -> np.ndarray:
        n = self.words if words is None else words
        out = np.empty(n, dtype=np.uint64)
        _check(_abi.lib().hs_rns_download(out.ctypes.data_as(_abi.U64P), self.ptr, n))
        return out

    def offset(self, words: int) -> int:
        return self.ptr + 8 * words

    def sub(self, words: int) -> "DeviceBuffer":
        """Non-owning view starting `words` words into this buffer."""
        v = object.__new__(DeviceBuffer)
        v.ptr, v.words, v._owner = self.ptr + 8 * words, self.words - words, self
        return v

    def free(self):
        if getattr(self, "_owner", None) is not None:  # a view owns nothing
            self.ptr = None
            return
        if self.ptr:
            _abi.lib().hs_rns_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _need(buf: "DeviceBuffer", words: int, what: str) -> "DeviceBuffer":
    """The hs_rns_* ops take raw device pointers: check the buffer covers what the op touches."""
    if buf.words < words:
        raise ValueError(f"{what}: device buffer of {buf.words} words, the op needs {words}")
    return buf


class RnsContext:
    """hs_rns: primes, twiddles and (lazily) keys for one parameter set."""

    def __init__(self, spec: RnsSpec):
        self.spec = spec
        h = C.c_void_p()
        _check(_abi.lib().hs_rns_create(C.byref(spec.c()), C.byref(h)))
        self.h = h.value

    def close(self):
        if self.h:
            _abi.lib().hs_rns_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def primes(self) -> np.ndarray:
        n = self.spec.L + 1 + self.spec.K
        out = np.zeros(n, dtype=np.uint64)
        _check(_abi.lib().hs_rns_primes(self.h, out.ctypes.data_as(_abi.U64P), n))
        return out

    def prepare_relin(self):
        _check(_abi.lib().hs_rns_prepare_relin(self.h))

    def prepare_rotation(self, k: int):
        _check(_abi.lib().hs_rns_prepare_rotation(self.h, k))

    def secret(self) -> np.ndarray:
        n = (self.spec.L + 1 + self.spec.K) * self.spec.N
        b = DeviceBuffer(n)
        _check(_abi.lib().hs_rns_secret(self.h, b.ptr))
        return b.download().reshape(self.spec.L + 1 + self.spec.K, self.spec.N)

    def random_ct(self, level: int, tag: int, out: DeviceBuffer | None = None, offset: int = 0) -> DeviceBuffer:
        out = out or DeviceBuffer(self.spec.ct_words(level))
        _need(out, offset + self.spec.ct_words(level), "random_ct out")
        _check(_abi.lib().hs_rns_random_ct(self.h, level, tag, out.offset(offset)))
        return out

    # ---- CKKS encoding / encryption ----
    def encode(self, z, scale: float) -> np.ndarray:
        return encode(self.spec.logN, z, scale)

    def decode(self, coeffs: np.ndarray, scale: float, n: int | None = None) -> np.ndarray:
        return decode(self.spec.logN, coeffs, scale, n)

    def add(self, level: int, a: DeviceBuffer, b: DeviceBuffer, out: DeviceBuffer | None = None,
            batch: int = 1, sub: bool = False) -> DeviceBuffer:
        w = batch * self.spec.ct_words(level)
        out = _need(out or DeviceBuffer(w), w, "add out")
        _need(a, w, "add a"), _need(b, w, "add b")
        f = _abi.lib().hs_rns_sub if sub else _abi.lib().hs_rns_add
        _check(f(self.h, level, a.ptr, b.ptr, out.ptr, batch))
        return out

    def add_const(self, level: int, a: DeviceBuffer, c: int, out: DeviceBuffer | None = None,
                  batch: int = 1) -> DeviceBuffer:
        w = batch * self.spec.ct_words(level)
        out = _need(out or DeviceBuffer(w), w, "add_const out")
        _need(a, w, "add_const a")
        _check(_abi.lib().hs_rns_add_const(self.h, level, a.ptr, int(c), out.ptr, batch))
        return out

    def mul_const(self, level: int, a: DeviceBuffer, c: int, out: DeviceBuffer | None = None,
                  batch: int = 1) -> DeviceBuffer:
        w = batch * self.spec.ct_words(level)
        out = _need(out or DeviceBuffer(w), w, "mul_const out")
        _need(a, w, "mul_const a")
        _check(_abi.lib().hs_rns_mul_const(self.h, level, a.ptr, int(c), out.ptr, batch))
        return out

    def encrypt_coeffs(self, level: int, coeffs: np.ndarray, tag: int, out: DeviceBuffer | None = None) -> DeviceBuffer:
        co = np.ascontiguousarray(coeffs, dtype=np.int64)
        out = _need(out or DeviceBuffer(self.spec.ct_words(level)), self.spec.ct_words(level), "encrypt out")
        if co.size != self.spec.N:
            raise ValueError(f"encrypt_coeffs: {co.size} coefficients, N = {self.spec.N}")
        _check(_abi.lib().hs_rns_encrypt_coeffs(self.h, level, co.ctypes.data_as(C.POINTER(C.c_int64)), tag, out.ptr))
        return out

    def encrypt(self, level: int, z, scale: float, tag: int, out: DeviceBuffer | None = None) -> DeviceBuffer:
        z = np.ascontiguousarray(np.asarray(z, dtype=np.float64).reshape(-1))
        out = _need(out or DeviceBuffer(self.spec.ct_words(level)), self.spec.ct_words(level), "encrypt out")
        _check(_abi.lib().hs_rns_encrypt(self.h, level, z.ctypes.data_as(C.POINTER(C.c_double)), z.size, scale, tag,
                                         out.ptr))
        return out

    def decrypt_coeffs(self, level: int, ct: DeviceBuffer) -> np.ndarray:
        _need(ct, self.spec.ct_words(level), "decrypt ct")
        out = np.zeros(self.spec.N, dtype=np.int64)
        _check(_abi.lib().hs_rns_decrypt_coeffs(self.h, level, ct.ptr, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    def decrypt(self, level: int, ct: DeviceBuffer, scale: float, n: int | None = None) -> np.ndarray:
        n = self.spec.N // 2 if n is None else n
        _need(ct, self.spec.ct_words(level), "decrypt ct")
        out = np.zeros(n, dtype=np.float64)
        _check(_abi.lib().hs_rns_decrypt(self.h, level, ct.ptr, scale, out.ctypes.data_as(C.POINTER(C.c_double)), n))
        return out

    def ntt(self, buf: DeviceBuffer, first_prime: int, nlimbs: int, batch: int = 1, inverse: bool = False):
        _need(buf, batch * nlimbs * self.spec.N, "ntt buffer")
        _check(_abi.lib().hs_rns_ntt(self.h, buf.ptr, first_prime, nlimbs, batch, int(inverse)))

    def mul_relin(self, level: int, a: DeviceBuffer, b: DeviceBuffer, out: DeviceBuffer | None = None,
                  batch: int = 1) -> DeviceBuffer:
        w = batch * self.spec.ct_words(level)
        out = _need(out or DeviceBuffer(w), w, "mul_relin out")
        _need(a, w, "mul_relin a"), _need(b, w, "mul_relin b")
        _check(_abi.lib().hs_rns_mul_relin(self.h, level, a.ptr, b.ptr, out.ptr, batch))
        return out

    def mul_relin_rescale(self, level: int, a: DeviceBuffer, b: DeviceBuffer, out: DeviceBuffer | None = None,
                          batch: int = 1) -> DeviceBuffer:
        w = batch * self.spec.ct_words(level)
        out = _need(out or DeviceBuffer(batch * self.spec.ct_words(level - 1)), batch * self.spec.ct_words(level - 1),
                    "mul_relin_rescale out")
        _need(a, w, "mul_relin_rescale a"), _need(b, w, "mul_relin_rescale b")
        _check(_abi.lib().hs_rns_mul_relin_rescale(self.h, level, a.ptr, b.ptr, out.ptr, batch))
        return out

    def rescale(self, level: int, a: DeviceBuffer, out: DeviceBuffer | None = None, batch: int = 1) -> DeviceBuffer:
        out = _need(out or DeviceBuffer(batch * self.spec.ct_words(level - 1)), batch * self.spec.ct_words(level - 1),
                    "rescale out")
        _need(a, batch * self.spec.ct_words(level), "rescale a")
        _check(_abi.lib().hs_rns_rescale(self.h, level, a.ptr, out.ptr, batch))
        return out

    def rescale_mul_const(self, level: int, a: DeviceBuffer, c: int, out: DeviceBuffer | None = None,
                          batch: int = 1) -> DeviceBuffer:
        """rescale(c * a) without materialising c * a (|c| < 2^53: passed exactly as a double)."""
        out = _need(out or DeviceBuffer(batch * self.spec.ct_words(level - 1)), batch * self.spec.ct_words(level - 1),
                    "rescale_mul_const out")
        _need(a, batch * self.spec.ct_words(level), "rescale_mul_const a")
        _check(_abi.lib().hs_rns_rescale_mul_const(self.h, level, a.ptr, int(c), out.ptr, batch))
        return out

    def rotate(self, level: int, k: int, a: DeviceBuffer, out: DeviceBuffer | None = None,
               batch: int = 1) -> DeviceBuffer:
        w = batch * self.spec.ct_words(level)
        out = _need(out or DeviceBuffer(w), w, "rotate out")
        _need(a, w, "rotate a")
        _check(_abi.lib().hs_rns_rotate(self.h, level, k, a.ptr, out.ptr, batch))
        return out


# ---- the reference's statistics over RNS ciphertexts (hs_rns_eval_*) --------------------------
INVSQRT, MEAN, VARIANCE, MOMENTS, ZNORM, KURTOSIS, SKEWNESS, PEARSON = range(8)


class RnsEval:
    """EvalContext semantics (levels, CostMeter, errors) over Tier-R ciphertexts:
    inputs are encrypted, the reference's DAG runs on RNS kernels, outputs are
    decrypted.  params.slot_count must be N/2 of the RNS context."""

    def __init__(self, ctx: RnsContext, params=None):
        from .hestat import CkksParams
        self.ctx = ctx
        self.params = params or CkksParams(slot_count=ctx.spec.N // 2)
        h = C.c_void_p()
        _check(_abi.lib().hs_rns_eval_create(ctx.h, C.byref(self.params._c()), C.byref(h)))
        self.h = h.value

    def close(self):
        if self.h:
            _abi.lib().hs_rns_eval_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def meter(self):
        from .hestat import CostMeter
        m = _abi.hs_meter()
        _check(_abi.lib().hs_rns_eval_meter(self.h, C.byref(m)))
        return CostMeter(m.mul_ct, m.mul_pt, m.add, m.rotate, m.bootstrap)

    def reset_meter(self):
        _check(_abi.lib().hs_rns_eval_set_meter(self.h, C.byref(_abi.hs_meter())))

    def stat(self, which: int, x, B: float, y=None, cfg=None, out_n: int = 1):
        """Returns (values, levels): values are the first out_n decrypted slots of each
        result (znorm: the n normalised values); levels the results' logical levels."""
        from .hestat import InvRootConfig
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))
        yp, ny = None, 0
        if y is not None:
            y = np.ascontiguousarray(np.asarray(y, dtype=np.float64).reshape(-1))
            yp, ny = y.ctypes.data_as(C.POINTER(C.c_double)), y.size
        nres = 2 if which == MOMENTS else 1
        if which == ZNORM:
            out_n = x.size
        out = np.zeros(out_n * (1 if which == ZNORM else nres), dtype=np.float64)
        levels = np.zeros(max(nres, (x.size + self.params.slot_count - 1) // self.params.slot_count), dtype=np.int32)
        c = (cfg or InvRootConfig())._c()
        _check(_abi.lib().hs_rns_eval_stat(self.h, which, x.ctypes.data_as(C.POINTER(C.c_double)), x.size, yp, ny,
                                           float(B), C.byref(c), out.ctypes.data_as(C.POINTER(C.c_double)), out_n,
                                           levels.ctypes.data_as(C.POINTER(C.c_int32))))
        return out, levels
