"""ctypes harness over the Tier-R RNS oracle (oracle/rns_oracle.c) plus big-int
helpers (CRT, centred lift) to check the RNS-CKKS identities the kernels must
satisfy.  TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from oracle_abi import ORACLE_SO

U64P = C.POINTER(C.c_uint64)


class RnsSpec(C.Structure):
    _fields_ = [("logN", C.c_uint32), ("L", C.c_uint32), ("K", C.c_uint32), ("dnum", C.c_uint32),
                ("logq0", C.c_uint32), ("logq", C.c_uint32), ("logp", C.c_uint32), ("h", C.c_uint32),
                ("seed", C.c_uint64)]


@dataclass
class Spec:
    logN: int = 10
    L: int = 3
    K: int = 2
    dnum: int = 2
    logq0: int = 60
    logq: int = 40
    logp: int = 61
    seed: int = 2025
    h: int = 0

    def c(self) -> RnsSpec:
        return RnsSpec(self.logN, self.L, self.K, self.dnum, self.logq0, self.logq, self.logp, self.h, self.seed)

    @property
    def N(self) -> int:
        return 1 << self.logN


def _u(a: np.ndarray):
    return a.ctypes.data_as(U64P)


class RnsOracle:
    def __init__(self):
        self.lib = C.CDLL(ORACLE_SO)

    def primes(self, s: Spec) -> np.ndarray:
        out = np.zeros(s.L + 1 + s.K, dtype=np.uint64)
        assert self.lib.rnso_primes(C.byref(s.c()), _u(out)) == 0
        return out

    def ntt(self, s: Spec, pi: int, a: np.ndarray, inverse: bool = False) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        (self.lib.rnso_intt if inverse else self.lib.rnso_ntt)(C.byref(s.c()), C.c_uint32(pi), _u(a))
        return a

    def random_ct(self, s: Spec, level: int, tag: int) -> np.ndarray:
        out = np.zeros(2 * (level + 1) * s.N, dtype=np.uint64)
        self.lib.rnso_random_ct(C.byref(s.c()), C.c_uint32(level), C.c_uint64(tag), _u(out))
        return out

    def secret(self, s: Spec) -> np.ndarray:
        out = np.zeros((s.L + 1 + s.K) * s.N, dtype=np.uint64)
        self.lib.rnso_secret(C.byref(s.c()), _u(out))
        return out.reshape(s.L + 1 + s.K, s.N)

    def mul_relin(self, s: Spec, level: int, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        out = np.zeros(2 * (level + 1) * s.N, dtype=np.uint64)
        self.lib.rnso_mul_relin(C.byref(s.c()), C.c_uint32(level), _u(a), _u(b), _u(out))
        return out

    def encrypt_coeffs(self, s: Spec, level: int, coeffs: np.ndarray, tag: int) -> np.ndarray:
        co = np.ascontiguousarray(coeffs, dtype=np.int64)
        out = np.zeros(2 * (level + 1) * s.N, dtype=np.uint64)
        self.lib.rnso_encrypt_coeffs(C.byref(s.c()), C.c_uint32(level), co.ctypes.data_as(C.POINTER(C.c_int64)),
                                     C.c_uint64(tag), _u(out))
        return out

    def decrypt_coeffs(self, s: Spec, level: int, ct: np.ndarray) -> np.ndarray:
        out = np.zeros(s.N, dtype=np.int64)
        self.lib.rnso_decrypt_coeffs(C.byref(s.c()), C.c_uint32(level), _u(np.ascontiguousarray(ct)),
                                     out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out

    def mul_relin_many(self, s: Spec, level: int, a: np.ndarray, b: np.ndarray, count: int) -> np.ndarray:
        out = np.zeros(count * 2 * (level + 1) * s.N, dtype=np.uint64)
        self.lib.rnso_mul_relin_many(C.byref(s.c()), C.c_uint32(level), C.c_uint32(count), _u(a), _u(b), _u(out))
        return out

    def mul_relin_rescale(self, s: Spec, level: int, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        """HMult + relin + rescale with the rescale merged into ModDown (ModDown by P q_level)."""
        out = np.zeros(2 * level * s.N, dtype=np.uint64)
        self.lib.rnso_mul_relin_rescale(C.byref(s.c()), C.c_uint32(level), _u(a), _u(b), _u(out))
        return out

    def rescale(self, s: Spec, level: int, a: np.ndarray) -> np.ndarray:
        out = np.zeros(2 * level * s.N, dtype=np.uint64)
        self.lib.rnso_rescale(C.byref(s.c()), C.c_uint32(level), _u(a), _u(out))
        return out

    def rotate(self, s: Spec, level: int, k: int, a: np.ndarray) -> np.ndarray:
        out = np.zeros(2 * (level + 1) * s.N, dtype=np.uint64)
        self.lib.rnso_rotate(C.byref(s.c()), C.c_uint32(level), C.c_int64(k), _u(a), _u(out))
        return out


# ---- exact big-int helpers ---------------------------------------------------------------
def mulmod_vec(a: np.ndarray, b: np.ndarray, q: int) -> np.ndarray:
    return np.array([(int(x) * int(y)) % q for x, y in zip(a, b)], dtype=np.uint64)


def crt_centred(limbs, primes) -> list:
    """[nl][N] residues -> centred integers mod prod(primes)."""
    Q = 1
    for p in primes:
        Q *= int(p)
    terms = []
    for p in primes:
        p = int(p)
        Qh = Q // p
        terms.append((Qh, pow(Qh % p, -1, p)))
    out = []
    for n in range(len(limbs[0])):
        v = 0
        for (Qh, inv), lim, p in zip(terms, limbs, primes):
            v += (int(lim[n]) * inv % int(p)) * Qh
        v %= Q
        out.append(v - Q if v > Q // 2 else v)
    return out


def galois_src(n: int, g: int, logN: int) -> int:
    def br(x):
        return int(format(x, f"0{logN}b")[::-1], 2)
    e = (2 * br(n) + 1) * g % (2 << logN)
    return br((e - 1) // 2)


def galois_elt(k: int, logN: int) -> int:
    half = 1 << (logN - 1)
    return pow(5, k % half, 2 << logN)
