"""CPU: validate the Tier-R RNS oracle (oracle/rns_oracle.c) by the algebraic
identities of RNS-CKKS, checked with exact big-integer CRT in Python:

  * primes are distinct, prime, = 1 mod 2N, of the requested sizes;
  * NTT/iNTT round-trip and the negacyclic convolution theorem (vs schoolbook);
  * HMult+relin: phase(out) = phase(a) * phase(b) + e_ks with |e_ks| small;
  * rescale: q_l * phase(out) - phase(in) is small (rounding term);
  * rotation: phase(out) = sigma_g(phase(in)) + e_ks.
phase(c) = c0 + c1 * s over Q_l, s = the oracle's ternary secret.
"""
import numpy as np
import pytest

from rns_abi import RnsOracle, Spec, crt_centred, galois_elt, galois_src

O = RnsOracle()
SPEC = Spec(logN=9, L=3, K=2, dnum=2)


def _is_prime(n):
    if n < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def test_primes():
    for spec in (SPEC, Spec(logN=16, L=24, K=9, dnum=3)):
        ps = [int(p) for p in O.primes(spec)]
        assert len(set(ps)) == len(ps) == spec.L + 1 + spec.K
        for i, p in enumerate(ps):
            assert _is_prime(p) and p % (2 * spec.N) == 1
            bits = spec.logq0 if i == 0 else (spec.logq if i <= spec.L else spec.logp)
            assert p < (1 << bits) and p > (1 << (bits - 1))


def test_ntt_roundtrip_and_convolution():
    rng = np.random.default_rng(1)
    N = SPEC.N
    for pi, q in enumerate(O.primes(SPEC)):
        q = int(q)
        a = rng.integers(0, q, N, dtype=np.uint64)
        b = rng.integers(0, q, N, dtype=np.uint64)
        fa, fb = O.ntt(SPEC, pi, a), O.ntt(SPEC, pi, b)
        assert np.array_equal(O.ntt(SPEC, pi, fa, inverse=True), a)
        prod = O.ntt(SPEC, pi, np.array([(int(x) * int(y)) % q for x, y in zip(fa, fb)], dtype=np.uint64), True)
        if pi < 2:  # schoolbook negacyclic product (O(N^2) in Python: two primes suffice)
            ai, bi = [int(x) for x in a], [int(x) for x in b]
            ref = [0] * N
            for i in range(N):
                if ai[i] == 0:
                    continue
                for j in range(N):
                    k = i + j
                    if k < N:
                        ref[k] += ai[i] * bi[j]
                    else:
                        ref[k - N] -= ai[i] * bi[j]
            assert [int(x) for x in prod] == [r % q for r in ref]


def _phase(ct, level, sk, primes, N):
    """c0 + c1*s in the NTT domain, per limb -> coefficient form (iNTT)."""
    nl = level + 1
    c = ct.reshape(2, nl, N)
    limbs = []
    for i in range(nl):
        q = int(primes[i])
        v = np.array([(int(c[0, i, n]) + int(c[1, i, n]) * int(sk[i, n])) % q for n in range(N)], dtype=np.uint64)
        limbs.append(O.ntt(SPEC, i, v, inverse=True))
    return limbs


def _ntt_phase(ct, level, sk, primes, N):
    nl = level + 1
    c = ct.reshape(2, nl, N)
    return [[(int(c[0, i, n]) + int(c[1, i, n]) * int(sk[i, n])) % int(primes[i]) for n in range(N)]
            for i in range(nl)]


@pytest.mark.parametrize("level", [3, 1])
def test_mul_relin_identity(level):
    N, primes, sk = SPEC.N, O.primes(SPEC), O.secret(SPEC)
    a, b = O.random_ct(SPEC, level, 1), O.random_ct(SPEC, level, 2)
    out = O.mul_relin(SPEC, level, a, b)
    pa, pb, po = (_ntt_phase(x, level, sk, primes, N) for x in (a, b, out))
    diff = []
    for i in range(level + 1):
        q = int(primes[i])
        d = np.array([(po[i][n] - pa[i][n] * pb[i][n]) % q for n in range(N)], dtype=np.uint64)
        diff.append(O.ntt(SPEC, i, d, inverse=True))
    err = crt_centred(diff, primes[: level + 1])
    assert max(abs(e) for e in err) < 2 ** 30, max(abs(e) for e in err)


def test_sparse_secret_weight_and_identity():
    s = Spec(logN=9, L=3, K=2, dnum=2, seed=4, h=32)
    sk = O.secret(s)
    q0 = int(O.primes(s)[0])
    coeff = O.ntt(s, 0, sk[0], inverse=True)
    nz = [int(v) for v in coeff if v != 0]
    assert 16 <= len(nz) <= 56 and all(v in (1, q0 - 1) for v in nz)
    # HMult+relin still decrypts to the product under the sparse key
    level = 3
    primes = O.primes(s)
    a, b = O.random_ct(s, level, 1), O.random_ct(s, level, 2)
    out = O.mul_relin(s, level, a, b)
    pa, pb, po = (_ntt_phase(x, level, sk, primes, s.N) for x in (a, b, out))
    diff = []
    for i in range(level + 1):
        q = int(primes[i])
        d = np.array([(po[i][n] - pa[i][n] * pb[i][n]) % q for n in range(s.N)], dtype=np.uint64)
        diff.append(O.ntt(s, i, d, inverse=True))
    err = crt_centred(diff, primes[: level + 1])
    assert max(abs(e) for e in err) < 2 ** 30


def test_rescale_identity():
    level = 3
    N, primes, sk = SPEC.N, O.primes(SPEC), O.secret(SPEC)
    a = O.random_ct(SPEC, level, 3)
    out = O.rescale(SPEC, level, a)
    pin = crt_centred(_phase(a, level, sk, primes, N), primes[: level + 1])
    pout = crt_centred(_phase(out, level - 1, sk, primes, N), primes[:level])
    Q = 1
    for p in primes[: level + 1]:
        Q *= int(p)
    ql = int(primes[level])
    worst = 0
    for x, y in zip(pin, pout):
        r = (y * ql - x) % Q
        r = r - Q if r > Q // 2 else r
        worst = max(worst, abs(r))
    assert worst <= ql * (N + 2)


@pytest.mark.parametrize("level", [3, 1])
def test_fused_mul_relin_rescale_identity(level):
    """ModDown by P q_level with the tensor term folded in (rnso_mul_relin_rescale) decrypts to the
    same value as mul_relin followed by rescale, up to the rounding of the two divisions."""
    N, primes, sk = SPEC.N, O.primes(SPEC), O.secret(SPEC)
    a, b = O.random_ct(SPEC, level, 11), O.random_ct(SPEC, level, 12)
    fused = O.mul_relin_rescale(SPEC, level, a, b)
    composed = O.rescale(SPEC, level, O.mul_relin(SPEC, level, a, b))
    assert fused.shape == composed.shape and not np.array_equal(fused, composed)
    pf = crt_centred(_phase(fused, level - 1, sk, primes, N), primes[:level])
    pc = crt_centred(_phase(composed, level - 1, sk, primes, N), primes[:level])
    Q = 1
    for p in primes[:level]:
        Q *= int(p)
    worst = 0
    for x, y in zip(pf, pc):
        r = (x - y) % Q
        r = r - Q if r > Q // 2 else r
        worst = max(worst, abs(r))
    assert worst <= 4 * N, worst


@pytest.mark.parametrize("k", [1, 5, -3])
def test_rotate_identity(k):
    level = 2
    N, primes, sk = SPEC.N, O.primes(SPEC), O.secret(SPEC)
    a = O.random_ct(SPEC, level, 4)
    out = O.rotate(SPEC, level, k, a)
    g = galois_elt(k, SPEC.logN)
    pa, po = _ntt_phase(a, level, sk, primes, N), _ntt_phase(out, level, sk, primes, N)
    # sigma(s) must be applied to phase(in) through sigma of the whole polynomial:
    # phase(out) ~ sigma(c0 + c1 s) -> in the NTT domain index-permuted
    src = [galois_src(n, g, SPEC.logN) for n in range(N)]
    diff = []
    for i in range(level + 1):
        q = int(primes[i])
        d = np.array([(po[i][n] - pa[i][src[n]]) % q for n in range(N)], dtype=np.uint64)
        diff.append(O.ntt(SPEC, i, d, inverse=True))
    err = crt_centred(diff, primes[: level + 1])
    assert max(abs(e) for e in err) < 2 ** 30, max(abs(e) for e in err)


# ---- CKKS codec (host functions of libhestat_gpu.so; no device work) and oracle encryption ----------
def _codec():
    from paper_2508_12093_b200 import rns
    return rns


@pytest.mark.parametrize("logN", [6, 10, 14, 16])
def test_codec_round_trip(logN):
    R = _codec()
    rng = np.random.default_rng(logN)
    S = 1 << (logN - 1)
    z = rng.uniform(-100, 100, S)
    co = R.encode(logN, z, 2.0 ** 40)
    back = R.decode(logN, co, 2.0 ** 40)
    assert np.max(np.abs(back - z)) < 1e-9
    # a constant vector encodes to the constant polynomial
    c = R.encode(logN, np.full(S, 1.5), 2.0 ** 40)
    assert c[0] == round(1.5 * 2 ** 40) and np.max(np.abs(c[1:])) <= 1


def _negacyclic(a, b):
    N = len(a)
    out = [0] * N
    for i, x in enumerate(a):
        if x == 0:
            continue
        for j, y in enumerate(b):
            k = i + j
            if k < N:
                out[k] += x * y
            else:
                out[k - N] -= x * y
    return out


def test_codec_slot_semantics():
    """Polynomial product = slot-wise product; X -> X^(5^k) = left rotation by k (ckks.hpp:193)."""
    R = _codec()
    logN, N = 6, 64
    rng = np.random.default_rng(3)
    z1, z2 = rng.uniform(-1, 1, N // 2), rng.uniform(-1, 1, N // 2)
    s = 2.0 ** 20
    m1, m2 = [int(v) for v in R.encode(logN, z1, s)], [int(v) for v in R.encode(logN, z2, s)]
    prod = np.array(_negacyclic(m1, m2), dtype=np.float64)
    got = R.decode(logN, np.rint(prod / s).astype(np.int64), s)
    assert np.max(np.abs(got - z1 * z2)) < 1e-4
    for k in (1, 3, -2):
        g = galois_elt(k, logN)
        rot = [0] * N
        for i, v in enumerate(m1):
            e = i * g % (2 * N)
            if e < N:
                rot[e] += v
            else:
                rot[e - N] -= v
        out = R.decode(logN, np.array(rot, dtype=np.int64), s)
        assert np.max(np.abs(out - np.roll(z1, -k))) < 1e-5


def test_codec_errors():
    from paper_2508_12093_b200 import hestat as H
    R = _codec()
    with pytest.raises(H.too_many_values):
        R.encode(6, np.zeros(33), 2.0 ** 40)
    with pytest.raises(H.non_finite_value):
        R.encode(6, np.array([1.0, float("nan")]), 2.0 ** 40)


def test_oracle_encrypt_decrypt():
    N = SPEC.N
    rng = np.random.default_rng(9)
    m = rng.integers(-(2 ** 50), 2 ** 50, N)
    for level in (SPEC.L, 0):
        ct = O.encrypt_coeffs(SPEC, level, m, 7)
        d = O.decrypt_coeffs(SPEC, level, ct)
        assert np.max(np.abs(d - m)) <= 21  # centred-binomial error
