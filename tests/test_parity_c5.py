"""GPU: config C5 (BASELINE.json configs[4], the primitive sweep) limb-for-limb against the
CPU RNS oracle (oracle/rns_oracle.c): the rotation steps 2^0 .. 2^14 at N = 2^16 (2^15 slots;
every power-of-two step of the reference's rotate-and-sum, ckks.hpp:218-230), and the sweep
shapes N in {2^14, 2^15, 2^16} x L in {8, 16, 24, 32} at a small batch (NTT, iNTT, HMult+relin,
HMult+relin+rescale, rescale, rotate), with the bench's parameter rule (logq0 60, logq 40,
logp 44, K so that P exceeds every digit modulus, dnum 3)."""
import numpy as np
import pytest

from rns_abi import RnsOracle, Spec

pytestmark = pytest.mark.gpu

O = RnsOracle()


def _ctx(s):
    from paper_2508_12093_b200.rns import RnsContext, RnsSpec
    return RnsContext(RnsSpec(s.logN, s.L, s.K, s.dnum, s.logq0, s.logq, s.logp, seed=s.seed, h=s.h))


def _buf(a):
    from paper_2508_12093_b200.rns import DeviceBuffer
    return DeviceBuffer(a.size).upload(a)


def _k(L, dnum=3, logq0=60, logq=40, logp=44):
    alpha = (L + 1 + dnum - 1) // dnum
    return -(-(logq0 + (alpha - 1) * logq + 1) // logp)


def test_rotation_steps_pow2_full_ring():
    """rotate(2^j), j = 0..14, at N = 2^16, two limbs plus a partial digit, against the oracle
    (Galois element 5^(2^j) mod 2^17, its key, the automorphism inside the key switch)."""
    s = Spec(logN=16, L=2, K=_k(2, dnum=2, logp=61), dnum=2, seed=31, logp=61)
    c = _ctx(s)
    a = O.random_ct(s, s.L, 1)
    da = _buf(a)
    for j in range(15):
        got = c.rotate(s.L, 1 << j, da).download()
        assert np.array_equal(got, O.rotate(s, s.L, 1 << j, a)), j


@pytest.mark.parametrize("logN,L", [(14, 8), (14, 16), (14, 32), (15, 8), (15, 16), (15, 32), (16, 8)])
def test_sweep_shape_matches_oracle(logN, L):
    s = Spec(logN=logN, L=L, K=_k(L), dnum=3, seed=40 + L, logp=44)
    c = _ctx(s)
    B = 2
    a = np.concatenate([O.random_ct(s, L, 1 + i) for i in range(B)])
    b = np.concatenate([O.random_ct(s, L, 50 + i) for i in range(B)])
    W = 2 * (L + 1) * s.N
    da, db = _buf(a), _buf(b)
    m = c.mul_relin(L, da, db, batch=B).download()
    mr = c.mul_relin_rescale(L, da, db, batch=B).download()
    r = c.rescale(L, da, batch=B).download()
    rot = c.rotate(L, 1, da, batch=B).download()
    Wr = 2 * L * s.N
    for i in range(B):
        ai, bi = a[i * W:(i + 1) * W], b[i * W:(i + 1) * W]
        assert np.array_equal(m[i * W:(i + 1) * W], O.mul_relin(s, L, ai, bi)), i
        assert np.array_equal(mr[i * Wr:(i + 1) * Wr], O.mul_relin_rescale(s, L, ai, bi)), i
        assert np.array_equal(r[i * Wr:(i + 1) * Wr], O.rescale(s, L, ai)), i
        assert np.array_equal(rot[i * W:(i + 1) * W], O.rotate(s, L, 1, ai)), i
    # NTT / iNTT of every limb of one ciphertext
    x = _buf(a[:W])
    c.ntt(x, 0, L + 1, batch=2, inverse=True)
    primes = O.primes(s)
    got = x.download().reshape(2, L + 1, s.N)
    src = a[:W].reshape(2, L + 1, s.N)
    for p in range(2):
        for i in (0, 1, L):
            assert np.array_equal(got[p, i], O.ntt(s, i, src[p, i], inverse=True)), (p, i)
    c.ntt(x, 0, L + 1, batch=2)
    assert np.array_equal(x.download(), a[:W])
    assert len(primes) == L + 1 + s.K
