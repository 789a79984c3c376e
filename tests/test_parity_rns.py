"""GPU: Tier-R kernels (include/hestat_rns.h) limb-for-limb against the CPU RNS
oracle (oracle/rns_oracle.c) on the same seeded keys and ciphertexts.

Bar: bit-exact u64 limbs for every op (NTT, iNTT, key generation, HMult+relin,
rescale, rotate), for several (logN, L, K, dnum) shapes including a digit
count that does not divide L+1, partial top digits at lower levels, batches,
and the full north_star size N=2^16, L=24.
"""
import numpy as np
import pytest

from rns_abi import RnsOracle, Spec

pytestmark = pytest.mark.gpu

O = RnsOracle()

SHAPES = [
    Spec(logN=9, L=3, K=2, dnum=2),
    Spec(logN=10, L=5, K=2, dnum=4, seed=7),      # alpha=2, 3 digits at the top level
    Spec(logN=12, L=7, K=3, dnum=3, seed=11),     # alpha=3: partial last digit
    Spec(logN=13, L=4, K=1, dnum=5, seed=3),      # alpha=1, K=1
    Spec(logN=12, L=5, K=3, dnum=3, seed=8, h=64),  # sparse secret (~64 nonzeros)
    Spec(logN=13, L=6, K=4, dnum=3, seed=9, logp=44),  # 44-bit special primes: FP64 NTT path at its bound
]


def _ctx(s: Spec):
    from paper_2508_12093_b200.rns import RnsContext, RnsSpec
    return RnsContext(RnsSpec(s.logN, s.L, s.K, s.dnum, s.logq0, s.logq, s.logp, seed=s.seed, h=s.h))


def _buf(a):
    from paper_2508_12093_b200.rns import DeviceBuffer
    return DeviceBuffer(a.size).upload(a)


_CTX = {}


def ctx(s: Spec):
    key = (s.logN, s.L, s.K, s.dnum, s.logq0, s.logq, s.logp, s.seed, s.h)
    if key not in _CTX:
        _CTX[key] = _ctx(s)
    return _CTX[key]


@pytest.mark.parametrize("s", SHAPES + [Spec(logN=16, L=24, K=9, dnum=3, seed=1)], ids=str)
def test_primes_and_secret(s):
    c = ctx(s)
    assert np.array_equal(c.primes(), O.primes(s))
    if s.logN <= 13:
        assert np.array_equal(c.secret(), O.secret(s))


@pytest.mark.parametrize("logN,logp", [(9, 61), (10, 61), (11, 61), (12, 61), (13, 61), (14, 61), (15, 61),
                                        (16, 61), (17, 61), (16, 44), (17, 44)])
def test_ntt_matches_oracle(logN, logp):
    s = Spec(logN=logN, L=2, K=1 if logp == 61 else 2, dnum=3, seed=5, logp=logp)
    c = ctx(s)
    primes = O.primes(s)
    rng = np.random.default_rng(logN)
    n = len(primes)
    a = np.stack([rng.integers(0, int(q), s.N, dtype=np.uint64) for q in primes])
    # two batch groups of all primes
    host = np.concatenate([a, a[::-1] % primes[:, None]]).reshape(-1)
    b = _buf(host)
    c.ntt(b, 0, n, batch=2)
    got = b.download().reshape(2, n, s.N)
    for g in range(2):
        src = a if g == 0 else a[::-1] % primes[:, None]
        for i in range(n):
            assert np.array_equal(got[g, i], O.ntt(s, i, src[i])), (g, i)
    c.ntt(b, 0, n, batch=2, inverse=True)
    assert np.array_equal(b.download(), host)
    # inverse of arbitrary (non-NTT) data matches the oracle's iNTT too
    b2 = _buf(a.reshape(-1))
    c.ntt(b2, 0, n, inverse=True)
    got = b2.download().reshape(n, s.N)
    for i in range(n):
        assert np.array_equal(got[i], O.ntt(s, i, a[i], inverse=True))


@pytest.mark.parametrize("logp", [61, 44])
def test_ntt_extreme_values(logp):
    s = Spec(logN=16, L=1, K=1 if logp == 61 else 2, dnum=2, seed=5, logp=logp)
    c = ctx(s)
    primes = O.primes(s)
    for fill in ("zero", "qm1", "one"):
        a = np.stack([np.full(s.N, {"zero": 0, "qm1": int(q) - 1, "one": 1}[fill], dtype=np.uint64) for q in primes])
        b = _buf(a.reshape(-1))
        c.ntt(b, 0, len(primes))
        got = b.download().reshape(len(primes), s.N)
        for i in range(len(primes)):
            assert np.array_equal(got[i], O.ntt(s, i, a[i]))


@pytest.mark.parametrize("s", SHAPES, ids=str)
def test_random_ct(s):
    c = ctx(s)
    for level, tag in ((s.L, 1), (1, 9)):
        assert np.array_equal(c.random_ct(level, tag).download(), O.random_ct(s, level, tag))


@pytest.mark.parametrize("s", SHAPES, ids=str)
def test_mul_relin_matches_oracle(s):
    c = ctx(s)
    for level in sorted({s.L, max(s.L - 2, 0), 0}):
        a, b = O.random_ct(s, level, 21), O.random_ct(s, level, 22)
        got = c.mul_relin(level, _buf(a), _buf(b)).download()
        assert np.array_equal(got, O.mul_relin(s, level, a, b)), level


@pytest.mark.parametrize("s", SHAPES, ids=str)
def test_mul_relin_rescale_matches_oracle(s):
    """HMult + relin + rescale with the rescale merged into ModDown (ModDown by P q_l)."""
    c = ctx(s)
    for level in sorted({s.L, max(s.L // 2, 1), 1}):
        a, b = O.random_ct(s, level, 23), O.random_ct(s, level, 24)
        got = c.mul_relin_rescale(level, _buf(a), _buf(b)).download()
        assert np.array_equal(got, O.mul_relin_rescale(s, level, a, b)), level


def test_mul_relin_rescale_composed_option_matches_oracle():
    """HS_MD_RESCALE=0: mul_relin followed by rescale (two roundings) -- the oracle's composition."""
    import os
    import subprocess
    import sys
    code = r'''
import sys; sys.path[:0] = ["tests", "."]
import numpy as np
from rns_abi import RnsOracle, Spec
from paper_2508_12093_b200.rns import RnsContext, RnsSpec, DeviceBuffer
O = RnsOracle()
for s in (Spec(logN=12, L=5, K=2, dnum=3, seed=9), Spec(logN=13, L=6, K=4, dnum=3, seed=9, logp=44)):
    c = RnsContext(RnsSpec(s.logN, s.L, s.K, s.dnum, s.logq0, s.logq, s.logp, seed=s.seed))
    a, b = O.random_ct(s, s.L, 1), O.random_ct(s, s.L, 2)
    got = c.mul_relin_rescale(s.L, DeviceBuffer(a.size).upload(a), DeviceBuffer(b.size).upload(b)).download()
    assert np.array_equal(got, O.rescale(s, s.L, O.mul_relin(s, s.L, a, b))), s
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, "HS_MD_RESCALE": "0"},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def _const_mul(s, level, a, k):
    """c * a limb by limb (numpy restatement with exact integers)."""
    primes = [int(p) for p in O.primes(s)]
    ct = a.reshape(2, level + 1, s.N)
    out = np.empty_like(ct)
    for i in range(level + 1):
        q = primes[i]
        kr = k % q
        out[:, i, :] = np.array([(int(v) * kr) % q for v in ct[:, i, :].reshape(-1)], dtype=np.uint64).reshape(2, s.N)
    return out.reshape(-1)


@pytest.mark.parametrize("s", SHAPES[:3], ids=str)
@pytest.mark.parametrize("k", [3, -7, (1 << 50) + 12345])
def test_rescale_mul_const_matches_oracle(s, k):
    """rescale(k c) fused (spread multiplies the last limb by k_l, combine computes k_i c_i) equals
    the oracle's rescale of the materialised product, word for word."""
    c = ctx(s)
    level = s.L
    a = O.random_ct(s, level, 41)
    got = c.rescale_mul_const(level, _buf(a), k).download()
    assert np.array_equal(got, O.rescale(s, level, _const_mul(s, level, a, k)))


@pytest.mark.parametrize("s", SHAPES, ids=str)
def test_rescale_matches_oracle(s):
    c = ctx(s)
    for level in sorted({s.L, 1}):
        a = O.random_ct(s, level, 31)
        got = c.rescale(level, _buf(a)).download()
        assert np.array_equal(got, O.rescale(s, level, a)), level


@pytest.mark.parametrize("s", SHAPES[:3], ids=str)
@pytest.mark.parametrize("k", [1, 2, 5, -3, 0])
def test_rotate_matches_oracle(s, k):
    c = ctx(s)
    level = s.L - 1
    a = O.random_ct(s, level, 41)
    got = c.rotate(level, k, _buf(a)).download()
    assert np.array_equal(got, O.rotate(s, level, k, a))


def test_batched_ops_equal_single():
    s = SHAPES[1]
    c = ctx(s)
    level, B = s.L, 3
    a = np.concatenate([O.random_ct(s, level, 50 + i) for i in range(B)])
    b = np.concatenate([O.random_ct(s, level, 60 + i) for i in range(B)])
    W = s.N * 2 * (level + 1)
    da, db = _buf(a), _buf(b)
    m = c.mul_relin(level, da, db, batch=B).download()
    r = c.rescale(level, da, batch=B).download()
    rot = c.rotate(level, 3, da, batch=B).download()
    Wr = s.N * 2 * level
    assert np.array_equal(m, O.mul_relin_many(s, level, a, b, B))
    for i in range(B):
        ai, bi = a[i * W:(i + 1) * W], b[i * W:(i + 1) * W]
        assert np.array_equal(m[i * W:(i + 1) * W], O.mul_relin(s, level, ai, bi))
        assert np.array_equal(r[i * Wr:(i + 1) * Wr], O.rescale(s, level, ai))
        assert np.array_equal(rot[i * W:(i + 1) * W], O.rotate(s, level, 3, ai))


def test_errors():
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200.rns import RnsSpec, RnsContext
    with pytest.raises(H.error):
        RnsContext(RnsSpec(logN=8, L=2, K=1, dnum=1))
    c = ctx(SHAPES[0])
    a = c.random_ct(1, 1)
    with pytest.raises(H.error):
        c.rescale(0, a)
    with pytest.raises((H.error, ValueError)):  # level > L (the buffer check fires first)
        c.mul_relin(SHAPES[0].L + 1, a, a)
    # raw-pointer ops: an undersized device buffer is refused before the call (no OOB access)
    top = c.random_ct(SHAPES[0].L, 2)
    with pytest.raises(ValueError):
        c.mul_relin(SHAPES[0].L, top, a)
    with pytest.raises(ValueError):
        c.rotate(SHAPES[0].L, 1, top, out=a)


def test_full_size_north_star():
    """N=2^16, L=24, K=9, dnum=3 (BASELINE north_star shape): HMult+relin,
    rescale and rotate at the top level, limb-exact vs the oracle."""
    s = Spec(logN=16, L=24, K=9, dnum=3, seed=1)
    c = ctx(s)
    level = s.L
    a, b = O.random_ct(s, level, 1), O.random_ct(s, level, 2)
    da, db = _buf(a), _buf(b)
    assert np.array_equal(c.mul_relin(level, da, db).download(), O.mul_relin(s, level, a, b))
    assert np.array_equal(c.rescale(level, da).download(), O.rescale(s, level, a))
    assert np.array_equal(c.rotate(level, 1, da).download(), O.rotate(s, level, 1, a))


# Base-conversion widths of k_conv_mma (KS = ceil(sources / 4) k-steps): alpha 1..16 sources per
# digit, ModDown with K special primes, 61-bit targets (integer epilogue) and 44-bit ones (FP64
# epilogue), and alpha = 17 (more than 16 sources: the ALU conversion kernel).
CONV_SHAPES = [
    Spec(logN=10, L=15, K=11, dnum=1, seed=21),           # alpha=16: KS=4; ModDown K=11: KS=3
    Spec(logN=10, L=11, K=6, dnum=2, seed=22, logp=44),   # alpha=6: KS=2; K=6: KS=2
    Spec(logN=10, L=9, K=12, dnum=5, seed=23, logp=44),   # alpha=2; ModDown 12 sources: KS=3
    Spec(logN=10, L=16, K=12, dnum=1, seed=24),           # alpha=17: fallback conversion
    Spec(logN=11, L=13, K=5, dnum=2, seed=25),            # alpha=7, 61-bit special targets
]


@pytest.mark.parametrize("s", CONV_SHAPES, ids=str)
def test_conv_widths_mul_relin_and_rotate(s):
    c = ctx(s)
    for level in (s.L, s.L - 1, max(1, s.L // 2)):
        a, b = O.random_ct(s, level, 31 + level), O.random_ct(s, level, 57 + level)
        got = c.mul_relin(level, _buf(a), _buf(b)).download()
        assert np.array_equal(got, O.mul_relin(s, level, a, b)), level
        assert np.array_equal(c.rotate(level, 3, _buf(a)).download(), O.rotate(s, level, 3, a)), level


@pytest.mark.parametrize("mode", ["0", "1"])
def test_alu_conversion_option_matches_oracle(mode):
    """HS_CONV_MMA=0 (the ALU/FP64 base conversion) and =1 (the legacy mma.sync IMMA kernel) give the
    same limbs as the default tcgen05 conversion and the oracle."""
    import os
    import subprocess
    import sys
    code = r'''
import sys; sys.path[:0] = ["tests", "."]
import numpy as np
from rns_abi import RnsOracle, Spec
from paper_2508_12093_b200.rns import RnsContext, RnsSpec, DeviceBuffer
O = RnsOracle()
for s in (Spec(logN=12, L=7, K=3, dnum=3, seed=11), Spec(logN=13, L=6, K=4, dnum=3, seed=9, logp=44),
          Spec(logN=10, L=15, K=11, dnum=1, seed=21), Spec(logN=10, L=9, K=12, dnum=5, seed=23, logp=44)):
    c = RnsContext(RnsSpec(s.logN, s.L, s.K, s.dnum, s.logq0, s.logq, s.logp, seed=s.seed))
    a, b = O.random_ct(s, s.L, 1), O.random_ct(s, s.L, 2)
    got = c.mul_relin(s.L, DeviceBuffer(a.size).upload(a), DeviceBuffer(b.size).upload(b)).download()
    assert np.array_equal(got, O.mul_relin(s, s.L, a, b)), s
    assert np.array_equal(c.rotate(s.L, 3, DeviceBuffer(a.size).upload(a)).download(), O.rotate(s, s.L, 3, a)), s
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, "HS_CONV_MMA": mode},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("mode", ["0", "3"])
def test_key_switch_fusion_options_match_oracle(mode):
    """HS_KS_FUSION=0 (tensor and automorphism materialised) / =3 (both computed inside the key
    switch's passes) give the same limbs as the oracle for HMult and rotations."""
    import os
    import subprocess
    import sys
    code = r'''
import sys; sys.path[:0] = ["tests", "."]
import numpy as np
from rns_abi import RnsOracle, Spec
from paper_2508_12093_b200.rns import RnsContext, RnsSpec, DeviceBuffer
O = RnsOracle()
for s in (Spec(logN=9, L=3, K=2, dnum=2), Spec(logN=12, L=7, K=3, dnum=3, seed=11),
          Spec(logN=13, L=6, K=4, dnum=3, seed=9, logp=44)):
    c = RnsContext(RnsSpec(s.logN, s.L, s.K, s.dnum, s.logq0, s.logq, s.logp, seed=s.seed))
    for level in (s.L, s.L - 1):
        a, b = O.random_ct(s, level, 1), O.random_ct(s, level, 2)
        A, B = DeviceBuffer(a.size).upload(a), DeviceBuffer(b.size).upload(b)
        assert np.array_equal(c.mul_relin(level, A, B).download(), O.mul_relin(s, level, a, b)), s
        for k in (1, -3):
            assert np.array_equal(c.rotate(level, k, A).download(), O.rotate(s, level, k, a)), (s, k)
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root,
                       env={**os.environ, "HS_KS_FUSION": mode},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
