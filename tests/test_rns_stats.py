"""GPU: the reference's statistics evaluated on real RNS-CKKS ciphertexts
(hs_rns_eval_*, RnsB backend of flow.h) against the reference's decrypted
outputs (the compiled oracle), at north_star's tolerance:

  * decrypted statistics within 1e-6 relative of the reference's outputs;
  * identical CostMeter counts and logical levels (the DAG is the reference's);
  * bootstrap() is a logical reset over a deep modulus chain; a chain shorter than
    the statistic's depth fails with level_exhausted.
"""
import numpy as np
import pytest

from oracle_abi import (Cfg, Params, ST_KURT, ST_MEAN, ST_MOMENTS, ST_PEARSON, ST_SKEW, ST_VAR, ST_ZNORM, oracle)

pytestmark = pytest.mark.gpu

TOL = 1e-6
_CTX = {}


def _rns(logN, L, seed=3):
    from paper_2508_12093_b200.rns import RnsContext, RnsSpec
    key = (logN, L, seed)
    if key not in _CTX:
        # 60-bit rescaling primes (scale 2^60) and a sparse secret (h = 192): the
        # reference's DAG amplifies per-op noise (cancellation in the variance, degree-511
        # BSGS), so 1e-6 relative needs ~1e-14 absolute CKKS noise; 61-bit q_0 / special
        # primes, K = alpha + 1
        _CTX[key] = RnsContext(RnsSpec(logN=logN, L=L, K=(L + 1 + 2) // 3 + 1, dnum=3, logq0=61, logq=60, logp=61,
                                       seed=seed, h=192))
    return _CTX[key]


def _eval(logN, L, **kw):
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200.rns import RnsEval
    return RnsEval(_rns(logN, L), H.CkksParams(slot_count=1 << (logN - 1), **kw))


def _normal(seed, n, mu, sd):
    rng = np.random.default_rng(seed)
    return mu + sd * rng.standard_normal(n)


def _check_scalar(got, ref):
    assert abs(got - ref) <= TOL * abs(ref), (got, ref, abs(got - ref) / abs(ref))


def _check_vector(got, ref):
    err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
    assert err <= TOL, err


def _meter(e):
    m = e.meter()
    return (m.mul_ct, m.mul_pt, m.add, m.rotate, m.bootstrap)


LOGN, L = 13, 28          # S = 4096 (the C1 shape); chain deeper than every statistic's depth (26) + 1
S = 1 << (LOGN - 1)


@pytest.mark.parametrize("deg,iters", [(15, 2), (511, 6)])
def test_invsqrt_c1(deg, iters):
    from paper_2508_12093_b200 import rns as R
    from paper_2508_12093_b200.hestat import InvRootConfig
    t = np.random.default_rng(1).uniform(0.01, 1.0, S)
    e = _eval(LOGN, L)
    out, lv = e.stat(R.INVSQRT, t, 1.0, cfg=InvRootConfig(cheb_degree=deg, newton_iters=iters), out_n=S)
    ref = oracle().invroot(Params(slot_count=S), 0, t, 11, 1.0, Cfg(cheb_degree=deg, newton_iters=iters))
    assert ref.rc == 0
    _check_vector(out, ref.out)
    assert _meter(e) == ref.meter and lv[0] == ref.levels[0]
    if deg == 511:  # the approximation itself (15/2 is coarse near t = 0.01, as in the reference)
        assert np.max(np.abs(out - 1 / np.sqrt(t))) < 1e-6


@pytest.mark.parametrize("which,ow", [("mean", ST_MEAN), ("var", ST_VAR), ("moments", ST_MOMENTS)])
def test_moments(which, ow):
    from paper_2508_12093_b200 import rns as R
    x = _normal(2, 4000, 50.0, 10.0)
    e = _eval(LOGN, L)
    code = {"mean": R.MEAN, "var": R.VARIANCE, "moments": R.MOMENTS}[which]
    B = 1.0 if which == "mean" else 100.0
    out, lv = e.stat(code, x, B, out_n=1)
    ref = oracle().stat(Params(slot_count=S), ow, x, B)
    assert ref.rc == 0
    if which == "moments":
        _check_scalar(out[0], ref.out[0])
        _check_scalar(out[1], ref.out[S])
        assert tuple(lv[:2]) == ref.levels
    else:
        _check_scalar(out[0], ref.out[0])
        assert lv[0] == ref.levels[0]
    assert _meter(e) == ref.meter


def test_znorm_c2_shape():
    from paper_2508_12093_b200 import rns as R
    x = _normal(3, 4000, 50.0, 10.0)
    e = _eval(LOGN, L)
    z, lv = e.stat(R.ZNORM, x, 100.0)
    ref = oracle().stat(Params(slot_count=S), ST_ZNORM, x, 100.0)
    assert ref.rc == 0
    _check_vector(z, ref.out)
    assert _meter(e) == ref.meter and lv[0] == ref.levels[0]


@pytest.mark.parametrize("which", ["kurt", "skew"])
def test_std_moments_c3_shape(which):
    from paper_2508_12093_b200 import rns as R
    rng = np.random.default_rng(4)
    x = np.exp(0.5 * rng.standard_normal(S))  # log-normal (C3), skew ~1.75
    e = _eval(LOGN, L)
    code, ow = (R.KURTOSIS, ST_KURT) if which == "kurt" else (R.SKEWNESS, ST_SKEW)
    out, lv = e.stat(code, x, 20.0)
    ref = oracle().stat(Params(slot_count=S), ow, x, 20.0)
    assert ref.rc == 0
    _check_scalar(out[0], ref.out[0])
    assert _meter(e) == ref.meter and lv[0] == ref.levels[0]


def test_pearson_c4_shape():
    from paper_2508_12093_b200 import rns as R
    rng = np.random.default_rng(5)
    z = rng.standard_normal(S)
    x = np.sqrt(0.6) * z + np.sqrt(0.4) * rng.standard_normal(S)
    y = np.sqrt(0.6) * z + np.sqrt(0.4) * rng.standard_normal(S)
    e = _eval(LOGN, L)
    out, lv = e.stat(R.PEARSON, x, 20.0, y=y)
    ref = oracle().stat(Params(slot_count=S), ST_PEARSON, x, 20.0, y=y)
    assert ref.rc == 0
    _check_scalar(out[0], ref.out[0])
    assert _meter(e) == ref.meter and lv[0] == ref.levels[0]


def test_multichunk_kurtosis_masks_padding():
    """n > S: two chunks, the partial one masked by a plaintext-vector multiply (stats.hpp:56-75)."""
    from paper_2508_12093_b200 import rns as R
    x = _normal(6, S + 900, 0.0, 1.0)
    e = _eval(LOGN, L)
    out, lv = e.stat(R.KURTOSIS, x, 20.0)
    ref = oracle().stat(Params(slot_count=S), ST_KURT, x, 20.0)
    assert ref.rc == 0
    _check_scalar(out[0], ref.out[0])
    assert _meter(e) == ref.meter


def test_short_chain_fails_like_level_exhaustion():
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import rns as R
    e = _eval(LOGN, 8)
    with pytest.raises(H.level_exhausted):
        e.stat(R.ZNORM, _normal(7, 100, 50.0, 10.0), 100.0)


def test_errors_match_reference():
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import rns as R
    e = _eval(LOGN, L)
    with pytest.raises(H.empty_column):
        e.stat(R.MEAN, np.zeros(0), 1.0)
    with pytest.raises(H.non_finite_value):
        e.stat(R.MEAN, np.array([1.0, np.inf]), 1.0)
    with pytest.raises(H.length_mismatch):
        e.stat(R.PEARSON, np.ones(10), 1.0, y=np.ones(11))
    from paper_2508_12093_b200.rns import RnsEval
    with pytest.raises(H.error):
        RnsEval(_rns(LOGN, L), H.CkksParams(slot_count=S // 2))  # slot_count != N/2


@pytest.mark.parametrize("which", ["kurt", "skew", "pearson", "kurt_normal", "skew_normal"])
def test_full_size_c3_c4(which):
    """N = 2^16: the cancellation-prone statistics at full size, within 1e-6 (C3's two datasets:
    LogNormal(0, 0.5) and N(0,1), whose skewness ~1e-2 is the cancellation-prone case)."""
    from paper_2508_12093_b200 import rns as R
    rng = np.random.default_rng(12)
    Sf = 32768
    if which == "pearson":
        z = rng.standard_normal(Sf)
        x = np.sqrt(0.6) * z + np.sqrt(0.4) * rng.standard_normal(Sf)
        y = np.sqrt(0.6) * z + np.sqrt(0.4) * rng.standard_normal(Sf)
        code, ow = R.PEARSON, ST_PEARSON
    else:
        x = rng.standard_normal(Sf) if which.endswith("_normal") else np.exp(0.5 * rng.standard_normal(Sf))
        y = None
        code, ow = (R.KURTOSIS, ST_KURT) if which.startswith("kurt") else (R.SKEWNESS, ST_SKEW)
    e = _eval(16, 28)
    out, lv = e.stat(code, x, 20.0, y=y)
    ref = oracle().stat(Params(slot_count=Sf), ow, x, 20.0, y=y)
    assert ref.rc == 0
    _check_scalar(out[0], ref.out[0])
    assert _meter(e) == ref.meter and lv[0] == ref.levels[0]


def test_znorm_full_size_north_star():
    """C2: 32768 x N(50, 10^2) in one 2^15-slot ciphertext (N = 2^16), B = 100,
    invsqrt 511/6 — decrypted z within 1e-6 of the reference's decrypted output."""
    from paper_2508_12093_b200 import rns as R
    x = _normal(8, 32768, 50.0, 10.0)
    e = _eval(16, 28)
    z, lv = e.stat(R.ZNORM, x, 100.0)
    ref = oracle().stat(Params(slot_count=32768), ST_ZNORM, x, 100.0)
    assert ref.rc == 0
    _check_vector(z, ref.out)
    assert _meter(e) == ref.meter and lv[0] == ref.levels[0]


def test_batched_bsgs_matches_recursion():
    """RnsB's level-order batched BSGS (one batched op per tree stage) and batched chunk ops
    (mul_pt / squares over a column's chunks) against the op-by-op paths (HS_RNS_BSGS=0):
    bit-identical decrypted outputs, meters and levels."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, hashlib; sys.path[:0] = ["tests", "."]
import numpy as np
import test_rns_stats as T
from paper_2508_12093_b200 import rns as R
from paper_2508_12093_b200 import hestat as H
x = T._normal(5, T.S, 50.0, 10.0)
y = 0.6 * x + T._normal(6, T.S, 0.0, 4.0)
out = []
e = T._eval(T.LOGN, T.L)
v, lv = e.stat(R.ZNORM, x, 100.0)
out.append((v.tobytes(), tuple(lv), T._meter(e)))
e = T._eval(T.LOGN, T.L)
v, lv = e.stat(R.PEARSON, x, 20.0, y=y)
out.append((v.tobytes(), tuple(lv), T._meter(e)))
e = T._eval(T.LOGN, T.L)
v, lv = e.stat(R.INVSQRT, np.linspace(0.01, 1.0, T.S), 1.0, cfg=H.InvRootConfig(cheb_degree=15, newton_iters=2))
out.append((v.tobytes(), tuple(lv), T._meter(e)))
x3 = T._normal(9, 3 * T.S + 100, 50.0, 10.0)   # 4 chunks, the last partial: batched chunk ops
e = T._eval(T.LOGN, T.L)
v, lv = e.stat(R.ZNORM, x3, 100.0)
out.append((v.tobytes(), tuple(lv), T._meter(e)))
e = T._eval(T.LOGN, T.L)
v, lv = e.stat(R.KURTOSIS, x3, 20.0)
out.append((v.tobytes(), tuple(lv), T._meter(e)))
print(hashlib.sha256(repr(out).encode()).hexdigest())
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    digests = []
    for mode in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, "HS_RNS_BSGS": mode},
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        digests.append(r.stdout.strip().splitlines()[-1])
    assert digests[0] == digests[1]
