"""GPU: the reference's operator surface (EvalContext, ckks.hpp:83-257, and every entry point
built on it) backed by RNS-CKKS ciphertexts -- an EvalContext created with backend="rns"
(hs_ctx_create_rns; HESTAT_BACKEND=rns for unmodified programs).

Checked against the compiled reference's semantics (the C oracle, run live on the same inputs):
  * identical CostMeter counts, logical levels and error types (the reference's DAG and ledger);
  * decrypted outputs within north_star's 1e-6 relative of the reference's decrypted outputs, at
    every BASELINE config: C1 inverse sqrt (4096 slots, 15/2 and 511/6), C2 Z-score, C3 skewness
    and kurtosis of N(0,1) and LogNormal(0, 0.5), all 28 C4 Pearson pairs (2^15 slots, N = 2^16);
  * per-op values (encrypt/decrypt, add/sub/add_pt/mul_ct/mul_pt/rotate/sum_all_slots/bootstrap)
    within the CKKS noise of the reference's slot values.
Both bootstrap models run: BOOT_REFRESH (secret-key refresh at the reference's bootstraps, chain
max_level + 1 = 13 primes, logQP ~1150 bits: inside the 128-bit budget at N = 2^16 with a dense
secret) and BOOT_LOGICAL (deep chain, logical reset only).
"""
import numpy as np
import pytest

from oracle_abi import Cfg, Params, ST_KURT, ST_PEARSON, ST_SKEW, ST_ZNORM, oracle

pytestmark = pytest.mark.gpu

TOL = 1e-6
_CTX = {}


def _ctx(S, boot=0, **kw):
    from paper_2508_12093_b200 import hestat as H
    return H.EvalContext(H.CkksParams(slot_count=S, **kw), rng_seed=7, backend="rns", boot=boot)


def _m(ctx):
    return ctx.meter().as_tuple()


def _rel(got, ref):
    return abs(got - ref) / abs(ref)


def test_context_parameters_are_128bit_budget():
    c = _ctx(32768)
    s, boot = c.rns_spec()
    assert c.rns_backed() and boot == 0
    assert s.logN == 16 and s.L == 12 and s.h == 0  # max_level 11 + 1, dense ternary secret
    logqp = s.logq0 + s.L * s.logq + s.K * s.logp
    assert logqp <= 1760, logqp  # HE-standard 128-bit bound for N = 2^16 (ternary secret)


def test_encrypt_decrypt_and_ops_match_reference_values():
    from paper_2508_12093_b200 import hestat as H
    S = 4096
    c = _ctx(S)
    rng = np.random.default_rng(1)
    x, y = rng.uniform(-1, 1, S), rng.uniform(-1, 1, S)
    a, b = c.encrypt(x), c.encrypt(y)
    assert a.level() == 11 and a.size() == S
    assert np.max(np.abs(c.decrypt(a, S) - x)) < 1e-9
    assert np.max(np.abs(np.asarray(a.slots()) - x)) < 1e-9  # Ciphertext::slots() decrypts
    ref = H.EvalContext(H.CkksParams(slot_count=S))         # the emulator semantics (Tier E)
    ra, rb = ref.encrypt(x), ref.encrypt(y)
    cases = [
        (c.add_ct(a, b), ref.add_ct(ra, rb)),
        (c.sub_ct(a, b), ref.sub_ct(ra, rb)),
        (c.add_pt(a, 0.25), ref.add_pt(ra, 0.25)),
        (c.mul_ct(a, b), ref.mul_ct(ra, rb)),
        (c.mul_pt(a, -3.5), ref.mul_pt(ra, -3.5)),
        (c.mul_pt(a, y), ref.mul_pt(ra, y)),
        (c.rotate(a, 5), ref.rotate(ra, 5)),
        (c.rotate(a, -3), ref.rotate(ra, -3)),
        (c.bootstrap(c.mul_ct(a, b)), ref.bootstrap(ref.mul_ct(ra, rb))),
        (c.sum_all_slots(a, S), ref.sum_all_slots(ra, S)),
    ]
    for i, (g, r) in enumerate(cases):
        assert g.level() == r.level(), i
        tol = 1e-9 * (S if i == len(cases) - 1 else 1)
        assert np.max(np.abs(c.decrypt(g, S) - ref.decrypt(r, S))) < tol, i
    assert _m(c) == _m(ref)


def test_ledger_errors_match_reference():
    from paper_2508_12093_b200 import hestat as H
    c = _ctx(4096, max_level=2, auto_bootstrap=False)
    a = c.encrypt(np.full(4096, 0.5))
    a2 = c.mul_ct(a, a)
    a1 = c.mul_ct(a2, a2)
    with pytest.raises(H.level_exhausted):
        c.mul_ct(c.mul_ct(a1, a1), a1)
    with pytest.raises(H.too_many_values):
        c.encrypt(np.zeros(4097))
    with pytest.raises(H.length_mismatch):
        c.add_ct(a, H.Ciphertext([1.0, 2.0], 2))  # a host Ciphertext of another size


def test_host_constructed_ciphertext_is_encrypted_on_use():
    from paper_2508_12093_b200 import hestat as H
    c = _ctx(4096)
    v = np.linspace(-1, 1, 4096)
    h = H.Ciphertext(v, 5)
    s = c.add_ct(h, h)
    assert s.level() == 5
    assert np.max(np.abs(c.decrypt(s, 4096) - 2 * v)) < 1e-9


def _cfg_for(key):
    from paper_2508_12093_b200 import workloads as W
    return W.CONFIG_CASES[key]


def _inputs(key):
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import workloads as W
    return W.make_inputs(W.CONFIG_CASES[key], H.synthetic_uniform)


@pytest.mark.parametrize("key", ["C1_d15", "C1_d511"])
@pytest.mark.parametrize("boot", [0, 1])
def test_c1_invsqrt(key, boot):
    from paper_2508_12093_b200 import hestat as H
    spec = _cfg_for(key)
    x, _ = _inputs(key)
    cf = spec["kwargs"]["cfg"]
    cfg = H.InvRootConfig(cheb_degree=cf["cheb_degree"], newton_iters=cf["newton_iters"])
    c = _ctx(4096, boot=boot)
    y = H.crypto_invsqrt(c, c.encrypt(x), 1.0, cfg, 4096)
    ref = oracle().invroot(Params(slot_count=4096), 0, x, 11, 1.0, Cfg(cheb_degree=cf["cheb_degree"],
                                                                     newton_iters=cf["newton_iters"]))
    got = c.decrypt(y, 4096)
    assert np.max(np.abs(got - ref.out[:4096]) / np.abs(ref.out[:4096])) <= TOL
    assert _m(c) == ref.meter and y.level() == ref.levels[0]


@pytest.mark.parametrize("boot", [0, 1])
def test_c2_znorm(boot):
    from paper_2508_12093_b200 import hestat as H
    x, _ = _inputs("C2_B100")
    c = _ctx(32768, boot=boot)
    z = H.decode_column(c, H.znorm(c, H.encode_column(c, x), 100.0))
    ref = oracle().stat(Params(slot_count=32768), ST_ZNORM, x, 100.0)
    assert np.max(np.abs(z - ref.out)) / np.max(np.abs(ref.out)) <= TOL
    assert _m(c) == ref.meter


@pytest.mark.parametrize("key", ["C3_skew_normal", "C3_kurt_normal", "C3_skew_lognormal", "C3_kurt_lognormal"])
def test_c3_moments(key):
    """N(0,1) skewness (~1e-2, the cancellation-prone case) and kurtosis, and LogNormal(0, 0.5)."""
    from paper_2508_12093_b200 import hestat as H
    x, _ = _inputs(key)
    c = _ctx(32768)
    col = H.encode_column(c, x)
    skew = "skew" in key
    r = (H.skewness if skew else H.kurtosis)(c, col, 20.0)
    got = c.decrypt(r, 1)[0]
    ref = oracle().stat(Params(slot_count=32768), ST_SKEW if skew else ST_KURT, x, 20.0)
    assert _rel(got, ref.out[0]) <= TOL, (got, ref.out[0])
    assert _m(c) == ref.meter and r.level() == ref.levels[0]


def test_c4_all_28_pairs():
    """The 28-pair correlation table: columns encrypted once, 28 pearson calls (stats.hpp:239-265)."""
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import workloads as W
    tab = W.c4_table(H.synthetic_uniform)
    c = _ctx(32768)
    cols = [H.encode_column(c, tab[k]) for k in range(W.C4_COLS)]
    worst = 0.0
    for i, j in W.C4_PAIRS:
        c.set_meter(H.CostMeter())
        r = H.pearson(c, cols[i], cols[j], 20.0)
        got = c.decrypt(r, 1)[0]
        ref = oracle().stat(Params(slot_count=32768), ST_PEARSON, tab[i], 20.0, y=tab[j])
        assert _m(c) == ref.meter and r.level() == ref.levels[0], (i, j)
        worst = max(worst, _rel(got, ref.out[0]))
    assert worst <= TOL, worst


def test_multichunk_column_and_coeff_variation():
    """n > S (masked partial chunk, stats.hpp:56-75) and the fifth statistic (CV, stats.hpp:216-233)."""
    from paper_2508_12093_b200 import hestat as H
    from oracle_abi import ST_CV
    x = H.synthetic_uniform(1004, 3 * 4096 + 700, 0.0, 20.0)
    c = _ctx(4096)
    col = H.encode_column(c, x)
    r = H.coeff_variation(c, col, 20.0)
    got = c.decrypt(r, 1)[0]
    ref = oracle().stat(Params(slot_count=4096), ST_CV, x, 20.0)
    assert ref.rc == 0
    assert _rel(got, ref.out[0]) <= TOL and _m(c) == ref.meter
