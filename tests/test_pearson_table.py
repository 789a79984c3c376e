"""hs_pearson_table (C4's 28 pairs in one launch, one inverse square root per column) against the
28 sequential pearson calls it stands for (stats.hpp:239-265): identical slots (bits), levels and
meter, on the fused path and on every fallback (debug_checks, quantize off, multi-chunk columns,
sums beyond the exact-sum bound), plus the reference oracle on one pair."""
import numpy as np
import pytest

from oracle_abi import Params, ST_PEARSON, bits, oracle

pytestmark = pytest.mark.gpu


def _table(S, n, ncols, seed=41, rho=0.6, scale=1.0, shift=0.0):
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import workloads as W
    t = W.correlated_table(H.synthetic_uniform, seed, ncols, n, rho)
    return [shift + scale * c for c in t]


def _compare(params, cols, B=20.0, chunks_ok=True):
    from paper_2508_12093_b200 import hestat as H
    ctx_t = H.EvalContext(params)
    ctx_s = H.EvalContext(params)
    enc_t = [H.encode_column(ctx_t, c) for c in cols]
    enc_s = [H.encode_column(ctx_s, c) for c in cols]
    before = H.kernel_launches()
    tab = H.pearson_table(ctx_t, enc_t, B)
    launched = H.kernel_launches() - before
    seq = [H.pearson(ctx_s, enc_s[i], enc_s[j], B) for i in range(len(cols)) for j in range(i + 1, len(cols))]
    S = params.slot_count
    assert len(tab) == len(seq)
    for a, b in zip(tab, seq):
        assert a.level() == b.level()
        assert np.array_equal(bits(np.asarray(ctx_t.decrypt(a, S))), bits(np.asarray(ctx_s.decrypt(b, S))))
    assert ctx_t.meter().as_tuple() == ctx_s.meter().as_tuple()
    return launched, tab, ctx_t


def test_c4_table_one_launch_matches_sequential_and_oracle():
    from paper_2508_12093_b200 import hestat as H
    S = 4096
    cols = _table(S, 4000, 8)  # n_valid < S: the x side of every product is masked
    launched, tab, ctx = _compare(H.CkksParams(slot_count=S), cols)
    assert launched <= 2, launched
    ref = oracle().stat(Params(slot_count=S), ST_PEARSON, cols[2], 20.0, y=cols[5])
    k = [(i, j) for i in range(8) for j in range(i + 1, 8)].index((2, 5))
    assert np.array_equal(bits(np.asarray(ctx.decrypt(tab[k], S))), bits(ref.out[:S]))


def test_full_size_three_columns():
    from paper_2508_12093_b200 import hestat as H
    S = 32768
    launched, _, _ = _compare(H.CkksParams(slot_count=S), _table(S, S, 3, seed=7))
    assert launched <= 2


@pytest.mark.parametrize("case", ["debug", "noquant", "multichunk", "inexact"])
def test_fallbacks_match_sequential(case):
    from paper_2508_12093_b200 import hestat as H
    S = 1024
    if case == "debug":
        _compare(H.CkksParams(slot_count=S, debug_checks=True), _table(S, 1000, 4))
    elif case == "noquant":
        _compare(H.CkksParams(slot_count=S, quantize=False), _table(S, 1000, 4))
    elif case == "multichunk":
        _compare(H.CkksParams(slot_count=S), _table(S, 2500, 3))
    else:  # |terms| far beyond 2^52 grid units: the exact-sum shortcut cannot be proven
        launched, _, _ = _compare(H.CkksParams(slot_count=S), _table(S, 1000, 3, scale=1e7, shift=3e7), B=1.0)


def test_length_mismatch_raises_like_the_calls():
    from paper_2508_12093_b200 import hestat as H
    S = 1024
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    cols = [H.encode_column(ctx, c) for c in (np.ones(900), np.arange(900.0), np.arange(800.0))]
    with pytest.raises(H.length_mismatch):
        H.pearson_table(ctx, cols, 20.0)
