"""hs_znorm_batch (many independent Z-scores in one launch) against the znorm calls it stands for
(stats.hpp:153-166): identical chunks (bits), levels and meter on the fused path (varying n_valid,
> 64 columns = several launches) and on every fallback (debug_checks, quantize off, multi-chunk
columns, sums beyond the exact-sum bound), plus the C oracle on one column."""
import numpy as np
import pytest

from oracle_abi import Params, ST_ZNORM, bits, oracle

pytestmark = pytest.mark.gpu


def _cols(S, ncols, n=None, seed=5, scale=10.0, shift=50.0):
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import workloads as W
    return [W.normal(H.synthetic_uniform, seed + k, n or S - 3 * k, shift, scale) for k in range(ncols)]


def _compare(params, xs, B=100.0):
    from paper_2508_12093_b200 import hestat as H
    ct, cs = H.EvalContext(params), H.EvalContext(params)
    ea, eb = [H.encode_column(ct, x) for x in xs], [H.encode_column(cs, x) for x in xs]
    before = H.kernel_launches()
    zb = H.znorm_batch(ct, ea, B)
    launched = H.kernel_launches() - before
    zs = [H.znorm(cs, c, B) for c in eb]
    for a, b in zip(zb, zs):
        assert [c.level() for c in a.chunks] == [c.level() for c in b.chunks]
        assert np.array_equal(bits(H.decode_column(ct, a)), bits(H.decode_column(cs, b)))
    assert ct.meter().as_tuple() == cs.meter().as_tuple()
    return launched, zb, ct


def test_batch_matches_calls_and_oracle():
    from paper_2508_12093_b200 import hestat as H
    S = 4096
    xs = _cols(S, 12)
    launched, zb, ctx = _compare(H.CkksParams(slot_count=S), xs)
    assert launched <= 2
    ref = oracle().stat(Params(slot_count=S), ST_ZNORM, xs[7], 100.0)
    assert np.array_equal(bits(H.decode_column(ctx, zb[7])), bits(ref.out))


def test_more_than_64_columns():
    from paper_2508_12093_b200 import hestat as H
    launched, _, _ = _compare(H.CkksParams(slot_count=1024), _cols(1024, 70))
    assert launched <= 4


@pytest.mark.parametrize("case", ["debug", "noquant", "multichunk", "inexact"])
def test_fallbacks_match_calls(case):
    from paper_2508_12093_b200 import hestat as H
    S = 1024
    if case == "debug":
        _compare(H.CkksParams(slot_count=S, debug_checks=True), _cols(S, 3))
    elif case == "noquant":
        _compare(H.CkksParams(slot_count=S, quantize=False), _cols(S, 3))
    elif case == "multichunk":
        _compare(H.CkksParams(slot_count=S), _cols(S, 3, n=2500))
    else:
        _compare(H.CkksParams(slot_count=S), _cols(S, 3, scale=1e7, shift=3e8), B=1e9)


def test_proven_exact_batch_is_capturable_and_matches():
    """encode_column's magnitude bound proves the exact-sum path on the host: no flag read, so the
    batch runs inside a CUDA graph; replaying it reproduces the eager result bit for bit."""
    from paper_2508_12093_b200 import hestat as H
    S = 4096
    xs = _cols(S, 6)
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    cols = [H.encode_column(ctx, x) for x in xs]
    eager = [H.decode_column(ctx, z) for z in H.znorm_batch(ctx, cols, 100.0)]
    with H.Graph() as g:
        zg = H.znorm_batch(ctx, cols, 100.0)
    g.launch()
    H.sync()
    for e, z in zip(eager, zg):
        assert np.array_equal(bits(e), bits(H.decode_column(ctx, z)))


def test_constant_bank_tree_in_graph_replay_and_between_tables():
    """One lane per slot (>= 1024 items per block): the degree-511 table is copied into the constant
    bank before each launch.  A captured batch carries its own copy node, so replaying it after an
    eager batch with a different table (another B) still gives the eager bits; HS_CONST_TREE-free
    semantics are checked against the per-column calls."""
    from paper_2508_12093_b200 import hestat as H
    S = 4096
    xs = _cols(S, 40)
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    cols = [H.encode_column(ctx, x) for x in xs]
    eager100 = [H.decode_column(ctx, z) for z in H.znorm_batch(ctx, cols, 100.0)]
    with H.Graph() as g:
        zg = H.znorm_batch(ctx, cols, 100.0)
    other = [H.decode_column(ctx, z) for z in H.znorm_batch(ctx, cols, 60.0)]  # another table in the bank
    g.launch()
    H.sync()
    for k in (0, 17, 39):
        assert np.array_equal(bits(eager100[k]), bits(H.decode_column(ctx, zg[k])))
        assert np.array_equal(bits(eager100[k]), bits(H.decode_column(ctx, H.znorm(ctx, cols[k], 100.0))))
        assert np.array_equal(bits(other[k]), bits(H.decode_column(ctx, H.znorm(ctx, cols[k], 60.0))))
    again = H.znorm_batch(ctx, cols, 60.0)  # eager after the replay: uploads its own table again
    assert np.array_equal(bits(other[5]), bits(H.decode_column(ctx, again[5])))
