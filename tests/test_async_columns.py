"""encode_column_async / decode_column_async (hs_encode_column_async, hs_decode_column_async,
hs_pending_wait): the same chunks, slots and errors as the synchronous column.hpp:25-56 calls,
with the wait deferred; a column still being uploaded can be consumed at once."""
import numpy as np
import pytest

from oracle_abi import Params, ST_ZNORM, bits, oracle

pytestmark = pytest.mark.gpu


def _x(n, seed=3):
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import workloads as W
    return W.normal(H.synthetic_uniform, seed, n, 50.0, 10.0)


@pytest.mark.parametrize("n", [1, 1000, 4096, 10000])
def test_async_round_trip_matches_sync(n):
    from paper_2508_12093_b200 import hestat as H
    S = 4096
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    x = _x(n)
    col, pend = H.encode_column_async(ctx, x)
    ref = H.encode_column(ctx, x)
    assert len(col.chunks) == len(ref.chunks) and col.n_valid == ref.n_valid
    out = np.empty(n)
    d = H.decode_column_async(ctx, col, out)  # consumed while the upload may still be in flight
    pend.wait()
    d.wait()
    assert np.array_equal(bits(out), bits(H.decode_column(ctx, ref)))
    for a, b in zip(col.chunks, ref.chunks):
        assert a.level() == b.level()
        assert np.array_equal(bits(a.slots()), bits(b.slots()))


def test_pinned_large_column_and_pipeline_matches_oracle():
    """The bench's e2e shape at a small size: pinned buffers, chunks of an in-flight encode fed to
    znorm_batch, results fetched by decode_column_async; three steps deep."""
    import torch
    from paper_2508_12093_b200 import hestat as H
    S, KB = 4096, 70  # > 2 MiB: the DMA-staged path; > 64 columns: two launches
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    x = _x(S, seed=9)
    ref = oracle().stat(Params(slot_count=S), ST_ZNORM, x, 100.0)
    hx = torch.empty(KB * S, dtype=torch.float64).pin_memory().numpy()
    for j in range(KB):
        hx[j * S:(j + 1) * S] = np.roll(x, j)
    outs = [torch.zeros(KB * S, dtype=torch.float64).pin_memory().numpy() for _ in range(3)]
    pend_d = []
    for k in range(3):
        big, pe = H.encode_column_async(ctx, hx)
        zs = H.znorm_batch(ctx, [H.EncryptedColumn([c], S) for c in big.chunks], 100.0)
        pend_d.append(H.decode_column_async(ctx, H.EncryptedColumn([z.chunks[0] for z in zs], KB * S), outs[k]))
        pe.wait()
    for d in pend_d:
        d.wait()
    for o in outs:
        assert np.array_equal(bits(o[:S]), bits(ref.out))
        z1 = oracle().stat(Params(slot_count=S), ST_ZNORM, np.roll(x, 69), 100.0)
        assert np.array_equal(bits(o[69 * S:70 * S]), bits(z1.out))


def test_non_finite_verdict_is_raised_by_wait():
    from paper_2508_12093_b200 import hestat as H
    ctx = H.EvalContext(H.CkksParams(slot_count=1024))
    x = _x(3000)
    x[2500] = np.inf
    with pytest.raises(H.non_finite_value):
        H.encode_column(ctx, x)
    col, pend = H.encode_column_async(ctx, x)
    with pytest.raises(H.non_finite_value):
        pend.wait()
    with pytest.raises(H.non_finite_value):  # idempotent: the verdict is kept
        pend.wait()
    x[2500] = 1.0
    col, pend = H.encode_column_async(ctx, x)
    pend.wait()
    pend.wait()
    assert np.array_equal(bits(H.decode_column(ctx, col)), bits(H.decode_column(ctx, H.encode_column(ctx, x))))


def test_sync_decode_of_statistic_output_uses_one_copy_and_matches():
    """decode_column of a 64-chunk column made of znorm_batch outputs (one allocation) and of
    separately allocated chunks gives the same slots."""
    from paper_2508_12093_b200 import hestat as H
    S = 1024
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    xs = [_x(S, seed=20 + k) for k in range(5)]
    cols = [H.encode_column(ctx, x) for x in xs]
    zb = H.znorm_batch(ctx, cols, 100.0)
    joined = H.decode_column(ctx, H.EncryptedColumn([z.chunks[0] for z in zb], 5 * S))
    for k in range(5):
        assert np.array_equal(bits(joined[k * S:(k + 1) * S]), bits(H.decode_column(ctx, H.znorm(ctx, cols[k], 100.0))))
    mixed = H.decode_column(ctx, H.EncryptedColumn([zb[0].chunks[0], cols[1].chunks[0], zb[2].chunks[0]], 3 * S))
    assert np.array_equal(bits(mixed[S:2 * S]), bits(H.decode_column(ctx, cols[1])))
    assert np.array_equal(bits(mixed[2 * S:]), bits(joined[2 * S:3 * S]))


def test_rns_context_async_calls_complete_synchronously():
    from paper_2508_12093_b200 import hestat as H
    ctx = H.EvalContext(H.CkksParams(slot_count=512), rng_seed=7, backend="rns")
    x = _x(300) / 100.0
    col, pend = H.encode_column_async(ctx, x)
    pend.wait()
    out = np.empty(300)
    H.decode_column_async(ctx, col, out).wait()
    assert np.allclose(out, x, rtol=0, atol=1e-6)


def test_pending_column_used_inside_graph_capture():
    """A column whose upload is still in flight can be the input of captured work: the library
    settles the upload on the host instead of making an outside event a capture dependency."""
    from paper_2508_12093_b200 import hestat as H
    S = 4096
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    x = _x(S, seed=31)
    col, pend = H.encode_column_async(ctx, x)
    with H.Graph() as g:
        z = H.znorm(ctx, col, 100.0)
    pend.wait()
    g.launch()
    H.sync()
    ref = oracle().stat(Params(slot_count=S), ST_ZNORM, x, 100.0)
    assert np.array_equal(bits(H.decode_column(ctx, z)), bits(ref.out))


def test_edge_cases_empty_host_side_and_release_without_wait():
    from paper_2508_12093_b200 import hestat as H
    S = 1024
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    # empty column: nothing to upload, the pending is complete at once
    col, pend = H.encode_column_async(ctx, np.empty(0))
    pend.wait()
    assert len(col.chunks) == 0 and col.n_valid == 0
    H.decode_column_async(ctx, col, np.empty(0)).wait()
    # a column of host-constructed ciphertexts (no device buffer yet): decoded by a host copy
    v = _x(S, seed=41)
    hc = H.EncryptedColumn([H.Ciphertext(v, 3)], S)
    out = np.zeros(S)
    H.decode_column_async(ctx, hc, out).wait()
    assert np.array_equal(bits(out), bits(v))
    # an out buffer that is too short is refused before anything is enqueued
    with pytest.raises(H.length_mismatch):
        H.decode_column_async(ctx, hc, np.zeros(S - 1))
    # dropping a Pending without wait() settles it (the library waits inside hs_pending_release)
    x = _x(5 * S, seed=42)
    col, pend = H.encode_column_async(ctx, x)
    del pend
    assert np.array_equal(bits(H.decode_column(ctx, col)), bits(H.decode_column(ctx, H.encode_column(ctx, x))))
    big = np.zeros(5 * S)
    d = H.decode_column_async(ctx, col, big)
    del d
    H.sync()
    assert np.array_equal(bits(big), bits(H.decode_column(ctx, col)))


def test_too_many_chunks_and_mixed_readiness_decode():
    """A column mixing a statistic's outputs (completion event), an upload still in flight and a
    plain op result decodes to the same slots as chunk-by-chunk reads."""
    from paper_2508_12093_b200 import hestat as H
    S = 2048
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    a = H.encode_column(ctx, _x(S, seed=51))
    z = H.znorm(ctx, a, 100.0).chunks[0]                       # fused statistic output
    up, pend = H.encode_column_async(ctx, _x(S, seed=52))      # upload in flight
    plain = ctx.add_pt(a.chunks[0], 1.5)                       # op-by-op result
    mixed = H.EncryptedColumn([z, up.chunks[0], plain], 3 * S)
    out = np.zeros(3 * S)
    d = H.decode_column_async(ctx, mixed, out)
    pend.wait()
    d.wait()
    for k, c in enumerate((z, up.chunks[0], plain)):
        assert np.array_equal(bits(out[k * S:(k + 1) * S]), bits(c.slots()))
