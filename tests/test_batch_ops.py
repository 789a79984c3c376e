"""GPU: batched EvalContext ops (hs_*_batch, the C5 workloads) equal the single
ops element by element: slot bits, levels, CostMeter, auto-bootstrap and errors
(ckks.hpp:113-202), and match the oracle's single-op results."""
import numpy as np
import pytest

from oracle_abi import Params, bits, oracle

pytestmark = pytest.mark.gpu

S = 8192


def _ctx(**kw):
    from paper_2508_12093_b200 import hestat as H
    return H.EvalContext(H.CkksParams(slot_count=S, **kw))


def _cts(ctx, n, seed, levels=None):
    from paper_2508_12093_b200 import hestat as H
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        c = ctx.encrypt(rng.uniform(-1, 1, S))
        if levels is not None and levels[i] != ctx.params().max_level:
            c = H.Ciphertext(c.slots(), levels[i])
        out.append(c)
    return out


@pytest.mark.parametrize("op", ["add", "sub", "mul"])
@pytest.mark.parametrize("n", [1, 7, 64, 130])
def test_binary_batch_equals_single(op, n):
    ctx, ref = _ctx(), _ctx()
    a, b = _cts(ctx, n, 1), _cts(ctx, n, 2)
    out = getattr(ctx, f"{op}_ct_batch")(a, b)
    single = [getattr(ref, f"{op}_ct")(x, y) for x, y in zip(a, b)]
    for o, s in zip(out, single):
        assert np.array_equal(bits(o.slots()), bits(s.slots())) and o.level() == s.level()
    assert ctx.meter().as_tuple() == ref.meter().as_tuple()


@pytest.mark.parametrize("op,c", [("add_pt", -0.375), ("mul_pt", 1.0 / 3.0)])
def test_scalar_batch_equals_single(op, c):
    ctx, ref = _ctx(), _ctx()
    a = _cts(ctx, 65, 3)
    out = getattr(ctx, f"{op}_batch")(a, c)
    single = [getattr(ref, op)(x, c) for x in a]
    for o, s in zip(out, single):
        assert np.array_equal(bits(o.slots()), bits(s.slots())) and o.level() == s.level()
    assert ctx.meter().as_tuple() == ref.meter().as_tuple()


@pytest.mark.parametrize("k", [0, 1, 2, 3, 1024, 1023, -5, S - 1, S + 3])
def test_rotate_batch_equals_single(k):
    ctx, ref = _ctx(), _ctx()
    a = _cts(ctx, 9, 4)
    out = ctx.rotate_batch(a, k)
    for o, x in zip(out, a):
        s = ref.rotate(x, k)
        assert np.array_equal(bits(o.slots()), bits(s.slots())) and o.level() == s.level()
    assert ctx.meter().as_tuple() == ref.meter().as_tuple()


@pytest.mark.parametrize("slots", [1, 2, 64])
def test_rotate_batch_small(slots):
    from paper_2508_12093_b200 import hestat as H
    ctx = H.EvalContext(H.CkksParams(slot_count=slots))
    a = [ctx.encrypt(np.arange(slots) + 10.0 * i) for i in range(3)]
    for k in (0, 1, 3):
        out = ctx.rotate_batch(a, k)
        for o, x in zip(out, a):
            assert np.array_equal(o.slots(), np.roll(x.slots(), -k))


def test_batch_auto_bootstrap_per_element():
    """Exhausted elements are bootstrapped (and counted) individually, as single calls do."""
    ctx, ref = _ctx(), _ctx()
    lv = [0, 3, 0, 5, 11, 0]
    a, b = _cts(ctx, 6, 5, lv), _cts(ctx, 6, 6, lv[::-1])
    out = ctx.mul_ct_batch(a, b)
    single = [ref.mul_ct(x, y) for x, y in zip(a, b)]
    for o, s in zip(out, single):
        assert np.array_equal(bits(o.slots()), bits(s.slots())) and o.level() == s.level()
    assert ctx.meter().as_tuple() == ref.meter().as_tuple()
    assert ctx.meter().bootstrap == sum(1 for x, y in zip(lv, lv[::-1]) for v in (x, y) if v < 1)
    m = _cts(ctx, 3, 7, [0, 0, 2])
    out = ctx.mul_pt_batch(m, 0.5)
    assert [o.level() for o in out] == [10, 10, 1]


def test_batch_errors():
    from paper_2508_12093_b200 import hestat as H
    ctx = _ctx(auto_bootstrap=False)
    a = _cts(ctx, 3, 8, [2, 0, 2])
    with pytest.raises(H.level_exhausted):
        ctx.mul_ct_batch(a, a)
    with pytest.raises(H.length_mismatch):
        ctx.add_ct_batch(a, a[:2])
    other = H.EvalContext(H.CkksParams(slot_count=S // 2)).encrypt(np.ones(4))
    with pytest.raises(H.length_mismatch):
        ctx.add_ct_batch([a[0], other], [a[0], a[0]])


def test_batch_matches_oracle():
    ctx = _ctx()
    rng = np.random.default_rng(9)
    xs = [rng.uniform(-1, 1, S) for _ in range(4)]
    ys = [rng.uniform(-1, 1, S) for _ in range(4)]
    a = [ctx.encrypt(x) for x in xs]
    b = [ctx.encrypt(y) for y in ys]
    out = ctx.mul_ct_batch(a, b)
    p = Params(slot_count=S)
    for o, x, y in zip(out, xs, ys):
        ex = oracle().encrypt(p, x)
        ey = oracle().encrypt(p, y)
        r = oracle().op(p, 3, ex.out, ex.levels[0], ey.out, ey.levels[0])  # OP_MUL_CT
        assert r.rc == 0 and np.array_equal(bits(o.slots()), bits(r.out)) and o.level() == r.levels[0]
