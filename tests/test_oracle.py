"""CPU: pin the C restatement (oracle/hestat_oracle.c) to the reference.

1. every golden case produced by the COMPILED reference (tests/golden) replays
   bit-for-bit through the restatement: status code, slot bit patterns, levels,
   meter;
2. the config-shaped workloads (C1-C4 at 4096 / 32768 slots) reproduce the
   reference's SHA-256 digests, meters and levels;
3. the reference test suites' known-answer tests hold (ckks_test.cpp,
   chebyshev_test.cpp, primitives_test.cpp, stats_test.cpp);
4. where oracle/_ref was built, randomized cases agree with the live reference.
"""
import hashlib
import math

import numpy as np
import pytest

from golden_io import cases, config_digests, run_case
from oracle_abi import (ALL_SLOTS, FIT_EXP, FIT_IDENT, FIT_INVSQRT_SHIFTED, FIT_SQUARE, OP_ADD, OP_MUL_CT,
                        OP_MUL_PT, OP_ROTATE, OP_SUM_ALL, ST_MEAN, ST_SKEW, ST_VAR, ST_ZNORM, Cfg, Params, bits,
                        oracle, reference)

GOLDEN = cases()


@pytest.mark.parametrize("entry,params,kw,expected", GOLDEN, ids=[c[0]["name"] for c in GOLDEN])
def test_golden_bitwise(entry, params, kw, expected):
    rc, out, levels, meter = run_case(oracle(), entry["api"], params, kw)
    assert rc == entry["rc"], oracle().last_error()
    assert list(meter) == entry["meter"]
    if rc == 0:
        n = len(expected)
        assert np.array_equal(bits(out[:n]), bits(expected))
        assert list(levels) == entry["levels"][: len(levels)]


from paper_2508_12093_b200 import workloads as W  # noqa: E402

DIGESTS = config_digests()


@pytest.mark.parametrize("key", sorted(k for k in DIGESTS if not k.startswith("C4") or k in ("C4_p01", "C4_p67")))
def test_config_digest(key):
    spec = W.CONFIG_CASES[key]
    o = oracle()
    x, y = W.make_inputs(spec, o.synthetic_uniform)
    d = DIGESTS[key]
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == d["input_sha256"]
    kw = dict(spec["kwargs"], x=x, y=y)
    kw["cfg"] = Cfg(**kw["cfg"])
    rc, out, levels, meter = run_case(o, spec["api"], Params(**spec["params"]), kw)
    assert rc == d["rc"]
    assert list(meter) == d["meter"]
    assert list(levels) == d["levels"][: len(levels)]
    assert hashlib.sha256(np.ascontiguousarray(out).view(np.uint64).tobytes()).hexdigest() == d["sha256"]


# --- known-answer tests of the reference suites ---------------------------------------

def test_kat_ckks():
    o = oracle()
    p = Params(slot_count=4, quantize=False, auto_bootstrap=False)
    r = o.op(p, OP_ADD, [1, 2, 0, 0], 11, b=[3, 4, 0, 0], lb=11)          # ckks_test.cpp:87
    assert list(r.out[:2]) == [4, 6] and r.levels == (11,)
    r = o.op(p, OP_MUL_CT, [1, 2, 0, 0], 11, b=[3, 4, 0, 0], lb=11)       # ckks_test.cpp:110-111
    assert list(r.out[:2]) == [3, 8] and r.levels == (10,)
    r = o.op(p, OP_ROTATE, [1, 2, 3, 4], 11, k=-1)                        # ckks_test.cpp:161
    assert list(r.out) == [4, 1, 2, 3]
    r = o.op(p, OP_SUM_ALL, [1, 2, 3, 0], 11, n_valid=3)                  # ckks_test.cpp:182
    assert list(r.out) == [6, 6, 6, 6]
    r = o.op(p, OP_MUL_CT, [1, 0, 0, 0], 0, b=[1, 0, 0, 0], lb=0)         # ckks_test.cpp:117
    assert r.rc == 3  # level_exhausted
    pa = Params(slot_count=4, quantize=False)
    r = o.op(pa, OP_MUL_CT, [2, 0, 0, 0], 0, b=[2, 0, 0, 0], lb=0)        # ckks_test.cpp:120-129
    assert r.out[0] == 4.0 and r.levels == (10,) and r.meter[4] == 2
    pq = Params(slot_count=4, quantize=True)
    r = o.encrypt(pq, [0.3])                                               # ckks_test.cpp:58-67
    assert r.out[0] == math.ldexp(round(0.3 * 2.0 ** 40), -40)
    r = o.op(pq, OP_MUL_CT, o.encrypt(pq, [0.1]).out, 11, b=o.encrypt(pq, [0.3]).out, lb=11)
    assert abs(r.out[0] - 0.03) <= 2.0 ** -39                              # ckks_test.cpp:131-136
    r = o.op(p, OP_SUM_ALL, np.arange(8.0), 11, n_valid=8) if False else None


def test_kat_chebyshev():
    o = oracle()
    rc, c = o.fit(FIT_IDENT, 1, 3)                                         # chebyshev_test.cpp:37-45
    assert abs(c[1] - 1) < 1e-12 and max(abs(c[0]), abs(c[2]), abs(c[3])) < 1e-12
    rc, c = o.fit(FIT_SQUARE, 1, 2)                                        # chebyshev_test.cpp:47-53
    assert abs(c[0] - 0.5) < 1e-12 and abs(c[2] - 0.5) < 1e-12
    rc, c = o.fit(FIT_INVSQRT_SHIFTED, 100.0, 511)                         # chebyshev_test.cpp:63-70
    rc2, wide = o.fit(FIT_INVSQRT_SHIFTED, 100.0, 575)
    assert abs(o.eval_plain(c, -1, 1, 0.0)[0] - 0.1) <= np.abs(wide[512:]).sum()
    rc, c = o.fit(FIT_EXP, 1, 511)                                         # chebyshev_test.cpp:117-127
    r = o.eval_encrypted(Params(slot_count=8, quantize=False), c, -1, 1, [-0.5, 0, 0.25, 0, 0, 0, 0, 0], 11)
    assert r.levels == (2,) and r.meter[4] == 0
    rc, c = o.fit(FIT_EXP, 1, 255)                                         # chebyshev_test.cpp:161-170
    r = o.eval_encrypted(Params(slot_count=8, quantize=False), c, -1, 1, [0.5] + [0] * 7, 3)
    assert r.meter[4] == 1 and abs(r.out[0] - math.exp(0.5)) < 1e-9
    rc, _ = o.fit(9, 1, 8)                                                 # sqrt: non_finite_target
    assert rc == 6


def test_kat_primitives():
    o = oracle()
    p = Params(slot_count=4, quantize=False)
    r = o.newton_refine(p, [1, 0, 0, 0], 11, [1, 0, 0, 0], 11, 2, 3)       # primitives_test.cpp:46-52
    assert r.out[0] == 1.0
    r = o.newton_refine(p, [0.25, 0, 0, 0], 11, [1.8, 0, 0, 0], 11, 2, 4)  # primitives_test.cpp:54-62
    assert abs(r.out[0] - 2.0) < 1e-6
    pq = Params(slot_count=256, quantize=True)                             # primitives_test.cpp:108-119
    xs = o.synthetic_grid(256, 0.001, 100.0)
    r = o.invroot(pq, 0, o.encrypt(pq, xs / 100.0).out, 11, 100.0, Cfg(), 256)
    assert r.meter[4] == 2
    assert np.all(np.abs(r.out - 1 / np.sqrt(xs)) <= 1e-4 / np.sqrt(xs))


def test_kat_stats():
    o = oracle()
    p4 = Params(slot_count=4, quantize=False)
    r = o.stat(p4, ST_MEAN, [1, 2, 3, 4], 1.0)                            # stats_test.cpp:69-79
    assert list(r.out) == [2.5] * 4 and r.levels[0] == 10
    r = o.stat(p4, ST_VAR, [1, 2, 3, 4], 1.0)                             # stats_test.cpp:94-101
    assert abs(r.out[0] - 1.25) < 1e-12 and r.levels[0] == 9
    r = o.stat(Params(slot_count=8, quantize=False), ST_SKEW, [0, 0, 0, 10], 5.0)  # stats_test.cpp:193-201
    assert abs(r.out[0] - 2 / math.sqrt(3)) < 1e-4 and r.meter[4] == 2
    pz = Params(slot_count=2048, quantize=True)                           # stats_test.cpp:132-144
    v = o.synthetic_uniform(42, 2000, 0.0, 100.0)
    r = o.stat(pz, ST_ZNORM, v, 100.0)
    z = (v - v.mean()) / v.std()
    assert np.mean(np.abs(r.out - z) / np.abs(z)) <= 1e-4 and r.meter[4] == 2


# --- live reference (only where oracle/_ref was built) ---------------------------------

@pytest.mark.skipif(reference() is None, reason="oracle/_ref not built here")
@pytest.mark.parametrize("seed", range(6))
def test_random_vs_live_reference(seed):
    rng = np.random.default_rng(1000 + seed)
    o, ref = oracle(), reference()
    S = int(2 ** rng.integers(2, 11))
    q = bool(seed % 2)
    p = Params(slot_count=S, quantize=q, debug_checks=bool(seed % 3 == 0))
    x = rng.uniform(0.05, 1.5, S)
    cfg = Cfg(cheb_degree=int(rng.integers(0, 600)), newton_iters=int(rng.integers(0, 5)))
    for lib_call in (lambda L: L.invroot(p, 0, x, int(rng.integers(0, 12)), 2.0, cfg),
                     lambda L: L.stat(p, int(seed % 9), x * 10, 10.0, y=x[::-1] * 3, cfg=cfg)):
        st = rng.bit_generator.state
        a = lib_call(o)
        rng.bit_generator.state = st
        b = lib_call(ref)
        assert a.rc == b.rc and a.meter == b.meter and a.levels == b.levels
        assert np.array_equal(bits(a.out), bits(b.out))
