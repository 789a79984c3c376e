"""GPU parity: every golden case produced by the COMPILED REFERENCE replays
bit-for-bit through the CUDA product (status code, slot bit patterns, levels,
meter), on both execution paths:

  fused     symbolic ledger + fused kernels (the performance path), and
  op-by-op  one kernel per EvalContext op (debug / fallback path).
"""
import numpy as np
import pytest

from golden_io import cases
from oracle_abi import bits

GOLDEN = cases()


@pytest.fixture(params=["fused", "opbyop"])
def mode(request):
    from paper_2508_12093_b200 import hestat as H
    H.set_fused(request.param == "fused")
    yield request.param
    H.set_fused(True)


@pytest.mark.gpu
@pytest.mark.parametrize("entry,params,kw,expected", GOLDEN, ids=[c[0]["name"] for c in GOLDEN])
def test_golden_gpu(entry, params, kw, expected, mode):
    from gpu_harness import run_case
    rc, out, levels, meter = run_case(entry["api"], params, kw)
    assert rc == entry["rc"], f"rc {rc} != {entry['rc']} ({entry['msg']})"
    assert list(meter) == entry["meter"]
    if rc == 0:
        n = len(expected)
        assert np.array_equal(bits(out[:n]), bits(expected)), \
            f"max |diff| {np.max(np.abs(out[:n] - expected))}"
        assert list(levels) == entry["levels"][: len(levels)]
