"""GPU parity at BASELINE.json's config sizes (C1: 4096 slots; C2-C4: 32768 slots).

Each config workload runs through the product's public API (fused path) and
must reproduce, bit for bit, the output of the C oracle run live on the same
inputs, and — when the regenerated inputs match the fixture's input digest —
the compiled reference's SHA-256 digest, meter and levels in
tests/golden/golden_configs.json.
"""
import hashlib

import numpy as np
import pytest

from golden_io import config_digests
from oracle_abi import Cfg, Params, bits, oracle
from golden_io import run_case as oracle_run

DIGESTS = config_digests()


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint64).tobytes()).hexdigest()


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(DIGESTS))
def test_config_gpu(key):
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import workloads as W
    from gpu_harness import run_case
    H.set_fused(True)
    spec = W.CONFIG_CASES[key]
    x, y = W.make_inputs(spec, H.synthetic_uniform)
    params = Params(**spec["params"])
    kw = dict(spec["kwargs"], x=x, y=y)
    rc, out, levels, meter = run_case(spec["api"], params, dict(kw))
    d = DIGESTS[key]
    assert rc == d["rc"]
    assert list(meter) == d["meter"]
    assert list(levels) == d["levels"][: len(levels)]
    okw = dict(kw)
    okw["cfg"] = Cfg(**okw["cfg"])
    orc, oout, olev, om = oracle_run(oracle(), spec["api"], params, okw)
    assert orc == rc and tuple(om) == tuple(meter)
    assert np.array_equal(bits(out), bits(oout[: len(out)]))
    if hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == d["input_sha256"]:
        assert _sha(out) == d["sha256"]
