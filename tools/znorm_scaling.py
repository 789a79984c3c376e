"""Device time (graph replay) of znorm / moments / crypto_invsqrt versus slot count:
separates the fixed per-call cost (launch, grid barriers, table staging) from the per-slot work."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2508_12093_b200 import _abi  # noqa: E402
if os.environ.get("HESTAT_LIB"):  # A/B a variant build of the library
    _abi.LIB_PATH = os.environ["HESTAT_LIB"]
from paper_2508_12093_b200 import hestat as H  # noqa: E402
from paper_2508_12093_b200 import workloads as W  # noqa: E402

H.init(0)
stream = torch.cuda.ExternalStream(H.stream_handle())


def graph_us(fn, reps=100):
    for _ in range(3):
        fn()
    H.sync()
    with H.Graph() as g:
        for _ in range(reps):
            r = fn()
            del r
    g.launch()
    H.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.launch()
    e1.record(stream)
    e1.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps


for S in (1024, 4096, 8192, 16384, 32768):
    x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    col = H.encode_column(ctx, x)
    var = H.moments(ctx, col, 100.0).ct_var
    z = graph_us(lambda: H.znorm(ctx, col, 100.0))
    m = graph_us(lambda: H.moments(ctx, col, 100.0))
    inv = graph_us(lambda: H.crypto_invsqrt(ctx, var, 100.0 * 100.0))
    print(f"S={S:6d} znorm {z:6.2f} us  moments {m:6.2f} us  invsqrt {inv:6.2f} us", flush=True)
