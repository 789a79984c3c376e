"""One C2 Z-score on an RNS-backed EvalContext (the bench's 128-bit refresh chain) inside a
profiler range, for an ncu launch list; also prints wall / GPU-span / kernel-sum timings and the
host-side share (codec, ledger, launch enqueue).

    python tools/rns_znorm_breakdown.py            # timings
    ncu --metrics gpu__time_duration.sum --profile-from-start off --csv \\
        python tools/rns_znorm_breakdown.py --prof  # launch list of one call
"""
import os
import sys
import time

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2508_12093_b200 import hestat as H  # noqa: E402
from paper_2508_12093_b200 import workloads as W  # noqa: E402

S, B = 32768, 100.0
x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
ctx = H.EvalContext(H.CkksParams(slot_count=S), rng_seed=5, backend="rns", boot=H.BOOT_REFRESH)
for _ in range(2):
    H.decode_column(ctx, H.znorm(ctx, H.encode_column(ctx, x), B))
H.sync()
stream = torch.cuda.ExternalStream(H.stream_handle())
if "--prof" in sys.argv:
    torch.cuda.cudart().cudaProfilerStart()
    H.decode_column(ctx, H.znorm(ctx, H.encode_column(ctx, x), B))
    H.sync()
    torch.cuda.cudart().cudaProfilerStop()
    print("ok")
    sys.exit(0)
for _ in range(3):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    H.sync()
    t0 = time.perf_counter()
    e[0].record(stream)
    col = H.encode_column(ctx, x)
    e[1].record(stream)
    t1 = time.perf_counter()
    z = H.znorm(ctx, col, B)
    e[2].record(stream)
    t2 = time.perf_counter()
    out = H.decode_column(ctx, z)
    e[3].record(stream)
    e[3].synchronize()
    t3 = time.perf_counter()
    print(f"wall ms: encode {1e3 * (t1 - t0):.2f} znorm-enqueue {1e3 * (t2 - t1):.2f} decode {1e3 * (t3 - t2):.2f} "
          f"total {1e3 * (t3 - t0):.2f} | gpu span ms: encode {e[0].elapsed_time(e[1]):.2f} "
          f"znorm {e[1].elapsed_time(e[2]):.2f} decode {e[2].elapsed_time(e[3]):.2f} | launches {H.kernel_launches()}")
