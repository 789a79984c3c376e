"""Wall vs device time of the RNS ZNorm (is the RNS statistics path host-bound?)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2508_12093_b200 import hestat as H  # noqa: E402
from paper_2508_12093_b200 import rns as R  # noqa: E402

L = 28
ctx = R.RnsContext(R.RnsSpec(logN=16, L=L, K=(L + 3) // 3 + 1, dnum=3, logq0=61, logq=60, logp=61, seed=5, h=192))
ev = R.RnsEval(ctx, H.CkksParams(slot_count=32768))
x = 50 + 10 * np.random.default_rng(1).standard_normal(32768)
ev.stat(R.ZNORM, x, 100.0)
stream = torch.cuda.ExternalStream(H.stream_handle())
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    H.sync()
    e0.record(stream)
    t0 = time.perf_counter()
    ev.stat(R.ZNORM, x, 100.0)
    e1.record(stream)
    e1.synchronize()
    wall = time.perf_counter() - t0
    print(f"wall {1e3 * wall:.1f} ms, device span {e0.elapsed_time(e1):.1f} ms, launches {H.kernel_launches()}")
