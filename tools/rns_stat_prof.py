"""One RNS ZNorm (N=2^16) inside a profiler range, for an ncu launch list."""
import os
import sys

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
H.sync()
torch.cuda.cudart().cudaProfilerStart()
ev.stat(R.ZNORM, x, 100.0)
H.sync()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
