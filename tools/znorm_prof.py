"""A few C2 znorm calls (Tier E) for ncu capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2508_12093_b200 import hestat as H  # noqa: E402
from paper_2508_12093_b200 import workloads as W  # noqa: E402

H.init(0)
S = 32768
x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
ctx = H.EvalContext(H.CkksParams(slot_count=S))
col = H.encode_column(ctx, x)
for _ in range(3):
    z = H.znorm(ctx, col, 100.0)
H.sync()
import torch  # noqa: E402
torch.cuda.cudart().cudaProfilerStart()
z = H.znorm(ctx, col, 100.0)
H.sync()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
