"""Quick device-time probe of the C2 pipeline pieces (run on the GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch
from paper_2508_12093_b200 import hestat as H
from paper_2508_12093_b200 import workloads as W
H.init(0)
st = torch.cuda.ExternalStream(H.stream_handle())
x = W.normal(H.synthetic_uniform, 21, 32768, 50.0, 10.0)
ctx = H.EvalContext(H.CkksParams(slot_count=32768))
cols = [H.encode_column(ctx, np.roll(x, 97 * i)) for i in range(64)]
m = H.moments(ctx, cols[0], 100.0)

def t(fn, reps=100):
    for i in range(5): fn(i)
    H.sync(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter(); a.record(st)
    for i in range(reps): fn(i)
    b.record(st); H.sync(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps, (time.perf_counter() - w0) * 1e6 / reps

res = {}
res["invsqrt"] = t(lambda i: H.crypto_invsqrt(ctx, m.ct_var, 1e4))
res["moments"] = t(lambda i: H.moments(ctx, cols[i % 64], 100.0))
res["znorm"] = t(lambda i: H.znorm(ctx, cols[i % 64], 100.0))
res["kurtosis"] = t(lambda i: H.kurtosis(ctx, cols[i % 64], 20.0))
res["pearson"] = t(lambda i: H.pearson(ctx, cols[i % 64], cols[(i + 1) % 64], 20.0))
print(os.environ.get("HESTAT_LANES", "4"), {k: (round(v[0], 1), round(v[1], 1)) for k, v in res.items()})
