"""Quick device-time probe of the C2 pipeline pieces (run on the GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2508_12093_b200 import hestat as H
from paper_2508_12093_b200 import workloads as W
H.init(0)
st = torch.cuda.ExternalStream(H.stream_handle())
x = W.normal(H.synthetic_uniform, 21, 32768, 50.0, 10.0)
ctx = H.EvalContext(H.CkksParams(slot_count=32768))
cols = [H.encode_column(ctx, np.roll(x, 97 * i)) for i in range(64)]
z01 = W.normal(H.synthetic_uniform, 31, 32768, 0.0, 1.0)
ncols = [H.encode_column(ctx, np.roll(z01, 89 * i)) for i in range(64)]
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
res["kurtosis"] = t(lambda i: H.kurtosis(ctx, ncols[i % 64], 20.0))
res["pearson"] = t(lambda i: H.pearson(ctx, ncols[i % 64], ncols[(i + 1) % 64], 20.0))
print(os.environ.get("HESTAT_LANES", "4"), {k: (round(v[0], 1), round(v[1], 1)) for k, v in res.items()})

# host enqueue rate (no sync inside the loop): if it matches the device time, we are host-bound
def enq(fn, reps=200):
    for i in range(5): fn(i)
    H.sync()
    w0 = time.perf_counter()
    keep = [fn(i) for i in range(reps)]
    w1 = time.perf_counter()
    H.sync()
    return (w1 - w0) * 1e6 / reps
print("enqueue_us", {"invsqrt": round(enq(lambda i: H.crypto_invsqrt(ctx, m.ct_var, 1e4)), 1),
                     "moments": round(enq(lambda i: H.moments(ctx, cols[i % 64], 100.0)), 1),
                     "znorm": round(enq(lambda i: H.znorm(ctx, cols[i % 64], 100.0)), 1)})

# device-only time: the same calls captured into one CUDA graph and replayed
def gt(fn, reps=50):
    for i in range(3):
        fn(i)
    H.sync()
    with H.Graph() as g:
        for i in range(reps):
            r = fn(i)
            del r
    g.launch()
    H.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    g.launch()
    b.record(st)
    H.sync(); torch.cuda.synchronize()
    return round(a.elapsed_time(b) * 1e3 / reps, 2)
try:
    print("graph_us", {"invsqrt": gt(lambda i: H.crypto_invsqrt(ctx, m.ct_var, 1e4)),
                       "moments": gt(lambda i: H.moments(ctx, cols[i % 64], 100.0)),
                       "znorm": gt(lambda i: H.znorm(ctx, cols[i % 64], 100.0)),
                       "kurtosis": gt(lambda i: H.kurtosis(ctx, ncols[i % 64], 20.0)),
                       "pearson": gt(lambda i: H.pearson(ctx, ncols[i % 64], ncols[(i + 1) % 64], 20.0))})
except Exception as e:
    print("graph failed", repr(e))

# e2e breakdown (wall clock, pinned host buffers)
hx = torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
hp = torch.empty(32768, dtype=torch.float64).pin_memory()
def wall(fn, reps=200):
    for _ in range(5): fn()
    H.sync()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    H.sync()
    return round((time.perf_counter() - t0) * 1e6 / reps, 1)
col0 = H.encode_column(ctx, hx)
z0 = H.znorm(ctx, col0, 100.0)
print("e2e_parts_us", {"encode": wall(lambda: H.encode_column(ctx, hx)),
                       "znorm_call": wall(lambda: H.znorm(ctx, col0, 100.0)),
                       "decode": wall(lambda: H.decode_column(ctx, z0)),
                       "decode_pinned": wall(lambda: H.decode_column(ctx, z0, out=hp.numpy())),
                       "all": wall(lambda: H.decode_column(ctx, H.znorm(ctx, H.encode_column(ctx, hx), 100.0)))})

# raw transfer costs for 256 KiB (pinned <-> device), torch copies on the default stream
ht = torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
dt = torch.empty(32768, dtype=torch.float64, device="cuda")
hp = torch.empty(32768, dtype=torch.float64).pin_memory()
def tw(fn, reps=200):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn(); torch.cuda.synchronize()
    return round((time.perf_counter() - t0) * 1e6 / reps, 1)
print("xfer_us", {"h2d_256k": tw(lambda: dt.copy_(ht, non_blocking=True)),
                  "d2h_256k": tw(lambda: hp.copy_(dt, non_blocking=True)),
                  "sync_only": tw(lambda: None)})
