"""Device time of the Tier-E per-slot program's parts at C2 size (graph replay of 50 calls):
crypto_invsqrt (degree 511 + 6 Newton), eval_encrypted of the same degree-511 series alone,
newton_refine (6 iterations) alone, and a degree-63 / degree-7 series (tree-size scaling)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2508_12093_b200 import hestat as H  # noqa: E402

H.init(0)
S = 32768
ctx = H.EvalContext(H.CkksParams(slot_count=S, max_level=40))
t = ctx.encrypt(np.linspace(0.02, 1.9, S))
arg = ctx.encrypt(np.linspace(-0.98, 0.9, S))
y0 = ctx.encrypt(np.full(S, 1.1))
s = torch.cuda.ExternalStream(H.stream_handle())


def gt(fn, reps=50):
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
    e0.record(s)
    g.launch()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


ser = {d: H.fit(lambda v: H.scaled_target(H.ScaledTargetKind(0), 100.0 * 100.0, v), d) for d in (511, 63, 7)}
print(f"crypto_invsqrt 511/6: {gt(lambda: H.crypto_invsqrt(ctx, t, 1.0)):.2f} us")
for d, sr in ser.items():
    print(f"eval_encrypted degree {d}: {gt(lambda: H.eval_encrypted(ctx, sr, arg)):.2f} us")
print(f"newton_refine n=2 x6: {gt(lambda: H.newton_refine(ctx, t, y0, 2, 6)):.2f} us")
print(f"newton_refine n=2 x1: {gt(lambda: H.newton_refine(ctx, t, y0, 2, 1)):.2f} us")
