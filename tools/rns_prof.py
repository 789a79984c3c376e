"""Eager Tier-R op launches for ncu capture (no timing here).
  python tools/rns_prof.py OP [--logN 16 --L 24 --batch 8]   OP in ntt intt mul_relin rescale rotate"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_12093_b200 import _abi  # noqa: E402
from paper_2508_12093_b200.rns import DeviceBuffer, RnsContext, RnsSpec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("op")
ap.add_argument("--logN", type=int, default=16)
ap.add_argument("--L", type=int, default=24)
ap.add_argument("--K", type=int, default=9)
ap.add_argument("--dnum", type=int, default=3)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--logp", type=int, default=44)
ap.add_argument("--logq", type=int, default=40)
ap.add_argument("--logq0", type=int, default=60)
a = ap.parse_args()
spec = RnsSpec(a.logN, a.L, a.K, a.dnum, logq0=a.logq0, logq=a.logq, logp=a.logp, seed=1)
c = RnsContext(spec)
c.prepare_relin()
c.prepare_rotation(1)
l, B = a.L, a.batch
W = spec.ct_words(l)
x, y, out = DeviceBuffer(B * W), DeviceBuffer(B * W), DeviceBuffer(B * W)
for i in range(B):
    c.random_ct(l, 1 + i, x, i * W)
    c.random_ct(l, 100 + i, y, i * W)
_abi.lib().hs_sync()
import torch  # noqa: E402
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.reps):
    if a.op == "ntt":
        c.ntt(x, 0, l + 1, batch=2 * B)
    elif a.op == "intt":
        c.ntt(x, 0, l + 1, batch=2 * B, inverse=True)
    elif a.op == "mul_relin":
        c.mul_relin(l, x, y, out, batch=B)
    elif a.op == "mul_relin_rescale":
        c.mul_relin_rescale(l, x, y, out, batch=B)
    elif a.op == "rescale":
        c.rescale(l, x, out, batch=B)
    elif a.op == "rotate":
        c.rotate(l, 1, x, out, batch=B)
_abi.lib().hs_sync()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
