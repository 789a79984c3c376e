"""How per-ciphertext Tier-R op time depends on the sub-batch size of the calls
(L2 residency of the key switch's intermediates versus key amortisation).

  python tools/rns_batch_probe.py [--logN 16 --L 24 --total 64]
For each sub-batch s, one CUDA graph issues total/s calls of s ciphertexts each;
prints us per ciphertext-op.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from rns_probe import graph_time  # noqa: E402
from paper_2508_12093_b200.rns import DeviceBuffer, RnsContext, RnsSpec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logN", type=int, default=16)
    ap.add_argument("--L", type=int, default=24)
    ap.add_argument("--K", type=int, default=9)
    ap.add_argument("--dnum", type=int, default=3)
    ap.add_argument("--logp", type=int, default=44)
    ap.add_argument("--total", type=int, default=64)
    ap.add_argument("--subs", default="1,2,4,8,16,64")
    ap.add_argument("--ops", default="ntt,mul_relin,rotate")
    a = ap.parse_args()
    spec = RnsSpec(a.logN, a.L, a.K, a.dnum, logp=a.logp, seed=1)
    c = RnsContext(spec)
    c.prepare_relin()
    c.prepare_rotation(1)
    l, T = a.L, a.total
    W = spec.ct_words(l)
    x, y, out = DeviceBuffer(T * W), DeviceBuffer(T * W), DeviceBuffer(T * W)
    for i in range(T):
        c.random_ct(l, 1 + i, x, i * W)
        c.random_ct(l, 100 + i, y, i * W)
    for s in [int(v) for v in a.subs.split(",")]:
        for op in a.ops.split(","):
            def run(op=op, s=s):
                for k in range(0, T, s):
                    if op == "ntt":
                        c.ntt(x.sub(k * W), 0, l + 1, batch=2 * s)
                    elif op == "mul_relin":
                        c.mul_relin(l, x.sub(k * W), y.sub(k * W), out.sub(k * W), batch=s)
                    elif op == "mul_relin_rescale":
                        c.mul_relin_rescale(l, x.sub(k * W), y.sub(k * W), out.sub(k * W), batch=s)
                    elif op == "rotate":
                        c.rotate(l, 1, x.sub(k * W), out.sub(k * W), batch=s)
            us = graph_time(run, reps=5) / T
            print(json.dumps({"op": op, "sub_batch": s, "total": T, "us_per_ct": round(us, 2)}), flush=True)


if __name__ == "__main__":
    main()
