"""Time the Tier-R kernels (device time, CUDA graph replay) at the C5 shapes.

  python tools/rns_probe.py [--logN 16] [--L 24] [--batch 8]
Prints one line per op: us per ciphertext-op and the HBM-roofline fraction
computed from the algorithmic bytes (DESIGN.md §Tier R).
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2508_12093_b200 import _abi  # noqa: E402
if os.environ.get("HESTAT_LIB"):  # A/B a variant build of the library
    _abi.LIB_PATH = os.environ["HESTAT_LIB"]
from paper_2508_12093_b200.rns import DeviceBuffer, RnsContext, RnsSpec  # noqa: E402


def graph_time(fn, reps=20):
    L = _abi.lib()
    fn()
    L.hs_sync()
    assert L.hs_graph_begin() == 0
    fn()
    g = C.c_void_p()
    assert L.hs_graph_end(C.byref(g)) == 0, L.hs_last_error()
    import torch
    L.hs_graph_launch(g)
    L.hs_sync()
    s = torch.cuda.ExternalStream(L.hs_stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        L.hs_graph_launch(g)
    e1.record(s)
    e1.synchronize()
    L.hs_graph_destroy(g)
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logN", type=int, default=16)
    ap.add_argument("--L", type=int, default=24)
    ap.add_argument("--K", type=int, default=9)
    ap.add_argument("--dnum", type=int, default=3)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--logp", type=int, default=44)
    ap.add_argument("--peak", type=float, default=6.5456e12)
    a = ap.parse_args()
    spec = RnsSpec(a.logN, a.L, a.K, a.dnum, logp=a.logp, seed=1)
    t = time.time()
    c = RnsContext(spec)
    c.prepare_relin()
    c.prepare_rotation(1)
    print(f"ctx+keys {time.time() - t:.2f}s", flush=True)
    N, l, B = spec.N, a.L, a.batch
    W = spec.ct_words(l)
    x = DeviceBuffer(B * W)
    y = DeviceBuffer(B * W)
    for i in range(B):
        c.random_ct(l, 1 + i, x, i * W)
        c.random_ct(l, 100 + i, y, i * W)
    out = DeviceBuffer(B * W)
    nl, K, dnum = l + 1, a.K, a.dnum
    alpha = (a.L + 1 + dnum - 1) // dnum
    nd = (nl + alpha - 1) // alpha
    key_bytes = 2 * nd * (nl + K) * N * 8  # the key rows one HMult reads
    res = {}
    us = graph_time(lambda: c.ntt(x, 0, nl, batch=2 * B)) / B
    res["ntt"] = (us, 2 * 2 * nl * N * 8)
    us = graph_time(lambda: c.ntt(x, 0, nl, batch=2 * B, inverse=True)) / B
    res["intt"] = (us, 2 * 2 * nl * N * 8)
    us = graph_time(lambda: c.mul_relin(l, x, y, out, batch=B)) / B
    res["mul_relin"] = (us, 3 * 2 * nl * N * 8 + key_bytes / B)
    us = graph_time(lambda: c.rescale(l, x, out, batch=B)) / B
    res["rescale"] = (us, (2 * nl + 2 * l) * N * 8)
    us = graph_time(lambda: c.rotate(l, 1, x, out, batch=B)) / B
    res["rotate"] = (us, 2 * 2 * nl * N * 8 + key_bytes / B)
    for k, (us, by) in res.items():
        print(json.dumps({"op": k, "logN": a.logN, "L": l, "batch": B, "us_per_ct": round(us, 2),
                          "alg_bytes": int(by), "GBps": round(by / us / 1e3, 1),
                          "hbm_frac": round(by / us / 1e3 / (a.peak / 1e9), 3)}), flush=True)


if __name__ == "__main__":
    main()
