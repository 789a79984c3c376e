"""Batched end-to-end Z-score through the public API: where the step time goes, the loop over
the blocking calls, and the one-thread pipeline over the asynchronous calls
(encode_column_async k+1 | znorm_batch k | decode_column_async k, waits for k / k-1).
(Host threads over the blocking calls were tried first: 11.5-20 us per ciphertext and erratic,
the interpreter lock serialises the per-chunk wrapper work; the asynchronous calls need no threads.)

  python tools/e2e_batch_probe.py [--kb 64] [--steps 40]

Pieces are host-timed with a synchronisation after each (encode_column of kb x 2^15 pinned
values, znorm_batch, decode_column of the kb results).  The loops are timed wall-clock and
with CUDA events on the compute stream.
"""
import argparse
import concurrent.futures as cf
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kb", type=int, default=64)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--lag", type=int, default=2, help="decodes in flight before the host waits for the oldest")
    args = ap.parse_args()
    import torch
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import workloads as W
    from oracle_abi import Params, ST_ZNORM, bits, oracle
    H.init(0)
    S, B, KB = 32768, 100.0, args.kb
    x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
    ref = oracle().stat(Params(slot_count=S), ST_ZNORM, x, B)
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    nbuf = 6
    XB = [torch.empty(KB * S, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
    ZB = [torch.empty(KB * S, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
    xb = [t.numpy() for t in XB]
    zb = [t.numpy() for t in ZB]
    for b in xb:
        for j in range(KB):
            b[j * S:(j + 1) * S] = np.roll(x, 97 * j)

    def benc(i):
        big = H.encode_column(ctx, xb[i % nbuf])
        return [H.EncryptedColumn([c], S) for c in big.chunks]

    def bdec(zs, i):
        H.decode_column(ctx, H.EncryptedColumn([z.chunks[0] for z in zs], KB * S), out=zb[i % nbuf])

    for i in range(5):
        bdec(H.znorm_batch(ctx, benc(i), B), i)
    H.sync()

    def timed(fn, reps=10):
        H.sync()
        t0 = time.perf_counter()
        for _ in range(reps):
            r = fn()
        H.sync()
        return 1e3 * (time.perf_counter() - t0) / reps, r

    t_enc, col = timed(lambda: benc(0))
    l0 = H.kernel_launches()
    t_z, zs = timed(lambda: H.znorm_batch(ctx, col, B))
    print("launches per znorm_batch (block-encoded columns):", (H.kernel_launches() - l0) / 10)
    sep = [H.encode_column(ctx, np.roll(x, 97 * j)) for j in range(KB)]
    l0 = H.kernel_launches()
    t_zs, _ = timed(lambda: H.znorm_batch(ctx, sep, B))
    print(f"znorm_batch on separately encoded columns: {t_zs:.3f} ms, launches {(H.kernel_launches() - l0) / 10}")
    stream = torch.cuda.ExternalStream(H.stream_handle())
    for name, cc in (("block", col), ("separate", sep)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        H.sync()
        e0.record(stream)
        for _ in range(10):
            r = H.znorm_batch(ctx, cc, B)
        e1.record(stream)
        H.sync()
        print(f"znorm_batch device span ({name}): {e0.elapsed_time(e1) / 10:.3f} ms")
    t_dec, _ = timed(lambda: bdec(zs, 0))
    mb = KB * S * 8 / 1e6
    print(f"pieces (ms per {KB}-ciphertext step): encode {t_enc:.3f} ({mb / t_enc:.1f} GB/s)  "
          f"znorm_batch {t_z:.3f}  decode {t_dec:.3f} ({mb / t_dec:.1f} GB/s)")

    steps = args.steps
    # round-2 loop: encode k+1 overlaps znorm k, decode k serial
    H.sync()
    t0 = time.perf_counter()
    col = benc(0)
    for k in range(steps):
        zs = H.znorm_batch(ctx, col, B)
        col = benc(k + 1) if k + 1 < steps else None
        bdec(zs, k)
    H.sync()
    t_old = 1e3 * (time.perf_counter() - t0) / steps
    print(f"two-stage loop: {t_old:.3f} ms/step = {1e3 * t_old / KB:.2f} us/ciphertext")

    import collections
    # single-threaded asynchronous pipeline: encode k+1 | znorm_batch k | decode k, wait k-1
    def aenc(i):
        big, pend = H.encode_column_async(ctx, xb[i % nbuf])
        return [H.EncryptedColumn([c], S) for c in big.chunks], pend

    def adec(zs, i):
        return H.decode_column_async(ctx, H.EncryptedColumn([z.chunks[0] for z in zs], KB * S), zb[i % nbuf])

    for rep in range(2):
        for b in zb:
            b[:] = 0.0
        H.sync()
        t0 = time.perf_counter()
        col, pe = aenc(0)
        dq = collections.deque()
        ht = {"znorm_batch": 0.0, "encode_async": 0.0, "decode_async": 0.0, "wait_enc": 0.0, "wait_dec": 0.0}
        pc = time.perf_counter
        for k in range(steps):
            a0 = pc()
            zs = H.znorm_batch(ctx, col, B)  # ordered behind encode k on the device
            a1 = pc()
            pk = pe
            if k + 1 < steps:
                col, pe = aenc(k + 1)
            a2 = pc()
            dq.append(adec(zs, k))
            a3 = pc()
            pk.wait()  # encode k's finiteness verdict
            a4 = pc()
            while len(dq) > args.lag - 1:
                dq.popleft().wait()
            a5 = pc()
            for n_, v_ in zip(ht, (a1 - a0, a2 - a1, a3 - a2, a4 - a3, a5 - a4)):
                ht[n_] += v_
        while dq:
            dq.popleft().wait()
        if rep:
            print("async loop host time per step (ms):", {n_: round(1e3 * v_ / steps, 3) for n_, v_ in ht.items()})
        H.sync()
        t_async = 1e3 * (time.perf_counter() - t0) / steps
    ok2 = all(np.array_equal(bits(zb[i][:S]), bits(ref.out)) for i in range(nbuf))
    print(f"async single-thread pipeline: {t_async:.3f} ms/step = {1e3 * t_async / KB:.2f} us/ciphertext  parity {ok2}")
    ok = all(np.array_equal(bits(zb[i][:S]), bits(ref.out)) for i in range(nbuf))


if __name__ == "__main__":
    main()
