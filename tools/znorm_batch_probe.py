"""Per-ciphertext device/wall time of hs_znorm_batch at C2 size for several batch widths
(inputs resident, distinct columns per call, L2 flushed before each timed call)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_2508_12093_b200 import _abi  # noqa: E402
if os.environ.get("HESTAT_LIB"):  # A/B a variant build of the library
    _abi.LIB_PATH = os.path.abspath(os.environ["HESTAT_LIB"])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2508_12093_b200 import hestat as H  # noqa: E402
from paper_2508_12093_b200 import workloads as W  # noqa: E402
from oracle_abi import Params, ST_ZNORM, bits, oracle  # noqa: E402

H.init(0)
S, B = 32768, 100.0
x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
ctx = H.EvalContext(H.CkksParams(slot_count=S))
pool = [H.encode_column(ctx, np.roll(x, 97 * i)) for i in range(256)]
ref = oracle().stat(Params(slot_count=S), ST_ZNORM, x, B)
ok = np.array_equal(bits(H.decode_column(ctx, H.znorm_batch(ctx, pool[:4], B)[0])), bits(ref.out))
s = torch.cuda.ExternalStream(H.stream_handle())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for K in (1, 8, 16, 32, 64, 128):
    best = None
    for r in range(4):
        cols = [pool[(r * K + i) % 256] for i in range(K)]
        with torch.cuda.stream(s):
            flush.fill_(1)
        H.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        z = H.znorm_batch(ctx, cols, B)
        e1.record(s)
        e1.synchronize()
        w = time.perf_counter() - t0
        if best is None or w < best[0]:
            best = (w, e0.elapsed_time(e1))
        del z
    print(f"K={K}: wall {1e6 * best[0] / K:.2f} us/ct, device {1e3 * best[1] / K:.2f} us/ct, parity {ok}")
