"""A/B of a Tier-E library variant: C2 znorm device time (graph replay of K steps on distinct
resident columns, L2 flushed) and bit-exactness vs the oracle.
    python tools/tier_e_ab.py [path/to/libhestat_variant.so]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_2508_12093_b200 import _abi  # noqa: E402
if len(sys.argv) > 1:
    _abi.LIB_PATH = os.path.abspath(sys.argv[1])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2508_12093_b200 import hestat as H  # noqa: E402
from paper_2508_12093_b200 import workloads as W  # noqa: E402
from oracle_abi import Params, ST_ZNORM, bits, oracle  # noqa: E402

H.init(0)
S, B, K = 32768, 100.0, 200
x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
ctx = H.EvalContext(H.CkksParams(slot_count=S))
pool = [H.encode_column(ctx, np.roll(x, 97 * i)) for i in range(K)]
ok = np.array_equal(bits(H.decode_column(ctx, H.znorm(ctx, pool[0], B))),
                    bits(oracle().stat(Params(slot_count=S), ST_ZNORM, x, B).out))
for i in range(5):
    H.znorm(ctx, pool[i], B)
H.sync()
with H.Graph() as g:
    for i in range(K):
        z = H.znorm(ctx, pool[i], B)
        del z
g.launch()
H.sync()
s = torch.cuda.ExternalStream(H.stream_handle())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
best = 1e9
for _ in range(3):
    with torch.cuda.stream(s):
        flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.launch()
    e1.record(s)
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / K * 1e3)
print(f"{os.path.basename(_abi.LIB_PATH)}: {best:.2f} us/znorm, bit-exact {ok}")
