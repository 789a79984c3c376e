"""bench.py — encrypted Z-score on B200 (BASELINE.json metric, config C2).

Workload (configs[1]): one CKKS-emulated ciphertext of 2^15 slots holding
32768 fp64 values ~ N(50, 10^2), seed-drawn; znorm with B = 100 and the
reference's default inverse-root configuration (Chebyshev degree 511 seed, 6
Newton iterations, 2 bootstraps), scale 2^-40 quantisation.  A step is one
znorm of one ciphertext.

  value  device time per ciphertext, inputs already resident in HBM: each step
         is --batch-cols (64) independent C2 ciphertexts through hs_znorm_batch
         (every ciphertext its own moments, inverse square root and
         normalisation; one cooperative launch per step), K steps captured into
         a CUDA graph and replayed; the inputs cycle through a pool of distinct
         encrypted columns larger than L2 (config.l2).  `single_call` reports
         the same with one znorm call (one launch) per ciphertext.
  e2e    the same metric through the public API with HOST buffers: every step
         encodes its 64 ciphertexts' values from pinned host memory (16 MiB H2D),
         runs znorm_batch and decodes the results (16 MiB D2H), all inside the
         timed region, as a one-thread software pipeline over the asynchronous
         calls (encode_column_async k+1 | znorm_batch k | decode_column_async k,
         then the waits for k's verdict and k-2's results).
         `e2e_single_call` is the one-ciphertext-per-step loop (and its
         strictly sequential latency and pageable-buffer variants).

N > 1 (torchrun): replicas only — every rank runs its own ciphertexts, no
collective on the data path; value = max-over-ranks time /
ciphertexts processed by all ranks.

--impl reference runs the reference's own CPU implementation (oracle/_ref, the
unmodified reference headers compiled here; else the oracle port) on all host
cores on the same workload.

tier_r (same JSON line): the north_star RNS-CKKS primitives at N=2^16, L=24,
K=9, dnum=3 on a batch of 64 random ciphertexts under seeded keys (C5 shape):
HMult+relin/s, HMult+relin+rescale, rotate, rescale, NTT, each as device time
per ciphertext and as a fraction of the HBM roofline using BASELINE.md §4's
algorithmic bytes; the RNS oracle (port, 1 core) is the CPU stand-in.
`python bench.py --c5` prints the full C5 sweep (N in 2^14..2^16 x L in
8/16/24/32), one JSON line per (N, L).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "encrypted Z-score ms per 2^15-slot ciphertext"
UNIT = "ms/ciphertext"
S = 32768
B = 100.0
SEED = 21
# the same wording in both arms' config (the driver compares the dictionaries)
STEP_TEXT = ("independent C2 Z-scores (each its own moments, inverse square root and normalisation); "
             "value per ciphertext")
POOL = 640  # 640 x 256 KiB = 160 MiB of distinct inputs > 126 MB L2


def workload_config(extra=None):
    cfg = {"workload": "C2 znorm: 32768 x N(50,10^2) in one 2^15-slot ciphertext, B=100, "
                       "invsqrt degree 511 + 6 Newton, scale 2^-40",
           "slots": S, "B": B, "cheb_degree": 511, "newton_iters": 6,
           "l2": f"L2 flushed (256 MiB write) right before the timed region; every step reads its own resident "
                 f"ciphertexts, cycled over a pool of {POOL} ({POOL * S * 8 // (1 << 20)} MiB > L2)"}
    if extra:
        cfg.update(extra)
    return cfg


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---- clocks ----------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.out = self.p.communicate(timeout=5)[0]
            except Exception:
                self.out = ""

    def summary(self):
        rows = []
        for line in (getattr(self, "out", "") or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(rows[0][2]),
                "reasons": sorted(reasons), "samples": len(rows)}


# ---- CPU reference / oracle leg --------------------------------------------------------------------
def cpu_lib():
    from oracle_abi import oracle, reference
    ref = reference()
    if ref is not None:
        return ref, "reference"
    return oracle(), "port"


def cpu_znorm_sample(x, threads: int, total: int):
    """`total` independent znorm runs (one EvalContext each) over `threads` host
    threads; returns (wall seconds, output of one run)."""
    from oracle_abi import Params
    lib, kind = cpu_lib()
    p = Params(slot_count=S)
    per = [total // threads + (1 if i < total % threads else 0) for i in range(threads)]
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        futs = [ex.submit(lib.znorm_reps, p, x, B, n) for n in per if n > 0]
        outs = [f.result() for f in futs]
    wall = time.perf_counter() - t0
    assert all(o[0] == 0 for o in outs)
    return wall, outs[0][1], kind


def cpu_baseline(x):
    threads = os.cpu_count() or 1
    total = max(threads, 40)  # ~40 znorms x ~0.25 s = ~10 s of CPU work
    wall, out, kind = cpu_znorm_sample(x, threads, total)
    t1, _, _ = cpu_znorm_sample(x, 1, 1)
    return {"value": 1e3 * wall / total, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{total} independent C2 znorm runs (one EvalContext each) on {threads} host threads",
            "latency_1core_ms": 1e3 * t1}, out


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2508_12093_b200 import workloads as W
    from oracle_abi import oracle
    x = W.normal(oracle().synthetic_uniform, SEED, S, 50.0, 10.0)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_znorm_sample(x, threads, threads)
    walls = []
    for _ in range(args.steps):
        w, _, kind = cpu_znorm_sample(x, threads, threads)
        walls.append(w / threads)
    v = 1e3 * float(np.mean(walls))
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "config": workload_config({"parallelism": f"replicas x{max(args.gpus, 1)} (no data-path collective)",
                                       "ciphertexts_per_step": max(1, min(args.batch_cols, 64)),
                                       "step": STEP_TEXT}),
            "step_detail": "each Z-score its own EvalContext on a host thread (the reference's sanctioned "
                           "concurrency, SPEC.md:141)",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": kind,
                             "sample": f"per step: {threads} independent C2 znorm runs on {threads} threads"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---- Tier R (RNS-CKKS primitives) -----------------------------------------------------------------
def hbm_peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 7700.0, "B200_PROFILING.md fallback (no MEASURED_PEAKS.json)"


def rns_alg_bytes(logN, L, K, dnum, level):
    """BASELINE.md §4 algorithmic bytes per ciphertext-op (u64 words)."""
    N, l = 1 << logN, level
    key = 2 * dnum * (l + 1 + K) * N * 8
    return {
        "ntt": 2 * 2 * (l + 1) * N * 8,  # both polynomials of one ciphertext, read + write
        "mul_relin": 4 * (l + 1) * N * 8 + key + 2 * (l + 1) * N * 8,
        "mul_relin_rescale": 4 * (l + 1) * N * 8 + key + 2 * l * N * 8,
        "rotate": 2 * (l + 1) * N * 8 + key + 2 * (l + 1) * N * 8,
        "rescale": 2 * (l + 1) * N * 8 + 2 * l * N * 8,
    }


def special_primes(L, dnum, logq0=60, logq=40, logp=44):
    """K special primes of logp bits with P >= the largest digit modulus (q_0 + alpha-1 q's)."""
    alpha = (L + 1 + dnum - 1) // dnum
    return -(-(logq0 + (alpha - 1) * logq) // logp)


def rns_measure(torch, stream, logN, L, K, dnum, batch, reps=3, ops=None, logp=44, rot_steps=()):
    """Device time per ciphertext of each Tier-R op (CUDA-graph replay of `reps`
    batched calls), inputs resident; returns {op: us_per_ct}, launches per op."""
    from paper_2508_12093_b200 import _abi
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200.rns import DeviceBuffer, RnsContext, RnsSpec
    spec = RnsSpec(logN, L, K, dnum, logp=logp, seed=1)
    c = RnsContext(spec)
    c.prepare_relin()
    c.prepare_rotation(1)
    W = spec.ct_words(L)
    x, y, out = DeviceBuffer(batch * W), DeviceBuffer(batch * W), DeviceBuffer(batch * W)
    for i in range(batch):
        c.random_ct(L, 1 + i, x, i * W)
        c.random_ct(L, 1000 + i, y, i * W)
    H.sync()
    fns = {
        "ntt": lambda: c.ntt(x, 0, L + 1, batch=2 * batch),
        "intt": lambda: c.ntt(x, 0, L + 1, batch=2 * batch, inverse=True),
        "mul_relin": lambda: c.mul_relin(L, x, y, out, batch=batch),
        "mul_relin_rescale": lambda: c.mul_relin_rescale(L, x, y, out, batch=batch),
        "rescale": lambda: c.rescale(L, x, out, batch=batch),
        "rotate": lambda: c.rotate(L, 1, x, out, batch=batch),
    }
    for st_ in rot_steps:  # C5: rotation steps 1, 2, 4 ... 2^14 (each its own Galois key)
        c.prepare_rotation(st_)
        fns[f"rotate_{st_}"] = (lambda st__: lambda: c.rotate(L, st__, x, out, batch=batch))(st_)
    res, launches = {}, {}
    for name, fn in fns.items():
        if ops and name not in ops:
            continue
        fn()
        H.sync()
        l0 = H.kernel_launches()
        with H.Graph() as g:
            for _ in range(reps):
                fn()
        launches[name] = (H.kernel_launches() - l0) // reps
        g.launch()
        H.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.launch()
        e1.record(stream)
        e1.synchronize()
        res[name] = 1e3 * e0.elapsed_time(e1) / (reps * batch)
        del g
    for b in (x, y, out):
        b.free()
    c.close()
    H.sync()
    return res, launches


def rns_parity_small():
    """Limb-exact check of the bench path at a small shape against the RNS oracle."""
    from rns_abi import RnsOracle, Spec
    from paper_2508_12093_b200.rns import DeviceBuffer, RnsContext, RnsSpec
    s = Spec(logN=12, L=5, K=2, dnum=3, seed=9)
    O = RnsOracle()
    c = RnsContext(RnsSpec(s.logN, s.L, s.K, s.dnum, s.logq0, s.logq, s.logp, seed=s.seed, h=s.h))
    a, b = O.random_ct(s, s.L, 1), O.random_ct(s, s.L, 2)
    da, db = DeviceBuffer(a.size).upload(a), DeviceBuffer(b.size).upload(b)
    ok = np.array_equal(c.mul_relin_rescale(s.L, da, db).download(), O.mul_relin_rescale(s, s.L, a, b))
    ok &= np.array_equal(c.mul_relin(s.L, da, db).download(), O.mul_relin(s, s.L, a, b))
    ok &= np.array_equal(c.rotate(s.L, 1, da).download(), O.rotate(s, s.L, 1, a))
    c.close()
    return bool(ok)


def rns_cpu_baseline(logN, L, K, dnum, logp=44):
    """RNS oracle (plain C, 1 core) HMult+relin per ciphertext: (t(3 cts) - t(1 ct)) / 2,
    so the once-per-call key generation drops out."""
    from rns_abi import RnsOracle, Spec
    O = RnsOracle()
    s = Spec(logN=logN, L=L, K=K, dnum=dnum, seed=1, logp=logp)
    a = np.concatenate([O.random_ct(s, L, 1 + i) for i in range(3)])
    b = np.concatenate([O.random_ct(s, L, 100 + i) for i in range(3)])
    W = 2 * (L + 1) * s.N
    t0 = time.perf_counter()
    O.mul_relin_many(s, L, a[:W], b[:W], 1)
    t1 = time.perf_counter()
    O.mul_relin_many(s, L, a, b, 3)
    t3 = time.perf_counter() - t1
    per = (t3 - (t1 - t0)) / 2
    return {"value": 1.0 / per, "unit": "HMult+relin/s", "cores": 1, "kind": "port",
            "sample": f"RNS oracle (oracle/rns_oracle.c), N=2^{logN} L={L} K={K} dnum={dnum} logp={logp}: "
                      "3 HMult+relin minus 1 (key generation excluded), single thread",
            "ms_per_op": 1e3 * per}


def _znorm_rns_ctx(torch, ctx, x, reps):
    """best-of-reps wall time and GPU span (CUDA events on the library stream) of one
    encode_column + znorm + decode_column through the public API on an RNS-backed context."""
    from paper_2508_12093_b200 import _abi
    from paper_2508_12093_b200 import hestat as H
    s = torch.cuda.ExternalStream(_abi.lib().hs_stream())
    best = None
    for _ in range(reps):
        ctx.set_meter(H.CostMeter())
        H.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        z = H.decode_column(ctx, H.znorm(ctx, H.encode_column(ctx, x), B))
        e1.record(s)
        e1.synchronize()
        wall = time.perf_counter() - t0
        if best is None or wall < best[0]:
            best = (wall, e0.elapsed_time(e1), z, ctx.meter().as_tuple())
    return best


def rns_znorm(torch, stream, reps=3):
    """C2 Z-score on real RNS-CKKS ciphertexts through the reference's operator surface (an
    RNS-backed EvalContext: encode_column -> znorm -> decode_column), decrypted and compared with
    the reference's output.  Primary: bootstrap = secret-key refresh at the reference's bootstrap
    points on a chain of max_level + 1 = 13 primes (logQP ~1150 bits, dense ternary secret: inside
    the 128-bit budget at N=2^16).  Also the deep chain (bootstrap = logical level reset only;
    functional, not 128-bit) and the paper's 1M-sample Z-score."""
    from oracle_abi import Params, ST_ZNORM, oracle
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import rns as R
    from paper_2508_12093_b200 import workloads as W
    x = W.normal(H.synthetic_uniform, SEED, S, 50.0, 10.0)
    ref = oracle().stat(Params(slot_count=S), ST_ZNORM, x, B)
    ctx = H.EvalContext(H.CkksParams(slot_count=S), rng_seed=5, backend="rns", boot=H.BOOT_REFRESH)
    sp, _ = ctx.rns_spec()
    logqp = sp.logq0 + sp.L * sp.logq + sp.K * sp.logp
    _znorm_rns_ctx(torch, ctx, x, 1)  # keys (relin + 15 rotations), plans
    wall, gpu, z, meter = _znorm_rns_ctx(torch, ctx, x, reps)
    out = {"metric": "encrypted Z-score ms per 2^15-slot ciphertext (RNS-CKKS, public API)",
           "value": round(1e3 * wall, 2), "unit": "ms/ciphertext", "gpu_span_ms": round(gpu, 2),
           "config": {"logN": sp.logN, "L": sp.L, "K": sp.K, "dnum": sp.dnum, "logq0": sp.logq0, "logq": sp.logq,
                      "logp": sp.logp, "secret": "dense ternary" if sp.h == 0 else f"sparse h={sp.h}",
                      "logQP_bits": logqp, "bootstrap": "secret-key refresh at the reference's bootstrap points "
                                                        "(decrypt + re-encrypt at the top of the chain)",
                      "api": "EvalContext(params, seed, backend='rns'): encode_column, znorm, decode_column",
                      "timing": "wall and GPU span (CUDA events), keys warm, best of %d" % reps},
           "security": "evaluation on a 128-bit parameter set (logQP %d <= 1761 at N=2^16); bootstrapping "
                       "modelled as a trusted secret-key refresh" % logqp,
           "rel_err_vs_reference": float(np.max(np.abs(z - ref.out)) / np.max(np.abs(ref.out))),
           "meter_equal": tuple(meter) == tuple(ref.meter)}
    x1m = np.random.default_rng(SEED).uniform(0.0, 100.0, 1_000_000)
    r1 = oracle().stat(Params(slot_count=S), ST_ZNORM, x1m, B)
    w1, g1, z1, m1 = _znorm_rns_ctx(torch, ctx, x1m, 2)
    out["znorm_1m"] = {"value": round(1e3 * w1, 1), "unit": "ms per 1M-sample column (31 ciphertexts)",
                       "gpu_span_ms": round(g1, 1),
                       "rel_err_vs_reference": float(np.max(np.abs(z1 - r1.out)) / np.max(np.abs(r1.out))),
                       "meter_equal": tuple(m1) == tuple(r1.meter),
                       "note": "the paper's Lattigo CPU Z-score of 1M samples is 141.29 s with 2 real bootstraps "
                               "(PAPER.md:498); different work, no ratio claimed"}
    del ctx
    # deep chain: logical bootstraps only, L = 25 (the DAG's depth 24 + 1), dnum = 2
    spec = R.RnsSpec(logN=16, L=25, K=14, dnum=2, logq0=61, logq=60, logp=61, seed=5, h=192)
    dctx = H.EvalContext(H.CkksParams(slot_count=S), rng_seed=5, backend="rns", boot=H.BOOT_LOGICAL, rns_spec=spec)
    _znorm_rns_ctx(torch, dctx, x, 1)
    wall, gpu, z, meter = _znorm_rns_ctx(torch, dctx, x, reps)
    out["deep_chain"] = {"value": round(1e3 * wall, 2), "unit": "ms/ciphertext", "gpu_span_ms": round(gpu, 2),
                         "config": {"logN": 16, "L": 25, "K": 14, "dnum": 2, "logq0": 61, "logq": 60, "logp": 61,
                                    "secret": "sparse h=192", "logQP_bits": 61 + 25 * 60 + 14 * 61,
                                    "bootstrap": "logical level reset over the deep chain"},
                         "security": "functional, not 128-bit (logQP 2415 > 1761)",
                         "rel_err_vs_reference": float(np.max(np.abs(z - ref.out)) / np.max(np.abs(ref.out))),
                         "meter_equal": tuple(meter) == tuple(ref.meter)}
    return out


def tier_r_section(torch, stream, batch=64, with_cpu=True):
    # dnum = 2 (K = 13 x 44-bit so P exceeds the 13-prime digits): HMult 154 vs 168 us at dnum = 3
    # (K = 9) and 183 us at dnum = 4 with the round-2 kernels (profiles/r2_summary.md)
    logN, L, dnum, logp = 16, 24, 2, 44
    K = special_primes(L, dnum, logp=logp)
    peak, src = hbm_peak_gbs()
    us, launches = rns_measure(torch, stream, logN, L, K, dnum, batch)
    ab = rns_alg_bytes(logN, L, K, dnum, L)
    ab["intt"] = ab["ntt"]
    ops = {}
    for k, v in us.items():
        gbs = ab[k] / (v * 1e-6) / 1e9
        ops[k] = {"us_per_ct": round(v, 2), "ops_per_s": round(1e6 / v, 1), "alg_bytes": ab[k],
                  "achieved_gbs": round(gbs, 1), "hbm_frac": round(gbs / peak, 4), "launches": launches[k]}
        tr = rns_traffic("ntt" if k == "intt" else k, logN, L, K)
        if tr:  # real DRAM bytes (ncu) moved per ciphertext at this op's bench time
            ops[k]["dram_bytes"] = round(tr)
            ops[k]["dram_gbs"] = round(tr / (v * 1e-6) / 1e9, 1)
            ops[k]["dram_frac"] = round(tr / (v * 1e-6) / 1e9 / peak, 4)
    sec = {"metric": "HMult+relin/s", "value": round(1e6 / us["mul_relin"], 1), "unit": "HMult+relin/s",
           "config": {"workload": "C5 tier R: batch of 64 random ciphertexts under seeded keys",
                      "logN": logN, "L": L, "K": K, "dnum": dnum, "level": L, "batch": batch,
                      "logq0": 60, "logq": 40, "logp": logp, "word": "u64",
                      "security": "logQP %d bits, dense ternary secret: inside the 128-bit budget at N=2^16 "
                                  "(1761)" % (60 + 40 * L + logp * K),
                      "l2": "inputs > L2 (64 x 25.6 MiB per operand)"},
           "ops": ops,
           "roofline": {"bound": "hbm", "kernel": "HMult+relin (whole op, BASELINE.md §4 bytes)",
                        "achieved": ops["mul_relin"]["achieved_gbs"], "peak": peak, "unit": "GB/s",
                        "frac": ops["mul_relin"]["hbm_frac"], "traffic": rns_traffic("mul_relin", logN, L, K),
                        "peak_source": src,
                        "traffic_source": "profiles/r2_tier_r_traffic.json (ncu dram bytes per ciphertext, "
                                          "tools/rns_traffic.py, batch 16)",
                        "note": "the key switch's intermediates and the two-pass NTTs go through HBM (real traffic "
                                "~3.5x the algorithmic bytes); the NTT passes are FP64-issue/latency bound "
                                "(ncu: FP64 pipe 42-54%, issue 46-51%); base conversion on tcgen05 (k_conv_tc), "
                                "see profiles/r2_summary.md"},
           "parity_vs_oracle": rns_parity_small(),
           "znorm": rns_znorm(torch, stream)}
    if with_cpu:
        sec["cpu_baseline"] = rns_cpu_baseline(logN, L, K, dnum, logp)
    return sec


def rns_traffic(op, logN, L, K):
    """DRAM bytes per ciphertext of a Tier-R op from profiles/r2_tier_r_traffic.json (or round 1's),
    None if absent or captured at another shape."""
    for name in ("r2_tier_r_traffic.json", "r1_tier_r_traffic.json"):
        p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name)
        try:
            with open(p) as f:
                d = json.load(f)
            sh = d["shape"]
            if (sh["logN"], sh["L"], sh["K"]) == (logN, L, K):
                return d["ops"][op]["dram_bytes_per_ct"]
        except (OSError, KeyError, ValueError):
            pass
    return None


def zbatch_lanes():
    """Threads per slot of the batched Z-score kernel (the library's default, or HESTAT_BATCH_LANES)."""
    v = os.environ.get("HESTAT_BATCH_LANES", "")
    return int(v) if v in ("1", "2", "4") else 1  # the library's choice for a 64-ciphertext step


def zbatch_traffic(kb):
    """DRAM bytes per k_zbatch launch of kb ciphertexts from the committed ncu --set full summary."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r2_zbatch_ct_ncu.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if d["ciphertexts"] != kb:
            return None
        return d["dram_bytes_read"] + d["dram_bytes_write"]
    except (OSError, KeyError, ValueError):
        return None


def kstat_traffic():
    """DRAM bytes per k_stat launch from the committed ncu --set full summary (None if absent)."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_kstat_ncu.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d["dram_bytes_read"] + d["dram_bytes_write"]
    except (OSError, KeyError, ValueError):
        return None


def c5_tier_e(torch, stream, S_, batch=64, pools=8, reps=3, ops=None):
    """C5 tier E: batched EvalContext ops on `batch` ciphertexts of S_ U[-1,1] slots.
    Device time per batch via graph replay over `pools` distinct input batches (> L2);
    HBM roofline with SURVEY §8(d) bytes: 24 B/slot (add, mul_ct), 16 B/slot (mul_pt, rotate)."""
    from paper_2508_12093_b200 import hestat as H
    ctx = H.EvalContext(H.CkksParams(slot_count=S_))
    rng = np.random.default_rng(S_)
    base = [ctx.encrypt(rng.uniform(-1, 1, S_)) for _ in range(batch)]
    # distinct pools: rotated copies (each its own allocation)
    a = [ctx.rotate_batch(base, 97 * p + 1) for p in range(pools)]
    b = [ctx.rotate_batch(base, 131 * p + 7) for p in range(pools)]
    H.sync()
    logS = S_.bit_length() - 1
    fns = {"mul_ct": (lambda p: ctx.mul_ct_batch(a[p], b[p]), 24),
           "add": (lambda p: ctx.add_ct_batch(a[p], b[p]), 24),
           "mul_pt": (lambda p: ctx.mul_pt_batch(a[p], 0.731), 16)}
    for j in range(logS):
        fns[f"rotate_{1 << j}"] = ((lambda k: (lambda p: ctx.rotate_batch(a[p], k)))(1 << j), 16)
    peak, _ = hbm_peak_gbs()
    res = {}
    for name, (fn, bps) in fns.items():
        if ops and name not in ops:
            continue
        for p in range(pools):
            fn(p)
        H.sync()
        with H.Graph() as g:
            for r in range(reps):
                for p in range(pools):
                    fn(p)
        g.launch()
        H.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.launch()
        e1.record(stream)
        e1.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / (reps * pools)  # per batch
        gbs = bps * S_ * batch / (us * 1e-6) / 1e9
        res[name] = {"us_per_batch": round(us, 2), "ops_per_s": round(batch / (us * 1e-6), 1),
                     "achieved_gbs": round(gbs, 1), "hbm_frac": round(gbs / peak, 4)}
        del g
    return res


def c5_tier_e_cpu(S_, batch=64):
    """The reference's own op (oracle/_ref shim) on all host threads: mul_ct over a batch."""
    from oracle_abi import Params
    lib, kind = cpu_lib()
    p = Params(slot_count=S_)
    rng = np.random.default_rng(S_)
    xs = [rng.uniform(-1, 1, S_) for _ in range(batch)]
    enc = [lib.encrypt(p, x) for x in xs]
    threads = min(os.cpu_count() or 1, batch)
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(lambda e: lib.op(p, 3, e.out, e.levels[0], e.out, e.levels[0]), enc))
    wall = time.perf_counter() - t0
    return {"value": round(batch / wall, 1), "unit": "mul_ct/s", "cores": threads, "kind": kind,
            "sample": f"{batch} mul_ct of {S_} slots through the reference's EvalContext::mul_ct, {threads} threads"}


def c5_sweep(args):
    import torch
    torch.cuda.set_device(0)
    from paper_2508_12093_b200 import hestat as H
    H.init(0)
    stream = torch.cuda.ExternalStream(H.stream_handle())
    for S_ in (8192, 16384, 32768):
        line = {"sweep": "C5 tier E", "slots": S_, "batch": args.batch, "ops": c5_tier_e(torch, stream, S_, args.batch),
                "cpu_baseline": c5_tier_e_cpu(S_, args.batch)}
        print(json.dumps(line), flush=True)
    peak, src = hbm_peak_gbs()
    for logN in (14, 15, 16):
        for L in (8, 16, 24, 32):
            # dnum = 2 measured fastest with the round-2 kernels (profiles/r2_summary.md; the bench shape); the
            # tensor-core base conversion takes digits of up to 16 primes, so L = 32 runs dnum = 3
            dnum = 2 if (L + 2) // 2 <= 16 else 3
            K = special_primes(L, dnum)
            steps_ = tuple(1 << j for j in range(1, logN - 1)) if (logN, L) == (16, 24) else ()
            us, launches = rns_measure(torch, stream, logN, L, K, dnum, args.batch, rot_steps=steps_)
            ab = rns_alg_bytes(logN, L, K, dnum, L)
            ab["intt"] = ab["ntt"]
            for st_ in steps_:
                ab[f"rotate_{st_}"] = ab["rotate"]
            line = {"sweep": "C5 tier R", "logN": logN, "L": L, "K": K, "dnum": dnum, "logp": 44, "batch": args.batch,
                    "peak_gbs": peak, "ops": {k: {"us_per_ct": round(v, 2), "ops_per_s": round(1e6 / v, 1),
                                                  "hbm_frac": round(ab[k] / (v * 1e-6) / 1e9 / peak, 4)}
                                              for k, v in us.items()}}
            print(json.dumps(line), flush=True)
    return 0


# ---- GPU leg ---------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tier-r", action="store_true")
    ap.add_argument("--c5", action="store_true", help="print the C5 tier-R sweep instead")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--profile-step", action="store_true",
                    help="only the timed step, eagerly, between cudaProfilerStart/Stop (for ncu "
                         "--profile-from-start off: the launch list of exactly the K timed steps)")
    ap.add_argument("--batch-cols", type=int, default=64,
                    help="independent C2 ciphertexts per step (hs_znorm_batch, <= 64 per launch)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.c5:
        return c5_sweep(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import workloads as W
    H.init(local)
    stream = torch.cuda.ExternalStream(H.stream_handle())

    def barrier_sync():
        torch.cuda.synchronize()
        H.sync()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # inputs: the seeded C2 column (identical on every rank) + a pool of distinct
    # rolled copies so each step reads a column that is not L2-resident
    x = W.normal(H.synthetic_uniform, SEED, S, 50.0, 10.0)
    ctx = H.EvalContext(H.CkksParams(slot_count=S), rng_seed=rank)
    pool = [H.encode_column(ctx, np.roll(x, 97 * i)) for i in range(POOL)]
    H.sync()

    # correctness gate: output of the bench path == oracle, bit for bit
    from oracle_abi import Params, ST_ZNORM, bits, oracle
    z = H.decode_column(ctx, H.znorm(ctx, pool[0], B))
    ref = oracle().stat(Params(slot_count=S), ST_ZNORM, x, B)
    parity = bool(np.array_equal(bits(z), bits(ref.out)))

    # ---- value: device time, inputs resident ----------------------------------------------
    # The K timed steps are captured once into a CUDA graph (hs_graph_*) and
    # replayed: every step is a full znorm launch on a distinct resident column;
    # the graph only removes per-call host/launch overhead (measured separately
    # below as api_loop_ms_per_step).
    for i in range(args.warmup):
        H.znorm(ctx, pool[i % POOL], B)
    barrier_sync()
    launches0 = H.kernel_launches()
    with H.Graph() as graph:
        for i in range(args.steps):
            zc = H.znorm(ctx, pool[i % POOL], B)
            del zc
    launches = H.kernel_launches() - launches0
    graph.launch()  # warm replay (untimed)
    barrier_sync()
    # L2 flush before the timed region (the timed steps then read inputs no step has touched since)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        flush.fill_(1)
    e0.record(stream)
    graph.launch()
    e1.record(stream)
    barrier_sync()
    dev_ms = e0.elapsed_time(e1)
    del graph

    # ---- value (headline): KB independent C2 ciphertexts per step, one hs_znorm_batch launch ----
    # Every ciphertext gets its whole Z-score DAG (moments, degree-511 + 6-Newton inverse square
    # root of ITS variance, (x - mu) inv); the batch shares one launch, one grid barrier and the
    # SMs' latency hiding.  encode_column's magnitude bound proves the exact sums on the host, so the
    # call has no synchronisation and the K steps are captured into one CUDA graph.
    KB = max(1, min(args.batch_cols, 64))

    def bcols(i):
        return [pool[(i * KB + j) % POOL] for j in range(KB)]

    zb0 = H.znorm_batch(ctx, bcols(0), B)
    bparity = bool(np.array_equal(bits(H.decode_column(ctx, zb0[0])), bits(ref.out)))
    del zb0
    for i in range(args.warmup):
        zb = H.znorm_batch(ctx, bcols(i), B)
        del zb
    barrier_sync()
    if args.profile_step:  # the K steps of the timed region, eager, inside the profiler range
        torch.cuda.cudart().cudaProfilerStart()
        for i in range(args.steps):
            zb = H.znorm_batch(ctx, bcols(i), B)
            del zb
        barrier_sync()
        torch.cuda.cudart().cudaProfilerStop()
        print(json.dumps({"profile_step": True, "steps": args.steps, "parity_vs_oracle": parity and bparity}))
        return 0
    bl0 = H.kernel_launches()
    with H.Graph() as bgraph:
        for i in range(args.steps):
            zb = H.znorm_batch(ctx, bcols(i), B)
            del zb
    blaunches = H.kernel_launches() - bl0
    bgraph.launch()  # warm replay (untimed)
    barrier_sync()
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.3)  # let the sampler start
        with torch.cuda.stream(stream):
            flush.fill_(1)
        b0.record(stream)
        bgraph.launch()
        b1.record(stream)
        barrier_sync()
        t_end = time.perf_counter() + 1.0  # keep the same load on for the clock samples
        while time.perf_counter() < t_end:
            bgraph.launch()
            H.sync()
    bdev_ms = b0.elapsed_time(b1)
    del bgraph

    # same K steps as plain API calls (host enqueue included)
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for i in range(args.steps):
        zc = H.znorm(ctx, pool[i % POOL], B)
        del zc
    a1.record(stream)
    barrier_sync()
    api_ms = a0.elapsed_time(a1)

    # ---- e2e: host buffers through the public API ----------------------------------------------
    hx = torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
    hz = torch.empty(S, dtype=torch.float64).pin_memory()
    xin = hx.numpy()
    hzn = hz.numpy()
    # warm-up (host clocks, the memory pool's cross-stream blocks): both loop shapes
    for _ in range(max(args.warmup, 100)):
        H.decode_column(ctx, H.znorm(ctx, H.encode_column(ctx, xin), B), out=hzn)
    col = H.encode_column(ctx, xin)
    for k_ in range(max(args.warmup, 100)):
        zc = H.znorm(ctx, col, B)
        col = H.encode_column(ctx, xin)
        H.decode_column(ctx, zc, out=hzn)
    del col, zc
    barrier_sync()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(100, args.steps)
    # strictly sequential: one ciphertext in flight
    t0 = time.perf_counter()
    f0.record(stream)
    for _ in range(e2e_steps):
        zc = H.znorm(ctx, H.encode_column(ctx, xin), B)
        H.decode_column(ctx, zc, out=hzn)
    f1.record(stream)
    barrier_sync()
    seq_wall_ms = 1e3 * (time.perf_counter() - t0)
    seq_ms = f0.elapsed_time(f1)
    # steady state: encode step k+1 while step k computes (every step still copies its input
    # H2D and its result D2H inside the timed region)
    t0 = time.perf_counter()
    f0.record(stream)
    col = H.encode_column(ctx, xin)
    for k_ in range(e2e_steps):
        zc = H.znorm(ctx, col, B)
        col = H.encode_column(ctx, xin) if k_ + 1 < e2e_steps else None
        H.decode_column(ctx, zc, out=hzn)
    f1.record(stream)
    barrier_sync()
    e2e_wall_ms = 1e3 * (time.perf_counter() - t0)
    e2e_ms = f0.elapsed_time(f1)
    e2e_ok = bool(np.array_equal(bits(hzn), bits(ref.out)))
    # one ciphertext per step over the asynchronous calls (encode k+1 | znorm k | decode k, waits for k's
    # verdict and k-2's slots); four pinned buffer pairs rotate
    hxs = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy() for _ in range(4)]
    hzs = [torch.zeros(S, dtype=torch.float64).pin_memory().numpy() for _ in range(4)]

    def single_async(steps):
        col_, pe_ = H.encode_column_async(ctx, hxs[0])
        dq_ = []
        for k_ in range(steps):
            zc_ = H.znorm(ctx, col_, B)
            pk_ = pe_
            if k_ + 1 < steps:
                col_, pe_ = H.encode_column_async(ctx, hxs[(k_ + 1) % 4])
            dq_.append(H.decode_column_async(ctx, zc_, hzs[k_ % 4]))
            pk_.wait()
            while len(dq_) > 2:
                dq_.pop(0).wait()
        while dq_:
            dq_.pop(0).wait()

    single_async(50)
    barrier_sync()
    t0 = time.perf_counter()
    single_async(e2e_steps)
    barrier_sync()
    sa_wall_ms = 1e3 * (time.perf_counter() - t0)
    sa_ok = all(bool(np.array_equal(bits(b_), bits(ref.out))) for b_ in hzs)
    # the same pipelined loop from pageable (ordinary numpy) host buffers: the library stages them
    px = np.array(x)
    pz = np.empty(S)
    col = H.encode_column(ctx, px)
    for k_ in range(20):
        zc = H.znorm(ctx, col, B)
        col = H.encode_column(ctx, px)
        H.decode_column(ctx, zc, out=pz)
    del col, zc
    barrier_sync()
    t0 = time.perf_counter()
    f0.record(stream)
    col = H.encode_column(ctx, px)
    for k_ in range(e2e_steps):
        zc = H.znorm(ctx, col, B)
        col = H.encode_column(ctx, px) if k_ + 1 < e2e_steps else None
        H.decode_column(ctx, zc, out=pz)
    f1.record(stream)
    barrier_sync()
    pg_wall_ms = 1e3 * (time.perf_counter() - t0)
    pg_ms = f0.elapsed_time(f1)
    pg_ok = bool(np.array_equal(bits(pz), bits(ref.out)))

    # ---- e2e (headline): KB ciphertexts per step through the public API from pinned host memory --
    # Per step: encode_column_async of the step's KB x 2^15 values (one 16 MiB H2D DMA + one encrypt
    # launch on an upload stream), each chunk its own single-chunk column, znorm_batch (ordered
    # behind the upload on the device), decode_column_async of the KB result chunks as one column
    # (one 16 MiB D2H DMA on the download stream); the host waits for step k's finiteness verdict
    # and step k-2's results while step k computes, so both copy engines and the SMs stay busy.
    # Every step's input is copied H2D and its whole result D2H inside the timed region; host
    # buffers rotate over NBUF pinned pairs.
    NBUF = 4
    XB = [torch.empty(KB * S, dtype=torch.float64).pin_memory() for _ in range(NBUF)]
    ZB = [torch.empty(KB * S, dtype=torch.float64).pin_memory() for _ in range(NBUF)]
    xbn, zbn = [t_.numpy() for t_ in XB], [t_.numpy() for t_ in ZB]
    for b_ in xbn:
        for j in range(KB):
            b_[j * S:(j + 1) * S] = np.roll(x, 97 * j)

    def benc(i):
        big, pend = H.encode_column_async(ctx, xbn[i % NBUF])
        return [H.EncryptedColumn([c], S) for c in big.chunks], pend

    def bdec(zs, i):
        return H.decode_column_async(ctx, H.EncryptedColumn([zc_.chunks[0] for zc_ in zs], KB * S), zbn[i % NBUF])

    def e2e_loop(steps):
        col_, pe = benc(0)
        dq = []
        for k_ in range(steps):
            zs_ = H.znorm_batch(ctx, col_, B)  # ordered behind encode k on the device
            pk = pe
            if k_ + 1 < steps:
                col_, pe = benc(k_ + 1)
            dq.append(bdec(zs_, k_))
            pk.wait()  # encode k's finiteness verdict
            while len(dq) > 2:
                dq.pop(0).wait()  # step k-2's results are in host memory
        while dq:
            dq.pop(0).wait()

    e2e_loop(max(args.warmup, 24))  # also grows the stream-ordered pool to the loop's working set
    for b_ in zbn:
        b_[:] = 0.0
    barrier_sync()
    be2e_steps = max(50, args.steps // 4)  # the pipeline's fill and drain are inside the timed region
    t0 = time.perf_counter()
    f0.record(stream)
    e2e_loop(be2e_steps)
    f1.record(stream)
    barrier_sync()
    be2e_wall_ms = 1e3 * (time.perf_counter() - t0)
    be2e_ms = max(f0.elapsed_time(f1), be2e_wall_ms)  # events bracket the loop on the compute stream; the
    # last results land on the download stream, which the final wait() has already drained
    be2e_ok = all(bool(np.array_equal(bits(b_[:S]), bits(ref.out))) for b_ in zbn)
    # the round-2 synchronous loop for comparison (encode k+1 beside znorm_batch k, decode k serial)
    def benc_sync():
        return [H.EncryptedColumn([c], S) for c in H.encode_column(ctx, xbn[0]).chunks]

    def bdec_sync(zs):
        H.decode_column(ctx, H.EncryptedColumn([zc_.chunks[0] for zc_ in zs], KB * S), out=zbn[0])

    bcol = benc_sync()
    for _ in range(5):
        zs_ = H.znorm_batch(ctx, bcol, B)
        bcol = benc_sync()
        bdec_sync(zs_)
    barrier_sync()
    t0 = time.perf_counter()
    for k_ in range(be2e_steps):
        zs_ = H.znorm_batch(ctx, bcol, B)
        bcol = benc_sync()
        bdec_sync(zs_)
    barrier_sync()
    be2e_sync_wall_ms = 1e3 * (time.perf_counter() - t0)
    del bcol, zs_
    # the same pipeline from a C++ host over the drop-in headers (tests/dropin/ext_pipeline.cpp,
    # built by build(); it checks its results against decode_column(znorm(encode_column(x))))
    cpp_e2e = None
    cpp_bin = os.path.join(ROOT, "build", "ext_pipeline_gpu")
    if ws == 1 and os.path.exists(cpp_bin):
        barrier_sync()
        try:
            r_ = subprocess.run([cpp_bin, str(S), str(KB), str(max(be2e_steps, 40))], capture_output=True, text=True,
                                timeout=300)
            if r_.returncode == 0 and "ext_pipeline ok" in r_.stdout:
                cpp_e2e = float(r_.stdout.split("steps,")[1].split("us/ciphertext")[0]) / 1e3
        except (OSError, ValueError, IndexError, subprocess.TimeoutExpired):
            cpp_e2e = None

    # ---- kernel roofline: the fused inverse-sqrt program (dominant phase) -------------------
    # Both probes replay CUDA graphs of `reps` calls (device time only).
    m = H.moments(ctx, pool[0], B)
    var = m.ct_var

    def graph_us(fn, reps=50):
        for i in range(3):
            fn(i)
        H.sync()
        with H.Graph() as g:
            for i in range(reps):
                r = fn(i)
                del r
        g.launch()
        barrier_sync()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        g.launch()
        g1.record(stream)
        barrier_sync()
        return 1e3 * g0.elapsed_time(g1) / reps

    prog_us = graph_us(lambda i: H.crypto_invsqrt(ctx, var, B * B))
    mom_us = graph_us(lambda i: H.moments(ctx, pool[i % POOL], B))
    # FP64 pipe instructions per slot of crypto_invsqrt (degree 511, 6 iterations) in the
    # grid-unit formulation of quant.cuh: mul_ct 3, mul_pt 2, add_pt 2, add/sub 1
    mul_ct, mul_pt, add_pt, add_ct = 263 + 18, 256 + 6 + 1, 256 + 8 + 1, 255 + 8 + 6
    fp64_per_slot = 3 * mul_ct + 2 * mul_pt + 2 * add_pt + add_ct
    prog_achieved = fp64_per_slot * S / (prog_us * 1e-6) / 1e12
    # the step kernel (k_stat, one launch per znorm) adds to the invsqrt program, per slot:
    # phase A moment terms (3 mul_pt + 1 mul_ct = 9), their exact sums (sum and |sum| of 3 terms = 6),
    # the variance (sub + mul_ct = 4) and z = (x - mu) * inv (sub + mul_ct = 4)
    step_per_slot = fp64_per_slot + 9 + 6 + 4 + 4
    from paper_2508_12093_b200 import _abi
    import ctypes
    rate = ctypes.c_double(0)
    _abi.lib().hs_diag_fp64_rate(0, ctypes.byref(rate))
    peak = rate.value / 1e12

    # ---- debug_checks = true (the reference CLI's / acceptance runner's default): checked fusion ----
    # (device predicates + one 4-byte flag read per call) vs the op-by-op debug path (set_fused(False))
    ctxd = H.EvalContext(H.CkksParams(slot_count=S, debug_checks=True), rng_seed=rank)
    refd = oracle().stat(Params(slot_count=S, debug_checks=True), ST_ZNORM, x, B)

    def debug_loop(reps):
        for i in range(2):
            H.znorm(ctxd, pool[i % POOL], B)
        barrier_sync()
        l0 = H.kernel_launches()
        t0_ = time.perf_counter()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        for i in range(reps):
            zc = H.znorm(ctxd, pool[i % POOL], B)
        d1.record(stream)
        barrier_sync()
        zz = H.decode_column(ctxd, H.znorm(ctxd, pool[0], B))
        return (1e3 * (time.perf_counter() - t0_) / reps, d0.elapsed_time(d1) / reps,
                (H.kernel_launches() - l0) / (reps + 1), bool(np.array_equal(bits(zz), bits(refd.out))))

    dbg_wall, dbg_dev, dbg_launch, dbg_ok = debug_loop(50)
    H.set_fused(False)
    obo_wall, obo_dev, obo_launch, obo_ok = debug_loop(3)
    H.set_fused(True)
    debug_line = {"metric": "C2 znorm with debug_checks=true, ms per call (public API, host-timed)",
                  "checked_fusion": {"wall_ms": dbg_wall, "device_ms": dbg_dev, "launches_per_call": dbg_launch,
                                     "matches_oracle": dbg_ok},
                  "op_by_op": {"wall_ms": obo_wall, "device_ms": obo_dev, "launches_per_call": obo_launch,
                               "matches_oracle": obo_ok},
                  "note": "checked fusion: the reference's value checks as device predicates in the one "
                          "statistics kernel, one 4-byte flag read per call; a failing check replays the call op "
                          "by op (the reference's error and meter)"}

    # ---- C4: all 28 Pearson pairs of 8 columns (reference semantics: 28 pearson calls) ----------
    cols8 = W.c4_table(H.synthetic_uniform)  # 8 x 32768, pairwise rho 0.6 (seeded)
    c4_line = None
    if True:
        ctx4 = H.EvalContext(H.CkksParams(slot_count=S), rng_seed=rank)
        enc8 = [H.encode_column(ctx4, c) for c in cols8]
        pairs = [(i, j) for i in range(8) for j in range(i + 1, 8)]
        for i, j in pairs[:3]:
            H.pearson(ctx4, enc8[i], enc8[j], 20.0)
        H.sync()
        with H.Graph() as g4:  # outputs freed inside the graph (a graph's live allocations block a relaunch)
            for i, j in pairs:
                r4 = H.pearson(ctx4, enc8[i], enc8[j], 20.0)
                del r4
        g4.launch()
        barrier_sync()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        g4.launch()
        c1.record(stream)
        barrier_sync()
        c0_c1_graph = c0.elapsed_time(c1)
        r01 = float(ctx4.decrypt(H.pearson(ctx4, enc8[0], enc8[1], 20.0), 1)[0])
        from oracle_abi import ST_PEARSON
        refp = oracle().stat(Params(slot_count=S), ST_PEARSON, cols8[0], 20.0, y=cols8[1])
        # the same table through hs_pearson_table: one launch, one inverse square root per column
        tab = H.pearson_table(ctx4, enc8, 20.0)
        tab_ok = bool(np.array_equal(bits(np.array([float(ctx4.decrypt(tab[0], 1)[0])])), bits(refp.out[:1])))
        del tab
        best = None
        for _ in range(5):
            barrier_sync()
            t0_ = time.perf_counter()
            c0.record(stream)
            tab = H.pearson_table(ctx4, enc8, 20.0)
            c1.record(stream)
            c1.synchronize()
            w_ = 1e3 * (time.perf_counter() - t0_)
            if best is None or w_ < best[0]:
                best = (w_, c0.elapsed_time(c1))
            del tab
        c4_line = {"metric": "C4: 28 Pearson pairs of 8 x 32768 columns, device ms per table (graph replay)",
                   "value": c0_c1_graph, "unit": "ms", "B": 20.0, "rho": 0.6,
                   "pair01_matches_oracle": bool(np.array_equal(bits(np.array([r01])), bits(refp.out[:1]))),
                   "pearson_table": {"wall_ms": best[0], "device_ms": best[1], "pair01_matches_oracle": tab_ok,
                                     "note": "hs_pearson_table: one cooperative launch (8 inverse square roots "
                                             "instead of 56) + a 4-byte flag read; same slots, levels and meter "
                                             "as the 28 calls"}}

    # ---- max over ranks ---------------------------------------------------------------------------
    t = torch.tensor([dev_ms, e2e_ms, seq_ms, bdev_ms, be2e_ms], dtype=torch.float64, device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    dev_ms, e2e_ms, seq_ms, bdev_ms, be2e_ms = (float(v) for v in t)
    if rank == 0:
        value = bdev_ms / (args.steps * KB * ws)
        bstep_us = 1e3 * bdev_ms / args.steps  # one k_zbatch launch per step, CUDA events over the timed region
        bachieved = step_per_slot * S * KB / (bstep_us * 1e-6) / 1e12
        step_us = 1e3 * dev_ms / args.steps  # single call: one k_stat launch per step
        achieved = step_per_slot * S / (step_us * 1e-6) / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": bdev_ms / args.steps, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded N(50,10^2) via mt19937_64 + Box-Muller (paper datasets absent)",
            "config": workload_config({"parallelism": f"replicas x{ws} (no data-path collective)",
                                       "ciphertexts_per_step": KB,
                                       "step": STEP_TEXT}),
            "step_detail": f"{KB} Z-scores through hs_znorm_batch: one k_zbatch launch per step, graph-replayed",
            "parity_vs_oracle": parity and bparity,
            "e2e": {"value": be2e_ms / (be2e_steps * KB * ws), "unit": UNIT, "h2d_bytes_per_step": KB * S * 8,
                    "d2h_bytes_per_step": KB * S * 8, "wall_ms_per_ciphertext": be2e_wall_ms / (be2e_steps * KB),
                    "mode": f"pipelined, {KB} ciphertexts per step, one host thread: encode_column_async of step "
                            f"k+1's {KB} x 2^15 values (16 MiB H2D DMA + encrypt on an upload stream), znorm_batch "
                            "of step k, decode_column_async of its results (16 MiB D2H DMA on the download "
                            "stream), then the waits for step k's finiteness verdict and step k-2's results; "
                            "public API calls only",
                    "cpp_host_ms_per_ciphertext": cpp_e2e,
                    "cpp_host": "the same pipeline from a C++ host over include/hestat/*.hpp "
                                "(build/ext_pipeline_gpu, own process, bit-checked against the blocking calls)",
                    "synchronous_calls_wall_ms_per_ciphertext": be2e_sync_wall_ms / (be2e_steps * KB),
                    "synchronous_calls_mode": "the same step with the reference-shaped blocking calls "
                                              "(encode_column k+1 beside znorm_batch k, decode_column k)",
                    "output_matches_oracle": be2e_ok, "host_buffers": f"pinned (torch pin_memory), {NBUF} rotating pairs"},
            "single_call": {
                "value": dev_ms / (args.steps * ws), "unit": UNIT, "ms_per_step": dev_ms / args.steps,
                "mode": "one znorm call per step (one k_stat launch), graph-replayed",
                "roofline_frac": achieved / peak, "achieved": achieved, "duration_us": step_us},
            "e2e_single_call": {"value": e2e_ms / (e2e_steps * ws), "unit": UNIT, "h2d_bytes_per_step": S * 8,
                    "d2h_bytes_per_step": S * 8, "wall_ms_per_step": e2e_wall_ms / e2e_steps,
                    "mode": "pipelined: encode of step k+1 overlaps znorm of step k (public API calls only)",
                    "latency_ms_per_step": seq_ms / e2e_steps, "latency_wall_ms_per_step": seq_wall_ms / e2e_steps,
                    "output_matches_oracle": e2e_ok, "host_buffers": "pinned (torch pin_memory)",
                    "async_pipeline": {"value": sa_wall_ms / e2e_steps, "output_matches_oracle": sa_ok,
                                       "mode": "encode_column_async k+1 | znorm k | decode_column_async k, waits "
                                               "for k's verdict and k-2's slots (wall clock)"},
                    "pageable": {"value": pg_ms / e2e_steps, "wall_ms_per_step": pg_wall_ms / e2e_steps,
                                 "host_buffers": "pageable numpy arrays (staged by the library)",
                                 "output_matches_oracle": pg_ok}},
            "gpu_launches": int(blaunches),
            "api_loop_ms_per_step_single_call": api_ms / args.steps,
            "roofline": {"bound": "fp64",
                         "kernel": f"k_zbatch<QGrid,{zbatch_lanes()}> (the step: {KB} fused C2 Z-scores = moments, grid-wide exact "
                                   "sums, invsqrt degree 511 + 6 Newton per ciphertext, (x - mu) * inv)",
                         "achieved": bachieved, "peak": peak, "unit": "TFLOP/s", "frac": bachieved / peak,
                         "traffic": zbatch_traffic(KB), "duration_us": bstep_us,
                         "work": f"{step_per_slot} fp64 ops/slot x {S} slots x {KB} ciphertexts",
                         "peak_source": "measured DMUL rate on this GPU (hs_diag_fp64_rate); "
                                        "MEASURED_PEAKS.json has no FP64 figure",
                         "traffic_source": "profiles/r2_zbatch_ct_ncu.json (ncu --set full, one k_zbatch launch of "
                                           "64 ciphertexts, dram read+write; algorithmic: 16 B per slot and "
                                           "ciphertext, 32 MiB per launch)",
                         "program_kernel": {"kernel": "k_prog<QGrid,2> (crypto_invsqrt alone)",
                                            "duration_us": prog_us, "achieved": prog_achieved,
                                            "frac": prog_achieved / peak,
                                            "work": f"{fp64_per_slot} fp64 ops/slot x {S} slots"}},
            "kernels_us": {"moments_stat_kernel": mom_us, "invsqrt_prog_kernel": prog_us,
                           "note": "graph replay per call, includes ~1-2 us node overhead"},
            "clocks": clk.summary(),
            "debug_checks": debug_line,
        }
        if c4_line is not None:
            line["c4_pearson_table"] = c4_line
        c5 = c5_tier_e(torch, stream, S, args.batch, ops=("mul_ct", "add", "mul_pt", "rotate_1"))
        line["c5_tier_e"] = {"metric": "mul_ct/s (batch of 64 x 2^15 slots)", "value": c5["mul_ct"]["ops_per_s"],
                             "unit": "mul_ct/s", "ops": c5,
                             "l2": "8 distinct input batches (384 MiB for mul_ct) cycled per replay"}
        if not args.no_cpu_baseline and ws == 1:
            line["c5_tier_e"]["cpu_baseline"] = c5_tier_e_cpu(S, args.batch)
        if not args.no_tier_r:
            line["tier_r"] = tier_r_section(torch, stream, args.batch, with_cpu=not args.no_cpu_baseline and ws == 1)
        if not args.no_cpu_baseline and ws == 1:
            cb, cout = cpu_baseline(x)
            cb["parity_vs_gpu"] = bool(np.array_equal(bits(cout), bits(z)))
            line["cpu_baseline"] = cb
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
