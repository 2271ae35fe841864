"""BASELINE.json's metric swept over n: attention TFLOP/s and % of bf16 peak vs n, and scratch bytes
vs n (SURVEY.md §8(d) "n-sweep"), on one B200.

    python tools/sweep.py [--out profiles/r01_sweep.json] [--max-log2n 18]

Rows:
  * self-attention forward (default schedule, and the paper's q_chunk 1024 / k_chunk 4096 key-split
    schedule) and backward (fused default and deterministic), B=1 H=16 d=64 bf16, n = 2^10 .. 2^18;
  * single query, B=H=1 d=64 bf16, n_k = 2^16 .. 2^24 (HBM GB/s of the K+V stream).
Each row: device time (median of CUDA-event-timed calls, 512 MiB L2 read-flush before each call,
outside the events), TFLOP/s (fwd 4 n^2 d H, bwd 10 n^2 d H — algorithmic, PAPER.md/BASELINE.json),
% of the measured peak (MEASURED_PEAKS.json), and scratch: the torch peak-allocation delta of the
call with outputs pre-allocated (= the library workspace, PAPER.md:220's definition), next to the
analytic standard-attention score matrix n^2 H 4 B (fwd) / 2 n^2 H 4 B (bwd).
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import Clocks, peaks as bench_peaks  # noqa: E402
from paper_2112_05682_b200 import api  # noqa: E402

H, D = 16, 64


def peaks():
    pk = bench_peaks()
    return pk["tflops"], pk["hbm_gbs"]


def sweep_one(n, lg, d, rows, fill, scratch, timed, peak_tf):
    """Forward (default and, at d = 64, the paper's chunk schedule) and both backward entry
    points at B = 1, H = 16, head dimension d."""
    q, k, v, do = (fill((1, n, H, d), t) for t in (1, 2, 3, 4))
    dev = q.device
    out = torch.empty_like(q)
    lse = torch.empty((1, H, n), dtype=torch.float32, device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ffl, bfl = 4.0 * n * n * d * H, 10.0 * n * n * d * H
    cases = [
        ("fwd", "default (online, no key split)", ffl, lambda: api.mea_attention_fwd(q, k, v, out=out, lse=lse)),
        ("bwd", "mea_attention_bwd" + (" (fused, dQ by TMA reduce-add)" if d == 64 else " (two kernels at d = 128)"),
         bfl, lambda: api.mea_attention_bwd(q, k, v, out, do, lse=lse, dq=dq, dk=dk, dv=dv)),
        ("bwd", "deterministic (dK/dV + dQ kernels)", bfl,
         lambda: api.mea_attention_bwd_deterministic(q, k, v, out, do, lse=lse, dq=dq, dk=dk, dv=dv)),
    ]
    if d == 64 and n > 4096:
        cases.insert(1, ("fwd", "paper q_chunk=1024 k_chunk=4096 (key split + merge)", ffl,
                         lambda: api.mea_attention_fwd(q, k, v, out=out, lse=lse, q_chunk=1024, k_chunk=4096)))
    api.mea_attention_fwd(q, k, v, out=out, lse=lse)
    for kind, sched, fl, fn in cases:
        sb = scratch(fn)
        med, mn, it = timed(fn, budget_s=1.0 if lg <= 16 else 3.0)
        tf = fl / (med * 1e-3) / 1e12
        std = (1 if kind == "fwd" else 2) * n * n * H * 4
        r = {"op": kind, "schedule": sched, "B": 1, "H": H, "n": n, "d": d, "ms_median": round(med, 4),
             "ms_min": round(mn, 4), "iters": it, "tflops": round(tf, 1), "pct_peak": round(100 * tf / peak_tf, 1),
             "scratch_bytes": sb, "standard_attention_scores_bytes": std,
             "reduction_vs_standard": round(std / sb, 1) if sb else None}
        rows.append(r)
        print(json.dumps(r), flush=True)
    del q, k, v, do, out, lse, dq, dk, dv
    torch.cuda.empty_cache()


def sweep_causal(n, lg, rows, fill, scratch, timed, peak_tf):
    """Causal forward / backward at d = 64 (flops of the visible pairs, n(n+1)/2 per head)."""
    q, k, v, do = (fill((1, n, H, D), t) for t in (1, 2, 3, 4))
    out = torch.empty_like(q)
    lse = torch.empty((1, H, n), dtype=torch.float32, device=q.device)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    vis = n * (n + 1) / 2 * D * H
    api.mea_attention_fwd_causal(q, k, v, out=out, lse=lse)
    for kind, fl, fn in (("fwd_causal", 4 * vis, lambda: api.mea_attention_fwd_causal(q, k, v, out=out, lse=lse)),
                         ("bwd_causal", 10 * vis, lambda: api.mea_attention_bwd_causal(q, k, v, out, do, lse=lse, dq=dq,
                                                                                       dk=dk, dv=dv))):
        sb = scratch(fn)
        med, mn, it = timed(fn, budget_s=1.0)
        tf = fl / (med * 1e-3) / 1e12
        r = {"op": kind, "schedule": "causal, visible pairs", "B": 1, "H": H, "n": n, "d": D,
             "ms_median": round(med, 4), "ms_min": round(mn, 4), "iters": it, "tflops": round(tf, 1),
             "pct_peak": round(100 * tf / peak_tf, 1), "scratch_bytes": sb}
        rows.append(r)
        print(json.dumps(r), flush=True)
    del q, k, v, do, out, lse, dq, dk, dv
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_sweep.json"))
    ap.add_argument("--max-log2n", type=int, default=18)
    ap.add_argument("--max-log2nk", type=int, default=24)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    peak_tf, peak_gbs = peaks()
    flush_buf = torch.ones(128 << 20, dtype=torch.float32, device=dev)
    sink = torch.empty((), device=dev)

    def timed(fn, budget_s=1.0):
        fn()  # warm-up (also first-touch of the workspace allocation)
        fn()
        fn()
        torch.cuda.synchronize()
        ts = []
        while len(ts) < 3 or (sum(ts) < budget_s * 1e3 and len(ts) < 50):
            torch.sum(flush_buf, dim=0, out=sink)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts), min(ts), len(ts)

    def scratch(fn):
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
        base = torch.cuda.memory_allocated(dev)
        fn()
        torch.cuda.synchronize()
        return torch.cuda.max_memory_allocated(dev) - base

    def fill(shape, tid, seed=0):
        t = torch.empty(shape, dtype=torch.bfloat16, device=dev)
        api.mea_fill_synthetic(t, seed, tid)
        return t

    rows = []
    clk = Clocks(0)
    clk.start()
    for lg in range(10, a.max_log2n + 1, 2):
        n = 1 << lg
        sweep_one(n, lg, D, rows, fill, scratch, timed, peak_tf)
    for lg in range(10, min(a.max_log2n, 16) + 1, 2):   # d = 128 and causal (d = 64) up to 2^16
        sweep_one(1 << lg, lg, 128, rows, fill, scratch, timed, peak_tf)
        sweep_causal(1 << lg, lg, rows, fill, scratch, timed, peak_tf)
    for lg in range(16, a.max_log2nk + 1, 2):
        n_k = 1 << lg
        q = fill((1, 1, D), 1)
        k, v = fill((1, n_k, 1, D), 2), fill((1, n_k, 1, D), 3)
        o = torch.empty((1, 1, D), dtype=torch.bfloat16, device=dev)
        fn = lambda: api.mea_single_query_fwd(q, k, v, out=o)  # noqa: E731
        sb = scratch(fn)
        med, mn, it = timed(fn, budget_s=0.3)
        byts = 2 * n_k * D * 2
        gbs = byts / (med * 1e-3) / 1e9
        r = {"op": "single_query", "B": 1, "H": 1, "n_k": n_k, "d": D, "us_median": round(med * 1e3, 2),
             "us_min": round(mn * 1e3, 2), "iters": it, "GBps": round(gbs, 0), "pct_peak_hbm": round(100 * gbs / peak_gbs, 1),
             "scratch_bytes": sb, "standard_attention_scores_bytes": n_k * 4}
        rows.append(r)
        print(json.dumps(r), flush=True)
        del q, k, v, o
        torch.cuda.empty_cache()
    clocks = clk.stop()
    res = {"about": __doc__.strip().splitlines()[0], "peak_bf16_tflops": peak_tf, "peak_hbm_GBps": peak_gbs,
           "clocks": clocks, "device": torch.cuda.get_device_name(dev), "rows": rows}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    print("clocks", json.dumps(clocks))


if __name__ == "__main__":
    main()
