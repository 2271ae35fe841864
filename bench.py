#!/usr/bin/env python
"""Benchmark of the hot path: exact chunked attention (arXiv 2112.05682) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mea|reference]
                    [--n N] [--heads H] [--dim D] [--dtype bf16|f32] [--query-chunk QC] [--key-chunk KC]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself under
torch.distributed.run with N ranks (one process per GPU, NCCL); under torchrun, WORLD_SIZE must
equal --gpus.

One STEP = one pass of the whole hot path over one batch of synthetic inputs:
  forward  (mea_attention_fwd, lse saved)          - SURVEY 8(a) F0-F8
  backward (mea_attention_bwd, recompute from lse)  - SURVEY 8(a) B1-B7
at BASELINE.json configs[2]/[3] shapes (B=1 per GPU, H=16, n=16384, d=64, bf16). The metric
is attention TFLOP/s = (4 + 10) * n^2 * d * H * B / time (BASELINE.json north_star flop
convention). Weak scaling: every rank processes its own batch element (no collective on
the data path), value = all ranks' flops / max-over-ranks time.

Also measured in the same run (extra keys): forward alone (bf16 and the paper's fp32 output),
backward alone, causal, d = 128, the paper's literal key-chunk schedule (q_chunk 1024 /
k_chunk 4096), a small vs-n sweep with scratch bytes, the single-query path at configs[1]
(n = 2^20, HBM-bound) and a decode batch (16 heads x 2^20 keys) against the copy peak and a
read-only HBM probe measured in the run, configs[4] (B=8 H=16 n=2^20) strong-scaled over the
ranks, query-chunk sharding (B*H = 1 < ranks), key-sharded single query / self-attention (one
NCCL all-gather of packed triples), the float64 oracle on the host cores (cpu_baseline) and the
end-to-end number through the public API with host buffers (e2e).

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events on the
launching stream with a 512 MiB L2 flush (read) before each step outside the events;
barrier + synchronize around the timed loop; the max over ranks is reported.
"""
import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DEF, H_DEF, D_DEF = 16384, 16, 64
SQ_NK = 1 << 20                   # configs[1]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["mea", "reference"], default="mea")
    ap.add_argument("--workload", choices=["cfg3", "cfg5"], default="cfg3",
                    help="cfg3: the headline fwd+bwd step; cfg5: configs[4] forward as the step")
    ap.add_argument("--n", type=int, default=N_DEF, help="sequence length (n_q = n_k) of the headline step")
    ap.add_argument("--heads", type=int, default=H_DEF)
    ap.add_argument("--dim", type=int, default=D_DEF, choices=[64, 128])
    ap.add_argument("--dtype", choices=["bf16", "f32"], default="bf16",
                    help="f32: exact fp32 inputs (SIMT forward only)")
    ap.add_argument("--query-chunk", type=int, default=0, help="paper's query chunk for the headline forward")
    ap.add_argument("--key-chunk", type=int, default=0, help="paper's key chunk (0: online, no key split)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the configs[4] strong-scaling extra")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--fwd-only", action="store_true", help="time the forward pass alone as the step")
    ap.add_argument("--no-extras", action="store_true",
                    help="only the headline step (e.g. for an ncu launch list whose shares match the step)")
    return ap.parse_args()


EXTRA_IDLE_S = 0.3   # idle before each extra's timing (tmean)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(a):
    """--gpus N > 1 outside torchrun: start N ranks (one per GPU) with torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        mp = json.load(open(path))
        return {"tflops": mp["bf16_tflops"], "tflops_sustained": mp.get("bf16_tflops_sustained"),
                "hbm_gbs": mp["hbm_gbs"], "sm_max_mhz": mp.get("sm_max_mhz", 1965.0),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"tflops": 1590.0, "tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "sm_max_mhz": 1965.0,
                "source": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
            except (ValueError, IndexError):
                continue
            for nm, val in zip(names, r[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- reference arm
def oracle_sample(rows, n=N_DEF, d=D_DEF, seed=0, heads=1, H=H_DEF):
    """Float64 oracle (oracle/) on a bounded sample of the workload: `heads` heads, the first
    `rows` query rows of each against all n keys; forward (naive, O1) + backward (O6).
    Returns (seconds, algorithmic flops of the sample)."""
    import numpy as np
    import oracle as O
    from synth import gen
    shape = (1, n, H, d)
    secs = 0.0
    for h in range(heads):
        q = gen.rows_of(shape, seed, gen.TENSOR_Q, 0, np.arange(rows), h)
        k = gen.rows_of(shape, seed, gen.TENSOR_K, 0, np.arange(n), h)
        v = gen.rows_of(shape, seed, gen.TENSOR_V, 0, np.arange(n), h)
        do = gen.rows_of(shape, seed, gen.TENSOR_DO, 0, np.arange(rows), h)
        t0 = time.perf_counter()
        O.naive(q, k, v, 1 / math.sqrt(d))
        O.backward(q, k, v, do, 1 / math.sqrt(d))
        secs += time.perf_counter() - t0
    return secs, 14 * rows * n * d * heads


def arm_metric_config(a, run_bwd, world, Bl, Hl, n, d):
    """The metric string and config dict both arms report (the reference arm times the oracle
    on a sample of this same workload)."""
    default = (n, Hl, d, a.dtype, a.query_chunk, a.key_chunk) == (N_DEF, H_DEF, D_DEF, "bf16", 0, 0)
    if a.workload == "cfg5":
        wl = "cfg5: self-attention fwd B=8 H=16 n=2^20 d=64 bf16, sharded over the ranks"
    elif default:
        wl = "cfg3+cfg4: self-attention fwd+bwd (recompute from lse), B=1/GPU H=16 n=16384 d=64 bf16"
    else:
        wl = (f"custom: self-attention {'fwd' if not run_bwd else 'fwd+bwd'} B=1/GPU H={Hl} n={n} d={d} {a.dtype}"
              f" q_chunk={a.query_chunk} k_chunk={a.key_chunk}")
    metric = ("attention TFLOP/s (fwd 4*n^2*d + bwd 10*n^2*d per head)" if run_bwd
              else "attention TFLOP/s (fwd 4*n^2*d per head)")
    config = {"workload": wl, "B_per_gpu": Bl, "H": Hl, "n": n, "d": d, "global_batch": Bl * world,
              "seq_len": n, "parallelism": f"dp{world} (batch x head sharding, no collective)",
              "l2": "flushed before every timed step (512 MiB read, outside the events)"}
    return metric, config


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(a):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0     # the oracle is one host process: the other ranks exit without work
    rows = 2048
    n, H, d = a.n, a.heads, a.dim
    for _ in range(a.warmup):
        oracle_sample(rows, n=n, d=d, seed=a.seed, H=H)
    times, flops = [], 0
    for _ in range(a.steps):
        t, flops = oracle_sample(rows, n=n, d=d, seed=a.seed, H=H)
        times.append(t)
    ms = statistics.mean(times) * 1e3
    val = flops / (ms * 1e-3) / 1e12
    sample = (f"float64 oracle (naive fwd O1 + analytic bwd O6): 1 of {H} heads, {rows} of {n} query rows "
              f"vs all {n} keys, d={d}, per step, one host process")
    metric, config = arm_metric_config(a, True, world, 1, H, n, d)   # the mea arm's metric and config
    line = {"impl": "reference", "metric": metric, "value": val,
            "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (counter-based Irwin-Hall(12), N(0,1)-like, PAPER.md:231)",
            "config": config,
            "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "host_processes": 1}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- mea arm
def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(a)
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != a.gpus:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}", file=sys.stderr)
        return 2
    if a.impl == "reference":
        return run_reference(a)
    if a.dtype == "f32":
        a.fwd_only = True

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    distributed = "WORLD_SIZE" in os.environ    # launched by torchrun (also with one rank)
    if distributed:
        # communicator set-up visible in the log (stderr, so stdout keeps one JSON line)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import torch
    import torch.distributed as dist
    if distributed:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2112_05682_b200 import api
    from paper_2112_05682_b200 import dist as mdist
    from synth import gen

    def barrier():
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if not distributed:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    D = a.dim
    tdt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
    if a.workload == "cfg5":
        B_glob, n, H = 8, 1 << 20, 16     # configs[4]: B=8 H=16 n=2^20, batch elements over the ranks
        assert B_glob % world == 0
        Bl, Hl = B_glob // world, H
    else:
        Bl, Hl, n = 1, a.heads, a.n       # weak scaling: one batch element per rank
    flop_fwd = 4 * n * n * D * Hl * Bl
    flop_bwd = 10 * n * n * D * Hl * Bl
    run_bwd = a.workload == "cfg3" and not a.fwd_only

    shape = (Bl, n, Hl, D)
    numel = Bl * n * Hl * D
    q = torch.empty(shape, dtype=tdt, device=dev)
    k, v = torch.empty_like(q), torch.empty_like(q)
    do = torch.empty_like(q) if run_bwd else None
    for t, tid in ((q, gen.TENSOR_Q), (k, gen.TENSOR_K), (v, gen.TENSOR_V), (do, gen.TENSOR_DO)):
        if t is not None:
            api.mea_fill_synthetic(t, a.seed, tid, offset=rank * numel)   # rank r = batch element r
    out = torch.empty_like(q)
    lse = torch.empty((Bl, Hl, n), dtype=torch.float32, device=dev)
    dq, dk, dv = (torch.empty_like(q) for _ in range(3)) if run_bwd else (None, None, None)
    bwd_ws = None
    if run_bwd:
        nb = api.mea_attention_bwd_workspace_size(Bl, Hl, n, n, D, api.MEA_BF16, True)
        bwd_ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    fwd_ws = None
    if a.query_chunk or a.key_chunk:
        nb = api.mea_attention_fwd_workspace_size(Bl, Hl, n, n, D, api.MEA_BF16 if a.dtype == "bf16" else api.MEA_F32,
                                                  a.query_chunk, a.key_chunk)
        fwd_ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
    # L2 flush by READING 512 MiB (> 126 MB L2): a write-based flush would leave ~126 MB of
    # dirty lines whose write-back steals HBM bandwidth from the next timed kernel.
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
    flush_sink = torch.empty((), dtype=torch.float32, device=dev)

    def flush_l2():
        torch.sum(flush, dim=0, out=flush_sink)

    def fwd():
        api.mea_attention_fwd(q, k, v, out=out, lse=lse, q_chunk=a.query_chunk, k_chunk=a.key_chunk,
                              workspace=fwd_ws)

    def step():
        fwd()
        if run_bwd:
            api.mea_attention_bwd(q, k, v, out, do, lse=lse, dq=dq, dk=dk, dv=dv, workspace=bwd_ws)

    def timed(fn, steps, warmup, flush_each=True):
        for _ in range(warmup):
            fn()
        barrier()
        evs = []
        for _ in range(steps):
            if flush_each:
                flush_l2()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            evs.append((e0, e1))
        barrier()
        return [e0.elapsed_time(e1) for e0, e1 in evs]

    def tmean(fn, steps, warmup=1):
        """median event time of fn over `steps` (ms), max over ranks (the extras: a median, so one
        stalled call among a few does not move the number; the headline step keeps its own timing).
        Each extra starts after EXTRA_IDLE_S of idle, so it meets the board in the state the headline
        step starts in, not in the power cap the previous extra drove it into (measured: the causal
        forward 0.74 ms right after the other extras, 0.62 ms from idle)."""
        torch.cuda.synchronize()
        time.sleep(EXTRA_IDLE_S)
        return max_over_ranks(statistics.median(timed(fn, steps, warmup)))

    # ---------------- the timed step (headline)
    for _ in range(a.warmup):
        step()
    barrier()
    clocks = Clocks(local)
    clocks.start()
    api.profile_enable(True)
    api.profile_read()
    step_ms = timed(step, a.steps, 0)
    prof = api.profile_read()
    api.profile_enable(False)
    clk = clocks.stop()
    total_ms = max_over_ranks(sum(step_ms))
    ms_per_step = total_ms / a.steps
    flops_step = flop_fwd + (flop_bwd if run_bwd else 0)
    value = world * flops_step / (ms_per_step * 1e-3) / 1e12
    gpu_launches = sum(c for c, _ in prof.values())

    pk = peaks()
    kernels = {}
    for name, (cnt, ms) in prof.items():
        kernels[name] = {"launches": cnt, "avg_ms": ms / cnt}
    # dominant kernel: the largest share of the step
    dom = max(prof.items(), key=lambda kv: kv[1][1])[0]
    dom_flops = {"fwd_bf16": flop_fwd, "fwd128_bf16": flop_fwd, "bwd_bf16": flop_bwd}.get(dom)
    dom_ms = kernels[dom]["avg_ms"]
    achieved = dom_flops / (dom_ms * 1e-3) / 1e12 if dom_flops else None
    traffic = None
    if a.workload == "cfg3" and (n, Hl, D) == (N_DEF, H_DEF, D_DEF):   # ncu captures at configs[2]/[3]
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
            traffic = tr.get(dom)
        except Exception:
            pass
    roofline = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": pk["tflops"], "unit": "TFLOP/s",
                "frac": (achieved / pk["tflops"]) if achieved else None, "traffic": traffic,
                "peak_source": pk["source"] + " bf16 dense burst",
                "frac_of_sustained": (achieved / pk["tflops_sustained"]) if achieved and pk["tflops_sustained"]
                else None,
                "per_launch_flops": dom_flops}

    extras = {}
    standard = a.workload == "cfg3" and (n, Hl, D, a.dtype) == (N_DEF, H_DEF, D_DEF, "bf16")
    if not a.no_extras and a.workload == "cfg3":
        # ---------------- HBM: read-only probe (the single query's roofline) + single query + decode batch,
        # measured first among the extras, before the compute-bound extras heat the board into its
        # power cap (the latency-bound parts of a 50 us call run on the SM clock), and after a short
        # idle so the headline step's power-cap clock has recovered (decode-shaped calls do not run
        # on a board that has just drawn 1 kW for the training step)
        torch.cuda.synchronize()
        time.sleep(0.5)
        buf = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
        probe_ms = statistics.median(timed(lambda: api.debug_read_probe(buf, 296), 10, 2))
        read_gbs = buf.numel() / (probe_ms * 1e-3) / 1e9
        del buf

        def sq_case(Bq, Hq, nk):
            sq_q = torch.empty((Bq, Hq, D), dtype=torch.bfloat16, device=dev)
            sq_k = torch.empty((Bq, nk, Hq, D), dtype=torch.bfloat16, device=dev)
            sq_v = torch.empty_like(sq_k)
            for t, tid in ((sq_q, gen.TENSOR_Q), (sq_k, gen.TENSOR_K), (sq_v, gen.TENSOR_V)):
                api.mea_fill_synthetic(t, a.seed, tid)
            sq_o = torch.empty((Bq, Hq, D), dtype=torch.bfloat16, device=dev)
            sq_ws = torch.empty(api.mea_single_query_workspace_size(Bq, Hq, nk, D, api.MEA_BF16), dtype=torch.uint8,
                                device=dev)
            call = lambda: api.mea_single_query_fwd(sq_q, sq_k, sq_v, out=sq_o, workspace=sq_ws)
            call_ms = statistics.median(timed(call, max(a.steps, 20), 2))   # launch profiler off
            api.profile_enable(True)
            api.profile_read()
            timed(call, max(a.steps, 20), 2)
            sp = api.profile_read()
            api.profile_enable(False)
            kern_ms = sp["sq_fused"][1] / sp["sq_fused"][0]
            nbytes = 2 * Bq * Hq * nk * D * 2 + 2 * Bq * Hq * D * 2
            gbs = nbytes / (call_ms * 1e-3) / 1e9
            return {"B": Bq, "H": Hq, "n_k": nk, "call_us": call_ms * 1e3, "kernel_us_events": kern_ms * 1e3,
                    "launches_per_call": sum(c for c, _ in sp.values()) / max(1, sp["sq_fused"][0]),
                    "gbs": gbs, "frac_hbm_copy_peak": gbs / pk["hbm_gbs"], "frac_hbm_read_probe": gbs / read_gbs,
                    "scratch_bytes": sq_ws.numel()}

        sq = sq_case(1, 1, SQ_NK)
        sq.update({"peak_gbs": pk["hbm_gbs"], "peak_source": "MEASURED_PEAKS.json copy (read + write)",
                   "read_probe_gbs": read_gbs,
                   "read_probe": "1 GiB streamed by the library's read-only probe kernel (296 CTAs x 512 threads, "
                                 "16-B non-caching loads), median of 10, L2 flushed"})
        extras["single_query_cfg2"] = sq
        extras["single_query_decode_batch"] = sq_case(1, 16, SQ_NK)
        extras["hbm_read_probe_gbs"] = read_gbs
    if not a.no_extras and a.workload == "cfg3":
        # ---------------- forward alone (bf16 out, and the paper's fp32 output), backward alone
        fwd_ms = tmean(fwd, max(3, a.steps // 2))
        extras["fwd"] = {"ms": fwd_ms, "tflops": flop_fwd / (fwd_ms * 1e-3) / 1e12,
                         "frac": flop_fwd / (fwd_ms * 1e-3) / 1e12 / pk["tflops"]}
        if D == 64 and a.dtype == "bf16":
            # the d = 64 forward's own roofline is the exponential unit (2 exps per 256 flops):
            # 16 ex2 / clk / SM (tools/micro/exp_throughput.cu measured 16.4) x 148 SMs x the max SM clock
            exps = flop_fwd / (4 * D)
            exp_peak = 16 * 148 * pk["sm_max_mhz"] * 1e6
            extras["fwd"]["exp_roofline"] = {
                "bound": "alu (MUFU ex2)", "achieved": exps / (fwd_ms * 1e-3) / 1e12, "peak": exp_peak / 1e12,
                "unit": "Tex2/s", "frac": exps / (fwd_ms * 1e-3) / exp_peak,
                "peak_basis": "16 exp/clk/SM x 148 SMs x %d MHz (max SM clock); 1 of 24 exponential pairs runs on "
                              "the FMA pipe, so the frac can exceed the MUFU-only reading" % pk["sm_max_mhz"]}
            # with the scores' TMEM load and the P store each tile also needs (.16x256b / .16x128b shapes), the
            # exponential loop runs at 16.3 cycles per pair per SM sub-partition (tools/micro/mio_mix.cu): the
            # kernel's practical floor
            pairs_per_smsp = exps / 64 / (148 * 4)   # warp-wide pairs: 32 lanes x 2 exponentials
            floor_ms = pairs_per_smsp * 16.3 / (pk["sm_max_mhz"] * 1e6) * 1e3
            extras["fwd"]["exp_roofline"].update({"practical_floor_ms": floor_ms, "frac_of_practical_floor": floor_ms / fwd_ms,
                                                  "practical_floor_basis": "16.3 cycles per exp pair per SMSP incl. "
                                                  "the per-tile tcgen05.ld of S (.16x256b) / st of P (.16x128b), at the max SM clock"})
        if a.dtype == "bf16":
            out32 = torch.empty(shape, dtype=torch.float32, device=dev)
            f32_ms = tmean(lambda: api.mea_attention_fwd(q, k, v, out=out32, lse=lse), max(3, a.steps // 2))
            extras["fwd_f32_out"] = {"ms": f32_ms, "tflops": flop_fwd / (f32_ms * 1e-3) / 1e12,
                                     "frac": flop_fwd / (f32_ms * 1e-3) / 1e12 / pk["tflops"],
                                     "setting": "bf16 q/k/v, float32 output: the paper's Table 1 setting (P:219)"}
            del out32
        if run_bwd:
            bwd_ms = tmean(lambda: api.mea_attention_bwd(q, k, v, out, do, lse=lse, dq=dq, dk=dk, dv=dv,
                                                         workspace=bwd_ws), max(3, a.steps // 2))
            extras["bwd"] = {"ms": bwd_ms, "tflops": flop_bwd / (bwd_ms * 1e-3) / 1e12,
                             "frac": flop_bwd / (bwd_ms * 1e-3) / 1e12 / pk["tflops"]}
            # B0: the backward without lse (stats recomputed), its workspace
            ws0 = torch.empty(api.mea_attention_bwd_workspace_size(Bl, Hl, n, n, D, api.MEA_BF16, False),
                              dtype=torch.uint8, device=dev)
            b0_ms = tmean(lambda: api.mea_attention_bwd(q, k, v, out, do, lse=None, dq=dq, dk=dk, dv=dv,
                                                        workspace=ws0), 3)
            extras["bwd_lse_recomputed"] = {"ms": b0_ms, "workspace_bytes": ws0.numel(),
                                            "workspace_bytes_with_lse": bwd_ws.numel()}
            del ws0
    if not a.no_extras and standard:
        # ---------------- causal masking: flops of the visible (i, j <= i) pairs only
        if run_bwd:
            vis = n * (n + 1) / 2 * D * Hl * Bl
            cf_ms = tmean(lambda: api.mea_attention_fwd_causal(q, k, v, out=out, lse=lse), max(3, a.steps // 2))
            cb_ms = tmean(lambda: api.mea_attention_bwd_causal(q, k, v, out, do, lse=lse, dq=dq, dk=dk, dv=dv,
                                                               workspace=bwd_ws), max(3, a.steps // 2))
            extras["causal"] = {"fwd_ms": cf_ms, "fwd_tflops": 4 * vis / (cf_ms * 1e-3) / 1e12,
                                "bwd_ms": cb_ms, "bwd_tflops": 10 * vis / (cb_ms * 1e-3) / 1e12,
                                "flops": "visible pairs only: 4 (fwd) / 10 (bwd) x n(n+1)/2 x d x H"}
        # ---------------- head dimension 128: configs[2]'s B, H, n
        q128 = torch.empty((Bl, n, Hl, 128), dtype=torch.bfloat16, device=dev)
        k128, v128 = torch.empty_like(q128), torch.empty_like(q128)
        for t, tid in ((q128, gen.TENSOR_Q), (k128, gen.TENSOR_K), (v128, gen.TENSOR_V)):
            api.mea_fill_synthetic(t, a.seed, tid, offset=rank * q128.numel())
        o128 = torch.empty_like(q128)
        l128 = torch.empty((Bl, Hl, n), dtype=torch.float32, device=dev)
        f128_ms = tmean(lambda: api.mea_attention_fwd(q128, k128, v128, out=o128, lse=l128), max(3, a.steps // 2))
        fl128 = 4 * n * n * 128 * Hl * Bl
        extras["fwd_d128"] = {"ms": f128_ms, "tflops": fl128 / (f128_ms * 1e-3) / 1e12,
                              "frac": fl128 / (f128_ms * 1e-3) / 1e12 / pk["tflops"], "kernel": "fwd128_bf16"}
        if run_bwd:
            do128 = torch.empty_like(q128)
            api.mea_fill_synthetic(do128, a.seed, gen.TENSOR_DO, offset=rank * do128.numel())
            g128 = [torch.empty_like(q128) for _ in range(3)]
            ws128 = torch.empty(api.mea_attention_bwd_workspace_size(Bl, Hl, n, n, 128, api.MEA_BF16, True),
                                dtype=torch.uint8, device=dev)
            b128_ms = tmean(lambda: api.mea_attention_bwd(q128, k128, v128, o128, do128, lse=l128, dq=g128[0],
                                                          dk=g128[1], dv=g128[2], workspace=ws128),
                            max(3, a.steps // 2))
            extras["bwd_d128"] = {"ms": b128_ms, "tflops": 2.5 * fl128 / (b128_ms * 1e-3) / 1e12,
                                  "frac": 2.5 * fl128 / (b128_ms * 1e-3) / 1e12 / pk["tflops"]}
            del do128, g128, ws128
        del q128, k128, v128, o128, l128
        # ---------------- the paper's literal schedule (query chunk 1024 / key chunk 4096)
        ws_kc = api.mea_attention_fwd_workspace_size(Bl, Hl, n, n, D, api.MEA_BF16, 1024, 4096)
        wsb = torch.empty(ws_kc, dtype=torch.uint8, device=dev)
        kc_ms = tmean(lambda: api.mea_attention_fwd(q, k, v, out=out, lse=lse, q_chunk=1024, k_chunk=4096,
                                                    workspace=wsb), 3)
        extras["fwd_paper_chunks_qc1024_kc4096"] = {"ms": kc_ms, "tflops": flop_fwd / (kc_ms * 1e-3) / 1e12,
                                                    "scratch_bytes": ws_kc}
        del wsb
        # ---------------- vs n (the metric's axis): fwd / bwd TFLOP/s and scratch bytes
        sweep = []
        for lg in (12, 13, 14, 15, 16):
            ns = 1 << lg
            qs = torch.empty((1, ns, Hl, D), dtype=torch.bfloat16, device=dev)
            ks, vs_, dos = torch.empty_like(qs), torch.empty_like(qs), torch.empty_like(qs)
            for t, tid in ((qs, gen.TENSOR_Q), (ks, gen.TENSOR_K), (vs_, gen.TENSOR_V), (dos, gen.TENSOR_DO)):
                api.mea_fill_synthetic(t, a.seed, tid)
            os_, ls_ = torch.empty_like(qs), torch.empty((1, Hl, ns), dtype=torch.float32, device=dev)
            gs = [torch.empty_like(qs) for _ in range(3)]
            wss = torch.empty(api.mea_attention_bwd_workspace_size(1, Hl, ns, ns, D, api.MEA_BF16, True),
                              dtype=torch.uint8, device=dev)
            it = 5 if lg <= 14 else 2
            fm = tmean(lambda: api.mea_attention_fwd(qs, ks, vs_, out=os_, lse=ls_), it)
            bm = tmean(lambda: api.mea_attention_bwd(qs, ks, vs_, os_, dos, lse=ls_, dq=gs[0], dk=gs[1], dv=gs[2],
                                                     workspace=wss), it)
            ff = 4 * ns * ns * D * Hl
            sweep.append({"n": ns, "fwd_ms": fm, "fwd_tflops": ff / (fm * 1e-3) / 1e12,
                          "bwd_ms": bm, "bwd_tflops": 2.5 * ff / (bm * 1e-3) / 1e12,
                          "fwd_scratch_bytes": 0, "bwd_scratch_bytes": wss.numel(),
                          "lse_residual_bytes": ls_.numel() * 4,
                          "standard_fwd_bytes": ns * ns * Hl * 4, "standard_bwd_bytes": 2 * ns * ns * Hl * 4})
            del qs, ks, vs_, dos, os_, ls_, gs, wss
        extras["vs_n"] = {"B": 1, "H": Hl, "d": D, "rows": sweep}
    if not a.no_extras:
        # ---------------- configs[4]: B=8 H=16 n=2^20 forward, strong scaling over the ranks
        if not a.no_cfg5 and D == 64 and a.dtype == "bf16":
            B5, H5, n5 = 8, 16, 1 << 20
            plan = mdist.shard_plan(B5, H5, n5, world, rank)
            (b0, b1), (h0, h1), (r0, r1) = plan["b"], plan["h"], plan["q"]
            Bq5, Hq5 = b1 - b0, h1 - h0
            q5 = torch.empty((Bq5, r1 - r0, Hq5, D), dtype=torch.bfloat16, device=dev)
            k5 = torch.empty((Bq5, n5, Hq5, D), dtype=torch.bfloat16, device=dev)
            v5 = torch.empty_like(k5)
            for t, tid in ((q5, gen.TENSOR_Q), (k5, gen.TENSOR_K), (v5, gen.TENSOR_V)):
                api.mea_fill_synthetic(t, a.seed, tid, offset=rank * t.numel())
            o5 = torch.empty_like(q5)
            l5 = torch.empty((Bq5, Hq5, r1 - r0), dtype=torch.float32, device=dev)
            c5_ms = max_over_ranks(timed(lambda: api.mea_attention_fwd(q5, k5, v5, out=o5, lse=l5), 1, 0)[0])
            fl5 = 4 * n5 * n5 * D * B5 * H5
            extras["cfg5_strong"] = {"B": B5, "H": H5, "n": n5, "n_gpus": world, "shard": plan["mode"],
                                     "per_rank": {"B": Bq5, "H": Hq5, "q_rows": r1 - r0}, "ms": c5_ms,
                                     "tflops_total": fl5 / (c5_ms * 1e-3) / 1e12,
                                     "frac_per_gpu": fl5 / (c5_ms * 1e-3) / 1e12 / world / pk["tflops"],
                                     "steps": 1, "collective": "none (rows independent, PAPER.md:68-70)"}
            del q5, k5, v5, o5, l5
        # ---------------- query-chunk sharding: B*H = 1 < ranks (strong scaling, K/V replicated)
        if D == 64 and a.dtype == "bf16":
            nq1 = 1 << 18
            plan = mdist.shard_plan(1, 1, nq1, world, rank)
            r0, r1 = plan["q"]
            qq = torch.empty((1, r1 - r0, 1, D), dtype=torch.bfloat16, device=dev)
            kq = torch.empty((1, nq1, 1, D), dtype=torch.bfloat16, device=dev)
            vq = torch.empty_like(kq)
            api.mea_fill_synthetic(qq, a.seed, gen.TENSOR_Q, offset=r0 * D)   # the global tensor's rows r0..r1
            api.mea_fill_synthetic(kq, a.seed, gen.TENSOR_K)
            api.mea_fill_synthetic(vq, a.seed, gen.TENSOR_V)
            oq = torch.empty_like(qq)
            qc_ms = tmean(lambda: api.mea_attention_fwd(qq, kq, vq, out=oq), 3)
            flq = 4 * nq1 * nq1 * D
            extras["query_chunk_sharded"] = {"B": 1, "H": 1, "n": nq1, "n_gpus": world, "shard": plan["mode"],
                                             "rows_per_rank": r1 - r0, "ms": qc_ms,
                                             "tflops_total": flq / (qc_ms * 1e-3) / 1e12,
                                             "collective": "none (K/V replicated, query rows split)"}
            del qq, kq, vq, oq
        # ---------------- key-sharded single query: per-rank packed triples, ONE NCCL all-gather, merge
        if D == 64 and a.dtype == "bf16":
            Bq, Hq, n_local = 1, 16, SQ_NK
            sq_q = torch.empty((Bq, Hq, D), dtype=torch.bfloat16, device=dev)
            sq_k = torch.empty((Bq, n_local, Hq, D), dtype=torch.bfloat16, device=dev)
            sq_v = torch.empty_like(sq_k)
            api.mea_fill_synthetic(sq_q, a.seed, gen.TENSOR_Q)
            api.mea_fill_synthetic(sq_k, a.seed, gen.TENSOR_K, offset=rank * sq_k.numel())
            api.mea_fill_synthetic(sq_v, a.seed, gen.TENSOR_V, offset=rank * sq_v.numel())
            sws = torch.empty(api.mea_single_query_workspace_size(Bq, Hq, n_local, D, api.MEA_BF16),
                              dtype=torch.uint8, device=dev)
            run = lambda: mdist.sharded_single_query(sq_q, sq_k, sq_v, workspace=sws)
            sh_ms = tmean(run, max(5, a.steps // 3), 2)
            gb = world * 2 * n_local * Hq * D * 2 / 1e9
            extras["single_query_key_sharded"] = {
                "keys_total": n_local * world, "heads": Hq, "n_gpus": world, "ms": sh_ms,
                "gbs_total": gb / (sh_ms * 1e-3),
                "collective": "one all_gather_into_tensor of packed (v*, m*, s*) records per (b,h), NCCL"
                              if world > 1 else "none (one rank)"}
            del sq_k, sq_v
        # ---------------- key-range sharded self-attention (long context beyond one GPU)
        if distributed and world > 1 and a.workload == "cfg3" and D == 64 and a.dtype == "bf16":
            lo, hi = mdist.shard_range(n, world, rank)
            q_all = torch.empty_like(q)                 # the same query rows on every rank (batch element 0)
            api.mea_fill_synthetic(q_all, a.seed, gen.TENSOR_Q)
            k_loc = torch.empty((Bl, hi - lo, Hl, D), dtype=torch.bfloat16, device=dev)
            v_loc = torch.empty_like(k_loc)             # this rank's key range of batch element 0
            api.mea_fill_synthetic(k_loc, a.seed, gen.TENSOR_K, offset=lo * Hl * D)
            api.mea_fill_synthetic(v_loc, a.seed, gen.TENSOR_V, offset=lo * Hl * D)
            run = lambda: mdist.sharded_self_attention(q_all, k_loc, v_loc)
            sa_ms = tmean(run, max(3, a.steps // 3))
            extras["self_attention_key_sharded"] = {
                "n": n, "heads": Hl, "keys_per_rank": hi - lo, "ms": sa_ms,
                "tflops_total": flop_fwd / (sa_ms * 1e-3) / 1e12,
                "exchange_bytes_per_rank": Bl * n * Hl * (D + 4) * 4,
                "collective": "one all_gather_into_tensor of packed per-row (v*, m*, s*) records, NCCL"}
            del q_all, k_loc, v_loc
    # ---------------- scratch bytes vs the paper's accounting (standard attention: n^2*4 B/head)
    scratch = {"fwd_workspace_bytes": fwd_ws.numel() if fwd_ws is not None else 0,
               "fwd_lse_residual_bytes": lse.numel() * 4,
               "bwd_workspace_bytes": bwd_ws.numel() if bwd_ws is not None else None,
               "standard_attention_fwd_bytes": n * n * 4 * Hl * Bl,
               "standard_attention_bwd_bytes": 2 * n * n * 4 * Hl * Bl}
    torch.cuda.reset_peak_memory_stats(dev)
    base = torch.cuda.memory_allocated(dev)
    step()
    torch.cuda.synchronize()
    scratch["torch_peak_delta_bytes_step"] = torch.cuda.max_memory_allocated(dev) - base

    # ---------------- e2e: through the public API with host buffers (H2D inputs, D2H results)
    # Every step copies its inputs (q, k, v, dO) from pinned host memory and reads its results
    # (out, dq, dk, dv) back. The steps are software-pipelined the way a training input pipeline
    # runs: the H2D copy of step i+1 and the D2H copy of step i-1 run on their own streams while
    # step i computes, with two device buffer sets and events ordering reuse.
    e2e = None
    if not a.no_e2e and a.workload == "cfg3":
        ins = [t for t in (q, k, v, do) if t is not None]
        hin = [t.cpu().pin_memory() for t in ins]
        hout = [torch.empty(shape, dtype=tdt).pin_memory() for _ in range(4 if run_bwd else 1)]
        bufs = [dict(q=q, k=k, v=v, do=do, out=out, lse=lse, dq=dq, dk=dk, dv=dv)]
        bufs.append({nm: (torch.empty_like(t) if t is not None else None) for nm, t in bufs[0].items()})
        ws_e2e = [bwd_ws, torch.empty_like(bwd_ws) if bwd_ws is not None else None]
        s_in, s_c, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_qkv = [torch.cuda.Event() for _ in range(2)]   # q, k, v of a set have landed
        ev_in = [torch.cuda.Event() for _ in range(2)]    # ... and dO
        ev_f = [torch.cuda.Event() for _ in range(2)]     # forward of a set done (out final)
        ev_c = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def e2e_run(steps):
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream(dev)
            start.record(cur)
            for st_ in (s_in, s_c, s_out):
                st_.wait_event(start)
            for i in range(steps):
                bi = i % 2
                S = bufs[bi]
                with torch.cuda.stream(s_in):
                    if i >= 2:
                        s_in.wait_event(ev_c[bi])      # step i-2 has finished reading this set
                    S["q"].copy_(hin[0], non_blocking=True); S["k"].copy_(hin[1], non_blocking=True)
                    S["v"].copy_(hin[2], non_blocking=True)
                    ev_qkv[bi].record(s_in)
                    if run_bwd:
                        S["do"].copy_(hin[3], non_blocking=True)
                    ev_in[bi].record(s_in)
                with torch.cuda.stream(s_c):
                    s_c.wait_event(ev_qkv[bi])         # the forward needs q, k, v only
                    if i >= 2:
                        s_c.wait_event(ev_out[bi])     # step i-2's results have been copied out
                    api.mea_attention_fwd(S["q"], S["k"], S["v"], out=S["out"], lse=S["lse"], q_chunk=a.query_chunk,
                                          k_chunk=a.key_chunk, workspace=fwd_ws)
                    ev_f[bi].record(s_c)
                    if run_bwd:
                        s_c.wait_event(ev_in[bi])
                        api.mea_attention_bwd(S["q"], S["k"], S["v"], S["out"], S["do"], lse=S["lse"], dq=S["dq"],
                                              dk=S["dk"], dv=S["dv"], workspace=ws_e2e[bi])
                    ev_c[bi].record(s_c)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_f[bi])         # out is final once the forward is done
                    hout[0].copy_(S["out"], non_blocking=True)
                    s_out.wait_event(ev_c[bi])
                    if run_bwd:
                        hout[1].copy_(S["dq"], non_blocking=True); hout[2].copy_(S["dk"], non_blocking=True)
                        hout[3].copy_(S["dv"], non_blocking=True)
                    ev_out[bi].record(s_out)
            for st_ in (s_in, s_c, s_out):
                cur.wait_stream(st_)
            end.record(cur)
            return start, end

        e2e_run(max(2, a.warmup))
        barrier()
        e0_, e1_ = e2e_run(a.steps)
        barrier()
        e_ms = max_over_ranks(e0_.elapsed_time(e1_)) / a.steps
        esz = q.element_size()
        h2d = len(ins) * numel * esz
        d2h = len(hout) * numel * esz
        e2e = {"value": world * flops_step / (e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "pipelining": "H2D of step i+1 and D2H of step i-1 overlap step i (3 streams, 2 buffer sets); "
                              "the forward starts once q, k, v have landed and out is read back while the "
                              "backward runs"}
        del bufs, ws_e2e

    # ---------------- cpu baseline: the oracle on the host cores (rank 0, N == 1 only)
    cpu = None
    if world == 1 and not a.no_cpu_baseline:
        rows, heads = 4096, 8    # ~10 s of host work on a 16-core box
        secs, fl = oracle_sample(rows, n=min(n, N_DEF), d=D, seed=a.seed, heads=min(heads, Hl), H=Hl)
        cpu = {"value": fl / secs / 1e12, "unit": "TFLOP/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": f"float64 oracle fwd (O1) + bwd (O6): {min(heads, Hl)} of {Hl} heads x {rows} query rows x "
                         f"{min(n, N_DEF)} keys, d={D} (threads: numpy/OpenBLAS default)",
               "seconds": secs}

    if rank == 0:
        metric, config = arm_metric_config(a, run_bwd, world, Bl, Hl, n, D)
        line = {
            "metric": metric,
            "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16" if a.dtype == "bf16" else "f32",
            "data": "synthetic (counter-based Irwin-Hall(12), N(0,1)-like, PAPER.md:231)",
            "config": config,
            "clocks": clk, "gpu_launches": gpu_launches, "roofline": roofline, "kernels": kernels,
            "cpu_baseline": cpu, "e2e": e2e, "scratch": scratch,
            **({"extras_idle_s": EXTRA_IDLE_S} if extras else {}), **extras,
            "paper_context": {"tpu_v3_fwd_ms_n16384_h1": 11.3, "tpu_v3_diff_ms_n16384_h1": 21.0,
                              "memory_reduction_fwd": "59x", "memory_reduction_diff": "32x"},
        }
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
