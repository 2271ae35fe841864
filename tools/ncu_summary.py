"""Summarise ncu outputs into profiles/: per-kernel key metrics (from --set full reports) and
per-kernel time shares (from a gpu__time_duration launch list).

    python tools/ncu_summary.py --rep gpurun_out/prof_fwd_r01.ncu-rep [...] --launches gpurun_out/launches_r01.csv --out profiles/r01
"""
import argparse
import collections
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active": "tensor_hmma_pct",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tc_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_mufu_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            out[name] = f"{vals[i]} {units[i]}".strip()
    return out


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv:
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[iu], 1.0)
        name = r[ik].split("(")[0].split("::")[-1]
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", "")) * scale
    total = sum(v[1] for v in agg.values())
    return {k: {"launches": v[0], "total_us": round(v[1], 3), "share": round(v[1] / total, 4)}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    res = {"kernels": [raw(r) for r in a.rep]}
    if a.launches:
        res["launch_list"] = launches(a.launches)
    json.dump(res, open(a.out + "_ncu_summary.json", "w"), indent=1)
    print(json.dumps(res, indent=1))
