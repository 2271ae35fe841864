"""Per-source-line warp-stall attribution from an ncu report captured with --import-source on
(`ncu -i REP --page source --print-source cuda,sass`): top lines by stall samples.

    python tools/ncu_stalls.py gpurun_out/prof_fwd_r01c.ncu-rep [--top 30]
"""
import argparse
import collections
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()
txt = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
fname = ""
hdr = None
line = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 5:
        continue
    if r[0]:
        line = (fname, r[0])
        src[line] = r[1].strip()
    if line is None:
        continue
    for i, c in enumerate(hdr):
        if i >= len(r):
            break
        if c == "Warp Stall Sampling (All Samples)" or (c.startswith("stall_") and "Not Issued" not in c):
            try:
                agg[line][c] += float(r[i] or 0)
            except ValueError:
                pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values()) or 1
top = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[: a.top]
for (f, ln), c in top:
    st = sorted(((v, k[6:]) for k, v in c.items() if k.startswith("stall_")), reverse=True)[:3]
    print(f"{f}:{ln:>5} {100 * c['Warp Stall Sampling (All Samples)'] / tot:5.2f}%  {src.get((f, ln), '')[:70]:70s} "
          + " ".join(f"{k}={100 * v / tot:.2f}" for v, k in st if v))
