"""SASS opcode histogram of every kernel in libmea.so (cuobjdump -sass): the instructions that
prove the Blackwell-native paths — UTCHMMA / UTCQMMA (tcgen05.mma), UTMALDG / UTMAREDG / UTMASTG
(TMA), LDTM / STTM (tcgen05.ld / st), MUFU.EX2, FFMA2 / FADD2 / FMUL2, F2FP, LDG / STG widths.

    python tools/sass_hist.py [--so paper_2112_05682_b200/libmea.so] [--out profiles/r02_sass_opcodes.json]
"""
import argparse
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = ("UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMAREDG", "UTMASTG", "UTMAPF", "LDTM", "STTM",
        "MUFU.EX2", "FFMA2", "FADD2", "FMUL2", "FFMA", "F2FP", "SHFL", "SYNCS", "ELECT", "LDG", "STG",
        "LDS", "STS", "REDG", "ATOMG", "BAR", "ACQBULK", "USETMAXREG")


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        return name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", default=os.path.join(ROOT, "paper_2112_05682_b200", "libmea.so"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sass_opcodes.json"))
    a = ap.parse_args()
    txt = subprocess.run(["cuobjdump", "-sass", a.so], capture_output=True, text=True, check=True).stdout
    kernels, cur = {}, None
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = demangle(m.group(1))
            cur = re.sub(r"\(anonymous namespace\)::", "", cur)
            kernels[cur] = collections.Counter()
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            op = m.group(1)
            kernels[cur]["_total"] += 1
            for k in KEEP:
                if op == k or op.startswith(k + "."):
                    # keep the width / form suffix for memory ops and MUFU, the bare opcode otherwise
                    key = op if k in ("LDG", "STG", "MUFU.EX2", "LDS", "STS", "REDG") else k
                    kernels[cur][key] += 1
                    break
    out = {"so": os.path.relpath(a.so, ROOT), "tool": "cuobjdump -sass (static instruction counts, not dynamic)",
           "kernels": {k: dict(sorted(v.items())) for k, v in sorted(kernels.items())}}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    for k, v in sorted(kernels.items()):
        short = {x: v[x] for x in ("UTCHMMA", "UTMALDG", "UTMAREDG", "LDTM", "STTM", "MUFU.EX2", "FFMA2") if v[x]}
        print(k[:90], short)


if __name__ == "__main__":
    main()
