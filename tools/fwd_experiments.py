"""Time forward-kernel variants (separate .so builds, tools/build_variant.sh) at configs[2]
(B=1, H=16, n=16384, d=64 bf16). Calls are interleaved variant by variant (A B C A B C ...) so
every variant sees the same clock / power state; outputs are compared with the first variant's.

    ITERS=60 python tools/fwd_experiments.py exp_so/exp_a.so exp_so/exp_b.so [...]
"""
import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import _lib, api

libs = sys.argv[1:]
dev = torch.device("cuda", 0)
H = 16
q = torch.empty((1, 16384, H, 64), dtype=torch.bfloat16, device=dev)
k, v = torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3)):
    api.mea_fill_synthetic(t, 0, tid)
outs = {p: torch.empty_like(q) for p in libs}
lse = torch.empty((1, H, 16384), dtype=torch.float32, device=dev)
FLUSH = os.environ.get("FLUSH", "0") == "1"   # 512 MiB read before every call (bench.py's protocol)
flush = torch.ones(128 << 20, dtype=torch.float32, device=dev) if FLUSH else None
sink = torch.empty((), dtype=torch.float32, device=dev)
fns = {}
for path in libs:
    lib = ctypes.CDLL(path)
    for name, (r, args) in _lib.SIGNATURES.items():
        if not hasattr(lib, name): continue
        f = getattr(lib, name); f.restype = r; f.argtypes = args
    fns[path] = lib


def call(path):
    _lib._lib = fns[path]
    api.mea_attention_fwd(q, k, v, out=outs[path], lse=lse)


res = {p: [] for p in libs}
ITERS = int(os.environ.get("ITERS", "40"))
for i in range(ITERS + 2):
    for path in libs:
        if FLUSH:
            torch.sum(flush, dim=0, out=sink)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); call(path); e1.record()
        torch.cuda.synchronize()
        if i >= 2: res[path].append(e0.elapsed_time(e1))
ref = outs[libs[0]].float()
for path in libs[1:]:
    print(f"{os.path.basename(path)}: max|diff| vs first {(outs[path].float() - ref).abs().max().item():.3e}")
base = statistics.median(res[libs[0]])
for path, ts in res.items():
    ms = statistics.median(ts)
    print(f"{os.path.basename(path):24s} fwd {ms:.3f} ms (min {min(ts):.3f}, {100 * (ms / base - 1):+.1f}%)  "
          f"{4*16384*16384*64*H/ms/1e9:.1f} TFLOP/s")
