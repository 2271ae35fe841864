"""Sustained-load A/B of forward variants: each variant runs configs[2]'s forward back to back for
SECS seconds (blocks alternate between variants, 3 blocks each). GPU time per call from CUDA events
around batches of 20 calls; SM clock sampled by nvidia-smi in the background (bench.Clocks)."""
import ctypes, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import Clocks
from paper_2112_05682_b200 import _lib, api
libs = sys.argv[1:]
SECS = float(os.environ.get("SECS", "8"))
fns = {}
for path in libs:
    lib = ctypes.CDLL(path)
    for name, (r, args) in _lib.SIGNATURES.items():
        if not hasattr(lib, name): continue
        f = getattr(lib, name); f.restype = r; f.argtypes = args
    fns[path] = lib
q = torch.empty((1, 16384, 16, 64), dtype=torch.bfloat16, device="cuda")
k, v = torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3)): api.mea_fill_synthetic(t, 0, tid)
out = torch.empty_like(q)
res = {p: [] for p in libs}
clk = {p: [] for p in libs}
for blk in range(3):
    for path in libs:
        _lib._lib = fns[path]
        c = Clocks(0)
        c.start()
        t_end = time.time() + SECS
        tot, n = 0.0, 0
        while time.time() < t_end:
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(20):
                api.mea_attention_fwd(q, k, v, out=out)
            e1.record()
            e1.synchronize()
            tot += e0.elapsed_time(e1)
            n += 20
        cl = c.stop()
        res[path].append(tot / n)
        clk[path].append(cl["sm_mhz"])
for path in libs:
    ms = statistics.mean(res[path])
    print(f"{os.path.basename(path):20s} {ms:.3f} ms/call {[round(x, 3) for x in res[path]]}  "
          f"{4 * 16384 * 16384 * 64 * 16 / ms / 1e9:.0f} TFLOP/s  clocks {clk[path]}")
