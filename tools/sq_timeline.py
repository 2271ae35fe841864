"""Per-CTA timeline of the single-query kernel (exp_so/exp_sqt.so, -DMEA_SQ_TIMING build):
start / streaming done / record written / merge done per CTA, relative to the first start."""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2112_05682_b200 import _lib, api
lib = ctypes.CDLL(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "exp_so", "exp_sqt.so"))
for name, (r, args) in _lib.SIGNATURES.items():
    if hasattr(lib, name):
        f = getattr(lib, name); f.restype = r; f.argtypes = args
_lib._lib = lib
B, H, n_k = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1, 1, 1 << 20))]
q = torch.empty((B, H, 64), dtype=torch.bfloat16, device="cuda")
k = torch.empty((B, n_k, H, 64), dtype=torch.bfloat16, device="cuda")
v = torch.empty_like(k)
for t, tid in ((q, 1), (k, 2), (v, 3)):
    api.mea_fill_synthetic(t, 0, tid)
ws = torch.empty(api.mea_single_query_workspace_size(B, H, n_k, 64, api.MEA_BF16), dtype=torch.uint8, device="cuda")
flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), device="cuda")
for it in range(6):
    torch.sum(flush, dim=0, out=sink)
    torch.cuda.synchronize()
    api.mea_single_query_fwd(q, k, v, workspace=ws)
    torch.cuda.synchronize()
n = 148 * 16
buf = (ctypes.c_ulonglong * (8 * n))()
lib.mea_debug_sq_times(buf, n)
a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8).astype(np.int64)
splits = api.mea_single_query_workspace_size  # noqa
nz = a[:, 0] > 0
a = a[nz]
t0 = a[:, 0].min()
r = (a - t0) / 1e3
r[a == 0] = np.nan
print(f"CTAs {len(a)}: start  min {np.nanmin(r[:,0]):.2f} max {np.nanmax(r[:,0]):.2f} us")
print(f"stream done: min {np.nanmin(r[:,1]):.2f} med {np.nanmedian(r[:,1]):.2f} max {np.nanmax(r[:,1]):.2f}")
print(f"record done: min {np.nanmin(r[:,2]):.2f} med {np.nanmedian(r[:,2]):.2f} max {np.nanmax(r[:,2]):.2f}")
print(f"merge done : {np.nanmax(r[:,3]):.2f}")
m = int(np.nanargmax(r[:, 3]))
print(f"merging CTA {m}: record {r[m, 2]:.2f}, ticket taken {r[m, 4]:.2f}, merge loads (thread 0) {r[m, 5]:.2f}, "
      f"done {r[m, 3]:.2f}; last record of any CTA {np.nanmax(r[:, 2]):.2f}")
print("stream done deciles:", np.round(np.nanpercentile(r[:, 1], [0, 10, 25, 50, 75, 90, 100]), 2))
print("per-CTA stream time (done - start) deciles:", np.round(np.nanpercentile(r[:, 1] - r[:, 0], [0, 10, 50, 90, 100]), 2))
order = np.argsort(r[:, 1])
print("slowest CTAs (idx, start, done):", [(int(i), round(float(r[i, 0]), 2), round(float(r[i, 1]), 2)) for i in order[-8:]])
