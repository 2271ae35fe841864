import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_2112_05682_b200 import _lib, api
lib = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _lib.SIGNATURES.items():
    if not hasattr(lib, name): continue
    f = getattr(lib, name); f.restype = res; f.argtypes = args
_lib._lib = lib
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64   # d = 128 (or DET=1): the two-kernel path's dK/dV kernel
q = torch.empty((1, 16384, 16, d), dtype=torch.bfloat16, device="cuda")
k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)): api.mea_fill_synthetic(t, 0, tid)
out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
dv = torch.zeros_like(q)
fn = api.mea_attention_bwd_deterministic if os.environ.get("DET") == "1" else api.mea_attention_bwd
for _ in range(2): fn(q, k, v, out, do, lse=lse, dv=dv)
torch.cuda.synchronize()
raw = dv.view(torch.int64).flatten()[:512 + 16 * 8].cpu().numpy().astype(np.int64)
ts = raw[:512].reshape(4, 16, 8)
mm = raw[512:].reshape(16, 8)
base = ts[0, 0, 0]
names = ["wait_S", "compute", "wait_pfree", "store+arrive"]
for g in range(4):
    for i in range(3):
        r = ts[g, i, :5] - base
        print(f"g{g} i={i+8}", " ".join(f"{x:7d}" for x in r), "| dt:", " ".join(f"{n}={x}" for n, x in zip(names, np.diff(r))))

sub = ts[:, :, [3, 5, 6, 7, 4]]
dd = np.diff(sub, axis=2).mean(axis=1)
print("store phase split (p_free seen -> tmem_st issued -> STS done -> proxy fence done -> st_wait+arrive):")
for g in range(4):
    print(f"  g{g} " + " ".join(f"{x:.0f}" for x in dd[g]))
print("softmax means over 16 tiles (cycles):")
for g in range(4):
    dd = np.diff(ts[g, :, :5], axis=1).mean(axis=0)
    per = np.diff(ts[g, :, 0]).mean()
    print(f"  g{g} period {per:7.0f} | " + " ".join(f"{n}={x:.0f}" for n, x in zip(names, dd)))
if d != 64 or os.environ.get("DET") == "1":
    sys.exit(0)   # the dK/dV kernel has no MMA-warp probes
mn = ["wait_qdo", "wait_s_loaded", "wait_p_full(+issue S)", "wait_dq_empty(+issue dV dK)"]
print("MMA warp means (cycles):", " ".join(f"{n}={x:.0f}" for n, x in zip(mn, np.diff(mm[:, :5], axis=1).mean(axis=0))),
      f"period {np.diff(mm[:, 0]).mean():.0f}")
for i in range(4):
    print("  MMA", i + 8, " ".join(f"{x - base:7d}" for x in mm[i, :5]))
