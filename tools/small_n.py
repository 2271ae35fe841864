import sys, os, statistics, torch
sys.path.insert(0, '/root/repo')
from paper_2112_05682_b200 import api
from synth import gen
dev = 'cuda'
flush = torch.ones(128 << 20, dtype=torch.float32, device=dev); sink = torch.empty((), device=dev)
for lg in (12, 13, 14):
    ns = 1 << lg; H = 16; D = 64
    qs = torch.empty((1, ns, H, D), dtype=torch.bfloat16, device=dev)
    ks, vs_, dos = torch.empty_like(qs), torch.empty_like(qs), torch.empty_like(qs)
    for t, tid in ((qs, gen.TENSOR_Q), (ks, gen.TENSOR_K), (vs_, gen.TENSOR_V), (dos, gen.TENSOR_DO)):
        api.mea_fill_synthetic(t, 0, tid)
    os_, ls_ = torch.empty_like(qs), torch.empty((1, H, ns), dtype=torch.float32, device=dev)
    gs = [torch.empty_like(qs) for _ in range(3)]
    wss = torch.empty(api.mea_attention_bwd_workspace_size(1, H, ns, ns, D, api.MEA_BF16, True), dtype=torch.uint8, device=dev)
    f = lambda: api.mea_attention_fwd(qs, ks, vs_, out=os_, lse=ls_)
    b = lambda: api.mea_attention_bwd(qs, ks, vs_, os_, dos, lse=ls_, dq=gs[0], dk=gs[1], dv=gs[2], workspace=wss)
    for name, fn in (("fwd", f), ("bwd", b)):
        ts = []
        for i in range(12):
            torch.sum(flush, dim=0, out=sink)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(lg, name, " ".join(f"{t:.3f}" for t in ts), flush=True)
