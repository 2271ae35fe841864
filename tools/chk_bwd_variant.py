import ctypes, os, sys, math
sys.path.insert(0, '/root/repo')
import torch, numpy as np
from paper_2112_05682_b200 import _lib, api
lib = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _lib.SIGNATURES.items():
    f = getattr(lib, name); f.restype = res; f.argtypes = args
_lib._lib = lib
import oracle as O
from tests import helpers as Hh
q, k, v, do = Hh.host_inputs(1, 300, 257, 2, 64, seed=21, with_dout=True)
qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
out, lse = api.mea_attention_fwd(qd, kd, vd, want_lse=True)
dq, dk, dv = api.mea_attention_bwd(qd, kd, vd, out, dod, lse=lse)
rq, rk, rv = O.mha_backward(q, k, v, do, 1/8)
print("dq err", np.abs(dq.double().cpu().numpy() - rq).max())
