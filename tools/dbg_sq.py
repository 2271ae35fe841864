import faulthandler, sys, os
faulthandler.dump_traceback_later(40, exit=True)
sys.path.insert(0, os.getcwd())
import torch
from paper_2112_05682_b200 import api
print("ws", api.mea_single_query_workspace_size(1, 1, 1, 64, 1), flush=True)
q = torch.randn(1, 1, 64, device="cuda").bfloat16()
k = torch.randn(1, 1, 1, 64, device="cuda").bfloat16()
v = torch.randn(1, 1, 1, 64, device="cuda").bfloat16()
print("launch", flush=True)
o = api.mea_single_query_fwd(q, k, v, out_dtype=torch.float32)
print("launched", flush=True)
torch.cuda.synchronize()
print("done", o[0, 0, :4], v[0, 0, 0, :4], flush=True)
