import torch, sys
sys.path.insert(0,'.')
from paper_2112_05682_b200 import api
q=torch.randn(1,300,2,64,device='cuda').bfloat16(); k=torch.randn(1,700,2,64,device='cuda').bfloat16()
o=api.mea_attention_fwd(q,k,k); torch.cuda.synchronize(); print("ok", o.float().abs().mean().item())
