import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import torch
from test_prefill_attention_gpu import _setup
c, kv = _setup(torch, 8, 128, 300, seed=300)
q = (torch.randn(300, 64, 128, device="cuda") * 0.5).to(torch.bfloat16)
out = torch.empty_like(q)
c.paged_prefill_attention_async(1, (0, 300), 0, 64, 8, 128, 128**-0.5, q.data_ptr(), out.data_ptr(), 0)
torch.cuda.synchronize(); print("ok")
