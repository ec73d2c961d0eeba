import torch
X=torch.randn(4095,4096,device="cuda",dtype=torch.bfloat16); W=torch.randn(4096,53248,device="cuda",dtype=torch.bfloat16); Y=torch.empty(4095,53248,device="cuda",dtype=torch.bfloat16)
for _ in range(3): torch.matmul(X,W,out=Y)
torch.cuda.synchronize()
