import sys, torch
sys.path.insert(0,'.')
from paper_2510_14126_b200 import ops
M,N,K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
w=(torch.randn(N,K,device='cuda')*0.05).to(torch.bfloat16); x=torch.randn(M,K,device='cuda').to(torch.bfloat16)
out=torch.empty(M,N,device='cuda',dtype=torch.bfloat16); ws=ops.GemmWorkspace('cuda')
print("path", ops.gemm_path(M,N,K), flush=True)
ops.gemm(ops.weight_map(w), ops.act_map(x), M, out, ws); torch.cuda.synchronize(); print("ok", M,N,K)
