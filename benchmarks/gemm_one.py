"""One GEMM shape a few times (for ncu): python benchmarks/gemm_one.py NAME M [SK]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_14126_b200 import ops  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm import SHAPES  # noqa: E402

name, M = sys.argv[1], int(sys.argv[2])
if len(sys.argv) > 3:
    ops.gemm_set_stream_k(int(sys.argv[3]))
N, K = SHAPES[name]
w = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
out = torch.empty(M, N, device="cuda", dtype=torch.float32)
res = torch.randn(M, N, device="cuda")
ws = ops.GemmWorkspace("cuda")
wm, xm = ops.weight_map(w), ops.act_map(x)
for _ in range(4):
    ops.gemm(wm, xm, M, out, ws, residual=res)
torch.cuda.synchronize()
print(name, M, ops.lib().cortex_gemm2_tile(M, N, K))
