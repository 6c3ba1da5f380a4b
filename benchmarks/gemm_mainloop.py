"""Mainloop timing of the 2-SM GEMM from a -DCORTEX_GEMM_TRACE build (globaltimer stamps):
median over pairs of tile 0's accumulator-ready time minus its MMA start, the kernel
span, and the per-launch time.  CORTEX_LIB=variants/libcortex_gtrace*.so
python benchmarks/gemm_mainloop.py NAME M"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

from gemm import SHAPES  # noqa: E402
from paper_2510_14126_b200 import ops  # noqa: E402

name, M = sys.argv[1], int(sys.argv[2])
ops.gemm_set_stream_k(0)
N, K = SHAPES[name]
w = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
ws = ops.GemmWorkspace("cuda")
wm, xm = ops.weight_map(w), ops.act_map(x)
for _ in range(3):
    ws.ws[15 << 20:].zero_()
    ops.gemm(wm, xm, M, out, ws)
torch.cuda.synchronize()
tr = ws.ws[15 << 20:(15 << 20) + 148 * 32].view(torch.int64).view(148, 16).cpu()
t0 = int(tr[tr > 0].min())
acc = sorted((int(tr[c][1]) - int(tr[c][0])) / 1e3 for c in range(0, 148, 2) if tr[c][1] > 0)
span = max((int(v) - t0) / 1e3 for v in tr.flatten().tolist() if v > 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    ops.gemm(wm, xm, M, out, ws)
e1.record()
torch.cuda.synchronize()
tn = ops.lib().cortex_gemm2_tile(M, N, K) & 0xffff
mma_us = (K // 64) * (256 * tn * 64 * 2 / 16384) / 1.965e3
print(f"{os.path.basename(os.environ.get('CORTEX_LIB', 'default'))} {name} M={M} TN={tn}: "
      f"tile-0 mainloop median {acc[len(acc) // 2]:.1f} us (MMA-rate floor {mma_us:.1f} us at "
      f"1.965 GHz), span {span:.1f} us, per launch {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
