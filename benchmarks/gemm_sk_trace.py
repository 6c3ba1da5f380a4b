"""Per-CTA timeline of one cluster split-K GEMM (needs a -DCORTEX_SK_TRACE build):
CORTEX_LIB=variants/libcortex_sktrace.so python benchmarks/gemm_sk_trace.py NAME M KS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

from gemm import SHAPES  # noqa: E402
from paper_2510_14126_b200 import ops  # noqa: E402

name, M, ks = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
ops.gemm_set_mode(3)
from paper_2510_14126_b200 import _lib  # noqa: E402

_lib.set_knob("SK_KS", ks)
N, K = SHAPES[name]
w = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
ws = ops.GemmWorkspace("cuda")
wm, xm = ops.weight_map(w), ops.act_map(x)
for _ in range(3):
    ws.ws[15 << 20:].zero_()
    ops.gemm(wm, xm, M, out, ws)
torch.cuda.synchronize()
n_cta = (N // 256) * ks * 2
tr = ws.ws[15 << 20:(15 << 20) + n_cta * 16].view(torch.int64).view(n_cta, 8).cpu()
t0 = int(tr[:, 0][tr[:, 0] > 0].min())
rel = ((tr - t0).float() / 1e3)
print(f"{name} M={M} ks={ks}: CTAs {n_cta}; end-to-end {float(rel[:, 5].max()):.1f} us")
for ev, lab in enumerate(["start", "setup", "acc", "partial", "barrier", "reduced"]):
    col = rel[:, ev]
    print(f"  {lab:8s} min {float(col.min()):7.1f}  median {float(col.median()):7.1f}  "
          f"max {float(col.max()):7.1f}")
