"""Per-pair event times of one stream-K GEMM (needs a -DCORTEX_GEMM_TRACE build):
CORTEX_LIB=variants/libcortex_trace.so python benchmarks/gemm_trace.py NAME M."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

from paper_2510_14126_b200 import ops  # noqa: E402
from gemm import SHAPES  # noqa: E402

name, M = sys.argv[1], int(sys.argv[2])
ops.gemm_set_stream_k(int(sys.argv[3]) if len(sys.argv) > 3 else 1)
N, K = SHAPES[name]
w = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
res = out if len(sys.argv) > 4 and sys.argv[4] == "res" else None  # in-place residual
ws = ops.GemmWorkspace("cuda")
wm, xm = ops.weight_map(w), ops.act_map(x)
for _ in range(3):
    ws.ws[15 << 20:].zero_()
    ops.gemm(wm, xm, M, out, ws, residual=res)
torch.cuda.synchronize()
tr = ws.ws[15 << 20:(15 << 20) + 148 * 32].view(torch.int64).view(148, 16).cpu()
t0 = int(tr[tr > 0].min())
for cta in range(0, 148, 1):
    ev = [(i, (int(v) - t0) / 1e3) for i, v in enumerate(tr[cta].tolist()) if v > 0]
    if cta % 2 == 0 and cta < 40:
        print("pair", cta // 2, " ".join(f"{i}:{t:.1f}" for i, t in ev))
last = [(max((int(v) - t0) / 1e3 for v in tr[c].tolist() if v > 0), c // 2) for c in range(148)
        if (tr[c] > 0).any()]
last.sort()
print("latest events:", last[-6:], "earliest last:", last[:3])
starts = sorted((int(tr[c][15]) - t0) / 1e3 for c in range(148) if tr[c][15] > 0)
ends13 = sorted((int(tr[c][13]) - t0) / 1e3 for c in range(148) if tr[c][13] > 0)
ends14 = sorted((int(tr[c][14]) - t0) / 1e3 for c in range(148) if tr[c][14] > 0)
print("kernel entry first/last", starts[0], starts[-1], "loop exit first/last", ends13[0], ends13[-1],
      "after syncthreads first/last", ends14[0], ends14[-1])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    ops.gemm(wm, xm, M, out, ws, residual=res)
e1.record()
torch.cuda.synchronize()
print("per launch us", e0.elapsed_time(e1) / 20 * 1e3)
tile2 = ops.lib().cortex_gemm2_tile(M, N, K)
TN = tile2 & 0xffff
tkb = K // 64
tiles = (N // 256) * ((M + TN - 1) // TN)
U = tiles * tkb
P = 74
rows = []
for p in range(P):
    a_, b_ = p * U // P, (p + 1) * U // P
    segs, u = [], a_
    while u < b_:
        t, k0 = divmod(u, tkb)
        k1 = min(tkb, k0 + (b_ - u))
        segs.append((t, k0, k1))
        u += k1 - k0
    ex = (int(tr[2 * p][13]) - t0) / 1e3 if tr[2 * p][13] > 0 else -1
    rows.append((ex, p, segs, [(i, round((int(v) - t0) / 1e3, 1)) for i, v in enumerate(tr[2 * p][:13].tolist()) if v > 0]))
rows.sort()
for r in rows[:3] + rows[-8:]:
    print("exit %.1f pair %d segs %s ev %s" % r)
