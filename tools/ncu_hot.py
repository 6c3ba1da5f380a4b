"""Hot SASS lines of one kernel in an ncu report: python tools/ncu_hot.py REP [N]."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Address" in r)
body = [r for r in rows if r and r[0].startswith("0x") and len(r) == len(hdr)]
f = lambda v: float(v) if v not in ("", "-") else 0.0
si = hdr.index("Warp Stall Sampling (All Samples)")
ni = hdr.index("Warp Stall Sampling (Not-issued Samples)")
tot = sum(f(r[si]) for r in body)
print(f"samples {tot:.0f}  instructions {len(body)}")
top = sorted(range(len(body)), key=lambda i: -f(body[i][si]))[:n]
for i in sorted(top):
    r = body[i]
    print(f"{i:5d} {f(r[si]):6.0f} {100 * f(r[si]) / tot:5.1f}%  {r[1].strip()[:80]}")
