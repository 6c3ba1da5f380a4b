"""Build a tuning variant of libcortex_b200.so with extra -D flags into variants/NAME.so
(git-ignored; it travels to the GPU box). Select it with CORTEX_LIB=variants/NAME.so.
Usage: python tools/build_variant.py NAME -DFOO=1 [-DBAR=2 ...]"""

import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_14126_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = b.ROOT / "variants" / f"{name}.so"
out.parent.mkdir(exist_ok=True)
cmd = [b._nvcc(), *b.NVCC_FLAGS, *defs, f"-I{b.INCLUDE}", f"-I{b.CSRC}", "-o", str(out),
       *map(str, b.sources())]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-4000:])
print(out)
