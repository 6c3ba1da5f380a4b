"""One FMHA launch of a chosen shape (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmha  # noqa: E402
kind = sys.argv[1] if len(sys.argv) > 1 else "prefill"
if kind == "prefill":
    print(fmha.prefill(0, [8192]))
else:
    print(fmha.cascade(8192, 128))
