"""The ctypes mirrors of cortex_decoder_t / cortex_step_t (paper_2510_14126_b200/_lib.py)
have the C layout of include/cortex_b200.h: every field's offset and both sizes, from a
C program compiled against the header (gcc, no GPU)."""

from __future__ import annotations

import ctypes
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_descriptor_layout_matches_header(tmp_path):
    from paper_2510_14126_b200 import _lib

    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "cortex_b200.h"',
             "int main(void) {"]
    for cname, cls in (("cortex_decoder_t", _lib.DecoderDesc), ("cortex_step_t", _lib.StepDesc)):
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", f"-I{ROOT / 'include'}", "-o", str(exe), str(src)],
                   check=True, capture_output=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out.splitlines()}
    for cname, cls in (("cortex_decoder_t", _lib.DecoderDesc), ("cortex_step_t", _lib.StepDesc)):
        assert got[(cname, "size")] == ctypes.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert got[(cname, f)] == getattr(cls, f).offset, (cname, f)


def test_decoder_layers_rejects_bad_descriptors():
    """Argument validation happens before any CUDA call (runs without a GPU): a missing
    descriptor, an empty step, a layer range outside the model, or no tcgen05 Q map."""
    from paper_2510_14126_b200 import _lib

    lib = _lib.load()
    m, st = _lib.DecoderDesc(), _lib.StepDesc()
    assert lib.cortex_decoder_layers(None, ctypes.byref(st)) == -1
    assert lib.cortex_decoder_layers(ctypes.byref(m), None) == -1
    m.n_layers, m.hq, m.hkv = 2, 8, 2
    st.n_tok, st.n_dec, st.layer_begin, st.layer_end = 4, 4, 0, 2
    assert lib.cortex_decoder_layers(ctypes.byref(m), ctypes.byref(st)) == -1  # no weights
    st.layer_end = 3
    assert lib.cortex_decoder_layers(ctypes.byref(m), ctypes.byref(st)) == -1  # past n_layers
