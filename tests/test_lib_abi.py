"""The C ABI library loads (no GPU needed) and exports every symbol the header declares."""

from __future__ import annotations

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_symbols(path=ROOT / "include" / "cortex_b200.h") -> list[str]:
    text = path.read_text()
    return sorted(set(re.findall(r"^int32_t (cortex_\w+)\(", text, flags=re.M)))


DEV_HEADER = ROOT / "paper_2510_14126_b200" / "csrc" / "cortex_dev.h"


def test_header_matches_binding_table():
    """The public boundary (include/cortex_b200.h) and the private tuning interface
    (csrc/cortex_dev.h) are disjoint and each matches its binding table."""
    from paper_2510_14126_b200 import _lib

    assert header_symbols() == sorted(_lib.SIGNATURES)
    assert header_symbols(DEV_HEADER) == sorted(_lib.DEV_SIGNATURES)
    assert not set(_lib.SIGNATURES) & set(_lib.DEV_SIGNATURES)


def test_library_reads_no_environment():
    """Kernel behaviour is fixed by the build and the knobs of cortex_dev.h, never by
    environment variables read inside the library."""
    for src in (ROOT / "paper_2510_14126_b200" / "csrc").glob("*.cu"):
        assert "getenv" not in src.read_text(), src.name


def test_library_loads_and_exports_everything():
    from paper_2510_14126_b200 import _lib

    if not _lib.LIB_PATH.exists():
        pytest.fail(f"{_lib.LIB_PATH} not built (run python -m paper_2510_14126_b200.build)")
    lib = _lib.load()
    for name in header_symbols() + header_symbols(DEV_HEADER):
        assert hasattr(lib, name), name
    assert lib.cortex_abi_version() == 103
    # pure host helpers are callable without a GPU
    assert lib.cortex_gemm_splits(32, 6144, 4096) >= 1
    assert lib.cortex_decode_splits(1000, 1300) == 3  # 82 tiles in 32-tile splits
    # balanced plan: 2 waves of 55 chunks x 8 kv heads on 148 SMs -> 37 tiles per chunk
    assert lib.cortex_decode_tiles_per_chunk(4000, 8) == 37
    assert lib.cortex_gemm_path(700, 4096, 4096) == 2
    assert lib.cortex_gemm_path(64, 4096, 4096) == 3  # cluster split-K (decode M)
    assert lib.cortex_gemm_path(64, 128256, 4096) == 1  # lm_head: too many tiles to split


def test_no_cpu_fallback_without_library(monkeypatch, tmp_path):
    from paper_2510_14126_b200 import _lib

    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "missing.so")
    monkeypatch.setattr(_lib, "_LIB", None)
    with pytest.raises(ImportError):
        _lib.load()
