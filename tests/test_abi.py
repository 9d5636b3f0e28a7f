"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute calls: these run without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pacloud_b200.h"
LIB = ROOT / "paper_2412_03898_b200" / "libpacloud_b200.so"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pc_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared_symbols()
    for must in ("pc_forward_traces", "pc_residual_state_grads",
                 "pc_deform_states", "pc_deform_backward",
                 "pc_adam_segments", "pc_compact_index", "pc_prune_mask"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not LIB.exists():
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(LIB))
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2412_03898_b200 import _lib
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_version_string_without_gpu():
    if not LIB.exists():
        pytest.skip("library not built")
    from paper_2412_03898_b200 import _lib
    lib = _lib.load_library(require_cuda=False)
    assert b"sm_100a" in lib.pc_version()


def test_workspace_queries_are_host_only():
    if not LIB.exists():
        pytest.skip("library not built")
    from paper_2412_03898_b200 import _lib
    lib = _lib.load_library(require_cuda=False)
    assert lib.pc_compact_workspace_bytes(1000) > 0


def test_product_has_no_oracle_dependency():
    """The product package never imports the CPU oracle."""
    pkg = ROOT / "paper_2412_03898_b200"
    for py in pkg.rglob("*.py"):
        src = py.read_text()
        assert "import oracle" not in src and "from oracle" not in src, py
