"""CPU-only: the C-ABI library loads and exports every symbol include/pgk.h
declares; the product has no CPU fallback and never imports the oracle."""
import ast
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "pgk.h"
PKG = ROOT / "paper_2410_01231_b200"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(pgk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2410_01231_b200 import _lib
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(pgk_[a-z0-9_]+)", out))
    assert set(syms) <= exported
    assert set(_lib.EXPORTS) <= exported


def test_library_is_sm100a():
    from paper_2410_01231_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_without_gpu():
    import torch
    from paper_2410_01231_b200 import _lib
    assert _lib.lib().pgk_version().startswith(b"pgk")
    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError):
            _lib.device()


def test_product_never_imports_oracle():
    for p in PKG.rglob("*.py"):
        tree = ast.parse(p.read_text())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert not any(a.name.split(".")[0] == "oracle" for a in node.names), p
            if isinstance(node, ast.ImportFrom):
                assert (node.module or "").split(".")[0] != "oracle", p


def test_workspace_queries_need_no_gpu():
    import ctypes
    from paper_2410_01231_b200 import _lib
    b = ctypes.c_size_t(0)
    assert _lib.lib().pgk_reverse_workspace(1000, 24, ctypes.byref(b)) == 0
    assert b.value > 1000 * 24 * 2 * 8
    assert _lib.lib().pgk_knn_workspace(1000, 1000, 32, 64, 0, ctypes.byref(b)) == 0
    assert b.value >= 1000 * 64 * 8
