"""The C-ABI boundary: liblmx.so loads, exports every entry point declared in
include/lmx.h, and fails loudly (no CPU fallback) without a GPU."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "lmx.h")
LIB = os.path.join(ROOT, "paper_1302_4587_b200", "liblmx.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lmx_[a-z0-9_]+)\s*\(", text)))


def test_library_built():
    assert os.path.exists(LIB), "run __graft_entry__.build() first"


def test_every_declared_symbol_is_exported():
    syms = declared_symbols()
    assert len(syms) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (lmx_[a-z0-9_]+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(LIB)
    for s in syms:
        assert getattr(lib, s) is not None


def test_python_binding_covers_header():
    from paper_1302_4587_b200.engine import EXPORTED_SYMBOLS
    assert sorted(EXPORTED_SYMBOLS) == declared_symbols()


def test_abi_version():
    from paper_1302_4587_b200 import load_library
    assert load_library().lmx_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    for other in ("sm_80", "sm_90", "sm_103"):
        assert other + "." not in out.stdout


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    from paper_1302_4587_b200 import Engine, local_max_b200
    from paper_1302_4587_b200.graph import Graph
    with pytest.raises(RuntimeError, match="CUDA"):
        Engine(0)
    g = Graph(3, np.array([0, 1]), np.array([1, 2]), np.array([1.0, 2.0]))
    with pytest.raises(RuntimeError):
        local_max_b200(g, 0)


def test_oracle_not_imported_by_product():
    import paper_1302_4587_b200  # noqa: F401
    pkg = os.path.join(ROOT, "paper_1302_4587_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                # no import, load or link of the checker from the product path
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), f
                assert "liblmx_oracle" not in src and "lmxo_" not in src, f
                assert "oracle/" not in src.replace("oracle/oracle.py:", ""), f


def test_result_types_without_reference():
    """Without locmax on the path the package's own RoundStats still compares
    equal to any object with the same three fields (a locmax.RoundStats)."""
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "from paper_1302_4587_b200 import graph as G\n"
        "assert not G.REFERENCE_TYPES\n"
        "class R:\n"
        "    edges_before, edges_matched, edges_removed = 5, 2, 4\n"
        "assert G.RoundStats(5, 2, 4) == R() and [G.RoundStats(5, 2, 4)] == [R()]\n"
        "import numpy as np\n"
        "m = G.Matching(np.array([2, 0]), np.array([1, 0, -1, -1]))\n"
        "assert m.size == 2 and m.edges == frozenset({0, 2})\n"
    ) % ROOT
    env = dict(os.environ)
    env["PYTHONPATH"] = ""
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
