"""Boundary hygiene (CPU): the product path never reaches the oracle and fails loudly without
its CUDA library; the oracle and the CUDA path share no code."""
import ast
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1707_01007_b200")


def _py_imports(path):
    tree = ast.parse(open(path).read())
    mods = set()
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            mods |= {a.name.split(".")[0] for a in node.names}
        elif isinstance(node, ast.ImportFrom) and node.module:
            mods.add(node.module.split(".")[0])
    return mods


def test_product_package_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            p = os.path.join(dirpath, f)
            if f.endswith(".py"):
                assert "oracle" not in _py_imports(p), p
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                src = open(p).read()
                assert not re.search(r'#include\s*[<"][^>"]*oracle', src), p
                assert "oracle_" not in src, p   # no oracle symbol is called or linked


def test_oracle_shares_no_code_with_the_cuda_path():
    odir = os.path.join(ROOT, "oracle")
    for f in os.listdir(odir):
        p = os.path.join(odir, f)
        if f.endswith(".py"):
            mods = _py_imports(p)
            assert "paper_1707_01007_b200" not in mods, p
        if f.endswith((".cpp", ".h", ".cu")):
            src = open(p).read()
            assert "cfpq_internal" not in src and "cfpq.h" not in src, p


def test_binding_fails_loudly_without_the_library(tmp_path):
    """With libcfpq.so absent, the first call raises instead of falling back to anything."""
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "from paper_1707_01007_b200 import cfpq as C\n"
        "C.LIB_PATH = %r\n"
        "try:\n"
        "    C.Grammar(2, 1, [], [[0, 0]])\n"
        "except ImportError as e:\n"
        "    print('raised', e)\n"
        "else:\n"
        "    print('no error')\n" % (ROOT, str(tmp_path / "missing" / "libcfpq.so")))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert "raised" in out.stdout, (out.stdout, out.stderr[-1000:])


def test_bench_and_smoke_are_the_only_oracle_users_outside_tests():
    """Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / reference arm) may
    touch oracle/ (task contract ③)."""
    allowed = {"__graft_entry__.py", "bench.py"}
    for f in os.listdir(ROOT):
        if f.endswith(".py") and f not in allowed:
            assert "oracle" not in _py_imports(os.path.join(ROOT, f)), f
