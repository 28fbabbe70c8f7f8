"""CPU-only checks of the C-ABI boundary: the library loads, exports exactly what
include/cfpq.h declares, and validates grammar input on the host (no GPU needed)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "cfpq.h")).read()
    return sorted(set(re.findall(r"CFPQ_API\s+[\w\s\*]*?\b(cfpq_\w+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_1707_01007_b200 import build
    build.build()
    from paper_1707_01007_b200 import cfpq as C
    lib = C.load()
    decl = _declared()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(C.EXPORTS) == decl
    assert "sm_100a" in C.version()


def test_grammar_validation_on_host():
    from paper_1707_01007_b200 import cfpq as C
    g = C.Grammar(3, 2, [[0, 1, 2]], [[1, 0], [2, 1]])
    assert g._h
    with pytest.raises(C.CfpqError) as e:
        C.Grammar(3, 2, [[0, 1, 3]], [])
    assert e.value.status == C.CFPQ_E_INVAL
    with pytest.raises(C.CfpqError):
        C.Grammar(3, 2, [], [[0, 2]])          # label id out of range
    with pytest.raises(C.CfpqError):
        C.Grammar(0, 2, [], [])                # no NTs
    with pytest.raises(C.CfpqError):
        C.Grammar(2000, 2, [], [])             # more than 1024 NTs


def test_sass_has_no_legacy_tensor_or_fallback():
    """The closure kernel is CUDA-core bitwise/atomic code compiled for sm_100a."""
    import subprocess
    lib = os.path.join(ROOT, "paper_1707_01007_b200", "libcfpq.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
