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


def build_c_client():
    """gcc the plain C client (tests/c/abi_example.c) against include/cfpq.h and libcfpq.so."""
    import subprocess
    from paper_1707_01007_b200 import build
    build.build()
    libdir = os.path.join(ROOT, "paper_1707_01007_b200")
    exe = os.path.join(ROOT, "tests", "c", "abi_example")
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "abi_example.c"), "-L", libdir, "-lcfpq",
                           "-Wl,-rpath," + libdir, "-o", exe])
    return exe


def test_c_client_compiles_and_options_layout_matches_the_binding():
    """The header compiles as plain C99 and the ctypes mirror of cfpq_options has the C layout
    (every field offset and the size), so no option is marshalled into the wrong slot."""
    import subprocess
    from paper_1707_01007_b200 import cfpq as C
    exe = build_c_client()
    out = subprocess.run([exe, "layout"], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    got = dict((k, int(v)) for k, v in (ln.split() for ln in out.stdout.strip().splitlines()))
    assert got.pop("sizeof") == ctypes.sizeof(C.Options)
    names = {"reserved_emulate": "emulate_ranks"}
    assert len(got) == len(C.Options._fields_)
    for field, off in got.items():
        assert getattr(C.Options, names.get(field, field)).offset == off, field
