"""The plain C client (tests/c/abi_example.c) runs the paper's worked example through the raw
C-ABI on the GPU: 6 loop bodies and R_S = {(0,0), (0,2), (1,2)} for the sparse,
tensor and bit-row engines, plus the argument and edge validation."""
import subprocess

import pytest

from tests.gpu_util import cuda_ok
from tests.test_abi import build_c_client

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def test_c_client_runs_the_example():
    exe = build_c_client()
    out = subprocess.run([exe, "run"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.startswith("OK"), (out.stdout, out.stderr)
