#!/bin/bash
# CSR read-back tests (long rows, n > 2^18, full-size CSR digests)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_csrtests.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_csr.py tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider --timeout 600 -rf 2>&1 | tail -3
