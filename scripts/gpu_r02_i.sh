#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_i.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_fullsize.py tests/test_gpu_abi_c.py -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/pytest_i.txt 2>&1
timeout 900 python scripts/c4_variants.py > gpurun_out/c4_variants_i.txt 2>&1
tail -n 3 gpurun_out/pytest_i.txt
