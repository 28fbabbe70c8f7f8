#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_m.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py tests/test_gpu_gauss_seidel.py tests/test_gpu_hashed.py tests/test_gpu_witness.py tests/test_gpu_async.py -m gpu -x -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_m.txt 2>&1
timeout 900 python scripts/c4_variants.py > gpurun_out/c4_variants_m.txt 2>&1
timeout 300 python scripts/phase_profile.py config4 > gpurun_out/phase_m.txt 2>&1
tail -n 3 gpurun_out/pytest_m.txt; head -8 gpurun_out/c4_variants_m.txt
