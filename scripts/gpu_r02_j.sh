#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_j.txt 2>&1
timeout 900 python scripts/c4_variants.py > gpurun_out/c4_variants_j.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_gauss_seidel.py tests/test_gpu_tensor.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider --timeout 900 -rf --durations=8 > gpurun_out/pytest_j.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_edges.py -k "gauss" -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_j2.txt 2>&1
for sch in 0 3; do
  timeout 300 python bench.py --steps 5 --warmup 3 --workload config3 --schedule $sch --no-supplementary --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_s${sch}_j.json 2>&1
done
tail -n 14 gpurun_out/pytest_j.txt; tail -2 gpurun_out/pytest_j2.txt
