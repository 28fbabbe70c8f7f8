#!/bin/bash
# round-2 first pass: build, new GPU tests, the round-1 suite, one bench line
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/build.txt
timeout 1500 python -m pytest tests/test_gpu_gauss_seidel.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py \
  -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/pytest_new.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf \
  --deselect tests/test_gpu_gauss_seidel.py --deselect tests/test_gpu_edges.py --deselect tests/test_gpu_fullsize.py \
  > gpurun_out/pytest_old.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --steps 5 --warmup 3 --workload config3 --no-supplementary --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --workload config3 --schedule 3 --no-supplementary --no-cpu-baseline > gpurun_out/bench_c3_gs.json 2>&1
tail -3 gpurun_out/pytest_new.txt gpurun_out/pytest_old.txt
