#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_d.txt 2>&1
timeout 600 python scripts/c4_variants.py > gpurun_out/c4_variants_d.txt 2>&1
timeout 300 python scripts/phase_profile.py config4 cell_set=1 > gpurun_out/phase_bitmaps_d.txt 2>&1
for sch in 0 3; do
  timeout 300 python bench.py --steps 5 --warmup 3 --workload config3 --schedule $sch --no-supplementary --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_s${sch}_d.json 2>&1
done
timeout 600 torchrun --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --force-sharded --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun1_sharded.json 2> gpurun_out/bench_torchrun1_sharded.err
timeout 1800 python -m pytest tests/test_gpu_gauss_seidel.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py tests/test_gpu_async.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_d.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_d.txt 2>&1
tail -n 3 gpurun_out/pytest_d.txt gpurun_out/smoke_d.txt
