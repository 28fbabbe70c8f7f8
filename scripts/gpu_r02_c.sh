#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_c.txt 2>&1
timeout 600 python scripts/c4_variants.py > gpurun_out/c4_variants_c.txt 2>&1
timeout 300 python scripts/phase_profile.py config4 cell_set=1 > gpurun_out/phase_bitmaps_c.txt 2>&1
for sch in 0 3; do
  timeout 300 python bench.py --steps 5 --warmup 3 --workload config3 --schedule $sch --no-supplementary --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_s${sch}_c.json 2>&1
done
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_c.txt 2>&1
tail -n 5 gpurun_out/pytest_c.txt
