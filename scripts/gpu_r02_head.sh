#!/bin/bash
# Full validation of HEAD: build, every GPU test, smoke, the default bench line.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_head.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_head.txt 2>&1
echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_head.json 2> gpurun_out/bench_head.err
echo "bench rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf --durations=25 > gpurun_out/pytest_head.txt 2>&1
echo "pytest rc=$?"
tail -40 gpurun_out/pytest_head.txt; tail -2 gpurun_out/smoke_head.txt; cut -c1-600 gpurun_out/bench_head.json
