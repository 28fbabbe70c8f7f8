#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/solo
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for W in config3 config5 config2 config4; do
  timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-supplementary > $O/bench_$W.json 2> $O/bench_$W.err
  python -c "import json; d=json.load(open('$O/bench_$W.json')); print('$W', d['ms_per_step'])"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gauss_seidel.py tests/test_gpu_witness.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py tests/test_gpu_async.py tests/test_gpu_hashed.py -m gpu -x -q -p no:cacheprovider --timeout 600 -rf > $O/pytest.txt 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.txt
