#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/csr
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_csr.py tests/test_gpu_abi_c.py -m gpu -q -p no:cacheprovider --timeout 600 -rf > $O/pytest.txt 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-supplementary > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print(d['ms_per_step'], d['e2e'])"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-supplementary --e2e-format pairs > $O/bench_pairs.json 2> $O/bench_pairs.err
python -c "import json; d=json.load(open('$O/bench_pairs.json')); print(d['ms_per_step'], d['e2e'])"
