#!/bin/bash
# bucketed CSR extraction: tests (release + checked build), result-read probe, e2e bench line
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/csr2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
python paper_1707_01007_b200/build.py --checked >> $O/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_csr.py tests/test_gpu_fullsize.py tests/test_gpu_abi_c.py -m gpu -x -q -p no:cacheprovider --timeout 600 -rf > $O/pytest.txt 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.txt
CFPQ_CHECKED=1 timeout 600 python -m pytest tests/test_gpu_csr.py -m gpu -x -q -p no:cacheprovider --timeout 600 -rf > $O/pytest_checked.txt 2>&1
echo "checked rc=$?"; tail -2 $O/pytest_checked.txt
timeout 300 python scripts/csr_probe.py 30 2>&1 | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python scripts/csr_probe.py 4 > /dev/null 2>&1
python scripts/launch_summary.py $O/launches.csv 2>&1 | head -14
timeout 600 python bench.py --no-supplementary > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'])"
