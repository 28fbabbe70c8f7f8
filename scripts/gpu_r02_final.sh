#!/bin/bash
# Final round-2 evidence: build, smoke, every GPU test, default bench line, checked build over
# every GPU test, bench lines of every workload + launch lists + ncu captures.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/final
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf --durations=10 > $O/pytest.txt 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest.txt
timeout 600 python bench.py > $O/bench_config4.json 2> $O/bench_config4.err; echo "bench rc=$?"
python paper_1707_01007_b200/build.py --checked >> $O/build.txt 2>&1
CFPQ_CHECKED=1 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > $O/pytest_checked.txt 2>&1; echo "checked pytest rc=$?"
tail -2 $O/pytest_checked.txt
CFPQ_CHECKED=1 timeout 900 python scripts/sanitize.py > $O/checked_cases.txt 2>&1; echo "checked cases rc=$?"
CFPQ_CHECKED=1 timeout 600 python scripts/rows_time.py 0 > $O/checked_rows.txt 2>&1; echo "checked rows rc=$?"
echo "assert hits: $(grep -h CFPQ_DASSERT $O/*checked* 2>/dev/null | wc -l)"
rm -f paper_1707_01007_b200/libcfpq_checked.so
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/launches_rows_config4.csv python /tmp/rows1.py > /dev/null 2>&1 || true
cat > /tmp/rows1.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r=C.closure(g,d,path_policy=3)
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/launches_rows_config4.csv python /tmp/rows1.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_compact_kernel -s 12 -c 1 -o $O/prof_rows_compact python /tmp/rows1.py > $O/ncu_rows_compact.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_lmerge_kernel -s 6 -c 1 -o $O/prof_rows_lmerge python /tmp/rows1.py > $O/ncu_rows_lmerge.txt 2>&1
python scripts/launch_summary.py $O/launches_rows_config4.csv > $O/launches_rows_summary.txt 2>&1
ls $O
