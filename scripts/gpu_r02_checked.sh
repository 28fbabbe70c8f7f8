#!/bin/bash
# Checked build (device bounds assertions) over every GPU test, the sanitizer case list, and one
# closure of every benchmark workload (compute-sanitizer is closed on this pool).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/checked
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
python paper_1707_01007_b200/build.py --checked >> $O/build.txt 2>&1
export CFPQ_CHECKED=1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > $O/pytest.txt 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.txt
timeout 900 python scripts/sanitize.py > $O/cases.txt 2>&1; echo "cases rc=$?"; tail -2 $O/cases.txt
for W in config4 configS config3 config2; do
  timeout 600 python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-supplementary > $O/bench_$W.json 2> $O/bench_$W.err
  echo "$W rc=$?"
done
timeout 600 python scripts/rows_time.py 0 > $O/rows.txt 2>&1; echo "rows rc=$?"; cat $O/rows.txt
grep -l "CFPQ_DASSERT" $O/* 2>/dev/null; echo "assert hits: $(grep -h CFPQ_DASSERT $O/* 2>/dev/null | wc -l)"
