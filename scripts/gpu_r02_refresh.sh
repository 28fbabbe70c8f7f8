#!/bin/bash
# after the per-warp log append became the default: checked build over every GPU test, the
# bench lines it changes, the config-4 launch list, one ncu full capture of closure_kernel,
# the phase profile
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02b
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
python paper_1707_01007_b200/build.py --checked >> $O/build.txt 2>&1
CFPQ_CHECKED=1 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > $O/pytest_checked.txt 2>&1
echo "checked pytest rc=$?"; tail -2 $O/pytest_checked.txt
echo "assert hits: $(grep -h CFPQ_DASSERT $O/pytest_checked.txt | wc -l)"
for W in config2 configS; do
  timeout 900 python bench.py --workload $W --steps 10 --warmup 3 > $O/bench_$W.json 2> $O/bench_$W.err
done
timeout 600 python bench.py --workload config4 --schedule 3 --steps 10 --warmup 3 --no-cpu-baseline --no-supplementary > $O/bench_config4_gs.json 2>&1
timeout 300 python scripts/phase_profile.py config4 > $O/phase_config4.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_config4.csv \
   python bench.py --workload config4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-supplementary > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:closure_kernel -s 5 -c 1 \
   -o $O/prof_config4 python bench.py --workload config4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-supplementary > $O/ncu_c4.txt 2>&1
ls $O
