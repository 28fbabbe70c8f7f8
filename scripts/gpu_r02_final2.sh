#!/bin/bash
# Final evidence at HEAD: checked build over every GPU test + the case list; bench lines of
# every workload and the reference arm; launch lists; ncu of the closure kernel.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/final2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
python paper_1707_01007_b200/build.py --checked >> $O/build.txt 2>&1
CFPQ_CHECKED=1 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > $O/pytest_checked.txt 2>&1; echo "checked pytest rc=$?"
tail -2 $O/pytest_checked.txt
CFPQ_CHECKED=1 timeout 900 python scripts/sanitize.py > $O/checked_cases.txt 2>&1; echo "checked cases rc=$?"
for W in config3 config5; do CFPQ_CHECKED=1 timeout 600 python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-supplementary > $O/checked_bench_$W.json 2>&1; echo "checked $W rc=$?"; done
echo "assert hits: $(grep -h CFPQ_DASSERT $O/* 2>/dev/null | wc -l)"
rm -f paper_1707_01007_b200/libcfpq_checked.so
for W in configS config3 config5 config2; do
  timeout 900 python bench.py --workload $W --steps 10 --warmup 3 > $O/bench_$W.json 2> $O/bench_$W.err
done
timeout 600 python bench.py --workload config3 --schedule 3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_config3_gs.json 2>&1
timeout 600 python bench.py --workload config4 --schedule 3 --steps 10 --warmup 3 --no-cpu-baseline --no-supplementary > $O/bench_config4_gs.json 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2>&1
timeout 600 torchrun --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --force-sharded --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_torchrun1_sharded.json 2> $O/bench_torchrun1_sharded.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_config4.csv \
   python bench.py --workload config4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-supplementary > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:closure_kernel -s 5 -c 1 \
   -o $O/prof_config4 python bench.py --workload config4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-supplementary > $O/ncu_c4.txt 2>&1
python scripts/phase_profile.py config4 > $O/phase_config4.txt 2>&1
python scripts/e2e_breakdown.py > $O/e2e_config4.txt 2>&1
python scripts/table1.py > $O/table1.md 2> $O/table1.err
ls $O
