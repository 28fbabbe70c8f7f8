# ncu evidence for profiles/: launch list of one bench step and one full capture of the closure kernel
set -x
W=${1:-config4}
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
    python bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$W.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:closure_kernel -s 4 -c 1 \
    -o gpurun_out/prof_$W python bench.py --workload $W --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$W.txt 2>&1
tail -3 gpurun_out/ncu_full_$W.txt
