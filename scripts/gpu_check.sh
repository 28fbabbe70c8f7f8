set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -3 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 600 python bench.py --workload config3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2>&1; cat gpurun_out/bench_c3.json
timeout 600 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2>&1; cat gpurun_out/bench_c5.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_stdout.txt 2>&1; tail -2 gpurun_out/ncu_launch_stdout.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:closure_kernel -s 4 -c 1 -o gpurun_out/prof_c4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_stdout.txt 2>&1; tail -5 gpurun_out/ncu_full_stdout.txt
ls -la gpurun_out
