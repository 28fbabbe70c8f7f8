set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -2 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 600 python bench.py --workload configS --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_cS.json 2> gpurun_out/bench_cS.err; tail -2 gpurun_out/bench_cS.err; cat gpurun_out/bench_cS.json
timeout 600 python bench.py --workload config3 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c3.json 2>&1; cat gpurun_out/bench_c3.json
timeout 600 python bench.py --workload config5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.json 2>&1; cat gpurun_out/bench_c5.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_configS.csv python bench.py --workload configS --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 12 -c 1 -o gpurun_out/prof_configS python bench.py --workload configS --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_configS.txt 2>&1; tail -2 gpurun_out/ncu_full_configS.txt
