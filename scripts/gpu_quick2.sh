set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python scripts/iter_profile.py config4 -1
python scripts/iter_profile.py config3 -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:closure_kernel -s 2 -c 1 -o gpurun_out/prof_config3 python bench.py --workload config3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_config3.txt 2>&1; tail -2 gpurun_out/ncu_full_config3.txt
