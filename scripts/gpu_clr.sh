set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hashed.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -4
python scripts/e2e_breakdown.py
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-supplementary --no-e2e 2>&1 | tail -1 | cut -c1-400
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-supplementary 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e'], d['config']['seed_phase_ms'], d['roofline']['kernel_ms'])"
