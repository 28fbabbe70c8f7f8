set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
python scripts/iter_profile.py config4 -1,0
python scripts/iter_profile.py config3 -1
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
