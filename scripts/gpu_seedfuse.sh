set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python scripts/ab_flags.py base=0
python scripts/trace_e2e.py 2>&1 | grep -B2 -A12 "seed_kernel" | head -30
