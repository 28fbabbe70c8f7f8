set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python scripts/ab_flags.py base=0 no_self_clear=4 precheck=1
python scripts/e2e_breakdown.py
