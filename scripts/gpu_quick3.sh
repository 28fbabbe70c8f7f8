set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python scripts/solo_exp.py
python scripts/iter_profile.py config4 -1
