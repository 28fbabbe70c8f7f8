set -x
python -c "import __graft_entry__ as g; g.build()"
./scripts/tlb_probe
python scripts/phase_profile.py config4
python scripts/phase_profile.py config4 max_ctas=74
