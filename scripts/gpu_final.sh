set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()"
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
bash scripts/gpu_sanitize.sh
