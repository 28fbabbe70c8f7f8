# end-of-session check: smoke, the whole GPU suite, then the evidence refresh (run under gpurun)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
bash scripts/gpu_refresh.sh
