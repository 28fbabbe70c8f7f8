#!/bin/bash
# node-order probe (scripts/reorder_probe.py) on config 4
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_reorder.txt 2>&1
timeout 600 python scripts/reorder_probe.py 2>&1 | tail -8
