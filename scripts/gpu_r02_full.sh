#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_full.txt 2>&1
timeout 3600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf --durations=30 > gpurun_out/pytest_full.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_full.txt 2>&1
tail -45 gpurun_out/pytest_full.txt | head -42; tail -2 gpurun_out/smoke_full.txt
