#!/bin/bash
# generic A/B: build, then ab_flags with the given variants (name=flags ...), plus a phase profile
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/ab
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python scripts/ab_flags.py "$@" 2>&1 | tail -8
timeout 300 python scripts/phase_profile.py config4 2>&1 | tail -3
