#!/bin/bash
# Per-iteration phases: bitmap vs hashed cell set (config 4).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/hash
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for v in "cell_set=1" "cell_set=2" "cell_set=1 flags=4" "cell_set=1 flags=1"; do
  echo "== $v"; timeout 300 python scripts/phase_profile.py config4 $v 2>&1 | tail -24
done > $O/phases.txt
cat $O/phases.txt
