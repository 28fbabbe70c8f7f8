#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_e.txt 2>&1
timeout 600 python scripts/c4_variants.py > gpurun_out/c4_variants_e.txt 2>&1
timeout 300 python scripts/phase_profile.py config4 cell_set=1 > gpurun_out/phase_bitmaps_e.txt 2>&1
timeout 300 python scripts/phase_profile.py config4 cell_set=1 flags=8 > gpurun_out/phase_warpflush_e.txt 2>&1
