#!/bin/bash
# closure kernel CTA shape: 1 x 1024 threads per SM (default) vs 2 x 512 (built on the box only)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_blk.txt 2>&1
echo "== 1x1024"; timeout 300 python scripts/ab_flags.py base=0 base_b=0 2>&1 | grep step
sed -i 's/constexpr int kBlock = 1024;/constexpr int kBlock = 512;/; s/__launch_bounds__(kBlock, 1)/__launch_bounds__(kBlock, 2)/g' paper_1707_01007_b200/csrc/engine.cu
python paper_1707_01007_b200/build.py --force >> gpurun_out/build_blk.txt 2>&1 || python paper_1707_01007_b200/build.py >> gpurun_out/build_blk.txt 2>&1
echo "== 2x512"; timeout 300 python scripts/ab_flags.py base=0 base_b=0 2>&1 | grep step
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
