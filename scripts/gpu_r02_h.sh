#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_h.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_edges.py -k "all_zero and rows and 1025" -q -p no:cacheprovider > gpurun_out/h_alone.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_edges.py -k "all_zero and rows and 1025" -q -p no:cacheprovider > gpurun_out/sanitize_h2.txt 2>&1
tail -5 gpurun_out/h_alone.txt; grep -v "^    \|^$" gpurun_out/sanitize_h2.txt | head -60
