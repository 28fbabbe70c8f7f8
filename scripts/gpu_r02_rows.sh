#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/rows
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python scripts/rows_time.py 0 0 > $O/time.txt 2>&1
cat $O/time.txt
timeout 1200 python -m pytest tests/test_gpu_rows.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -m gpu -x -q -p no:cacheprovider --timeout 600 -rf > $O/pytest.txt 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.txt
