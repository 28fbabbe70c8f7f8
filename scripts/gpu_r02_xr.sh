#!/bin/bash
# emulated peer-memory exchange: every sharded test, repeated
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/xr
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for rep in 1 2 3 4; do
  timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider --timeout 300 -rf > $O/sh_$rep.txt 2>&1
  echo "rep $rep rc=$?"; tail -2 $O/sh_$rep.txt
done
timeout 600 python scripts/c4_variants.py > $O/variants.txt 2>&1; grep -E "bitmaps |xr|shard" $O/variants.txt
