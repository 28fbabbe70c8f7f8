#!/bin/bash
# grid-barrier wait: pure spin for 20 us then backoff (default) vs a fixed 32 / 128 ns sleep
# between polls from the start (built on the box only)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_spin.txt 2>&1
echo "== spin"; timeout 300 python scripts/ab_flags.py base=0 base_b=0 2>&1 | grep step
cp paper_1707_01007_b200/csrc/engine.cu /tmp/engine.cu.orig
for NS in 32 128; do
  cp /tmp/engine.cu.orig paper_1707_01007_b200/csrc/engine.cu
  sed -i "1044s/.*/                        ns = ${NS}u;/; 1077s/.*/                ns = ${NS}u;/" paper_1707_01007_b200/csrc/engine.cu
  sed -n '1043,1044p;1076,1077p' paper_1707_01007_b200/csrc/engine.cu
  python paper_1707_01007_b200/build.py --force >> gpurun_out/build_spin.txt 2>&1
  echo "== sleep $NS"; timeout 300 python scripts/ab_flags.py base=0 base_b=0 2>&1 | grep step
done
