#!/bin/bash
# result-read breakdown (scripts/csr_probe.py) and the kernels of the csr calls (ncu launch list)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/csrprobe
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python scripts/csr_probe.py 30 2>&1 | tail -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python scripts/csr_probe.py 4 > /dev/null 2>&1
python scripts/launch_summary.py $O/launches.csv 2>&1 | head -20
