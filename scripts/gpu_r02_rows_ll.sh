#!/bin/bash
# ncu launch list (time, DRAM bytes, L2 hit rate) of one bit-row-engine closure of config 4
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/rowsll
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
cat > /tmp/rows1.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r=C.closure(g,d,path_policy=3)
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv \
   --log-file $O/launches_rows.csv python /tmp/rows1.py > /dev/null 2>&1
python scripts/launch_summary.py $O/launches_rows.csv > $O/summary.txt 2>&1
cat $O/summary.txt
