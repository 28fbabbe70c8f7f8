#!/bin/bash
# ncu source-level capture of the warp-solo loop (config 3: one new cell per iteration)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/soloprof
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
cat > /tmp/c3.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w = I.anbn_workload(2, 16383)
g = C.Grammar.from_workload(w); d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r = C.closure(g, d)
C.closure_reuse(g, d, r)
torch.cuda.synchronize(); print(r.iterations, r.stats()["loop_ns"] / 1e6)
PY
timeout 600 python /tmp/c3.py > $O/plain.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:closure_kernel -s 1 -c 1 -o $O/prof_c3 python /tmp/c3.py > $O/ncu.txt 2>&1
ncu -i $O/prof_c3.ncu-rep --page source --csv --print-source sass > $O/src_sass.csv 2>&1
ls -la $O; cat $O/plain.txt
