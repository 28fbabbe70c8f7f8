set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_rgather -s 6 -c 1 -o gpurun_out/prof_rows_rgather \
   python -c "
import sys; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r=C.closure(g,d,path_policy=3)
" > gpurun_out/ncu_rgather.txt 2>&1
tail -2 gpurun_out/ncu_rgather.txt
