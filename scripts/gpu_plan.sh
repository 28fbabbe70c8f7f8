set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r1=C.closure(g,d,path_policy=1)
r=C.closure(g,d,path_policy=3)
t=[]
for _ in range(3): C.closure_reuse(g,d,r,path_policy=3); t.append(r.stats()['loop_ns']/1e6)
nc,_=r.iteration_stats(); nc1,_=r1.iteration_stats()
print('rows', t, nc.tolist()==nc1.tolist())
"
timeout 900 python -m pytest tests/test_gpu_rows.py -q -x 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/launches_rows_config4.csv python -c "
import sys; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r=C.closure(g,d,path_policy=3)
" > /dev/null 2>&1
