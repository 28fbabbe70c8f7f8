set -x
python -c "import __graft_entry__ as g; g.build()"
for V in 64 32 16; do CFPQ_ROWS_CHUNKL=$V timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r1=C.closure(g,d,path_policy=1)
r=C.closure(g,d,path_policy=3)
t=[]
for _ in range(3): C.closure_reuse(g,d,r,path_policy=3); t.append(r.stats()['loop_ns']/1e6)
nc,_=r.iteration_stats(); nc1,_=r1.iteration_stats()
print('chunkl $V', t, nc.tolist()==nc1.tolist())
"; done
