# 2-SM (cta_group::2) tensor kernel A/B (run under gpurun)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import inputs as I
from tests.gpu_util import gpu_closure, assert_parity
for n in (64, 300):
    w = I.dense_stress_workload(n, 2, seed=n)
    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=2)
    assert_parity(w, r)
print('2sm fp4 small ok')
"
timeout 120 python scripts/dense_perf.py 16384 2
CFPQ_DENSE_2SM=0 timeout 120 python scripts/dense_perf.py 16384 2
CFPQ_DENSE_2SM=1 timeout 120 python scripts/dense_perf.py 16384 1
timeout 900 python -m pytest tests/test_gpu_tensor.py tests/test_gpu_rows.py -q -x 2>&1 | tail -4
timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r1=C.closure(g,d,path_policy=1)
r=C.closure(g,d,path_policy=3)
for _ in range(2): C.closure_reuse(g,d,r,path_policy=3)
st=r.stats(); nc,_=r.iteration_stats(); nc1,_=r1.iteration_stats()
print(json.dumps({'rows_loop_ms': st['loop_ns']/1e6, 'same': nc.tolist()==nc1.tolist()}))
"
