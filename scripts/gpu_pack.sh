set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import inputs as I
from tests.gpu_util import gpu_closure, assert_parity
for fmt in (1, 2):
    for n in (64, 300, 257):
        w = I.dense_stress_workload(n, 2, seed=n)
        r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt)
        assert_parity(w, r)
print('pack small ok')
"
timeout 120 python scripts/dense_perf.py 16384 1,2
for O in 4 6 8; do CFPQ_ROWS_SCATTER_OCC=$O timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r=C.closure(g,d,path_policy=3)
for _ in range(3): C.closure_reuse(g,d,r,path_policy=3)
print('rows occ $O', r.stats()['loop_ns']/1e6)
"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_configS.csv \
   python bench.py --workload configS --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
