# bit-row path: parity + config-4 timing + launch list (run under gpurun)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_rows.py -q -x 2>&1 | tail -15
timeout 600 python -c "
import sys, time, json; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r1=C.closure(g,d,path_policy=1)
r=C.closure(g,d,path_policy=3)
for _ in range(2): C.closure_reuse(g,d,r,path_policy=3)
st=r.stats()
print(json.dumps({'iters': r.iterations, 'sparse_iters': r1.iterations, 'loop_ms': st['loop_ns']/1e6, 'seed_ms': st['seed_ns']/1e6,
  'same': all(r.count(X)==r1.count(X) for X in range(w.n_nt))}))
nc,_=r.iteration_stats(); nc1,_=r1.iteration_stats(); print(nc.tolist()==nc1.tolist())
"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_rows.csv python -c "
import sys; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r=C.closure(g,d,path_policy=3)
" > /dev/null 2>&1
CFPQ_DENSE_PAIR=1 timeout 300 python scripts/dense_perf.py 16384 2
timeout 300 python scripts/dense_perf.py 16384 2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 3 -c 1 -o gpurun_out/prof_configS_fp4 python scripts/dense_perf.py 16384 2 > gpurun_out/ncu_cS_fp4.txt 2>&1
tail -2 gpurun_out/ncu_cS_fp4.txt
