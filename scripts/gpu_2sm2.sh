set -x
python -c "import __graft_entry__ as g; g.build()"
CFPQ_DENSE_2SM=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import inputs as I
from tests.gpu_util import gpu_closure, assert_parity
for fmt in (1, 2):
  for n in (64, 300, 700):
    w = I.dense_stress_workload(n, 2, seed=n)
    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt)
    assert_parity(w, r)
print('2sm mask small ok')
"
CFPQ_DENSE_2SM=1 timeout 120 python scripts/dense_perf.py 16384 2,1
timeout 120 python scripts/dense_perf.py 16384 2,1
CFPQ_DENSE_PAIR=1 timeout 120 python scripts/dense_perf.py 16384 2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 3 -c 1 -o gpurun_out/prof_configS_mask python scripts/dense_perf.py 16384 2 > gpurun_out/ncu_mask.txt 2>&1
tail -1 gpurun_out/ncu_mask.txt
