# FP4 tensor path bring-up (run under gpurun)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import inputs as I
from tests.gpu_util import gpu_closure, assert_parity
for n in (64, 300):
    w = I.dense_stress_workload(n, 2, seed=n)
    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=2)
    print(n, r.iterations, r.count(0))
    assert_parity(w, r)
print('fp4 small ok')
"
timeout 600 python -m pytest tests/test_gpu_tensor.py -q -x 2>&1 | tail -5
timeout 300 python scripts/dense_perf.py 4096,16384 1,2
