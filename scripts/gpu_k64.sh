# fp4 64-byte K blocks (9 stages) A/B (run under gpurun)
set -x
python -c "import __graft_entry__ as g; g.build()"
CFPQ_DENSE_K64=1 timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import inputs as I
from tests.gpu_util import gpu_closure, assert_parity
for n in (64, 300):
    w = I.dense_stress_workload(n, 2, seed=n)
    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=2)
    assert_parity(w, r)
print('k64 small ok')
"
CFPQ_DENSE_K64=1 timeout 120 python scripts/dense_perf.py 16384 2
timeout 120 python scripts/dense_perf.py 16384 2
CFPQ_DENSE_K64=1 timeout 900 python -m pytest tests/test_gpu_tensor.py -q -x -k "k64 or full_size" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_rows.py -q -x -k "full_size" 2>&1 | tail -3
