set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import inputs as I
from tests.gpu_util import gpu_closure, assert_parity
for fmt in (1, 2):
  for n in (64, 300, 257, 700):
    w = I.dense_stress_workload(n, 2, seed=n)
    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt)
    o = assert_parity(w, r)
print('mask small ok')
"
timeout 120 python scripts/dense_perf.py 16384 2,1
timeout 120 python scripts/dense_perf.py 4096,16384 2
timeout 900 python -m pytest tests/test_gpu_tensor.py -q -x 2>&1 | tail -3
