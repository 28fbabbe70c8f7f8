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
    assert_parity(w, r)
print('pack3 small ok')
"
timeout 120 python scripts/dense_perf.py 16384 2,1
timeout 120 python scripts/dense_perf.py 16384 2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pack3.csv python scripts/dense_perf.py 16384 2 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_tensor.py -q -x -k "example or stress or random or ontology or anbn or shards" 2>&1 | tail -2
