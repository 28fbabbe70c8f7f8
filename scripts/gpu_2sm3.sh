set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_tensor.py -q -x 2>&1 | tail -3
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -c "
import sys; sys.path.insert(0,'.')
import inputs as I
from tests.gpu_util import gpu_closure, assert_parity
for fmt in (1, 2):
    for n, ranks in ((200, 0), (150, 3)):
        w = I.dense_stress_workload(n, 2)
        r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt, emulate_ranks=ranks)
        assert_parity(w, r)
print('ok 2sm default')
" > gpurun_out/sanitize_2sm_$tool.txt 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_2sm_$tool.txt
done
