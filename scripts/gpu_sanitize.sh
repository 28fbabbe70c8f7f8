python -c "import __graft_entry__ as g; g.build()"
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done
echo "== memcheck, 1-CTA-per-SM tensor variant"
CFPQ_DENSE_2SM=0 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -c "
import sys; sys.path.insert(0,'.')
import inputs as I
from tests.gpu_util import gpu_closure, assert_parity
for fmt in (1, 2):
    w = I.dense_stress_workload(200, 2)
    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt)
    assert_parity(w, r)
print('ok 2sm')
" > gpurun_out/sanitize_2sm.txt 2>&1
echo "rc=$?"; tail -3 gpurun_out/sanitize_2sm.txt
