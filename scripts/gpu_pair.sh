set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python -m pytest tests/test_gpu_tensor.py -q -x -k "example" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_tensor.py -q -x 2>&1 | tail -4
timeout 300 python scripts/dense_perf.py 4096,16384
CFPQ_DENSE_PAIR=0 timeout 300 python scripts/dense_perf.py 4096,16384
