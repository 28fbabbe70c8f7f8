python -c "import __graft_entry__ as g; g.build()" > /dev/null
python scripts/dense_perf.py 4096,16384; python scripts/dense_perf.py 16384
timeout 900 python -m pytest tests/test_gpu_tensor.py -q -x 2>&1 | tail -2
