set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_witness.py tests/test_gpu_tensor.py -q -x 2>&1 | tail -4
python scripts/e2e_breakdown.py
python scripts/trace_e2e.py 2>&1 | tail -22
