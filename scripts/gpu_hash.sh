set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_hashed.py -q -x 2>&1 | tail -3
python scripts/phase_profile.py config4 | tail -1
python scripts/phase_profile.py config4 cell_set=1 | tail -1
python scripts/iter_profile.py config3 -1 | head -3
timeout 300 python -c "
import sys; sys.argv=['x','config3','-1']
" 
