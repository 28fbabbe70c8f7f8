"""Config-3 single-CTA iteration experiments (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs as I
from paper_1707_01007_b200 import cfpq as C
q = int(sys.argv[1]) if len(sys.argv) > 1 else 16383
w = I.anbn_workload(2, q)
g = C.Grammar.from_workload(w)
d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
for mc in (0, 1, 8):
    r = C.closure(g, d, max_ctas=mc)
    C.closure_reuse(g, d, r, max_ctas=mc)
    st = r.stats()
    print(f"max_ctas={mc} ctas={st['ctas']} loop_ms={st['loop_ns']/1e6:.2f} us/iter={st['loop_ns']/1e3/r.iterations:.3f}")
r = C.closure(g, d, record_times=True)
C.closure_reuse(g, d, r, record_times=True)
st = r.stats(); it = st['solo_iterations']
print({k: round(v / it, 1) for k, v in st.items() if k.startswith('prof')}, "cycles/iter")
