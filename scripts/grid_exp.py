"""Sparse engine experiments: per-iteration fixed cost and CTA-count sensitivity."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs as I
from paper_1707_01007_b200 import cfpq as C

def loop_ms(w, reps=3, **kw):
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
    r = C.closure(g, d, **kw)
    t = []
    for _ in range(reps):
        C.closure_reuse(g, d, r, **kw)
        t.append(r.stats()["loop_ns"] / 1e6)
    return min(t), r.iterations

w3 = I.anbn_workload(2, 2047)
for solo in (-1, 0):
    ms, it = loop_ms(w3, solo_threshold=solo)
    print(f"config3-small solo={solo}: {ms:.2f} ms, {1e3*ms/it:.2f} us/iter")
w4 = I.config4_workload()
for mc in (0, 74, 37, 16):
    ms, it = loop_ms(w4, max_ctas=mc)
    print(f"config4 max_ctas={mc}: loop {ms:.3f} ms ({1e3*ms/it:.1f} us/iter)")
