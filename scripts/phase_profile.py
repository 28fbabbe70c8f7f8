"""Per-iteration phase breakdown of the grid-wide sparse iterations (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import inputs as I
from paper_1707_01007_b200 import cfpq as C

name = sys.argv[1] if len(sys.argv) > 1 else "config4"
w = {"config4": lambda: I.config4_workload(), "q1": lambda: I.ontology_workload("q1", 3808, depth=8, seed=0)}[name]()
g = C.Grammar.from_workload(w)
d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
extra = {}
for a in sys.argv[2:]:
    k, v = a.split("=")
    extra[k] = int(v)
r = C.closure(g, d, record_times=True, **extra)
for _ in range(3):
    C.closure_reuse(g, d, r, record_times=True, **extra)
nc, _ = r.iteration_stats()
t = r.iteration_times()
ph = r.iteration_phases()
st = r.stats()
mhz = 1965.0
print(f"{name} {extra} iters={r.iterations} loop_ms={st['loop_ns']/1e6:.3f} cells={st['cells']} cand={st['candidates']}")
prev = 0
print("   k      new   dt_us  expand  flush  barrier(last)  close   (us, max over CTAs)")
for k in range(len(nc)):
    e, f, b, c = (ph[k] / mhz)
    print(f"{k+1:4d} {nc[k]:8d} {(t[k]-prev)/1e3:7.1f} {e:7.2f} {f:6.2f} {b:8.2f} {c:7.2f}")
    prev = t[k]
s = ph.sum(0) / mhz
print("sum us: expand %.1f flush %.1f barrier %.1f close %.1f; total dt %.1f" % (*s, t[-1] / 1e3))
