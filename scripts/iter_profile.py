"""Per-iteration Δ sizes and device times of one closure (diagnostics)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs as I
from paper_1707_01007_b200 import cfpq as C

name = sys.argv[1] if len(sys.argv) > 1 else "config4"
solos = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [-1]
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
w = {"config4": lambda: I.config4_workload(), "config3": lambda: I.anbn_workload(2, 16383),
     "q1": lambda: I.ontology_workload("q1", 3808, depth=8, seed=0)}[name]()
g = C.Grammar.from_workload(w)
d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
for solo in solos:
    r = C.closure(g, d, solo_threshold=solo, record_times=True, flags=flags)
    for _ in range(3):
        C.closure_reuse(g, d, r, solo_threshold=solo, record_times=True, flags=flags)
    st = r.stats()
    nc, _ = r.iteration_stats()
    t = r.iteration_times()
    print(f"solo={solo} iters={r.iterations} loop_ms={st['loop_ns']/1e6:.3f} seed_ms={st['seed_ns']/1e6:.3f} "
          f"cells={st['cells']} cand={st['candidates']} exps={st['expansions']} solo_iters={st['solo_iterations']}")
    prev = 0
    if len(nc) <= 40:
        for k in range(len(nc)):
            print(f"  k={k+1:3d} new={nc[k]:8d} dt_us={(t[k]-prev)/1e3:9.1f}")
            prev = t[k]
    else:
        dt = np.diff(np.concatenate([[0], t])) / 1e3
        print("  per-iter us: median", np.median(dt), "mean", dt.mean(), "max", dt.max())
    r2 = C.closure(g, d, solo_threshold=solo, flags=flags)
    C.closure_reuse(g, d, r2, solo_threshold=solo, flags=flags)
    print(f"  without timestamps: loop_ms={r2.stats()['loop_ns']/1e6:.3f}")
