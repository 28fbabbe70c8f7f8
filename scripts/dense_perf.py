"""Config S (S -> S S | a) on the tcgen05 dense engine: closure time and issued tensor work."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs as I
from paper_1707_01007_b200 import cfpq as C
ns = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [4096, 8192, 16384]
fmts = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2]
for n, fmt in [(n, f) for n in ns for f in fmts]:
    w = I.dense_stress_workload(n, 2, 0)
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
    r = C.closure(g, d, path_policy=2, tensor_format=fmt)
    for _ in range(2):
        C.closure_reuse(g, d, r, path_policy=2, tensor_format=fmt)
    st = r.stats()
    nc, _ = r.iteration_stats()
    ops = st["mma_kblocks"] * 2 * 128 * 32 * 128
    t = st["loop_ns"] * 1e-9
    print(json.dumps({"n": n, "fmt": fmt, "iters": r.iterations, "loop_ms": t * 1e3, "seed_ms": st["seed_ns"] / 1e6,
                      "kblocks": st["mma_kblocks"], "issued_TOPS": ops / t / 1e12,
                      "count": r.count(0), "density": r.count(0) / n / n, "new": nc.tolist()}))
