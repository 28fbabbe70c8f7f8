"""Config-4 bit-row (path_policy 3) closure time: median of reuses, L2 flushed (diagnostics)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs as I
from paper_1707_01007_b200 import cfpq as C

w = I.config4_workload()
g = C.Grammar.from_workload(w)
s = torch.cuda.current_stream()
d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda(), stream=s)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for flags in [int(a) for a in sys.argv[1:]] or [0]:
    r = C.closure(g, d, stream=s, path_policy=3, flags=flags)
    ts, loops = [], []
    for _ in range(6):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        C.closure_reuse(g, d, r, stream=s, path_policy=3, flags=flags)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        loops.append(r.stats()["loop_ns"] / 1e6)
    print(f"rows flags={flags}: step {statistics.median(ts):.3f} ms loop {statistics.median(loops):.3f} ms "
          f"iterations {r.iterations} cells {sum(r.count(a) for a in range(w.n_nt))}", flush=True)
    del r
