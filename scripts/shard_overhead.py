"""Per-iteration cost of the row-sharded sparse loop on one GPU (NCCL world of one rank):
host-driven launches + count/cell all-gathers vs the persistent single-launch engine."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import inputs as I
from paper_1707_01007_b200 import cfpq as C

w = I.config4_workload()
stream = torch.cuda.current_stream()
g = C.Grammar.from_workload(w)
d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda(), stream=stream)
uid = C.nccl_unique_id()
for name, kw in [("persistent", {}), ("sharded_nccl_1rank", dict(world_size=1, rank=0, nccl_unique_id=uid)),
                 ("emulated_2", dict(emulate_ranks=2)), ("emulated_4", dict(emulate_ranks=4))]:
    r = C.closure(g, d, stream=stream, **kw)
    ts = []
    for _ in range(8):
        C.closure_reuse(g, d, r, stream=stream, **kw)
        st = r.stats()
        ts.append((st["seed_ns"] + st["loop_ns"]) / 1e6)
    print(f"{name:22s} closure {statistics.median(ts):.3f} ms  iterations {r.iterations}  launches {r.stats()['launches']}")
