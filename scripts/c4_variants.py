"""Config-4 closure time by engine option (diagnostics): median of 10 reuses, L2 flushed."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import inputs as I
from paper_1707_01007_b200 import cfpq as C

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w = I.config4_workload(n=n)
g = C.Grammar.from_workload(w)
s = torch.cuda.current_stream()
d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda(), stream=s)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
variants = {
    "bitmaps": dict(cell_set=1),
    "bitmaps_noprecheck": dict(cell_set=1, flags=1),
    "bitmaps_noreset": dict(cell_set=1, flags=4),
    "bitmaps_selfreset": dict(cell_set=1, flags=128),
    "bitmaps_ctamajor": dict(cell_set=1, flags=256),
    "bitmaps_seed_kernels": dict(cell_set=1, flags=512),
    "hashed": dict(cell_set=2),
    "solo0": dict(cell_set=1, solo_threshold=0),
    "gauss_seidel": dict(cell_set=1, schedule=3),
    "gauss_seidel_hashed": dict(cell_set=2, schedule=3),
    "async": dict(schedule=2),
    "rows": dict(path_policy=3),
    "rows_R_1x4rows": dict(path_policy=3, flags=1 << 4),
    "rows_R_2x1row": dict(path_policy=3, flags=2 << 4),
    "rows_R_2x4rows": dict(path_policy=3, flags=3 << 4),
    "rows_R_1x8rows": dict(path_policy=3, flags=4 << 4),
    "cta_flush": dict(cell_set=1, flags=8),
    "xr2_peer": dict(emulate_ranks=2, exchange=1),
    "xr8_peer": dict(emulate_ranks=8, exchange=1),
    "shard8_hostloop": dict(emulate_ranks=8),
    "ctas111": dict(cell_set=1, max_ctas=111),
    "ctas74": dict(cell_set=1, max_ctas=74),
    "ctas37": dict(cell_set=1, max_ctas=37),
}
for name, kw in variants.items():
    r = C.closure(g, d, stream=s, **kw)
    ts, loops = [], []
    for _ in range(10):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        C.closure_reuse(g, d, r, stream=s, **kw)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        loops.append(r.stats()["loop_ns"] / 1e6)
    print(f"{name:22s} step {statistics.median(ts):.3f} ms  loop {statistics.median(loops):.3f} ms  "
          f"iterations {r.iterations}  cells {r.stats()['cells']}", flush=True)
    del r
