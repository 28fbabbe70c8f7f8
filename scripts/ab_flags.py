"""A/B of config-4 closure knobs (flags bit 0 = precheck, bit 1 = side-stream clear instead of
the in-kernel clear), interleaved to cancel drift; device ms per closure_reuse (CUDA events)."""
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
variants = {name: int(v) for name, v in (a.split("=") for a in sys.argv[1:])} or {"base": 0, "side_clear": 2}
res = {k: C.closure(g, d, stream=stream, flags=v) for k, v in variants.items()}
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
t = {k: [] for k in variants}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(40):
    for k, v in variants.items():
        flush.fill_(1)
        e0.record(stream)
        C.closure_reuse(g, d, res[k], stream=stream, flags=v)
        e1.record(stream)
        e1.synchronize()
        if rep >= 5:
            t[k].append(e0.elapsed_time(e1))
for k in variants:
    st = res[k].stats()
    print(f"{k:12s} step {statistics.median(t[k]):.4f} ms (min {min(t[k]):.4f})  loop {st['loop_ns']/1e6:.3f}  seed {st['seed_ns']/1e6:.3f}")
