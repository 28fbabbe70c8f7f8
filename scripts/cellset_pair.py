"""One config-4 closure with the bit-matrix cell set, then one with the hashed set (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import inputs as I
from paper_1707_01007_b200 import cfpq as C

w = I.config4_workload()
g = C.Grammar.from_workload(w)
d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
for cs in (1, 2):
    r = C.closure(g, d, cell_set=cs)
    torch.cuda.synchronize()
    print(cs, r.stats()["loop_ns"] / 1e6, r.stats()["hashed"])
