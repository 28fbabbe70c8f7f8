"""Small closures on every engine, for compute-sanitizer (memcheck / racecheck / synccheck):
sparse, hashed, sharded (NCCL-style host loop and peer-memory exchange), async, Gauss-Seidel,
tensor (fp4 and int8; CTA pairs by default, dense_launch 2 / 3 for the other variants; 2-D
grids), bit rows (forms L, R, V, P; row shards; list and chunk overflow)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import inputs as I
import oracle as O
from paper_1707_01007_b200 import cfpq as C

def run(w, **kw):
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, w.edges)
    r = C.closure(g, d, **kw)
    o = O.run(w, lengths=kw.get("semantics", 0) == 1)
    for A in range(w.n_nt):
        assert np.array_equal(r.pairs(A), o.pairs(A)), (w.name, kw)
    return r

cases = [(I.example_workload(), dict()), (I.example_workload(), dict(semantics=1)),
         (I.anbn_workload(3, 5), dict(semantics=1)),
         (I.ontology_workload("union", 300, depth=5, seed=1), dict(solo_threshold=0)),
         (I.ontology_workload("union", 300, depth=5, seed=1), dict(log_capacity=64)),
         (I.dense_stress_workload(100, 2), dict(semantics=1)),
         (I.dense_stress_workload(200, 2), dict(path_policy=2, tensor_format=1)),
         (I.dense_stress_workload(200, 2), dict(path_policy=2, tensor_format=2)),
         (I.dense_stress_workload(200, 2), dict(path_policy=3)),
         (I.ontology_workload("q1", 300, depth=5, seed=6), dict(path_policy=3)),
         (I.ontology_workload("union", 300, depth=5, seed=7), dict(path_policy=3)),
         (I.dense_stress_workload(150, 2), dict(path_policy=2, emulate_ranks=2)),
         (I.dense_stress_workload(150, 2), dict(path_policy=2, tensor_format=1, emulate_ranks=2)),
         (I.dense_stress_workload(300, 2), dict()),
         (I.ontology_workload("union", 300, depth=5, seed=2), dict(cell_set=2)),
         (I.ontology_workload("union", 300, depth=5, seed=2), dict(cell_set=2, log_capacity=64)),
         (I.ontology_workload("union", 300, depth=5, seed=3), dict(emulate_ranks=3)),
         (I.ontology_workload("q1", 200, depth=5, seed=4), dict(schedule=2)),
         (I.ontology_workload("union", 300, depth=5, seed=8), dict(schedule=3)),
         (I.anbn_workload(3, 5), dict(schedule=3)),
         (I.dense_stress_workload(150, 2), dict(schedule=3)),
         (I.ontology_workload("union", 300, depth=5, seed=9), dict(emulate_ranks=3, exchange=1)),
         (I.ontology_workload("union", 300, depth=5, seed=9), dict(emulate_ranks=4, exchange=1, log_capacity=64)),
         (I.ontology_workload("union", 300, depth=5, seed=10), dict(path_policy=3, emulate_ranks=3)),
         (I.ontology_workload("union", 300, depth=5, seed=10), dict(path_policy=3, rows_list_capacity=8)),
         (I.ontology_workload("union", 300, depth=5, seed=10), dict(path_policy=3, emulate_ranks=2, rows_list_capacity=8)),
         (I.dense_stress_workload(150, 2), dict(path_policy=2, emulate_ranks=4, grid=(2, 2))),
         (I.dense_stress_workload(150, 2), dict(path_policy=2, tensor_format=1, dense_launch=2)),
         (I.dense_stress_workload(150, 2), dict(path_policy=2, tensor_format=1, dense_launch=3))]
for w, kw in cases:
    run(w, **kw)
    print("ok", w.name, kw, flush=True)
# reuse with bank rotation (the other bank is cleared inside the closure kernel)
w = I.ontology_workload("union", 300, depth=5, seed=5)
g = C.Grammar.from_workload(w)
d = C.Graph(w.n_nodes, w.edges)
r = C.closure(g, d)
for _ in range(3):
    C.closure_reuse(g, d, r)
o = O.run(w)
assert all(np.array_equal(r.pairs(A), o.pairs(A)) for A in range(w.n_nt))
print("ok reuse", flush=True)
# single-path witness
w = I.anbn_workload(3, 5)
g = C.Grammar.from_workload(w)
d = C.Graph(w.n_nodes, w.edges)
r = C.closure(g, d, semantics=1)
p = r.witness(d, 0, *r.pairs(0)[0].tolist())
assert O.cyk(w, p[:, 1].tolist(), 0)
print("ok witness", flush=True)
