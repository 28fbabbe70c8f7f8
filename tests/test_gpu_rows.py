"""GPU parity of the bit-row CUDA-core path (path_policy = 3): the paper-faithful
full-operand Jacobi products over packed rows (Alg. 1 line 9).  Every product is
recomputed from the whole T_{k-1}, so the per-iteration new-cell counts must equal the
oracle's Jacobi states T_k exactly (not only the fixpoint)."""
import pytest

import inputs as I
from tests.gpu_util import assert_parity, cuda_ok, gpu_closure

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def test_rows_example(example_golden):
    g = example_golden
    w = I.bind("example", I.same_generation_grammar(), 3, g["edges"], "S")
    r, _, _ = gpu_closure(w, path_policy=3)
    assert r.iterations == 6
    ores = assert_parity(w, r)
    nc, _ = r.iteration_stats()
    assert nc.tolist() == ores.stats()["new_bits"].tolist()


def test_rows_random_and_dense():
    for s in range(40):
        w = I.random_workload(60_000 + s, max_nodes=60, max_edges=200, max_nt=5, max_bin=10, max_term=5)
        r, _, _ = gpu_closure(w, path_policy=3)
        ores = assert_parity(w, r)
        nc, _ = r.iteration_stats()
        assert nc.tolist() == ores.stats()["new_bits"].tolist(), w.name
    for n, d in ((100, 2), (257, 1), (300, 3)):
        w = I.dense_stress_workload(n, d, seed=n)
        r, _, _ = gpu_closure(w, path_policy=3)
        ores = assert_parity(w, r)
        nc, _ = r.iteration_stats()
        assert nc.tolist() == ores.stats()["new_bits"].tolist()


@pytest.mark.parametrize("n", [700, 2048])
def test_rows_union_grammar(n):
    w = I.config4_workload(n=n)
    r, _, _ = gpu_closure(w, path_policy=3)
    ores = assert_parity(w, r)
    nc, _ = r.iteration_stats()
    assert nc.tolist() == ores.stats()["new_bits"].tolist()


@pytest.mark.parametrize("query", ["q1", "q2"])
def test_rows_ontology_and_reuse(query):
    """Q1 / Q2 (forms L, R, P) and reuse of the result: the second run starts from the
    cleared buffers and the seed cells again, on a different graph."""
    from paper_1707_01007_b200 import cfpq as C
    w = I.ontology_workload(query, 800, depth=7, seed=5)
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, w.edges)
    r = C.closure(g, d, path_policy=3)
    ores = assert_parity(w, r)
    nc, _ = r.iteration_stats()
    assert nc.tolist() == ores.stats()["new_bits"].tolist()
    w2 = I.ontology_workload(query, 800, depth=6, seed=6)
    d.set_edges(w2.edges)
    C.closure_reuse(g, d, r, path_policy=3)
    ores2 = assert_parity(w2, r)
    nc, _ = r.iteration_stats()
    assert nc.tolist() == ores2.stats()["new_bits"].tolist()


def test_rows_delta_list_overflow_fallback():
    """A Δ word list that overflows makes the next iteration copy whole matrices instead
    (and the list grows): same states.  rows_list_capacity = 8 forces it from iteration 1;
    the row-sharded variant rebuilds the shard's list from T_k minus T_{k-1} instead."""
    for w in (I.config4_workload(n=1500), I.dense_stress_workload(200, 2, seed=1)):
        for kw in (dict(), dict(emulate_ranks=3)):
            r, _, _ = gpu_closure(w, path_policy=3, rows_list_capacity=8, **kw)
            o = assert_parity(w, r)
            nc, _ = r.iteration_stats()
            assert nc.tolist() == o.stats()["new_bits"].tolist(), (w.name, kw)


def test_rows_wide_rows_agree_with_sparse():
    """n = 9000 spans several 256-word slices per row: the row path equals the sparse engine."""
    import numpy as np
    w = I.ontology_workload("q1", 9000, depth=7, seed=4)
    r3, _, _ = gpu_closure(w, path_policy=3)
    r1, _, _ = gpu_closure(w, path_policy=1)
    assert r3.iterations == r1.iterations
    for A in range(w.n_nt):
        assert np.array_equal(r3.pairs(A), r1.pairs(A))


def test_config4_full_size_engines_agree():
    """Config 4 at its bench size (n = 65,536, union grammar): three independent closures —
    the sparse semi-naive engine on bit matrices, the sparse engine on the hashed cell set,
    and the full-operand bit-row path — give the same relations for every NT, the same
    iteration count and (sparse vs rows, both Jacobi) the same per-iteration new-cell counts;
    the union grammar's S_Q1 / S_Q2 equal Q1's / Q2's start relations closed separately."""
    import numpy as np
    w = I.config4_workload()
    r1, _, _ = gpu_closure(w, path_policy=1, cell_set=1)
    r2, _, _ = gpu_closure(w, path_policy=1, cell_set=2)
    r3, _, _ = gpu_closure(w, path_policy=3)
    assert r1.iterations == r2.iterations == r3.iterations
    for A in range(w.n_nt):
        p1 = r1.pairs(A)
        assert np.array_equal(p1, r2.pairs(A)) and np.array_equal(p1, r3.pairs(A)), w.nt_names[A]
    assert r1.iteration_stats()[0].tolist() == r3.iteration_stats()[0].tolist()
    for q in ("q1", "q2"):
        wq = I.ontology_workload(q, 65536, depth=10, seed=0)
        # same triples (label ids are numbered per grammar)
        assert np.array_equal(np.sort(wq.edges[:, [0, 2]], axis=0), np.sort(w.edges[:, [0, 2]], axis=0))
        rq, _, _ = gpu_closure(wq, path_policy=1)
        A = w.nt_names.index("S_Q1" if q == "q1" else "S_Q2")
        assert np.array_equal(rq.pairs(wq.start), r1.pairs(A)), q


def test_rows_wider_than_config4():
    """n = 100,003 (ragged, 3,126 words per row: more scan batches per L chunk and 13 row
    slices per R chunk than config 4's 8 KiB rows): Q1 on the bit-row path equals the sparse
    engine, per iteration."""
    import numpy as np
    w = I.ontology_workload("q1", 100_003, depth=9, seed=11)
    r3, _, _ = gpu_closure(w, path_policy=3)
    r1, _, _ = gpu_closure(w, path_policy=1)
    assert r3.iterations == r1.iterations
    assert r3.iteration_stats()[0].tolist() == r1.iteration_stats()[0].tolist()
    for A in range(w.n_nt):
        assert np.array_equal(r3.pairs(A), r1.pairs(A)), w.nt_names[A]


@pytest.mark.parametrize("ranks", [2, 3, 8])
def test_rows_shards_emulated(ranks):
    """Row-block sharded bit-row engine (§8(e)): every shard derives its rows from full
    replicas, the Δ_k word lists go through the padded exchange buffer and the rank-order
    compaction, every word is applied to T_k (flip-counted).  Jacobi states per iteration."""
    for w in (I.ontology_workload("q1", 700, depth=7, seed=ranks), I.ontology_workload("q2", 500, depth=6, seed=1),
              I.config4_workload(n=1500, seed=ranks), I.anbn_workload(3, 7), I.dense_stress_workload(300, 2, seed=2),
              I.example_workload()):
        r, _, _ = gpu_closure(w, path_policy=3, emulate_ranks=ranks)
        ores = assert_parity(w, r)
        nc, _ = r.iteration_stats()
        assert nc.tolist() == ores.stats()["new_bits"].tolist(), (w.name, ranks)


def test_rows_shards_random_grammars():
    for s in range(60):
        w = I.random_workload(90_000 + s, max_nodes=80, max_edges=240, max_nt=6, max_bin=10, max_term=5)
        r, _, _ = gpu_closure(w, path_policy=3, emulate_ranks=2 + s % 5)
        ores = assert_parity(w, r)
        nc, _ = r.iteration_stats()
        assert nc.tolist() == ores.stats()["new_bits"].tolist(), w.name


def test_rows_nccl_single_rank():
    """The NCCL exchange of the word lists with one rank (libnccl dlopen'ed, counts + padded
    words all-gathered every iteration)."""
    from paper_1707_01007_b200 import cfpq as C
    uid = C.nccl_unique_id()
    w = I.config4_workload(n=2000, seed=4)
    r, _, _ = gpu_closure(w, path_policy=3, world_size=1, rank=0, nccl_unique_id=uid)
    ores = assert_parity(w, r)
    nc, _ = r.iteration_stats()
    assert nc.tolist() == ores.stats()["new_bits"].tolist()


def test_rows_pipelined_iterations_match_unpipelined():
    """Pipelined bit-row iterations (the next one enqueued before the host reads this one's
    outcome; a device stop flag gates the speculative one) give the same per-iteration states
    as the host-synchronised loop (diag_flags bit 11), at the fixpoint and under a cap, with
    the entry lists overflowing and redone (rows_list_capacity = 8)."""
    import numpy as np
    from paper_1707_01007_b200 import cfpq as C
    for w in (I.config4_workload(n=1500, seed=2), I.ontology_workload("q2", 700, depth=6, seed=3)):
        for extra in (dict(), dict(rows_list_capacity=8)):
            ra, _, _ = gpu_closure(w, path_policy=3, **extra)
            rb, _, _ = gpu_closure(w, path_policy=3, flags=1 << 11, **extra)
            assert ra.iterations == rb.iterations
            assert ra.iteration_stats()[0].tolist() == rb.iteration_stats()[0].tolist()
            for A in range(w.n_nt):
                assert np.array_equal(ra.pairs(A), rb.pairs(A)), (w.name, extra, A)
        g, d = C.Grammar.from_workload(w), C.Graph(w.n_nodes, w.edges)
        ca = C.closure(g, d, path_policy=3, max_iterations=3)
        cb = C.closure(g, d, path_policy=3, max_iterations=3, flags=1 << 11)
        assert ca.status == cb.status == C.CFPQ_E_NOT_CONVERGED
        assert ca.iterations == cb.iterations == 3
        for A in range(w.n_nt):
            assert np.array_equal(ca.pairs(A), cb.pairs(A))
