"""GPU parity of the dense tensor-core engine (path_policy = 2: tcgen05 MMA on 0/1 tiles,
TMA-staged, TMEM accumulators, thresholded to bits) against the oracle, in both operand
formats: tensor_format 1 = kind::i8 (s32 accumulator), 2 = kind::mxf4 (e2m1 nibbles, unit
block scales, f32 accumulator)."""
from collections import deque

import numpy as np
import pytest

import inputs as I
import oracle as O
from tests.gpu_util import assert_parity, cuda_ok, gpu_closure

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def _bfs_closure_pairs(n, edges):
    adj = [[] for _ in range(n)]
    for s, _, d in edges:
        adj[s].append(d)
    out = []
    for s in range(n):
        seen = set(adj[s])
        dq = deque(adj[s])
        while dq:
            u = dq.popleft()
            for v in adj[u]:
                if v not in seen:
                    seen.add(v)
                    dq.append(v)
        out += [(s, v) for v in sorted(seen)]
    return np.array(out, dtype=np.int32).reshape(-1, 2)


@pytest.mark.parametrize("fmt", [1, 2])
def test_tensor_example_and_iterations(example_golden, fmt):
    g = example_golden
    w = I.bind("example", I.same_generation_grammar(), 3, g["edges"], "S")
    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt)
    assert r.iterations == 6
    ores = assert_parity(w, r)
    nc, _ = r.iteration_stats()
    assert nc.tolist() == ores.stats()["new_bits"].tolist()


@pytest.mark.parametrize("n,d", [(64, 1), (150, 2), (300, 1), (257, 3)])
@pytest.mark.parametrize("fmt", [1, 2])
def test_tensor_dense_stress_parity(n, d, fmt):
    """S -> S S | a (both operands change): several 128x256 tiles and K blocks, ragged n."""
    w = I.dense_stress_workload(n, d, seed=n)
    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt, account_work=True)
    ores = assert_parity(w, r)
    nc, jt = r.iteration_stats(work=True)
    assert nc.tolist() == ores.stats()["new_bits"].tolist()
    assert jt.tolist() == ores.stats()["jacobi_triples"].tolist()


@pytest.mark.parametrize("n,d", [(1000, 2), (2048, 1), (1537, 4)])
@pytest.mark.parametrize("fmt", [1, 2])
def test_tensor_dense_stress_bfs(n, d, fmt):
    """Larger n against the textbook BFS transitive closure (the pin of S -> S S | a)."""
    w = I.dense_stress_workload(n, d, seed=7)
    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt)
    assert np.array_equal(r.pairs(0), _bfs_closure_pairs(n, w.edges.tolist()))


@pytest.mark.parametrize("fmt", [1, 2])
def test_tensor_random_parity(fmt):
    for s in range(60):
        w = I.random_workload(40_000 + s, max_nodes=40, max_edges=120, max_nt=5, max_bin=10, max_term=5)
        r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt)
        ores = assert_parity(w, r)
        nc, _ = r.iteration_stats()
        assert nc.tolist() == ores.stats()["new_bits"].tolist(), w.name


@pytest.mark.parametrize("query", ["q1", "q2", "union"])
@pytest.mark.parametrize("fmt", [1, 2])
def test_tensor_ontology_parity(query, fmt):
    w = I.ontology_workload(query, 600, depth=6, seed=2)
    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt)
    assert_parity(w, r)


@pytest.mark.parametrize("fmt", [1, 2])
def test_tensor_anbn_and_reuse(fmt):
    from paper_1707_01007_b200 import cfpq as C
    w = I.anbn_workload(3, 5)
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, w.edges)
    r = C.closure(g, d, path_policy=2, tensor_format=fmt)
    assert r.iterations == 2 * 3 * 5 + 1
    assert_parity(w, r)
    C.closure_reuse(g, d, r, path_policy=2, tensor_format=fmt)
    assert_parity(w, r)
    w2 = I.anbn_workload(3, 5)
    w2.edges = w2.edges[::-1].copy()
    d.set_edges(w2.edges)
    C.closure_reuse(g, d, r, path_policy=2, tensor_format=fmt)
    assert_parity(w2, r)


def test_tensor_empty_and_lengths_rejected():
    from paper_1707_01007_b200 import cfpq as C
    w = I.bind("empty", I.dense_stress_grammar(), 10, [], "S")
    r, _, _ = gpu_closure(w, path_policy=2)
    assert r.iterations == 1 and r.count(0) == 0
    w2 = I.dense_stress_workload(20, 1)
    with pytest.raises(C.CfpqError) as e:
        gpu_closure(w2, path_policy=2, semantics=1)
    assert e.value.status == C.CFPQ_E_UNSUPPORTED


@pytest.mark.parametrize("ranks", [2, 3, 8])
@pytest.mark.parametrize("fmt", [1, 2])
def test_tensor_row_block_shards_emulated(ranks, fmt):
    """Row-block sharding of the dense engine (the multi-GPU partition, §8(e)) emulated with
    `ranks` shards in one process: identical closure, iterations and per-iteration counts."""
    for w in (I.dense_stress_workload(400, 2, seed=ranks), I.random_workload(50_000 + ranks, max_nodes=200,
                                                                               max_edges=600, max_nt=5, max_bin=10,
                                                                               max_term=5, n_labels=4),
              I.ontology_workload("union", 400, depth=5, seed=ranks)):
        r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt, emulate_ranks=ranks)
        ores = assert_parity(w, r)
        nc, _ = r.iteration_stats()
        assert nc.tolist() == ores.stats()["new_bits"].tolist()


def test_tensor_nccl_single_rank_path():
    """The NCCL exchange path (dlopen'ed libnccl, ncclCommInitRank, grouped in-place
    all-gather of the row blocks + all-reduce of the new-cell count) with one rank."""
    from paper_1707_01007_b200 import cfpq as C
    uid = C.nccl_unique_id()
    w = I.dense_stress_workload(500, 2, seed=3)
    r, _, _ = gpu_closure(w, path_policy=2, world_size=1, rank=0, nccl_unique_id=uid)
    assert_parity(w, r)


@pytest.mark.parametrize("n,d", [(300, 2), (400, 2)])
def test_auto_policy_switches_to_tensor(n, d):
    """Auto policy: sparse iterations while Δ is small, then the tcgen05 engine once Δ is
    dense (rule S -> S S has two changing operands); same fixpoint, iterations and counts."""
    w = I.dense_stress_workload(n, d, seed=11)
    r, _, _ = gpu_closure(w, account_work=True)
    assert r.stats()["dense_finish"] == 1
    ores = assert_parity(w, r)
    nc, jt = r.iteration_stats(work=True)
    assert nc.tolist() == ores.stats()["new_bits"].tolist()
    assert jt.tolist() == ores.stats()["jacobi_triples"].tolist()
    # the paper's grammars (all rules have a preterminal operand) never switch
    w2 = I.ontology_workload("union", 800, depth=6, seed=1)
    r2, _, _ = gpu_closure(w2)
    assert r2.stats()["dense_finish"] == 0
    assert_parity(w2, r2)


def test_tensor_cta_pairs_multicast():
    """dense_launch = 3: CTA pairs (clusters of 2) sharing the B tile through TMA multicast,
    MMA commits arriving on both CTAs' stage barriers; same closure, including an odd number
    of row tiles (the second tile of the last pair does not exist)."""
    for n, d in [(300, 2), (700, 2), (130, 1)]:
        w = I.dense_stress_workload(n, d, seed=n)
        r, _, _ = gpu_closure(w, path_policy=2, tensor_format=1, dense_launch=3)
        assert_parity(w, r)
        r, _, _ = gpu_closure(w, path_policy=2, tensor_format=1, dense_launch=3, emulate_ranks=3)
        assert_parity(w, r)


def test_tensor_one_cta_per_sm():
    """dense_launch = 2: the one-CTA-per-SM kernel (the default is the 2-SM pair kernel:
    cta_group::2, M = 256 UMMAs issued by the even CTA, each CTA staging its A rows and half
    of B, TMA bytes of both CTAs completing on the leader's barrier) in both formats,
    including the emulated row-block shards."""
    for fmt in (1, 2):
        for n, d in [(300, 2), (700, 2), (130, 1)]:
            w = I.dense_stress_workload(n, d, seed=n)
            r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt, dense_launch=2)
            o = assert_parity(w, r)
            nc, _ = r.iteration_stats()
            assert nc.tolist() == o.stats()["new_bits"].tolist()
        w = I.ontology_workload("union", 500, depth=5, seed=3)
        r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt, dense_launch=2, emulate_ranks=3)
        assert_parity(w, r)


@pytest.mark.parametrize("fmt", [1, 2])
def test_tensor_config_s_full_size_sampled(fmt):
    """Config S at its bench size (S -> S S | a on G(16384, 32768), the launch configuration
    bench.py times): R_S rows of 48 sampled source nodes against BFS from each source (the
    pin of S -> S S | a: the strict transitive closure of the a-edges), plus the closure's
    iteration count and the symmetric property |R_S| = sum of the BFS set sizes on the sample."""
    import numpy as np
    from paper_1707_01007_b200 import cfpq as C
    n = 16384
    w = I.dense_stress_workload(n, 2, 0)
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, w.edges)
    r = C.closure(g, d, path_policy=2, tensor_format=fmt)
    pairs = r.pairs(0)
    adj = [[] for _ in range(n)]
    for s, _, t in w.edges.tolist():
        adj[s].append(t)
    rng = np.random.default_rng(5)
    starts = np.searchsorted(pairs[:, 0], np.arange(n + 1))
    for s in rng.choice(n, 48, replace=False).tolist():
        seen = set(adj[s])
        dq = deque(adj[s])
        while dq:
            u = dq.popleft()
            for v in adj[u]:
                if v not in seen:
                    seen.add(v)
                    dq.append(v)
        got = pairs[starts[s]:starts[s + 1], 1]
        assert np.array_equal(got, np.array(sorted(seen), dtype=got.dtype)), s
    assert r.iterations == 7


@pytest.mark.parametrize("grid", [(2, 2), (2, 3), (3, 2), (1, 4), (4, 1), (2, 4)])
@pytest.mark.parametrize("fmt", [1, 2])
def test_tensor_2d_grid_emulated(grid, fmt):
    """2-D (SUMMA-style) block sharding: shard (a, b) derives block (I_a, J_b)
    of every T_A from the row panel I_a of the left and the column panel J_b of the right
    operands; blocks go through the staging buffer.  Jacobi states per iteration."""
    for w in (I.dense_stress_workload(300, 2, seed=7), I.dense_stress_workload(700, 2, seed=8),
              I.dense_stress_workload(129, 1, seed=9), I.ontology_workload("union", 600, depth=6, seed=4),
              I.anbn_workload(5, 7)):
        r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt, emulate_ranks=grid[0] * grid[1], grid=grid)
        o = assert_parity(w, r)
        nc, _ = r.iteration_stats()
        assert nc.tolist() == o.stats()["new_bits"].tolist(), (w.name, grid)


def test_tensor_2d_grid_random_grammars():
    for s in range(30):
        w = I.random_workload(70_000 + s, max_nodes=300, max_edges=900, max_nt=4, max_bin=8, max_term=4)
        grid = [(2, 2), (1, 3), (3, 1), (2, 3)][s % 4]
        r, _, _ = gpu_closure(w, path_policy=2, emulate_ranks=grid[0] * grid[1], grid=grid)
        o = assert_parity(w, r)
        nc, _ = r.iteration_stats()
        assert nc.tolist() == o.stats()["new_bits"].tolist(), (w.name, grid)


def test_tensor_2d_grid_rejections():
    from paper_1707_01007_b200 import cfpq as C
    w = I.dense_stress_workload(50, 1)
    for kw in (dict(path_policy=2, emulate_ranks=4, grid=(2, 3)), dict(path_policy=1, emulate_ranks=4, grid=(2, 2)),
               dict(path_policy=3, emulate_ranks=4, grid=(2, 2))):
        with pytest.raises(C.CfpqError):
            gpu_closure(w, **kw)


@pytest.mark.parametrize("variant", ["pairs_fp4", "pairs_int8", "grid_2x4_fp4"])
def test_tensor_config_s_full_size_all_rows(variant):
    """Config S at its bench size (S -> S S | a on G(16384, 32768)): EVERY row of R_S equals
    the strict transitive closure of the a-edges (tests/closure_pin.py: SCC condensation,
    pinned to the oracle on CPU), bit for bit, for the default CTA-pair kernel in both operand
    formats and for the 2-D block-sharded run on an emulated 2 x 4 grid."""
    import torch

    from paper_1707_01007_b200 import cfpq as C
    from tests.closure_pin import strict_closure_bits
    w = I.dense_stress_workload(16384, 2, 0)
    e = np.asarray(w.edges)
    exp = strict_closure_bits(w.n_nodes, e[:, 0], e[:, 2])
    kw = {"pairs_fp4": dict(tensor_format=2), "pairs_int8": dict(tensor_format=1),
          "grid_2x4_fp4": dict(tensor_format=2, emulate_ranks=8, grid=(2, 4))}[variant]
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda(), stream=torch.cuda.current_stream())
    r = C.closure(g, d, path_policy=2, stream=torch.cuda.current_stream(), **kw)
    got = r.matrix(0)
    assert got.shape == exp.shape
    bad = np.nonzero((got != exp).any(axis=1))[0]
    assert len(bad) == 0, (variant, len(bad), bad[:5])
    assert r.count(0) == int(np.unpackbits(exp.view(np.uint8)).sum())
