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
    """The opt-in CTA-pair variant (clusters of 2 sharing the B tile through TMA multicast,
    MMA commits arriving on both CTAs' stage barriers) gives the same closure, including an
    odd number of row tiles (the second tile of the last pair does not exist)."""
    import os
    import subprocess
    import sys
    code = (
        "import inputs as I, numpy as np\n"
        "from tests.gpu_util import gpu_closure, assert_parity\n"
        "for n, d in [(300, 2), (1000, 2), (130, 1)]:\n"
        "    w = I.dense_stress_workload(n, d, seed=n)\n"
        "    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=1)\n"
        "    assert_parity(w, r)\n"
        "    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=1, emulate_ranks=3)\n"
        "    assert_parity(w, r)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CFPQ_DENSE_PAIR="1", PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_tensor_one_cta_per_sm():
    """The one-CTA-per-SM kernel (CFPQ_DENSE_2SM=0; the default is the 2-SM pair kernel:
    cta_group::2, M = 256 UMMAs issued by the even CTA, each CTA staging its A rows and half
    of B, TMA bytes of both CTAs completing on the leader's barrier) in both formats,
    including the emulated row-block shards."""
    import os
    import subprocess
    import sys
    code = (
        "import inputs as I\n"
        "from tests.gpu_util import gpu_closure, assert_parity\n"
        "for fmt in (1, 2):\n"
        "    for n, d in [(300, 2), (700, 2), (130, 1)]:\n"
        "        w = I.dense_stress_workload(n, d, seed=n)\n"
        "        r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt)\n"
        "        o = assert_parity(w, r)\n"
        "        nc, _ = r.iteration_stats()\n"
        "        assert nc.tolist() == o.stats()['new_bits'].tolist()\n"
        "    w = I.ontology_workload('union', 500, depth=5, seed=3)\n"
        "    r, _, _ = gpu_closure(w, path_policy=2, tensor_format=fmt, emulate_ranks=3)\n"
        "    assert_parity(w, r)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CFPQ_DENSE_2SM="0", PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


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
