"""Seeded synthetic grammars and graphs (the workloads of SURVEY.md §8(d)).

Every generator is deterministic in its `seed` (numpy PCG64).  A workload is a
CNF grammar (rules A->BC and A->x, no start symbol) plus an
edge-labelled digraph D=(V,E) with E ⊆ V×Σ×V, with labels interned to
ids that index one vocabulary shared by grammar and graph.  Labels that occur in
the graph but have no terminal rule stay in the vocabulary (they seed nothing,
S:249).

Nothing here computes any part of the CFPQ method.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "Workload", "Grammar", "bind",
    "same_generation_grammar", "q2_grammar", "union_grammar", "anbn_grammar",
    "dense_stress_grammar", "random_grammar",
    "example_edges", "two_cycle_edges", "ontology_triples", "triples_to_edges",
    "disjoint_copies", "random_digraph_edges", "random_labeled_edges",
    "example_workload", "anbn_workload", "ontology_workload", "dense_stress_workload",
    "random_workload", "relabel_nodes", "TABLE1_TRIPLES", "config4_workload",
]


@dataclass
class Grammar:
    """CNF grammar G=(N,Σ,P).  NTs and terminals are named."""
    nt_names: List[str]
    binary: List[Tuple[str, str, str]]          # A -> B C
    terminal: List[Tuple[str, str]]             # A -> x

    @property
    def terminals(self) -> List[str]:
        out: List[str] = []
        for _, x in self.terminal:
            if x not in out:
                out.append(x)
        return out


@dataclass
class Workload:
    """A bound (grammar, graph) pair with integer ids, ready for either side."""
    name: str
    n_nodes: int
    nt_names: List[str]
    labels: List[str]
    bin: np.ndarray            # int32 [n_bin, 3] (A, B, C)
    term: np.ndarray           # int32 [n_term, 2] (A, label)
    edges: np.ndarray          # int32 [n_edges, 3] (src, label, dst)
    start: int = 0             # NT whose |R| is the "#results"
    meta: Dict = field(default_factory=dict)

    @property
    def n_nt(self) -> int:
        return len(self.nt_names)

    @property
    def n_labels(self) -> int:
        return len(self.labels)

    def nt(self, name: str) -> int:
        return self.nt_names.index(name)


def bind(name: str, g: Grammar, n_nodes: int, named_edges: Sequence[Tuple[int, str, int]],
         start: str, extra_labels: Sequence[str] = (), meta: Optional[Dict] = None) -> Workload:
    """Intern labels: the grammar's terminals first, then any other graph labels."""
    labels = list(g.terminals)
    for x in extra_labels:
        if x not in labels:
            labels.append(x)
    for _, x, _ in named_edges:
        if x not in labels:
            labels.append(x)
    lid = {x: k for k, x in enumerate(labels)}
    nid = {a: k for k, a in enumerate(g.nt_names)}
    b = np.array([[nid[a], nid[bb], nid[c]] for a, bb, c in g.binary], dtype=np.int32).reshape(-1, 3)
    t = np.array([[nid[a], lid[x]] for a, x in g.terminal], dtype=np.int32).reshape(-1, 2)
    if len(named_edges):
        e = np.array([[s, lid[x], d] for s, x, d in named_edges], dtype=np.int32).reshape(-1, 3)
    else:
        e = np.zeros((0, 3), dtype=np.int32)
    return Workload(name, int(n_nodes), list(g.nt_names), labels, b, t, e, nid[start], dict(meta or {}))


# ---------------------------------------------------------------------------------------------
# Grammars
# ---------------------------------------------------------------------------------------------

SC, SCR, T, TR = "subClassOf", "subClassOf_r", "type", "type_r"


def same_generation_grammar() -> Grammar:
    """G' of P:279-296 (CNF of the same-generation query, = Query 1)."""
    binary = [("S", "S1", "S5"), ("S", "S3", "S6"), ("S", "S1", "S2"), ("S", "S3", "S4"),
              ("S5", "S", "S2"), ("S6", "S", "S4")]
    terminal = [("S1", SCR), ("S2", SC), ("S3", TR), ("S4", T)]
    return Grammar(["S", "S1", "S2", "S3", "S4", "S5", "S6"], binary, terminal)


def q2_grammar() -> Grammar:
    """A CNF of Query 2; the paper does not print it, reading c9."""
    binary = [("S", "B", "P_sc"), ("B", "P_scr", "B1"), ("B1", "B", "P_sc"), ("B", "P_scr", "P_sc")]
    terminal = [("S", SC), ("P_scr", SCR), ("P_sc", SC)]
    return Grammar(["S", "B", "B1", "P_scr", "P_sc"], binary, terminal)


def union_grammar() -> Grammar:
    """Config-4 grammar: Q1' ∪ Q2' with shared preterminals -> 10 NTs."""
    binary = [("S_Q1", "P_scr", "S5"), ("S_Q1", "P_tr", "S6"), ("S_Q1", "P_scr", "P_sc"),
              ("S_Q1", "P_tr", "P_t"), ("S5", "S_Q1", "P_sc"), ("S6", "S_Q1", "P_t"),
              ("S_Q2", "B", "P_sc"), ("B", "P_scr", "B1"), ("B1", "B", "P_sc"), ("B", "P_scr", "P_sc")]
    terminal = [("S_Q2", SC), ("P_scr", SCR), ("P_sc", SC), ("P_tr", TR), ("P_t", T)]
    return Grammar(["S_Q1", "S5", "S6", "S_Q2", "B", "B1", "P_scr", "P_sc", "P_tr", "P_t"],
                   binary, terminal)


def anbn_grammar() -> Grammar:
    """a^n b^n in CNF: S->AB | A S1, S1->S B, A->a, B->b (BASELINE.json configs[0])."""
    return Grammar(["S", "S1", "A", "B"],
                   [("S", "A", "B"), ("S", "A", "S1"), ("S1", "S", "B")],
                   [("A", "a"), ("B", "b")])


def dense_stress_grammar() -> Grammar:
    """S -> S S | a: closure = strict transitive closure of the a-edges (SURVEY V-5)."""
    return Grammar(["S"], [("S", "S", "S")], [("S", "a")])


def random_grammar(rng: np.random.Generator, n_nt: int, n_bin: int, n_term: int,
                   n_labels: int) -> Grammar:
    names = [f"N{k}" for k in range(n_nt)]
    labels = [f"l{k}" for k in range(n_labels)]
    binary = []
    for _ in range(n_bin):
        a, b, c = rng.integers(0, n_nt, size=3)
        binary.append((names[a], names[b], names[c]))
    terminal = []
    for _ in range(n_term):
        a = rng.integers(0, n_nt)
        x = rng.integers(0, n_labels)
        terminal.append((names[a], labels[x]))
    return Grammar(names, binary, terminal)


# ---------------------------------------------------------------------------------------------
# Graphs
# ---------------------------------------------------------------------------------------------

def example_edges() -> List[Tuple[int, str, int]]:
    """The graph of P:298-306 (figure missing), reconstructed uniquely from T0
    through the terminal rules P:288-291 (reading c1; same as S:129)."""
    return [(0, SCR, 0), (0, TR, 1), (1, TR, 2), (2, SC, 0), (2, T, 2)]


def two_cycle_edges(p: int, q: int) -> Tuple[int, List[Tuple[int, str, int]]]:
    """a-cycle 0->1->..->p-1->0 and b-cycle 0->p->p+1->..->p+q-2->0 sharing node 0.

    n = p+q-1 nodes, p 'a' edges and q 'b' edges (reading c2)."""
    n = p + q - 1
    e = [(k, "a", (k + 1) % p) for k in range(p)]
    bnodes = [0] + list(range(p, p + q - 1))
    e += [(bnodes[k], "b", bnodes[(k + 1) % q]) for k in range(q)]
    return n, e


def ontology_triples(n: int, depth: int = 10, seed: int = 0, n_triples: Optional[int] = None,
                     p_second_parent: float = 0.25, p_second_type: float = 0.4,
                     noise_per_node: float = 0.5, class_frac: float = 0.45
                     ) -> List[Tuple[int, str, int]]:
    """RDF-ontology-shaped triple set (SURVEY §8(d) 'Ontology-shaped generator').

    Node 0 = owl:Class (hub), node 1 = owl:Thing (root class, level 0); `class_frac`
    of the rest are classes on levels 1..depth, the others instances.  Every class
    has `type` owl:Class and `subClassOf` a class one level up (+ a second parent
    with p=0.25); every instance has `type` one class (+ a second with p=0.4).
    Noise triples on labels p0..p4 (no grammar rule) pad to `n_triples` exactly.
    """
    assert n >= depth + 3
    rng = np.random.default_rng(seed)
    HUB, ROOT = 0, 1
    n_rest = n - 2
    n_cls = max(depth, int(round(class_frac * n_rest)))
    cls = np.arange(2, 2 + n_cls)
    inst = np.arange(2 + n_cls, n)
    level = np.empty(n_cls, dtype=np.int64)
    level[:depth] = np.arange(1, depth + 1)
    level[depth:] = rng.integers(1, depth + 1, size=n_cls - depth)
    by_level: List[np.ndarray] = [np.array([ROOT])]
    for lv in range(1, depth + 1):
        by_level.append(cls[level == lv])
    trip = set()
    trip.add((ROOT, T, HUB))
    for c, lv in zip(cls.tolist(), level.tolist()):
        trip.add((c, T, HUB))
        up = by_level[lv - 1]
        trip.add((c, SC, int(up[rng.integers(0, len(up))])))
        if rng.random() < p_second_parent and len(up) > 1:
            trip.add((c, SC, int(up[rng.integers(0, len(up))])))
    all_cls = np.concatenate([[ROOT], cls])
    for x in inst.tolist():
        trip.add((x, T, int(all_cls[rng.integers(0, len(all_cls))])))
        if rng.random() < p_second_type:
            trip.add((x, T, int(all_cls[rng.integers(0, len(all_cls))])))
    structural = sorted(trip)
    n_noise = int(round(noise_per_node * n)) if n_triples is None else n_triples - len(structural)
    if n_noise < 0:
        raise ValueError(f"n_triples={n_triples} below the structural triple count {len(structural)}")
    noise = set()
    while len(noise) < n_noise:
        k = n_noise - len(noise)
        u = rng.integers(0, n, size=k)
        v = rng.integers(0, n, size=k)
        lab = rng.integers(0, 5, size=k)
        for a, b, l in zip(u.tolist(), v.tolist(), lab.tolist()):
            if len(noise) < n_noise:
                noise.add((a, f"p{l}", b))
    return structural + sorted(noise)


def triples_to_edges(triples: Sequence[Tuple[int, str, int]]) -> List[Tuple[int, str, int]]:
    """RDF -> graph: each triple (o,p,s) adds (o,p,s) and (s,p^-1,o); p^-1 spelt p_r
    (reading c10).  Triples are a set (deduplicated)."""
    out = []
    for o, p, s in sorted(set(triples)):
        out.append((o, p, s))
        out.append((s, p + "_r", o))
    return out


def disjoint_copies(n: int, edges: Sequence[Tuple[int, str, int]], k: int
                    ) -> Tuple[int, List[Tuple[int, str, int]]]:
    """g1..g3 of P:422 'simply repeating the existing graphs' = k disjoint copies (c11)."""
    out = []
    for c in range(k):
        out += [(s + c * n, x, d + c * n) for s, x, d in edges]
    return n * k, out


def relabel_nodes(n: int, edges: Sequence[Tuple[int, str, int]], seed: int
                  ) -> List[Tuple[int, str, int]]:
    perm = np.random.default_rng(seed + 7919).permutation(n)
    return [(int(perm[s]), x, int(perm[d])) for s, x, d in edges]


def random_digraph_edges(n: int, m: int, seed: int, label: str = "a"
                         ) -> List[Tuple[int, str, int]]:
    """G(n, m): m distinct directed non-loop edges, uniform."""
    rng = np.random.default_rng(seed)
    m = min(m, n * (n - 1))
    got = set()
    while len(got) < m:
        k = m - len(got)
        u = rng.integers(0, n, size=2 * k)
        v = rng.integers(0, n, size=2 * k)
        for a, b in zip(u.tolist(), v.tolist()):
            if a != b and len(got) < m:
                got.add((a, b))
    return [(a, label, b) for a, b in sorted(got)]


def random_labeled_edges(rng: np.random.Generator, n: int, n_edges: int, labels: Sequence[str]
                         ) -> List[Tuple[int, str, int]]:
    """Uniform random labelled edges; duplicates and self-loops allowed (c5, c6)."""
    e = []
    for _ in range(n_edges):
        e.append((int(rng.integers(0, n)), labels[int(rng.integers(0, len(labels)))],
                  int(rng.integers(0, n))))
    return e


# ---------------------------------------------------------------------------------------------
# Named workloads
# ---------------------------------------------------------------------------------------------

# Table 1 #triples of the 11 ontologies, used to size config 2.
TABLE1_TRIPLES = {"skos": 252, "generations": 273, "travel": 277, "univ-bench": 293,
                  "atom-primitive": 425, "biomedical-measure-primitive": 459, "foaf": 631,
                  "people-pets": 640, "funding": 1086, "wine": 1839, "pizza": 1980}


def example_workload() -> Workload:
    """Config 1b: P:249-386."""
    return bind("example", same_generation_grammar(), 3, example_edges(), "S")


def anbn_workload(p: int, q: int) -> Workload:
    """Config 1a (p=3,q=2) / 3 / 5 (p=2, q=n-1)."""
    n, e = two_cycle_edges(p, q)
    return bind(f"anbn_p{p}_q{q}", anbn_grammar(), n, e, "S", meta={"p": p, "q": q})


def ontology_workload(query: str, n: int, depth: int = 10, seed: int = 0,
                      n_triples: Optional[int] = None, copies: int = 1,
                      relabel: bool = True, name: Optional[str] = None) -> Workload:
    """Config 2 / 4: Q1 ('q1'), Q2 ('q2') or the union grammar ('union')."""
    trip = ontology_triples(n, depth=depth, seed=seed, n_triples=n_triples)
    edges = triples_to_edges(trip)
    nn = n
    if copies > 1:
        nn, edges = disjoint_copies(n, edges, copies)
    if relabel:
        edges = relabel_nodes(nn, edges, seed)
    g = {"q1": same_generation_grammar, "q2": q2_grammar, "union": union_grammar}[query]()
    start = {"q1": "S", "q2": "S", "union": "S_Q1"}[query]
    extra = [f"p{k}" for k in range(5)] + [f"p{k}_r" for k in range(5)] + [SC, SCR, T, TR]
    return bind(name or f"{query}_ont_n{nn}_d{depth}_s{seed}", g, nn, edges, start,
                extra_labels=extra,
                meta={"triples": len(trip) * copies, "depth": depth, "seed": seed, "copies": copies})


def config4_workload(seed: int = 0, n: int = 65536, depth: int = 10) -> Workload:
    """Config 4: union grammar on a 64k-node ontology-shaped graph."""
    return ontology_workload("union", n, depth=depth, seed=seed, name=f"config4_union_n{n}_d{depth}_s{seed}")


def dense_stress_workload(n: int, d: int, seed: int = 0) -> Workload:
    """Config S: S->SS|a on G(n, d*n)."""
    return bind(f"dense_n{n}_d{d}_s{seed}", dense_stress_grammar(), n,
                random_digraph_edges(n, d * n, seed), "S")


def random_workload(seed: int, max_nodes: int = 12, max_edges: int = 40, max_nt: int = 4,
                    max_bin: int = 8, max_term: int = 4, n_labels: int = 3) -> Workload:
    """SPEC S:456-style random instance (|V|<=12, |E|<=40, |N|<=4, <=8 binary, <=4 terminal)."""
    rng = np.random.default_rng(seed)
    n_nt = int(rng.integers(1, max_nt + 1))
    g = random_grammar(rng, n_nt, int(rng.integers(0, max_bin + 1)),
                       int(rng.integers(1, max_term + 1)), n_labels)
    n = int(rng.integers(1, max_nodes + 1))
    labels = [f"l{k}" for k in range(n_labels)]
    e = random_labeled_edges(rng, n, int(rng.integers(0, max_edges + 1)), labels)
    return bind(f"random_s{seed}", g, n, e, g.nt_names[0], extra_labels=labels)
