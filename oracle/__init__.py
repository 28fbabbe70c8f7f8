"""ORACLE — TEST INFRASTRUCTURE ONLY (never on the product path).

Python face of the plain CPU oracle for the CFPQ closure of arXiv 1707.01007
(P:n = PAPER.md line n).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no
code with paper_1707_01007_b200/ and neither imports the other.

* `run()`            — Algorithm 1 in C++ (cfpq_oracle.cpp): seed,
                       Jacobi loop T <- T ∪ T×T, relations, lengths (min
                       tie-break = reading c7), per-iteration work counts.
* `witness()`        — single-path reconstruction "by a simple search".
* `cyk()`            — CYK membership for a word.
* `valiant_closure()`— Valiant's a⁺ = ∪ a⁽ⁱ⁾₊ with a⁽ⁱ⁾₊ = ∪_j a⁽ʲ⁾₊ × a⁽ⁱ⁻ʲ⁾₊,
                       pure Python, for tiny matrices (Theorem 1 pin).
* `paths_relations()`— brute force: every path of ≤ L edges, its word CYK-checked
                       (definition of R_A), pure Python, tiny graphs only.

Parity status: every function here is pinned by tests/test_oracle_*.py (see
DESIGN.md "Oracle pins"); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from itertools import product as _iproduct
from typing import Dict, List, Optional, Sequence, Set, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cfpq_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with plain g++ (no CUDA, no shared headers)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i32, i64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
        lib.oracle_run.restype = vp
        lib.oracle_run.argtypes = [i64, i32, vp, i64, vp, i64, vp, i64, i32, i32, i64]
        lib.oracle_free.argtypes = [vp]
        lib.oracle_status.argtypes = [vp]
        lib.oracle_status.restype = i32
        lib.oracle_iterations.argtypes = [vp]
        lib.oracle_iterations.restype = i64
        lib.oracle_count.argtypes = [vp, i32, i64]
        lib.oracle_count.restype = i64
        lib.oracle_pairs.argtypes = [vp, i32, i64, vp]
        lib.oracle_pairs.restype = i64
        lib.oracle_num_snapshots.argtypes = [vp]
        lib.oracle_num_snapshots.restype = i64
        lib.oracle_stats.argtypes = [vp, vp, vp, vp]
        lib.oracle_lengths.argtypes = [vp, i32, vp]
        lib.oracle_lengths.restype = i64
        lib.oracle_witness.argtypes = [i64, i32, vp, i64, vp, i64, vp, i64, vp, i64, i32, i64, i64, vp, i64]
        lib.oracle_witness.restype = i64
        lib.oracle_cyk.argtypes = [i32, vp, i64, vp, i64, vp, i64, i32]
        lib.oracle_cyk.restype = i32
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a.size else None


def _c32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class OracleResult:
    """Handle on one oracle run.  NT ids and node ids are the workload's."""

    def __init__(self, handle, n_nt: int):
        self._h = handle
        self.n_nt = n_nt

    def __del__(self):
        if getattr(self, "_h", None):
            _L().oracle_free(self._h)
            self._h = None

    @property
    def status(self) -> int:
        return _L().oracle_status(self._h)

    @property
    def iterations(self) -> int:
        """Loop bodies of Alg. 1 including the final no-change pass."""
        return _L().oracle_iterations(self._h)

    @property
    def num_snapshots(self) -> int:
        return _L().oracle_num_snapshots(self._h)

    def count(self, A: int, snap: int = -1) -> int:
        return _L().oracle_count(self._h, A, snap)

    def pairs(self, A: int, snap: int = -1) -> np.ndarray:
        """R_A (Theorem 2) as int32 [m,2], ascending (i,j); snap=k gives T_k."""
        c = self.count(A, snap)
        out = np.zeros((max(c, 0), 2), dtype=np.int32)
        if c > 0:
            _L().oracle_pairs(self._h, A, snap, _p(out))
        return out

    def relation_sets(self, snap: int = -1) -> Dict[int, Set[Tuple[int, int]]]:
        return {A: set(map(tuple, self.pairs(A, snap).tolist())) for A in range(self.n_nt)}

    def stats(self) -> Dict[str, np.ndarray]:
        k = self.iterations
        nb = np.zeros(k, np.int64)
        jt = np.zeros(k, np.int64)
        st = np.zeros(k, np.int64)
        _L().oracle_stats(self._h, _p(nb), _p(jt), _p(st))
        return {"new_bits": nb, "jacobi_triples": jt, "seminaive_triples": st}

    def lengths(self, A: int) -> np.ndarray:
        """(i, j, l_A) int64 [m,3] ascending (i,j) (reading c7)."""
        c = self.count(A)
        out = np.zeros((max(c, 0), 3), dtype=np.int64)
        if c > 0:
            got = _L().oracle_lengths(self._h, A, _p(out))
            if got < 0:
                raise RuntimeError("oracle run had no lengths")
        return out


def run(w, lengths: bool = False, snapshots: bool = False, max_iterations: int = 0) -> OracleResult:
    """Algorithm 1 on workload `w` (inputs.Workload or any object with the same fields)."""
    b = _c32(w.bin).reshape(-1, 3)
    t = _c32(w.term).reshape(-1, 2)
    e = _c32(w.edges).reshape(-1, 3)
    h = _L().oracle_run(int(w.n_nodes), int(w.n_nt), _p(b), len(b), _p(t), len(t), _p(e), len(e),
                        int(lengths), int(snapshots), int(max_iterations))
    if not h:
        raise ValueError("oracle_run rejected its input")
    return OracleResult(h, int(w.n_nt))


def witness(w, cells: np.ndarray, A: int, i: int, j: int, cap: Optional[int] = None
            ) -> Optional[np.ndarray]:
    """Reconstruct a path of the recorded length for (A,i,j) from a length table
    `cells` = int64 [m,4] rows (A, i, j, l).  Returns int32 [l,3] edges or None."""
    b = _c32(w.bin).reshape(-1, 3)
    t = _c32(w.term).reshape(-1, 2)
    e = _c32(w.edges).reshape(-1, 3)
    c = np.ascontiguousarray(np.asarray(cells, dtype=np.int64).reshape(-1, 4))
    if cap is None:
        sel = c[(c[:, 0] == A) & (c[:, 1] == i) & (c[:, 2] == j)]
        cap = int(sel[0, 3]) if len(sel) else 1
    out = np.zeros((max(cap, 1), 3), dtype=np.int32)
    m = _L().oracle_witness(int(w.n_nodes), int(w.n_nt), _p(b), len(b), _p(t), len(t), _p(e), len(e),
                            _p(c), len(c), int(A), int(i), int(j), _p(out), int(cap))
    if m < 0:
        return None
    return out[:m]


def cyk(w, word: Sequence[int], A: int) -> bool:
    """Does A derive the label word (label ids)?  CYK over the CNF rules."""
    b = _c32(w.bin).reshape(-1, 3)
    t = _c32(w.term).reshape(-1, 2)
    wd = _c32(list(word))
    return bool(_L().oracle_cyk(int(w.n_nt), _p(b), len(b), _p(t), len(t), _p(wd), len(wd), int(A)))


# ---------------------------------------------------------------------------------------------
# Pure-Python definitions for tiny inputs
# ---------------------------------------------------------------------------------------------

Cell = frozenset
SetMatrix = List[List[frozenset]]


def set_product(n1: frozenset, n2: frozenset, rules: Sequence[Tuple[int, int, int]]) -> frozenset:
    """N1 · N2 = {A | ∃B∈N1, ∃C∈N2, (A->BC)∈P}."""
    return frozenset(a for a, b, c in rules if b in n1 and c in n2)


def set_matmul(x: SetMatrix, y: SetMatrix, rules) -> SetMatrix:
    """c_ij = ∪_k a_ik · b_kj."""
    n = len(x)
    out = []
    for i in range(n):
        row = []
        for j in range(n):
            acc = frozenset()
            for k in range(n):
                acc = acc | set_product(x[i][k], y[k][j], rules)
            row.append(acc)
        out.append(row)
    return out


def set_union(x: SetMatrix, y: SetMatrix) -> SetMatrix:
    return [[x[i][j] | y[i][j] for j in range(len(x))] for i in range(len(x))]


def valiant_closure(a: SetMatrix, rules, n_terms: int) -> SetMatrix:
    """∪_{i=1..n_terms} a⁽ⁱ⁾₊ with a⁽¹⁾₊ = a, a⁽ⁱ⁾₊ = ∪_{j=1}^{i-1} a⁽ʲ⁾₊ × a⁽ⁱ⁻ʲ⁾₊."""
    terms = [None, a]
    for i in range(2, n_terms + 1):
        acc = [[frozenset() for _ in a] for _ in a]
        for j in range(1, i):
            acc = set_union(acc, set_matmul(terms[j], terms[i - j], rules))
        terms.append(acc)
    out = terms[1]
    for i in range(2, n_terms + 1):
        out = set_union(out, terms[i])
    return out


def paths_relations(w, max_len: int, max_paths: int = 2_000_000) -> Dict[int, Set[Tuple[int, int]]]:
    """Brute force of the definition R_A = {(n,m) | ∃ n π m, l(π) ∈ L(G_A)}:
    enumerate every path with 1..max_len edges, CYK its word for every A."""
    n = int(w.n_nodes)
    edges = sorted(set(map(tuple, np.asarray(w.edges).tolist())))
    out_e: List[List[Tuple[int, int]]] = [[] for _ in range(n)]
    for s, x, d in edges:
        out_e[s].append((x, d))
    rel: Dict[int, Set[Tuple[int, int]]] = {A: set() for A in range(int(w.n_nt))}
    seen_words: Dict[Tuple[int, ...], List[int]] = {}
    budget = [max_paths]

    def derivers(word: Tuple[int, ...]) -> List[int]:
        if word not in seen_words:
            seen_words[word] = [A for A in range(int(w.n_nt)) if cyk(w, word, A)]
        return seen_words[word]

    def dfs(start: int, node: int, word: Tuple[int, ...]):
        budget[0] -= 1
        if budget[0] < 0:
            raise RuntimeError("path enumeration budget exceeded")
        for A in derivers(word):
            rel[A].add((start, node))
        if len(word) == max_len:
            return
        for x, d in out_e[node]:
            dfs(start, d, word + (x,))

    for s in range(n):
        for x, d in out_e[s]:
            dfs(s, d, (x,))
    return rel


def seed_set_matrix(w) -> SetMatrix:
    """a_ij = {A_k | (i,x,j)∈E ∧ (A_k->x)∈P}."""
    n = int(w.n_nodes)
    m = [[set() for _ in range(n)] for _ in range(n)]
    for s, x, d in np.asarray(w.edges).tolist():
        for a, lab in np.asarray(w.term).tolist():
            if lab == x:
                m[s][d].add(a)
    return [[frozenset(c) for c in row] for row in m]
