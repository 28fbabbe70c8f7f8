"""Thin Python binding of libcfpq (include/cfpq.h): argument marshalling only.

Every step of the CFPQ hot path (seed, semi-naive products, fused update and change
detection, fixpoint loop, extraction) runs in the CUDA kernels of libcfpq.so.  There
is no CPU fallback: if the library or a CUDA device is missing, calls raise.

Names follow the C-ABI: `cfpq_grammar_create` -> `grammar_create`, etc.
PyTorch is used only for device buffers and streams.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# CFPQ_CHECKED=1 selects the checked build (device bounds assertions; diagnostics only,
# `python paper_1707_01007_b200/build.py --checked`): the library itself reads no environment
LIB_PATH = os.path.join(HERE, "libcfpq_checked.so" if os.environ.get("CFPQ_CHECKED") == "1" else "libcfpq.so")

CFPQ_OK, CFPQ_E_INVAL, CFPQ_E_NOMEM, CFPQ_E_CUDA, CFPQ_E_NCCL = 0, -1, -2, -3, -4
CFPQ_E_NOT_CONVERGED, CFPQ_E_OVERFLOW, CFPQ_E_UNSUPPORTED = -5, -6, -7
_STATUS = {0: "CFPQ_OK", -1: "CFPQ_E_INVAL", -2: "CFPQ_E_NOMEM", -3: "CFPQ_E_CUDA", -4: "CFPQ_E_NCCL",
           -5: "CFPQ_E_NOT_CONVERGED", -6: "CFPQ_E_OVERFLOW", -7: "CFPQ_E_UNSUPPORTED"}

EXPORTS = [
    "cfpq_grammar_create", "cfpq_grammar_destroy", "cfpq_graph_create", "cfpq_graph_set_edges",
    "cfpq_graph_destroy", "cfpq_options_default", "cfpq_closure", "cfpq_closure_reuse",
    "cfpq_result_destroy", "cfpq_result_iterations", "cfpq_result_count", "cfpq_result_count_at",
    "cfpq_result_pairs", "cfpq_result_pairs_at", "cfpq_result_csr", "cfpq_result_matrix", "cfpq_result_lengths",
    "cfpq_result_stats", "cfpq_result_iteration_stats", "cfpq_result_iteration_stats2",
    "cfpq_result_iteration_phases", "cfpq_result_witness", "cfpq_last_error",
    "cfpq_version", "cfpq_nccl_unique_id", "cfpq_shard_rows", "cfpq_shard_block",
]


class CfpqError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {_STATUS.get(status, status)}: {msg}")
        self.status = status


class Options(ctypes.Structure):
    _fields_ = [("semantics", ctypes.c_int32), ("schedule", ctypes.c_int32),
                ("path_policy", ctypes.c_int32), ("account_work", ctypes.c_int32),
                ("max_iterations", ctypes.c_int64), ("cuda_stream", ctypes.c_void_p),
                ("world_size", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("log_capacity", ctypes.c_int64),
                ("solo_threshold", ctypes.c_int32), ("record_times", ctypes.c_int32),
                ("max_ctas", ctypes.c_int32), ("emulate_ranks", ctypes.c_int32),
                ("cell_set", ctypes.c_int32),
                ("tensor_format", ctypes.c_int32),
                ("dense_launch", ctypes.c_int32), ("diag_flags", ctypes.c_int32),
                ("grid_rows", ctypes.c_int32), ("grid_cols", ctypes.c_int32),
                ("rows_list_capacity", ctypes.c_int64), ("exchange", ctypes.c_int32)]


_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree libcfpq.so (built by __graft_entry__.build()); fail loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    i32, i64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
    P = ctypes.POINTER
    sig = {
        "cfpq_grammar_create": (i32, [i32, i32, vp, i64, vp, i64, P(vp)]),
        "cfpq_grammar_destroy": (None, [vp]),
        "cfpq_graph_create": (i32, [i64, vp, i64, i32, vp, P(vp)]),
        "cfpq_graph_set_edges": (i32, [vp, vp, i64, i32, vp]),
        "cfpq_graph_destroy": (None, [vp]),
        "cfpq_options_default": (None, [P(Options)]),
        "cfpq_closure": (i32, [vp, vp, P(Options), P(vp)]),
        "cfpq_closure_reuse": (i32, [vp, vp, P(Options), vp]),
        "cfpq_result_destroy": (None, [vp]),
        "cfpq_result_iterations": (i32, [vp, P(i64)]),
        "cfpq_result_count": (i32, [vp, i32, P(i64)]),
        "cfpq_result_count_at": (i32, [vp, i32, i64, P(i64)]),
        "cfpq_result_pairs": (i32, [vp, i32, vp, i64, i32, P(i64)]),
        "cfpq_result_pairs_at": (i32, [vp, i32, i64, vp, i64, i32, P(i64)]),
        "cfpq_result_matrix": (i32, [vp, i32, vp, i64, i32]),
        "cfpq_result_csr": (i32, [vp, i32, vp, vp, i64, i32, P(i64)]),
        "cfpq_result_lengths": (i32, [vp, i32, vp, i64, i32, P(i64)]),
        "cfpq_result_stats": (i32, [vp, P(i64), i32]),
        "cfpq_result_iteration_stats": (i32, [vp, vp, vp, i64]),
        "cfpq_result_iteration_stats2": (i32, [vp, vp, vp, vp, i64]),
        "cfpq_result_iteration_phases": (i32, [vp, vp, i64]),
        "cfpq_result_witness": (i32, [vp, vp, i32, i32, i32, vp, i64, i32, P(i64)]),
        "cfpq_last_error": (ctypes.c_char_p, []),
        "cfpq_version": (ctypes.c_char_p, []),
        "cfpq_nccl_unique_id": (i32, [vp, i64]),
        "cfpq_shard_rows": (i32, [i64, i32, i32, P(i64), P(i64)]),
        "cfpq_shard_block": (i32, [i64, i32, i32, i32, P(i64), P(i64), P(i64), P(i64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(st: int, where: str, ok=(CFPQ_OK,)):
    if st not in ok:
        raise CfpqError(st, where, load().cfpq_last_error().decode())
    return st


def version() -> str:
    return load().cfpq_version().decode()


def _host_i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr() if a.numel() else None
    return a.ctypes.data if a.size else None


def _is_device(a) -> bool:
    return hasattr(a, "is_cuda") and a.is_cuda


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Grammar:
    """cfpq_grammar_create: CNF rules A->BC (bin [m,3]) and A->x (term [t,2])."""

    def __init__(self, n_nt: int, n_labels: int, bin, term):
        self.n_nt, self.n_labels = int(n_nt), int(n_labels)
        b = _host_i32(bin).reshape(-1, 3)
        t = _host_i32(term).reshape(-1, 2)
        h = ctypes.c_void_p()
        _check(load().cfpq_grammar_create(self.n_nt, self.n_labels, _ptr(b), len(b), _ptr(t), len(t),
                                          ctypes.byref(h)), "cfpq_grammar_create")
        self._h = h

    @classmethod
    def from_workload(cls, w) -> "Grammar":
        return cls(w.n_nt, w.n_labels, w.bin, w.term)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cfpq_grammar_destroy(self._h)
            self._h = None


class Graph:
    """cfpq_graph_create: edges int32 [E,3] (src,label,dst) from host (numpy) or device (torch)."""

    def __init__(self, n_nodes: int, edges, stream=None):
        self.n_nodes = int(n_nodes)
        dev = _is_device(edges)
        e = edges.contiguous() if dev else _host_i32(edges).reshape(-1, 3)
        n_e = e.shape[0] if e.ndim == 2 else e.numel() // 3
        h = ctypes.c_void_p()
        _check(load().cfpq_graph_create(self.n_nodes, _ptr(e), int(n_e), int(dev), _stream_ptr(stream),
                                        ctypes.byref(h)), "cfpq_graph_create")
        self._h = h
        self.n_edges = int(n_e)

    def set_edges(self, edges, stream=None):
        """cfpq_graph_set_edges (the per-query host->device upload)."""
        dev = _is_device(edges)
        e = edges.contiguous() if dev else _host_i32(edges).reshape(-1, 3)
        n_e = e.shape[0] if e.ndim == 2 else e.numel() // 3
        _check(load().cfpq_graph_set_edges(self._h, _ptr(e), int(n_e), int(dev), _stream_ptr(stream)),
               "cfpq_graph_set_edges")
        self.n_edges = int(n_e)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cfpq_graph_destroy(self._h)
            self._h = None


def options(semantics: int = 0, schedule: int = 0, path_policy: int = 0, account_work: bool = False,
            max_iterations: int = 0, stream=None, log_capacity: int = 0, solo_threshold: int = -1,
            record_times: bool = False, max_ctas: int = 0, world_size: int = 1, rank: int = 0,
            nccl_unique_id=None, emulate_ranks: int = 0, flags: int = 0, cell_set: int = 0,
            tensor_format: int = 0, dense_launch: int = 0, grid: Tuple[int, int] = (0, 0),
            rows_list_capacity: int = 0, exchange: int = 0) -> Options:
    o = Options()
    load().cfpq_options_default(ctypes.byref(o))
    o.semantics, o.schedule, o.path_policy = int(semantics), int(schedule), int(path_policy)
    o.account_work = int(bool(account_work))
    o.max_iterations = int(max_iterations)
    o.cuda_stream = _stream_ptr(stream)
    o.log_capacity = int(log_capacity)
    o.solo_threshold = int(solo_threshold)
    o.record_times = int(bool(record_times))
    o.max_ctas = int(max_ctas)
    o.world_size = int(world_size)
    o.rank = int(rank)
    o.emulate_ranks = int(emulate_ranks)
    o.diag_flags = int(flags)
    o.dense_launch = int(dense_launch)
    o.grid_rows, o.grid_cols = int(grid[0]), int(grid[1])
    o.rows_list_capacity = int(rows_list_capacity)
    o.exchange = int(exchange)
    o.cell_set = int(cell_set)
    o.tensor_format = int(tensor_format)
    if nccl_unique_id is not None:
        buf = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
        o._uid = buf                     # keep alive with the options
        o.nccl_unique_id = ctypes.cast(buf, ctypes.c_void_p)
    return o


def nccl_unique_id() -> bytes:
    """cfpq_nccl_unique_id: 128 bytes to broadcast to every rank (torch.distributed)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().cfpq_nccl_unique_id(buf, 128), "cfpq_nccl_unique_id")
    return buf.raw


def shard_rows(n_nodes: int, world_size: int, rank: int) -> Tuple[int, int]:
    """cfpq_shard_rows: the row block [lo, hi) that `rank` computes."""
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(load().cfpq_shard_rows(int(n_nodes), int(world_size), int(rank), ctypes.byref(lo), ctypes.byref(hi)),
           "cfpq_shard_rows")
    return lo.value, hi.value


def shard_block(n_nodes: int, grid_rows: int, grid_cols: int, rank: int) -> Tuple[int, int, int, int]:
    """cfpq_shard_block: the 2-D block (row_lo, row_hi, col_lo, col_hi) of shard `rank`."""
    v = [ctypes.c_int64() for _ in range(4)]
    _check(load().cfpq_shard_block(int(n_nodes), int(grid_rows), int(grid_cols), int(rank), *[ctypes.byref(x) for x in v]),
           "cfpq_shard_block")
    return tuple(x.value for x in v)


class Result:
    """cfpq_result: the closure T^cf on the device plus its derived-cell log."""

    def __init__(self, handle, status: int, n_nt: int, n_nodes: int):
        self._h = handle
        self.status = status
        self.n_nt = n_nt
        self.n_nodes = n_nodes

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cfpq_result_destroy(self._h)
            self._h = None

    @property
    def iterations(self) -> int:
        v = ctypes.c_int64()
        _check(load().cfpq_result_iterations(self._h, ctypes.byref(v)), "cfpq_result_iterations")
        return v.value

    def count(self, A: int) -> int:
        v = ctypes.c_int64()
        _check(load().cfpq_result_count(self._h, int(A), ctypes.byref(v)), "cfpq_result_count")
        return v.value

    def count_at(self, A: int, k: int) -> int:
        v = ctypes.c_int64()
        _check(load().cfpq_result_count_at(self._h, int(A), int(k), ctypes.byref(v)), "cfpq_result_count_at")
        return v.value

    def pairs(self, A: int, out=None):
        """R_A as int32 [m,2] ascending (numpy).  `out` may be an int32 torch tensor [cap,2] on
        the device or in (pinned) host memory; then the pairs are written there and a view of
        its first |R_A| rows is returned."""
        w = ctypes.c_int64()
        if out is not None:
            _check(load().cfpq_result_pairs(self._h, int(A), _ptr(out), int(out.shape[0]), int(_is_device(out)),
                                            ctypes.byref(w)), "cfpq_result_pairs")
            return out[: w.value]
        m = self.count(A)
        buf = np.zeros((m, 2), dtype=np.int32)
        _check(load().cfpq_result_pairs(self._h, int(A), _ptr(buf), m, 0, ctypes.byref(w)), "cfpq_result_pairs")
        return buf[: w.value]

    def csr(self, A: int, row_ptr=None, cols=None):
        """R_A in compressed-row form: (row_ptr int64 [n+1], cols int32 [|R_A|]), columns ascending
        per row.  `row_ptr` / `cols` may be torch tensors (both on the device, or both in (pinned)
        host memory); then they are written and (row_ptr, cols[:|R_A|]) is returned."""
        w = ctypes.c_int64()
        if row_ptr is not None:
            _check(load().cfpq_result_csr(self._h, int(A), _ptr(row_ptr), _ptr(cols), int(cols.shape[0]),
                                          int(_is_device(row_ptr)), ctypes.byref(w)), "cfpq_result_csr")
            return row_ptr, cols[: w.value]
        m = self.count(A)
        rp = np.zeros(self.n_nodes + 1, dtype=np.int64)
        cs = np.zeros(max(m, 1), dtype=np.int32)
        _check(load().cfpq_result_csr(self._h, int(A), _ptr(rp), _ptr(cs), m, 0, ctypes.byref(w)), "cfpq_result_csr")
        return rp, cs[: w.value]

    def pairs_at(self, A: int, k: int) -> np.ndarray:
        """Pairs of A in T_k (Alg. 1 state after k loop bodies)."""
        m = self.count_at(A, k)
        buf = np.zeros((m, 2), dtype=np.int32)
        w = ctypes.c_int64()
        _check(load().cfpq_result_pairs_at(self._h, int(A), int(k), _ptr(buf), m, 0, ctypes.byref(w)),
               "cfpq_result_pairs_at")
        return buf[: w.value]

    def matrix(self, A: int) -> np.ndarray:
        """Bit matrix of A: uint32 [n, ceil(n/32)], bit j of row i = word j>>5 bit j&31."""
        wn = (self.n_nodes + 31) // 32
        buf = np.zeros((self.n_nodes, max(wn, 1)), dtype=np.uint32)
        _check(load().cfpq_result_matrix(self._h, int(A), _ptr(buf), max(wn, 1), 0), "cfpq_result_matrix")
        return buf

    def lengths(self, A: int) -> np.ndarray:
        """Single-path lengths of A, aligned with pairs(A)."""
        m = self.count(A)
        buf = np.zeros(m, dtype=np.uint32)
        w = ctypes.c_int64()
        _check(load().cfpq_result_lengths(self._h, int(A), _ptr(buf), m, 0, ctypes.byref(w)), "cfpq_result_lengths")
        return buf[: w.value]

    def stats(self) -> dict:
        v = (ctypes.c_int64 * 22)()
        _check(load().cfpq_result_stats(self._h, v, 22), "cfpq_result_stats")
        keys = ["iterations", "cells", "log_capacity", "regrows", "launches", "solo_iterations", "candidates",
                "expansions", "seed_ns", "loop_ns", "ctas", "prof_loop", "prof_expand", "prof_bar1",
                "prof_close", "prof_4", "prof_head", "prof_atomic", "mma_kblocks", "dense_finish", "hashed",
                "hash_capacity"]
        return dict(zip(keys, list(v)))

    def iteration_stats(self, work: bool = False) -> Tuple[np.ndarray, Optional[np.ndarray]]:
        k = self.iterations
        nc = np.zeros(k, dtype=np.int64)
        jt = np.zeros(k, dtype=np.int64) if work else None
        _check(load().cfpq_result_iteration_stats(self._h, _ptr(nc), _ptr(jt) if work else None, k),
               "cfpq_result_iteration_stats")
        return nc, jt

    def iteration_times(self) -> np.ndarray:
        """Device ns from the end of seeding to the end of each iteration."""
        k = self.iterations
        t = np.zeros(k, dtype=np.int64)
        _check(load().cfpq_result_iteration_stats2(self._h, None, None, _ptr(t), k), "cfpq_result_iteration_stats2")
        return t

    def witness(self, graph: "Graph", A: int, i: int, j: int) -> np.ndarray:
        """cfpq_result_witness: int32 [l, 3] edges (src, label, dst) of a path i -> j of the
        recorded single-path length l whose word A derives (semantics=1 runs)."""
        n = ctypes.c_int64(0)
        st = load().cfpq_result_witness(self._h, graph._h, int(A), int(i), int(j), None, 0, 0, ctypes.byref(n))
        if n.value <= 0:
            _check(st, "cfpq_result_witness")
        out = np.zeros((n.value, 3), dtype=np.int32)
        _check(load().cfpq_result_witness(self._h, graph._h, int(A), int(i), int(j), _ptr(out), n.value, 0,
                                          ctypes.byref(n)), "cfpq_result_witness")
        return out

    def iteration_phases(self) -> np.ndarray:
        """[k, 4] SM cycles per grid-wide iteration: expand, CTA flush, barrier (last
        arriver), close (record_times runs only)."""
        k = self.iterations
        c = np.zeros((k, 4), dtype=np.int64)
        _check(load().cfpq_result_iteration_phases(self._h, _ptr(c), k), "cfpq_result_iteration_phases")
        return c


def closure(grammar: Grammar, graph: Graph, opts: Optional[Options] = None, **kw) -> Result:
    """cfpq_closure: seed + Algorithm 1 loop to the fixpoint on the GPU."""
    o = opts if opts is not None else options(**kw)
    h = ctypes.c_void_p()
    st = _check(load().cfpq_closure(grammar._h, graph._h, ctypes.byref(o), ctypes.byref(h)), "cfpq_closure",
                ok=(CFPQ_OK, CFPQ_E_NOT_CONVERGED, CFPQ_E_OVERFLOW))
    return Result(h, st, grammar.n_nt, graph.n_nodes)


def closure_reuse(grammar: Grammar, graph: Graph, result: Result, opts: Optional[Options] = None, **kw) -> int:
    """cfpq_closure_reuse: re-run into an existing result's workspace."""
    o = opts if opts is not None else options(**kw)
    st = _check(load().cfpq_closure_reuse(grammar._h, graph._h, ctypes.byref(o), result._h),
                "cfpq_closure_reuse", ok=(CFPQ_OK, CFPQ_E_NOT_CONVERGED, CFPQ_E_OVERFLOW))
    result.status = st
    return st
