"""CPU bitset baseline of the CFPQ closure: uint64 bit rows,
semi-naive deltas, OpenMP over the host cores.

A second, independent CPU program: it shares no code with the oracle (`oracle/`, the root
of trust) nor with the CUDA product (`paper_1707_01007_b200/`).  bench.py times it on the
benched configuration itself (config 4, n = 65,536) beside the GPU number; tests check it
against the oracle and against the oracle's golden digests (tests/golden/config4_*.json).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bitset_cfpq.cpp")
_LIB = os.path.join(_HERE, "libbitset.so")
_lib = None


def build(force: bool = False) -> str:
    """g++ -O3 -fopenmp (portable flags: the .so may run on another host CPU)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O3", "-std=c++17", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i32, i64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
        lib.bitset_create.restype = vp
        lib.bitset_create.argtypes = [i64, i32, vp, i64, vp, i64]
        lib.bitset_destroy.argtypes = [vp]
        lib.bitset_run.restype = i64
        lib.bitset_run.argtypes = [vp, vp, i64, i32, i64]
        lib.bitset_seconds.restype = ctypes.c_double
        lib.bitset_seconds.argtypes = [vp]
        lib.bitset_threads.restype = i32
        lib.bitset_threads.argtypes = [vp]
        lib.bitset_num_cells.restype = i64
        lib.bitset_num_cells.argtypes = [vp]
        lib.bitset_iteration_stats.argtypes = [vp, vp, vp]
        lib.bitset_count.restype = i64
        lib.bitset_count.argtypes = [vp, i32]
        lib.bitset_pairs.restype = i64
        lib.bitset_pairs.argtypes = [vp, i32, vp]
        _lib = lib
    return _lib


def _c32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class BitsetBaseline:
    """One handle per (grammar, n): bitsets allocated and zeroed once; run() re-seeds."""

    def __init__(self, w):
        b = _c32(w.bin).reshape(-1, 3)
        t = _c32(w.term).reshape(-1, 2)
        self._keep = (b, t)
        self.n_nt = int(w.n_nt)
        self._h = _L().bitset_create(int(w.n_nodes), self.n_nt, b.ctypes.data if b.size else None, len(b),
                                     t.ctypes.data if t.size else None, len(t))
        if not self._h:
            raise MemoryError("bitset baseline: allocation failed or bad input")

    def __del__(self):
        if getattr(self, "_h", None):
            _L().bitset_destroy(self._h)
            self._h = None

    def run(self, edges, threads: int = 0, max_iterations: int = 0) -> int:
        e = _c32(edges).reshape(-1, 3)
        k = _L().bitset_run(self._h, e.ctypes.data if e.size else None, len(e), int(threads), int(max_iterations))
        if k < 0:
            raise ValueError("bitset baseline: edge out of range")
        return int(k)

    @property
    def seconds(self) -> float:
        return float(_L().bitset_seconds(self._h))

    @property
    def threads(self) -> int:
        return int(_L().bitset_threads(self._h))

    def iteration_stats(self, k: int):
        nc = np.zeros(k, np.int64)
        cand = np.zeros(k, np.int64)
        _L().bitset_iteration_stats(self._h, nc.ctypes.data, cand.ctypes.data)
        return nc, cand

    def count(self, A: int) -> int:
        return int(_L().bitset_count(self._h, int(A)))

    def pairs(self, A: int) -> np.ndarray:
        m = self.count(A)
        out = np.zeros((max(m, 1), 2), np.int32)
        _L().bitset_pairs(self._h, int(A), out.ctypes.data)
        return out[:m]
