#!/usr/bin/env python
"""Write full-size golden digests of the ORACLE's closure (test infrastructure only).

Calls only `oracle/` (Algorithm 1, plain std::set Jacobi loop) and the seeded
generators in `inputs/` — never the CUDA path — so that the -m gpu tests can compare every
engine with the oracle at the benched size (config 4, n = 65,536) and at n = 16,384.

Digest per workload (tests/golden/<name>.json):
  iterations            loop bodies incl. the final no-change pass
  new_cells[k-1]        |T_k \\ T_{k-1}| over all NTs (per-iteration Jacobi states)
  jacobi_triples[k-1]   AND-true triples of T_{k-1} x T_{k-1} (the work of Alg. 1 line 9)
  seminaive_triples[k-1] AND-true triples of the semi-naive pairs of iteration k
  count[A]              |R_A| (Theorem 2)
  sha256[A]             SHA-256 of R_A as int32 little-endian (i, j) pairs, ascending

  python scripts/golden_oracle_digest.py config4 65536 0
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs as I  # noqa: E402
import oracle as O  # noqa: E402


def digest(w, lengths=False):
    t0 = time.perf_counter()
    res = O.run(w, lengths=lengths)
    secs = time.perf_counter() - t0
    st = res.stats()
    out = {"workload": w.name, "n_nodes": int(w.n_nodes), "n_edges": int(len(w.edges)),
           "n_nt": int(w.n_nt), "nt_names": list(w.nt_names), "start": int(w.start),
           "status": int(res.status), "iterations": int(res.iterations),
           "new_cells": [int(x) for x in st["new_bits"]],
           "jacobi_triples": [int(x) for x in st["jacobi_triples"]],
           "seminaive_triples": [int(x) for x in st["seminaive_triples"]],
           "count": [], "sha256": [], "oracle_seconds": secs,
           "generated_by": "scripts/golden_oracle_digest.py (oracle/ only)"}
    for A in range(w.n_nt):
        p = np.ascontiguousarray(res.pairs(A).astype("<i4"))
        out["count"].append(int(len(p)))
        out["sha256"].append(hashlib.sha256(p.tobytes()).hexdigest())
    return out


def main():
    kind, n, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    if kind == "config4":
        w = I.config4_workload(seed=seed, n=n)
    else:
        raise SystemExit("unknown workload kind " + kind)
    d = digest(w)
    path = os.path.join(ROOT, "tests", "golden", f"{kind}_n{n}_s{seed}.json")
    with open(path, "w") as f:
        json.dump(d, f, indent=1)
    print(path, d["iterations"], d["count"][w.start], "%.1f s" % d["oracle_seconds"])


if __name__ == "__main__":
    main()
