#!/usr/bin/env python
"""Benchmark of the CFPQ closure hot path (arXiv 1707.01007, Algorithm 1) on B200.

One step = one full closure of the workload: seed T_0 from the edges and
run T <- T ∪ T×T to the fixpoint, inputs resident in HBM.  Default
workload = SURVEY §8(d) config 4: the 10-NT Q1∪Q2 union grammar on a 64k-node
ontology-shaped graph (the largest config, the one BASELINE's metric quotes at
1/2/4/8 GPUs).

value = effective boolean Gop/s of the EXECUTED schedule (SURVEY §8(d) "useful boolean
ops ... summed over the semi-naive pairs"): 2 x the (Δ entry, neighbour) pairs the
semi-naive engine expands (stats.candidates: AND-true triples of Δ_B x T_C and T_B x Δ_C
on the operand sides the engine expands) / closure time.  The dense tensor engine executes
full Jacobi products, so its numerator is 2 x the AND-true triples of T_{k-1} x T_{k-1}.
The Jacobi-equivalent rate (2 x AND-true triples of Alg. 1 line 9 on sparse operands,
identical for every exact schedule) is reported beside it as `jacobi_equivalent`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload config4|config3|config5|config2|configS]
  python bench.py --impl reference ...   # the CPU oracle as the reference arm

Multi-GPU (torchrun, N>1): one process per GPU; time = max over ranks of the
device-timed region.  config 4 and config S close ONE problem row-block sharded over the
ranks ("scaling": "strong"): config 4 on the sparse engine (each rank derives the cells
of its rows, Δ_k exchanged as index lists over NCCL every iteration) with the
paper-faithful bit-row engine sharded the same way as a supplement (Δ word lists
exchanged); config S on the tcgen05 engine (row blocks all-gathered).  N independent
seeded replicas are timed as a supplement (--replicas makes them the headline).
config2/3/5: replicas.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CFPQ closure time (ms) & boolean Gop/s vs roofline at 1/2/4/8 B200"
UNIT = "Gop/s"
HBM_FALLBACK = 6650.0   # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ------------------------------------------------------------------------------------------
# workloads
# ------------------------------------------------------------------------------------------

def make_workload(name: str, seed: int):
    import inputs as I
    if name == "config4":
        w = I.config4_workload(seed=seed)
        desc = {"workload": "config4: Q1∪Q2 union CNF (10 NTs) on ontology-shaped graph, n=65536, depth 10",
                "grammar": "union (S_Q1,S5,S6,S_Q2,B,B1,P_scr,P_sc,P_tr,P_t)"}
    elif name in ("config3", "config5"):
        w = I.anbn_workload(2, 16383)
        desc = {"workload": f"{name}: a^n b^n on coprime cycles p=2, q=16383 (n=16384), worst case"
                            + (", single-path lengths" if name == "config5" else ""),
                "grammar": "a^n b^n CNF (S,S1,A,B)"}
    elif name == "config2":
        w = I.ontology_workload("q1", int(1980 / 2.28), depth=8, seed=seed, n_triples=1980, copies=8)
        desc = {"workload": "config2: Q1 on 8 disjoint copies of a pizza-sized (1980 triples) ontology graph",
                "grammar": "same-generation G' (P:279-296)"}
    elif name == "configS":
        w = I.dense_stress_workload(16384, 2, seed)
        desc = {"workload": "configS: S->SS|a on G(n=16384, m=2n), dense tcgen05 engine (fp4 kind::mxf4)",
                "grammar": "S->SS|a"}
    else:
        raise SystemExit(f"unknown workload {name}")
    desc.update({"n_nodes": w.n_nodes, "n_edges": int(len(w.edges)), "seed": seed})
    return w, desc


def policy_for(name):
    """Dense var x var grammar -> the tcgen05 engine; the paper's grammars -> sparse engine."""
    return 2 if name == "configS" else 0


def jacobi_ops(w, name, g, d, C, stream):
    """2 x AND-true triples of T_{k-1} x T_{k-1} over all iterations (untimed accounting)."""
    if name in ("config3", "config5"):
        # closed form (tests/test_oracle_pins.py): iteration k has exactly k triples
        p, q = w.meta["p"], w.meta["q"]
        it = 2 * p * q + 1
        return 2 * it * (it + 1) // 2
    r = C.closure(g, d, account_work=True, stream=stream, semantics=int(name == "config5"),
                  path_policy=policy_for(name))
    _, jt = r.iteration_stats(work=True)
    return 2 * int(jt.sum())


# ------------------------------------------------------------------------------------------
# clocks (NVML polled during the timed region)
# ------------------------------------------------------------------------------------------

class ClockSampler:
    def __init__(self, index: int, period: float = 0.002):
        self.index, self.period = index, period
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        N = self.N
        names = {"hw_slowdown": getattr(N, "nvmlClocksEventReasonHwSlowdown", 0x8),
                 "hw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                 "sw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                 "sw_power_cap": getattr(N, "nvmlClocksEventReasonSwPowerCap", 0x4),
                 "hw_power_brake": getattr(N, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80)}
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                try:
                    rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    rs = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if rs & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------
# peaks, profiles
# ------------------------------------------------------------------------------------------

def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str):
    """dram bytes per launch of the closure kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "closure_kernel_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(workload)
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


def probe_random_access(footprint_bytes: int, n_ops: int = 1 << 25):
    """Random-access peaks over a buffer the size of the bit matrices, measured on this GPU
    with library kernels (like the int8 peak): independent random 4-byte atomicAdds
    (`index_add_`, the read-modify-write a bit insertion costs) and random 4-byte loads
    (`take`), G ops/s, best of 3.  The closure kernel's unit of work is one random bit test
    (+ set) per candidate into 5.4 GB of matrices, so these rates — not streaming bandwidth —
    are what its memory system can deliver."""
    import torch
    words = max(1, footprint_bytes // 4)
    try:
        buf = torch.zeros(words, dtype=torch.int32, device="cuda")
        idx = torch.randint(0, words, (n_ops,), dtype=torch.int64, device="cuda")
        one = torch.ones(n_ops, dtype=torch.int32, device="cuda")
        res = {}
        for name, fn in (("atomic", lambda: buf.index_add_(0, idx, one)), ("load", lambda: torch.take(buf, idx))):
            fn()
            best = None
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                e1.synchronize()
                ms = e0.elapsed_time(e1)
                best = ms if best is None else min(best, ms)
            res[name] = n_ops / (best * 1e-3) / 1e9
        del buf, idx, one
        torch.cuda.empty_cache()
        return res
    except Exception as ex:   # e.g. not enough free memory next to the closure's buffers
        return {"error": str(ex)[:120]}


_INT8_PROBE = {}


def probe_int8_tops():
    """Dense int8 tensor throughput measured on this GPU: torch._int_mm (cuBLASLt) on
    8192^3 int8 -> int32, best of 10 (the same method as MEASURED_PEAKS' bf16 probe).
    Cached per process; None if the probe is unavailable."""
    if "tops" in _INT8_PROBE:
        return _INT8_PROBE["tops"]
    tops = None
    try:
        import torch
        n = 8192
        a = torch.randint(-4, 4, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-4, 4, (n, n), dtype=torch.int8, device="cuda")
        for _ in range(3):
            torch._int_mm(a, b)
        best = None
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        tops = 2.0 * n ** 3 / (best * 1e-3) / 1e12
        del a, b
    except Exception:
        tops = None
    _INT8_PROBE["tops"] = tops
    return tops


def int8_peak():
    """Dense int8 tensor peak: the torch._int_mm probe on this GPU when available, else the
    measured bf16 (MEASURED_PEAKS.json) x the nominal int8/bf16 ratio (2)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        derived = 2.0 * float(d["bf16_tflops"]), 2.0 * float(d["bf16_tflops_sustained"]), \
            "measured bf16 x 2 (nominal int8/bf16)"
    except Exception:
        derived = 2.0 * 1590.0, 2.0 * 1400.0, "fallback bf16 x 2 (B200_PROFILING.md)"
    probed = probe_int8_tops()
    if probed:
        return probed, probed * derived[1] / derived[0], "measured: torch._int_mm 8192^3 int8, best of 10 (this run)"
    return derived


def fp4_peak():
    """Dense FP4 (kind::mxf4) tensor peak = the int8 peak x the nominal fp4/int8 ratio
    (9 / 4.5 = 2; no fp4 library GEMM to probe)."""
    b, s, src = int8_peak()
    return 2.0 * b, 2.0 * s, src + " x 2 (nominal fp4/int8)"


TENSOR_FORMATS = {1: "int8", 2: "fp4"}


def tensor_roofline(stats, step_ms, fmt=2):
    """Issued tensor work of the dense engine over the device time of the fixpoint loop (all
    tcgen05 product launches + packs of every iteration): the library counts issued MMA work in
    units of 128 x 32 x 128 multiply-adds (2*128*32*128 ops; an M=128 x N=256 int8 k-block is
    8 units, a 256-deep fp4 k-block 16).  Peak of the format:
    int8 = bf16 x 2, fp4 = bf16 x 4 (measured bf16, nominal ratios)."""
    ops = stats["mma_kblocks"] * 2 * 128 * 32 * 128
    loop_s = stats["loop_ns"] * 1e-9
    burst, sustained, src = fp4_peak() if fmt == 2 else int8_peak()
    achieved = ops / loop_s / 1e12
    kind = "kind::mxf4, e2m1 0/1, unit ue8m0 scales, f32 accumulator" if fmt == 2 else "kind::i8"
    nominal = 9000.0 if fmt == 2 else 4500.0   # dense fp4 / int8 datasheet figures (context only)
    return {"bound": "tensor", "achieved": achieved, "peak": burst, "unit": "TFLOP/s", "frac": achieved / burst,
            "int8_probe_tops": probe_int8_tops(),
            "frac_of_sustained": achieved / sustained, "frac_of_nominal": achieved / nominal, "traffic": ncu_traffic("configS" if fmt == 2 else "configS_int8"),
            "kernel": f"cfpq::dense2sm_kernel (tcgen05.mma.cta_group::2 {kind}, CTA pairs)", "format": TENSOR_FORMATS[fmt],
            "loop_ms": loop_s * 1e3, "share_of_step": loop_s * 1e3 / step_ms, "issued_ops": ops, "peak_source": src,
            "note": f"{TENSOR_FORMATS[fmt]} TOPS reported in the TFLOP/s slot; issued work counts whole output "
                    "tiles x live K blocks (zeros inside tiles included); the peak is the measured cuBLAS bf16 "
                    "burst x the nominal format ratio, which a tuned kernel can exceed slightly (frac_of_nominal "
                    "is against the datasheet's dense figure)"}


def supplementary_tensor(C, stream, steps=3, fmt=2):
    """Config S (S->SS|a, n=16384) on the tcgen05 engine: the tensor-path roofline beside the
    headline line (untimed by the driver's contract; its own CUDA-event timing)."""
    import inputs as I
    import torch
    w = I.dense_stress_workload(16384, 2, 0)
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda(), stream=stream)
    r = C.closure(g, d, path_policy=2, tensor_format=fmt, stream=stream)
    C.closure_reuse(g, d, r, path_policy=2, tensor_format=fmt, stream=stream)
    t = []
    st = None
    for _ in range(steps):
        C.closure_reuse(g, d, r, path_policy=2, tensor_format=fmt, stream=stream)
        st = r.stats()
        t.append(st["loop_ns"] + st["seed_ns"])
    ms = statistics.mean(t) * 1e-6
    roof = tensor_roofline(st, ms, fmt)
    out = {"workload": "configS: S->SS|a, G(16384, 32768)", "format": TENSOR_FORMATS[fmt], "closure_ms": ms,
           "iterations": r.iterations, "cells": r.count(0), "roofline": roof}
    del r
    return out


def rows_alg_bytes(w, r_sparse):
    """Algorithmic bytes of the bit-row path (path_policy 3): the full Jacobi product
    T_{k-1} x T_{k-1} of every rule at every iteration k, in the form the kernels evaluate it
    (DESIGN §3.3), each distinct row / index entry read once per rule and iteration:
      L (B changes, C preterminal): 4W per non-empty row of T_B (bit-row scan, once per B for
        all L rules sharing it) + 8 B per set
        bit (its CSR_C row pointers) + 4 B per CSR_C entry reached (candidate index)
      R (B preterminal, C changes): 8 B per row of CSR_B + 4 B per CSR_B entry + 4W per
        distinct non-empty row of T_C referenced
      V (both change): 4W per non-empty row of T_B + 4W per distinct non-empty row of T_C
        referenced
      P (both preterminal, iteration 1 only): 8 B per CSR_B row + 4 B per CSR_B entry + 8 B
        per entry (CSR_C pointers) + 4 B per candidate
      every form: 8 B per distinct output word the product touches (pre-check read + merge)
      per iteration: 32 B per word of T_k that gained bits (Δ_k word list: write + apply);
        iteration 1: 8 B per seed cell (T_0 into the second buffer).
    W = ceil(n/32) words per row.  T_{k-1} per NT comes from the sparse run's log."""
    import numpy as np
    import scipy.sparse as sp
    n = w.n_nodes
    W = (n + 31) // 32
    K = r_sparse.iterations
    rules = [tuple(x) for x in np.unique(w.bin.reshape(-1, 3), axis=0).tolist()]
    lhs = {A for A, _, _ in rules}
    pre = [X not in lhs for X in range(w.n_nt)]
    cache = {}

    def at(X, k):
        if (X, k) not in cache:
            cache[(X, k)] = r_sparse.pairs_at(X, k)
        return cache[(X, k)]

    def mat(pairs):
        return sp.csr_matrix((np.ones(len(pairs), np.int8), (pairs[:, 0], pairs[:, 1])), shape=(n, n))

    def words(P):
        P = P.tocoo()
        return len(np.unique(P.row.astype(np.int64) * W + P.col // 32)) if P.nnz else 0

    total = 8 * sum(len(at(X, 0)) for X in range(w.n_nt))
    for k in range(1, K + 1):
        scanned = set()   # L-form rules with the same B share one scan of each row of T_B
        for A, B, C in rules:
            pb, pc = at(B, k - 1), at(C, k - 1)
            lform = not pre[B] and pre[C]
            scan = 4 * W * len(np.unique(pb[:, 0])) if len(pb) else 0
            if lform:
                scan = 0 if B in scanned else scan
                scanned.add(B)
            if len(pb) == 0 or len(pc) == 0:
                if not pre[B] and len(pb):
                    total += scan   # the row is still scanned
                continue
            MB, MC = mat(pb), mat(pc)
            degC = np.diff(MC.indptr)
            P = (MB.astype(np.int32) @ MC.astype(np.int32))
            if lform:
                total += scan + 8 * len(pb) + 4 * int(degC[pb[:, 1]].sum())
            elif pre[B] and not pre[C]:
                ref = np.unique(pb[:, 1])
                total += 8 * len(np.unique(pb[:, 0])) + 4 * len(pb) + 4 * W * int((degC[ref] > 0).sum())
            elif not pre[B] and not pre[C]:
                ref = np.unique(pb[:, 1])
                total += 4 * W * len(np.unique(pb[:, 0])) + 4 * W * int((degC[ref] > 0).sum())
            else:
                if k > 1:
                    continue
                total += 8 * len(np.unique(pb[:, 0])) + 12 * len(pb) + 4 * int(degC[pb[:, 1]].sum())
            total += 8 * words(P)
        # Δ_k word list: words of T_k that gained bits
        for A in lhs:
            new = at(A, k)
            if len(new) == len(at(A, k - 1)):
                continue
            Mk, Mp = mat(new), mat(at(A, k - 1)) if len(at(A, k - 1)) else None
            D = Mk if Mp is None else (Mk - Mp)
            D.eliminate_zeros()
            total += 32 * words(D)
    return total


def supplementary_rows(C, w, g, d, r_sparse, stream, steps=3):
    """Config 4 in the paper-faithful full-operand mode (path_policy 3, bit-row CUDA-core
    products of Alg. 1 line 9 over whole matrices), with its HBM roofline on SURVEY §8(d)'s
    algorithmic bytes (rows_alg_bytes)."""
    n = w.n_nodes
    K = r_sparse.iterations
    alg = rows_alg_bytes(w, r_sparse)
    r = C.closure(g, d, path_policy=3, stream=stream)
    t = []
    for _ in range(steps):
        C.closure_reuse(g, d, r, path_policy=3, stream=stream)
        t.append(r.stats()["loop_ns"] * 1e-9)
    loop_s = statistics.mean(t)
    ok = r.iterations == K and all(r.count(X) == r_sparse.count(X) for X in range(w.n_nt))
    peak, src = hbm_peak()
    return {"workload": "config4 (same graph), path_policy 3: full-operand bit-row products",
            "closure_ms": (loop_s + r.stats()["seed_ns"] * 1e-9) * 1e3, "iterations": r.iterations,
            "same_result_as_sparse": ok,
            "roofline": {"bound": "hbm", "achieved": alg / loop_s / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / loop_s / 1e9 / peak, "traffic": ncu_traffic("config4_rows"),
                         "kernel": "cfpq::rows_compact_kernel<0/1> + rows_lmerge/rows_rmerge_kernel (+ plan, delta, "
                                   "reset, end): every launch of the loop; alg_bytes and traffic per closure",
                         "alg_bytes": alg, "peak_source": src,
                         "note": "model of the implemented full-operand forms (DESIGN 3.3, bench.rows_alg_bytes): "
                                 "each distinct bit row / CSR entry read once per rule and iteration, 8 B per "
                                 "output word touched, 32 B per Delta word"}}


def job_totals(dist, world, sharded, total_ms, useful, jac, device):
    """Whole-job aggregation over the ranks: time = MAX over ranks of the device-timed region;
    work per step = the one sharded problem's work counted once, or the sum over replicas."""
    import torch
    if world <= 1:
        return float(total_ms), float(useful), float(jac)
    my = torch.tensor([total_ms, float(useful), float(jac)], dtype=torch.float64, device=device)
    t_max = my[0:1].clone()
    dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    o_sum = my[1:3].clone()
    if not sharded:
        dist.all_reduce(o_sum, op=dist.ReduceOp.SUM)
    return float(t_max.item()), float(o_sum[0].item()), float(o_sum[1].item())


def supplementary_rows_sharded(C, w, g, d, args, rank, world, stream, dist, shard_kw):
    """Config 4 in the paper-faithful full-operand mode (bit-row engine, path_policy 3) closed
    as ONE problem row-block sharded over the ranks (Δ_k word lists exchanged over NCCL),
    time = max over ranks; rank 0 also times the unsharded 1-GPU closure of the same problem
    (the other ranks wait) so the line carries its own speedup."""
    import torch
    r = C.closure(g, d, stream=stream, path_policy=3, **shard_kw)
    for _ in range(max(args.warmup // 2, 1)):
        C.closure_reuse(g, d, r, stream=stream, path_policy=3, **shard_kw)
    torch.cuda.synchronize()
    dist.barrier()
    steps = max(args.steps // 4, 2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        C.closure_reuse(g, d, r, stream=stream, path_policy=3, **shard_kw)
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / steps
    one = None
    if rank == 0:
        r1 = C.closure(g, d, stream=stream, path_policy=3)
        C.closure_reuse(g, d, r1, stream=stream, path_policy=3)
        e0.record(stream)
        for _ in range(steps):
            C.closure_reuse(g, d, r1, stream=stream, path_policy=3)
        e1.record(stream)
        torch.cuda.synchronize()
        one = e0.elapsed_time(e1) / steps
        del r1
    dist.barrier()
    return {"workload": "config4, ONE problem, bit-row engine row-sharded over %d GPUs (NCCL word-list exchange)"
                        % world, "ms_per_step": ms, "iterations": r.iterations, "scaling": "strong",
            "one_gpu_ms_per_step": one, "speedup_vs_1gpu": (one / ms) if one else None}


def supplementary_replicas(C, args, rank, world, stream, dist):
    """N > 1: N independent seeded config-4 problems (seed + rank), one per GPU, single-GPU
    engine, no data-path collective ("scaling": "weak").  Time = max over ranks."""
    import torch
    w, _ = make_workload(args.workload, args.seed + rank)
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda(), stream=stream)
    r = C.closure(g, d, stream=stream)
    useful = 2 * int(r.stats()["candidates"])
    for _ in range(args.warmup):
        C.closure_reuse(g, d, r, stream=stream)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        C.closure_reuse(g, d, r, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1), float(useful)], dtype=torch.float64, device="cuda")
    tm, us = t[0:1].clone(), t[1:2].clone()
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    dist.all_reduce(us, op=dist.ReduceOp.SUM)
    ms = float(tm.item()) / args.steps
    return {"workload": "%d independent config-4 problems (seed + rank), one per GPU" % world, "ms_per_step": ms,
            "value": float(us.item()) / (ms * 1e-3) / 1e9, "unit": "Gop/s", "scaling": "weak"}


# ------------------------------------------------------------------------------------------
# CPU baselines: the oracle (reference arm / cpu_baseline, bounded sample) and the
# independent OpenMP bitset program (cpu_bitset, the full benched configuration)
# ------------------------------------------------------------------------------------------

def oracle_sample(name: str, seed: int, n4: int = 2048):
    import inputs as I
    if name == "config4":
        return I.config4_workload(seed=seed, n=n4), f"config-4 generator at n={n4} (depth 10): full closure"
    if name in ("config3", "config5"):
        return I.anbn_workload(2, 255), "a^n b^n p=2, q=255 (n=256, 1021 iterations): full closure"
    if name == "config2":
        return (I.ontology_workload("q1", int(1980 / 2.28), depth=8, seed=seed, n_triples=1980),
                "one pizza-sized copy (1980 triples) of the config-2 graph: full closure")
    return I.dense_stress_workload(320, 2, seed), "S->SS|a on G(320, 640): full closure"


def sample_numerator(name: str, w):
    """The work unit of `value` on a CPU sample, in the same definition as our arm: 2 x the
    semi-naive (Δ entry, neighbour) pairs (counted by the independent bitset program, whose
    expansion rules are the engine's: tests/test_gpu_units.py) — or, for the dense config S,
    2 x the Jacobi AND-true triples (the oracle's own count)."""
    if name == "configS":
        return None
    import cpu_baseline as CB
    b = CB.BitsetBaseline(w)
    k = b.run(w.edges)
    _, cand = b.iteration_stats(k)
    return 2 * int(cand.sum())


def time_oracle(name: str, seed: int, reps: int = 1, n4: int = 2048):
    import oracle as O
    w, sample = oracle_sample(name, seed, n4)
    lengths = name == "config5"
    num = sample_numerator(name, w)
    ts, ops = [], 0
    for _ in range(reps):
        t0 = time.perf_counter()
        res = O.run(w, lengths=lengths)
        ts.append(time.perf_counter() - t0)
        ops = num if num is not None else 2 * int(res.stats()["jacobi_triples"].sum())
    return ops, ts, sample, w


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    _, desc = make_workload(args.workload, args.seed)
    _, _, sample, sw = time_oracle(args.workload, args.seed)   # warm the oracle build / sample
    for _ in range(max(args.warmup - 1, 0)):
        time_oracle(args.workload, args.seed)
    ops, ts = 0, []
    for _ in range(args.steps):
        o, t, sample, sw = time_oracle(args.workload, args.seed)
        ops += o
        ts += t
    total = sum(ts)
    value = ops / total / 1e9
    ms = 1e3 * total / len(ts)
    sdesc = {"what": sample, "n_nodes": int(sw.n_nodes), "n_edges": int(len(sw.edges))}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "set<int> cells (CPU)", "data": "synthetic",
            "config": {**desc, "sample": sdesc, "same_config": False,
                       "note": "each step closes the bounded sample (n_nodes/n_edges above), not the full "
                               "workload; value is in the same unit as our arm (2 x semi-naive pairs of the "
                               "instance / time), so the ratio compares rates on instances of different size"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_bitset(name: str, w, r, n_nt: int, reps: int = 3):
    """The independent OpenMP bitset program on the FULL benched instance (all host cores),
    single-thread time beside it; its relations are checked against the GPU result's counts."""
    if name == "configS":
        return None
    import cpu_baseline as CB
    b = CB.BitsetBaseline(w)
    cores = host_cores()
    k = b.run(w.edges, threads=cores)
    ts = []
    for _ in range(reps):
        b.run(w.edges, threads=cores)
        ts.append(b.seconds)
    _, cand = b.iteration_stats(k)
    num = 2 * int(cand.sum())
    same = k == r.iterations and all(b.count(A) == r.count(A) for A in range(n_nt))
    b.run(w.edges, threads=1)
    t1 = b.seconds
    sec = statistics.median(ts)
    return {"value": num / sec / 1e9, "unit": UNIT, "cores": cores, "kind": "bitset (uint64 rows, semi-naive, OpenMP)",
            "sample": "the full benched instance", "seconds": sec, "single_thread_seconds": t1,
            "single_thread_value": num / t1 / 1e9, "iterations": k, "same_relations_as_gpu": bool(same),
            "source": "cpu_baseline/bitset_cfpq.cpp"}


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config4", choices=["config4", "config3", "config5", "config2", "configS"])
    ap.add_argument("--tensor-format", type=int, default=0, choices=[0, 1, 2],
                    help="tensor engine operands: 0 auto (fp4), 1 int8 (kind::i8), 2 fp4 (kind::mxf4)")
    ap.add_argument("--schedule", type=int, default=0, choices=[0, 3],
                    help="0 Jacobi (Alg. 1 states), 3 Gauss-Seidel (in-place stages, same fixpoint)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-format", default="csr", choices=["csr", "pairs"],
                    help="end-to-end result read back: CSR (default) or (i, j) pairs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-supplementary", action="store_true")
    ap.add_argument("--solo", type=int, default=-1)
    ap.add_argument("--replicas", action="store_true",
                    help="N>1, config4/configS: headline = N independent problems (weak) instead of ONE sharded problem")
    ap.add_argument("--exchange", type=int, default=1, choices=[0, 1],
                    help="sharded config4: 1 device-resident peer-memory exchange (default), 0 NCCL host loop")
    ap.add_argument("--force-sharded", action="store_true",
                    help="testing: take the N>1 code path (NCCL communicator, sharded engines, supplements) "
                         "even with one process")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(args.warmup, 3)

    import torch
    import torch.distributed as dist

    from paper_1707_01007_b200 import build as B
    B.build()
    from paper_1707_01007_b200 import cfpq as C

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    multi = world > 1 or args.force_sharded
    if multi:
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world)
    stream = torch.cuda.current_stream()
    dev_index = torch.cuda.current_device()

    # config 4 / config S: ONE problem row-block sharded over the ranks (strong scaling);
    # the other workloads close one independent seeded problem per GPU (weak scaling)
    sharded = multi and args.workload in ("config4", "configS") and not args.replicas
    w, desc = make_workload(args.workload, args.seed + (0 if sharded else rank))
    shard_kw = {}
    if sharded:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.tensor(list(C.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, src=0)
        shard_kw = {"world_size": world, "rank": rank, "nccl_unique_id": bytes(uid.cpu().tolist())}
        if args.workload == "config4":
            shard_kw["exchange"] = args.exchange
    lengths = args.workload == "config5"
    g = C.Grammar.from_workload(w)
    edges_dev = torch.from_numpy(w.edges).cuda()
    d = C.Graph(w.n_nodes, edges_dev, stream=stream)
    pol = policy_for(args.workload)
    kw = dict(stream=stream, semantics=int(lengths), solo_threshold=args.solo, path_policy=pol,
              tensor_format=args.tensor_format, schedule=args.schedule)

    # numerators (untimed): the executed semi-naive pairs of this instance on one GPU (the
    # sparse engine's stats.candidates; the tensor engine executes Jacobi products) and the
    # Jacobi-equivalent work of Alg. 1 line 9
    jac = jacobi_ops(w, args.workload, g, d, C, stream)
    r0 = C.closure(g, d, **kw)
    useful = jac if pol == 2 else 2 * int(r0.stats()["candidates"])
    del r0

    exchange_note = None
    r, err = None, None
    try:
        r = C.closure(g, d, **kw, **shard_kw)
    except C.CfpqError as ex:
        if shard_kw.get("exchange") != 1:
            raise
        err = ex
    if shard_kw.get("exchange") == 1 and multi and dist.is_initialized():
        # every rank takes the same path: one rank that could not map its peers sends all of
        # them to the NCCL host loop
        ok = torch.tensor([0 if err is not None else 1], dtype=torch.int32, device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0 and err is None:
            err = RuntimeError("a peer rank could not use the peer-memory exchange")
    if err is not None:
        # the peer-memory path could not map the peers (e.g. no CUDA IPC between these
        # processes): fall back to the NCCL host loop, and say so in the line
        exchange_note = "peer-memory exchange failed (%s); NCCL host loop used" % str(err)[:200]
        r = None
        shard_kw["exchange"] = 0
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.tensor(list(C.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, src=0)
        shard_kw["nccl_unique_id"] = bytes(uid.cpu().tolist())
        r = C.closure(g, d, **kw, **shard_kw)
    iterations = r.iterations
    cells = r.stats()["cells"]
    cells_total = sum(r.count(A) for A in range(w.n_nt)) if pol == 2 else cells
    results_start = r.count(w.start)
    nc, _ = r.iteration_stats()
    delta0 = int(cells - nc.sum())

    # L2 flush buffer (> 126 MB L2), written between timed steps, outside the events
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        C.closure_reuse(g, d, r, **kw, **shard_kw)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    step_ms, loop_ns, seed_ns, launches, cands = [], [], [], 0, []
    stats = None
    with ClockSampler(dev_index) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            ev0.record(stream)
            C.closure_reuse(g, d, r, **kw, **shard_kw)
            ev1.record(stream)
            ev1.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
            stats = r.stats()
            loop_ns.append(stats["loop_ns"])
            seed_ns.append(stats["seed_ns"])
            cands.append(stats["candidates"])
            launches += stats["launches"]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    assert r.iterations == iterations and r.stats()["cells"] == cells

    total_ms = float(sum(step_ms))
    total_ms_max, useful_job, jac_job = job_totals(dist, world, sharded, total_ms, useful, jac, "cuda")
    value = useful_job * args.steps / (total_ms_max * 1e-3) / 1e9
    ms_per_step = total_ms_max / args.steps

    # ---- roofline of the dominant kernel (the persistent closure kernel) ----
    # algorithmic bytes per launch: 8 B per Δ entry read, 8 B per (entry, rule)
    # expansion (two adjacency offsets), 12 B per candidate (4 B adjacency index + 4 B read +
    # 4 B write of its bit-matrix word), 8 B per appended cell; single-path adds 16 B per
    # candidate (key read+write) and 8 B per entry (own key).
    peak, peak_src = hbm_peak()
    if pol == 2:
        roofline = tensor_roofline(stats, total_ms / args.steps, 1 if args.tensor_format == 1 else 2)
    cand, exps = stats["candidates"], stats["expansions"]
    new_cells = cells - delta0
    alg_bytes = 8 * cells + 8 * exps + 12 * cand + 8 * new_cells
    if lengths:
        alg_bytes += 16 * cand + 8 * cells
    elif not sharded:
        # relational runs reset their bit words at the fixpoint inside the same launch:
        # 8 B log read + 4 B word store per cell
        alg_bytes += 12 * cells
    loop_s = statistics.mean(loop_ns) * 1e-9
    if pol != 2:
        achieved = alg_bytes / loop_s / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": ncu_traffic(args.workload), "kernel": "cfpq::closure_kernel",
                    "kernel_ms": loop_s * 1e3, "share_of_step": (loop_s * 1e3) / (total_ms / args.steps),
                    "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                    "note": ("latency-bound (SURVEY V-9): ~20 iterations of ~1e5 new cells, ~4 dependent memory "
                             "round trips each" if args.workload in ("config4", "config2") else
                             "latency-bound worst case: 2pq+1 iterations, one new cell each (SURVEY V-2)")}
        if args.workload in ("config4", "config2") and not lengths and not args.no_supplementary:
            # second roofline: candidates (one random bit test + set each) per second against the
            # measured random 4-byte RMW rate over a buffer the size of the bit matrices
            foot = int(w.n_nt) * int(w.n_nodes) * (((int(w.n_nodes) + 31) // 32 + 31) // 32 * 32) * 4
            pr = probe_random_access(foot)
            cand_rate = cand / loop_s / 1e9
            roofline["random_access"] = {
                "bound": "random 4-byte RMW into the bit matrices", "achieved": cand_rate,
                "peak": pr.get("atomic"), "unit": "G candidates/s vs G random atomics/s",
                "frac": (cand_rate / pr["atomic"]) if pr.get("atomic") else None,
                "random_load_peak": pr.get("load"), "footprint_bytes": foot,
                "peak_source": "measured in this run: torch index_add_ (int32 atomicAdd) / take, 2^25 uniform "
                               "random indices over the footprint, best of 3" if "atomic" in pr else pr.get("error")}

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(w.edges.copy()).pin_memory()
        csr = args.e2e_format == "csr"
        if csr:   # R_start as row pointers + columns (cfpq_result_csr): 4 B per pair + 8(n+1) B
            out_ptr = torch.empty((w.n_nodes + 1,), dtype=torch.int64).pin_memory()
            out_cols = torch.empty((max(results_start, 1),), dtype=torch.int32).pin_memory()
        else:
            out_pairs = torch.empty((max(results_start, 1), 2), dtype=torch.int32).pin_memory()
        h2d = pinned.numel() * 4
        d2h = 0
        ts, t_run, t_read = [], [], []
        for it in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            d.set_edges(pinned, stream=stream)
            C.closure_reuse(g, d, r, **kw, **shard_kw)
            ta = time.perf_counter()
            if csr:
                rp, cols = r.csr(w.start, out_ptr, out_cols)
            else:
                pairs = r.pairs(w.start, out=out_pairs)
            t1 = time.perf_counter()
            if it >= args.warmup:
                ts.append(t1 - t0)
                t_run.append(ta - t0)
                t_read.append(t1 - ta)
                d2h = rp.numel() * 8 + cols.numel() * 4 if csr else pairs.numel() * 4
        e_total = torch.tensor([sum(ts)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(e_total, op=dist.ReduceOp.MAX)
        e2e = {"value": useful_job * len(ts) / float(e_total.item()) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * float(e_total.item()) / len(ts),
               "median_ms": {"upload_and_closure": 1e3 * statistics.median(t_run),
                             "result_read": 1e3 * statistics.median(t_read)},
               "result": ("R_start as CSR (cfpq_result_csr: int64 row pointers + int32 columns)" if csr else
                          "R_start as sorted (i, j) int32 pairs (cfpq_result_pairs)") + " into pinned host memory"}

    supp = None
    if multi and args.workload == "config4" and not args.no_supplementary:
        supp = {}
        if sharded:
            supp["replicas"] = supplementary_replicas(C, args, rank, world, stream, dist)
            try:
                supp["paper_faithful_rows_sharded"] = supplementary_rows_sharded(C, w, g, d, args, rank, world,
                                                                                 stream, dist, shard_kw)
            except Exception as ex:
                supp["paper_faithful_rows_sharded_error"] = repr(ex)
    if rank == 0 and not multi and args.workload == "config4" and not args.no_supplementary:
        supp = {}
        try:
            supp["tensor_path"] = supplementary_tensor(C, stream, fmt=2)
        except Exception as ex:   # never lose the headline line over a supplement
            supp["tensor_path_error"] = repr(ex)
        try:
            supp["tensor_path_int8"] = supplementary_tensor(C, stream, fmt=1)
        except Exception as ex:
            supp["tensor_path_int8_error"] = repr(ex)
        try:
            supp["paper_faithful_rows"] = supplementary_rows(C, w, g, d, r, stream)
        except Exception as ex:
            supp["paper_faithful_rows_error"] = repr(ex)

    cpu = bits = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        o, t, sample, sw = time_oracle(args.workload, args.seed, n4=4096)
        cpu = {"value": o / sum(t) / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
               "sample_n_nodes": int(sw.n_nodes), "sample_n_edges": int(len(sw.edges)), "seconds": sum(t)}
        try:
            bits = cpu_bitset(args.workload, w, r, w.n_nt)
        except Exception as ex:
            bits = {"error": repr(ex)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if sharded else "weak", "vs_baseline": None,
                "dtype": (("int8 0/1 tiles -> s32 (tcgen05 kind::i8)" if args.tensor_format == 1 else
                           "e2m1 (fp4) 0/1 tiles, unit ue8m0 scales -> f32 (tcgen05 kind::mxf4)")
                          if pol == 2 else "u32 bit-words (boolean)"),
                "data": "synthetic",
                "config": {**desc, "iterations": iterations, "cells": int(cells_total),
                           "results_start_nt": int(results_start),
                           "ops_per_step": int(useful_job),
                           "ops_definition": ("2 x Jacobi AND-true triples (the tensor engine executes full products)"
                                              if pol == 2 else "2 x executed semi-naive (Δ entry, neighbour) pairs "
                                              "= 2 x stats.candidates"),
                           "candidates_per_step": int(statistics.median(cands)) if cands else None,
                           "schedule": {0: "jacobi", 3: "gauss-seidel"}[args.schedule],
                           "l2": "flushed between steps (512 MiB write outside the timed events)",
                           "parallelism": (("ONE problem row-block sharded over %d GPUs: %s" % (world, (
                                               "Δ cells appended to every rank's log over NVLink peer memory inside "
                                               "one persistent kernel per GPU, cross-GPU barrier per iteration"
                                               if shard_kw.get("exchange") == 1 else
                                               "NCCL all-gather per iteration of "
                                               + ("Δ index lists" if pol != 2 else "dense row blocks"))))
                                           if sharded else f"{world} independent replicas (seed+rank)")
                           if world > 1 else "1 GPU",
                           "exchange_note": exchange_note,
                           "engine": ("dense tcgen05 int8 (kind::i8)" if args.tensor_format == 1 else
                                      "dense tcgen05 fp4 (kind::mxf4)") + ", CTA pairs" if pol == 2 else
                                     "sparse semi-naive persistent kernel",
                           "seed_phase_ms": statistics.mean(seed_ns) * 1e-6},
                "jacobi_equivalent": {"value": jac_job * args.steps / (total_ms_max * 1e-3) / 1e9, "unit": UNIT,
                                      "ops_per_step": int(jac_job),
                                      "definition": "2 x AND-true triples of T_{k-1} x T_{k-1} over all iterations "
                                                    "(Alg. 1 line 9 on sparse operands), same closure time"},
                "roofline": roofline, "cpu_baseline": cpu, "cpu_bitset": bits, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clk.summary(), "supplementary": supp}
        print(json.dumps(line), flush=True)
    if multi:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
