#!/usr/bin/env python
"""Benchmark: APD (A-DEF1 with higher-order deflation vectors) + CSLP preconditioned FGMRES
time-to-1e-6 on B200 (BASELINE.json metric "FGMRES time-to-1e-6 & its/s at 1-8 GPUs").

One "step" = one complete solve A x = b to ||b - Ax||/||b|| <= 1e-6 from x0 = 0 (every row of
the hot path: stencil applies, V-cycles, deflation Z/Z^T and the coarse solve, Krylov
dots/axpys).  Default workload: BASELINE.json configs[4]'s weak-scaling block on one GPU,
`c4_weak_2049` = the unit-square Dirichlet point-source problem with a 2047 x 2047 interior
grid (h = 1/2048) and k = 1280 (kh = 0.625), complex128, inputs resident in HBM (the 126 MB L2
is flushed between timed steps, outside the events).
`value` = `ms_per_step` / 1000 = mean time to 1e-6 in seconds (lower is better); the outer
FGMRES iterations per second ("its/s") are reported beside it.  N > 1 (torchrun): weak scaling,
one 2047 x 2048 row strip per GPU of N unit squares stacked in y at the same h and k (kh =
0.625 at every N), decomposed solve over NCCL; value = max-over-ranks time to 1e-6.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c4_weak_2049] [--inner-maxit 200] [--inner-restart 50] ...

--impl reference times the oracle (numpy, host cores) on a bounded sample of the same
workload: the base contract's reference arm for this tier.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Method of the timed workload: higher-order deflation vectors (APD, the paper's
# wavenumber-independent variant, Table 4) with the Galerkin coarse operator E; outer flexible
# GMRES (§6.3: a flexible outer method keeps the outer accuracy with a loose coarse
# tolerance); the coarse problem by CSLP-FGMRES(48) (reading R25) to 1e-1 capped at 192 steps;
# the CSLP hierarchy stops at the first level with <= 512 unknowns (§4 "predefined
# coarsest grid size"), solved exactly (R8).  Chosen by the time-to-1e-6 sweeps on c4_weak_2049
# (profiles/r02_c4_sweep.jsonl, one-vector coarse solve: cap/restart 120/30 .. 200/50 within 5 %,
# 160/40 the fastest; profiles/r02_c4_sweep_sstep.jsonl, s-step coarse solve, restart a multiple
# of s = 8: 192/48 and 224/56 the fastest, 462 / 396 outer iterations; any outer restart stagnates).
DEFAULT_METHOD = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 1e-1, "inner_maxit": 192,
                  "inner_restart": 48, "coarsest_n": 512, "restart": 0}
DEFAULT_WORKLOAD = "c4_weak_2049"
# Device form of the coarse solve (reading R28, §6d): the basis generated and
# orthogonalised 8 vectors at a time (one block Gram-Schmidt pass), measured 25.2 -> 16.9 s on
# c4_weak_2049 (profiles/r02_sstep_probe.jsonl).
DEFAULT_SSTEP = {"sstep": 8, "sstep_passes": 1}

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return dict(PEAKS_FALLBACK)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if "Active" in r[2 + i] and "Not" not in r[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def method_of(args):
    return {"vectors": args.vectors, "coarse_op": args.coarse_op, "inner_tol": args.inner_tol,
            "inner_maxit": args.inner_maxit, "inner_restart": args.inner_restart, "coarsest_n": args.coarsest_n,
            "restart": args.restart, "outer": args.outer}


def gpu_method(args):
    """The GPU parameters of the method: the paper's method (method_of, shared with the oracle) plus
    the form the coarse solve takes on the device (s-step blocks, reading R28: the same GMRES(m)
    iterates in exact arithmetic), which the oracle does not have."""
    return dict(method_of(args), sstep=args.sstep, sstep_passes=args.sstep_passes)


def oracle_params(args, **kw):
    import oracle
    m = dict(method_of(args), **kw)
    return oracle.SolverParams(**m)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


COUNTS_FILE = os.path.join(ROOT, "profiles", "r02_bench_counts.json")


def method_counts(args):
    """Outer / inner iteration counts of a converged GPU solve of this workload with this method
    (profiles/r02_bench_counts.json, written by `bench.py --record-counts`): the reference arm
    extrapolates the oracle's per-iteration cost with them.  None if unrecorded."""
    try:
        with open(COUNTS_FILE) as fh:
            d = json.load(fh)
        e = d.get(args.workload)
        if e and e.get("method") == method_of(args):
            return e
    except (OSError, ValueError):
        pass
    return None


def oracle_cores():
    try:
        import threadpoolctl
        return max([i.get("num_threads", 1) for i in threadpoolctl.threadpool_info()] or [1])
    except Exception:
        return 1


class OracleSample:
    """The oracle (numpy, host cores) on a bounded sample of the workload: the first outer FGMRES
    iteration from x0 = 0 with its coarse solve truncated to c inner iterations.  Two sample sizes
    separate the cost of one inner iteration from the rest of an outer iteration:
        t_inner = (T(c2) - T(c1)) / (c2 - c1),   t_outer = T(c1) - c1 t_inner,
    and the time to 1e-6 is extrapolated as N_outer t_outer + N_inner t_inner with the method's
    iteration counts on this workload (method_counts).  The Gram-Schmidt work of the sampled
    iterations is that of the first basis columns only, so the estimate is a lower bound for
    the oracle."""

    def __init__(self, args, c1=1, c2=2):
        import oracle
        from workloads import config_problem
        self.args = args
        self.p = config_problem(args.workload)
        self.c1, self.c2 = c1, c2
        prm = oracle_params(args, maxit=1)
        self.solver = oracle.Solver(self.p.k, self.p.h, self.p.bc, prm)

    def run(self, c):
        s = self.solver
        s.p.inner_maxit = c
        s.p.inner_tol = 0.0          # exactly c inner iterations (reading R15)
        t0 = time.perf_counter()
        s.solve(self.p.b)
        return time.perf_counter() - t0

    def estimate(self, t1, t2):
        t_inner = max(0.0, (t2 - t1) / (self.c2 - self.c1))
        t_outer = max(0.0, t1 - self.c1 * t_inner)
        cnt = method_counts(self.args)
        if cnt is None:
            return None, t_inner, t_outer, None
        return cnt["outer"] * t_outer + cnt["inner_total"] * t_inner, t_inner, t_outer, cnt

    def describe(self, t_inner, t_outer, cnt, secs):
        c = f"counts outer {cnt['outer']}, inner {cnt['inner_total']} ({os.path.basename(COUNTS_FILE)})" if cnt \
            else "no recorded counts"
        return (f"oracle on {self.args.workload}: first outer FGMRES iteration from x0=0 with the coarse solve "
                f"truncated to {self.c1} and {self.c2} inner iterations ({secs:.1f} s of CPU work); "
                f"{t_inner:.2f} s per inner iteration, {t_outer:.2f} s per outer iteration otherwise; "
                f"time to 1e-6 extrapolated with the method's {c} (a lower bound: later basis columns "
                f"cost more Gram-Schmidt)")


def run_reference(args, rank, world):
    """The oracle (numpy) on the host cores: each step one bounded sample (OracleSample, the larger
    truncation); value = the extrapolated time to 1e-6 in seconds, like the GPU arm's."""
    if rank != 0:
        return
    smp = OracleSample(args)
    t1 = smp.run(smp.c1)                          # the split needs the smaller sample once
    times = []
    for step in range(args.warmup + args.steps):
        dt = smp.run(smp.c2)
        if step >= args.warmup:
            times.append(dt)
    t2 = statistics.mean(times)
    est, t_inner, t_outer, cnt = smp.estimate(t1, t2)
    val = est if est is not None else t2
    vdef = ("extrapolated time to 1e-6 (s); ms_per_step = one bounded sample" if est is not None else
            "no recorded iteration counts for this workload/method: value = one bounded sample (s)")
    cores = oracle_cores()
    p = smp.p
    desc = smp.describe(t_inner, t_outer, cnt, t1 + sum(times))
    line = {
        "impl": "reference", "metric": "fgmres_time_to_1e-6_s", "value": val, "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t2,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": args.workload, **method_of(args), "nx": p.nx, "ny": p.ny, "h": p.h,
                   "k": p.meta.get("k"), "tol": 1e-6, "l2": "n/a (host)",
                   "value_definition": vdef},
        "cpu_baseline": {"value": val, "unit": "s", "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": val, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(args):
    """cpu_baseline of the GPU arm's line: the oracle on the host cores, one bounded sample of
    each size (OracleSample), extrapolated to the time to 1e-6."""
    smp = OracleSample(args)
    t1 = smp.run(smp.c1)
    t2 = smp.run(smp.c2)
    est, t_inner, t_outer, cnt = smp.estimate(t1, t2)
    return {"value": est, "unit": "s", "cores": oracle_cores(), "kind": "oracle",
            "sample": smp.describe(t_inner, t_outer, cnt, t1 + t2)}


def mean_inner_column(rep, method):
    """Mean Arnoldi column j over the solve's inner iterations: a coarse solve of I steps in
    cycles of m (inner_restart) visits j = 0..min(I, m)-1 per cycle."""
    I = rep["inner_iterations_total"] / max(1, rep["inner_solves"])
    m = method.get("inner_restart") or 0
    span = min(I, m) if m > 0 else I
    return max(1, int(round((span - 1) / 2)))


def kernel_roofline(H, rep, method, peaks, workload):
    """The roofline line of the step's dominant kernel, measured live here with CUDA events.

    The solve is a chain of dependent kernels inside one CUDA graph, so each kernel is timed the
    way it runs there: back-to-back instances of exactly the solve's launch (helm_bench_graph
    regions that call the solve's own Arnoldi-step code) captured into a graph and replayed warm,
    at the solve's mean inner basis column.  Launch counts per step are the solve's own counts;
    the dominant kernel is the one with the largest count x time.  Algorithmic bytes per launch
    (per coarse unknown n1 / fine unknown n0): E 64 (x 16, fine k 4 x 8, y 16);
    pass 1 16 (j + 2) (V_0..V_j and w); fused E + pass 1 (64 + 16(j+1) + 16); pass 2 (16 j + 64);
    V-cycle from level 1 sum_l 104 n_l + the dense coarsest inverse; A 40 n0."""
    inner_its = rep["inner_iterations_total"]
    outer_its = rep["outer_iterations"]
    jm = mean_inner_column(rep, method)
    lv = [ny * nx for (ny, nx, _) in H.levels]
    n0, n1 = lv[0], lv[1]
    tiles = -(-H.levels[1][1] // 16) * -(-H.levels[1][0] // 8)
    vbytes = sum(104.0 * lv[l] for l in range(1, len(lv) - 1)) + 16.0 * lv[-1] ** 2 + 32.0 * lv[-1]
    prm = H.params
    galerkin = method.get("coarse_op", "galerkin") == "galerkin"
    fused = galerkin and bool(prm.fuse_dots)
    comps = []
    ss = int(method.get("sstep") or 0)
    if ss > 0:
        # s-step coarse solve (reading R28): per step one V-cycle + E in residual mode; per block
        # of s steps `passes` x (pass partials, reduction, update) at the mean block column
        m = method.get("inner_restart") or method.get("inner_maxit")
        Jm = ss * ((m // ss - 1) // 2)
        blocks = -(-inner_its // ss)
        passes = int(method.get("sstep_passes") or 1)
        comps += [
            ("k_glk_stream<2,1> (E = Z^T A Z in residual mode, w = sigma f - E x)" if galerkin and prm.e_stream else
             "E apply (residual mode)", "ss_e", 0, 10, inner_its, 80.0 * n1),
            ("k_bgs_dots_smem (block pass partials [Q W]^H W)", "ss_dots", Jm, 5, blocks * passes,
             16.0 * (Jm + 1 + ss) * n1),
            ("k_bgs_update (W <- (W - Q C) R^-1)", "ss_update", Jm, 5, blocks * passes, 16.0 * (Jm + 1 + 2 * ss) * n1),
            ("k_bgs_reduce (partial sums + Cholesky)", "ss_reduce", Jm, 10, blocks * passes,
             16.0 * (Jm + 1 + ss) * ss * 148),
        ]
    elif fused:
        comps.append(("k_galerkin_apply<2,0,16,8,true> (E = Z^T A Z fused with DCGS2 pass 1)", "e_dots", jm, 4,
                      inner_its, (64.0 + 16 * (jm + 1) + 16) * n1))
    else:
        comps.append(("k_glk_stream<2,0> (E = Z^T A Z, column streaming)" if galerkin and prm.e_stream else
                      "E apply (coarse operator)", "apply_E", 0, 10, inner_its, 64.0 * n1))
        comps.append(("k_dcgs_dots (DCGS2 pass 1)", "dcgs_dots", jm, 4, inner_its, 16.0 * (jm + 2) * n1))
    if ss <= 0:
        comps += [
            ("k_dcgs_update (DCGS2 pass 2 + step B)", "dcgs_update", jm, 4, inner_its, (16.0 * jm + 64) * n1),
            ("k_dcgs_reduceA (pass-1 partial sums + step A)", "dcgs_reduce", jm, 4, inner_its,
             (2 * jm + 2) * 16.0 * (tiles if fused else -(-n1 // 256))),
        ]
    # the inner V-cycle by kernel: the two level-1 legs (the largest V-cycle kernels of the launch
    # list) and the rest of the cycle from level 2 (11 kernels on levels <= 511^2 + the coarsest)
    n2 = lv[2] if len(lv) > 2 else 0
    vbytes2 = sum(104.0 * lv[l] for l in range(2, len(lv) - 1)) + 16.0 * lv[-1] ** 2 + 32.0 * lv[-1]
    if len(lv) > 3 and H.params.nu_pre == 1 and H.params.nu_post == 1:
        comps += [
            ("k_vc_down (V-cycle down leg, level 1)", "vc_down", 1, 10, inner_its + outer_its, 44.0 * n1 + 0 * n2),
            ("k_vc_up (V-cycle up leg, level 1)", "vc_up", 1, 10, inner_its + outer_its, 60.0 * n1),
            ("V-cycle from level 2 (11 kernels)", "vcycle", 2, 10, inner_its + outer_its, vbytes2),
        ]
    else:
        comps.append(("V-cycle from level 1 (inner CSLP preconditioner)", "vcycle", 1, 10, inner_its + outer_its,
                      vbytes))
    comps += [
        ("k_apply_op A (level 0)", "apply_A", 0, 10, 2 * outer_its, 40.0 * n0),
    ]
    # the outer FGMRES's DCGS2 step over the level-0 basis at the solve's mean column (pass 1 reads
    # V_0..V_j, v~_j, w; pass 2 reads V_0..V_{j-1}, v~_j, w and writes v_j, w'): a group, not chosen
    jo = max(1, outer_its // 2)
    if method.get("outer", "fgmres") == "fgmres" and not method.get("restart"):
        comps.append(("outer DCGS2 step, level-0 basis (3 kernels)", "outer_dcgs", jo, 3, outer_its,
                      (32.0 * jo + 112.0) * n0))
    rows = {}
    for label, region, arg, nrep, count, nbytes in comps:
        try:
            us = H.helm_bench_graph(region, arg, nrep)
        except RuntimeError:
            if region != "outer_dcgs":   # needs the outer basis of a finished solve on this context
                raise
            continue
        gbs = nbytes / (us * 1e-6) / 1e9
        rows[label] = {"kernel": label, "bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                       "frac": gbs / peaks["hbm_gbs"], "traffic": None, "bytes_per_launch": nbytes,
                       "us_per_launch": us, "launches_per_step": count, "est_ms_per_step": count * us * 1e-3,
                       "column": arg if region in ("e_dots", "dcgs_dots", "dcgs_update", "dcgs_reduce", "ss_dots",
                                                   "ss_update", "ss_reduce", "outer_dcgs") else None,
                       "timing": "in-graph, warm (helm_bench_graph: the solve's own launch, replayed)",
                       "peak_src": peaks["src"]}
    # the dominant KERNEL (groups of kernels are reported, not chosen)
    dom = max((r for r in rows.values() if "kernels)" not in r["kernel"]), key=lambda r: r["est_ms_per_step"])
    # DRAM traffic per launch of the dominant kernel from the committed ncu --set full capture of
    # the same launch at this workload (tools/ncu_regions.py; cold caches)
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")) as fh:
            prof = json.load(fh)
        key = f"{workload}:{dom['kernel'].split(' ')[0]}"
        if key in prof:
            e = prof[key]
            # per basis column the kernel streams 16 n1 bytes more: scale to this column
            dom["traffic"] = e["dram_bytes"] + e.get("bytes_per_column", 0.0) * ((dom["column"] or 0) - (e.get("column") or 0))
            dom["traffic_src"] = e["src"]
    except (OSError, KeyError, ValueError, TypeError):
        pass
    return dict(dom), {"components": {k: {kk: v[kk] for kk in ("achieved", "frac", "us_per_launch", "bytes_per_launch",
                                                              "launches_per_step", "est_ms_per_step")}
                                      for k, v in rows.items()},
                       "mean_inner_column": jm}


def microbench(peaks, n=16385, reps=10):
    """BASELINE configs[4] microbenchmark: isolated stencil apply, fused V-cycle legs and one whole
    V-cycle from level 0 on a 16385^2-node (16383^2 Dirichlet unknowns) complex128 grid.  Single
    kernels: L2 flushed before each launch.  Whole V-cycle: 5 back-to-back cycles in a graph (the
    4.3 GB fields are 34x the L2).  Algorithmic bytes of a V-cycle: 104 B per unknown of every
    level above the coarsest (down leg 44, up leg 60) + the dense coarsest inverse."""
    import torch
    from paper_2308_06152_b200 import helm
    m = n - 2
    h = 1.0 / (n - 1)
    k = torch.full((m, m), 0.625 / h, dtype=torch.float64, device="cuda")
    H = helm.Helm(m, m, h, "dirichlet", k, {"inner_maxit": 2, "coarsest_n": 512})
    out = {"grid": f"{m}x{m} unknowns (h=1/{n - 1}), complex128"}
    for name, arg in (("apply_A", 0), ("vc_down", 0), ("vc_up", 0)):
        us, nb = H.helm_bench_kernel(name, arg=arg, reps=reps, flush=True)
        gbs = nb / (us * 1e-6) / 1e9
        out[name] = {"us": us, "GB/s": gbs, "frac": gbs / peaks["hbm_gbs"], "bytes": nb}
    lv = [ny * nx for (ny, nx, _) in H.levels]
    vb = sum(104.0 * lv[l] for l in range(len(lv) - 1)) + 16.0 * lv[-1] ** 2 + 32.0 * lv[-1]
    us = H.helm_bench_graph("vcycle", 0, 5)
    out["vcycle_from_level0"] = {"us": us, "GB/s": vb / (us * 1e-6) / 1e9, "frac": vb / (us * 1e-6) / 1e9 / peaks["hbm_gbs"],
                                 "bytes": vb, "levels": len(lv)}
    H.close()
    del k
    torch.cuda.empty_cache()
    return out


class _StdoutToStderr:
    """Route fd 1 to stderr while libraries (NCCL prints a version banner on stdout) run, so that
    rank 0's stdout carries exactly the one JSON line of the contract."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def run_decomposed(args, rank, world, local):
    from paper_2308_06152_b200 import helm
    with _StdoutToStderr():
        line = _run_decomposed(args, rank, world, local)
    if line is not None:
        print(json.dumps(line), flush=True)


def _run_decomposed(args, rank, world, local):
    """Weak scaling of ONE solve over the ranks: the workload's unit square
    stacked `world` times in y (strip_problem: same h and k, so kh = 0.625 and one 2047 x 2048
    block per GPU at every N; point source at the centre), one row strip per GPU; halos by
    grouped ncclSend/ncclRecv, dots by ncclAllReduce, the coarse levels below the decomposed ones
    all-gathered and replicated.  value = max-over-ranks device time to 1e-6 (s).  The same
    outer restart length at every N.  A transport failure raises on every rank (no rerun)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2308_06152_b200 import helm
    from workloads import config_problem, strip_problem
    torch.cuda.set_device(local)
    peaks = load_peaks()
    base = config_problem(args.workload)
    if args.scaling == "strong":
        # strong scaling: the workload's own grid (e.g. c4_strong_8193, BASELINE configs[4]) cut
        # into `world` row strips
        p = base
    else:
        p = strip_problem(base.meta["k"], base.meta["n_cells"], world, f"{args.workload}_x{world}")
    method = gpu_method(args)
    uid = peer_exchange = None
    if args.transport == "peer":        # NVLink peer memory through CUDA IPC (peer.cuh), no NCCL
        def peer_exchange(handle):
            if world == 1:
                return [handle]
            out = [None] * world
            dist.all_gather_object(out, handle)
            return out
    elif world > 1:
        obj = [helm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    else:
        uid = helm.nccl_unique_id()
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        # decomposed levels per N (the all-gather and the replicated coarse levels
        # shrink 4x per extra decomposed level, each extra level adds one halo exchange)
        prm = dict(method, dist_levels=args.dist_levels or (3 if world <= 2 else 4 if world <= 4 else 5))
        H = helm.HelmDist(p.nx, p.ny, p.h, p.bc, p.k, rank, world, nccl_id=uid, params=prm, stream=stream,
                          peer_exchange=peer_exchange)
        try:
            bo = np.ascontiguousarray(p.b[H.row0:H.row0 + H.nrows])
            b = torch.from_numpy(bo).cuda()
            x = torch.empty_like(b)
            for _ in range(args.warmup):
                H.solve(b, 1e-6, args.maxit, x)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            reps = []
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            wall0 = time.perf_counter()
            with ClockSampler(local) as clk:
                for s in range(args.steps):
                    H.helm_flush_l2(256 << 20)
                    ev[s][0].record(stream)
                    _, rep = H.solve(b, 1e-6, args.maxit, x)
                    ev[s][1].record(stream)
                    reps.append(rep)
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
            wall = time.perf_counter() - wall0
            dev_s = sum(a.elapsed_time(b_) for a, b_ in ev) * 1e-3
            if world > 1:
                tt = torch.tensor([dev_s], device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dev_s = float(tt.item())
            its = sum(r["outer_iterations"] for r in reps)
            bh = torch.from_numpy(bo).pin_memory().numpy()
            xh = torch.empty(bo.shape, dtype=torch.complex128).pin_memory().numpy()
            e2e_t = []
            for s in range(max(1, args.e2e_steps)):
                H.helm_flush_l2(256 << 20)
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                H.solve_host(bh, xh, 1e-6, args.maxit)
                e2e_t.append(time.perf_counter() - t0)
            e2e_s = statistics.mean(e2e_t)
            if world > 1:
                tt = torch.tensor([e2e_s], device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                e2e_s = float(tt.item())
            launches = sum(r["kernels"] for r in reps)
        finally:
            H.close()
        roof = roof_all = None
        if rank == 0:   # kernel rooflines at the per-GPU block size (single-GPU context)
            Hs = helm.helm_setup(base, method, stream=stream)
            roof, roof_all = kernel_roofline(Hs, reps[-1], method, peaks, args.workload)
            Hs.close()
    if rank != 0:
        return None
    tts = dev_s / args.steps
    r = reps[-1]
    line = {
        "metric": "fgmres_time_to_1e-6_s", "value": tts, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tts,
        "higher_is_better": False, "scaling": args.scaling, "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "outer_its_per_s": its / dev_s, "time_to_solution_s": tts,
        "converged": all(x_["converged"] for x_ in reps),
        "config": {"workload": p.name, "per_gpu_block": args.workload, **method, "nx": p.nx, "ny": p.ny,
                   "h": p.h, "k": p.meta["k"], "tol": 1e-6, "maxit": args.maxit,
                   "l2": "flushed between timed steps (256 MiB read)",
                   "outer_iterations": r["outer_iterations"],
                   "inner_iterations_total": r["inner_iterations_total"],
                   "inner_iterations_mean": r["inner_iterations_total"] / max(1, r["inner_solves"]),
                   "parallelism": f"row-strip decomposition x{world} ({args.transport} transport)",
                   "dist_levels": prm["dist_levels"], "transport": args.transport,
                   "value_definition": "max-over-ranks device time to 1e-6 (s)"},
        "wall_s": wall,
        "gpu_launches": launches,
        "e2e": {"value": e2e_s, "unit": "s", "steps": len(e2e_t), "h2d_bytes_per_step": int(bo.nbytes) * world,
                "d2h_bytes_per_step": int(bo.nbytes) * world},
        "roofline": roof,
        "roofline_kernels": roof_all,
        "clocks": clk.summary(),
    }
    if not line["converged"]:
        # DESIGN.md R27: the stacked-strip weak family gets harder with N at the N = 1 method's
        # coarse cap (one-GPU runs of the N = 2..8 grids, profiles/r02_weak_family_counts.jsonl)
        line["note"] = (f"not converged to 1e-6 within maxit = {args.maxit}: value is the time to maxit, "
                        "not a time to solution (DESIGN.md R27)")
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD)
    ap.add_argument("--coarse-op", default=DEFAULT_METHOD["coarse_op"])
    ap.add_argument("--vectors", default=DEFAULT_METHOD["vectors"])
    ap.add_argument("--outer", default="fgmres", choices=["fgmres", "gcr"])
    ap.add_argument("--inner-tol", type=float, default=DEFAULT_METHOD["inner_tol"])
    ap.add_argument("--inner-maxit", type=int, default=DEFAULT_METHOD["inner_maxit"])
    ap.add_argument("--inner-restart", type=int, default=DEFAULT_METHOD["inner_restart"])
    ap.add_argument("--restart", type=int, default=DEFAULT_METHOD["restart"],
                    help="outer FGMRES(m); 0 = full basis (the same at every N)")
    ap.add_argument("--coarsest-n", type=int, default=DEFAULT_METHOD["coarsest_n"])
    ap.add_argument("--sstep", type=int, default=DEFAULT_SSTEP["sstep"],
                    help="coarse solve in s-step form (0 = one vector per step, delayed CGS2)")
    ap.add_argument("--sstep-passes", type=int, default=DEFAULT_SSTEP["sstep_passes"])
    ap.add_argument("--maxit", type=int, default=1000)
    ap.add_argument("--e2e-steps", type=int, default=1, help="end-to-end solves (host buffers) after the timed ones")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-micro", action="store_true")
    ap.add_argument("--record-counts", action="store_true",
                    help="write this run's iteration counts to profiles/r02_bench_counts.json (reference arm)")
    ap.add_argument("--dist-levels", type=int, default=0, help="decomposed levels (0: 3)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="decomposed solve: weak = the workload's block per GPU (stacked strips, default); "
                         "strong = the workload's own grid cut into N strips (e.g. --workload c4_strong_8193)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer"],
                    help="decomposed solve: NCCL collectives (default) or NVLink peer memory through CUDA IPC")
    ap.add_argument("--decomp", default="auto", choices=["auto", "on", "off"],
                    help="row-strip decomposed solve over the ranks; auto = on when N > 1")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        with _StdoutToStderr():
            dist.init_process_group("nccl")
    if args.decomp == "on" or (args.decomp == "auto" and world > 1):
        return run_decomposed(args, rank, world, local)
    import torch
    from paper_2308_06152_b200 import helm
    from workloads import config_problem
    torch.cuda.set_device(local)
    peaks = load_peaks()
    p = config_problem(args.workload)
    method = gpu_method(args)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        H = helm.helm_setup(p, method, stream=stream)
        b = torch.from_numpy(p.b).cuda()
        x = torch.empty_like(b)
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            H.solve(b, 1e-6, args.maxit, x)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        reps = []
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        with ClockSampler(local) as clk:
            for s in range(args.steps):
                H.helm_flush_l2(256 << 20)
                ev[s][0].record(stream)
                _, rep = H.solve(b, 1e-6, args.maxit, x)
                ev[s][1].record(stream)
                reps.append(rep)
            torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
        launches = sum(r["kernels"] for r in reps)
        dev_s = sum(a.elapsed_time(b_) for a, b_ in ev) * 1e-3
        its = sum(r["outer_iterations"] for r in reps)
        converged = all(r["converged"] for r in reps)
        # true residual of the last solution (the device estimate is the stopping test)
        rr = float(torch.linalg.vector_norm(H.apply_A(x) - b) / torch.linalg.vector_norm(b))
        # end-to-end through the public API with host buffers (H2D of b, D2H of x inside)
        bh = torch.from_numpy(p.b).pin_memory().numpy()
        xh = torch.empty(p.shape, dtype=torch.complex128).pin_memory().numpy()
        e2e_t = []
        for s in range(max(1, args.e2e_steps)):
            H.helm_flush_l2(256 << 20)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, r2 = H.solve_host(bh, xh, 1e-6, args.maxit)
            e2e_t.append(time.perf_counter() - t0)
        roof, roof_all = kernel_roofline(H, reps[-1], method, peaks, args.workload)
        H.close()
    tts = dev_s / args.steps
    r = reps[-1]
    if args.record_counts and converged:
        try:
            with open(COUNTS_FILE) as fh:
                d = json.load(fh)
        except (OSError, ValueError):
            d = {}
        d[args.workload] = {"method": method_of(args), "outer": r["outer_iterations"], "inner_total": r["inner_iterations_total"],
                            "inner_solves": r["inner_solves"], "time_to_solution_s": tts}
        with open(COUNTS_FILE, "w") as fh:
            json.dump(d, fh, indent=1, sort_keys=True)
    line = {
        "metric": "fgmres_time_to_1e-6_s", "value": tts, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tts,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "outer_its_per_s": its / dev_s, "time_to_solution_s": tts, "converged": converged, "true_relres": rr,
        "config": {"workload": args.workload, **method, "nx": p.nx, "ny": p.ny, "h": p.h,
                   "k": p.meta.get("k"), "tol": 1e-6, "maxit": args.maxit,
                   "l2": "flushed between timed steps (256 MiB read)",
                   "outer_iterations": r["outer_iterations"],
                   "inner_iterations_total": r["inner_iterations_total"],
                   "inner_iterations_mean": r["inner_iterations_total"] / max(1, r["inner_solves"]),
                   "inner_iterations_max": r["inner_iterations_max"], "inner_restarts": r["inner_restarts"],
                   "outer_restarts": r["restarts"], "parallelism": "single"},
        "wall_s": wall,
        "gpu_launches": launches,
        "e2e": {"value": statistics.mean(e2e_t), "unit": "s", "steps": len(e2e_t),
                "h2d_bytes_per_step": p.nx * p.ny * 16, "d2h_bytes_per_step": p.nx * p.ny * 16},
        "roofline": roof,
        "roofline_kernels": roof_all,
        "clocks": clk.summary(),
    }
    if not args.no_micro:
        line["microbench"] = microbench(peaks)
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline_sample(args)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
