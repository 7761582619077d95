#!/usr/bin/env python
"""Benchmark: A-DEF1 + CSLP preconditioned FGMRES time-to-1e-6 on B200 (BASELINE.json).

One "step" = one complete solve A x = b to ||b - Ax||/||b|| <= 1e-6 from x0 = 0 (every row
of the hot path: stencil applies, V-cycles, deflation Z/Z^T and the coarse solve, Krylov
dots/axpys) for the workload of BASELINE.json configs[1] at its largest size (k = 400,
h = 1/640, kh = 0.625, Dirichlet point source, Galerkin E), inputs resident in HBM.
`value` = outer FGMRES iterations per second over the K timed steps; `ms_per_step` is
the time-to-solution.  The L2 (126 MB) is flushed between timed steps (outside the
events).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c1_k400] [--coarse-op galerkin]

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

# Method of the timed workload: higher-order deflation vectors (APD, the
# paper's wavenumber-independent variant, Table 4) with the Galerkin coarse operator E; the
# coarse problem solved by CSLP-FGMRES to 1e-1 (§6.3, the GCR/FGMRES setting) capped
# at 50 iterations, the inner counts the paper reports for that setting (Tables 9-10); the
# CSLP hierarchy stops at the first level with <= 512 unknowns (§4 "predefined
# coarsest grid size"), solved exactly (R8).
DEFAULT_METHOD = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 1e-1, "inner_maxit": 50,
                  "coarsest_n": 512}

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
            "inner_maxit": args.inner_maxit, "coarsest_n": args.coarsest_n}


def oracle_params(args, **kw):
    import oracle
    m = method_of(args)
    return oracle.SolverParams(vectors=m["vectors"], coarse_op=m["coarse_op"], inner_tol=m["inner_tol"],
                               inner_maxit=m["inner_maxit"], coarsest_n=m["coarsest_n"], **kw)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def run_reference(args, rank, world):
    """The oracle (numpy) on the host cores, bounded sample: full solves of the same
    workload family at a size the oracle finishes in seconds is NOT the same workload, so
    we time whole outer FGMRES iterations of the real workload (c1_k400) instead."""
    import numpy as np
    import oracle
    from workloads import config_problem
    if rank != 0:
        return
    p = config_problem(args.workload)
    prm = oracle_params(args, maxit=args.ref_iters)
    s = oracle.Solver(p.k, p.h, p.bc, prm)
    times, iters = [], []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        x, rep = s.solve(p.b)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
            iters.append(rep["outer_iterations"])
    total = sum(times)
    its = sum(iters)
    cores = 1
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        cores = max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:
        pass
    val = its / total
    line = {
        "impl": "reference", "metric": "fgmres_outer_iterations_per_s", "value": val, "unit": "it/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": args.workload, **method_of(args), "nx": p.nx, "ny": p.ny, "h": p.h,
                   "k": p.meta.get("k"), "l2": "n/a (host)"},
        "cpu_baseline": {"value": val, "unit": "it/s", "cores": cores, "kind": "oracle",
                         "sample": f"first {args.ref_iters} outer FGMRES iterations of {args.workload} per step"},
        "e2e": {"value": val, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(args, n_outer=1):
    """Oracle timed on the host cores on a bounded sample of the workload: its first
    `n_outer` outer FGMRES iteration(s) from x0 = 0, each including its full inner coarse
    solve (same method parameters as the GPU run)."""
    import oracle
    from workloads import config_problem
    p = config_problem(args.workload)
    prm = oracle_params(args, maxit=n_outer)
    s = oracle.Solver(p.k, p.h, p.bc, prm)
    t0 = time.perf_counter()
    x, rep = s.solve(p.b)
    dt = time.perf_counter() - t0
    cores = 1
    try:
        import threadpoolctl
        cores = max([i.get("num_threads", 1) for i in threadpoolctl.threadpool_info()] or [1])
    except Exception:
        pass
    inner = rep["inner_iterations"]
    return {"value": rep["outer_iterations"] / dt, "unit": "it/s", "cores": cores, "kind": "oracle",
            "sample": f"first {rep['outer_iterations']} outer FGMRES iteration(s) of {args.workload} from x0=0 "
                      f"(inner coarse solve: {sum(inner)} iterations), {dt:.1f} s"}


def kernel_roofline(H, rep, peaks, reps=20):
    """The roofline line of the step's dominant component, measured live here with CUDA events.

    The solve is a chain of small dependent kernels, so each component is timed the way it runs
    inside the solve: `reps` back-to-back instances captured into one CUDA graph and replayed
    (helm_bench_graph, warm).  Components: one delayed-CGS2 step of the inner FGMRES at the
    mean basis size (pass 1, reduction + step A, pass 2 + step B), one V-cycle from level 1,
    one E apply, one A apply.  Counts per step come from the solve's own iteration counts.
    Algorithmic bytes: DCGS2 step (2j + 7) * 16 n1; V-cycle sum over levels of
    (40 + 56) n_l + 32 n_{l+1} plus the dense coarsest inverse; E 32 n1 + 8 n0; A 40 n0.  The
    isolated per-kernel timings (L2 flushed before each launch) are reported beside it."""
    inner_its = rep["inner_iterations_total"]
    outer_its = rep["outer_iterations"]
    jm = max(1, int(round(rep["inner_iterations_total"] / max(1, rep["inner_solves"]) / 2)))
    lv = [ny * nx for (ny, nx, _) in H.levels]
    n0, n1 = lv[0], lv[1]
    vbytes = sum(96.0 * lv[l] + 32.0 * lv[l + 1] for l in range(1, len(lv) - 1)) + 16.0 * lv[-1] ** 2
    comps = [("dcgs2 step (inner, j=%d)" % jm, "dcgs", jm, 10, inner_its, (2 * jm + 7) * 16.0 * n1),
             ("V-cycle from level 1 (inner preconditioner)", "vcycle", 1, 20, inner_its + outer_its, vbytes),
             ("galerkin_apply E (level 1)", "apply_E", 0, 50, inner_its, 32.0 * n1 + 8.0 * n0),
             ("apply_op A (level 0)", "apply_A", 0, 50, 2 * outer_its, 40.0 * n0)]
    rows = {}
    for label, region, arg, nrep, count, nbytes in comps:
        us = H.helm_bench_graph(region, arg, nrep)
        gbs = nbytes / (us * 1e-6) / 1e9
        rows[label] = {"kernel": label, "bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                       "frac": gbs / peaks["hbm_gbs"], "traffic": None, "bytes_per_launch": nbytes,
                       "us_per_launch": us, "launches_per_step": count, "est_ms_per_step": count * us * 1e-3,
                       "timing": "in-graph, warm (helm_bench_graph)", "peak_src": peaks["src"]}
    dom = max(rows.values(), key=lambda r: r["est_ms_per_step"])
    # DRAM traffic of the dominant component from the committed ncu --set full capture of the
    # same component (cold caches): the kernels of one delayed-CGS2 step at inner column jm, or
    # of the first inner V-cycle from level 1 (tools/ncu_dcgs_summary.py)
    prof_name = ("dcgs_j%d" % jm) if dom["kernel"].startswith("dcgs2 step") else \
        ("vcycle1" if dom["kernel"].startswith("V-cycle from level 1") else None)
    if prof_name:
        try:
            with open(os.path.join(ROOT, "profiles", f"r01_ncu_{prof_name}.json")) as fh:
                prof = json.load(fh)
            dom["traffic"] = prof["dram_bytes_per_step"]
            dom["traffic_src"] = f"profiles/r01_ncu_{prof_name}.json (ncu --set full, cold caches)"
        except (OSError, KeyError, ValueError):
            pass
    iso = {}
    for name, arg in (("gs_dots", jm + 1), ("gs_update", jm + 1), ("apply_E", 0), ("apply_A", 0), ("vc_down", 0),
                      ("vc_up", 0), ("vc_down", 1), ("vc_up", 1)):
        us, nbytes = H.helm_bench_kernel(name, arg=arg, reps=reps, flush=True)
        gbs = nbytes / (us * 1e-6) / 1e9
        iso[f"{name}[{arg}]"] = {"us": us, "GB/s": gbs, "frac": gbs / peaks["hbm_gbs"]}
    return dict(dom), {"components": {k: {kk: v[kk] for kk in ("achieved", "frac", "us_per_launch",
                                                              "launches_per_step", "est_ms_per_step")}
                                      for k, v in rows.items()},
                       "isolated_kernels_l2_flushed": iso}


def microbench(peaks, n=16385, reps=10):
    """BASELINE configs[4] microbenchmark: isolated stencil apply and fused V-cycle legs on a
    16385^2-node (16383^2 Dirichlet unknowns) complex128 grid, L2 flushed before each launch."""
    import torch
    from paper_2308_06152_b200 import helm
    m = n - 2
    h = 1.0 / (n - 1)
    k = torch.full((m, m), 0.625 / h, dtype=torch.float64, device="cuda")
    H = helm.Helm(m, m, h, "dirichlet", k, {"inner_maxit": 2})
    out = {"grid": f"{m}x{m} unknowns (h=1/{n - 1}), complex128"}
    for name, arg in (("apply_A", 0), ("vc_down", 0), ("vc_up", 0)):
        us, nb = H.helm_bench_kernel(name, arg=arg, reps=reps, flush=True)
        gbs = nb / (us * 1e-6) / 1e9
        out[name] = {"us": us, "GB/s": gbs, "frac": gbs / peaks["hbm_gbs"], "bytes": nb}
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
        try:
            line = _run_decomposed(args, rank, world, local)
        except helm.HelmError as exc:
            # the peer transport reports a stalled peer (wait timeout) on every rank; the job then
            # reruns over NCCL instead of producing nothing
            if args.transport != "peer":
                raise
            print(f"[bench] peer transport failed ({exc}); rerunning over NCCL", file=sys.stderr, flush=True)
            args.transport = "nccl"
            args.transport_note = f"peer transport failed: {exc}"
            line = _run_decomposed(args, rank, world, local)
    if line is not None:
        print(json.dumps(line), flush=True)


def _run_decomposed(args, rank, world, local):
    """Weak scaling of ONE solve over the ranks: the workload's unit square
    stacked `world` times in y (strip_problem: same h and k, point source at the centre), one
    row strip per GPU; halos by grouped ncclSend/ncclRecv, dots by ncclAllReduce, the coarse
    levels below the decomposed ones all-gathered and replicated.  value = world x outer
    iterations / device time: each outer iteration covers `world` blocks of the N = 1
    workload, so value / (N x value at N = 1) is the time-per-iteration efficiency."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2308_06152_b200 import helm
    from workloads import config_problem, strip_problem
    torch.cuda.set_device(local)
    peaks = load_peaks()
    base = config_problem(args.workload)
    p = strip_problem(base.meta["k"], base.meta["n_cells"], world, f"{args.workload}_x{world}")
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
        # levels 0-2 decomposed, level 3 (79 x (80 N - 1) unknowns) and below replicated: 7 small
        # collectives per inner iteration instead of ~11 with the deepest possible split
        prm = dict(method_of(args), dist_levels=args.dist_levels or 3)
        H = helm.HelmDist(p.nx, p.ny, p.h, p.bc, p.k, rank, world, nccl_id=uid, params=prm, stream=stream,
                          peer_exchange=peer_exchange)
        bo = np.ascontiguousarray(p.b[H.row0:H.row0 + H.nrows])
        b = torch.from_numpy(bo).cuda()
        x = torch.empty_like(b)
        for _ in range(args.warmup):
            H.solve(b, 1e-6, args.maxit, x)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
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
        wall = time.perf_counter() - wall0
        dev_s = sum(a.elapsed_time(b_) for a, b_ in ev) * 1e-3
        if world > 1:
            tt = torch.tensor([dev_s], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dev_s = float(tt.item())
        its = sum(r["outer_iterations"] for r in reps)
        value = world * its / dev_s
        bh = torch.from_numpy(bo).pin_memory().numpy()
        xh = torch.empty(bo.shape, dtype=torch.complex128).pin_memory().numpy()
        H.solve_host(bh, xh, 1e-6, args.maxit)
        e2e_t, e2e_its = [], 0
        for s in range(args.steps):
            H.helm_flush_l2(256 << 20)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            _, r2 = H.solve_host(bh, xh, 1e-6, args.maxit)
            e2e_t.append(time.perf_counter() - t0)
            e2e_its += r2["outer_iterations"]
        e2e_s = sum(e2e_t)
        if world > 1:
            tt = torch.tensor([e2e_s], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        launches = sum(r["kernels"] for r in reps)
        H.close()
        roof = roof_all = None
        if rank == 0:   # kernel rooflines at the per-GPU block size (single-GPU context)
            Hs = helm.helm_setup(base, method_of(args), stream=stream)
            roof, roof_all = kernel_roofline(Hs, reps[-1], peaks)
            Hs.close()
    if rank != 0:
        return None
    line = {
        "metric": "fgmres_outer_iterations_per_s", "value": value, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps,
        "time_to_solution_s": dev_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": p.name, "per_gpu_block": args.workload, **method_of(args), "nx": p.nx, "ny": p.ny,
                   "h": p.h, "k": p.meta["k"], "tol": 1e-6, "l2": "flushed between timed steps (256 MiB read)",
                   "outer_iterations": reps[-1]["outer_iterations"],
                   "inner_iterations_mean": reps[-1]["inner_iterations_total"] / max(1, reps[-1]["inner_solves"]),
                   "parallelism": f"row-strip decomposition x{world} ({args.transport} transport)",
                   "dist_levels": prm["dist_levels"], "transport": args.transport,
                   **({"transport_note": args.transport_note} if getattr(args, "transport_note", None) else {}),
                   "value_definition": "world x outer iterations / max-over-ranks device time"},
        "wall_s": wall,
        "gpu_launches": launches,
        "e2e": {"value": world * e2e_its / e2e_s, "unit": "it/s", "h2d_bytes_per_step": int(bo.nbytes) * world,
                "d2h_bytes_per_step": int(bo.nbytes) * world},
        "roofline": roof,
        "roofline_kernels": roof_all,
        "clocks": clk.summary(),
    }
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c1_k400")
    ap.add_argument("--coarse-op", default=DEFAULT_METHOD["coarse_op"])
    ap.add_argument("--vectors", default=DEFAULT_METHOD["vectors"])
    ap.add_argument("--inner-tol", type=float, default=DEFAULT_METHOD["inner_tol"])
    ap.add_argument("--inner-maxit", type=int, default=DEFAULT_METHOD["inner_maxit"])
    ap.add_argument("--coarsest-n", type=int, default=DEFAULT_METHOD["coarsest_n"])
    ap.add_argument("--maxit", type=int, default=2000)
    ap.add_argument("--ref-iters", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-micro", action="store_true")
    ap.add_argument("--dist-levels", type=int, default=0, help="decomposed levels (0: 3)")
    ap.add_argument("--transport", default="peer", choices=["nccl", "peer"],
                    help="decomposed solve: NVLink peer memory through CUDA IPC (default; reruns over NCCL if a "
                         "peer stalls) or NCCL collectives")
    ap.add_argument("--decomp", default="auto", choices=["auto", "on", "off"],
                    help="row-strip decomposed solve over the ranks (NCCL); auto = on when N > 1")
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
    import numpy as np
    import torch
    from paper_2308_06152_b200 import helm
    from workloads import config_problem
    torch.cuda.set_device(local)
    peaks = load_peaks()
    p = config_problem(args.workload)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        H = helm.helm_setup(p, method_of(args), stream=stream)
        b = torch.from_numpy(p.b).cuda()
        x = torch.empty_like(b)
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            H.solve(b, 1e-6, args.maxit, x)
        launches0 = H.helm_launch_count()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        reps = []
        if world > 1:
            torch.distributed.barrier()
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
        if world > 1:
            t = torch.tensor([dev_s], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dev_s = float(t.item())
        its = sum(r["outer_iterations"] for r in reps)
        value = its * world / dev_s
        # end-to-end through the public API with host buffers (H2D of b, D2H of x)
        bh = torch.from_numpy(p.b).pin_memory().numpy()
        xh = torch.empty(p.shape, dtype=torch.complex128).pin_memory().numpy()
        H.solve_host(bh, xh, 1e-6, args.maxit)
        e2e_t = []
        e2e_its = 0
        for s in range(args.steps):
            H.helm_flush_l2(256 << 20)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, r2 = H.solve_host(bh, xh, 1e-6, args.maxit)
            e2e_t.append(time.perf_counter() - t0)
            e2e_its += r2["outer_iterations"]
        roof, roof_all = kernel_roofline(H, reps[-1], peaks)
    if rank != 0:
        return
    line = {
        "metric": "fgmres_outer_iterations_per_s", "value": value, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps,
        "time_to_solution_s": dev_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": args.workload, **method_of(args), "nx": p.nx, "ny": p.ny, "h": p.h,
                   "k": p.meta.get("k"), "tol": 1e-6, "l2": "flushed between timed steps (256 MiB write)",
                   "outer_iterations": reps[-1]["outer_iterations"],
                   "inner_iterations_mean": reps[-1]["inner_iterations_total"] / max(1, reps[-1]["inner_solves"]),
                   "inner_iterations_max": reps[-1]["inner_iterations_max"],
                   "parallelism": "replicas" if world > 1 else "single"},
        "wall_s": wall,
        "gpu_launches": launches,
        "e2e": {"value": e2e_its / sum(e2e_t), "unit": "it/s", "h2d_bytes_per_step": p.nx * p.ny * 16,
                "d2h_bytes_per_step": p.nx * p.ny * 16},
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
