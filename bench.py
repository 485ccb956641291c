#!/usr/bin/env python
"""Newton-step benchmark for the B200 hot path (BASELINE.json metric:
"Newton linear solves/s and BSR SpMV GB/s vs HBM peak").

One *step* = one first corrector pass of step_generalized_alpha
(timeint.cpp:54-176) on a seeded cube: predictor, stage blend, residual
assembly, tangent assembly with the kinematic fold-in, solve_block_system
with the nested (SCR) preconditioner -- including both AMG hierarchy setups
-- and the two-stage update.  Every step restarts from the same seeded state
(device-side copy), so K steps are K identical Newton linear solves.

Workload: BASELINE configs[1] (40^3 cube, fully incompressible, dt 1e-3,
the reference's solver settings) -- the configuration the reference itself
can run, so the reference arm times the SAME problem.  configs[4] (160^3)
is not runnable by the reference's algorithm in any practical sense: at dt
1e-3 its smoothed aggregation stops coarsening (level 1: 587,577 nodes ->
587,045 aggregates) and the hierarchy cannot be stored; at dt 0.1 the S_hat
hierarchy grows a 1.6e9-nonzero level whose RAP alone takes minutes even on
the B200.  --config 2|4 runs those sizes anyway.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: the path does not shard (exact Gauss-Seidel and greedy
aggregation are global-order dependent) -> N independent
replicas, one process per GPU, value = total solves / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Newton linear solves/s and BSR SpMV GB/s vs HBM peak (160^3 cube, 16.5M dofs)"
UNIT = "solves/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 4], help="BASELINE configs[i]")
    ap.add_argument("--n", type=int, default=None, help="override cells per cube edge")
    ap.add_argument("--nu", type=float, default=None)
    ap.add_argument("--dt", type=float, default=None)
    ap.add_argument("--cpu-sample-n", type=int, default=None, help="cube size of the CPU sample (default: the workload)")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg (profiling runs)")
    ap.add_argument("--spmv-n", type=int, default=160,
                    help="cube size of the 160^3 leg (the metric's BSR SpMV GB/s, assembly, Newton pass); 0 skips it")
    ap.add_argument("--big-dt", type=float, default=1e-2, help="time step of the 160^3 leg")
    ap.add_argument("--big-newton", type=int, default=1,
                    help="whole first Newton passes timed at 160^3 (0: skip; 1: one pass, which also builds the "
                         "mesh-static solver structures; 2: a warm-up pass first)")
    a = ap.parse_args()
    cfg = {0: (10, 0.4, 1e-3), 1: (40, 0.5, 1e-3), 2: (100, 0.45, 0.1), 4: (160, 0.5, 0.1)}[a.config]
    a.n = a.n or cfg[0]
    a.nu = a.nu if a.nu is not None else cfg[1]
    a.dt = a.dt if a.dt is not None else cfg[2]
    if a.cpu_sample_n is None:
        a.cpu_sample_n = a.n if a.n <= 40 else 16
    return a


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy test)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi clock/throttle sampling during the timed region."""

    def __init__(self, device):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        if os.environ.get("BENCH_NO_SMI"):
            self.p = None
            return
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "500"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        return world, rank, local, dist
    return 1, 0, 0, None


def max_over_ranks(dist, value):
    """Max over ranks (timing rule: the job is as slow as its slowest replica)."""
    if dist is None:
        return value
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(dist, world, steps, ms_local):
    """Whole-job throughput of N independent replicas: total solves / max time."""
    ms_max = max_over_ranks(dist, ms_local)
    return world * steps / (ms_max / 1e3), ms_max


def barrier(dist):
    if dist is not None:
        dist.barrier()


def cpu_reference_step(n, nu, dt):
    """The reference CPU path (oracle/_ref, single-threaded like the
    reference) on one seeded cube: one first corrector pass."""
    from oracle import ref
    from paper_1809_06350_b200 import CubeProblem

    cp = CubeProblem(n=n, nu=nu, dt=dt)
    P = ref.RefProblem(ref.cube_params(n, nu=nu, dt=dt))
    st = cp.seeded_state()
    opts = ref.SolverOptions.from_buffer_copy(bytes(cp.solver_options()))
    P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    t0 = time.perf_counter()
    out = P.newton_first_pass(opts)
    return time.perf_counter() - t0, out, cp


def _ref_worker(a):
    n, nu, dt = a
    t, out, cp = cpu_reference_step(n, nu, dt)
    return t, out["stats"], cp.nv + cp.np


def _host_mem_gb():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) / 1e6
    except OSError:
        pass
    return 16.0


def run_reference(args, world, rank, dist):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference compiled from its sources) on the SAME workload as our arm:
    K full first corrector passes of the seeded configs[i] cube.  The
    reference is single-threaded, so the host's cores run K independent
    passes as replicas (one process each, at most one per core and as many
    as host memory allows); value = K / wall time of the timed set."""
    if rank != 0:
        return
    import concurrent.futures as cf
    import multiprocessing as mp

    from paper_1809_06350_b200 import CubeProblem

    cw = CubeProblem(n=args.n, nu=args.nu, dt=args.dt)
    unknowns = cw.nv + cw.np
    gb_per_pass = 0.5 + 13.5e-6 * unknowns  # measured peak RSS: 3.6 GB for the 40^3 pass
    cores = os.cpu_count() or 1
    procs = max(1, min(cores, args.steps, int(_host_mem_gb() * 0.8 / gb_per_pass)))
    ctx = mp.get_context("fork")
    with cf.ProcessPoolExecutor(max_workers=procs, mp_context=ctx) as ex:
        if args.warmup > 0:  # no JIT or caches to warm: one tiny cube per worker
            list(ex.map(_ref_worker, [(4, args.nu, args.dt)] * procs))
        t0 = time.perf_counter()
        res = list(ex.map(_ref_worker, [(args.n, args.nu, args.dt)] * args.steps))
        wall = time.perf_counter() - t0
    value = args.steps / wall
    per_pass = [r[0] for r in res]
    sample = (f"reference (oracle/_ref, the unmodified reference compiled from its sources) first corrector pass on "
              f"the {args.n}^3 cube ({unknowns} unknowns, seeded, nu={args.nu}, dt={args.dt}), {args.steps} passes "
              f"as {procs} concurrent single-threaded processes; mean single-pass time {statistics.mean(per_pass):.2f} s")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64 state)",
        "config": workload_config(args, cw),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "reference", "sample": sample,
                         "single_pass_s": per_pass, "stats": res[-1][1]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def workload_config(args, cp):
    return {"workload": f"configs[{args.config}]: cube {args.n}^3 first Newton corrector pass", "n": args.n,
            "nu": args.nu, "dt": args.dt, "unknowns": cp.nv + cp.np, "tets": cp.mesh.n_tets,
            "solver": "FGMRES(200) 1e-6 / SCR a,s,inner 1e-2, AMG SGS (reference defaults)"}


def cube_leg(n, dt, device, peak, newton):
    """The metric's 160^3 quantities (configs[4] size: 16.6 M unknowns, ~9 GB
    coupled matrix >> 126 MB L2).  Mesh, residual and tangent assembly on the
    device; the coupled / A-plane / S_hat SpMVs and the fine Gauss-Seidel half
    sweep, each timed with CUDA events over 5 launches; assembly rates; and,
    when `newton`, one whole first Newton corrector pass (both AMG setups and
    the nested FGMRES solve; a warm-up pass first builds the mesh-static
    structures), device-timed, with its counts and phase split."""
    import gc

    from paper_1809_06350_b200 import CubeProblem

    t0 = time.perf_counter()
    cp = CubeProblem(n=n, nu=0.5, dt=dt)
    st = cp.seeded_state()
    ctx = cp.context(device)
    ctx.set_state(st)
    ctx.assemble_residuals()
    ctx.assemble_tangent(cp.ts)
    k = ctx.bench_kernels(cp.solver_options(), n_rep=5)
    out = {"n": n, "dt": dt, "nu": 0.5, "unknowns": cp.nv + cp.np, "tets": cp.mesh.n_tets,
           "setup_s": round(time.perf_counter() - t0, 1)}
    spmv = {}
    for name, (ms, by) in k.items():
        gbs = by / (ms * 1e-3) / 1e9
        spmv[name] = {"ms": ms, "bytes": by, "achieved_gbs": gbs, "frac": gbs / peak, "frac_8tbs": gbs / 8000.0}
    out["spmv"] = spmv
    out["assembly"] = assembly_row(ctx.bench_assembly(cp.ts, n_rep=3), peak)
    if newton:
        opts = cp.solver_options()
        ctx.set_state(st)
        ctx.state_save()
        passes = []
        for rep in range(max(1, int(newton))):
            ctx.state_restore()
            ctx.timer_start()
            o = ctx.newton_first_pass(cp.ts, opts)
            ms = ctx.timer_stop()
            passes.append({"ms": ms, "stats": o["stats"], "norm": o["norm"], "history": [float(h) for h in o["history"]],
                           "phase_ms": o["times"]})
        last = passes[-1]
        out["newton"] = {"solves_per_s": 1e3 / last["ms"], "pass_ms": last["ms"],
                         "warm_pass_ms": passes[0]["ms"] if len(passes) > 1 else None,
                         "stats": last["stats"], "norm": last["norm"], "history": last["history"],
                         "phase_ms": last["phase_ms"],
                         "note": "device-timed first corrector pass (residual, tangent, both AMG setups, nested "
                                 "FGMRES, update) from the seeded state; the reference cannot run this size "
                                 "(DESIGN.md §5), so there is no same-config CPU number"}
    ctx.close()
    del ctx, cp
    gc.collect()
    return out


# FP64 flops per element of the tangent (element kernel + fold-in) and the
# residual kernels: ncu sm__sass_thread_inst_executed_op_{dadd,dmul,dfma}
# (fma = 2) of every colour launch of one pass over its elements (profiles/r02/assembly_fp64_ncu.md)
TANGENT_FLOP_PER_ELEM = 21298.0
RESIDUAL_FLOP_PER_ELEM = 1632.5


def assembly_row(a, peak):
    """Assembly at the metric's size: Melem/s, algorithmic GB/s
    against HBM, FP64 rate against the measured FMA peak."""
    E = a["elements"]
    row = {"elements": E, "fp64_peak_gflops_measured": a["fp64_peak_gflops"],
           "k4_staging_bytes": a["k4_bytes"], "plane_bytes": a["plane_bytes"]}
    for part, fpe in (("residual", RESIDUAL_FLOP_PER_ELEM), ("tangent", TANGENT_FLOP_PER_ELEM)):
        ms, by = a[f"{part}_ms"], a[f"{part}_bytes"]
        r = {"ms": ms, "melem_s": E / (ms * 1e-3) / 1e6, "bytes": by, "achieved_gbs": by / (ms * 1e-3) / 1e9,
             "hbm_frac": by / (ms * 1e-3) / 1e9 / peak}
        if fpe:
            r["fp64_gflops"] = fpe * E / (ms * 1e-3) / 1e9
            r["fp64_frac"] = r["fp64_gflops"] / a["fp64_peak_gflops"]
        row[part] = r
    return row


def _profiler_range():
    """cudaProfilerStart/Stop through the CUDA runtime torch already loaded
    (no-ops unless a profiler is attached)."""
    try:
        import torch

        def f(on):
            (torch.cuda.profiler.start if on else torch.cuda.profiler.stop)()
        return f
    except Exception:  # pragma: no cover
        return lambda on: None


def _ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    summary (profiles/traffic.json: {"kernel@level": bytes}), else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if kernel is None or not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f).get(kernel)


def _pinned_state(st):
    """The step's host inputs in page-locked memory (the e2e contract)."""
    import numpy as np
    import torch

    from paper_1809_06350_b200 import State

    def pin(a):
        t = torch.empty(a.shape[0], dtype=torch.float64, pin_memory=True)
        v = t.numpy()
        v[:] = a
        _pinned_state.keep.append(t)
        return v
    return State(*[pin(np.asarray(a)) for a in (st.u, st.udot, st.p, st.pdot, st.v, st.vdot)])


_pinned_state.keep = []


def run_ours(args, world, rank, local, dist):
    import numpy as np

    from paper_1809_06350_b200 import CubeProblem

    cp = CubeProblem(n=args.n, nu=args.nu, dt=args.dt)
    st = cp.seeded_state()
    ctx = cp.context(local)
    opts = cp.solver_options()
    ctx.set_state(st)
    ctx.state_save()
    # warm-up (builds every mesh-static structure: patterns, S_hat symbolic, level schedules)
    for _ in range(args.warmup):
        ctx.state_restore()
        out = ctx.newton_first_pass(cp.ts, opts)
    barrier(dist)
    clocks = Clocks(local)
    l0 = ctx.kernel_launches()
    prof = _profiler_range()
    prof(True)  # ncu --profile-from-start off captures exactly the timed steps
    acct_on = os.environ.get("BENCH_NO_ACCT") is None
    ctx.kernel_accounting(acct_on)  # CUDA events around every sparse launch, on the library stream
    ctx.timer_start()
    phase = []
    for _ in range(args.steps):
        ctx.state_restore()
        out = ctx.newton_first_pass(cp.ts, opts)
        phase.append(out["times"])
    ms = ctx.timer_stop()
    prof(False)
    acct = ctx.kernel_account()
    ctx.kernel_accounting(False)
    launches = ctx.kernel_launches() - l0
    clk = clocks.stop()
    value, ms_max = replica_value(dist, world, args.steps, ms)
    barrier(dist)

    # end to end through the public API: host state in, solution out
    h2d = 14 * 8 * cp.mesh.n_nodes
    d2h = 8 * (cp.nv + cp.np) + 8
    st_pinned = _pinned_state(st)
    e2e_ms, e2e_phase = [], None
    barrier(dist)
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        ctx.set_state(st_pinned)
        out_e = ctx.newton_first_pass(cp.ts, opts)
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
        e2e_phase = out_e["times"]
    e2e_mean = max_over_ranks(dist, sum(e2e_ms) / len(e2e_ms) if e2e_ms else 0.0)
    e2e_value = world / (e2e_mean / 1e3) if e2e_mean > 0 else None

    kern = ctx.bench_kernels(opts, n_rep=10)
    if rank != 0:
        return
    peak, peak_src = peaks()
    # kernels standalone (cold inputs, n_rep launches each): the metric's SpMV
    micro = {}
    for name, (kms, kbytes) in kern.items():
        gbs = kbytes / (kms * 1e-3) / 1e9
        micro[name] = {"ms": kms, "bytes": kbytes, "achieved_gbs": gbs, "frac": gbs / peak}
    # live, inside the timed steps: every sparse launch bracketed by events;
    # the dominant class (most device time) is the roofline headline
    step_ms = ms / args.steps
    live = {}
    for name, (n_l, kms, kbytes) in acct.items():
        live[name] = {"launches_per_step": n_l / args.steps, "ms_per_step": kms / args.steps,
                      "share_of_step": (kms / args.steps) / step_ms, "bytes_per_launch": kbytes / max(n_l, 1),
                      "ms_per_launch": kms / max(n_l, 1), "achieved_gbs": kbytes / (kms * 1e-3) / 1e9 if kms > 0 else 0.0}
    live = dict(sorted(live.items(), key=lambda kv: -kv[1]["ms_per_step"]))
    # SURVEY.md 8d solve roofline: algorithmic bytes of every accounted launch of
    # the solve (SpMV, sweeps, dense GEMV, Krylov vector kernels) / HBM peak,
    # against the measured FGMRES time (AMG setup excluded, reported beside it)
    solve_bytes = sum(kbytes for (_, _, kbytes) in acct.values()) / args.steps
    fg_ms = sum(p["fgmres_ms"] for p in phase) / len(phase)
    solve_roof = {"bytes_per_step": solve_bytes, "time_roof_ms": solve_bytes / (peak * 1e9) * 1e3,
                  "fgmres_ms": fg_ms, "frac": solve_bytes / (peak * 1e9) * 1e3 / fg_ms,
                  "time_roof_ms_8tbs": solve_bytes / 8e12 * 1e3,
                  "amg_setup_ms": sum(p["amg_setup_ms"] for p in phase) / len(phase)}
    top = next(iter(live)) if live else None
    head = live[top] if top else {"achieved_gbs": 0.0}
    traffic = _ncu_traffic(top)
    cpu = None
    if world == 1 and not args.no_cpu:
        t_cpu, _, cpc = cpu_reference_step(args.cpu_sample_n, args.nu, args.dt)
        cpu = {"value": 1.0 / t_cpu, "unit": UNIT, "cores": 1, "kind": "reference",
               "sample": f"reference (oracle/_ref, 1 thread) first corrector pass on the {args.cpu_sample_n}^3 cube "
                         f"({cpc.nv + cpc.np} unknowns) in {t_cpu:.2f} s"
                         + ("" if args.cpu_sample_n == args.n else f" (bounded sample of the {args.n}^3 workload)")}
    big = cube_leg(args.spmv_n, args.big_dt, local, peak, args.big_newton) if args.spmv_n > 0 else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64 state, SURVEY.md §8d)",
        "config": dict(workload_config(args, cp), parallelism=f"replicas{world}",
                       l2_flush="none needed for the step (AMG setup rewrites every level each step); kernel rows: cold inputs"),
        "roofline": {"bound": "hbm", "kernel": top, "achieved": head["achieved_gbs"], "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": head["achieved_gbs"] / peak,
                     "traffic": traffic,
                     "note": ("Gauss-Seidel half sweeps keep the reference's sequential semantics: their time is "
                              "dependency levels x per-level latency, not bytes (DESIGN.md §4)"),
                     "live_kernels": dict(list(live.items())[:10]), "standalone_kernels": micro,
                     "solve": solve_roof},
        "cfg4": big,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms": e2e_ms, "host_inputs": "pinned", "phase_ms_last": e2e_phase},
        "gpu_launches": launches,
        "clocks": clk,
        "newton": {"norm": out["norm"], "stats": out["stats"], "phase_ms_last": phase[-1] if phase else None,
                   "setup_fgmres_ms_per_step": [[round(p["amg_setup_ms"], 1), round(p["fgmres_ms"], 1)] for p in phase]},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local, dist = dist_init(args)
    if args.impl == "reference":
        run_reference(args, world, rank, dist)
    else:
        run_ours(args, world, rank, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
