#!/usr/bin/env python3
"""bench.py — throughput of the B200 MR/FV Euler hot path (and the reference arm).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4|cfg2|cfg3|cfg1|cfg5]
    python bench.py --impl reference ...      # the reference's own CPU path

Default workload: "cfg4" (BASELINE.json configs[3]), the largest config that
fits one GPU and the one north_star's scaling target names: 3D Euler on the
uniform 512^3 mesh, fp64, seeded ellipsoid, outflow BCs, MUSCL/minmod +
AUSM+ + RK2, CFL 0.4. A "step" is one RK2 step over the whole mesh (two fused
stage launches); the default K is the config's own 100 steps. The state (5.4
GB) is far larger than L2, so no flush is needed between steps. The metric
is BASELINE.json's: leaf-cell RK-stage updates / s. The MR workloads (cfg2,
cfg3) time run_mr cycles (refine, virtual leaves, the RK2 step, coarsen).
Multi-GPU (torchrun): slabs with NCCL halo exchange.

Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-updates/sec (fp64, leaf cells x RK stages)"
UNIT = "cell-updates/s"

WORKLOADS = {
    # name: (BASELINE config index, case kind, dim, level, cfl, seed, steps in the config)
    "cfg1": (0, 0, 2, 8, 0.5, 1, 200),
    "cfg2": (1, 0, 2, 10, 0.5, 1, 500),
    "cfg3": (2, 1, 2, 13, 0.5, 1, 64),
    "cfg4": (3, 2, 3, 9, 0.4, 1, 100),
    # 3D MRLT at 1024^3 is an 8-GPU config (one rank's windowed share is ~1/5 of
    # the ~217 GB tree); --level runs it smaller
    "cfg5": (4, 3, 3, 10, 0.4, 1, 16),
}
# The AMR patch path (not a BASELINE.json config: these lines are
# recorded under profiles/, the default line stays cfg4). The reference's AMR preset
# (AUSMDV / minmod / MUSCL-Hancock), time-refined, its paper base meshes (64^2, 8^3).
AMR_WORKLOADS = {
    # name: (case kind, dim, base_exp, level, dt_finest, seed, cycles)
    "amr2d": (0, 2, 6, 10, 2.5e-4, 1, 4),
    "amr3d": (3, 3, 3, 8, 3.5e-4, 1, 2),
}
BASE_LEVEL = {k: v[3] for k, v in WORKLOADS.items()}
# MR options per MR workload (BASELINE.json configs[1], configs[2])
MR_OPTS = {
    "cfg2": dict(eps=1e-3, eps_scaled=True, min_leaf=3, local_time=False, gap=3),
    "cfg3": dict(eps=1e-3, eps_scaled=False, min_leaf=0, local_time=True, gap=3),
    # coarsest 16^3 = min leaf level 4 with gap = L - 4 (the gap
    # of 3 would otherwise force leaves to level >= 7)
    "cfg5": dict(eps=1e-3, eps_scaled=True, min_leaf=4, local_time=True, gap=6),
}


def mr_options(workload):
    o = MR_OPTS[workload]
    _, _, dim, level, _, _, _ = WORKLOADS[workload]
    epsl = ([o["eps"] * 2.0 ** (dim * (l - level)) for l in range(level + 1)]
            if o["eps_scaled"] else None)
    return o, epsl


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks --
def fp64_info():
    """The fp64-pipe side of the roofline: measured fp64
    throughput (tools/micro/fp64peak.cu) and the stage kernel's fp64-pipe
    utilisation from its ncu capture (profiles/fp64_peaks.json)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "fp64_peaks.json")))
        return {"peak_dadd_per_s": d["dadd_per_s"], "peak_ddiv_per_s": d["ddiv_ieee_per_s"],
                "stage_pipe_frac": d["fv3d_stage_fp64_pipe_frac"], "source": d["source"]}
    except Exception:
        return None


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region, in
    process through NVML (the nvidia-smi query fields clocks.sm,
    clocks.max.sm, clocks_event_reasons.*): one sample when the region
    starts, one every `period` s from a background thread, one when it ends.
    NVML is initialised before the region so its start-up cost stays out."""

    HW_SLOWDOWN, SW_THERMAL, HW_THERMAL, SW_POWER = 0x8, 0x20, 0x40, 0x4

    def __init__(self, device: int, period: float = 0.005):
        self.period = period
        self.rows = []
        self.thread = None
        self.stop_evt = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.sample()
            self.rows.clear()
        except Exception:
            self.nv = None

    def sample(self):
        nv = self.nv
        self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                          nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))

    def _loop(self):
        while not self.stop_evt.wait(self.period):
            self.sample()

    def start(self):
        if self.nv is None:
            return
        self.sample()
        self.thread = threading.Thread(target=self._loop, daemon=True)
        self.thread.start()

    def stop(self):
        if self.nv is None:
            return None
        self.sample()
        self.stop_evt.set()
        self.thread.join()
        names = {self.HW_SLOWDOWN: "hw_slowdown", self.HW_THERMAL: "hw_thermal_slowdown",
                 self.SW_THERMAL: "sw_thermal_slowdown", self.SW_POWER: "sw_power_cap"}
        reasons = sorted({v for r in self.rows for k, v in names.items() if r[1] & k})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.rows),
                "source": "nvml"}


# ------------------------------------------------------------- CPU legs -----
CORE_RATE_3D = 4.5e6   # reference cell-stage updates/s per core on the 3D path (r01 B200 host)
PLANE_BYTES_3D = 4 * 40  # u, step_block's mid, rk2_stage's rhs and w per ghosted cell


def window_plan(n: int, threads: int, steps: int, budget_s: float):
    """z-window of the n^3 mesh the multi-core reference arm steps: the whole
    mesh when K steps fit the time budget and host memory, else the largest
    centred window that does (a multiple of the thread count)."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16e9
    per_plane = PLANE_BYTES_3D * (n + 4) ** 2
    mem_planes = int(0.5 * avail / per_plane) - 4 * threads
    time_planes = int(budget_s * threads * CORE_RATE_3D / (2.0 * n * n * max(1, steps)))
    nz = max(threads, min(n, mem_planes, time_planes))
    nz = max(threads, nz - nz % threads)
    return (n - nz) // 2, nz


def reference_cpu_rate(kind: str, workload: str, steps: int, warmup: int, threads: int,
                       level_override: int | None = None, budget_s: float = 150.0):
    """Times the CPU implementation (`kind` "reference" = oracle/_ref, the
    reference library compiled from its own sources; "port" = the C
    restatement). Returns (rate, sample description, wall, ran) where `ran`
    says exactly what was stepped.

    3D uniform (cfg4): the config's own n^3 mesh, or a centred z-window of it
    when K steps of the whole mesh would not fit `budget_s`, split into one
    z-slab per thread, each stepped by the reference's own step_block
    (oracle/ref_harness.cpp afref_uniform_window_run; bit-identical to the
    single-domain run on the whole mesh). Other workloads: `threads`
    independent single-threaded copies of the same generator at a smaller
    level (MR: the reference's from_uniform + coarsen takes minutes at L >= 8)."""
    from oracle import oracle as O
    _, case, dim, level, cfl, seed, _ = WORKLOADS[workload]
    is_mr = workload in MR_OPTS
    if dim == 3 and not is_mr and kind == "reference" and level_override is None:
        n = 1 << level
        z0, nz = window_plan(n, threads, steps + min(warmup, 1), budget_s)
        init = O.window_init(case, seed, level, z0, nz)
        p = O.make_params(dim, level, steps, cfl=cfl)
        _, res = O.uniform_window_run(p, init, z0, nz, threads, min(warmup, 1))
        if res["err_kind"]:
            raise RuntimeError(res["err"])
        wall = res["wall_seconds"]
        work = nz * n * n * 2 * steps
        whole = nz == n
        ran = {"mesh": f"{n}x{n}x{n}", "z_window": [z0, z0 + nz], "whole_mesh": whole,
               "threads": threads, "steps_timed": steps, "warmup_steps": min(warmup, 1)}
        sample = (f"{'the whole' if whole else f'z-planes [{z0},{z0 + nz}) of the'} "
                  f"{n}^3 {workload} mesh ({nz * n * n} cells), split into {threads} z-slabs, "
                  f"one thread each running the reference's step_block (unigrid.cpp:39) with "
                  f"neighbour ghost planes between stages; {steps} RK2 steps timed after "
                  f"{min(warmup, 1)} warm-up; steady_clock around the step loop; value = "
                  f"cell RK-stage updates / s")
        return work / wall, sample, wall, ran
    if level_override is not None:
        lvl = level_override
    elif is_mr:
        lvl = {"cfg2": 7, "cfg3": 8, "cfg5": 5}[workload]
    else:
        lvl = 7 if dim == 3 else level
    init = O.case_fill(case, seed, lvl)
    cells = init.shape[0]
    lib_kind = "ref" if kind == "reference" else "port"
    results = [None] * threads
    work = [0] * threads

    def params(n):
        if not is_mr:
            return O.make_params(dim, lvl, n, cfl=cfl)
        o = MR_OPTS[workload]
        epsl = ([o["eps"] * 2.0 ** (dim * (l - lvl)) for l in range(lvl + 1)]
                if o["eps_scaled"] else None)
        return O.make_params(dim, lvl, n, cfl=cfl, eps=o["eps"], eps_level=epsl,
                             min_leaf_level=o["min_leaf"], local_time=o["local_time"],
                             lt_gap=o["gap"])

    def one(i):
        if is_mr:
            if warmup:
                O.mr_run(lib_kind, params(warmup), init)
            _, _, cyc, _, res = O.mr_run(lib_kind, params(steps), init)
            work[i] = int(cyc[:, 4].sum())
        else:
            if warmup:
                O.uniform_run(lib_kind, params(warmup), init)
            _, _, res = O.uniform_run(lib_kind, params(steps), init)
            work[i] = cells * 2 * steps
        results[i] = res

    ts = [threading.Thread(target=one, args=(i,)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    wall = max(r["wall_seconds"] for r in results)
    rate = sum(work) / wall
    what = "MR cycles (refine/evolve/coarsen)" if is_mr else "RK2 steps"
    n = 1 << lvl
    ran = {"mesh": "x".join([str(n)] * dim), "finest_level": lvl, "copies": threads,
           "threads": threads, "steps_timed": steps, "warmup_steps": warmup}
    sample = (f"{threads} independent single-threaded copies of the {workload} generator at "
              f"level {lvl} ({cells} finest cells), {steps} {what} each after {warmup} "
              f"warm-up; steady_clock around the step loop only (unigrid.cpp:31-48, "
              f"mr_solver.cpp:339-395); value = leaf-cell RK-stage updates / s")
    return rate, sample, wall, ran


def host_threads(req: int) -> int:
    """Cores this process may run on (cgroup/affinity aware), capped by `req` if > 0."""
    try:
        avail = len(os.sched_getaffinity(0))
    except AttributeError:
        avail = os.cpu_count() or 1
    return max(1, min(avail, req) if req > 0 else avail)


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU implementation (rank 0 only)."""
    if rank != 0:
        return
    from oracle import oracle as O
    kind = "reference" if O.available("ref") else "port"
    if kind == "port" and not O.available("port"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle libraries not built"}))
        return
    threads = host_threads(args.cpu_threads)
    rate, sample, wall, ran = reference_cpu_rate(kind, args.workload, max(1, args.steps),
                                                 max(0, args.warmup), threads,
                                                 level_override=args.ref_level)
    idx, case, dim, level, cfl, seed, _ = WORKLOADS[args.workload]
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(1, args.steps), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(workload_config(args.workload, 1, "exact"),
                       parity_mode="the reference's own CPU implementation (oracle/_ref)"),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads,
                         "kind": kind, "sample": sample, "ran": ran},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


NUMERICS = {"tolerance": "tolerance: within 1e-10 relative L1 per field of the bit-exact result "
                         "(BASELINE.json north_star bar; reciprocal estimates + FMA, "
                         "tests/test_tolerance_gpu.py)",
            "exact": "bit-exact (--fmad=false, the reference's operations)"}


def workload_config(workload, n_gpus, numerics="exact"):
    idx, case, dim, level, cfl, seed, steps = WORKLOADS[workload]
    n = 1 << level
    c = {"workload": f"{workload}: BASELINE.json configs[{idx}]",
         "mesh": "x".join([str(n)] * dim), "dim": dim, "scheme": "AUSM+/minmod/RK2",
         "cfl": cfl, "cfl_rule": "dt_L = cfl*dx_L / max_leaves sum_a(|v_a|+c)", "seed": seed,
         "bc": "outflow",
         "l2": "inputs larger than L2 (no flush)" if (n ** dim) * 40 > 126e6
               else "working set fits in L2 (latency-bound config)",
         "parity_mode": NUMERICS["exact"]}
    if dim == 3 and workload not in MR_OPTS:
        c["parity_mode"] = NUMERICS[numerics]
    if dim == 2 and workload in MR_OPTS and numerics == "tolerance":
        c["parity_mode"] = ("tolerance: full-tile stages with reciprocal estimates + FMA, within "
                            "1e-10 relative L1 per field of the bit-exact run with identical leaf "
                            "sets (tests/test_mr_tolerance_gpu.py)")
    if BASE_LEVEL.get(workload, level) != level:
        c["level_override"] = f"finest level {level} instead of the config's {BASE_LEVEL[workload]}"
    if workload in MR_OPTS:
        o = MR_OPTS[workload]
        c.update({"method": "MRLT" if o["local_time"] else "MR (global dt)",
                  "finest_level": level, "min_leaf_level": o["min_leaf"],
                  "eps": ("1e-3*2^(d(l-L))" if o["eps_scaled"] else o["eps"]),
                  "lt_gap": o["gap"] if o["local_time"] else None,
                  "step": "one MR cycle (refine, virtual leaves, evolve, coarsen)",
                  "decomposition": "single GPU (per-level dense grids)"})
    else:
        c["decomposition"] = f"{n_gpus} slab(s) along the last axis"
    return c


# ----------------------------------------------------------------- GPU arm --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: the config's own step count, e.g. cfg2's 500 "
                         "cycles, cfg4's 100 steps)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=sorted(WORKLOADS) + sorted(AMR_WORKLOADS))
    ap.add_argument("--level", type=int, default=None,
                    help="run the workload at another finest level (not the config's own)")
    ap.add_argument("--mr-multi", default="auto", choices=["auto", "slabs", "replicas"],
                    help="MR at N>1: slab decomposition or independent replicas "
                         "(auto: replicas for the single-GPU cfg2, slabs otherwise)")
    ap.add_argument("--cpu-threads", type=int, default=0,
                    help="host threads for the CPU legs (0 = every core this process may use)")
    ap.add_argument("--ref-level", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-other-numerics", action="store_true")
    ap.add_argument("--numerics", default=None, choices=["tolerance", "exact"],
                    help="3D uniform stage numerics: 'tolerance' (reciprocal estimates + FMA, "
                         "within BASELINE.json's 1e-10 relative L1 per field of the exact result; "
                         "tests/test_tolerance_gpu.py) or 'exact' (bit-identical to the "
                         "reference). The other mode is timed too and reported beside it.")
    args = ap.parse_args()
    if args.workload in AMR_WORKLOADS:
        amr_main(args)
        return
    if args.numerics is None:  # uniform 3D: tolerance; MR: exact (its established bar)
        args.numerics = "exact" if args.workload in MR_OPTS else "tolerance"
    if args.steps is None:
        args.steps = WORKLOADS[args.workload][6]
    if args.level is not None:
        w = list(WORKLOADS[args.workload])
        w[3] = args.level
        WORKLOADS[args.workload] = tuple(w)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import ctypes as C
    from paper_1603_05211_b200 import _abi
    from paper_1603_05211_b200 import uniform as U

    lib = _abi.load()
    idx, case, dim, level, cfl, seed, _ = WORKLOADS[args.workload]
    comm = None
    needs_comm = world > 1 and (args.workload not in MR_OPTS or mr_decomposed(args, world))
    if needs_comm:  # NCCL only where the path exchanges (not for MR replicas)
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            assert lib.af_comm_unique_id(C.cast(uid, C.c_char_p)) == 0
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_ubyte * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        st = lib.af_comm_create(C.cast(uid, C.c_char_p), world, rank, local, C.byref(h))
        assert st == 0, "af_comm_create failed"
        comm = h

    if args.workload in MR_OPTS:
        line = mr_bench(args, rank, world, local, comm, torch, dist)
    else:
        line = uniform_bench(args, rank, world, local, comm, torch, dist)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def uniform_bench(args, rank, world, local, comm, torch, dist):
    from paper_1603_05211_b200 import uniform as U
    idx, case, dim, level, cfl, seed, _ = WORKLOADS[args.workload]
    solver = U.UniformSolver(dim, level, scheme=U.SchemeConfig(limiter=U.MINMOD),
                             device=local, comm=comm)
    tol = dim == 3 and args.numerics == "tolerance"
    solver.set_numerics(tol)
    # A dedicated (non-default) stream: the solver's kernels and the timing
    # events must be on the same stream.
    stream = torch.cuda.Stream(device=local)
    solver.set_stream(stream)
    n = 1 << level
    init_host = U.case_fill(case, seed, level, z0=solver.z0, nz=solver.nz)
    init_pinned = torch.from_numpy(init_host).pin_memory()
    init_dev = init_pinned.to(f"cuda:{local}")
    out_pinned = torch.empty_like(init_pinned).pin_memory()
    cells_local = solver.cells
    cells_total = n ** dim

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident throughput ("value") -------------------------------
    solver.upload(init_dev)
    solver.run(args.warmup, cfl=cfl, collect=False)   # W untimed warm-up steps
    solver.sync()
    l0 = solver.kernel_launches()
    sampler = ClockSampler(local)
    barrier()
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    solver.run(args.steps, cfl=cfl, collect=False)
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    launches = solver.kernel_launches() - l0
    solver.sync()
    ms = max_over_ranks(ms)
    value = cells_total * 2 * args.steps / (ms / 1e3)

    # ---- end to end through the C ABI with host buffers ----------------------
    e2e = None
    if not args.no_e2e:
        # untimed warm-up of the host-buffer path
        solver.upload(init_pinned.numpy())
        solver.run(1, cfl=cfl, collect=False)
        solver.download(out_pinned.numpy())
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        solver.upload(init_pinned.numpy())   # pinned host -> device
        solver.run(args.steps, cfl=cfl, collect=False)
        solver.download(out_pinned.numpy())  # device -> pinned host (synchronises)
        t1.record(stream)
        barrier()
        ems = max_over_ranks(t0.elapsed_time(t1))
        e2e = {"value": cells_total * 2 * args.steps / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(cells_local * 40 * world / args.steps),
               "d2h_bytes_per_step": int(cells_local * 40 * world / args.steps),
               "what": "one run_uniform-equivalent call: upload of the initial state from "
                       "pinned host memory, K steps, download of the final state"}

    # ---- the other 3D numerics mode, same steps, for reference ---------------
    other = None
    if dim == 3 and not args.no_other_numerics:
        solver.set_numerics(not tol)
        solver.upload(init_dev)
        solver.run(max(1, args.warmup), cfl=cfl, collect=False)
        barrier()
        o0, o1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        o0.record(stream)
        solver.run(args.steps, cfl=cfl, collect=False)
        o1.record(stream)
        barrier()
        oms = max_over_ranks(o0.elapsed_time(o1))
        solver.set_numerics(tol)
        oname = "exact" if tol else "tolerance"
        other = {"numerics": NUMERICS[oname], "value": cells_total * 2 * args.steps / (oms / 1e3),
                 "unit": UNIT, "ms_per_step": oms / args.steps,
                 "kernel": "fv3d_tile<16x15, exact>" if oname == "exact" else
                           "fv3d_tile<16x15, tolerance>"}

    if rank != 0:
        return None

    # ---- roofline of the dominant kernel (the fused RK2 stage) ---------------
    hbm, src = peaks()
    S = (dim + 2) * 8
    alg_bytes_per_launch = 2.5 * S * cells_local       # 2.5 S per cell-stage
    avg_launch_s = (ms / 1e3) / (2 * args.steps)        # timed region = 2 stage launches/step
    achieved = alg_bytes_per_launch / avg_launch_s / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "peak_source": src,
            "kernel": ("fv3d_tile<16x15, tolerance>" if tol else "fv3d_tile<16x15, exact>")
                      if dim == 3 else "fv2d_stage",
            "fp64": fp64_info(),
            "note": "fp64-pipe and issue bound (~400 fp64 instructions per cell-stage), not "
                    "HBM bound; see DESIGN.md"}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            from oracle import oracle as O
            kind = "reference" if O.available("ref") else "port"
            threads = host_threads(args.cpu_threads)
            rate, sample, _, ran = reference_cpu_rate(kind, args.workload, 2, 1, threads,
                                                      budget_s=20.0)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
                   "sample": sample, "ran": ran}
        except Exception as e:  # the CPU leg must not sink the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args.workload, world, args.numerics),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks, "other_numerics": other,
    }
    return line




def mr_partition_level(o, level, world):
    """The partition level af_mr_create_dist picks (MR::MR): smallest l with
    2^l >= 4N, capped at the minimum leaf level."""
    ml = max(o["min_leaf"], max(0, level - o["gap"])) if o["local_time"] else o["min_leaf"]
    lp = 0
    while (1 << lp) < 4 * world and lp < ml:
        lp += 1
    return lp


def mr_decomposed(args, world):
    """MR at N > 1: the slab decomposition of SURVEY §8(e) (one tree, strong
    scaling) for the multi-GPU MR configs (cfg3); cfg2 is a single-GPU config
    in BASELINE.json, so its N > 1 lines run independent replicas (weak)."""
    if world == 1:
        return False
    if args.mr_multi == "auto":
        return args.workload != "cfg2"
    return args.mr_multi == "slabs"


def mr_bench(args, rank, world, local, comm, torch, dist):
    """MR / MRLT workloads (cfg2, cfg3). A step = one macro cycle of run_mr
    (refine, virtual leaves, evolve, coarsen); value = leaf-cell RK-stage
    updates actually performed / s (whole job)."""
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    idx, case, dim, level, cfl, seed, _ = WORKLOADS[args.workload]
    o, epsl = mr_options(args.workload)
    opts = M.MROptions(epsilon=o["eps"], eps_level=epsl, min_leaf_level=o["min_leaf"],
                       local_time=o["local_time"], local_time_level_gap=o["gap"])
    slabs = mr_decomposed(args, world)
    solver = M.MRSolver(dim, level, opts, scheme=U.SchemeConfig(limiter=U.MINMOD), device=local,
                        comm=comm if slabs else None)
    stream = torch.cuda.Stream(device=local)
    solver.set_stream(stream)
    if dim == 2 and args.numerics == "tolerance":
        solver.set_numerics(True)
    init_host = U.case_fill(case, seed, level)
    init_pinned = torch.from_numpy(init_host).pin_memory()
    init_dev = init_pinned.to(f"cuda:{local}")
    out_pinned = torch.empty_like(init_pinned).pin_memory()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce(x, op):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=op)
        return float(t.item())

    # ---- device-resident throughput ------------------------------------------
    solver.build(init_dev)
    # W untimed warm-up cycles. The solver keeps one cycle graph per profiling
    # mode (the timed run records stage events, the e2e run does not), so the
    # warm-up instantiates both: W-1 cycles unprofiled, then one profiled.
    if args.warmup > 1:
        solver.run(args.warmup - 1, cfl=cfl)
    solver.profile(True)
    if args.warmup:
        solver.run(1, cfl=cfl)
    l0 = solver.kernel_launches()
    solver.profile(True)                        # resets the stage statistics
    sampler = ClockSampler(local)
    barrier()
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rep = solver.run(args.steps, cfl=cfl)
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    ms = reduce(e0.elapsed_time(e1), dist.ReduceOp.MAX if world > 1 else None)
    launches = solver.kernel_launches() - l0
    stage_ms, stage_launches, stage_updates = solver.stage_stats()
    solver.profile(False)
    # with slabs the cycle records are already global; replicas add up
    updates = rep.updates if slabs else reduce(float(rep.updates),
                                               dist.ReduceOp.SUM if world > 1 else None)
    value = updates / (ms / 1e3)

    # ---- end to end: pinned host input -> build -> K cycles -> to_uniform ----
    e2e = None
    if not args.no_e2e:
        # untimed warm-up of the host-buffer path (first-call allocations of
        # the staging buffers, the dense to_uniform prediction launches)
        solver.build(init_pinned.numpy())
        solver.run(1, cfl=cfl)
        solver._check(solver._lib.af_mr_to_uniform(
            solver._h, level, __import__("ctypes").c_void_p(out_pinned.data_ptr())))
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        solver.build(init_pinned.numpy())
        rep2 = solver.run(args.steps, cfl=cfl)
        solver._check(solver._lib.af_mr_to_uniform(
            solver._h, level, __import__("ctypes").c_void_p(out_pinned.data_ptr())))
        t1.record(stream)
        barrier()
        ems = reduce(t0.elapsed_time(t1), dist.ReduceOp.MAX if world > 1 else None)
        upd2 = rep2.updates if slabs else reduce(float(rep2.updates),
                                                 dist.ReduceOp.SUM if world > 1 else None)
        nbytes = init_host.nbytes
        e2e = {"value": upd2 / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(nbytes * world / args.steps),
               "d2h_bytes_per_step": int(nbytes * world / args.steps),
               "what": "one run_mr-equivalent call: build from the pinned host initial state, "
                       "K cycles, to_uniform(L) download to pinned host"}
    if rank != 0:
        return None

    hbm, src = peaks()
    S = (dim + 2) * 8
    # stage kernels: 2.5 S per leaf-cell stage, timed live by
    # CUDA events around each stage's launches on the solver stream
    achieved = 2.5 * S * stage_updates / (stage_ms / 1e3) / 1e9 if stage_ms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
            "peak_source": src, "kernel": "mr_stage_full2d + mr_stage_kernel" if dim == 2 else "mr_stage_kernel",
            "kernel_share_of_step": stage_ms / ms if ms > 0 else None,
            "stage_launches": stage_launches,
            "note": "per-launch average over the timed region; the MR cycle also runs "
                    "refine/coarsen/projection/prediction kernels and host decisions"}
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            from oracle import oracle as O
            kind = "reference" if O.available("ref") else "port"
            threads = host_threads(args.cpu_threads)
            rate, sample, _, ran = reference_cpu_rate(kind, args.workload, 8, 2, threads)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
                   "ran": ran}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                   "sample": f"unavailable: {e}"}
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if (slabs or world == 1) else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(workload_config(args.workload, world, args.numerics),
                       leaves_last_cycle=int(rep.cycles[-1, 0]) if len(rep.cycles) else None,
                       decomposition=(f"{world} slabs of rows along the last axis from level "
                                      f"{mr_partition_level(o, level, world)} up, halo "
                                      "exchange over NCCL" if slabs else
                                      ("single GPU (per-level dense grids)" if world == 1 else
                                       f"{world} independent replicas"))),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks,
    }


def amr_main(args):
    """AMR / AMRLT workloads. A step = one time-refined cycle of run_amr
    (2^max_levels finest steps: ghost syncs, remesh with the device
    clustering, patch stepping, average-down, refluxing). value = patch-cell
    updates / s over the cycle (cells of a level x its substeps). The run is
    host-driven (box lists come back at every remesh), so the timed region is
    wall clock between two device synchronisations. One GPU (N>1: replicas)."""
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    from paper_1603_05211_b200 import amr as A
    from paper_1603_05211_b200 import uniform as U
    kind, dim, base, level, dt, seed, cycles = AMR_WORKLOADS[args.workload]
    if args.level is not None:
        dt = dt * 2.0 ** (level - args.level)
        level = args.level
    steps_per_cycle = 1 << (level - base)
    cycles = args.steps if args.steps is not None else cycles
    scheme = U.SchemeConfig(1, U.MINMOD, 1)
    opts = A.AmrOptions(max_levels=level - base)

    def fresh():
        h = A.PatchHierarchy(dim, base, opts, scheme=scheme, device=local)
        h.initialize_case(kind, seed)
        return h

    if args.impl == "reference":
        if rank != 0:
            return
        from oracle import oracle as O
        lv = args.ref_level if args.ref_level is not None else level - 1
        n = (1 << (lv - base)) * max(1, cycles)
        r = O.ref_amr_run(dim, lv, base, n, dt * 2.0 ** (level - lv), case_kind=kind, seed=seed,
                          flux=1, integrator=1)
        upd = float(sum(r["cells_per_step"]))  # not exact per level; see sample
        # exact count: every level's cells x its substeps, from the final box lists
        rate = None
        if r["err_kind"] == 0:
            per = sum(len(l["data"]) * (1 << i) for i, l in enumerate(r["levels"]))
            rate = per * max(1, cycles) / r["wall_seconds"]
        line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": 0,
                "steps": cycles, "warmup": 0,
                "ms_per_step": 1e3 * r["wall_seconds"] / max(1, cycles),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": args.workload, "ran": {"finest_level": lv, "base_exp": base,
                                                              "finest_steps": n, "threads": 1}},
                "cpu_baseline": {"value": rate, "unit": UNIT, "cores": 1, "kind": "reference",
                                 "sample": f"the reference's PatchHierarchy/advance loop at finest level "
                                           f"{lv} (one below the workload's {level} unless --ref-level), {n} "
                                           "finest steps, one thread (the reference is serial); updates "
                                           "counted from the final box lists"},
                "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    h = fresh()
    for _ in range(max(args.warmup, 1)):
        h.run(steps_per_cycle, dt)
    h.profile(True)
    u0, l0, r0 = h.cell_updates(), h.kernel_launches(), h.remesh_stats()
    sampler = ClockSampler(local)
    torch.cuda.synchronize()
    sampler.start()
    t0 = time.perf_counter()
    rep = h.run(steps_per_cycle * cycles, dt)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    clocks = sampler.stop()
    upd = h.cell_updates() - u0
    launches = h.kernel_launches() - l0
    stage_ms, stage_launches, stage_updates = h.stage_stats()
    remesh_s = h.remesh_stats()[0] - r0[0]
    boxes = [h.level_info(l)[0] for l in range(h.n_levels())]
    cells = [h.level_info(l)[1] for l in range(h.n_levels())]
    h.close()

    # end to end: initial condition on the host -> hierarchy -> W+K cycles -> every patch back
    e2e = None
    if not args.no_e2e:
        t0 = time.perf_counter()
        g = fresh()
        u1 = g.cell_updates()
        g.run(steps_per_cycle * cycles, dt)
        out_bytes = 0
        for l in range(g.n_levels()):
            out_bytes += g.patch_data(l, 0).nbytes
        torch.cuda.synchronize()
        ew = time.perf_counter() - t0
        e2e = {"value": (g.cell_updates() - u1) / ew, "unit": UNIT,
               "h2d_bytes_per_step": int(sum(cells) * 40 / cycles),
               "d2h_bytes_per_step": int(out_bytes / cycles),
               "what": "create + initialize (initial condition evaluated on the host per patch cell, "
                       "uploaded) + K cycles + download of every patch interior"}
        g.close()
    if rank != 0:
        return
    hbm, src = peaks()
    S = (dim + 2) * 8
    # MUSCL-Hancock step: read u, write u' per patch cell (2 S), as hancock_step's row in DESIGN.md
    achieved = 2.0 * S * stage_updates / (stage_ms / 1e3) / 1e9 if stage_ms > 0 else None
    line = {
        "metric": METRIC, "value": upd * world / wall, "unit": UNIT, "n_gpus": world,
        "steps": cycles, "warmup": max(args.warmup, 1), "ms_per_step": 1e3 * wall / cycles,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.workload}: AMR patch path (SURVEY.md 8(f) #4), not a BASELINE.json config",
                   "method": "AMRLT", "dim": dim, "base_mesh": f"{1 << base}^{dim}",
                   "finest_mesh": f"{1 << level}^{dim}", "levels": level - base + 1,
                   "scheme": "AUSMDV/minmod/MUSCL-Hancock (the reference's AMR preset)",
                   "dt_finest": dt, "seed": seed, "bc": "outflow",
                   "step": f"one time-refined cycle = {steps_per_cycle} finest steps",
                   "patches_per_level": boxes, "cells_per_level": cells,
                   "timing": "wall clock between device synchronisations (host-driven recursion)",
                   "l2": "flushed by the cycle's own traffic (levels re-read between substeps)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": (achieved / hbm) if achieved else None, "traffic": None,
                     "peak_source": src,
                     "kernel": "amr_prims + amr_predict + amr_faces_hancock + amr_update (one update_level)",
                     "kernel_share_of_step": stage_ms / (1e3 * wall) if wall > 0 else None,
                     "stage_launches": stage_launches,
                     "note": "multi-pass global-memory kernels, latency and fp64 bound at these patch "
                             "counts; remesh (flags, device clustering, rebuild) took "
                             f"{remesh_s:.3f} s of the {wall:.3f} s"},
        "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
    }
    if not args.no_cpu_baseline and world == 1:
        try:
            from oracle import oracle as O
            lv = args.ref_level if args.ref_level is not None else level - 1
            n = 1 << (lv - base)
            r = O.ref_amr_run(dim, lv, base, n, dt * 2.0 ** (level - lv), case_kind=kind, seed=seed,
                              flux=1, integrator=1)
            per = sum(len(l["data"]) * (1 << i) for i, l in enumerate(r["levels"]))
            line["cpu_baseline"] = {
                "value": per / r["wall_seconds"], "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"the reference's PatchHierarchy/advance loop at finest level {lv} (one below "
                          f"the workload's {level}), one cycle of {n} finest steps, one thread (the "
                          "reference is serial); updates counted from the final box lists",
                "ran": {"finest_level": lv, "finest_steps": n, "wall_seconds": r["wall_seconds"]}}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
