#!/usr/bin/env python
"""Benchmark of the B200 two-stage s-step GMRES hot path (BASELINE.json metric).

Workload (BASELINE.json configs[2], the north-star config): 2D Laplace
5-point 8000×8000, row-partitioned by whole grid lines over the N ranks
(strong scaling: the grid is fixed, N = 1 holds all 64 M rows on one B200),
b = A·1, s-step GMRES(60), s = 5, two-stage BlkOrtho with ŝ = 60, fp64.
One timed *step* = one full restart cycle through the C ABI
(kry_sstep_gmres_device with max_iters = 60, warm-started from the current
x): 12 MPK blocks (60 stencil SpMVs), 12 first-stage BCGS-PIP, 1
second-stage BCGS-PIP finalize of the 61-column big panel,
Hessenberg/LSQ, solution update and explicit residual.  Inputs live in HBM
(the 31 GB basis is ≫ the 126 MB L2, so no L2 flush is needed between
steps).  --scaling weak keeps grid² rows per GPU instead (grid × grid·N).

`value` = aggregate BlkOrtho HBM GB/s: Σ_ranks algorithmic BlkOrtho bytes
(8·n·(2c0+3w) per BCGS-PIP) ÷ BlkOrtho device time (CUDA events
on the solver stream around Gram + allreduce + Cholesky + update, max over
ranks).  `e2e` = the same bytes ÷ the end-to-end wall time of the same cycles
through the host-buffer C ABI (kry_sstep_gmres: b and x0 copied H2D from
pinned memory, x copied D2H, every step).

  python bench.py                      # N=1, 3 warm-up + 30 timed cycles at 8000²
  python bench.py --impl reference     # the CPU reference's BlkOrtho on the same config
  torchrun --nproc-per-node N bench.py --gpus N
  python bench.py --workload random    # configs[4]: n = 20 M, 30 nnz/row, device Jacobi
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# Keep stdout to the one JSON line (NCCL prints its version banner otherwise).
os.environ.setdefault("NCCL_DEBUG", "WARN")

METRIC = "GMRES time-to-solution (s) & BlkOrtho HBM GB/s, 2D Laplace, 1/2/4/8 B200"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--grid", type=int, default=8000,
                   help="grid side (strong: of the whole grid; weak: per GPU, grid × grid·N)")
    p.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                   help="strong (default, BASELINE configs[2]): the grid is split over the ranks")
    p.add_argument("--dims", type=int, choices=[2, 3], default=2, help="2D 5-point or 3D 7-point Laplacian")
    p.add_argument("--workload", choices=["laplace", "random"], default="laplace",
                   help="random = BASELINE configs[4] (kry_gen_random_sparse, 30 nnz/row, device Jacobi)")
    p.add_argument("--random-rows", type=int, default=20_000_000,
                   help="rows of the random workload (strong: total; weak: per GPU)")
    p.add_argument("--random-nnz", type=int, default=30)
    p.add_argument("--diag-factor", type=float, default=0.15)
    p.add_argument("--shat", type=int, default=60)
    p.add_argument("--scheme", choices=["two-stage", "bcgs-pip2", "standard"], default="two-stage",
                   help="standard = standard_gmres (gmres.hpp:404: s = 1, CGS2), the paper's GMRES column")
    p.add_argument("--no-tts", action="store_true",
                   help="skip the full solves from x0 = 0 at the bench grid (two-stage and one-stage PIP2)")
    p.add_argument("--no-tts512", action="store_true", help="skip the 512² time-to-solution solves")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-sample-blocks", type=int, default=3)
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy test)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------
def cpu_slab(grid, dims):
    """The bounded CPU sample of the bench grid: a slab of whole grid lines
    (2-D: grid × lines, 3-D: grid × grid × planes) holding about 4 M rows.
    First-stage BCGS-PIP is row-separable (every Gram entry is a sum over
    rows, the update is row-local), so the reference's BlkOrtho GB/s on the
    slab is its rate on the whole grid at 1/k of the time."""
    plane = grid if dims == 2 else grid * grid
    lines = max(8, min(grid, (4 << 20) // plane))
    return lines, lines * plane


def reference_blkortho_sample(grid, dims, shat, blocks, threads, first_block=0, store=None):
    """Time the CPU reference's BlkOrtho (BasisStore::preprocess_block,
    basis_store.hpp:122-125 → bcgs_pip block_ortho.hpp:180) on blocks
    [first_block, first_block + blocks) of a restart cycle of the bench
    configuration, on the cpu_slab rows (the reference's own operator and
    MPK feed it).  Returns (GB/s, seconds, bytes, description, store)."""
    os.environ["KRYLOV_NUM_THREADS"] = str(threads)
    import numpy as np
    from oracle import ref

    lines, n = cpu_slab(grid, dims)
    m, s = 60, 5
    if store is None:
        a = ref.laplace2d(grid, lines) if dims == 2 else ref.laplace3d(grid, grid, lines)
        b = ref.spmv(a, np.ones(n))
        store = {"a": a, "v1": b / np.linalg.norm(b), "st": ref.Store(n, m, s, shat)}
    a, v1, st = store["a"], store["v1"], store["st"]
    secs, byts = 0.0, 0.0
    for k in range(first_block, first_block + blocks):
        info = st.info()
        if info.filled + s > m + 1:  # a new restart cycle
            st.reset()
            info = st.info()
        start = v1 if info.filled == 0 else st.column(info.filled - 1)
        blk = ref.mpk(a, start, s)
        c0 = 0 if info.filled == 0 else info.filled - 1
        t = time.perf_counter()
        st.preprocess_block(blk, info.filled != 0)
        secs += time.perf_counter() - t
        byts += 8.0 * n * (2 * c0 + 3 * (s + 1))
    shape = f"{grid}x{lines}" if dims == 2 else f"{grid}x{grid}x{lines}"
    desc = (f"CPU reference BasisStore::preprocess_block (first-stage BCGS-PIP, c0 cycling 0..55 as in a restart "
            f"cycle), {blocks} blocks on a {shape} slab of whole grid lines (n={n}) of the bench grid, "
            f"KRYLOV_NUM_THREADS={threads}")
    return byts / secs / 1e9, secs, byts, desc, store


def run_reference(args):
    """The reference arm: the unmodified CPU reference (oracle/_ref, built from
    /root/reference) on this box's host cores, same metric and unit (BlkOrtho
    GB/s).  One step = one first-stage BCGS-PIP block on the cpu_slab sample
    of the bench grid (a full 8000² cycle takes minutes on the CPU, SURVEY
    §6).  KRYLOV_NUM_THREADS: both 1 and all host threads are probed and the
    faster is timed (the reference's SpMV gets slower with threads, SURVEY
    A.5); both probes are recorded."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    K, W = args.steps, args.warmup
    g, dims = args.grid, args.dims
    nproc = os.cpu_count() or 1
    probes = {}
    for th in sorted({1, nproc}):
        gbs, secs, _, _, _ = reference_blkortho_sample(g, dims, args.shat, 3, th)
        probes[th] = gbs
    threads = max(probes, key=probes.get)
    store = None
    times, byts = [], []
    for k in range(W + K):
        gbs, secs, b, desc, store = reference_blkortho_sample(g, dims, args.shat, 1, threads, k, store)
        if k >= W:
            times.append(secs)
            byts.append(b)
    total = sum(times)
    value = sum(byts) / total / 1e9
    lines, n = cpu_slab(g, dims)
    shape = f"{g}x{g}" if dims == 2 else f"{g}x{g}x{g}"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * total / K, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{'2D Laplace 5-pt' if dims == 2 else '3D Laplace 7-pt'} {shape}, s-step GMRES(60) "
                               f"s=5, two-stage BlkOrtho shat={args.shat}",
                   "grid": [g, g] if dims == 2 else [g, g, g], "sample_rows": n,
                   "step": "one first-stage BCGS-PIP (BasisStore::preprocess_block) on a slab of whole grid lines "
                           "of the bench grid (BlkOrtho is row-separable; the GB/s rate is the metric)"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "reference",
                         "sample": f"{K} first-stage BCGS-PIP blocks (c0 cycling as in a restart cycle) on "
                                   f"{n} rows of the {shape} grid after {W} warm-up blocks",
                         "threads_probed_gbs": {str(k): v for k, v in probes.items()}},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    import paper_2402_15033_b200 as kb

    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        idb = torch.zeros(kb.lib().kry_nccl_unique_id_size(), dtype=torch.uint8, device="cuda")
        if rank == 0:
            idb.copy_(torch.frombuffer(bytearray(kb.Context.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idb, 0)
        nccl_id = bytes(idb.cpu().tolist())
    ctx = kb.Context(local, world, rank, nccl_id)
    ctx.set_timing(True)
    stream = torch.cuda.ExternalStream(ctx.stream_handle())

    g = args.grid
    strong = args.scaling == "strong"
    if args.workload == "random":
        # configs[4]: rows of the generator (kry_gen_random_sparse, SplitMix64
        # seed 1), b = A·1 of the unscaled matrix, then device Jacobi.
        n_glob = args.random_rows if strong else args.random_rows * world
        rb, re = rank * n_glob // world, (rank + 1) * n_glob // world
        op = kb.CsrOperator(*kb.gen_random_sparse(n_glob, rb, re - rb, args.random_nnz, seed=1,
                                                  diag_factor=args.diag_factor),
                            n_global=n_glob, row_begin=rb, ctx=ctx)
        nx, ny, nz = n_glob, 1, 1
        shape = (f"random sparse n={n_glob} ({args.random_nnz} nnz/row, SplitMix64 seed 1, "
                 f"diag 1+{args.diag_factor}*sum|off|, device Jacobi)")
    elif args.dims == 2:
        nx, ny, nz = (g, g, 1) if strong else (g, g * world, 1)
        op = kb.Laplace2D(nx, ny, ctx)
        shape = f"2D Laplace 5-pt {nx}x{ny}"
    else:
        nx, ny, nz = (g, g, g) if strong else (g, g, g * world)
        op = kb.Laplace3D(nx, ny, nz, ctx)
        shape = f"3D Laplace 7-pt {nx}x{ny}x{nz}"
    n = op.n
    kind = kb.OrthoKind.TWO_STAGE if args.scheme == "two-stage" else kb.OrthoKind.BCGS_PIP2
    std = args.scheme == "standard"
    solve_dev = kb.standard_gmres_device if std else kb.sstep_gmres_device
    solve_host = kb.lib().kry_standard_gmres if std else kb.lib().kry_sstep_gmres
    cfg_cycle = kb.SolverConfig(scheme=kb.OrthoScheme(kind, args.shat), big_step=args.shat if kind == 3 else 0,
                                max_iters=60)
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    kb.lib().kry_spmv_device(ctx.handle, op.handle, ones.data_ptr(), b.data_ptr())  # b = A·1 (gen_rhs_ones)
    if args.workload == "random":
        op.jacobi()  # from here the operator is D⁻¹A; the solver forms D⁻¹b on the device

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def cycle():
        return solve_dev(op, b.data_ptr(), x.data_ptr(), cfg_cycle, x.data_ptr())

    for _ in range(args.warmup):
        cycle()
    barrier()
    tel = {k: 0.0 for k in ("ortho_seconds", "ortho_bytes", "gram_kernel_seconds", "gram_bytes", "gram_launches",
                            "update_kernel_seconds", "update_bytes", "update_launches", "mpk_seconds", "mpk_bytes",
                            "restart_seconds", "gpu_launches")}
    iters, reduces = 0, 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            rep = cycle()
            for k in tel:
                tel[k] += rep.telemetry[k]
            iters += rep.iterations
            reduces += rep.sync.reduces
        ev1.record(stream)
        ev1.synchronize()
    barrier()
    elapsed = ev0.elapsed_time(ev1) * 1e-3

    # max over ranks of the times, sum over ranks of the bytes
    def allred(vals, op_):
        t = torch.tensor(vals, dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=op_)
        return t.cpu().tolist()

    MAX = dist.ReduceOp.MAX if world > 1 else None
    SUM = dist.ReduceOp.SUM if world > 1 else None
    t_el, t_ortho, t_gram, t_upd, t_mpk, t_rst = allred(
        [elapsed, tel["ortho_seconds"], tel["gram_kernel_seconds"], tel["update_kernel_seconds"],
         tel["mpk_seconds"], tel["restart_seconds"]], MAX)
    b_ortho, b_gram, b_upd, b_mpk = allred([tel["ortho_bytes"], tel["gram_bytes"], tel["update_bytes"],
                                            tel["mpk_bytes"]], SUM)
    value = b_ortho / t_ortho / 1e9

    # e2e: the host-buffer C ABI, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        hb = torch.empty(n, dtype=torch.float64, pin_memory=True)
        hb.copy_(b)
        hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
        hx.copy_(x)
        import ctypes as C
        P = lambda t: C.cast(C.c_void_p(t.data_ptr()), kb._capi.P_dbl)
        ccfg = cfg_cycle.to_c()
        def host_cycle():
            rep_c, cyc, pb, pbp = kb._new_report(1024)
            kb._check(solve_host(ctx.handle, op.handle, P(hb), P(hx), C.byref(ccfg), C.byref(rep_c), P(hx)))
            return rep_c.ortho_bytes

        for _ in range(args.warmup):  # the first host-buffer call sizes the upload buffers
            host_cycle()
        e_bytes = 0.0
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e_bytes += host_cycle()
        barrier()
        t_e2e = allred([time.perf_counter() - t0], MAX)[0]
        e_bytes = allred([e_bytes], SUM)[0]
        e2e = {"value": e_bytes / t_e2e / 1e9, "unit": "GB/s", "ms_per_step": 1e3 * t_e2e / args.steps,
               "ortho_bytes_per_step": e_bytes / args.steps / world, "h2d_bytes_per_step": 2 * 8 * n,
               "d2h_bytes_per_step": 8 * n,
               "definition": "BlkOrtho algorithmic bytes / end-to-end wall time of whole restart cycles via "
                             "kry_sstep_gmres with host (pinned) b, x0 in and x out per step"}

    # roofline: the dominant BlkOrtho kernel, per-launch average of this rank
    peak, peak_src = peaks()
    dom = "gram_kernel" if t_gram >= t_upd else "update_kernel"
    if dom == "gram_kernel":
        per_launch_b = tel["gram_bytes"] / max(tel["gram_launches"], 1)
        per_launch_t = tel["gram_kernel_seconds"] / max(tel["gram_launches"], 1)
    else:
        per_launch_b = tel["update_bytes"] / max(tel["update_launches"], 1)
        per_launch_t = tel["update_kernel_seconds"] / max(tel["update_launches"], 1)
    achieved = per_launch_b / per_launch_t / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            traffic = tj.get(f"{dom}@{shape}/{world}")
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "laplace":
        gbs, secs, byts, desc, _ = reference_blkortho_sample(g, args.dims, args.shat, args.cpu_sample_blocks, 1)
        cpu = {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "reference",
               "sample": desc + f"; {secs:.1f} s of CPU BlkOrtho ({byts / 1e9:.1f} GB algorithmic)"}

    # Time to solution at BASELINE config 1 (2D Laplace 512², tol 1e-6): full
    # solves from x0 = 0, one-stage BCGS-PIP2 (the CPU reference's config) and
    # two-stage ŝ = 60; inputs resident in HBM, wall clock around the call.
    tts512 = None
    ctx.set_timing(False)  # the time-to-solution runs need no phase events
    if world == 1 and not args.no_tts512:
        op5 = kb.Laplace2D(512, 512, ctx)
        one5 = torch.ones(op5.n, dtype=torch.float64, device="cuda")
        b5 = torch.empty_like(one5)
        x5 = torch.zeros_like(one5)
        torch.cuda.synchronize()
        kb.lib().kry_spmv_device(ctx.handle, op5.handle, one5.data_ptr(), b5.data_ptr())
        tts512 = {"grid": [512, 512], "rel_tol": 1e-6,
                  "cpu_reference_seconds_survey": {"bcgs_pip2_1thread": 329.5, "two_stage_8threads": 239.4,
                                                   "source": "BASELINE.md §2 (survey container, 8-core Xeon)"},
                  "cpu_reference_seconds_gpu_box": {"two_stage_1thread": 202.3, "two_stage_16threads": 157.7,
                                                    "bcgs_pip2_1thread": 198.1, "bcgs_pip2_16threads": 203.8,
                                                    "source": "profiles/cpu_ref_tts_512.jsonl (tools/cpu_ref_tts.py "
                                                              "on a B200 box host, 16 cores, round 1)"}}
        for label, knd, sh in [("bcgs_pip2", kb.OrthoKind.BCGS_PIP2, 0), ("two_stage_shat60", kb.OrthoKind.TWO_STAGE, 60)]:
            cfgf = kb.SolverConfig(scheme=kb.OrthoScheme(knd, sh), big_step=sh)
            kb.sstep_gmres_device(op5, b5.data_ptr(), None, cfgf, x5.data_ptr())  # warm (module load, workspace)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = kb.sstep_gmres_device(op5, b5.data_ptr(), None, cfgf, x5.data_ptr())
            torch.cuda.synchronize()
            tts512[label] = {"seconds": time.perf_counter() - t0, "status": rep.status.name.lower(),
                             "iterations": rep.iterations, "restarts": rep.restarts, "reduces": rep.sync.reduces,
                             "final_relative_residual": rep.final_relative_residual}
        del op5

    # Time to solution at the bench grid (BASELINE metric "GMRES time-to-
    # solution"): full solves from x0 = 0 to the reference's stopping rules,
    # two-stage (the configured ŝ) and one-stage BCGS-PIP2, wall clock
    # around the call with the inputs resident (max over ranks).
    tts = None
    if not args.no_tts and args.scheme != "standard":
        tts = {}
        for label, knd, sh in [(f"two_stage_shat{args.shat}", kb.OrthoKind.TWO_STAGE, args.shat),
                               ("bcgs_pip2", kb.OrthoKind.BCGS_PIP2, 0)]:
            x.zero_()
            cfg_full = kb.SolverConfig(scheme=kb.OrthoScheme(knd, sh), big_step=sh)
            barrier()
            t0 = time.perf_counter()
            rep = solve_dev(op, b.data_ptr(), None, cfg_full, x.data_ptr())
            barrier()
            t_tts = allred([time.perf_counter() - t0], MAX)[0]
            tts[label] = {"seconds": t_tts, "status": rep.status.name.lower(), "iterations": rep.iterations,
                          "restarts": rep.restarts, "final_relative_residual": rep.final_relative_residual,
                          "reduces": rep.sync.reduces}
        two = tts[f"two_stage_shat{args.shat}"]["seconds"]
        tts["speedup_two_stage_over_one_stage"] = tts["bcgs_pip2"]["seconds"] / two

    if rank == 0:
        steps = args.steps
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_el / steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (b = A*1, x0 = 0, then warm restarts)",
            "config": {"workload": f"{shape} ({n} rows per GPU), " + (
                           "standard GMRES(60) (s = 1, CGS2 as BCGS2-CholQR2)" if std else
                           f"s-step GMRES(60) s=5, {args.scheme} BlkOrtho shat={args.shat}"),
                       "grid": [nx, ny] if args.dims == 2 else [nx, ny, nz], "rows_per_gpu": n, "m": 60, "s": 5,
                       "shat": args.shat,
                       "step": "one full restart cycle (60 iterations) through kry_" +
                               ("standard" if std else "sstep") + "_gmres_device",
                       "parallelism": f"row-partitioned dp{world}", "l2": "inputs larger than L2 (basis 8*61*n B)"},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": per_launch_b, "avg_launch_ms": per_launch_t * 1e3},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(tel["gpu_launches"]),
            "clocks": clk.summary(),
            "phases_ms_per_step": {"mpk": 1e3 * t_mpk / steps, "blkortho": 1e3 * t_ortho / steps,
                                   "gram_kernels": 1e3 * t_gram / steps, "update_kernels": 1e3 * t_upd / steps,
                                   "restart": 1e3 * t_rst / steps},
            "phase_gbs": {"gram": b_gram / t_gram / 1e9, "update": b_upd / t_upd / 1e9,
                          "mpk": b_mpk / max(t_mpk, 1e-12) / 1e9},
            "iterations_per_step": iters / steps, "reduces_per_step": reduces / steps,
        }
        if tts512 is not None:
            line["time_to_solution_512"] = tts512
        if tts is not None:
            line["time_to_solution"] = tts
        print(json.dumps(line), flush=True)
    del op
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
