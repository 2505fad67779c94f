#!/usr/bin/env python
"""Benchmark: Mpixel-iterations/s of preconditioned AR-BC Landweber on B200.

Workload (default): BASELINE config C3 — a batch of 64 FP64 1024x1024 images
(seed per image), 31x31 Gaussian mask sigma=(4,4.5) offset (+1,0), 1% noise,
40 preconditioned (D-)Landweber iterations under anti-reflective BCs.  One
"step" is one complete 40-iteration restoration of the rank's 64-image batch
(histories, best-iterate tracking and all per-iteration norms included).
Multi-GPU: the fixed 64-image batch is sharded over the ranks
(64/N contiguous images per GPU, 8 at N = 8; strong scaling, no data-path
collective); --weak gives every rank its own 64 images instead.

  value  : device-resident inputs, CUDA events on the plan's stream, max over ranks
  e2e    : same solve through the public C-ABI with pinned HOST buffers, i.e.
           H2D of g and f_true + D2H of the restored images inside the timed region
  roofline: the dominant kernel (per-launch CUDA events of one extra eager
           step), with every kernel of the iteration listed in roofline.kernels
  cpu_baseline: the CPU oracle port (oracle/), rank 0 at N=1, bounded sample

`--impl reference` times the reference algorithm's CPU restatement (the oracle
port; the reference itself cannot be built: Eigen3/FFTW3 are absent) with all
host threads on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpixel-iterations/s of preconditioned AR-BC iteration"
UNIT = "Mpixel-iterations/s"
PEAKS_FILE = os.path.join(ROOT, "profiles", "r01_fp64_peak.json")
HBM_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
E2E_CHUNKS = int(os.environ.get("DBX_E2E_CHUNKS", "4"))  # with 2 in flight: measured best (r1s2bb, r1s2cc)


def e2e_split(B):
    """Chunk sizes of the e2e host run: DBX_E2E_SPLIT="a,b,..." (summing to
    the batch), else E2E_CHUNKS equal chunks."""
    sp = os.environ.get("DBX_E2E_SPLIT")
    if sp:
        sizes = [int(v) for v in sp.split(",") if v.strip()]
        if sum(sizes) == B and all(v > 0 for v in sizes):
            return sizes
    if B % 8 == 0 and "DBX_E2E_CHUNKS" not in os.environ:
        # short first / last chunks: less exposed upload before the first solve
        # and download after the last (measured: 8,24,24,8 -> e2e 20006 / 20085
        # vs 4 x 16 -> 19601 / 19505, r1s3 A/B)
        return [B // 8, 3 * B // 8, 3 * B // 8, B // 8]
    nch = E2E_CHUNKS if B % E2E_CHUNKS == 0 else 1
    return [B // nch] * nch


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--images", type=int, default=0, help="override images per rank")
    ap.add_argument("--weak", action="store_true",
                    help="every rank restores its own full batch (default: the batch is sharded over the ranks)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the single-GPU graph-path lines of the other BASELINE configs (C1, C2, C4, C5)")
    ap.add_argument("--slab", action="store_true",
                    help="row-slab decomposition of one image (default for C5 at N > 1)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


def cpu_sample(cfg, threads: int, iters: int):
    """Oracle (CPU restatement of the reference) on `threads` concurrent images,
    each `iters` D-Landweber iterations; returns (Mpx-it/s, seconds, sample str)."""
    from oracle import oracle as O
    from paper_1211_0393_b200 import configs as cf
    O.build()
    probs = [cf.make_problem(cfg, image=i) for i in range(threads)]
    taps = probs[0][2]
    d = O.build_tikhonov(taps, cfg.alpha, cfg.n, cfg.n)
    errs = []

    def work(i):
        try:
            f, g, _ = probs[i]
            O.landweber(taps, g, d=d, f_true=f, max_iters=iters)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    t0 = time.perf_counter()
    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    if errs:
        raise errs[0]
    px_it = threads * cfg.n * cfg.n * iters
    sample = (f"{threads} image(s) x {iters} D-Landweber iteration(s) of {cfg.name} ({cfg.n}^2, q={cfg.q}), "
              f"oracle port: reference algorithm (FFT correlation for q>7, FFT DST-I), {threads} thread(s)")
    return px_it / dt / 1e6, dt, sample


def cpu_per_config(cf):
    """1-core CPU oracle line for every BASELINE config, each
    a bounded sample of that config's D-Landweber run (iterations timed
    linearly extrapolate: the loop does the same work every iteration).  C5
    (8192^2) uses every host core (line-parallel oracle passes, results
    bit-identical to one thread) so that the sample stays within seconds."""
    from oracle import oracle as O
    O.build()
    out = {"unit": UNIT, "kind": "port", "note": "oracle port of the reference algorithm (FFT correlation for q>7, "
                                                 "FFT DST-I); the reference's FFTW is unavailable"}
    plan = {"C1": (10, 1), "C2": (5, 1), "C3": (2, 1), "C4": (1, 1), "C5": (1, os.cpu_count() or 1)}
    for name, (iters, threads) in plan.items():
        c = cf.CONFIGS[name]
        f, g, taps = cf.make_problem(c)
        d = O.build_tikhonov(taps, c.alpha, c.n, c.n)
        O.set_threads(threads)
        try:
            t0 = time.perf_counter()
            O.landweber(taps, g, d=d, f_true=f, max_iters=iters)
            dt = time.perf_counter() - t0
        finally:
            O.set_threads(1)
        out[name] = {"value": c.n * c.n * iters / dt / 1e6, "cores": threads,
                     "sample": f"1 image x {iters} D-Landweber iteration(s) of {c.n}^2, q={c.q}", "seconds": round(dt, 2)}
        del f, g, d
    return out


def other_configs(L, dbx, cf, torch, dev, local, reps=3):
    """Single-GPU graph-path throughput of the other BASELINE configs (the
    parity cases), same timing rules as the headline (warm-up, CUDA events on
    the plan's stream, device-resident inputs).  C2 also times plain Landweber
    (configs[1] names both); C1/C2 are single small images (L2-resident,
    launch/latency bound), C4/C5 single large images (separate-pass pipeline)."""
    out = {}
    for name in ("C1", "C2", "C4", "C5"):
        cfg = cf.CONFIGS[name]
        n, q, H = cfg.n, cfg.q, cfg.iters
        # inputs synthesised on the GPU straight into device buffers (§8f f4)
        g = torch.empty((1, n, n), dtype=torch.float64, device=dev)
        f = torch.empty_like(g)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, taps = cf.make_problem_device(cfg, device=local, out=(f, g))
        torch.cuda.synchronize()
        gen_s = time.perf_counter() - t0
        o = torch.empty_like(g)
        plan = C.c_void_p()
        dbx._check(L.dbx_plan_create(n, n, 1, dbx._ptr(taps), q, q, 3, local, C.byref(plan)))
        dbx._check(L.dbx_precond_build(plan, float(cfg.alpha)))
        stream = torch.cuda.ExternalStream(L.dbx_plan_stream(plan), device=dev)
        rre = np.zeros(H)
        res = np.zeros(H)
        best, done = (C.c_int * 1)(), (C.c_int * 1)()
        entry = {"n": n, "q": q, "iters": H, "alpha": cfg.alpha, "generation_s": round(gen_s, 3),
                 "generator": "device (dbx_gen_honest_device)"}
        fz = C.c_int()
        for prec in ((1, 0) if cfg.plain_too else (1,)):
            def solve():
                dbx._check(L.dbx_landweber_run(plan, dbx._ptr(g), dbx._ptr(f), 1.0, H, 1, 0, 0.0, prec,
                                               dbx._ptr(o), dbx._ptr(rre), dbx._ptr(res), best, done, None))
            for _ in range(3):
                solve()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
            for _ in range(reps):
                solve()
            with torch.cuda.stream(stream):
                e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            key = "value" if prec else "plain_value"
            entry[key] = n * n * H / (ms * 1e-3) / 1e6
            entry[("ms_per_run" if prec else "plain_ms_per_run")] = ms
            if prec:
                L.dbx_plan_pipeline(plan, C.byref(fz))
                entry["pipeline"] = {0: "separate passes", 1: "fused", 2: "fused separable"}.get(fz.value, "?")
        L.dbx_plan_destroy(plan)
        out[name] = entry
        del g, f, o
    return out


def images_per_rank(cfg, args, world):
    if args.images:
        return args.images
    if args.weak or cfg.batch % world:
        return cfg.batch
    return cfg.batch // world


def workload_config(cfg, B, world, weak):
    """The `config` object of both arms' JSON lines (identical by construction)."""
    return {"workload": f"{cfg.name}: {B * world if not weak else cfg.batch} x {cfg.n}x{cfg.n} FP64 images"
                        f"{' per GPU' if weak else ''}, q={cfg.q} mask, {cfg.iters} D-Landweber iterations, AR BCs, "
                        f"alpha={cfg.alpha}",
            "images_per_gpu": B, "global_images": B * world, "n": cfg.n, "q": cfg.q, "iters": cfg.iters,
            "parallelism": f"batch-sharded x{world} (no data-path collective)",
            "l2": f"inputs larger than L2 (each {B}x{cfg.n}^2 FP64 array = {B * cfg.n * cfg.n * 8 >> 20} MiB)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_1211_0393_b200 import configs as cf
    O.build()
    # inputs through the oracle's own build of the generators: this CPU arm
    # never maps the product library libdbx.so
    cf.use_generator_library(O.gen_lib_path())
    cfg = cf.CONFIGS[args.config]
    B = images_per_rank(cfg, args, world)
    threads = os.cpu_count() or 1
    vals = []
    for s in range(args.warmup + args.steps):
        v, dt, sample = cpu_sample(cfg, threads, 1)
        if s >= args.warmup:
            vals.append((v, dt))
    v = float(np.median([x[0] for x in vals]))
    ms = float(np.median([x[1] for x in vals])) * 1e3
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, host-generated)",
            "config": workload_config(cfg, B, world, args.weak),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference (Eigen3/FFTW3 header library) is unbuildable here; timed its CPU restatement "
                    "oracle/deblur_oracle.cpp (own Stockham/Bluestein FFT in place of FFTW), one image per host "
                    "thread, each step a bounded sample (1 iteration per image) of the same workload"}
    print(json.dumps(line), flush=True)
    return 0


def run_slab(args):
    """One image split into row slabs across the ranks (C5),
    through the C++ slab loop (dbx_slab_run): NCCL halo send/recv for the blur,
    all-to-all from grouped send/recv for the column blocks of D, device-side
    all-reduce of the norms and device bookkeeping; strong scaling (the image
    is fixed)."""
    import torch
    import torch.distributed as dist

    from paper_1211_0393_b200 import configs as cf
    from paper_1211_0393_b200.slab import NcclComm, SlabRun
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = cf.CONFIGS[args.config]
    n, q, H = cfg.n, cfg.q, cfg.iters
    F, G, taps = cf.make_batch(cfg, 1)
    R = n // world
    dev = torch.device("cuda", local)
    gh = torch.from_numpy(np.ascontiguousarray(G[0, rank * R:(rank + 1) * R])).pin_memory()
    fh = torch.from_numpy(np.ascontiguousarray(F[0, rank * R:(rank + 1) * R])).pin_memory()
    del F, G
    g, f = gh.to(dev), fh.to(dev)
    comm = NcclComm(local) if world > 1 else None
    solver = SlabRun(n, world, taps, q, cfg.alpha, rank=rank if world > 1 else -1, comm=comm, device=local)
    out = torch.empty_like(g)
    for _ in range(args.warmup):
        solver.run(g, f, H, out=out)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.ExternalStream(solver.stream())
    clocks = Clocks(local)
    clocks.start()
    l0 = solver.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        solver.run(g, f, H, out=out)
    t1.record(stream)
    torch.cuda.synchronize()
    launches = (solver.launch_count() - l0) // max(args.steps, 1)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    # e2e: the same call with the rank's slab uploaded from pinned host memory
    # and the restored slab read back inside the timed region
    oh = torch.empty_like(gh).pin_memory()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        g.copy_(gh, non_blocking=True)
        f.copy_(fh, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        solver.run(g, f, H, out=out)
        oh.copy_(out, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([t0.elapsed_time(t1), e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max, t_e2e = float(t[0].item()), float(t[1].item())
    px_it = n * n * H * args.steps
    value = px_it / (t_max * 1e-3) / 1e6
    separable = solver.separable
    solver.close()
    if comm is not None:
        comm.close()
    if rank == 0:
        hbm = float(json.load(open(HBM_FILE))["hbm_gbs"]) if os.path.exists(HBM_FILE) else 7700.0
        gbs = 72.0 * px_it / (t_max * 1e-3) / 1e9 / world
        slab_bytes = R * n * 8
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded scene/mask/noise, host-generated)",
                "config": {"workload": f"{cfg.name}: one {n}x{n} FP64 image in {world} row slabs of {R} rows, "
                                       f"q={q}, {H} D-Landweber iterations",
                           "parallelism": f"row slabs x{world} (C++ loop: NCCL halo send/recv, all-to-all from "
                                          "grouped send/recv, device all-reduce)",
                           "blur": "separable direct on halo-extended slabs" if separable else "FFT slab blur",
                           "l2": "slab arrays exceed L2"},
                "clocks": clk, "gpu_launches": int(launches),
                "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                             "traffic": None, "note": "SURVEY canonical 72 B per pixel-iteration, per GPU"},
                "e2e": {"value": px_it / (t_e2e * 1e-3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": 2 * slab_bytes,
                        "d2h_bytes_per_step": slab_bytes,
                        "path": "SlabRun.run (dbx_slab_run) with the slab uploaded from pinned host memory"},
                "cpu_baseline": None}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.slab or (args.config == "C5" and dist_env()[1] > 1):
        return run_slab(args)
    import torch
    import torch.distributed as dist

    import paper_1211_0393_b200 as dbx
    from paper_1211_0393_b200 import configs as cf

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    L = dbx.lib()
    cfg = cf.CONFIGS[args.config]
    B = images_per_rank(cfg, args, world)
    n, q = cfg.n, cfg.q
    N = n * n

    # ---- synthetic inputs (host, seeded per image; not timed) ----
    F, G, taps = cf.make_batch(cfg, B, first=rank * B)
    dev = torch.device("cuda", local)
    g_d = torch.from_numpy(G).to(dev)
    f_d = torch.from_numpy(F).to(dev)
    out_d = torch.empty_like(g_d)
    del F, G

    plan = C.c_void_p()
    dbx._check(L.dbx_plan_create(n, n, B, dbx._ptr(taps), q, q, 3, local, C.byref(plan)))
    dbx._check(L.dbx_precond_build(plan, float(cfg.alpha)))
    stream = torch.cuda.ExternalStream(L.dbx_plan_stream(plan), device=dev)
    H = cfg.iters
    rre_h = np.zeros((B, H))
    res_h = np.zeros((B, H))
    best = (C.c_int * B)()
    done = (C.c_int * B)()

    def solve(g, f, out):
        dbx._check(L.dbx_landweber_run(plan, dbx._ptr(g), dbx._ptr(f), 1.0, H, 1, 0, 0.0, 1, dbx._ptr(out),
                                       dbx._ptr(rre_h), dbx._ptr(res_h), best, done, None))

    for _ in range(args.warmup):
        solve(g_d, f_d, out_d)
    torch.cuda.synchronize()

    # ---- timed region: device-resident inputs, the production path (one CUDA
    # graph per run, replayed) ----
    clocks = Clocks(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = L.dbx_plan_launch_count(plan)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for s in range(args.steps):
        with torch.cuda.stream(stream):
            ev[s][0].record(stream)
        solve(g_d, f_d, out_d)
        with torch.cuda.stream(stream):
            ev[s][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = int(L.dbx_plan_launch_count(plan) - launches0)
    # ---- per-class kernel times: one more (untimed for the headline) step with
    # eager launches bracketed by CUDA events on the plan stream ----
    L.dbx_plan_set_timing(plan, 1)
    solve(g_d, f_d, out_d)
    torch.cuda.synchronize()
    ms = (C.c_double * 8)()
    cnt = (C.c_int * 8)()
    L.dbx_plan_kernel_times(plan, ms, cnt, 8)
    kms_tot = np.array(ms[:4]) * args.steps
    kcnt_tot = np.array(cnt[:4]) * args.steps
    kprof = {}
    nm = C.create_string_buffer(128)
    kms1, kc1 = C.c_double(), C.c_int()
    for i in range(L.dbx_plan_kernel_profile(plan, -1, None, 0, None, None)):
        L.dbx_plan_kernel_profile(plan, i, nm, 128, C.byref(kms1), C.byref(kc1))
        kprof[nm.value.decode()] = (kms1.value, kc1.value)
    L.dbx_plan_set_timing(plan, 0)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_ms = float(np.sum(step_ms))
    t_local = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    t_max = float(t_local.item())
    px_it = world * B * N * H * args.steps
    value = px_it / (t_max * 1e-3) / 1e6

    # ---- e2e: public C-ABI with pinned host buffers (H2D + D2H inside the
    # timed region).  dbx_landweber_run_chunks splits the batch over E2E_CHUNKS
    # plans so that every chunk's upload and its restored images' download
    # overlap the other chunks' solves ----
    e2e = None
    if not args.no_e2e:
        gh = g_d.cpu().pin_memory()
        fh = f_d.cpu().pin_memory()
        oh = torch.empty_like(gh).pin_memory()
        sizes = e2e_split(B)
        nch = len(sizes)
        cplans = []
        for bs in sizes:
            cp = C.c_void_p()
            dbx._check(L.dbx_plan_create(n, n, bs, dbx._ptr(taps), q, q, 3, local, C.byref(cp)))
            dbx._check(L.dbx_precond_build(cp, float(cfg.alpha)))
            cplans.append(cp)
        handles = (C.c_void_p * nch)(*cplans)

        def solve_host():
            dbx._check(L.dbx_landweber_run_chunks(handles, nch, dbx._ptr(gh), dbx._ptr(fh), 1.0, H, 1, 0, 0.0, 1,
                                                  dbx._ptr(oh), dbx._ptr(rre_h), dbx._ptr(res_h), best, done))

        solve_host()  # warm (graphs, staging buffers)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            solve_host()
        e1.record()
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": px_it / (float(te.item()) * 1e-3) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(2 * B * N * 8), "d2h_bytes_per_step": int(B * N * 8 + 2 * B * H * 8),
               "path": f"dbx_landweber_run_chunks: {nch} chunks of {'/'.join(map(str, sizes))} images, pinned host arrays, "
                       "uploads/downloads overlapped with the other chunks' solves"}
        for cp in cplans:
            L.dbx_plan_destroy(cp)
        del gh, fh, oh

    # ---- roofline of the dominant kernel (per-launch CUDA events of the
    # eager step; every kernel of the iteration listed) ----
    from paper_1211_0393_b200 import workmodel as wm
    names = ["blur_adjoint(A')", "blur(A)+residual", "ar_transform_pass", "finalize"]
    peaks = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
    if os.path.exists(HBM_FILE):
        hbm_peak, hsrc = float(json.load(open(HBM_FILE))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
    else:
        hbm_peak, hsrc = 7700.0, "B200_PROFILING.md fallback (7.7 TB/s nominal)"
    conv_e, dst_e, fz = C.c_int(), C.c_int(), C.c_int()
    L.dbx_plan_engines(plan, C.byref(conv_e), C.byref(dst_e))
    L.dbx_plan_pipeline(plan, C.byref(fz))
    separable = fz.value == 2
    p_fp64 = peaks.get("dfma_tflops_sustained", 34.0)
    fsrc = "measured DFMA FP64 sustained (profiles/r01_fp64_peak.json, SM clock 1965 MHz)"
    step_s = t_max * 1e-3 / args.steps
    traffic_tab = {}
    if os.path.exists(TRAFFIC_FILE):
        tj = json.load(open(TRAFFIC_FILE))
        if tj.get("images") == B:
            traffic_tab = tj.get("per_launch_bytes", {})
    kern = []
    model = wm.fused_sep_kernels(n, q, B) if separable else {}
    tot_ms = sum(v[0] for v in kprof.values()) or 1e-9
    for name, (kms_, kc_) in sorted(kprof.items(), key=lambda kv: -kv[1][0]):
        e = {"kernel": name, "ms_per_step": kms_, "launches_per_step": kc_, "share_of_step": kms_ / tot_ms,
             "avg_launch_ms": kms_ / max(kc_, 1)}
        if name in model:
            avg_s = e["avg_launch_ms"] * 1e-3
            e.update({"algorithmic_bytes_per_launch": model[name]["bytes"],
                      "achieved_gbs": model[name]["bytes"] / avg_s / 1e9,
                      "frac_hbm": model[name]["bytes"] / avg_s / 1e9 / hbm_peak,
                      "algorithmic_flops_per_launch": model[name]["flops"],
                      "achieved_tflops": model[name]["flops"] / avg_s / 1e12,
                      "frac_fp64": model[name]["flops"] / avg_s / 1e12 / p_fp64,
                      "traffic_per_launch": traffic_tab.get(name)})
        kern.append(e)
    dom = next((e for e in kern if "frac_hbm" in e), kern[0] if kern else None)
    roof = {"kernel": dom["kernel"] if dom else None, "bound": "hbm", "peak": hbm_peak, "unit": "GB/s",
            "peak_source": hsrc}
    if dom and "frac_hbm" in dom:
        t_hbm = dom["algorithmic_bytes_per_launch"] / (hbm_peak * 1e9)
        t_fp = dom["algorithmic_flops_per_launch"] / (p_fp64 * 1e12)
        roof.update({"avg_launch_ms": dom["avg_launch_ms"], "share_of_step": dom["share_of_step"],
                     "achieved": dom["achieved_gbs"], "frac": dom["frac_hbm"],
                     "algorithmic_bytes_per_launch": dom["algorithmic_bytes_per_launch"],
                     "traffic": dom["traffic_per_launch"],
                     "traffic_source": ("ncu --set full dram__bytes_read.sum + dram__bytes_write.sum per launch at "
                                        f"{B} images ({os.path.basename(TRAFFIC_FILE)})") if traffic_tab else None,
                     "binding": "hbm" if t_hbm >= t_fp else "fp64 (below the FP64 ridge the HBM floor binds)",
                     "secondary": {"achieved": dom["achieved_tflops"], "peak": p_fp64, "unit": "TFLOP/s",
                                   "frac": dom["frac_fp64"], "peak_source": fsrc,
                                   "algorithmic_flops_per_launch": dom["algorithmic_flops_per_launch"]},
                     "form": "fused separable pipeline (rank-1 mask: direct row/column correlation passes; "
                             "packed real FFT-form DST-I)",
                     "note": "bytes: every array the kernel must read/write once (workmodel.fused_sep_kernels); "
                             "flops: nominal 5 N log2 N per FFT, 2(2q+1) per pixel per direct pass"})
    roof["kernels"] = kern
    roof["class_ms_per_step"] = {names[i]: float(kms_tot[i] / args.steps) for i in range(4)}
    if separable:
        cls = wm.fused_sep_classes(n, q, B)["ar_transform_pass"]
        avg_cls = kms_tot[2] / max(kcnt_tot[2], 1) * 1e-3
        roof["class_aggregate"] = {"class": "ar_transform_pass (3 kernels)",
                                   "achieved": cls["bytes"] / cls["launches"] / avg_cls / 1e9,
                                   "frac": cls["bytes"] / cls["launches"] / avg_cls / 1e9 / hbm_peak}
    roof["dense_stencil_sol"] = wm.canonical(q, float(world * B * N * H) / world, step_s, hbm_peak, p_fp64)

    others = None
    if rank == 0 and world == 1 and not args.no_other_configs and args.config == "C3" and not args.images:
        others = other_configs(L, dbx, cf, torch, dev, local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, sample = cpu_sample(cfg, 1, 2)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample}
        if args.config == "C3" and not args.images:
            cpu["per_config"] = cpu_per_config(cf)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
                "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded scenes/masks/noise, host-generated; stands in for Cameraman/Bridge)",
                "config": workload_config(cfg, B, world, args.weak),
                "clocks": clk, "gpu_launches": launches, "roofline": roof, "e2e": e2e, "cpu_baseline": cpu}
        if others:
            line["other_configs"] = {"unit": UNIT, "note": "single-GPU graph path, D-Landweber unless plain_*; "
                                                          "parity cases, not the headline", **others}
        print(json.dumps(line), flush=True)
    L.dbx_plan_destroy(plan)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
