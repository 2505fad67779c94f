"""Alpha sweep on the GPU: the direct caller of the hot
path.  The reference's experiment driver (experiment.hpp:182-310) runs, per
boundary condition, one plain Landweber cell and one D-Landweber cell per
alpha of a log-spaced grid, keeps the best cell, and writes per-cell
`iter,rre,residual` CSVs, `summary.csv` and `metadata.txt`.  Here the alpha
cells are independent images of ONE batched run: every image of the batch is
the same blurred data g, image b is preconditioned with its own filter grid
d_b = 1/(lambda^2 + alpha_b) (dbx_precond_build_sweep), so a whole sweep is a
single CUDA-graph run.  Boundary conditions: anti-reflective (the path) and
reflective (its CosineIII algebra, §8f f3), one block of cells per BC like
the reference's `for (BoundaryCondition bc : cfg.bcs)` loop
(experiment.hpp:201-270), with the restored PGMs of the plain cell and of the
best preconditioned cell per BC (experiment.hpp:242-244, 266-268).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os
import time
from typing import List, Optional, Sequence

import numpy as np

from . import (DBX_EDIVERGED, BlurOperator, BoundaryCondition, Psf, RestorationRun, SolverConfig,
               SolverDivergence, StoppingRule, _check, _f64, _ptr, landweber, lib)
from .io import write_pgm

# to_string(BoundaryCondition), boundary.hpp:11-19 (the BCs this path runs)
BC_NAMES = {BoundaryCondition.AntiReflective: "antireflective", BoundaryCondition.Reflective: "reflective"}
BC_NAME = BC_NAMES[BoundaryCondition.AntiReflective]


def bc_name(bc) -> str:
    bc = BoundaryCondition(bc)
    if bc not in BC_NAMES:
        raise ValueError("run_experiment: no preconditioner algebra on this path for %s BCs" % bc.name)
    return BC_NAMES[bc]


def alpha_grid(min_alpha: float = 1e-6, max_alpha: float = 1e-1, count: int = 6) -> List[float]:
    """Log-spaced grid, endpoints included (experiment.hpp:36-46)."""
    if not (min_alpha > 0.0 and max_alpha >= min_alpha):
        raise ValueError("AlphaSweep: bounds must be positive and ordered")
    if count < 1:
        raise ValueError("AlphaSweep: need at least one point")
    if count == 1:
        return [min_alpha]
    la, lb = math.log(min_alpha), math.log(max_alpha)
    return [math.exp(la + (lb - la) * i / (count - 1)) for i in range(count)]


def format_double(v: float) -> str:
    return "%.17g" % v


def format_alpha(v: float) -> str:
    return "%.6g" % v


@dataclasses.dataclass
class CellResult:
    method: str            # "landweber" or "d-landweber"
    alpha: float
    run: RestorationRun
    seconds: float
    diverged: bool = False
    bc: BoundaryCondition = BoundaryCondition.AntiReflective

    def stem(self) -> str:  # experiment.hpp:160-164
        s = bc_name(self.bc) + "_" + self.method
        return s if self.method == "landweber" else s + "_alpha" + format_alpha(self.alpha)


@dataclasses.dataclass
class SummaryRow:
    method: str
    alpha: float
    best_rre: float
    best_iter: int
    seconds: float
    bc: BoundaryCondition = BoundaryCondition.AntiReflective


@dataclasses.dataclass
class ExperimentResult:
    cells: List[CellResult]
    summary: List[SummaryRow]


def history_csv(run: RestorationRun) -> str:  # experiment.hpp:149-158
    out = ["iter,rre,residual"]
    for k, r in enumerate(run.residual_history):
        e = format_double(run.rre_history[k]) if k < len(run.rre_history) else ""
        out.append("%d,%s,%s" % (k + 1, e, format_double(r)))
    return "\n".join(out) + "\n"


def _write(path: str, text: str):
    tmp = path + ".tmp"  # write-then-rename, like write_file_atomic
    with open(tmp, "w") as fh:
        fh.write(text)
    os.replace(tmp, path)


def sweep_d_landweber(taps, g, f_true, alphas: Sequence[float], max_iters: int, tau: float = 1.0,
                      device: int = 0, bc=BoundaryCondition.AntiReflective) -> List[CellResult]:
    """One batched D-Landweber run: image b = g with alpha_b (MinRre against
    f_true); the filter algebra follows the BC (detail::algebra_for,
    experiment.hpp:166-174: AntiReflective or CosineIII)."""
    g, f = _f64(g), _f64(f_true)
    B = len(alphas)
    n1, n2 = g.shape
    bc_name(bc)
    op = BlurOperator(Psf(taps), BoundaryCondition(bc), n1, n2, batch=B, device=device)
    L = lib()
    al = np.ascontiguousarray(alphas, dtype=np.float64)
    _check(L.dbx_precond_build_sweep(op.handle, _ptr(al)))
    gb = np.ascontiguousarray(np.broadcast_to(g, (B, n1, n2)))
    fb = np.ascontiguousarray(np.broadcast_to(f, (B, n1, n2)))
    H = max(max_iters, 1)
    restored = np.empty_like(gb)
    rre = np.zeros((B, H))
    res = np.zeros((B, H))
    best = (C.c_int * B)()
    done = (C.c_int * B)()
    stop = StoppingRule.min_rre()
    t0 = time.perf_counter()
    st = L.dbx_landweber_run(op.handle, _ptr(gb), _ptr(fb), float(tau), int(max_iters), int(stop.kind), 0, 0.0, 1,
                             _ptr(restored), _ptr(rre), _ptr(res), best, done, None)
    secs = time.perf_counter() - t0
    if st not in (0, DBX_EDIVERGED):
        _check(st)
    cells = []
    for b in range(B):
        k = done[b]
        diverged = st == DBX_EDIVERGED and k < max_iters  # the guard fired before recording
        run = RestorationRun(restored=restored[b], iterations_executed=k, best_iteration=best[b],
                             rre_history=list(rre[b, :k]), residual_history=list(res[b, :k]))
        cells.append(CellResult("d-landweber", float(alphas[b]), run, secs / B, diverged, BoundaryCondition(bc)))
    return cells


def run_experiment(taps, g, f_true, alphas: Sequence[float], max_iters: int, precond_max_iters: int = 0,
                   tau: float = 1.0, out_dir: Optional[str] = None, meta: Optional[dict] = None,
                   device: int = 0, bcs: Sequence = (BoundaryCondition.AntiReflective,)) -> ExperimentResult:
    """Per BC (experiment.hpp:201-270): the plain Landweber cell + the batched
    alpha sweep, a summary row per (bc, method) (the sweep's best alpha, strict
    '<' so the first best alpha wins), and, when out_dir is set, the files in
    the reference's formats: per-cell CSVs, `<bc>_landweber.pgm` (plain
    restored) and `<bc>_d-landweber.pgm` (best cell's restored), summary.csv,
    metadata.txt.  The same (Honest) data g, f serve every BC, as the
    reference's honest_data does."""
    g, f = _f64(g), _f64(f_true)
    n1, n2 = g.shape
    if not bcs:
        raise ValueError("run_experiment: need at least one BC")
    for bc in bcs:
        bc_name(bc)
    write = bool(out_dir)
    if write:
        os.makedirs(out_dir, exist_ok=True)
    cells: List[CellResult] = []
    summary: List[SummaryRow] = []
    piters = precond_max_iters if precond_max_iters > 0 else max_iters
    for bc in bcs:
        bc = BoundaryCondition(bc)
        name = bc_name(bc)
        op = BlurOperator(Psf(taps), bc, n1, n2, device=device)
        cfg = SolverConfig(tau=tau, max_iters=max_iters, stop=StoppingRule.min_rre(), track_rre_against=f)
        t0 = time.perf_counter()
        try:
            plain = CellResult("landweber", 0.0, landweber(op, g, cfg), 0.0, False, bc)
        except SolverDivergence:
            plain = CellResult("landweber", 0.0, RestorationRun(), 0.0, True, bc)
        plain.seconds = time.perf_counter() - t0
        cells.append(plain)
        pr = plain.run
        summary.append(SummaryRow("landweber", 0.0, pr.rre_history[pr.best_iteration - 1] if pr.best_iteration > 0
                                  else math.inf, pr.best_iteration, plain.seconds, bc))
        if write:
            write_pgm(os.path.join(out_dir, name + "_landweber.pgm"),
                      pr.restored if pr.restored is not None else np.zeros((0, 0)))
        if alphas:
            sweep = sweep_d_landweber(taps, g, f, alphas, piters, tau, device, bc)
            cells += sweep
            best = SummaryRow("d-landweber", 0.0, math.inf, 0, 0.0, bc)
            best_cell = None
            for c in sweep:
                if c.diverged or c.run.best_iteration == 0:
                    continue
                e = c.run.rre_history[c.run.best_iteration - 1]
                if e < best.best_rre:  # strict '<': first best alpha wins
                    best = SummaryRow("d-landweber", c.alpha, e, c.run.best_iteration, c.seconds, bc)
                    best_cell = c
            summary.append(best)
            if write and best_cell is not None:
                write_pgm(os.path.join(out_dir, name + "_d-landweber.pgm"), best_cell.run.restored)
    if write:
        for c in cells:
            if c.run.rre_history:
                _write(os.path.join(out_dir, c.stem() + ".csv"), history_csv(c.run))
        rows = ["bc,method,alpha,best_rre,best_iter,seconds"]
        for r in summary:
            rows.append("%s,%s,%s,%s,%d,%.3f" % (bc_name(r.bc), r.method, format_alpha(r.alpha),
                                                 format_double(r.best_rre), r.best_iter, r.seconds))
        _write(os.path.join(out_dir, "summary.csv"), "\n".join(rows) + "\n")
        m = {"fov": "%dx%d" % (n1, n2), "psf_support": "%dx%d" % taps.shape, "tau": format_double(tau),
             "x0": "zero", "iteration_convention": "completed-steps-from-1",
             "stopping": "min-rre (oracle stopping on the true image; non-blind)",
             "plain_max_iters": str(max_iters), "precond_max_iters": str(piters),
             "alphas": ",".join(format_alpha(a) for a in alphas),
             "bcs": ",".join(bc_name(b) for b in bcs), "engine": "B200 (batched alpha sweep)"}
        m.update(meta or {})
        _write(os.path.join(out_dir, "metadata.txt"), "".join("%s=%s\n" % kv for kv in m.items()))
    return ExperimentResult(cells, summary)
