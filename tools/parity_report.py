#!/usr/bin/env python
"""Parity floor report: for each BASELINE config, the
production GPU trajectory, the FP64 CPU oracle and the same oracle in long
double (64-bit mantissa) on identical seeded inputs:

  gpu_vs_oracle   max over iterations of ||x_gpu - x_orc|| / ||x_orc||
  oracle_vs_ld    the FP64 oracle's own rounding error (against long double)
  gpu_vs_ld       the GPU path's rounding error (against long double)
  best iteration  of all three (strict '<', solver.hpp:114)
  rre margin      (runner-up RRE - best RRE) / best RRE from the long-double
                  history: how far the 'identical best iteration' decision is
                  from being decided by rounding

Writes JSON to --out (default gpurun_out/parity_report.json).  Runs on the
GPU box; the oracle uses every host core (bit-identical for any count).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def margin(h):
    h = np.asarray(h)
    if len(h) < 2:
        return None
    s = np.sort(h)
    return float((s[1] - s[0]) / s[0])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C2plain,C3,C4,C5")
    ap.add_argument("--ld-iters", type=str, default="C5:3",
                    help="per-config iteration caps for the long-double runs, e.g. C5:3,C4:10")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_report.json"))
    args = ap.parse_args()
    import paper_1211_0393_b200 as dbx
    from oracle import oracle as O
    from paper_1211_0393_b200 import configs as cf
    O.build()
    O.set_threads(os.cpu_count() or 1)
    O.set_kernel_cache(True)
    caps = {}
    for tok in filter(None, args.ld_iters.split(",")):
        k, v = tok.split(":")
        caps[k] = int(v)
    report = {"host_threads": os.cpu_count(), "note": __doc__.strip().splitlines()[0], "configs": {}}
    for name in args.configs.split(","):
        plain = name.endswith("plain")
        base = name[:-5] if plain else name
        c = cf.CONFIGS[base]
        n = c.n
        iters = 5 if base == "C5" else c.iters
        t0 = time.time()
        f, g, taps = cf.make_problem(c)
        op = dbx.BlurOperator(dbx.Psf(taps), dbx.BoundaryCondition.AntiReflective, n, n)
        scfg = dbx.SolverConfig(max_iters=iters, track_rre_against=f)
        if plain:
            run = dbx.landweber(op, g, scfg, keep_iterates=True)
            ref = O.landweber(taps, g, f_true=f, max_iters=iters, keep_iterates=True)
        else:
            d = dbx.build_tikhonov(dbx.Psf(taps), dbx.PreconditionerSpec(dbx.Algebra.AntiReflective, c.alpha), n, n)
            run = dbx.d_landweber(op, d, g, scfg, keep_iterates=True)
            ref = O.landweber(taps, g, d=O.build_tikhonov(taps, c.alpha, n, n), f_true=f, max_iters=iters,
                              keep_iterates=True)
        t1 = time.time()
        ld_it = min(iters, caps.get(base, iters))
        ld = O.landweber(taps, g, f_true=f, max_iters=ld_it, keep_iterates=True,
                         long_double_alpha=(-1.0 if plain else c.alpha))
        t2 = time.time()
        go = [rel(run.iterates[k], ref["iterates"][k]) for k in range(iters)]
        ol = [rel(ref["iterates"][k], ld["iterates"][k]) for k in range(ld_it)]
        gl = [rel(run.iterates[k], ld["iterates"][k]) for k in range(ld_it)]
        ent = {
            "n": n, "q": c.q, "iters": iters, "method": "plain Landweber" if plain else f"D-Landweber alpha={c.alpha}",
            "pipeline": op.pipeline() if hasattr(op, "pipeline") else None,
            "gpu_vs_oracle_max": max(go), "gpu_vs_oracle_last": go[-1],
            "long_double_iters": ld_it,
            "oracle_vs_ld_max": max(ol), "gpu_vs_ld_max": max(gl),
            "best_iteration": {"gpu": run.best_iteration, "oracle": ref["best_iteration"],
                               "long_double": ld["best_iteration"] if ld_it == iters else None},
            "rre_margin_best_vs_runner_up": margin(ref["rre_history"]),
            "rre_margin_ld": margin(ld["rre_history"]) if ld_it == iters else None,
            "seconds": {"gpu+oracle": round(t1 - t0, 1), "long_double": round(t2 - t1, 1)},
        }
        report["configs"][name] = ent
        print(name, json.dumps(ent), flush=True)
        del run, ref, ld
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(report, fh, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
