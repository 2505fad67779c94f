"""Minimal C3 pipeline driver for ncu captures (B images, H iterations, run
twice so the second run is warm).  Diagnostic only."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_0393_b200 as dbx  # noqa: E402
from paper_1211_0393_b200 import configs as cf  # noqa: E402


def main(B=8, H=2):
    import torch
    L = dbx.lib()
    cfg = cf.CONFIGS["C3"]
    F, G, taps = cf.make_batch(cfg, B)
    g = torch.from_numpy(G).cuda()
    f = torch.from_numpy(F).cuda()
    out = torch.empty_like(g)
    plan = C.c_void_p()
    dbx._check(L.dbx_plan_create(cfg.n, cfg.n, B, dbx._ptr(taps), cfg.q, cfg.q, 3, 0, C.byref(plan)))
    dbx._check(L.dbx_precond_build(plan, float(cfg.alpha)))
    rre = np.zeros((B, H)); res = np.zeros((B, H)); best = (C.c_int * B)(); done = (C.c_int * B)()
    for _ in range(2):
        dbx._check(L.dbx_landweber_run(plan, dbx._ptr(g), dbx._ptr(f), 1.0, H, 1, 0, 0.0, 1, dbx._ptr(out),
                                       dbx._ptr(rre), dbx._ptr(res), best, done, None))
    torch.cuda.synchronize()
    L.dbx_plan_destroy(plan)
    print("ok")


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
