"""Per-phase clock shares of the instrumented fused kernels (build with
DBX_BUILD_TAG=phases DBX_BUILD_DEFS=-DDBX_PHASES, run with
DBX_LIB=paper_1211_0393_b200/libdbx_phases.so).  Diagnostic only."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_0393_b200 as dbx  # noqa: E402
from paper_1211_0393_b200 import configs as cf  # noqa: E402

NAMES = {0: "dst_tcols:stage", 1: "dst_tcols:fill1", 2: "dst_tcols:fft1", 3: "dst_tcols:split1",
         4: "dst_tcols:scan1", 5: "dst_tcols:fill2", 6: "dst_tcols:fft2", 7: "dst_tcols:split2",
         8: "dst_tcols:scan2", 9: "dst_tcols:store",
         10: "t_axpy:stage", 11: "t_axpy:fill", 12: "t_axpy:dft", 13: "t_axpy:split+scan",
         14: "t_axpy:x-update", 15: "t_axpy:conv-fwd", 20: "ainv_tt:load", 21: "ainv_tt:inv-fft",
         22: "ainv_tt:rows", 23: "ainv_tt:fill", 24: "ainv_tt:dft", 25: "ainv_tt:split+scan",
         26: "ainv_tt:store", 40: "dst-fft:stage1(r31)", 41: "dst-fft:stage2(r11)", 42: "dst-fft:stage3(r3)"}


def main():
    import torch
    L = dbx.lib()
    L.dbx_debug_phases.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    cfg = cf.CONFIGS["C3"]
    B, H = 8, 4
    F, G, taps = cf.make_batch(cfg, B)
    g = torch.from_numpy(G).cuda()
    f = torch.from_numpy(F).cuda()
    out = torch.empty_like(g)
    plan = C.c_void_p()
    dbx._check(L.dbx_plan_create(cfg.n, cfg.n, B, dbx._ptr(taps), cfg.q, cfg.q, 3, 0, C.byref(plan)))
    dbx._check(L.dbx_precond_build(plan, float(cfg.alpha)))
    rre = np.zeros((B, H)); res = np.zeros((B, H)); best = (C.c_int * B)(); done = (C.c_int * B)()
    run = lambda: dbx._check(L.dbx_landweber_run(plan, dbx._ptr(g), dbx._ptr(f), 1.0, H, 1, 0, 0.0, 1,
                                                 dbx._ptr(out), dbx._ptr(rre), dbx._ptr(res), best, done, None))
    run()
    buf = (C.c_ulonglong * 64)()
    L.dbx_debug_phases(buf, 64)  # reset
    run()
    L.dbx_debug_phases(buf, 64)
    v = np.array(buf[:64], dtype=np.float64)
    # CTAs per run: every fused kernel covers the image in 4-line blocks; the
    # DST FFT stages (40-42) run in rows_ainv_tt, dst_tcols (x2), rows_t_axpy
    ctas = (cfg.n // 4) * B * H
    per = {(0, 10): ctas, (10, 20): ctas, (20, 30): ctas, (40, 43): 4 * ctas}
    for (lo, hi), nc in per.items():
        tot = v[lo:hi].sum()
        if tot <= 0:
            continue
        print("%-22s %8.0f cycles per CTA (thread 0 wall clock)" % ("[group %d-%d]" % (lo, hi - 1), tot / nc))
        for i in range(lo, hi):
            if v[i] > 0:
                print("%-22s %6.1f%%  %8.0f" % (NAMES.get(i, "phase%d" % i), 100 * v[i] / tot, v[i] / nc))
    L.dbx_plan_destroy(plan)


if __name__ == "__main__":
    main()
