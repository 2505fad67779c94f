"""Graph-path throughput of one BASELINE config under engine overrides, with
per-class kernel times (diagnostic; bench.py is the contract).
Usage: config_probe.py CONFIG [conv=0|1|2] [fusion=0|1] [reps] [dst=0 auto|1 dense|2 fft]"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_0393_b200 as dbx  # noqa: E402
from paper_1211_0393_b200 import configs as cf  # noqa: E402


def main(name, conv=0, fusion=1, reps=3, dst=0):
    import torch
    L = dbx.lib()
    cfg = cf.CONFIGS[name]
    F, G, taps = cf.make_batch(cfg, 1)
    g = torch.from_numpy(G).cuda()
    f = torch.from_numpy(F).cuda()
    o = torch.empty_like(g)
    n, q, H = cfg.n, cfg.q, cfg.iters
    plan = C.c_void_p()
    dbx._check(L.dbx_plan_create(n, n, 1, dbx._ptr(taps), q, q, 3, 0, C.byref(plan)))
    dbx._check(L.dbx_plan_set_conv(plan, conv))
    dbx._check(L.dbx_plan_set_fusion(plan, fusion))
    dbx._check(L.dbx_plan_set_dst(plan, dst))
    dbx._check(L.dbx_precond_build(plan, float(cfg.alpha)))
    stream = torch.cuda.ExternalStream(L.dbx_plan_stream(plan))
    rre, res = np.zeros(H), np.zeros(H)
    best, done = (C.c_int * 1)(), (C.c_int * 1)()
    solve = lambda: dbx._check(L.dbx_landweber_run(plan, dbx._ptr(g), dbx._ptr(f), 1.0, H, 1, 0, 0.0, 1,
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
    L.dbx_plan_set_timing(plan, 1)
    solve()
    torch.cuda.synchronize()
    kt, kc = (C.c_double * 8)(), (C.c_int * 8)()
    L.dbx_plan_kernel_times(plan, kt, kc, 8)
    fz, ce, de = C.c_int(), C.c_int(), C.c_int()
    L.dbx_plan_pipeline(plan, C.byref(fz))
    L.dbx_plan_engines(plan, C.byref(ce), C.byref(de))
    print(json.dumps({"config": name, "conv": ce.value, "dst": de.value, "fused": fz.value, "ms_per_run": ms,
                      "mpx_it_s": n * n * H / (ms * 1e-3) / 1e6, "best": best[0], "rre_last": rre[-1],
                      "class_ms": [round(kt[i], 3) for i in range(4)], "class_launches": [kc[i] for i in range(4)]}))
    L.dbx_plan_destroy(plan)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], *[int(x) for x in a[1:]])
