"""C5 throughput through the C++ row-slab loop (P in-process ranks on one GPU;
P = 1 is the one-rank NCCL-free path the bench runs per rank) next to the
single-image graph path.  Usage: slab_probe.py P [reps]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1211_0393_b200 import configs as cf  # noqa: E402
from paper_1211_0393_b200.slab import SlabRun  # noqa: E402


def main(P=1, reps=3):
    c = cf.CONFIGS["C5"]
    t0 = time.time()
    F, G, taps = cf.make_batch(c, 1)
    dev = torch.device("cuda", 0)
    g, f = torch.from_numpy(G[0]).to(dev), torch.from_numpy(F[0]).to(dev)
    run = SlabRun(c.n, P, taps, c.q, c.alpha, rank=-1, device=0)
    out = torch.empty_like(g)
    run.run(g, f, c.iters, out=out)
    torch.cuda.synchronize()
    s = torch.cuda.ExternalStream(run.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        _, h = run.run(g, f, c.iters, out=out)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"config": "C5", "path": "cpp slab loop", "P": P, "ms_per_run": ms,
                      "mpx_it_s": c.n * c.n * c.iters / (ms * 1e-3) / 1e6, "best": h["best_iteration"],
                      "launches_per_run": run.launch_count() / (reps + 1), "separable": run.separable,
                      "setup_s": round(time.time() - t0, 2)}))
    run.close()


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
