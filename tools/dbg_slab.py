import sys, os, numpy as np, torch, ctypes as C
sys.path.insert(0, os.getcwd())
import paper_1211_0393_b200 as dbx
from paper_1211_0393_b200 import configs as cf
from paper_1211_0393_b200.slab import SlabLandweber, LocalWorld
n = int(sys.argv[1]); cfgname = sys.argv[2]; P = int(sys.argv[3])
c = cf.CONFIGS[cfgname]
f, g, taps = cf.make_problem(c, n=n)
op = dbx.BlurOperator(dbx.Psf(taps), dbx.BoundaryCondition.AntiReflective, n, n)
d = dbx.build_tikhonov(dbx.Psf(taps), dbx.PreconditionerSpec(dbx.Algebra.AntiReflective, c.alpha), n, n)
iters = 20
try:
    ref = dbx.d_landweber(op, d, g, dbx.SolverConfig(max_iters=iters, track_rre_against=f))
    print("single:", ref.iterations_executed, ref.best_iteration, ref.residual_history[:3], ref.residual_history[-3:])
except Exception as e:
    print("single failed:", e)
R = n // P; dev = torch.device("cuda", 0)
gs = {p: torch.from_numpy(np.ascontiguousarray(g[p*R:(p+1)*R])).to(dev) for p in range(P)}
fs = {p: torch.from_numpy(np.ascontiguousarray(f[p*R:(p+1)*R])).to(dev) for p in range(P)}
s = SlabLandweber(LocalWorld(P), n, taps, c.q, c.alpha, device=0)
try:
    run = s.run(gs, fs, iters)
    print("slab:", run["iterations_executed"], run["best_iteration"], run["residual_history"][:3], run["residual_history"][-3:])
except Exception as e:
    print("slab failed:", e)
