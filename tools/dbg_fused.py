import sys, numpy as np
sys.path.insert(0, '.')
import paper_1211_0393_b200 as dev
from paper_1211_0393_b200 import configs as cf
for name, n, conv in (("C2", 512, "Auto"), ("C3", 1024, "Auto"), ("C1", 256, "Fft")):
    c = cf.CONFIGS[name]
    f, g, taps = cf.make_problem(c, n=n)
    op = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, n, n)
    op.set_conv(getattr(dev.ConvEngine, conv)).set_fusion(True).set_timing(True)
    d = dev.build_tikhonov(dev.Psf(taps), dev.PreconditionerSpec(dev.Algebra.AntiReflective, c.alpha), n, n)
    try:
        run = dev.d_landweber(op, d, g, dev.SolverConfig(max_iters=2, track_rre_against=f))
        print(name, 'ok', run.rre_history, op.kernel_times(), flush=True)
    except Exception as e:
        print(name, 'ERR', e, flush=True)
