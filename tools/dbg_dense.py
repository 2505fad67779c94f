import numpy as np, sys
sys.path.insert(0, '.')
import paper_1211_0393_b200 as dev
from oracle import oracle as O
rng = np.random.default_rng(5)
rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
for (n1, n2) in [(520, 520), (520, 8), (8, 520), (130, 130), (136, 136), (200, 520), (513, 513), (576, 576)]:
    x = rng.uniform(-1, 1, (n1, n2))
    out = []
    for kind in (dev.TransformKind.SineI, dev.TransformKind.AntiReflectiveInverse):
        ref = O.tensor_apply(int(kind), x)
        a = dev.tensor_apply(kind, x, engine=dev.DstEngine.Dense)
        a2 = dev.tensor_apply(kind, x, engine=dev.DstEngine.Dense)
        out.append((int(kind), '%.1e' % rel(a, ref), bool(np.array_equal(a, a2))))
        if rel(a, ref) > 1e-10:
            bad = np.abs(a - ref) > 1e-8 * np.abs(ref).max()
            ii = np.argwhere(bad)
            out.append(('bad rows', sorted(set(ii[:, 0]))[:8], 'cols', sorted(set(ii[:, 1]))[:8], len(ii)))
    print(n1, n2, out, flush=True)
