"""Small fused-step repro for compute-sanitizer: python tools/repro_step.py DIM RES ORDER"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2402_14415_b200 as tg  # noqa: E402

dim, res, order = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
spec = tg.GridSpec(dim=dim, resolution=(res,) * dim, order=order)
g = tg.init_grid(spec, tg.InitOptions(mode=tg.InitMode.SmallUniform, epsilon=0.1, seed=1))
g.adam_reset(tg.AdamConfig(lr=1e-2))
rng = np.random.default_rng(0)
s = np.concatenate([rng.uniform(-1, 1, (3000, 3)), rng.uniform(-0.3, 0.3, (3000, 1))], 1)
if dim == 2:
    s[:, 2] = 0
print(tg.train_step(g, s, tg.LossConfig()))
