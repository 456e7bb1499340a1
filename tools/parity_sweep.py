"""Random-configuration parity sweep of the fused step against the fp64 oracle
(the generator of tests/test_gpu_parity.py::test_fused_step_random_configs).

    python tools/parity_sweep.py [--cases 300] [--start 0]

Prints, per case, the worst |d| / (|ref| * 1e-5 + mass_rel * mass) of the
full gradient for a few mass_rel values, and the worst loss-term error; the
last line summarises the maxima. Used to pick and justify the gradient bound.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_14415_b200 as tg  # noqa: E402
from oracle.pyoracle import Loss, Oracle, Spec  # noqa: E402


def case(O, seed):
    rng = np.random.default_rng(9000 + seed)
    dim = int(rng.choice([2, 3]))
    order = int(rng.integers(0, 3))
    res = tuple(int(r) for r in rng.integers(2, 42, dim)) + ((1,) if dim == 2 else ())
    n = int(rng.choice([1, 7, 513, int(rng.integers(1, 20001))]))
    cfg = tg.LossConfig(lambda1=float(rng.choice([0.0, 1e-4, 1e-2])), lambda2=float(rng.choice([0.0, 2e-5, 1e-3])),
                        k=float(rng.choice([5.0, 50.0])), use_weighting=bool(rng.integers(0, 2)),
                        use_tv=bool(rng.integers(0, 2)), differentiate_weight=bool(rng.integers(0, 2)))
    lr = float(rng.choice([1e-3, 1e-2]))
    s = Spec(dim=dim, res=res[:dim], order=order)
    c = (0.2 * rng.standard_normal(s.V * s.K)).astype(np.float32).astype(np.float64)
    pts = rng.uniform(-1.1, 1.1, (n, 3)).astype(np.float32)
    if dim == 2:
        pts[:, 2] = 0.0
    gt = rng.uniform(-0.5, 0.5, n).astype(np.float32)
    smp = np.concatenate([pts, gt[:, None]], 1).astype(np.float64)
    loss = Loss(cfg.lambda1, cfg.lambda2, cfg.k, cfg.use_weighting, cfg.use_tv, cfg.differentiate_weight)
    gref = np.zeros(s.V * s.K)
    tref = O.total_loss(s, c, smp, loss, gref)
    mass = O.total_loss_mass(s, c, smp, loss)
    g = tg.init_grid(tg.GridSpec(dim=dim, resolution=res, order=order))
    g.coeffs = c
    g.adam_reset(tg.AdamConfig(lr=lr))
    t = tg.train_step(g, smp, cfg, export_grad=True)
    d = np.abs(g.grad() - gref)
    out = {"seed": seed, "dim": dim, "order": order, "res": res[:dim], "n": n, "k": cfg.k, "l1": cfg.lambda1,
           "dw": cfg.differentiate_weight}
    for mr in (4e-6, 2e-6, 1e-6, 5e-7):
        out[f"grad/{mr:g}"] = float(np.max(d / (1e-5 * np.abs(gref) + mr * mass + 1e-300)))
    out["terms_rel"] = float(np.max(np.abs(t.as_array() - tref) / np.maximum(np.abs(tref), 1e-30)))
    g.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=300)
    ap.add_argument("--start", type=int, default=0)
    a = ap.parse_args()
    O = Oracle()
    worst = {}
    for sd in range(a.start, a.start + a.cases):
        r = case(O, sd)
        print(json.dumps(r), flush=True)
        for k, v in r.items():
            if k.startswith("grad/") or k == "terms_rel":
                if v > worst.get(k, (0, None))[0]:
                    worst[k] = (v, sd)
    print(json.dumps({"worst": worst}))


if __name__ == "__main__":
    main()
