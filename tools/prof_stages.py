"""Device timing of the §8f kernels (lattice query, upsample) with CUDA events.

Algorithmic bytes:
  sample_grid_field: 4 B per lattice value written + 4*K B per grid vertex read once
  upsample:          4*K B per new vertex written + 4*K B per old vertex read once
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2402_14415_b200 as tg  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = []
    for order, gres, lat in ((2, 128, 512), (2, 256, 256), (1, 512, 512), (2, 512, 512)):
        spec = tg.GridSpec(dim=3, resolution=(gres,) * 3, order=order)
        g = tg.init_grid(spec, tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.1, seed=1,
                                              memory_cap_bytes=1 << 40))
        K = spec.coeffs_per_vertex()
        vals = torch.empty(lat ** 3, dtype=torch.float32, device="cuda")
        ms = timed(lambda: tg.sample_grid_field(g, (lat,) * 3, out=vals))
        b = 4 * lat ** 3 + 4 * K * gres ** 3
        out.append(dict(kernel="sample_grid_field", order=order, grid=gres, lattice=lat, ms=ms,
                        gbs=b / ms / 1e6, frac=b / ms / 1e6 / peak, gpts=lat ** 3 / ms / 1e6))
        del g, vals
        torch.cuda.empty_cache()
    for order, a, b_ in ((2, 64, 128), (2, 128, 256), (1, 256, 512)):
        spec = tg.GridSpec(dim=3, resolution=(a,) * 3, order=order)
        g = tg.init_grid(spec, tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.1, seed=1,
                                              memory_cap_bytes=1 << 40))
        K = spec.coeffs_per_vertex()
        dst = tg.init_grid(tg.GridSpec(dim=3, resolution=(b_,) * 3, order=order),
                           tg.InitOptions(memory_cap_bytes=1 << 40))
        L = tg.lib()
        ms = timed(lambda: L.tgcu_grid_upsample(g.handle, dst.handle, 2, None))
        byt = 4 * K * (a ** 3 + b_ ** 3)
        out.append(dict(kernel="upsample", order=order, src=a, dst=b_, ms=ms, gbs=byt / ms / 1e6,
                        frac=byt / ms / 1e6 / peak))
        del g, dst
        torch.cuda.empty_cache()
    for r in out:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
