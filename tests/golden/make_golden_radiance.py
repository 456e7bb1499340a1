"""Golden vectors for the radiance density chain, generated
from the REFERENCE build (oracle/_ref/libtgref.so: tg::render_ray and
tg::photometric_loss, volume_render.cpp) on small seeded fp32-representable
inputs -> tests/golden/radiance.npz.

    python tests/golden/make_golden_radiance.py
"""
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Reference, Spec  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    R = Reference()
    rng = np.random.default_rng(20240601)
    out = {}
    # jit64: RenderOptions::jitter with a seed (per-ray Rng, volume_render.cpp:69-70)
    cases = [("soft64", 0, 64, 2, (8, 7, 9), 2, 0), ("soft100", 0, 100, 1, (6, 6, 7), 1, 0),
             ("relu64", 1, 64, 2, (7, 8, 6), 0, 0), ("jit64", 0, 64, 2, (8, 7, 9), 2, 987654321)]
    for name, act, ns, order, dres, deg, jseed in cases:
        ds = Spec(3, dres, order=order)
        dc = f32(rng.normal(0, 1.0, ds.V * ds.K))
        dc[::ds.K] = f32(rng.uniform(8.0, 14.0, ds.V) if act == 0 else rng.uniform(-2.0, 6.0, ds.V))
        ss = Spec(3, (5, 6, 4), order=0, origin=(-1.1, -1.0, -1.2), extent=(2.2, 2.1, 2.4))
        sc = f32(rng.normal(0, 0.5, ss.V * 3 * (deg + 1) ** 2))
        n = 96
        o = f32(rng.uniform(-0.9, 0.9, (n, 3)))
        d = rng.normal(size=(n, 3))
        d = f32(d / np.linalg.norm(d, axis=1, keepdims=True))
        near = f32(rng.uniform(0.0, 0.2, n))
        far = f32(near + rng.uniform(0.4, 1.6, n))
        gt = f32(rng.uniform(0, 1, (n, 3)))
        rays = dict(origins=o, dirs=d, near=near, far=far, gt=gt)
        r = R.photometric_loss(ds, dc, ss, deg, sc, rays, n_samples=ns, activation=act, want_grad=True, render=True,
                               jitter=jseed != 0, jitter_seed=jseed)
        pre = f"{name}_"
        out.update({pre + "meta": np.array([act, ns, order, deg]), pre + "dres": np.array(dres), pre + "dc": dc,
                    pre + "sc": sc, pre + "sres": np.array(ss.res), pre + "sorg": np.array(ss.origin),
                    pre + "sext": np.array(ss.extent), pre + "o": o, pre + "d": d, pre + "near": near,
                    pre + "far": far, pre + "gt": gt, pre + "loss": np.array([r["loss"]]),
                    pre + "gd": r["grad_density"], pre + "gs": r["grad_sh"], pre + "colors": r["colors"],
                    pre + "resid": r["residual"], pre + "jitter_seed": np.array([jseed], dtype=np.uint64)})
    np.savez_compressed(os.path.join(OUT, "radiance.npz"), **out)
    print("wrote radiance.npz", os.path.getsize(os.path.join(OUT, "radiance.npz")), "bytes")


if __name__ == "__main__":
    main()
