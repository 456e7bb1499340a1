"""C5 per-GPU load imbalance of the z-slab partition, measured slab by slab on
one GPU ("report per-GPU imbalance and halo-exchange time").

    python tools/c5_imbalance.py [--ranks 2 4 8] [--steps 10] [--res 512]

C5 = 512^3 order 2, 2^23 points/step, 90 % near the surface of the seeded
64-primitive SDF (sigma 0.005) and 10 % uniform. For N ranks the brick layers
are split (a) evenly and (b) by a per-layer weight of points + dense work
(slab.slab_ranges(weights=...)); each rank's slab is built in turn on this GPU
with its owner-sharded points (slab_point_mask) and its fused step is timed
with CUDA events (no rank waits on another: the partial sums are the slab's
own). Reports per-rank step ms, max / mean (the imbalance that caps scaling
efficiency), and the halo bytes a step moves per rank pair.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, nargs="*", default=[2, 4, 8])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--res", type=int, default=512)
    ap.add_argument("--points", type=int, default=1 << 23)
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_2402_14415_b200 as tg
    from paper_2402_14415_b200.slab import SlabGrid, brick_layers, point_cells_z, slab_point_mask, slab_ranges
    res = a.res
    spec = tg.GridSpec(dim=3, resolution=(res,) * 3, order=2)
    K = spec.coeffs_per_vertex()
    batch = tg.sample(tg.SHAPE_PRIMS, 3, 77, a.points, near_frac=0.9, sigma=0.005, param0=42)
    b64 = batch.astype(np.float64)
    nbz = brick_layers(res)
    # per brick layer: points whose cell lies in it, and owned vertices
    cz = point_cells_z(spec, b64[:, 2])
    pts_layer = np.bincount(np.minimum(cz // 8, nbz - 1), minlength=nbz).astype(np.float64)
    verts_layer = np.array([min(8, res - 8 * l) for l in range(nbz)], dtype=np.float64) * res * res
    cfg = tg.LossConfig()
    out = {"config": "C5 512^3 o2, 2^23 pts, 90% near-surface sigma 0.005", "plane_bytes": res * res * K * 4,
           "results": []}

    def time_partition(n, mode, ranges):
        per = []
        for r, (lo, hi) in enumerate(ranges):
            sg = SlabGrid(spec, lo, hi, tg.InitOptions(memory_cap_bytes=1 << 40))
            sg.adam_reset(tg.AdamConfig(lr=5e-3))
            local = np.ascontiguousarray(batch[slab_point_mask(spec, b64, lo, hi)])
            dev = torch.from_numpy(local).cuda()
            torch.cuda.synchronize()
            for _ in range(2):
                sg.finish(sg.begin(dev, cfg, n_global=len(batch), input_ready=True), asynchronous=True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                sg.finish(sg.begin(dev, cfg, n_global=len(batch), input_ready=True), asynchronous=True)
            e1.record()
            torch.cuda.synchronize()
            per.append({"rank": r, "brick_layers": [lo, hi], "points": int(len(local)),
                        "ms": e0.elapsed_time(e1) / a.steps})
            sg.close()
            del dev
            torch.cuda.empty_cache()
        ms = np.array([p["ms"] for p in per])
        out["results"].append({"ranks": n, "partition": mode, "per_rank": per, "max_ms": float(ms.max()),
                               "mean_ms": float(ms.mean()), "imbalance_max_over_mean": float(ms.max() / ms.mean()),
                               "halo_planes_per_step": 2 * (n - 1)})
        print(json.dumps(out["results"][-1]), flush=True)
        return per

    # even split first; the per-slab times then calibrate a per-layer cost
    # model t = a * points + b * vertices (least squares) for the weighted split
    rows, times = [], []
    for n in a.ranks:
        ranges = slab_ranges(nbz, n)
        for p, (lo, hi) in zip(time_partition(n, "even", ranges), ranges):
            rows.append([pts_layer[lo:hi].sum(), verts_layer[lo:hi].sum(), 1.0])
            times.append(p["ms"])
    coef, *_ = np.linalg.lstsq(np.array(rows), np.array(times), rcond=None)
    out["cost_model_ms"] = {"per_point": float(coef[0]), "per_vertex": float(coef[1]), "fixed": float(coef[2])}
    print(json.dumps(out["cost_model_ms"]), flush=True)
    w = np.maximum(coef[0] * pts_layer + coef[1] * verts_layer, 1e-12)
    for n in a.ranks:
        time_partition(n, "weighted", slab_ranges(nbz, n, weights=w))
    print(json.dumps({"summary": [(x["ranks"], x["partition"], round(x["imbalance_max_over_mean"], 3))
                                  for x in out["results"]]}))


if __name__ == "__main__":
    main()
