"""Time the fused train step on the larger BASELINE configs on one GPU.

    python tools/bench_configs.py [c3] [c5] [--steps 50]

C3: 256^3 order 2, 2^21 points/step (50% uniform / 50% near-surface sigma 0.01)
    of the 64-primitive procedural SDF; C5: 512^3 order 2, 2^23 points/step
    (10% uniform / 90% near-surface sigma 0.005), Adam lr 5e-3. Batches are
    device-resident (input_ready), steps asynchronous, CUDA events around K steps.
Prints one JSON object per config with points/s and the step's fraction of the
HBM roofline on SURVEY 8d's bytes B_t = N(4D+4) + 3*U*K*4 + 32*V*K.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CONFIGS = {
    "c1": dict(res=128, points=1 << 16, near=0.0, sigma=0.01, lr=1e-2, dim=2),
    "c3": dict(res=256, points=1 << 21, near=0.5, sigma=0.01, lr=1e-2),
    "c5": dict(res=512, points=1 << 23, near=0.9, sigma=0.005, lr=5e-3),
    # C2 in deterministic mode (tgcu_grid_set_deterministic): the cost of bit-reproducibility
    "c2det": dict(res=128, points=1 << 20, near=0.5, sigma=0.01, lr=1e-2, det=True, shape="sphere"),
}


def unique_vertex_coeffs(pts, res, K):
    import numpy as np
    h = 2.0 / (res - 1)
    c = np.clip(np.floor((pts[:, :3].astype(np.float64) + 1.0) / h).astype(np.int64), 0, res - 2)
    cells = np.unique((c[:, 2] * res + c[:, 1]) * res + c[:, 0])
    cz, r = np.divmod(cells, res * res)
    cy, cx = np.divmod(r, res)
    out = []
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                out.append(((cz + dz) * res + cy + dy) * res + cx + dx)
    return len(np.unique(np.concatenate(out))) * K


def run(name, steps, warmup):
    import numpy as np
    import torch
    import paper_2402_14415_b200 as tg
    cfg = CONFIGS[name]
    res = cfg["res"]
    dim = cfg.get("dim", 3)
    spec = tg.GridSpec(dim=dim, resolution=(res,) * dim + ((1,) if dim == 2 else ()), order=2)
    g = tg.init_grid(spec, tg.InitOptions(memory_cap_bytes=1 << 40))
    g.adam_reset(tg.AdamConfig(lr=cfg["lr"]))
    g.set_deterministic(cfg.get("det", False))
    if cfg.get("shape") == "sphere":
        host = [tg.sample(tg.SHAPE_SPHERE, 3, 1000 + i, cfg["points"], near_frac=0.5, sigma=0.01, param0=0.6)
                for i in range(2)]
    elif dim == 2:  # C1: circle r=0.5 union box, uniform points (sampling.cpp C1 restatement)
        host = [tg.sample(tg.SHAPE_C1_2D, 2, 500 + i, cfg["points"]) for i in range(2)]
    else:
        host = [tg.sample(tg.SHAPE_PRIMS, 3, 500 + i, cfg["points"], near_frac=cfg["near"], sigma=cfg["sigma"],
                          param0=42) for i in range(2)]
    dev = [torch.from_numpy(b).cuda() for b in host]
    torch.cuda.synchronize()
    lc = tg.LossConfig()
    for i in range(warmup):
        tg.train_step(g, dev[i % 2], lc, asynchronous=True, input_ready=True)
    g.sync()
    tg.reset_launch_count()
    tg.train_step(g, dev[0], lc, asynchronous=True, input_ready=True)
    launches = tg.launch_count()  # per step: 2 = small-grid path (small.cu), 5+ = brick path
    g.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if cfg.get("dim", 3) == 2:
        steps = max(steps, 4000)  # C1 steps take ~25 us: a longer window
    e0.record()
    for i in range(steps):
        tg.train_step(g, dev[i % 2], lc, asynchronous=True, input_ready=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    # the brick kernel's time from a second, profiled window (its per-launch
    # events would otherwise sit inside the timed steps: +45 % at C1)
    graph_leg = None
    if launches == 2:  # small-grid path: the same steps replayed from a CUDA graph (tgcu_train_graph_*)
        try:
            gs = torch.cuda.Stream()
            graph = tg.TrainGraph(g, [dev[i % 2] for i in range(100)], lc, stream=gs)
            for _ in range(3):
                graph.replay()
            g.sync()
            reps = max(1, steps // 100)
            with torch.cuda.stream(gs):
                e0.record(gs)
                for _ in range(reps):
                    graph.replay()
                e1.record(gs)
            torch.cuda.synchronize()
            graph_leg = {"ms_per_step": e0.elapsed_time(e1) / (reps * 100), "steps": reps * 100,
                         "api": "tgcu_train_graph_launch: 100 captured steps per replay (no host call per step)"}
            graph.close()
            g.sync()
        except Exception as ex:  # the leg is optional: report, keep the line
            graph_leg = {"unavailable": f"{type(ex).__name__}: {ex}"}
    g.profile_begin()
    for i in range(steps):
        tg.train_step(g, dev[i % 2], lc, asynchronous=True, input_ready=True)
    torch.cuda.synchronize()
    kms, kn = g.profile_end()
    last = g.sync()
    K = spec.coeffs_per_vertex()
    V = res ** dim
    N = cfg["points"]
    # 2D: U ~= V (uniform points on 127^2 cells); 3D: counted exactly
    UK = V * K if dim == 2 else np.mean([unique_vertex_coeffs(b, res, K) for b in host])
    bt = N * (4 * dim + 4) + 3 * UK * 4 + 32 * V * K
    ours = 24 * V * K + 16 * N
    peak = 6549.1
    try:
        peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    return {"config": name, "deterministic": bool(cfg.get("det", False)), "grid": [res] * dim, "order": 2, "points_per_step": N, "near_frac": cfg["near"],
            "sigma": cfg["sigma"], "ms_per_step": ms, "points_per_s": N / (ms * 1e-3),
            "step_path": "small (2 launches)" if launches == 2 else f"brick ({launches} launches)",
            "launches_per_step": launches,
            "brick_kernel_ms" if launches != 2 else "step_kernels_ms": kms / max(kn, 1), "survey_bytes_per_step": bt,
            "step_frac_survey_bytes": bt / (ms * 1e-3) / 1e9 / peak,
            "kernel_frac_survey_bytes": bt / (kms / max(kn, 1) * 1e-3) / 1e9 / peak,
            "kernel_frac_our_bytes": ours / (kms / max(kn, 1) * 1e-3) / 1e9 / peak, "peak_gbs": peak,
            "loss_last": last.total, "steps": steps, **({"graph": graph_leg} if graph_leg else {})}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c3", "c5"])
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args()
    for c in a.configs:
        print(json.dumps(run(c, a.steps, a.warmup)), flush=True)


if __name__ == "__main__":
    main()
