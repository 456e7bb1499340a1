"""Benchmark of the TaylorGrid query-and-optimise hot path on B200.

Workloads (BASELINE.json configs):
  c2  (default at N=1, configs[1]): 3D 128^3 grid, order 2 (10 fp32
      coefficients per vertex, zero init), target = analytic sphere r=0.6,
      2^20 points per step (50% uniform in the cube, 50% near-surface: sphere
      point + N(0, 0.01) per axis), Adam lr 1e-2.
  c3  (default at N>1, configs[2]): 256^3, order 2, 2^21 points per step
      (50% uniform / 50% near-surface sigma 0.01) of the seeded min-union of
      64 procedural primitives; strong scaling over z-slabs.
  c5  (configs[4], --workload c5): 512^3, order 2, 2^23 points per step
      (10% uniform / 90% near-surface sigma 0.005), Adam lr 5e-3; strong
      scaling over z-slabs, per-rank imbalance reported.
Every workload uses the paper loss (lambda1=1e-4 reuse-batch, lambda2=2e-5 TV,
k=50, weighting on). A step = zero grad -> total_loss -> finite check ->
adam_step (one run_schedule iteration), executed by the fused device pipeline
(tgcu_train_step; slabs: tgcu_slab_step_begin/finish). Metric: train points/s.

Extra keys: roofline (fused brick kernel, HBM), cpu_baseline (the reference's
own CPU code, oracle/_ref, on this host), e2e (through the C ABI with host
buffers), query (C4: 512^3 forward-only query, unsorted and brick-sorted,
with the reference's own eval timed on a bounded sample), larger_configs (C1,
C3, C5 on one GPU, each with a bounded reference CPU sample).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c5] [--impl reference]
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NBATCH = 4
METRIC = "TaylorGrid train points/s (fwd+bwd+Adam) & query Mpts/s; % of HBM roofline"
LOSS_DESC = "paper loss (lambda1=1e-4 reuse-batch, lambda2=2e-5 TV, k=50)"
STEP_DESC = "step = zero-grad + total_loss + finite check + adam_step"
WORKLOADS = {
    "c2": dict(res=128, points=1 << 20, shape="sphere", near=0.5, sigma=0.01, lr=1e-2,
               desc="C2: 3D 128^3 order-2 TaylorGrid SDF fit, sphere r=0.6, 2^20 points/step "
                    "(50% uniform / 50% near-surface sigma=0.01)"),
    "c3": dict(res=256, points=1 << 21, shape="prims", near=0.5, sigma=0.01, lr=1e-2,
               desc="C3: 3D 256^3 order-2 TaylorGrid SDF fit, min-union of 64 seeded primitives, 2^21 points/step "
                    "(50% uniform / 50% near-surface sigma=0.01)"),
    "c5": dict(res=512, points=1 << 23, shape="prims", near=0.9, sigma=0.005, lr=5e-3,
               desc="C5: 3D 512^3 order-2 TaylorGrid SDF fit, min-union of 64 seeded primitives, 2^23 points/step "
                    "(10% uniform / 90% near-surface sigma=0.005)"),
}
PRIM_SEED = 42  # seed of the 64 procedural primitives (tgcu_sample SHAPE_PRIMS param0)


def workload_config(wl, ws):
    """The config dict both arms print (identical keys and values)."""
    W = WORKLOADS[wl]
    return {"workload": f"{W['desc']}, {LOSS_DESC}, Adam lr {W['lr']:g}; {STEP_DESC}",
            "grid": [W["res"]] * 3, "order": 2, "points_per_step": W["points"],
            "parallelism": "single GPU" if ws == 1 else
            f"z-slab x{ws}: owner computes, points binned to their owning GPU, NCCL all-reduce of the loss partials, "
            "halo planes stored into the neighbours over peer memory"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def mem_available_bytes():
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except Exception:
        pass
    return 0


E2E_WINDOWS = 5


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed legs run."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                util = float(parts[6])
                s, m = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            if util < 5:
                continue
            sm.append(s)
            mx.append(m)
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- inputs ---------------------------------------------------------------------------


def make_batches(wl, seed0, count=NBATCH):
    """Seeded batches (x, y, z, gt) fp32 through the package's host sampler
    (tgcu_sample: the reference Rng mappings; the sphere batches equal
    sample_sphere_points(0.6, {1, 1, 0}, 0.01) bit for bit, test_abi_cpu.py)."""
    import paper_2402_14415_b200 as tg
    W = WORKLOADS[wl]
    if W["shape"] == "sphere":
        return [tg.sample(tg.SHAPE_SPHERE, 3, seed0 + i, W["points"], near_frac=0.5, sigma=0.01, param0=0.6)
                for i in range(count)]
    return [tg.sample(tg.SHAPE_PRIMS, 3, seed0 + i, W["points"], near_frac=W["near"], sigma=W["sigma"],
                      param0=PRIM_SEED) for i in range(count)]


def reference_batches(wl, seed0, count=NBATCH):
    """The same batches for the reference arm, without mapping libtgcu.so into
    the reference process: C2 from the reference's own sampler
    (sample_sphere_points, sampling.cpp:140-159, rounded to fp32 with gt from
    the fp32 point exactly as tgcu_sample does); C3 / C5 (procedural target,
    not in the reference) from a child process that writes them to a file."""
    W = WORKLOADS[wl]
    if W["shape"] == "sphere":
        from oracle.pyoracle import Reference
        R = Reference()
        out = []
        for i in range(count):
            s = R.sample_sphere(0.6, W["points"], ratio=(1, 1, 0), sigma_near=0.01, seed=seed0 + i)
            p = s[:, :3].astype(np.float32)
            gt = (np.linalg.norm(p.astype(np.float64), axis=1) - 0.6).astype(np.float32)
            out.append(np.ascontiguousarray(np.concatenate([p, gt[:, None]], 1)))
        return out
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "batches.npy")
        subprocess.run([sys.executable, os.path.abspath(__file__), "--gen-batches", wl, "--gen-seed", str(seed0),
                        "--gen-count", str(count), "--gen-out", path], check=True)
        a = np.load(path)
    return [np.ascontiguousarray(a[i]) for i in range(count)]


def unique_vertices(pts, res, zlo=0, zhi=None):
    """U of SURVEY 8d: vertices (with z in [zlo, zhi)) of the cells the points
    fall in, by the reference cell rule on a cubic grid over [-1, 1]^3.
    Untimed host pass."""
    h = 2.0 / (res - 1)
    zhi = res if zhi is None else zhi
    p = np.asarray(pts, dtype=np.float64)[:, :3]
    c = np.clip(np.floor((np.clip(p, -1.0, 1.0) + 1.0) / h).astype(np.int64), 0, res - 2)
    cells = np.unique((c[:, 2] * res + c[:, 1]) * res + c[:, 0])
    cz, r = np.divmod(cells, res * res)
    cy, cx = np.divmod(r, res)
    ids = []
    for dz in (0, 1):
        z = cz + dz
        keep = (z >= zlo) & (z < zhi)
        for dy in (0, 1):
            for dx in (0, 1):
                ids.append(((z[keep] * res + cy[keep] + dy) * res) + cx[keep] + dx)
    return int(np.unique(np.concatenate(ids)).size)


def traffic_from_profile(key="dram_bytes_per_launch"):
    """The fused kernel's DRAM bytes per launch (or its L2 hit rate) from the
    committed ncu capture (profiles/ncu_traffic.json, tools/ncu_traffic.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if key == "dram_bytes_per_launch":
            return d.get("k_brick_step", {}).get(key)
        ks = [v for k, v in d.get("kernels", {}).items() if k.startswith("k_brick_step")]
        return ks[-1].get(key) if ks else None
    except Exception:
        return None


# ---- reference CPU path (oracle/_ref: the reference's own sources) -------------------


def ref_train_threads(res):
    """total_loss keeps one dense fp64 gradient copy per thread (GradScratch,
    sdf_loss.cpp:96-103): cap the threads so the copies fit in ~1/3 of the
    available host memory (and at 64)."""
    vk = res ** 3 * 10
    budget = max(mem_available_bytes() // 3 - 4 * 8 * vk, 8 * vk)
    return int(max(1, min(os.cpu_count() or 1, 64, budget // (8 * vk))))


def ref_train_sample(wl, batches, steps, threads=None):
    """`steps` reference steps (tg::total_loss + tg::adam_step, zero init) on
    the workload's grid; returns (seconds, per-step terms, threads)."""
    from oracle.pyoracle import Loss, Reference, Spec
    W = WORKLOADS[wl]
    R = Reference()
    s = Spec(dim=3, res=(W["res"],) * 3, order=2)
    threads = threads or ref_train_threads(W["res"])
    _, terms, secs = R.train(s, None, np.array(batches, dtype=np.float64), Loss(), lr=W["lr"], threads=threads,
                             steps=steps)
    return secs, terms, threads


def cpu_baseline_train(wl, batches, steps=2):
    from oracle.pyoracle import reference_available
    if not reference_available():
        return None
    W = WORKLOADS[wl]
    need = 4 * 8 * W["res"] ** 3 * 10 * 1.6
    if mem_available_bytes() and mem_available_bytes() < need:
        return {"unavailable": f"host memory: {mem_available_bytes() / 1e9:.0f} GB available, the reference "
                               f"needs > {need / 1e9:.0f} GB for {wl}"}
    secs, terms, threads = ref_train_sample(wl, batches, steps)
    pts = steps * W["points"]
    return {"value": pts / secs, "unit": "points/s", "cores": threads, "kind": "reference",
            "sample": f"{steps} full {wl.upper()} steps ({pts} points) through tg::total_loss + tg::adam_step "
                      f"(oracle/_ref: unmodified reference sources, g++ -O3 -ffp-contract=off as its CMake build, "
                      f"no -march=native), threads={threads}",
            "seconds": secs, "loss_last": float(terms[-1, 0])}


def cpu_baseline_c1(steps=40):
    """C1 (BASELINE configs[0]: 2D 128^2 order 2, 65,536 uniform points of the
    circle-union-box target per step, lr 1e-2) through the reference's own
    tg::total_loss + tg::adam_step (oracle/_ref), all host threads, `steps`
    steps on two seeded batches from the package's host sampler."""
    from oracle.pyoracle import Loss, Reference, Spec, reference_available
    if not reference_available():
        return None
    import paper_2402_14415_b200 as tg
    batches = [tg.sample(tg.SHAPE_C1_2D, 2, 500 + i, 1 << 16) for i in range(2)]
    R = Reference()
    threads = int(min(os.cpu_count() or 1, 64))
    _, terms, secs = R.train(Spec(dim=2, res=(128, 128, 1), order=2), None, np.array(batches, dtype=np.float64),
                             Loss(), lr=1e-2, threads=threads, steps=steps)
    pts = steps * (1 << 16)
    return {"value": pts / secs, "unit": "points/s", "cores": threads, "kind": "reference",
            "sample": f"{steps} full C1 steps ({pts} points) through tg::total_loss + tg::adam_step "
                      f"(oracle/_ref, threads={threads})", "seconds": secs, "loss_last": float(terms[-1, 0])}


def stages_leg(device, hbm_peak, cpu=True):
    """SURVEY 8(f) rows on this GPU next to the reference's own code: upsample
    (128^3 -> 256^3 order 2), sample_grid_field (256^3 order-2 grid on a 256^3
    lattice) and the radiance photometric loss with density and SH gradients
    (128^3 grids, 2^16 rays x 64 samples). Device inputs resident, CUDA events
    after warm-up; algorithmic bytes: upsample 4K (old + new vertices), lattice
    4 B per value + 4K B per grid vertex (each read once). The reference
    (oracle/_ref, one thread) runs a bounded sample of each."""
    import ctypes as C
    import torch
    import paper_2402_14415_b200 as tg
    from paper_2402_14415_b200.radiance import _RO, make_rays
    dev = f"cuda:{device}"
    L = tg.lib()

    def timed(fn, reps=10):
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

    big = tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.1, seed=1, memory_cap_bytes=1 << 40)
    R = None
    if cpu:
        from oracle.pyoracle import Reference, Spec, reference_available
        R = Reference() if reference_available() else None
    out = {}
    # upsample
    a, b = 128, 256
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(a,) * 3, order=2), big, device=device)
    dst = tg.init_grid(tg.GridSpec(dim=3, resolution=(b,) * 3, order=2), tg.InitOptions(memory_cap_bytes=1 << 40),
                       device=device)
    ms = timed(lambda: tg._check(L.tgcu_grid_upsample(g.handle, dst.handle, tg.TGCU_ASYNC, None)))
    byt = 4 * 10 * (a ** 3 + b ** 3)
    up = {"grid": [a, b], "order": 2, "ms": ms, "achieved_gbs": byt / ms / 1e6, "frac": byt / ms / 1e6 / hbm_peak,
          "new_vertices_per_s": b ** 3 / (ms * 1e-3)}
    del g, dst
    if R is not None:
        sa, sb = 64, 128
        s = Spec(dim=3, res=(sa,) * 3, order=2)
        c = np.random.default_rng(1).normal(0.0, 0.1, s.V * s.K)
        t0 = time.perf_counter()
        R.upsample(s, c, (sb,) * 3)
        dt = time.perf_counter() - t0
        up["cpu_baseline"] = {"value": sb ** 3 / dt, "unit": "new vertices/s", "cores": 1, "kind": "reference",
                              "sample": f"tg::upsample {sa}^3 -> {sb}^3 order 2", "seconds": dt}
    out["upsample"] = up
    # lattice query
    gres, lat = 256, 256
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(gres,) * 3, order=2), big, device=device)
    vals = torch.empty(lat ** 3, dtype=torch.float32, device=dev)
    ms = timed(lambda: tg.sample_grid_field(g, (lat,) * 3, out=vals))
    byt = 4 * lat ** 3 + 4 * 10 * gres ** 3
    lq = {"grid": gres, "lattice": lat, "order": 2, "ms": ms, "achieved_gbs": byt / ms / 1e6,
          "frac": byt / ms / 1e6 / hbm_peak, "gvalues_per_s": lat ** 3 / ms / 1e6}
    del g, vals
    if R is not None:
        s = Spec(dim=3, res=(64,) * 3, order=2)
        c = np.random.default_rng(2).normal(0.0, 0.1, s.V * s.K)
        t0 = time.perf_counter()
        R.sample_grid_field(s, c, (128,) * 3)
        dt = time.perf_counter() - t0
        lq["cpu_baseline"] = {"value": 128 ** 3 / dt, "unit": "values/s", "cores": 1, "kind": "reference",
                              "sample": "tg::sample_grid_field, 64^3 order-2 grid, 128^3 lattice", "seconds": dt}
    out["lattice_query"] = lq
    # radiance photometric loss with gradients
    res, deg, n, ns = 128, 2, 1 << 16, 64
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(res,) * 3, order=2),
                     tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=1.0, seed=3), device=device)
    ss = tg.GridSpec(dim=3, resolution=(res,) * 3, order=0)
    gen = torch.Generator(device=dev).manual_seed(5)
    shc = torch.randn(res ** 3 * (deg + 1) ** 2 * 3, device=dev, generator=gen) * 0.5
    rng = np.random.default_rng(0)
    o = rng.uniform(-0.9, 0.9, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rays = torch.from_numpy(make_rays(o, d, 0.0, 1.0)).to(dev)
    gt = torch.rand((n, 3), device=dev, generator=gen)
    gd = torch.zeros(g.coeff_total(), device=dev)
    gs = torch.zeros_like(shc)
    ro = _RO(ns, 0, -10.0, (C.c_double * 3)(1.0, 1.0, 1.0), 0, 0)
    loss = C.c_double()
    spec = ss._c()
    ms = timed(lambda: tg._check(L.tgcu_photometric_loss(
        g.handle, C.byref(spec), deg, C.c_void_p(shc.data_ptr()), C.c_void_p(rays.data_ptr()),
        C.c_void_p(gt.data_ptr()), n, C.cast(C.pointer(ro), C.c_void_p), None, None, C.c_void_p(gd.data_ptr()),
        C.c_void_p(gs.data_ptr()), C.byref(loss), 0, None)), reps=5)
    rad = {"grid": res, "sh_degree": deg, "rays": n, "samples_per_ray": ns, "ms": ms,
           "gsamples_per_s": n * ns / ms / 1e6, "note": "loss + density and SH gradients (profiles/r02_rays_ncu.md)"}
    del g, shc, gd, gs
    if R is not None:
        m, r2 = 2048, 64
        ds = Spec(dim=3, res=(r2,) * 3, order=2)
        sss = Spec(dim=3, res=(r2,) * 3, order=0)
        dc = np.random.default_rng(3).normal(0.0, 1.0, ds.V * ds.K)
        sc = np.random.default_rng(4).normal(0.0, 0.5, sss.V * 3 * (deg + 1) ** 2)
        rr = {"origins": o[:m], "dirs": d[:m], "near": np.zeros(m), "far": np.ones(m), "gt": rng.random((m, 3))}
        t0 = time.perf_counter()
        R.photometric_loss(ds, dc, sss, deg, sc, rr, n_samples=ns, want_grad=True)
        dt = time.perf_counter() - t0
        rad["cpu_baseline"] = {"value": m * ns / dt, "unit": "samples/s", "cores": 1, "kind": "reference",
                               "sample": f"tg::photometric_loss with gradients, {m} rays x {ns} samples, "
                                         f"{r2}^3 grids", "seconds": dt}
    out["radiance"] = rad
    torch.cuda.empty_cache()
    return out


def cpu_baseline_query(order, pts_host):
    """The reference's query path (parallel_for + tg::eval, taylor_grid.cpp:197-203)
    on the C4 512^3 grid (built by the reference's init_grid, SmallUniform),
    over a bounded sample of the C4 points."""
    from oracle.pyoracle import Reference, Spec, reference_available
    if not reference_available():
        return None
    K = 4 if order == 1 else 10
    need = 512 ** 3 * K * 8 * 1.3
    if mem_available_bytes() and mem_available_bytes() < need:
        return {"unavailable": f"host memory: {mem_available_bytes() / 1e9:.0f} GB available, < {need / 1e9:.0f} GB"}
    threads = max(1, min(os.cpu_count() or 1, 64))
    R = Reference()
    s = Spec(dim=3, res=(512, 512, 512), order=order)
    _, secs = R.query_bench(s, pts_host, threads, epsilon=0.1, seed=7)
    return {"value": len(pts_host) / secs, "unit": "points/s", "cores": threads, "kind": "reference",
            "sample": f"{len(pts_host)} of the 2^26 C4 points (unsorted), tg::eval under tg::parallel_for on a "
                      f"512^3 order-{order} grid from tg::init_grid(SmallUniform, eps 0.1), threads={threads}",
            "seconds": secs}


def run_reference(args):
    """--impl reference: the reference CPU implementation on our arm's config
    (rank 0 only under torchrun; the other ranks exit without work). The
    reference process never imports this package (no libtgcu.so)."""
    rank = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    from oracle.pyoracle import reference_available
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtgref.so not built"}))
        return
    wl = args.workload or ("c2" if ws == 1 else "c3")
    W = WORKLOADS[wl]
    batches = reference_batches(wl, 1000)
    # warm-up probe (1 step), the rest of --warmup bounded to ~20 s of CPU work,
    # then a bounded number of timed steps (~60 s of CPU work)
    t1, _, threads = ref_train_sample(wl, batches, 1)
    warm = 1
    extra = int(max(0, min(args.warmup - 1, 20.0 // max(t1, 1e-3))))
    if extra:
        ref_train_sample(wl, batches, extra, threads)
        warm += extra
    steps = int(max(1, min(args.steps, 60.0 // max(t1, 1e-3))))
    secs, terms, _ = ref_train_sample(wl, batches, steps, threads)
    v = steps * W["points"] / secs
    sample = (f"{steps} full steps of the arm's config ({steps * W['points']} points, the arm's {NBATCH} batches "
              f"cycled), threads={threads} (bounded sample of --steps {args.steps})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 * secs / steps, "higher_is_better": True,
        "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": data_desc(wl), "config": workload_config(wl, ws),
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "loss_last": float(terms[-1, 0]),
    }))


def data_desc(wl):
    W = WORKLOADS[wl]
    tgt = "sphere samples" if W["shape"] == "sphere" else "procedural 64-primitive samples"
    return f"synthetic: seeded {tgt} (reference Rng mappings), {NBATCH} distinct batches cycled"


# ---- our arm --------------------------------------------------------------------------


def dist_setup():
    """One process per GPU (torchrun env). The device is bound before the
    process group so NCCL initialises on it. TGCU_DIST_BACKEND=gloo (tests
    only) runs the same flow with host-staged collectives, ranks wrapping onto
    the available devices. The process group is bench plumbing (barriers and
    the max over ranks of the timings); the slab step's own collectives run in
    libtgcu (SlabTrainer)."""
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group(os.environ.get("TGCU_DIST_BACKEND", "nccl"))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def count_unique_vertices(pts_dev, res):
    """U: vertices touched by a point set (untimed torch pass)."""
    import torch
    V = res[0] * res[1] * res[2]
    mark = torch.zeros(V, dtype=torch.bool, device=pts_dev.device)
    h = torch.tensor([2.0 / (r - 1) for r in res], dtype=torch.float64, device=pts_dev.device)
    for s0 in range(0, pts_dev.shape[0], 1 << 23):
        p = pts_dev[s0:s0 + (1 << 23)].double().clamp(-1, 1)
        c = torch.floor((p + 1.0) / h).long()
        for a in range(3):
            c[:, a].clamp_(0, res[a] - 2)
        base = c[:, 0] + res[0] * (c[:, 1] + res[1] * c[:, 2])
        for corner in range(8):
            off = (corner & 1) + ((corner >> 1) & 1) * res[0] + ((corner >> 2) & 1) * res[0] * res[1]
            mark[base + off] = True
    return int(mark.sum().item())


def query_leg(device, hbm_peak, reps=10, ws=1, rank=0, cpu=True):
    """C4: 512^3 forward-only query, orders 1 and 2, 2^26 uniform points,
    unsorted (binned inside the call) and brick-sorted (smem tile) kernels.
    With N ranks the grid is replicated and the points sharded (rank r takes
    the r-th contiguous N-th of the same seeded set; no collective); times are
    the max over ranks, throughput = all points / that time. Rank 0 at N=1
    also times the reference's eval on a bounded sample of the points."""
    import torch
    import paper_2402_14415_b200 as tg
    res = (512, 512, 512)
    n = 1 << 26
    full = torch.empty((n, 3), dtype=torch.float32, device=f"cuda:{device}")
    tg.sample_uniform_device(3, 4242, full)
    m = n // ws
    pts = full[rank * m:(rank + 1) * m] if ws > 1 else full
    spts = torch.empty_like(pts)
    vals = torch.empty(pts.shape[0], dtype=torch.float32, device=pts.device)
    st = torch.cuda.current_stream()
    out = {}
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    U = count_unique_vertices(full, res)
    cpu_pts = full[: 1 << 22].cpu().numpy() if (cpu and ws == 1 and rank == 0) else None
    del full
    offs = None
    for order in (1, 2):
        g = tg.init_grid(tg.GridSpec(dim=3, resolution=res, order=order),
                         tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.1, seed=7, memory_cap_bytes=1 << 40),
                         device=device)
        K = g.spec.coeffs_per_vertex()
        if offs is None:
            offs = torch.empty(tg.query_brick_codes(g) + 1, dtype=torch.int64, device=pts.device)
            tg.sort_points(g, pts, spts, None, offs)  # warm-up
            torch.cuda.synchronize()
            t0.record(st)
            tg.sort_points(g, pts, spts, None, offs)
            t1.record(st)
            torch.cuda.synchronize()
            out["sort_ms"] = max_over_ranks(t0.elapsed_time(t1), ws)
        alg = n * (4 * 3 + 4) + U * K * 4

        def run(mode):
            if mode == "unsorted":
                tg.eval_device(g, pts, vals, asynchronous=True)
            else:
                tg.eval_sorted(g, spts, offs, vals, asynchronous=True)

        for mode in ("unsorted", "sorted"):
            run(mode)  # warm-up
            torch.cuda.synchronize()
            barrier(ws)
            t0.record(st)
            for _ in range(reps):
                run(mode)
            t1.record(st)
            torch.cuda.synchronize()
            ms = max_over_ranks(t0.elapsed_time(t1) / reps, ws)
            gbs = alg / (ms * 1e-3) / 1e9
            out[f"o{order}_{mode}"] = {"gpts_per_s": n / (ms * 1e-3) / 1e9, "ms": ms, "achieved_gbs": gbs,
                                      "frac": gbs / hbm_peak}
        out[f"o{order}_sort_plus_sorted_ms"] = out["sort_ms"] + out[f"o{order}_sorted"]["ms"]
        g.close()
        if cpu_pts is not None:
            cb = cpu_baseline_query(order, cpu_pts)
            if cb is not None:
                out[f"o{order}_cpu_baseline"] = cb
    out["points"] = n
    out["sharding"] = f"grid replicated, points sharded over {ws} rank(s)" if ws > 1 else "single GPU"
    out["unique_vertices"] = U
    out["grid"] = list(res)
    out["coeffs"] = "0.1 N(0,1) from a counter hash (device init); the CPU sample's grid: reference SmallUniform"
    out["algorithmic_bytes"] = "N*(4D+4) + U*K*4 (SURVEY 8d B_q)"
    out["l2"] = "no flush: each call streams >= 2.1 GB of coefficients + 1 GB of points, > L2"
    del pts, spts, vals, offs
    torch.cuda.empty_cache()
    return out


def make_trainer(wl, ws, rank, dev):
    """(handle, step function, local host batches, spec) for this rank."""
    import paper_2402_14415_b200 as tg
    W = WORKLOADS[wl]
    spec = tg.GridSpec(dim=3, resolution=(W["res"],) * 3, order=2)
    cfg = tg.LossConfig()  # paper defaults
    opts = tg.InitOptions(memory_cap_bytes=1 << 40)
    if ws == 1:
        g = tg.init_grid(spec, opts, device=dev)
        g.adam_reset(tg.AdamConfig(lr=W["lr"]))

        def step(batch, sp, asynchronous=True):
            # device batches are uploaded and synchronized before use: input_ready
            # lets each step's binning overlap the previous brick kernel
            return tg.train_step(g, batch, cfg, asynchronous=asynchronous, stream=sp if asynchronous else None,
                                 input_ready=True)
        return g, step, None
    from paper_2402_14415_b200.slab import SlabTrainer
    trainer = SlabTrainer(spec, rank, ws, tg.AdamConfig(lr=W["lr"]), device=dev, opts=opts)

    def step(batch, sp, asynchronous=True):
        return trainer.step(batch, cfg, stream=sp, want_terms=not asynchronous, n_global=W["points"],
                            input_ready=True)
    return trainer.slab, step, trainer


def single_gpu_reference_value(wl, dev, host_batches, steps, warmup):
    """N>1: rank 0 times the whole workload on its own GPU first (the
    single-GPU point of the strong-scaling curve, same steps)."""
    import torch
    g, step, _ = make_trainer(wl, 1, 0, dev)
    db = [torch.from_numpy(b).to(f"cuda:{dev}") for b in host_batches]
    torch.cuda.synchronize()
    sp = torch.cuda.current_stream().cuda_stream
    for i in range(warmup):
        step(db[i % NBATCH], sp)
    g.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        step(db[i % NBATCH], sp)
    e1.record()
    torch.cuda.synchronize()
    g.sync()
    ms = e0.elapsed_time(e1) / steps
    g.close()
    del db
    torch.cuda.empty_cache()
    return {"value": WORKLOADS[wl]["points"] / (ms * 1e-3), "unit": "points/s", "ms_per_step": ms,
            "steps": steps, "note": "the same workload on rank 0's GPU alone, timed before the slab run"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=list(WORKLOADS),
                    help="default: c2 at N=1 (BASELINE configs[1]), c3 strong scaling at N>1 (configs[2])")
    ap.add_argument("--no-query", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1 / C3 / C5 step timings")
    ap.add_argument("--no-stages", action="store_true", help="skip the 8(f) legs (upsample, lattice, radiance)")
    ap.add_argument("--e2e-steps", type=int, default=500)
    ap.add_argument("--gen-batches", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--gen-seed", type=int, default=1000, help=argparse.SUPPRESS)
    ap.add_argument("--gen-count", type=int, default=NBATCH, help=argparse.SUPPRESS)
    ap.add_argument("--gen-out", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gen_batches:  # child of reference_batches: write the batches, nothing else
        np.save(args.gen_out, np.stack(make_batches(args.gen_batches, args.gen_seed, args.gen_count)))
        return
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(args.warmup, 3)

    ws, rank, local = dist_setup()
    wl = args.workload or ("c2" if ws == 1 else "c3")
    W = WORKLOADS[wl]
    import torch
    import paper_2402_14415_b200 as tg
    dev = local
    hbm_peak, peak_src = peaks()
    res = W["res"]
    K = 10
    npts_global = W["points"]
    # every rank builds the same seeded global batches
    host_global = make_batches(wl, 1000)
    single = None
    if ws > 1 and rank == 0:
        single = single_gpu_reference_value(wl, dev, host_global, min(args.steps, 200), args.warmup)
    barrier(ws)
    g, step, trainer = make_trainer(wl, ws, rank, dev)
    if trainer is not None:
        # data sharded by owner up front (outside the timed region): each rank
        # holds the points whose cells touch its slab; the loss keeps the
        # global 1/N (SURVEY 8e "bins points to their owning GPU")
        host_batches = [trainer.local_points(b) for b in host_global]
    else:
        host_batches = host_global
    dev_batches = [torch.from_numpy(b).to(f"cuda:{dev}") for b in host_batches]
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    torch.cuda.synchronize()

    for i in range(args.warmup):
        step(dev_batches[i % NBATCH], sp)
    g.sync()

    with ClockSampler(dev) as clocks:
        # ---- timed: K fused steps, inputs resident in HBM -------------------------
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        barrier(ws)
        torch.cuda.synchronize()
        l0 = tg.launch_count()
        # the brick kernel is timed live on every 8th step: event pairs around
        # every launch would cost the stream ~6 us per step
        g.profile_begin(every=8 if args.steps >= 64 else 1)
        ev0.record(stream)
        for i in range(args.steps):
            step(dev_batches[i % NBATCH], sp)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
        torch.cuda.synchronize()
        launches = tg.launch_count() - l0
        brick_ms, brick_n = g.profile_end()
        comm_prof = trainer.comm_profile() if trainer is not None else None
        last = g.sync()
        ms_total = max_over_ranks(ev0.elapsed_time(ev1), ws)
        ms_step = ms_total / args.steps

        # ---- e2e: host (pinned) samples in, LossTerms out, every step -------------
        # Single GPU: the pipelined C-ABI host path (TGCU_HOST|TGCU_ASYNC): each
        # step's H2D copy runs on the library's copy stream under the previous
        # step's kernels and each step's LossTerms are copied back to pinned
        # host memory. Slabs (N > 1): host samples, synchronous steps.
        pinned = [torch.from_numpy(b).pin_memory() for b in host_batches]
        ne = max(3, min(args.e2e_steps, args.steps))
        e2e_async = ws == 1
        for i in range(2 * NBATCH):  # every pinned buffer through the copy path twice
            step(pinned[i % NBATCH].numpy(), sp, asynchronous=e2e_async)
        g.sync()
        torch.cuda.synchronize()
        # E2E_WINDOWS back-to-back windows of ne steps, each timed whole (max
        # over ranks); the median window is reported, so one host stall (a
        # ~0.1 s scheduling hiccup against a ~0.16 s window) does not set it
        e2e_windows = []
        for _w in range(E2E_WINDOWS):
            barrier(ws)
            t0 = time.perf_counter()
            for i in range(ne):
                step(pinned[i % NBATCH].numpy(), sp, asynchronous=e2e_async)  # H2D inside, D2H of LossTerms
            e2e_last = g.sync()
            torch.cuda.synchronize()
            e2e_windows.append(max_over_ranks(time.perf_counter() - t0, ws))
        e2e_s = sorted(e2e_windows)[len(e2e_windows) // 2]
        barrier(ws)

        q = None
        if not args.no_query:
            q = query_leg(dev, hbm_peak, ws=ws, rank=rank, cpu=not args.no_cpu_baseline)

    clk = clocks.summary()
    value = npts_global * args.steps / (ms_total * 1e-3)  # whole job: one global batch per step
    kern_ms = brick_ms / max(brick_n, 1)
    per_rank_ms = [kern_ms]
    if ws > 1:  # per-GPU load imbalance of the fused kernel (report imbalance)
        import torch.distributed as dist
        per_rank_ms = [None] * ws
        dist.all_gather_object(per_rank_ms, kern_ms)
    vk_total = res ** 3 * K
    if ws == 1:
        vk_local, pts_local, zlo, zhi = vk_total, npts_global, 0, res
    else:  # this rank's kernel: its owned vertex planes and its local points
        vk_local = (g.z_own_hi - g.z_own_lo) * res * res * K
        pts_local = int(sum(b.shape[0] for b in host_batches) / len(host_batches))
        zlo, zhi = g.z_own_lo, g.z_own_hi
    # SURVEY 8d B_t = N(4D+4) + U*K*4 + 2*U*K*4 + 8*V*K*4 for this rank's kernel:
    # its points, U counted exactly (untimed host pass) over its owned vertices
    u_local = float(np.mean([unique_vertices(b, res, zlo, zhi) for b in host_batches]))
    bt_local = 16 * pts_local + 3 * u_local * K * 4 + 32 * vk_local
    achieved = bt_local / (kern_ms * 1e-3) / 1e9
    kern_bytes = 24 * vk_local + 16 * pts_local  # the fused kernel's own compulsory bytes (grad never stored)
    u_global = float(np.mean([unique_vertices(b, res) for b in host_global])) if ws > 1 else u_local
    survey_bytes = 16 * npts_global + 3 * u_global * K * 4 + 32 * vk_total
    line = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None, "dtype": "f32",
        "data": data_desc(wl), "config": workload_config(wl, ws),
        "l2": f"no flush: every step streams p,m,v ({24 * vk_local / 1e6:.0f} MB per GPU) + points, > the "
              f"{torch.cuda.get_device_properties(dev).L2_cache_size / 2**20:.0f} MiB L2 (cudaDevAttrL2CacheSize)",
        "roofline": {"bound": "hbm", "kernel": "k_brick_step<3,2,...> (fused loss+backward+TV+Adam)",
                     "achieved": achieved, "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic_from_profile() if wl == "c2" and ws == 1 else None,
                     "frac_nominal_8tbs": achieved / 8000.0,
                     "l2_hit_pct": traffic_from_profile("l2_hit_pct") if wl == "c2" and ws == 1 else None,
                     "algorithmic_bytes_per_launch": bt_local,
                     "algorithmic_bytes_def": "SURVEY 8d B_t = N*(4D+4) + 3*U*K*4 + 8*V*K*4 with U = unique vertices "
                                              "touched, counted exactly per batch (mean over the batches)"
                                              + ("" if ws == 1 else "; rank 0's local points and owned slab"),
                     "unique_vertices": u_local,
                     "fused_compulsory": {"bytes": kern_bytes,
                                          "def": "24 B/coeff (p,m,v read+write fp32; the fused step never stores "
                                                 "the gradient) + 16 B/point",
                                          "achieved": kern_bytes / (kern_ms * 1e-3) / 1e9,
                                          "frac": kern_bytes / (kern_ms * 1e-3) / 1e9 / hbm_peak},
                     "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / ms_step,
                     "step_frac_survey_bytes": survey_bytes / (ms_step * 1e-3) / 1e9 / hbm_peak / ws},
        "e2e": {"value": npts_global * ne / e2e_s, "unit": "points/s",
                "h2d_bytes_per_step": int(16 * ws * sum(b.shape[0] for b in host_batches) / len(host_batches)),
                "d2h_bytes_per_step": 32 * ws,
                "api": ("tgcu_train_step(TGCU_HOST|TGCU_ASYNC): pipelined H2D on a copy stream, per-step LossTerms "
                        "D2H to pinned memory" if ws == 1 else "SlabTrainer.step with host samples, synchronous"),
                "loss_last": e2e_last.total, "steps_per_window": ne,
                "window_points_per_s": [round(npts_global * ne / w) for w in e2e_windows],
                "statistic": f"median of {E2E_WINDOWS} windows"},
        "gpu_launches": int(launches),
        "clocks": clk,
        "loss_last": last.total,
    }
    if ws > 1:
        line["per_rank_kernel_ms"] = per_rank_ms
        line["kernel_imbalance_max_over_mean"] = max(per_rank_ms) / (sum(per_rank_ms) / ws)
        line["halo"] = ("fused: boundary planes stored into the neighbours' halo by the brick kernel (peer memory)"
                        if getattr(trainer, "fused_halo", False) else "NCCL send/recv of the boundary planes")
        line["collectives"] = getattr(trainer, "backend", None)
        # per-rank collective phase of the profiled steps: all-reduce of the
        # loss partials and the halo exchange (0 when the brick kernel stores
        # the planes into the neighbours), ms per step
        import torch.distributed as dist
        cp = [None] * ws
        ar, hx, nst = comm_prof
        dist.all_gather_object(cp, (ar / max(nst, 1), hx / max(nst, 1)))
        line["per_rank_allreduce_ms"] = [c[0] for c in cp]
        line["per_rank_halo_exchange_ms"] = [c[1] for c in cp]
        if single is not None:
            line["single_gpu"] = single
    if q is not None:
        line["query"] = q
    if rank == 0 and ws == 1 and not args.no_configs:
        # BASELINE configs C1 (2D 128^2, parity config), C3 (256^3, 2^21 pts) and C5 (512^3, 2^23 pts,
        # 90% near-surface) on this GPU: step time and fraction of the HBM roofline
        # (tools/bench_configs.py), each with a bounded reference CPU sample
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_configs
        with ClockSampler(dev) as cclk:
            line["larger_configs"] = [bench_configs.run(c, 30, 5) for c in ("c1", "c3", "c5", "c2det")]
        line["larger_configs_clocks"] = cclk.summary()
        if not args.no_cpu_baseline:
            for ent in line["larger_configs"]:
                if ent["config"] == "c1":
                    ent["cpu_baseline"] = cpu_baseline_c1()
                if ent["config"] in ("c3", "c5"):
                    ent["cpu_baseline"] = cpu_baseline_train(ent["config"], make_batches(ent["config"], 500, 2),
                                                             steps=1)
    if rank == 0 and ws == 1 and not args.no_stages:
        line["stages"] = stages_leg(dev, hbm_peak, cpu=not args.no_cpu_baseline)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline_train(wl, host_batches)
        if cb is not None:
            line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
