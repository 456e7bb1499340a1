"""Benchmark of the TaylorGrid query-and-optimise hot path on B200.

Default workload (BASELINE.json configs[1], "C2"): 3D 128^3 grid, order 2
(10 fp32 coefficients per vertex, zero init), target = analytic sphere r=0.6,
2^20 points per step (50% uniform in the cube, 50% near-surface: sphere point
+ N(0, 0.01) per axis), paper loss (lambda1=1e-4 reuse-batch, lambda2=2e-5,
k=50, weighting on), Adam lr 1e-2. A step = zero grad -> total_loss -> finite
check -> adam_step (one run_schedule iteration), executed by the fused device
pipeline (tgcu_train_step). Metric: train points/s.

Extra keys: roofline (fused brick kernel, HBM), cpu_baseline (the reference's
own CPU code, oracle/_ref, on this host), e2e (through the C ABI with host
buffers), query (C4: 512^3 forward-only query, unsorted and brick-sorted).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

RES = (128, 128, 128)
ORDER = 2
NPTS = 1 << 20
NBATCH = 4
LR = 1e-2
WORKLOAD = ("C2: 3D 128^3 order-2 TaylorGrid SDF fit, sphere r=0.6, 2^20 points/step "
            "(50% uniform / 50% near-surface sigma=0.01), paper loss (lambda1=1e-4 reuse-batch, "
            "lambda2=2e-5 TV, k=50), Adam lr 1e-2; step = zero-grad + total_loss + finite check + adam_step")
METRIC = "TaylorGrid train points/s (fwd+bwd+Adam) & query Mpts/s; % of HBM roofline"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


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


def dist_setup():
    """One process per GPU (torchrun env). The device is bound before the
    process group so NCCL initialises on it. TGCU_DIST_BACKEND=gloo (tests
    only) runs the same flow with host-staged collectives, ranks wrapping onto
    the available devices."""
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


def make_stacked_batches(ws, seed0, n=NPTS, count=NBATCH):
    """Weak scaling: N copies of the C2 problem stacked along z, one per rank's
    slab of 128 vertex planes (C2 spacing h = 2/127). Slab r's points are a C2
    batch (50 % uniform, 50 % near its sphere of radius 0.6) shifted by
    128 r h, its uniform half stretched over the slab's full thickness so the
    shared boundary cell layers get points; gt = the exact distance to the
    union of the spheres (nearest of slabs r-1, r, r+1), from the fp32
    coordinates."""
    import numpy as np
    import paper_2402_14415_b200 as tg
    h = 2.0 / (RES[2] - 1)
    th = RES[2] * h
    n_uni = n - int(np.floor(n * 0.5))
    out = []
    for i in range(count):
        parts = []
        for r in range(ws):
            b = tg.sample(tg.SHAPE_SPHERE, 3, seed0 + 7919 * r + i, n, near_frac=0.5, sigma=0.01,
                          param0=0.6).astype(np.float64)
            b[:n_uni, 2] = -1.0 + (b[:n_uni, 2] + 1.0) * (th / 2.0)
            b[:, 2] += 128 * r * h
            p = b[:, :3].astype(np.float32).astype(np.float64)
            gt = np.full(n, np.inf)
            for k in (r - 1, r, r + 1):
                if 0 <= k < ws:
                    c = np.array([0.0, 0.0, 128 * k * h])
                    gt = np.minimum(gt, np.linalg.norm(p - c, axis=1) - 0.6)
            parts.append(np.concatenate([p, gt[:, None]], 1).astype(np.float32))
        out.append(np.ascontiguousarray(np.concatenate(parts)))
    return out


def make_batches(seed0, n=NPTS, count=NBATCH):
    import paper_2402_14415_b200 as tg
    return [tg.sample(tg.SHAPE_SPHERE, 3, seed0 + i, n, near_frac=0.5, sigma=0.01, param0=0.6) for i in range(count)]


def unique_vertices(pts, res, zlo=0, zhi=None):
    """U of SURVEY 8d: vertices (with z in [zlo, zhi)) of the cells the points
    fall in, by the reference cell rule on the bench grid (spacing 2/127 on
    every axis, origin -1). Untimed host pass."""
    h = 2.0 / (RES[0] - 1)
    zhi = res[2] if zhi is None else zhi
    p = np.asarray(pts, dtype=np.float64)[:, :3]
    c = np.floor((p + 1.0) / h).astype(np.int64)
    for a in range(3):
        np.clip(c[:, a], 0, res[a] - 2, out=c[:, a])
    cells = np.unique((c[:, 2] * res[1] + c[:, 1]) * res[0] + c[:, 0])
    cz, r = np.divmod(cells, res[0] * res[1])
    cy, cx = np.divmod(r, res[0])
    ids = []
    for dz in (0, 1):
        z = cz + dz
        keep = (z >= zlo) & (z < zhi)
        for dy in (0, 1):
            for dx in (0, 1):
                ids.append(((z[keep] * res[1] + cy[keep] + dy) * res[0]) + cx[keep] + dx)
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


def cpu_baseline(batches, steps_cap=2):
    """The reference's own CPU path (oracle/_ref) on this host: bounded sample."""
    from oracle.pyoracle import Loss, Reference, Spec, reference_available
    if not reference_available():
        return None
    R = Reference()
    threads = max(1, min(os.cpu_count() or 1, 64))
    s = Spec(dim=3, res=RES, order=ORDER)
    b = np.array([x.astype(np.float64) for x in batches[:steps_cap]])
    _, terms, secs = R.train(s, np.zeros(s.V * s.K), b, Loss(), lr=LR, threads=threads)
    pts = steps_cap * NPTS
    return {"value": pts / secs, "unit": "points/s", "cores": threads, "kind": "reference",
            "sample": f"{steps_cap} full C2 steps ({pts} points) through tg::total_loss + tg::adam_step "
                      f"(oracle/_ref, unmodified reference sources, -O3), threads={threads}",
            "seconds": secs, "loss_last": float(terms[-1, 0])}


def run_reference(args):
    """--impl reference: the reference CPU implementation on the same config."""
    ws, rank, _ = dist_setup()
    try:
        if rank == 0:
            _run_reference_rank0(args, ws)
    finally:
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


def _run_reference_rank0(args, ws):
    from oracle.pyoracle import Loss, Reference, Spec, reference_available
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtgref.so not built"}))
        return
    import paper_2402_14415_b200 as tg  # host sampler only (same inputs as our arm)
    R = Reference()
    # our arm's config: C2 (N = 1) or N stacked C2 slabs (weak scaling, N > 1)
    res = (RES[0], RES[1], RES[2] * ws)
    s = Spec(dim=3, res=res, order=ORDER, extent=(2.0, 2.0, (res[2] - 1) * 2.0 / (RES[2] - 1)))
    npts = NPTS * ws
    # the reference keeps a dense fp64 gradient copy per thread: cap threads at ~16 GB of copies
    threads = max(1, min(os.cpu_count() or 1, 64, int(16e9 // (8 * s.V * s.K))))
    batches = [b.astype(np.float64) for b in
               (make_batches(1000, count=2) if ws == 1 else make_stacked_batches(ws, 1000, count=2))]
    # warm-up: a one-step probe, then the rest of --warmup (bounded to ~20 s of
    # CPU work); then a bounded number of timed steps (~60 s of CPU work)
    _, _, t1 = R.train(s, np.zeros(s.V * s.K), np.array(batches[:1]), Loss(), lr=LR, threads=threads)
    warm = 1
    extra = int(max(0, min(args.warmup - 1, 20.0 // max(t1, 1e-3))))
    if extra:
        R.train(s, np.zeros(s.V * s.K), np.array([batches[i % len(batches)] for i in range(extra)]), Loss(), lr=LR,
                threads=threads)
        warm += extra
    steps = int(max(1, min(args.steps, 60.0 // max(t1, 1e-3))))
    seq = np.array([batches[i % len(batches)] for i in range(steps)])
    _, terms, secs = R.train(s, np.zeros(s.V * s.K), seq, Loss(), lr=LR, threads=threads)
    v = steps * npts / secs
    sample = (f"{steps} full steps of the arm's config ({steps * npts} points), threads={threads} "
              f"(bounded sample of --steps {args.steps})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 * secs / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded sphere samples)",
        "config": {"workload": WORKLOAD if ws == 1 else f"C2 per GPU, {ws} C2 slabs stacked in z; " + WORKLOAD,
                   "grid": list(res), "order": ORDER, "points_per_step": npts},
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "loss_last": float(terms[-1, 0]),
    }))


def count_unique_vertices(pts_dev, res, order_K):
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


def query_leg(device, hbm_peak, reps=10, ws=1, rank=0):
    """C4: 512^3 forward-only query, orders 1 and 2, 2^26 uniform points,
    unsorted (binned inside the call) and brick-sorted (smem tile) kernels.
    With N ranks the grid is replicated and the points sharded (rank r takes
    the r-th contiguous N-th of the same seeded set; no collective); times are
    the max over ranks, throughput = all points / that time."""
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
    U = count_unique_vertices(full, res, 1)
    del full
    offs = None
    for order in (1, 2):
        g = tg.init_grid(tg.GridSpec(dim=3, resolution=res, order=order),
                         tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.1, seed=7, memory_cap_bytes=1 << 40),
                         device=device)
        K = g.spec.coeffs_per_vertex()
        if offs is None:
            offs = torch.empty(tg.query_brick_codes(g) + 1, dtype=torch.int64, device=pts.device)
            tg.sort_points(g, pts, spts, None, offs)  # warm-up: stream-pool growth, CUB module load
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
        g.close()
    out["points"] = n
    out["sharding"] = f"grid replicated, points sharded over {ws} rank(s)" if ws > 1 else "single GPU"
    out["unique_vertices"] = U
    out["grid"] = list(res)
    out["algorithmic_bytes"] = "N*(4D+4) + U*K*4 (SURVEY 8d B_q)"
    del pts, spts, vals, offs
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-query", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C3 / C5 step timings")
    ap.add_argument("--e2e-steps", type=int, default=500)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(args.warmup, 3)

    ws, rank, local = dist_setup()
    import torch
    import paper_2402_14415_b200 as tg
    torch.cuda.set_device(local)
    dev = local
    hbm_peak, peak_src = peaks()

    # N = 1: C2. N > 1: weak scaling, N C2 slabs stacked in z (make_stacked_batches).
    res = (RES[0], RES[1], RES[2] * ws)
    spec = tg.GridSpec(dim=3, resolution=res, order=ORDER,
                       extent=(2.0, 2.0, (res[2] - 1) * 2.0 / (RES[2] - 1)))
    K = spec.coeffs_per_vertex()
    VK = spec.coeff_total()
    cfg = tg.LossConfig()  # paper defaults
    npts_global = NPTS * ws
    # every rank builds the same seeded global batches
    host_batches = make_batches(1000) if ws == 1 else make_stacked_batches(ws, 1000)
    dev_batches = [torch.from_numpy(b).to(f"cuda:{dev}") for b in host_batches]
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    if ws == 1:
        g = tg.init_grid(spec, device=dev)
        g.adam_reset(tg.AdamConfig(lr=LR))

        def step(batch, asynchronous=True):
            # device batches are uploaded and synchronized before use: input_ready
            # lets each step's binning overlap the previous brick kernel
            return tg.train_step(g, batch, cfg, asynchronous=asynchronous, stream=None if not asynchronous else sp,
                                 input_ready=True)
    else:
        # weak scaling: rank r owns the r-th stacked C2 slab (16 brick layers;
        # owner computes; NCCL all-reduce of loss partials + halo planes)
        from paper_2402_14415_b200.slab import SlabTrainer
        trainer = SlabTrainer(spec, rank, ws, tg.AdamConfig(lr=LR), device=dev)
        g = trainer.slab

        # data sharded by owner up front (outside the timed region): each rank
        # holds the points whose cells touch its slab; the loss keeps the
        # global 1/N (SURVEY 8e "bins points to their owning GPU")
        local_host = [trainer.local_points(b) for b in host_batches]
        dev_batches = [torch.from_numpy(b).to(f"cuda:{dev}") for b in local_host]
        host_batches = local_host

        def step(batch, asynchronous=True):
            return trainer.step(batch, cfg, stream=sp, want_terms=not asynchronous, n_global=npts_global,
                                input_ready=True)

    for i in range(args.warmup):
        step(dev_batches[i % NBATCH])
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
            step(dev_batches[i % NBATCH])
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
        torch.cuda.synchronize()
        launches = tg.launch_count() - l0
        brick_ms, brick_n = g.profile_end()
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
            step(pinned[i % NBATCH].numpy(), asynchronous=e2e_async)
        g.sync()
        torch.cuda.synchronize()
        barrier(ws)
        t0 = time.perf_counter()
        for i in range(ne):
            step(pinned[i % NBATCH].numpy(), asynchronous=e2e_async)  # H2D inside, D2H of LossTerms
        e2e_last = g.sync()
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, ws)
        barrier(ws)

        q = None
        if not args.no_query:
            q = query_leg(dev, hbm_peak, ws=ws, rank=rank)

    clk = clocks.summary()
    value = npts_global * args.steps / (ms_total * 1e-3)  # whole job: one global batch per step
    kern_ms = brick_ms / max(brick_n, 1)
    per_rank_ms = [kern_ms]
    if ws > 1:  # per-GPU load imbalance of the fused kernel (report imbalance)
        import torch.distributed as dist
        per_rank_ms = [None] * ws
        dist.all_gather_object(per_rank_ms, kern_ms)
    if ws == 1:
        vk_local, pts_local = VK, NPTS
    else:  # this rank's kernel: its owned vertex planes and its local points
        vk_local = (g.z_own_hi - g.z_own_lo) * RES[0] * RES[1] * K
        pts_local = int(sum(b.shape[0] for b in host_batches) / len(host_batches))
    # SURVEY 8d B_t = N(4D+4) + U*K*4 + 2*U*K*4 + 8*V*K*4 for this rank's kernel:
    # its points, U counted exactly (untimed host pass) over its owned vertices
    if ws == 1:
        zlo, zhi = 0, res[2]
    else:
        zlo, zhi = g.z_own_lo, g.z_own_hi
    u_local = float(np.mean([unique_vertices(b, res, zlo, zhi) for b in host_batches]))
    bt_local = 16 * pts_local + 3 * u_local * K * 4 + 32 * vk_local
    achieved = bt_local / (kern_ms * 1e-3) / 1e9
    kern_bytes = 24 * vk_local + 16 * pts_local  # the fused kernel's own compulsory bytes (grad never stored)
    survey_bytes = 16 * npts_global + 3 * (u_local * ws) * K * 4 + 32 * VK  # whole step (U ~ per-rank U x N)
    line = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: seeded sphere samples (reference Rng mappings), 4 distinct batches cycled",
        "config": {"workload": WORKLOAD if ws == 1 else
                   (f"C2 per GPU, weak scaling: {ws} C2 slabs stacked in z (grid 128x128x{128 * ws}, "
                    f"{ws} x 2^20 points/step, sphere per slab, owner-sharded batch); " + WORKLOAD),
                   "grid": list(res), "order": ORDER, "points_per_step": npts_global,
                   "parallelism": f"z-slab x{ws} (owner computes, NCCL all-reduce + halo planes)" if ws > 1
                   else "single GPU",
                   "l2": f"no flush: every step streams p,m,v ({24 * vk_local / 1e6:.0f} MB per GPU) + points, > the "
                         f"{torch.cuda.get_device_properties(dev).L2_cache_size / 2**20:.0f} MiB L2 "
                         f"(cudaDevAttrL2CacheSize)"},
        "roofline": {"bound": "hbm", "kernel": "k_brick_step<3,2,true> (fused loss+backward+TV+Adam)",
                     "achieved": achieved, "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic_from_profile(),
                     "frac_nominal_8tbs": achieved / 8000.0, "l2_hit_pct": traffic_from_profile("l2_hit_pct"),
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
                     "step_frac_survey_bytes": survey_bytes / (ms_step * 1e-3) / 1e9 / hbm_peak},
        "e2e": {"value": npts_global * ne / e2e_s, "unit": "points/s",
                "h2d_bytes_per_step": int(16 * ws * sum(b.shape[0] for b in host_batches) / len(host_batches)),
                "d2h_bytes_per_step": 32,
                "api": ("tgcu_train_step(TGCU_HOST|TGCU_ASYNC): pipelined H2D on a copy stream, per-step LossTerms "
                        "D2H to pinned memory" if ws == 1 else "SlabTrainer.step with host samples, synchronous"),
                "loss_last": e2e_last.total},
        "gpu_launches": int(launches),
        "clocks": clk,
        "loss_last": last.total,
    }
    if ws > 1:
        line["per_rank_kernel_ms"] = per_rank_ms
        line["kernel_imbalance_max_over_mean"] = max(per_rank_ms) / (sum(per_rank_ms) / ws)
        line["halo"] = ("fused: boundary planes stored into the neighbours' halo by the brick kernel (peer memory)"
                        if getattr(trainer, "fused_halo", False) else "NCCL send/recv of the boundary planes")
    if q is not None:
        line["query"] = q
    if rank == 0 and ws == 1 and not args.no_configs:
        # BASELINE configs C1 (2D 128^2, parity config), C3 (256^3, 2^21 pts) and C5 (512^3, 2^23 pts,
        # 90% near-surface) on this GPU:
        # step time and fraction of the HBM roofline (tools/bench_configs.py)
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools"))
        import bench_configs
        with ClockSampler(dev) as cclk:
            line["larger_configs"] = [bench_configs.run(c, 30, 5) for c in ("c1", "c3", "c5")]
        line["larger_configs_clocks"] = cclk.summary()
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(host_batches)
        if cb is not None:
            line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
