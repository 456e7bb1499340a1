"""e2e diagnosis: host issue time vs device time of pipelined host-input C2 steps."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def gpu_local_cpus(dev=0):
    """CPUs on the GPU's NUMA node (NVML CPU affinity mask)."""
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(dev)
    words = pynvml.nvmlDeviceGetCpuAffinity(h, 64)
    cpus = [64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
    pynvml.nvmlShutdown()
    return cpus


def main():
    import torch
    if "--affinity" in sys.argv:
        cpus = gpu_local_cpus()
        os.sched_setaffinity(0, cpus)
        print(f"bound to {len(cpus)} GPU-local cpus")
    import paper_2402_14415_b200 as tg
    spec = tg.GridSpec(dim=3, resolution=(128,) * 3, order=2)
    g = tg.init_grid(spec)
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    hb = [torch.from_numpy(tg.sample(tg.SHAPE_SPHERE, 3, 1000 + i, 1 << 20, near_frac=0.5, sigma=0.01,
                                     param0=0.6)).pin_memory() for i in range(4)]
    arrs = [h.numpy() for h in hb]
    cfg = tg.LossConfig()
    for i in range(10):
        tg.train_step(g, arrs[i % 4], cfg, asynchronous=True)
    g.sync()
    n = 300
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    for i in range(n):
        tg.train_step(g, arrs[i % 4], cfg, asynchronous=True)
    t_issue = time.perf_counter() - t0
    e1.record()
    g.sync()
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t0
    print(f"host issue {t_issue / n * 1e3:.3f} ms/step, wall {t_wall / n * 1e3:.3f} ms/step, "
          f"legacy-stream events {e0.elapsed_time(e1) / n:.3f} ms/step, e2e {n * (1 << 20) / t_wall / 1e9:.2f} Gpts/s")
    # copies alone (no compute): the same 16 MB per step through the copy path
    d = torch.empty_like(hb[0], device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        h = hb[i % 4]
        m = h.shape[0] // 2
        with torch.cuda.stream(s1):
            d[:m].copy_(h[:m], non_blocking=True)
        with torch.cuda.stream(s2):
            d[m:].copy_(h[m:], non_blocking=True)
    torch.cuda.synchronize()
    print(f"copies alone {(time.perf_counter() - t0) / n * 1e3:.3f} ms/step")


if __name__ == "__main__":
    main()
