"""C1 small-grid steps captured into a CUDA graph (timing experiment: the
captured steps replay with the Adam t and trace slots of the capture, so the
numerics of replays are not a training run): device time per step without
the per-call host cost, next to the same steps issued call by call.

    python tools/c1_graph.py [--steps-per-graph 100] [--replays 40]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_14415_b200 as tg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps-per-graph", type=int, default=100)
    ap.add_argument("--replays", type=int, default=40)
    a = ap.parse_args()
    import torch
    dev = [torch.from_numpy(tg.sample(tg.SHAPE_C1_2D, 2, 500 + i, 1 << 16)).cuda() for i in range(2)]
    cfg = tg.LossConfig()
    g = tg.init_grid(tg.GridSpec(dim=2, resolution=(128, 128, 1), order=2))
    g.adam_reset(tg.AdamConfig(lr=1e-2))
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    with torch.cuda.stream(s):
        for i in range(200):
            tg.train_step(g, dev[i % 2], cfg, asynchronous=True, input_ready=True, stream=sp)
    torch.cuda.synchronize()
    # call by call on the same stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = a.steps_per_graph * a.replays
    with torch.cuda.stream(s):
        e0.record(s)
        for i in range(n):
            tg.train_step(g, dev[i % 2], cfg, asynchronous=True, input_ready=True, stream=sp)
        e1.record(s)
    torch.cuda.synchronize()
    print(f"calls: {1e3 * e0.elapsed_time(e1) / n:.2f} us/step over {n} steps", flush=True)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for i in range(a.steps_per_graph):
            tg.train_step(g, dev[i % 2], cfg, asynchronous=True, input_ready=True, stream=sp)
    torch.cuda.synchronize()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(a.replays):
            graph.replay()
        e1.record(s)
    torch.cuda.synchronize()
    print(f"graph: {1e3 * e0.elapsed_time(e1) / n:.2f} us/step over {n} steps "
          f"({a.replays} replays of {a.steps_per_graph})", flush=True)


if __name__ == "__main__":
    main()
