"""k_eval_direct vs point grouping on the C4 query (512^3, 2^26 points).

Times the direct (per-point L2/HBM gather) eval on uniform points in four
orders: as drawn, grouped by superbrick (64^3-cell Morton blocks, what one
9-bit partition pass gives), grouped by 32^3-cell blocks, and grouped by brick
(8^3 cells); beside them the binned path (two-pass partition + smem brick
tiles) on the drawn order. Answers whether one partition pass plus the direct
gather (L2 reuse inside a superbrick) beats the two-pass binned query.
Run: TGCU_QUERY_DIRECT=1 python tools/query_grouping.py [order]
(the env var only changes which kernel the unsorted calls reach).
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def spread3(v):
    import torch
    out = torch.zeros_like(v)
    for b in range(10):
        out |= ((v >> b) & 1) << (3 * b)
    return out


def timed(fn, reps=5):
    import torch
    for _ in range(2):
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
    import torch
    import paper_2402_14415_b200 as tg
    order = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    mode = os.environ.get("QG_MODE", "direct")
    g = tg.init_grid(tg.GridSpec(dim=3, resolution=(512,) * 3, order=order),
                     tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.1, seed=7, memory_cap_bytes=1 << 40))
    n = 1 << 26
    pts = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    tg.sample_uniform_device(3, 4242, pts)
    vals = torch.empty(n, dtype=torch.float32, device="cuda")
    res = {"order": order, "mode": mode}
    if mode == "binned":
        res["binned_ms"] = timed(lambda: tg.eval_device(g, pts, vals, asynchronous=True))
    else:
        cell = ((pts + 1.0) * (511 / 2.0)).floor().clamp(0, 510).to(torch.int64)
        ref = None
        for name, shift in (("drawn", None), ("sb64", 6), ("blk32", 5), ("brick8", 3)):
            if shift is None:
                q = pts
            else:
                c = cell >> shift
                key = spread3(c[:, 0]) | (spread3(c[:, 1]) << 1) | (spread3(c[:, 2]) << 2)
                idx = torch.sort(key, stable=True).indices
                q = pts[idx].contiguous()
                del key, idx, c
            res[name + "_ms"] = timed(lambda: tg.eval_device(g, q, vals, asynchronous=True))
            if shift is None:
                ref = vals.clone()
            del q
        res["direct_matches_binned_check"] = "n/a"
    print(json.dumps(res))


if __name__ == "__main__":
    if os.environ.get("QG_CHILD"):
        main()
    else:
        env = dict(os.environ, QG_CHILD="1")
        for order in (1, 2):
            for mode, direct in (("binned", "0"), ("direct", "1")):
                subprocess.run([sys.executable, __file__, str(order)],
                               env=dict(env, QG_MODE=mode, TGCU_QUERY_DIRECT=direct), check=True)
