"""A/B of TGCU_QP_FUSE_H2 (pass-2 tile histograms counted by the pass-1
scatter vs a histogram pass over the pass-1 records) on the C4 query:
512^3, 2^26 uniform points; binned eval o1/o2 (with gradients for o2) and
tgcu_sort_points. Each arm runs in a child process (the knob is read once);
values, gradients, the brick offsets and the sorted point multiset must be
identical across arms. Run: python tools/qp_fuse_ab.py [TGCU_QP_FUSE_H2|TGCU_QP_LUT]
(TGCU_QP_LUT: a table-driven Morton spread in the pass-1 histogram, measured
neutral in profiles/r02_qp_lut_ab.jsonl and removed again; the knob is inert now).
"""
import hashlib
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, reps=10):
    import torch
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


def digest(t):
    return hashlib.sha1(t.contiguous().cpu().numpy().tobytes()).hexdigest()[:16]


def child():
    import torch
    import paper_2402_14415_b200 as tg
    n = 1 << 26
    pts = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    tg.sample_uniform_device(3, 4242, pts)
    out = {"fuse_h2": os.environ.get("TGCU_QP_FUSE_H2", "0"), "lut": os.environ.get("TGCU_QP_LUT", "0")}
    for order in (1, 2):
        g = tg.init_grid(tg.GridSpec(dim=3, resolution=(512,) * 3, order=order),
                         tg.InitOptions(mode=tg.InitMode.HashGaussian, epsilon=0.1, seed=7, memory_cap_bytes=1 << 40))
        vals = torch.empty(n, dtype=torch.float32, device="cuda")
        grads = torch.empty((n, 3), dtype=torch.float32, device="cuda") if order == 2 else None
        out[f"o{order}_binned_ms"] = timed(lambda: tg.eval_device(g, pts, vals, grads, asynchronous=True))
        out[f"o{order}_vals"] = digest(vals)
        if grads is not None:
            out[f"o{order}_grads"] = digest(grads)
        if order == 2:
            srt = torch.empty_like(pts)
            perm = torch.empty(n, dtype=torch.int64, device="cuda")
            offs = torch.empty(tg.query_brick_codes(g) + 1, dtype=torch.int64, device="cuda")
            out["sort_ms"] = timed(lambda: tg.sort_points(g, pts, srt, perm, offs), reps=5)
            out["sort_offsets"] = digest(offs)
            out["sort_perm_sum"] = int(perm.sum().item())
            out["sort_gather_ok"] = bool(torch.equal(pts[perm], srt))
        del g
        torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if os.environ.get("QP_CHILD"):
        child()
    else:
        res = []
        for arm in ("0", "1", "0", "1"):
            knob = sys.argv[1] if len(sys.argv) > 1 else "TGCU_QP_FUSE_H2"
            env = dict(os.environ, QP_CHILD="1", TGCU_QP_FUSE_H2="0", TGCU_QP_LUT="0")
            env[knob] = arm
            r = subprocess.run([sys.executable, __file__], env=env,
                               capture_output=True, text=True, check=True)
            res.append(json.loads(r.stdout.strip().splitlines()[-1]))
            print(json.dumps(res[-1]), flush=True)
        keys = [k for k in res[0] if not k.endswith("_ms") and k not in ("fuse_h2", "lut")]
        same = all(r[k] == res[0][k] for r in res for k in keys)
        print(json.dumps({"identical_outputs": same}))
