"""Multi-GPU z-slab partition logic, world size 2 on CPU, over libtgcu's own
communicator (tgcu_comm, host backend: the TCP star, fixed-order host
all-reduce and routed point-to-point that carry the GPU job's bootstrap and
its host-staged collectives; no PyTorch, no GPU needed).

Each rank runs the owner-computes slab algorithm of paper_2402_14415_b200/slab.py
with the CPU oracle as compute engine: it keeps the points whose cells touch its
owned vertex planes (slab_point_mask), computes their gradient at its owned
vertices (global 1/N and TV normaliser), Adam-updates its owned coefficients,
sums the loss partials of its home points with an all-reduce, and exchanges its
boundary parameter planes with the neighbour (send/recv). After the run the
owned planes gathered from both ranks must equal a single-process training run
of the whole grid, and every step's loss must equal the single-process loss.
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


RES = (10, 9, 26)  # 4 brick layers along z -> slabs [0,2) and [2,4): planes [0,16) and [16,26)
STEPS = 4
N = 700


def _batches():
    rng = np.random.default_rng(5)
    out = []
    for s in range(STEPS):
        p = rng.uniform(-1.0, 1.0, (N, 3)).astype(np.float32).astype(np.float64)
        # points exactly on / next to the slab boundary plane z = 16h
        h = 2.0 / (RES[2] - 1)
        p[:40, 2] = -1.0 + 16 * h + rng.uniform(-1.5 * h, 1.5 * h, 40)
        p[:5, 2] = -1.0 + 16 * h
        p = p.astype(np.float32).astype(np.float64)
        gt = (np.linalg.norm(p, axis=1) - 0.6).astype(np.float32).astype(np.float64)
        out.append(np.concatenate([p, gt[:, None]], 1))
    return out


def _rank_main(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    from oracle.pyoracle import Loss, Oracle, Spec
    from paper_2402_14415_b200 import GridSpec
    from paper_2402_14415_b200.slab import (Comm, brick_layers, home_point_mask, owned_planes, slab_point_mask,
                                            slab_ranges)
    comm = Comm(rank, world, addr="127.0.0.1", port=port, backend="host")
    O = Oracle()
    s = Spec(dim=3, res=RES, order=2)
    gs = GridSpec(dim=3, resolution=RES, order=2)
    K = s.K
    plane = RES[0] * RES[1] * K
    lo, hi = slab_ranges(brick_layers(RES[2]), world)[rank]
    z0, z1 = owned_planes(RES[2], lo, hi)
    rng = np.random.default_rng(0)
    params = rng.uniform(-0.05, 0.05, s.V * K)  # identical initial grid on every rank
    m = np.zeros((z1 - z0) * plane)
    v = np.zeros_like(m)
    t = 0
    cfg = Loss()  # paper defaults: eikonal + TV
    losses = []
    for b in _batches():
        keep = slab_point_mask(gs, b, lo, hi)
        home = home_point_mask(gs, b, lo, hi)
        # point terms over this slab's points, with the global 1/N scale
        g = np.zeros(s.V * K)
        sub = b[keep]
        O.total_loss(s, params, sub, Loss(cfg.lambda1, 0.0, cfg.k, cfg.use_weighting, False), g)
        g *= len(sub) / N
        # TV gradient (global normaliser) added at owned vertices
        O.tv_loss(s, params, g, cfg.lambda2)
        # loss partials: home points' sums + TV pairs owned by the lower vertex
        hv = O.total_loss(s, params, b[home], Loss(cfg.lambda1, 0.0, cfg.k, cfg.use_weighting, False)) \
            if home.any() else np.zeros(4)
        nh = int(home.sum())
        own = params.reshape(RES[2], RES[1], RES[0], K)
        zt = min(z1, RES[2] - 1)
        tv_pairs = 0.0
        block = own[z0:z1]
        tv_pairs += np.sum((block[:, :, 1:] - block[:, :, :-1]) ** 2) + np.sum((block[:, 1:] - block[:, :-1]) ** 2)
        tv_pairs += np.sum((own[z0 + 1:zt + 1] - own[z0:zt]) ** 2)
        part = comm.allreduce([hv[1] * nh, hv[2] * nh, tv_pairs])
        P = (RES[0] - 1) * RES[1] * RES[2] + RES[0] * (RES[1] - 1) * RES[2] + RES[0] * RES[1] * (RES[2] - 1)
        fit, eik, tv = part[0] / N, part[1] / N, part[2] / (P * K)
        losses.append(fit + cfg.lambda1 * eik + cfg.lambda2 * tv)
        # Adam on the owned coefficients only
        ps = params[z0 * plane:z1 * plane].copy()
        t, bad = O.adam_step(ps, g[z0 * plane:z1 * plane].copy(), m, v, t, lr=1e-2)
        assert bad == -1
        params[z0 * plane:z1 * plane] = ps
        # halo exchange of the boundary parameter planes
        sends, recvs = [], []
        buf_lo, buf_hi = np.zeros(plane), np.zeros(plane)
        if rank > 0:
            sends.append((rank - 1, params[z0 * plane:(z0 + 1) * plane].copy()))
            recvs.append((rank - 1, buf_lo))
        if rank < world - 1:
            sends.append((rank + 1, params[(z1 - 1) * plane:z1 * plane].copy()))
            recvs.append((rank + 1, buf_hi))
        comm.exchange(sends, recvs)
        if rank > 0:
            params[(z0 - 1) * plane:z0 * plane] = buf_lo
        if rank < world - 1:
            params[z1 * plane:(z1 + 1) * plane] = buf_hi
    np.save(os.path.join(outdir, f"owned{rank}.npy"), params[z0 * plane:z1 * plane])
    np.save(os.path.join(outdir, f"loss{rank}.npy"), np.array(losses))
    comm.close()


def test_slab_partition_rules():
    from paper_2402_14415_b200 import GridSpec
    from paper_2402_14415_b200.slab import home_point_mask, slab_point_mask, slab_ranges, stored_planes
    assert slab_ranges(4, 2) == [(0, 2), (2, 4)]
    assert slab_ranges(5, 3) == [(0, 2), (2, 4), (4, 5)]
    assert slab_ranges(8, 2, weights=[1, 1, 1, 1, 10, 1, 1, 1])[0][1] >= 4
    assert stored_planes(26, 2, 4) == (15, 26)
    gs = GridSpec(dim=3, resolution=RES, order=2)
    b = np.concatenate(_batches())
    ranges = slab_ranges(4, 2)
    homes = [home_point_mask(gs, b, lo, hi) for lo, hi in ranges]
    keeps = [slab_point_mask(gs, b, lo, hi) for lo, hi in ranges]
    assert np.array_equal(homes[0] ^ homes[1], np.ones(len(b), bool))  # every point has exactly one home
    assert np.all(keeps[0] | keeps[1]) and np.all(~homes[0] | keeps[0])
    assert (keeps[0] & keeps[1]).sum() > 0  # boundary cell layer shared


def _spawn(fn, world, *args):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=fn, args=(r, world) + args) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]


def _comm_rank(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2402_14415_b200.slab import Comm
    c = Comm(rank, world, addr="127.0.0.1", port=port, backend="host")
    out = {}
    out["sum"] = c.allreduce([1.0 + rank, 0.1 * rank, 1e16 if rank == 0 else 1.0])
    out["max"] = c.allreduce([rank, -rank], op="max")
    out["min"] = c.allreduce([rank, -rank], op="min")
    out["gather"] = np.frombuffer(b"".join(c.allgather(bytes([rank, 7 * rank]))), np.uint8)
    c.barrier()
    # ring: send a block to both neighbours (world 3 routes through rank 0)
    sends = [((rank + 1) % world, np.full(5, rank, np.float64)), ((rank - 1) % world, np.full(3, -rank, np.int32))]
    a, b = np.zeros(5), np.zeros(3, np.int32)
    c.exchange(sends, [((rank - 1) % world, a), ((rank + 1) % world, b)])
    out["ring"] = np.concatenate([a, b.astype(np.float64)])
    np.savez(os.path.join(outdir, f"comm{rank}.npz"), **out)
    c.close()


@pytest.mark.parametrize("world", [2, 3])
def test_comm_host_collectives(tmp_path, world):
    """tgcu_comm (host backend) over world processes: rank-ordered sums (the
    same bits on every rank), max / min, allgather, barrier, routed p2p."""
    _spawn(_comm_rank, world, _free_port(), str(tmp_path))
    res = [np.load(tmp_path / f"comm{r}.npz") for r in range(world)]
    exp_sum = [sum(1.0 + r for r in range(world)), sum(0.1 * r for r in range(world)),
               1e16 + (world - 1) * 1.0]
    acc = 0.0
    for r in range(world):
        acc = acc + 0.1 * r  # rank order
    for r in range(world):
        assert np.array_equal(res[r]["sum"], res[0]["sum"])
        assert res[r]["sum"][0] == exp_sum[0] and res[r]["sum"][1] == acc
        assert list(res[r]["max"]) == [world - 1, 0] and list(res[r]["min"]) == [0, -(world - 1)]
        assert list(res[r]["gather"]) == [x for k in range(world) for x in (k, 7 * k)]
        lo, hi = (r - 1) % world, (r + 1) % world
        assert np.array_equal(res[r]["ring"], np.concatenate([np.full(5, lo), np.full(3, -hi)]).astype(np.float64))


def test_two_slabs_over_comm_match_single_process(tmp_path):
    import sys
    sys.path.insert(0, ROOT)
    from oracle.pyoracle import Loss, Oracle, Spec
    _spawn(_rank_main, 2, _free_port(), str(tmp_path))
    O = Oracle()
    s = Spec(dim=3, res=RES, order=2)
    rng = np.random.default_rng(0)
    c0 = rng.uniform(-0.05, 0.05, s.V * s.K)
    final, terms = O.train(s, c0, _batches(), Loss(), lr=1e-2)
    slabs = np.concatenate([np.load(tmp_path / "owned0.npy"), np.load(tmp_path / "owned1.npy")])
    assert np.allclose(slabs, final, rtol=1e-9, atol=1e-12)
    for r in range(2):
        assert np.allclose(np.load(tmp_path / f"loss{r}.npy"), terms[:, 0], rtol=1e-9)
