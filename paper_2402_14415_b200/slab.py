"""Multi-GPU z-slab training, owner computes.

The global grid is cut into slabs of whole brick layers (bricks of 8^3
vertices). Rank r owns the vertex planes of its brick layers and the Adam
state of those vertices; it stores one halo plane below and above. Every rank
is given the full global batch and keeps the points whose cells touch its
owned vertices (a point in a slab-boundary cell layer is used by both ranks,
exactly as a point in a brick-boundary cell layer is binned into both bricks
on one GPU; with `local_points` the batch can be sharded to the ranks up
front, the loss still normalised by the global batch size). Per step:

    partials = slab.begin(batch)          # bin + fused brick kernel, local sums
    all_reduce(partials)                  # {recon, eik, tv, nan flag, bad flag}
    terms = slab.finish(partials)         # same commit decision on every rank
    halo exchange of boundary parameter planes (send/recv with the neighbours)

With the fused halo (SlabTrainer default when every rank can open its
neighbours' parameter buffers through CUDA IPC, i.e. NVLink peers or one
shared device) the exchange disappears: the brick kernel of each boundary
brick layer also stores the new boundary plane into the neighbour's halo
plane of the same ping-pong slot, and the all-reduce of the partials is the
only collective per step.

No gradient is exchanged: each gradient is computed by its owner. The loss
scale 1/N and the TV normaliser P*K are global (sdf_loss.cpp:161-170), so the
slab steps reproduce the single-grid step.

The partition helpers are plain numpy so the CPU tests (gloo, world size 2)
exercise the same rules with the oracle as compute engine.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Tuple

import numpy as np

from . import (TGCU_ASYNC, TGCU_HOST, AdamConfig, GridSpec, InitOptions, LossConfig, LossTerms, _check, _ptr, _Terms,
               lib)

BRICK = 8


def brick_layers(res_z: int) -> int:
    return (res_z + BRICK - 1) // BRICK


def slab_ranges(nbz: int, world: int, weights: Optional[np.ndarray] = None) -> List[Tuple[int, int]]:
    """Split nbz brick layers into `world` contiguous ranges. With per-layer
    weights (e.g. point counts) the split balances weight + the dense work."""
    if world > nbz:
        raise ValueError(f"slab_ranges: {world} ranks for {nbz} brick layers")
    if weights is None:
        base, rem = divmod(nbz, world)
        out, lo = [], 0
        for r in range(world):
            hi = lo + base + (1 if r < rem else 0)
            out.append((lo, hi))
            lo = hi
        return out
    w = np.asarray(weights, dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    out, lo = [], 0
    for r in range(world):
        if r == world - 1:
            hi = nbz
        else:
            target = cum[-1] * (r + 1) / world
            hi = int(np.searchsorted(cum, target))
            hi = max(hi, lo + 1)
            hi = min(hi, nbz - (world - 1 - r))
        out.append((lo, hi))
        lo = hi
    return out


def owned_planes(res_z: int, zb_lo: int, zb_hi: int) -> Tuple[int, int]:
    return BRICK * zb_lo, min(res_z, BRICK * zb_hi)


def stored_planes(res_z: int, zb_lo: int, zb_hi: int) -> Tuple[int, int]:
    return max(0, BRICK * zb_lo - 1), min(res_z, BRICK * zb_hi + 1)


def point_cells_z(spec: GridSpec, z: np.ndarray) -> np.ndarray:
    """The reference's locate rule on the z axis (grid_spec.cpp:45-69), fp64."""
    lo = spec.origin[2]
    hi = spec.origin[2] + spec.extent[2]
    h = spec.extent[2] / (spec.resolution[2] - 1)
    p = np.clip(np.asarray(z, dtype=np.float64), lo, hi)
    c = np.floor((p - lo) / h).astype(np.int64)
    return np.clip(c, 0, spec.resolution[2] - 2)


def slab_point_mask(spec: GridSpec, points: np.ndarray, zb_lo: int, zb_hi: int) -> np.ndarray:
    """Points whose cell touches a vertex owned by brick layers [zb_lo, zb_hi):
    cells [8*zb_lo - 1, 8*zb_hi - 1] along z."""
    c = point_cells_z(spec, np.asarray(points)[:, 2])
    return (c >= BRICK * zb_lo - 1) & (c <= BRICK * zb_hi - 1)


def home_point_mask(spec: GridSpec, points: np.ndarray, zb_lo: int, zb_hi: int) -> np.ndarray:
    """Points whose loss terms this slab sums (cell's brick layer is its own)."""
    c = point_cells_z(spec, np.asarray(points)[:, 2])
    return (c >= BRICK * zb_lo) & (c <= BRICK * zb_hi - 1)


class _CudaBuf:
    """__cuda_array_interface__ view of a raw device pointer (torch.as_tensor)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def device_view(ptr: int, n: int, dtype: str = "<f4"):
    import torch
    return torch.as_tensor(_CudaBuf(ptr, n, dtype), device="cuda")


class SlabGrid:
    """Device handle of one slab (tgcu_grid_create_slab)."""

    def __init__(self, spec: GridSpec, zb_lo: int, zb_hi: int, opts: Optional[InitOptions] = None, device: int = 0):
        L = lib()
        self.spec = spec
        self.zb = (zb_lo, zb_hi)
        o = opts or InitOptions()
        from . import _Init
        ci = _Init(int(o.mode), o.constant, o.epsilon, o.seed, o.memory_cap_bytes)
        h = C.c_void_p()
        _check(L.tgcu_grid_create_slab(C.byref(spec._c()), zb_lo, zb_hi, C.byref(ci), device, C.byref(h)))
        self._h = h
        info = [C.c_int() for _ in range(5)]
        L.tgcu_slab_info(h, *[C.byref(x) for x in info])
        self.z_store_lo, self.z_store_n, self.z_own_lo, self.z_own_hi, self.brick_layers = [x.value for x in info]

    @property
    def handle(self):
        return self._h

    def set_deterministic(self, on: bool = True):
        """Bit-reproducible slab steps (tgcu_grid_set_deterministic): each brick's
        sums in a canonical order, so the slabs' parameters equal a single
        grid's in the same mode bit for bit."""
        _check(lib().tgcu_grid_set_deterministic(self._h, 1 if on else 0))

    def close(self):
        if getattr(self, "_h", None):
            lib().tgcu_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def adam_reset(self, cfg: AdamConfig = AdamConfig()):
        _check(lib().tgcu_adam_reset(self._h, C.byref(cfg._c())))

    def coeff_total(self) -> int:
        return int(lib().tgcu_grid_coeff_total(self._h))

    def coeffs(self) -> np.ndarray:
        out = np.empty(self.coeff_total())
        _check(lib().tgcu_grid_download_f64(self._h, _ptr(out), out.size))
        return out

    def set_coeffs(self, values):
        a = np.ascontiguousarray(values, dtype=np.float64).ravel()
        _check(lib().tgcu_grid_upload_f64(self._h, _ptr(a), a.size))

    def owned_coeffs(self) -> np.ndarray:
        """Coefficients of the owned vertex planes (reference AoS layout)."""
        K = self.spec.coeffs_per_vertex()
        plane = self.spec.resolution[0] * self.spec.resolution[1] * K
        c = self.coeffs()
        a = (self.z_own_lo - self.z_store_lo) * plane
        b = (self.z_own_hi - self.z_store_lo) * plane
        return c[a:b]

    def begin(self, samples, cfg: LossConfig, stream=None, export_grad=False, n_global: int = 0,
              input_ready: bool = False) -> int:
        """Phase 1; returns the device pointer of the 5 local partial sums.
        samples: the full global batch, or only this slab's points
        (slab_point_mask) with n_global = the global batch size.
        input_ready: see train_step (device samples known complete)."""
        from . import TGCU_EXPORT_GRAD, TGCU_INPUT_READY, _dev_f32, _is_torch
        flags = 0 if _is_torch(samples) else TGCU_HOST
        if flags == 0:
            _dev_f32(samples, 4, "slab samples")
        if export_grad:
            flags |= TGCU_EXPORT_GRAD
        if input_ready and not flags & TGCU_HOST:
            flags |= TGCU_INPUT_READY
        if not _is_torch(samples):
            samples = np.ascontiguousarray(np.asarray(samples, dtype=np.float32)).reshape(-1, 4)
        p = C.POINTER(C.c_double)()
        _check(lib().tgcu_slab_step_begin(self._h, _ptr(samples), samples.shape[0], int(n_global), C.byref(cfg._c()),
                                          C.byref(p), flags, C.c_void_p(stream) if stream else None))
        return C.cast(p, C.c_void_p).value

    def finish(self, reduced_ptr: Optional[int], asynchronous=False, stream=None) -> Optional[LossTerms]:
        if asynchronous:
            _check(lib().tgcu_slab_step_finish(self._h, C.c_void_p(reduced_ptr) if reduced_ptr else None, None,
                                               TGCU_ASYNC, C.c_void_p(stream) if stream else None))
            return None
        t = _Terms()
        _check(lib().tgcu_slab_step_finish(self._h, C.c_void_p(reduced_ptr) if reduced_ptr else None, C.byref(t), 0,
                                           C.c_void_p(stream) if stream else None))
        return LossTerms._from(t)

    def halo(self):
        """(send_lo, send_hi, recv_lo, recv_hi, plane_floats) device pointers (0 = none)."""
        ptrs = [C.c_void_p() for _ in range(4)]
        pf = C.c_int64()
        _check(lib().tgcu_slab_halo(self._h, *[C.byref(x) for x in ptrs], C.byref(pf)))
        return tuple((x.value or 0) for x in ptrs) + (pf.value,)

    def sync(self) -> LossTerms:
        t = _Terms()
        _check(lib().tgcu_sync(self._h, C.byref(t)))
        return LossTerms._from(t)

    # ---- fused halo: the brick kernel writes boundary planes into the neighbours ----
    def ipc_export(self) -> bytes:
        """144-byte blob: IPC handles of both parameter slots + halo plane offsets."""
        buf = (C.c_ubyte * 144)()
        _check(lib().tgcu_slab_ipc_export(self._h, C.cast(buf, C.c_void_p)))
        return bytes(buf)

    def ipc_import(self, side: int, blob: bytes):
        """side 0: the lower neighbour's blob, side 1: the upper neighbour's."""
        buf = (C.c_ubyte * 144).from_buffer_copy(blob)
        _check(lib().tgcu_slab_ipc_import(self._h, int(side), C.cast(buf, C.c_void_p)))

    def halo_slots(self) -> Tuple[Tuple[int, int], Tuple[int, int]]:
        """This slab's (lower, upper) halo plane addresses, each as (slot 0, slot 1); 0 = none."""
        lo, hi = (C.c_void_p * 2)(), (C.c_void_p * 2)()
        _check(lib().tgcu_slab_halo_slots(self._h, lo, hi))
        return (lo[0] or 0, lo[1] or 0), (hi[0] or 0, hi[1] or 0)

    def set_peer_planes(self, dst_lo: Tuple[int, int], dst_hi: Tuple[int, int]):
        """Same-device neighbours (tests): their halo plane addresses per slot."""
        lo = (C.c_void_p * 2)(*[C.c_void_p(x or None) for x in dst_lo])
        hi = (C.c_void_p * 2)(*[C.c_void_p(x or None) for x in dst_hi])
        _check(lib().tgcu_slab_set_peer_planes(self._h, lo, hi))

    def peer_probe(self, phase: int) -> bool:
        ok = C.c_int(0)
        _check(lib().tgcu_slab_peer_probe(self._h, int(phase), C.byref(ok)))
        return bool(ok.value)

    def profile_begin(self, every: int = 1):
        _check(lib().tgcu_profile_every(self._h, int(every)))
        _check(lib().tgcu_profile_begin(self._h))

    def profile_end(self):
        """(summed brick-kernel device ms, launches) since profile_begin."""
        ms, n = C.c_double(), C.c_int()
        _check(lib().tgcu_profile_end(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value


TGCU_COMM_NCCL, TGCU_COMM_HOST = 0, 1


class Comm:
    """One rank of a multi-GPU job (tgcu_comm, csrc/comm.cu): a TCP star
    rooted at rank 0 (addr:port) for the bootstrap and host collectives, and
    NCCL (backend "nccl", loaded by libtgcu at run time) or host-staged
    ("host": tests, ranks sharing a device) device collectives. No PyTorch.
    Defaults: MASTER_ADDR, TGCU_COMM_PORT (else MASTER_PORT + 17, clear of a
    torch.distributed store on MASTER_PORT), TGCU_COMM_BACKEND (else nccl)."""

    def __init__(self, rank: int, world: int, device: int = 0, addr: Optional[str] = None,
                 port: Optional[int] = None, backend: Optional[str] = None):
        import os
        addr = addr or os.environ.get("MASTER_ADDR", "127.0.0.1")
        if port is None:
            port = int(os.environ.get("TGCU_COMM_PORT", int(os.environ.get("MASTER_PORT", "29500")) + 17))
        backend = backend or os.environ.get("TGCU_COMM_BACKEND", "nccl")
        if backend not in ("nccl", "host"):
            raise ValueError(f"Comm: unknown backend {backend!r}")
        self.rank, self.world, self.backend = rank, world, backend
        h = C.c_void_p()
        _check(lib().tgcu_comm_create(addr.encode(), int(port), rank, world, device,
                                      TGCU_COMM_NCCL if backend == "nccl" else TGCU_COMM_HOST, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().tgcu_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def barrier(self):
        _check(lib().tgcu_comm_barrier(self._h))

    def allreduce(self, values, op: str = "sum") -> np.ndarray:
        """Host doubles reduced over the ranks in rank order (sum / max / min)."""
        a = np.ascontiguousarray(np.atleast_1d(np.asarray(values, dtype=np.float64))).copy()
        _check(lib().tgcu_comm_allreduce_host(self._h, _ptr(a), a.size, {"sum": 0, "max": 1, "min": 2}[op]))
        return a

    def allgather(self, blob: bytes) -> List[bytes]:
        n = len(blob)
        inb = (C.c_ubyte * max(n, 1)).from_buffer_copy(blob or b"\0")
        out = (C.c_ubyte * max(n * self.world, 1))()
        _check(lib().tgcu_comm_allgather_host(self._h, inb, n, out))
        raw = bytes(out)
        return [raw[r * n:(r + 1) * n] for r in range(self.world)]

    def exchange(self, sends, recvs):
        """Routed host point-to-point (collective). sends: [(dst, ndarray)],
        recvs: [(src, ndarray to fill)]."""
        sends = [(d, np.ascontiguousarray(a)) for d, a in sends]
        ns, nr = len(sends), len(recvs)
        dst = (C.c_int * max(ns, 1))(*[d for d, _ in sends])
        sb = (C.c_void_p * max(ns, 1))(*[a.ctypes.data for _, a in sends])
        sz = (C.c_int64 * max(ns, 1))(*[a.nbytes for _, a in sends])
        src = (C.c_int * max(nr, 1))(*[s_ for s_, _ in recvs])
        rb = (C.c_void_p * max(nr, 1))(*[a.ctypes.data for _, a in recvs])
        rz = (C.c_int64 * max(nr, 1))(*[a.nbytes for _, a in recvs])
        _check(lib().tgcu_comm_exchange_host(self._h, ns, dst, sb, sz, nr, src, rb, rz))


class SlabTrainer:
    """One rank of a slab-parallel training run: the slab grid, attached to
    the job's Comm (tgcu_slab_connect: initial halo, peer-memory halo set up
    when every rank can open its neighbours' buffers), stepped with
    tgcu_slab_train_step. No PyTorch on this path."""

    def __init__(self, spec: GridSpec, rank: int, world: int, adam: AdamConfig, device: int = 0,
                 opts: Optional[InitOptions] = None, ranges=None, comm: Optional[Comm] = None,
                 fused_halo: Optional[bool] = None):
        import os
        self.rank, self.world = rank, world
        nbz = brick_layers(spec.resolution[2])
        self.ranges = ranges or slab_ranges(nbz, world)
        lo, hi = self.ranges[rank]
        self.comm = comm or Comm(rank, world, device)
        self.backend = self.comm.backend
        self.slab = SlabGrid(spec, lo, hi, opts, device)
        self.slab.adam_reset(adam)
        if fused_halo is None:
            fused_halo = os.environ.get("TGCU_FUSED_HALO", "1") != "0"
        f = C.c_int(0)
        _check(lib().tgcu_slab_connect(self.slab.handle, self.comm.handle, 1 if fused_halo else 0, C.byref(f)))
        self.fused_halo = bool(f.value)

    def local_points(self, samples):
        """The points of a global batch this rank's slab needs (host numpy):
        cells touching its owned vertex planes (the reference cell rule)."""
        lo, hi = self.ranges[self.rank]
        a = np.asarray(samples)
        return np.ascontiguousarray(a[slab_point_mask(self.slab.spec, a.astype(np.float64), lo, hi)])

    def step(self, samples, cfg: LossConfig, stream=None, want_terms=False, n_global: int = 0,
             input_ready: bool = False):
        """One step (tgcu_slab_train_step). samples: the global batch, or this
        rank's local_points with n_global = the global batch size; host numpy
        or a CUDA tensor. want_terms=False: stream-ordered (NCCL backend)."""
        from . import TGCU_INPUT_READY, _dev_f32, _is_torch
        flags = 0 if _is_torch(samples) else TGCU_HOST
        if flags == 0:
            _dev_f32(samples, 4, "slab samples")
            if input_ready:
                flags |= TGCU_INPUT_READY
        else:
            samples = np.ascontiguousarray(np.asarray(samples, dtype=np.float32)).reshape(-1, 4)
        st = C.c_void_p(stream) if stream else None
        if want_terms:
            t = _Terms()
            _check(lib().tgcu_slab_train_step(self.slab.handle, _ptr(samples), samples.shape[0], int(n_global),
                                              C.byref(cfg._c()), C.byref(t), flags, st))
            return LossTerms._from(t)
        _check(lib().tgcu_slab_train_step(self.slab.handle, _ptr(samples), samples.shape[0], int(n_global),
                                          C.byref(cfg._c()), None, flags | TGCU_ASYNC, st))
        return None

    def comm_profile(self):
        """(all-reduce ms, halo-exchange ms, steps) summed over the profiled
        steps since the last call (tgcu_slab_comm_profile)."""
        ar, hx, n = C.c_double(), C.c_double(), C.c_int()
        _check(lib().tgcu_slab_comm_profile(self.slab.handle, C.byref(ar), C.byref(hx), C.byref(n)))
        return ar.value, hx.value, n.value

    def close(self):
        self.slab.close()
        self.comm.close()
