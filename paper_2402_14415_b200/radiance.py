"""Radiance density chain on the device.

Mirrors volume_render.hpp:11-54 and sh.hpp:11-45 of /root/reference/proj/core
for the hot part of TaylorGrid-density NeRF training: ``render_rays`` (batched
``render_ray``) and ``photometric_loss`` with gradients to the density grid
(through the activation, weights and transmittance) and to the SH color grid
(through the sigmoid, basis and interpolation), via ``tgcu_photometric_loss``.
Stratified jitter is not supported (the reference draws it from a per-ray
mt19937_64 stream).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Sequence

import numpy as np

from . import TGCU_HOST, GridSpec, TaylorGrid, _check, _ptr, _Spec, lib

__all__ = ["DensityActivation", "RenderOptions", "SHColorGrid", "sh_basis", "make_rays", "render_rays",
           "photometric_loss"]


class DensityActivation(IntEnum):
    """tg::DensityActivation (volume_render.hpp:11)."""
    ShiftedSoftplus = 0
    ClampRelu = 1


@dataclass
class RenderOptions:
    """tg::RenderOptions (volume_render.hpp:17-24)."""
    n_samples: int = 64
    activation: DensityActivation = DensityActivation.ShiftedSoftplus
    softplus_shift: float = -10.0
    background: Sequence[float] = (1.0, 1.0, 1.0)
    jitter: bool = False  # stratified jitter inside the N bins (per-ray Rng, ray id = batch index)
    jitter_seed: int = 0


class _RO(C.Structure):
    _fields_ = [("n_samples", C.c_int), ("activation", C.c_int), ("softplus_shift", C.c_double),
                ("background", C.c_double * 3), ("jitter", C.c_int), ("jitter_seed", C.c_uint64)]


@dataclass
class SHColorGrid:
    """tg::SHColorGrid (sh.hpp:19-29): per-vertex [R basis | G basis | B basis]
    coefficients (host numpy, fp32 on the device)."""
    spec: GridSpec
    degree: int = 2
    coeffs: Optional[np.ndarray] = None

    def basis_count(self) -> int:
        return (self.degree + 1) ** 2

    def channels(self) -> int:
        return 3 * self.basis_count()

    def __post_init__(self):
        if not 0 <= self.degree <= 2:
            raise ValueError("init_sh_grid: degree must be in [0,2]")
        if self.coeffs is None:
            self.coeffs = np.zeros(self.spec.vertex_count() * self.channels())


def sh_basis(degree: int, d) -> np.ndarray:
    """sh_basis (sh.cpp:43-60), host helper."""
    x, y, z = (float(v) for v in d)
    out = [0.28209479177387814]
    if degree >= 1:
        c1 = 0.4886025119029199
        out += [-c1 * y, c1 * z, -c1 * x]
    if degree >= 2:
        out += [1.0925484305920792 * x * y, -1.0925484305920792 * y * z,
                0.31539156525252005 * (2 * z * z - x * x - y * y), -1.0925484305920792 * x * z,
                0.5462742152960396 * (x * x - y * y)]
    return np.array(out)


def make_rays(origins, dirs, near, far) -> np.ndarray:
    """Pack a RayBatch (camera.hpp:47-55) as the ABI's n x 8 float array."""
    o = np.asarray(origins, dtype=np.float32).reshape(-1, 3)
    d = np.asarray(dirs, dtype=np.float32).reshape(-1, 3)
    n = o.shape[0]
    out = np.empty((n, 8), dtype=np.float32)
    out[:, 0:3] = o
    out[:, 3:6] = d
    out[:, 6] = np.broadcast_to(np.asarray(near, dtype=np.float32), (n,))
    out[:, 7] = np.broadcast_to(np.asarray(far, dtype=np.float32), (n,))
    return out


def _call(density: TaylorGrid, sh: SHColorGrid, rays, gt, opts: RenderOptions, want_colors: bool,
          want_grad: bool):
    L = lib()
    r = np.ascontiguousarray(np.asarray(rays, dtype=np.float32)).reshape(-1, 8)
    n = r.shape[0]
    g = None if gt is None else np.ascontiguousarray(np.asarray(gt, dtype=np.float32)).reshape(-1, 3)
    shc = np.ascontiguousarray(np.asarray(sh.coeffs, dtype=np.float32)).ravel()
    cols = np.empty((n, 3), dtype=np.float32) if want_colors else None
    res = np.empty(n, dtype=np.float32) if want_colors else None
    gd = np.zeros(density.coeff_total(), dtype=np.float32) if want_grad else None
    gs = np.zeros(shc.size, dtype=np.float32) if want_grad else None
    ro = _RO(int(opts.n_samples), int(opts.activation), float(opts.softplus_shift),
             (C.c_double * 3)(*[float(b) for b in opts.background]), int(bool(opts.jitter)), int(opts.jitter_seed))
    loss = C.c_double(0.0)
    _check(L.tgcu_photometric_loss(density.handle, C.byref(sh.spec._c()), sh.degree, _ptr(shc), _ptr(r), _ptr(g), n,
                                   C.cast(C.pointer(ro), C.c_void_p), _ptr(cols), _ptr(res), _ptr(gd), _ptr(gs),
                                   C.byref(loss), TGCU_HOST, None))
    return loss.value, cols, res, gd, gs


def render_rays(density: TaylorGrid, sh: SHColorGrid, rays, opts: RenderOptions = RenderOptions()):
    """Batched render_ray (volume_render.cpp:194-208) -> (colors n x 3, residual n)."""
    _, cols, res, _, _ = _call(density, sh, rays, None, opts, True, False)
    return cols.astype(np.float64), res.astype(np.float64)


def photometric_loss(density: TaylorGrid, sh: SHColorGrid, rays, gt, opts: RenderOptions = RenderOptions(),
                     want_grad: bool = True):
    """photometric_loss (volume_render.cpp:210-276): mean squared RGB error and,
    with want_grad, (grad_density, grad_sh) in the coefficient layouts (fp64)."""
    loss, _, _, gd, gs = _call(density, sh, rays, gt, opts, False, want_grad)
    if not want_grad:
        return loss
    return loss, gd.astype(np.float64), gs.astype(np.float64)
