"""TaylorGrid query-and-optimise hot path on B200 (sm_100a).

Python host mirror of the reference's ``tg::`` API for the hot path
(/root/reference/proj/core: grid_spec.hpp, taylor_grid.hpp, sdf_loss.hpp,
adam.hpp, schedule.hpp), layered on the C ABI of ``libtgcu.so``
(include/tgcu.h). Names, argument meaning and error classes follow the
reference; calls are batched (arrays of points instead of one ``Vec3``).

There is no CPU fallback: importing works without a GPU, but every call that
computes needs ``libtgcu.so`` and a CUDA device and raises otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "GridSpec", "InitMode", "InitOptions", "LossConfig", "LossTerms", "AdamConfig", "TaylorGrid",
    "coeff_count", "init_grid", "eval", "eval_with_spatial_gradient", "backprop_point",
    "backprop_spatial_chain", "backprop_value_and_spatial", "adaptive_weight", "tv_loss",
    "total_loss", "adam_step", "train_step", "sample", "sample_uniform", "shape_sdf",
    "ConfigError", "IngestError", "NumericalError", "ResourceError", "CudaError", "lib",
    "launch_count", "reset_launch_count", "LIB_PATH", "TrainGraph", "upsample", "multilinear_resample", "ScalarField3",
    "ScalarField2", "sample_grid_field", "sample_grid_field2", "StoragePrecision", "save_tgrid", "load_tgrid",
    "tgrid_file_size", "draw_batch",
]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtgcu.so")

# ---- error classes (errors.hpp:9-34) ---------------------------------------


class ConfigError(RuntimeError):
    """tg::ConfigError."""


class IngestError(RuntimeError):
    """tg::IngestError."""


class NumericalError(RuntimeError):
    """tg::NumericalError."""


class ResourceError(RuntimeError):
    """tg::ResourceError."""


class CudaError(RuntimeError):
    """CUDA runtime failure or no device (the product has no CPU fallback)."""


_ERR = {1: ValueError, 2: ConfigError, 3: IngestError, 4: NumericalError, 5: ResourceError, 6: CudaError}

TGCU_HOST, TGCU_ASYNC, TGCU_SORTED, TGCU_EXPORT_GRAD, TGCU_INPUT_READY = 1, 2, 4, 8, 16

# ---- C structs ----------------------------------------------------------------


class _Spec(C.Structure):
    _fields_ = [("dim", C.c_int), ("res", C.c_int * 3), ("origin", C.c_double * 3),
                ("extent", C.c_double * 3), ("order", C.c_int)]


class _Init(C.Structure):
    _fields_ = [("mode", C.c_int), ("constant", C.c_double), ("epsilon", C.c_double),
                ("seed", C.c_uint64), ("memory_cap_bytes", C.c_uint64)]


class _Loss(C.Structure):
    _fields_ = [("lambda1", C.c_double), ("lambda2", C.c_double), ("k", C.c_double),
                ("use_weighting", C.c_int), ("use_tv", C.c_int), ("differentiate_weight", C.c_int)]


class _Terms(C.Structure):
    _fields_ = [("total", C.c_double), ("fit", C.c_double), ("eik", C.c_double), ("tv", C.c_double)]


class _Adam(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)]


_lib = None


def lib():
    """Load libtgcu.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtgcu.so not built at {LIB_PATH}; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    L.tgcu_last_error.restype = C.c_char_p
    L.tgcu_version.restype = C.c_char_p
    L.tgcu_coeff_count.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int)]
    L.tgcu_grid_create.argtypes = [C.POINTER(_Spec), C.POINTER(_Init), C.c_int, C.POINTER(P)]
    L.tgcu_grid_destroy.argtypes = [P]
    L.tgcu_grid_spec_of.argtypes = [P, C.POINTER(_Spec)]
    L.tgcu_grid_coeff_total.argtypes = [P]
    L.tgcu_grid_coeff_total.restype = C.c_int64
    L.tgcu_grid_coeffs.argtypes = [P]
    L.tgcu_grid_coeffs.restype = P
    L.tgcu_grid_grad.argtypes = [P]
    L.tgcu_grid_grad.restype = P
    L.tgcu_grid_upload_f64.argtypes = [P, P, C.c_int64]
    L.tgcu_grid_download_f64.argtypes = [P, P, C.c_int64]
    L.tgcu_grid_upload_f32.argtypes = [P, P, C.c_int64, C.c_int]
    L.tgcu_grid_download_f32.argtypes = [P, P, C.c_int64, C.c_int]
    L.tgcu_grid_all_finite.argtypes = [P, C.POINTER(C.c_int)]
    L.tgcu_eval.argtypes = [P, P, C.c_int64, P, P, C.c_int, P]
    L.tgcu_sort_points.argtypes = [P, P, C.c_int64, P, P, P, P]
    L.tgcu_query_brick_codes.argtypes = [P]
    L.tgcu_query_brick_codes.restype = C.c_int64
    L.tgcu_eval_sorted.argtypes = [P, P, C.c_int64, P, P, P, C.c_int, P]
    L.tgcu_backprop.argtypes = [P, P, P, P, C.c_int64, P, C.c_int, P]
    L.tgcu_grad_zero.argtypes = [P, P, P]
    L.tgcu_grad_download_f64.argtypes = [P, P, P, C.c_int64]
    L.tgcu_tv_loss.argtypes = [P, P, C.c_double, C.POINTER(C.c_double), P]
    L.tgcu_total_loss.argtypes = [P, P, C.c_int64, C.POINTER(_Loss), P, C.POINTER(_Terms), C.c_int, P]
    L.tgcu_adam_reset.argtypes = [P, C.POINTER(_Adam)]
    L.tgcu_adam_get_t.argtypes = [P, C.POINTER(C.c_int64)]
    L.tgcu_adam_step.argtypes = [P, P, P]
    L.tgcu_adam_download_f64.argtypes = [P, P, P, C.c_int64]
    L.tgcu_train_step.argtypes = [P, P, C.c_int64, C.POINTER(_Loss), C.POINTER(_Terms), C.c_int, P]
    L.tgcu_sync.argtypes = [P, C.POINTER(_Terms)]
    L.tgcu_grid_steps_launched.argtypes = [P, C.POINTER(C.c_int64)]
    L.tgcu_grid_create_slab.argtypes = [C.POINTER(_Spec), C.c_int, C.c_int, C.POINTER(_Init), C.c_int, C.POINTER(P)]
    L.tgcu_slab_info.argtypes = [P] + [C.POINTER(C.c_int)] * 5
    L.tgcu_slab_step_begin.argtypes = [P, P, C.c_int64, C.c_int64, C.POINTER(_Loss),
                                       C.POINTER(C.POINTER(C.c_double)), C.c_int, P]
    L.tgcu_slab_step_finish.argtypes = [P, P, C.POINTER(_Terms), C.c_int, P]
    L.tgcu_slab_halo.argtypes = [P, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(C.c_int64)]
    L.tgcu_slab_ipc_export.argtypes = [P, P]
    L.tgcu_slab_ipc_import.argtypes = [P, C.c_int, P]
    L.tgcu_slab_set_peer_planes.argtypes = [P, C.POINTER(P), C.POINTER(P)]
    L.tgcu_slab_peer_probe.argtypes = [P, C.c_int, C.POINTER(C.c_int)]
    L.tgcu_slab_halo_slots.argtypes = [P, C.POINTER(P), C.POINTER(P)]
    L.tgcu_trace.argtypes = [P, C.POINTER(_Terms), C.c_int]
    L.tgcu_launch_count.restype = C.c_int64
    L.tgcu_profile_begin.argtypes = [P]
    L.tgcu_profile_every.argtypes = [P, C.c_int]
    L.tgcu_profile_end.argtypes = [P, C.POINTER(C.c_double), C.POINTER(C.c_int)]
    L.tgcu_sample.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int64, C.c_double, C.c_double, C.c_double, P]
    L.tgcu_sample_uniform.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_double, C.c_double, P]
    L.tgcu_sample_uniform_device.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_double, C.c_double, P, P]
    L.tgcu_shape_sdf.argtypes = [C.c_int, C.c_int, C.c_double, P, C.c_int64, P]
    L.tgcu_multilinear_resample.argtypes = [C.POINTER(_Spec), P, C.c_int64, C.c_int, C.POINTER(C.c_int), P, C.c_int, P]
    L.tgcu_grid_upsample.argtypes = [P, P, C.c_int, P]
    L.tgcu_sample_grid_field.argtypes = [P, C.POINTER(C.c_int), P, C.c_int, P]
    L.tgcu_draw_batch.argtypes = [P, C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, P, P]
    L.tgcu_save_tgrid.argtypes = [P, C.c_char_p, C.c_int]
    L.tgcu_load_tgrid.argtypes = [C.c_char_p, C.c_int, C.POINTER(P)]
    L.tgcu_tgrid_file_size.argtypes = [C.POINTER(_Spec), C.c_int]
    L.tgcu_tgrid_file_size.restype = C.c_int64
    # tgcu_render_options is declared in radiance.py (_RO); the pointer is passed as void*
    L.tgcu_photometric_loss.argtypes = [P, C.POINTER(_Spec), C.c_int, P, P, P, C.c_int64, P, P, P, P, P,
                                        C.POINTER(C.c_double), C.c_int, P]
    L.tgcu_rng_create.argtypes = [C.c_uint64, C.POINTER(P)]
    L.tgcu_rng_destroy.argtypes = [P]
    L.tgcu_rng_index.argtypes = [P, C.c_uint64, C.c_int64, P]
    L.tgcu_rng_uniform_box.argtypes = [P, C.c_int, P, P, C.c_int64, P]
    L.tgcu_recon_loss.argtypes = [P, P, C.c_int64, C.POINTER(_Loss), C.c_double, P, C.POINTER(C.c_double), C.c_int, P]
    L.tgcu_eikonal_loss.argtypes = [P, P, C.c_int64, C.c_double, P, C.POINTER(C.c_double), C.c_int, P]
    L.tgcu_train_step_fresh_eik.argtypes = [P, P, C.c_int64, P, C.POINTER(_Loss), C.POINTER(_Terms), C.c_int, P]
    L.tgcu_shuffle_order.argtypes = [C.c_uint64, C.c_int64, P]
    L.tgcu_grid_set_deterministic.argtypes = [P, C.c_int]
    L.tgcu_grid_set_step_path.argtypes = [P, C.c_int]
    L.tgcu_train_graph_create.argtypes = [P, C.POINTER(C.c_void_p), C.c_int, C.c_int64, C.POINTER(_Loss), P,
                                          C.POINTER(P)]
    L.tgcu_train_graph_launch.argtypes = [P, P]
    L.tgcu_train_graph_destroy.argtypes = [P]
    L.tgcu_slab_comm_profile.argtypes = [P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int)]
    L.tgcu_comm_create.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(P)]
    L.tgcu_comm_destroy.argtypes = [P]
    L.tgcu_comm_info.argtypes = [P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.tgcu_comm_barrier.argtypes = [P]
    L.tgcu_comm_allreduce_host.argtypes = [P, P, C.c_int, C.c_int]
    L.tgcu_comm_allgather_host.argtypes = [P, P, C.c_int64, P]
    L.tgcu_comm_exchange_host.argtypes = [P, C.c_int, P, P, P, C.c_int, P, P, P]
    L.tgcu_slab_connect.argtypes = [P, P, C.c_int, C.POINTER(C.c_int)]
    L.tgcu_slab_train_step.argtypes = [P, P, C.c_int64, C.c_int64, C.POINTER(_Loss), C.POINTER(_Terms), C.c_int, P]
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        msg = lib().tgcu_last_error().decode()
        raise _ERR.get(rc, RuntimeError)(msg)


def launch_count() -> int:
    return int(lib().tgcu_launch_count())


def reset_launch_count() -> None:
    lib().tgcu_reset_launch_count()


# ---- value types (mirrors of the reference structs) ----------------------------


def coeff_count(order: int, dim: int) -> int:
    """coeff_count (grid_spec.cpp:10-19)."""
    out = C.c_int()
    _check(lib().tgcu_coeff_count(order, dim, C.byref(out)))
    return out.value


@dataclass
class GridSpec:
    """tg::GridSpec (grid_spec.hpp:19-24)."""
    dim: int = 3
    resolution: Sequence[int] = (2, 2, 2)
    origin: Sequence[float] = (-1.0, -1.0, -1.0)
    extent: Sequence[float] = (2.0, 2.0, 2.0)
    order: int = 2

    def coeffs_per_vertex(self) -> int:
        return {0: 1, 1: 1 + self.dim, 2: 1 + self.dim + self.dim * (self.dim + 1) // 2}[self.order]

    def vertex_count(self) -> int:
        n = 1
        for a in range(self.dim):
            n *= int(self.resolution[a])
        return n

    def coeff_total(self) -> int:
        return self.vertex_count() * self.coeffs_per_vertex()

    def spacing(self, axis: int) -> float:
        return self.extent[axis] / (self.resolution[axis] - 1)

    def _c(self) -> _Spec:
        res = list(self.resolution) + [1] * (3 - len(self.resolution))
        org = list(self.origin) + [0.0] * (3 - len(self.origin))
        ext = list(self.extent) + [1.0] * (3 - len(self.extent))
        return _Spec(self.dim, (C.c_int * 3)(*map(int, res[:3])), (C.c_double * 3)(*map(float, org[:3])),
                     (C.c_double * 3)(*map(float, ext[:3])), self.order)


class InitMode(IntEnum):
    """tg::InitMode (taylor_grid.hpp:17)."""
    Zeros = 0
    Constant = 1
    SmallUniform = 2
    HashGaussian = 3  # device-side epsilon*N(0,1) (large synthetic grids)


@dataclass
class InitOptions:
    """tg::InitOptions (taylor_grid.hpp:19-25)."""
    mode: InitMode = InitMode.Zeros
    constant: float = 0.0
    epsilon: float = 1e-4
    seed: int = 0
    memory_cap_bytes: int = 4 << 30


@dataclass
class LossConfig:
    """tg::LossConfig (sdf_loss.hpp:15-25). eikonal_point_source: the batch
    itself (ReuseBatch, default) or |batch| fresh uniform points drawn from the
    step's Rng (FreshUniform, sdf_loss.cpp:274-283)."""
    lambda1: float = 1e-4
    lambda2: float = 2e-5
    k: float = 50.0
    use_weighting: bool = True
    use_tv: bool = True
    batch_size: int = 8192
    differentiate_weight: bool = False
    eikonal_point_source: int = 0  # EikonalPointSource

    def _c(self) -> _Loss:
        return _Loss(self.lambda1, self.lambda2, self.k, int(self.use_weighting), int(self.use_tv),
                     int(self.differentiate_weight))


class EikonalPointSource(IntEnum):
    """tg::EikonalPointSource (sdf_loss.hpp:13)."""
    ReuseBatch = 0
    FreshUniform = 1


class Rng:
    """tg::Rng (rng.hpp:14-74) on the host: mt19937_64, the reference's
    index / uniform_in_box draws (same streams as the reference)."""

    def __init__(self, seed: int):
        h = C.c_void_p()
        _check(lib().tgcu_rng_create(int(seed), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().tgcu_rng_destroy(self._h)
            self._h = None

    def index(self, n: int, count: int) -> np.ndarray:
        out = np.empty(int(count), dtype=np.int64)
        _check(lib().tgcu_rng_index(self._h, int(n), int(count), _ptr(out)))
        return out

    def uniform_in_box(self, dim: int, lo, hi, count: int) -> np.ndarray:
        """count points (count x 3, fp64; z = 0 in 2D)."""
        lo3 = np.ascontiguousarray(np.asarray(list(lo) + [0.0] * 3, dtype=np.float64)[:3])
        hi3 = np.ascontiguousarray(np.asarray(list(hi) + [0.0] * 3, dtype=np.float64)[:3])
        out = np.empty((int(count), 3), dtype=np.float64)
        _check(lib().tgcu_rng_uniform_box(self._h, int(dim), _ptr(lo3), _ptr(hi3), int(count), _ptr(out)))
        return out


@dataclass
class LossTerms:
    """tg::LossTerms (schedule.hpp:43-48)."""
    total: float = 0.0
    fit: float = 0.0
    eik: float = 0.0
    tv: float = 0.0

    @staticmethod
    def _from(t: _Terms) -> "LossTerms":
        return LossTerms(t.total, t.fit, t.eik, t.tv)

    def as_array(self):
        return np.array([self.total, self.fit, self.eik, self.tv])


@dataclass
class AdamConfig:
    """tg::AdamConfig (adam.hpp:9-14)."""
    lr: float = 0.003
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    def _c(self) -> _Adam:
        return _Adam(self.lr, self.beta1, self.beta2, self.eps)


# ---- array plumbing ---------------------------------------------------------


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _dev_f32(t, cols: int, what: str):
    """A device tensor passed straight to the C ABI: contiguous fp32 CUDA (n, cols)."""
    import torch
    if t.dtype != torch.float32:
        raise TypeError(f"{what}: device array must be float32, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError(f"{what}: torch tensor must live on a CUDA device")
    if t.dim() != 2 or t.shape[1] != cols or not t.is_contiguous():
        raise ValueError(f"{what}: expected a contiguous (n, {cols}) tensor, got shape {tuple(t.shape)}")
    return t


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        return C.c_void_p(x.data_ptr())
    return x.ctypes.data_as(C.c_void_p)


def _host_f32(x, cols: int) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    if cols == 3 and a.ndim == 2 and a.shape[1] == 2:  # 2D points -> pad z
        a = np.ascontiguousarray(np.concatenate([a, np.zeros((a.shape[0], 1), np.float32)], 1))
    return a.reshape(-1, cols)


class TaylorGrid:
    """Device-resident tg::TaylorGrid (taylor_grid.hpp:32-44) plus its AdamState
    and gradient buffer. ``coeffs`` round-trips the reference AoS layout."""

    def __init__(self, spec: GridSpec, opts: Optional[InitOptions] = None, device: int = 0):
        self.spec = spec
        h = C.c_void_p()
        o = opts or InitOptions()
        ci = _Init(int(o.mode), o.constant, o.epsilon, o.seed, o.memory_cap_bytes)
        _check(lib().tgcu_grid_create(C.byref(spec._c()), C.byref(ci), device, C.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            lib().tgcu_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def coeff_total(self) -> int:
        return int(lib().tgcu_grid_coeff_total(self._h))

    @property
    def coeffs(self) -> np.ndarray:
        out = np.empty(self.coeff_total(), dtype=np.float64)
        _check(lib().tgcu_grid_download_f64(self._h, _ptr(out), out.size))
        return out

    @coeffs.setter
    def coeffs(self, values):
        a = np.ascontiguousarray(values, dtype=np.float64).ravel()
        _check(lib().tgcu_grid_upload_f64(self._h, _ptr(a), a.size))

    def coeffs_f32(self) -> np.ndarray:
        out = np.empty(self.coeff_total(), dtype=np.float32)
        _check(lib().tgcu_grid_download_f32(self._h, _ptr(out), out.size, TGCU_HOST))
        return out

    def set_coeffs_f32(self, values):
        a = np.ascontiguousarray(values, dtype=np.float32).ravel()
        _check(lib().tgcu_grid_upload_f32(self._h, _ptr(a), a.size, TGCU_HOST))

    def device_coeffs_ptr(self) -> int:
        return int(lib().tgcu_grid_coeffs(self._h) or 0)

    def grad_ptr(self) -> int:
        p = lib().tgcu_grid_grad(self._h)
        if not p:
            _check(6)
        return int(p)

    def grad(self) -> np.ndarray:
        """Download the grid-owned gradient buffer (fp32 -> fp64)."""
        n = self.coeff_total()
        out = np.empty(n, dtype=np.float64)
        _check(lib().tgcu_grad_download_f64(self._h, None, _ptr(out), n))
        return out

    def zero_grad(self):
        _check(lib().tgcu_grad_zero(self._h, C.c_void_p(self.grad_ptr()), None))

    STEP_AUTO, STEP_BRICK, STEP_SINGLE = 0, 1, 2

    def set_step_path(self, path: int):
        """Fused-step path (tgcu_grid_set_step_path): STEP_AUTO, STEP_BRICK
        (binning + brick kernel + finalize) or STEP_SINGLE (one cooperative
        launch, for small grids such as BASELINE configs[0])."""
        _check(lib().tgcu_grid_set_step_path(self._h, int(path)))
        return self

    def set_deterministic(self, on: bool = True):
        """Bit-reproducible fused steps (tgcu_grid_set_deterministic): canonical
        summation orders, the reference's --deterministic (run_config.cpp:239-242)."""
        _check(lib().tgcu_grid_set_deterministic(self._h, 1 if on else 0))

    def all_finite(self) -> bool:
        r = C.c_int()
        _check(lib().tgcu_grid_all_finite(self._h, C.byref(r)))
        return bool(r.value)

    # AdamState (adam.hpp:17-32)
    def adam_reset(self, cfg: AdamConfig = AdamConfig()):
        _check(lib().tgcu_adam_reset(self._h, C.byref(cfg._c())))

    @property
    def adam_t(self) -> int:
        t = C.c_int64()
        lib().tgcu_adam_get_t(self._h, C.byref(t))
        return t.value

    def adam_moments(self):
        n = self.coeff_total()
        m = np.empty(n)
        v = np.empty(n)
        _check(lib().tgcu_adam_download_f64(self._h, _ptr(m), _ptr(v), n))
        return m, v

    @property
    def steps_launched(self) -> int:
        n = C.c_int64()
        lib().tgcu_grid_steps_launched(self._h, C.byref(n))
        return n.value

    def sync(self) -> LossTerms:
        t = _Terms()
        _check(lib().tgcu_sync(self._h, C.byref(t)))
        return LossTerms._from(t)

    def profile_begin(self, every: int = 1):
        """Time the fused brick launches (every `every`-th one) until profile_end."""
        _check(lib().tgcu_profile_every(self._h, int(every)))
        _check(lib().tgcu_profile_begin(self._h))

    def profile_end(self):
        """(summed brick-kernel device ms, launches) since profile_begin."""
        ms, n = C.c_double(), C.c_int()
        _check(lib().tgcu_profile_end(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def trace(self, count: int):
        arr = (_Terms * count)()
        _check(lib().tgcu_trace(self._h, arr, count))
        return np.array([[t.total, t.fit, t.eik, t.tv] for t in arr])


def init_grid(spec: GridSpec, opts: Optional[InitOptions] = None, device: int = 0) -> TaylorGrid:
    """init_grid (taylor_grid.cpp:162-188)."""
    return TaylorGrid(spec, opts, device)


# ---- queries ----------------------------------------------------------------


def eval(grid: TaylorGrid, points, sorted_points: bool = False) -> np.ndarray:  # noqa: A001
    """Batched eval (taylor_grid.cpp:197-199). points: (n, dim|3) host array or a
    CUDA tensor (n, 3) float32. Returns fp64 numpy (host input) or fills a tensor."""
    v, _ = _eval(grid, points, False, sorted_points)
    return v


def eval_with_spatial_gradient(grid: TaylorGrid, points, sorted_points: bool = False):
    """Batched eval_with_spatial_gradient (taylor_grid.cpp:201-203) -> (values, grads)."""
    return _eval(grid, points, True, sorted_points)


def _eval(grid, points, want_grad, sorted_points):
    flags = TGCU_SORTED if sorted_points else 0
    if _is_torch(points):
        import torch
        _dev_f32(points, 3, "eval")
        n = points.shape[0]
        vals = torch.empty(n, dtype=torch.float32, device=points.device)
        grads = torch.empty((n, 3), dtype=torch.float32, device=points.device) if want_grad else None
        _check(lib().tgcu_eval(grid.handle, _ptr(points), n, _ptr(vals), _ptr(grads), flags,
                               C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return vals, grads
    p = _host_f32(points, 3)
    n = p.shape[0]
    vals = np.empty(n, dtype=np.float32)
    grads = np.empty((n, 3), dtype=np.float32) if want_grad else None
    _check(lib().tgcu_eval(grid.handle, _ptr(p), n, _ptr(vals), _ptr(grads), flags | TGCU_HOST, None))
    return vals.astype(np.float64), (grads.astype(np.float64)[:, :grid.spec.dim] if want_grad else None)


def query_brick_codes(grid: TaylorGrid) -> int:
    return int(lib().tgcu_query_brick_codes(grid.handle))


def sort_points(grid: TaylorGrid, points_dev, out_dev, perm_dev=None, offsets_dev=None):
    """Brick/Morton sort of device query points for the brick-binned query.
    offsets_dev: optional int64 CUDA tensor of query_brick_codes(grid)+1 entries."""
    import torch
    _dev_f32(points_dev, 3, "sort_points")
    _check(lib().tgcu_sort_points(grid.handle, _ptr(points_dev), points_dev.shape[0], _ptr(out_dev),
                                  _ptr(perm_dev), _ptr(offsets_dev),
                                  C.c_void_p(torch.cuda.current_stream().cuda_stream)))


def eval_device(grid: TaylorGrid, points_dev, values_dev, grads_dev=None, asynchronous: bool = False):
    """Direct-gather query of device points into preallocated device outputs."""
    import torch
    _check(lib().tgcu_eval(grid.handle, _ptr(points_dev), points_dev.shape[0], _ptr(values_dev), _ptr(grads_dev),
                           TGCU_ASYNC if asynchronous else 0,
                           C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return values_dev


def eval_sorted(grid: TaylorGrid, sorted_dev, offsets_dev=None, values_dev=None, grads_dev=None,
                asynchronous: bool = False):
    """Brick-binned query of sorted device points (tgcu_eval_sorted)."""
    import torch
    n = sorted_dev.shape[0]
    if values_dev is None:
        values_dev = torch.empty(n, dtype=torch.float32, device=sorted_dev.device)
    _check(lib().tgcu_eval_sorted(grid.handle, _ptr(sorted_dev), n, _ptr(offsets_dev), _ptr(values_dev),
                                  _ptr(grads_dev), TGCU_ASYNC if asynchronous else 0,
                                  C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return values_dev


# ---- backward ---------------------------------------------------------------


def _backprop(grid, points, upstream, upstream_vec, grad_ptr=None):
    p = _host_f32(points, 3)
    n = p.shape[0]
    up = None if upstream is None else np.ascontiguousarray(np.broadcast_to(np.asarray(upstream, np.float32), (n,)))
    uv = None
    if upstream_vec is not None:
        uv = _host_f32(np.broadcast_to(np.asarray(upstream_vec, np.float32).reshape(-1, np.shape(upstream_vec)[-1]),
                                       (n, np.shape(upstream_vec)[-1])), 3)
    gp = grad_ptr if grad_ptr is not None else grid.grad_ptr()
    _check(lib().tgcu_backprop(grid.handle, _ptr(p), _ptr(up), _ptr(uv), n, C.c_void_p(gp), TGCU_HOST, None))


def backprop_point(grid: TaylorGrid, points, upstream, grad_ptr=None):
    """backprop_point (taylor_grid.cpp:205-213), batched, into the grid's grad buffer."""
    _backprop(grid, points, upstream, None, grad_ptr)


def backprop_spatial_chain(grid: TaylorGrid, points, upstream_vec, grad_ptr=None):
    """backprop_spatial_chain (taylor_grid.cpp:215-221), batched."""
    _backprop(grid, points, None, upstream_vec, grad_ptr)


def backprop_value_and_spatial(grid: TaylorGrid, points, upstream, upstream_vec, grad_ptr=None):
    """backprop_value_and_spatial (taylor_grid.cpp:223-229), batched."""
    _backprop(grid, points, upstream, upstream_vec, grad_ptr)


# ---- losses / optimiser -----------------------------------------------------------


def adaptive_weight(d_hat: float, d: float, k: float) -> float:
    """adaptive_weight (sdf_loss.cpp:125-128); host scalar helper."""
    if not k > 0.0:
        raise ValueError("adaptive_weight: k must be > 0")

    def wp(x):
        return 1.0 - abs(2.0 / (1.0 + np.exp(-k * x)) - 1.0)
    return float(max(wp(d_hat), wp(d)))


def tv_loss(grid: TaylorGrid, with_grad: bool = False, scale: float = 1.0) -> float:
    """tv_loss (sdf_loss.cpp:155-257); with_grad accumulates into the grid grad buffer."""
    out = C.c_double()
    gp = C.c_void_p(grid.grad_ptr()) if with_grad else None
    _check(lib().tgcu_tv_loss(grid.handle, gp, scale, C.byref(out), None))
    return out.value


def _samples(samples):
    if _is_torch(samples):
        return _dev_f32(samples, 4, "samples"), 0
    a = np.ascontiguousarray(np.asarray(samples, dtype=np.float32)).reshape(-1, 4)
    return a, TGCU_HOST


def total_loss(grid: TaylorGrid, samples, cfg: LossConfig = LossConfig(), with_grad: bool = True) -> LossTerms:
    """total_loss (sdf_loss.cpp:259-292), unfused path; samples (n, 4) = x, y, z, gt.
    with_grad accumulates into the grid-owned gradient buffer."""
    s, flags = _samples(samples)
    t = _Terms()
    gp = C.c_void_p(grid.grad_ptr()) if with_grad else None
    _check(lib().tgcu_total_loss(grid.handle, _ptr(s), s.shape[0], C.byref(cfg._c()), gp, C.byref(t), flags, None))
    return LossTerms._from(t)


def recon_loss(grid: TaylorGrid, samples, cfg: LossConfig = LossConfig(), scale: float = 1.0,
               with_grad: bool = True) -> float:
    """recon_loss (sdf_loss.cpp:130-135): mean weighted L1 residual; with_grad
    adds scale x its gradient into the grid-owned gradient buffer."""
    s, flags = _samples(samples)
    out = C.c_double()
    gp = C.c_void_p(grid.grad_ptr()) if with_grad else None
    _check(lib().tgcu_recon_loss(grid.handle, _ptr(s), s.shape[0], C.byref(cfg._c()), float(scale), gp,
                                 C.byref(out), flags, None))
    return out.value


def eikonal_loss(grid: TaylorGrid, points, scale: float = 1.0, with_grad: bool = True) -> float:
    """eikonal_loss (sdf_loss.cpp:137-153): mean (|grad f| - 1)^2 over the
    points (n, 3); with_grad adds scale x its gradient into the grid buffer."""
    if _is_torch(points):
        p, flags = _dev_f32(points, 3, "eikonal_loss"), 0
    else:
        p, flags = _host_f32(points, 3), TGCU_HOST
    out = C.c_double()
    gp = C.c_void_p(grid.grad_ptr()) if with_grad else None
    _check(lib().tgcu_eikonal_loss(grid.handle, _ptr(p), p.shape[0], float(scale), gp, C.byref(out), flags, None))
    return out.value


def adam_step(grid: TaylorGrid, grad_ptr: Optional[int] = None):
    """adam_step (adam.cpp:12-56) on the grid's coefficients with the grid's
    (or the given device) gradient buffer."""
    gp = grad_ptr if grad_ptr is not None else grid.grad_ptr()
    _check(lib().tgcu_adam_step(grid.handle, C.c_void_p(gp), None))


def train_step(grid: TaylorGrid, samples, cfg: LossConfig = LossConfig(), asynchronous: bool = False,
               stream=None, export_grad: bool = False, input_ready: bool = False,
               rng: Optional["Rng"] = None) -> Optional[LossTerms]:
    """One fused step: zero grad → total_loss → finite check → adam_step
    (schedule.cpp:66-92). Returns the LossTerms (None when asynchronous).
    export_grad also stores the full gradient in the grid grad buffer (validation).
    input_ready (device samples): the caller guarantees the samples are complete,
    so the step's binning overlaps the previous step's brick kernel.
    asynchronous=True with a host array: the copy to the device is queued on
    the library's copy stream and runs while earlier steps compute, so the
    array must stay alive AND unmodified until sync() (or until a later step
    is known to have consumed it): refilling one pinned buffer every step
    would overwrite samples whose copy is still in flight. Cycle through
    at least two buffers and sync() before reusing one."""
    s, flags = _samples(samples)
    if export_grad:
        flags |= TGCU_EXPORT_GRAD
    if cfg.eikonal_point_source == EikonalPointSource.FreshUniform and cfg.lambda1 > 0.0:
        # total_loss draws |batch| points with rng->uniform_in_box(origin, domain_max)
        if rng is None:
            raise ValueError("total_loss: fresh-uniform eikonal points need an rng")
        sp = grid.spec
        hi = [sp.origin[a] + sp.extent[a] for a in range(3)]
        eik = rng.uniform_in_box(sp.dim, sp.origin, hi, s.shape[0]).astype(np.float32)
        if not flags & TGCU_HOST:
            import torch
            eik = torch.from_numpy(eik).to(s.device)
        ef = flags | (TGCU_ASYNC if asynchronous else 0)
        t = _Terms()
        _check(lib().tgcu_train_step_fresh_eik(grid.handle, _ptr(s), s.shape[0], _ptr(eik), C.byref(cfg._c()),
                                               None if asynchronous else C.byref(t), ef,
                                               C.c_void_p(stream) if stream else None))
        return None if asynchronous else LossTerms._from(t)
    if input_ready and not flags & TGCU_HOST:
        flags |= TGCU_INPUT_READY
    if asynchronous:
        flags |= TGCU_ASYNC
        _check(lib().tgcu_train_step(grid.handle, _ptr(s), s.shape[0], C.byref(cfg._c()), None, flags,
                                     C.c_void_p(stream) if stream else None))
        return None
    t = _Terms()
    _check(lib().tgcu_train_step(grid.handle, _ptr(s), s.shape[0], C.byref(cfg._c()), C.byref(t), flags,
                                 C.c_void_p(stream) if stream else None))
    return LossTerms._from(t)


class TrainGraph:
    """CUDA-graph replay of small-grid fused steps (tgcu_train_graph_*): the
    steps train_step(grid, batches[i], cfg, asynchronous=True,
    input_ready=True) for i in 0..len(batches)-1 (an even count), captured
    once on `stream` (a torch.cuda.Stream or raw handle; a new stream if None)
    and replayed without a host call per step. The batches are CUDA float32
    (n, 4) tensors whose storage the graph keeps: refill them in place between
    replays. Errors are sticky and surface at grid.sync()."""

    def __init__(self, grid: TaylorGrid, batches, cfg: LossConfig = LossConfig(), stream=None):
        import torch
        self.grid = grid
        self.batches = [_dev_f32(b, 4, "samples") for b in batches]
        n = self.batches[0].shape[0]
        if any(b.shape[0] != n for b in self.batches):
            raise ValueError("train_graph_create: every batch needs the same size")
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.batches[0].device)
        ptrs = (C.c_void_p * len(self.batches))(*[b.data_ptr() for b in self.batches])
        h = C.c_void_p()
        _check(lib().tgcu_train_graph_create(grid.handle, ptrs, len(self.batches), n, C.byref(cfg._c()),
                                             C.c_void_p(self._raw(self.stream)), C.byref(h)))
        self._h = h

    @staticmethod
    def _raw(stream):
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)

    @property
    def steps(self) -> int:
        return len(self.batches)

    def replay(self, stream=None):
        s = self.stream if stream is None else stream
        _check(lib().tgcu_train_graph_launch(self._h, C.c_void_p(self._raw(s))))

    def close(self):
        if getattr(self, "_h", None):
            lib().tgcu_train_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- seeded inputs ------------------------------------------------------------------

SHAPE_SPHERE, SHAPE_C1_2D, SHAPE_PRIMS = 0, 1, 2


def sample(shape: int, dim: int, seed: int, n: int, near_frac: float = 0.0, sigma: float = 0.01,
           param0: float = 0.0) -> np.ndarray:
    """Seeded (x, y, z, gt) samples, reference Rng mappings (rng.hpp:14-74)."""
    out = np.empty((n, 4), dtype=np.float32)
    _check(lib().tgcu_sample(shape, dim, seed, n, near_frac, sigma, param0, _ptr(out)))
    return out


def sample_uniform(dim: int, seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    out = np.empty((n, 3), dtype=np.float32)
    _check(lib().tgcu_sample_uniform(dim, seed, n, lo, hi, _ptr(out)))
    return out


def sample_uniform_device(dim: int, seed: int, out, lo: float = -1.0, hi: float = 1.0, stream=None):
    """Fill a CUDA float32 tensor (n, 3) with hashed uniform points (device-side)."""
    _check(lib().tgcu_sample_uniform_device(dim, seed, out.shape[0], lo, hi, _ptr(out),
                                            C.c_void_p(stream) if stream else None))


def shape_sdf(shape: int, dim: int, param0: float, pts) -> np.ndarray:
    p = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    out = np.empty(p.shape[0])
    _check(lib().tgcu_shape_sdf(shape, dim, param0, _ptr(p), p.shape[0], _ptr(out)))
    return out


# ---- stage transitions, lattice query, .tgrid I/O ---------------------


def _res3(res, dim):
    r = [int(x) for x in res] + [1] * 3
    return (C.c_int * 3)(*r[:3])


def upsample(grid: TaylorGrid, new_resolution) -> TaylorGrid:
    """upsample (taylor_grid.cpp:273-284): a new device grid at new_resolution
    (>= the old one per axis) holding the multilinear resample of the
    coefficients. Raises ValueError "upsample: resolution may not shrink"."""
    s = grid.spec
    for a in range(s.dim):
        if int(new_resolution[a]) < int(s.resolution[a]):
            raise ValueError(f"upsample: resolution may not shrink (axis {a})")
    res = tuple(int(new_resolution[a]) for a in range(s.dim)) + tuple(s.resolution[s.dim:])
    ns = GridSpec(dim=s.dim, resolution=res, origin=tuple(s.origin), extent=tuple(s.extent), order=s.order)
    out = TaylorGrid(ns, InitOptions(memory_cap_bytes=1 << 62), grid.device)
    _check(lib().tgcu_grid_upsample(grid.handle, out.handle, 0, None))
    return out


def multilinear_resample(old_spec: GridSpec, data, channels: int, new_resolution) -> np.ndarray:
    """multilinear_resample (taylor_grid.cpp:231-271) of host data (fp32 in/out)."""
    a = np.ascontiguousarray(np.asarray(data, dtype=np.float32)).ravel()
    nr = _res3(new_resolution, old_spec.dim)
    nv = 1
    for ax in range(old_spec.dim):
        nv *= nr[ax]
    out = np.empty(nv * channels, dtype=np.float32)
    _check(lib().tgcu_multilinear_resample(C.byref(old_spec._c()), _ptr(a), a.size, channels, nr, _ptr(out),
                                           TGCU_HOST, None))
    return out


@dataclass
class ScalarField3:
    """tg::ScalarField3 (marching.hpp:12-25): lattice values, x fastest."""
    res: tuple
    origin: tuple
    extent: tuple
    values: np.ndarray

    def at(self, x: int, y: int, z: int) -> float:
        return float(self.values[(z * self.res[1] + y) * self.res[0] + x])

    def position(self, x: int, y: int, z: int):
        return tuple(self.origin[a] + self.extent[a] * v / (self.res[a] - 1) for a, v in enumerate((x, y, z)))


@dataclass
class ScalarField2:
    """tg::ScalarField2 (marching.hpp:27-37)."""
    res: tuple
    origin: tuple
    extent: tuple
    values: np.ndarray


def _lattice(grid: TaylorGrid, lat, out=None, stream=None):
    n = 1
    for a in range(grid.spec.dim):
        n *= int(lat[a])
    if out is not None:  # device output tensor
        _check(lib().tgcu_sample_grid_field(grid.handle, _res3(lat, grid.spec.dim), _ptr(out), 0,
                                            C.c_void_p(stream) if stream else None))
        return out
    vals = np.empty(n, dtype=np.float32)
    _check(lib().tgcu_sample_grid_field(grid.handle, _res3(lat, grid.spec.dim), _ptr(vals), TGCU_HOST, None))
    return vals.astype(np.float64)


def sample_grid_field(grid: TaylorGrid, res, out=None, stream=None):
    """sample_grid_field (marching.cpp:53-58) -> ScalarField3; with `out` (a CUDA
    float32 tensor of prod(res)) the values stay on the device."""
    if grid.spec.dim != 3:
        raise ValueError("sample_grid_field: needs a 3D grid")
    for r in res[:3]:
        if int(r) < 2:
            raise ValueError("sample_field3: resolution must be >= 2 per axis")
    v = _lattice(grid, res, out, stream)
    if out is not None:
        return v
    return ScalarField3(tuple(int(r) for r in res[:3]), tuple(grid.spec.origin[:3]), tuple(grid.spec.extent[:3]), v)


def sample_grid_field2(grid: TaylorGrid, nx: int, ny: int) -> ScalarField2:
    """The CLI's 2D lattice (tools/main.cpp:33-45) -> ScalarField2."""
    v = _lattice(grid, (nx, ny))
    return ScalarField2((nx, ny), tuple(grid.spec.origin[:2]), tuple(grid.spec.extent[:2]), v)


class StoragePrecision(IntEnum):
    """tg::StoragePrecision (grid_io.hpp:9)."""
    F64 = 0
    F32 = 1


def save_tgrid(grid: TaylorGrid, path, precision: StoragePrecision = StoragePrecision.F64) -> None:
    """save_tgrid (grid_io.cpp:44-65)."""
    _check(lib().tgcu_save_tgrid(grid.handle, os.fspath(path).encode(), int(precision)))


def load_tgrid(path, device: int = 0) -> TaylorGrid:
    """load_tgrid (grid_io.cpp:67-109) -> a device grid (F64 payloads narrowed to fp32)."""
    h = C.c_void_p()
    _check(lib().tgcu_load_tgrid(os.fspath(path).encode(), device, C.byref(h)))
    cs = _Spec()
    lib().tgcu_grid_spec_of(h, C.byref(cs))
    spec = GridSpec(dim=cs.dim, resolution=tuple(cs.res[:cs.dim]), origin=tuple(cs.origin[:cs.dim]),
                    extent=tuple(cs.extent[:cs.dim]), order=cs.order)
    g = TaylorGrid.__new__(TaylorGrid)
    g.spec, g._h, g.device = spec, h, device
    return g


def tgrid_file_size(spec: GridSpec, precision: StoragePrecision = StoragePrecision.F64) -> int:
    """tgrid_file_size (grid_io.cpp:36-40)."""
    n = int(lib().tgcu_tgrid_file_size(C.byref(spec._c()), int(precision)))
    if n < 0:
        raise ValueError("tgrid_file_size: invalid spec")
    return n


def draw_batch(pool_dev, n: int, seed: int, step: int, out_dev=None, stream=None):
    """Device batch draw with replacement from a (pool_n, 4) CUDA float32 pool
    (SdfProblem::compute, sdf_fit.cpp:21-23; hashed stream)."""
    import torch
    if out_dev is None:
        out_dev = torch.empty((n, 4), dtype=torch.float32, device=pool_dev.device)
    _check(lib().tgcu_draw_batch(_ptr(pool_dev), pool_dev.shape[0], n, seed, step, _ptr(out_dev),
                                 C.c_void_p(stream) if stream else None))
    return out_dev
