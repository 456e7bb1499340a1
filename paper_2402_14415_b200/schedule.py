"""Progressive training driver: Schedule / run_schedule / fit_sdf on the device.

Mirrors schedule.hpp:13-86 / schedule.cpp:13-129 and sdf_fit.hpp:11-55 /
sdf_fit.cpp:14-105 of /root/reference/proj/core. The reference's plugin point
is ``TrainProblem::compute(grid, grad) -> LossTerms``; here a problem comes in
two flavours:

* fused (default, ``TrainProblem.fused = True``): ``batch(grid, step)`` returns
  the step's samples and ``compute`` runs the fused device step
  {loss + backward + TV + finite check + Adam} (tgcu_train_step), so
  run_schedule adds nothing per step;
* unfused (``fused = False``): ``compute(grid)`` accumulates into the grid's
  gradient buffer (e.g. with total_loss / backprop_*) and returns LossTerms;
  run_schedule zeroes the buffer before and runs adam_step after, exactly the
  reference loop (schedule.cpp:84-92).

Per stage: upsample when the resolution changes (taylor_grid.cpp:273-284),
fresh Adam moments (schedule.cpp:79), on_stage_start, then the steps. A
non-finite loss raises NumericalError "run_schedule: non-finite loss at stage
s step k" (schedule.cpp:88-91).
"""
from __future__ import annotations

import io
import re
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import (AdamConfig, GridSpec, InitOptions, LossConfig, LossTerms, NumericalError, Rng, TaylorGrid, _check,
               _ptr, adam_step, draw_batch, eval as tg_eval, init_grid, lib, train_step, upsample)

__all__ = ["Stage", "Schedule", "TraceRow", "ScheduleResult", "TrainProblem", "BatchProblem", "SdfProblem",
           "run_schedule", "trace_csv_string", "write_trace_csv", "FitOptions", "FitReport", "FitResult", "fit_sdf",
           "mean_abs_error"]


@dataclass
class Stage:
    """Schedule::Stage (schedule.hpp:17-20)."""
    resolution: Sequence[int] = (2, 2, 2)
    steps: int = 0


@dataclass
class Schedule:
    """tg::Schedule (schedule.hpp:16-39)."""
    stages: List[Stage] = field(default_factory=list)

    def validate(self, dim: int) -> None:
        """Schedule::validate (schedule.cpp:13-25)."""
        if not self.stages:
            raise ValueError("Schedule: needs at least one stage")
        for s, st in enumerate(self.stages):
            if st.steps < 0:
                raise ValueError("Schedule: negative step count")
            for a in range(dim):
                if st.resolution[a] < 2:
                    raise ValueError("Schedule: stage resolution must be >= 2")
                if s > 0 and st.resolution[a] < self.stages[s - 1].resolution[a]:
                    raise ValueError("Schedule: resolutions must be non-decreasing across stages")

    def total_steps(self) -> int:
        return sum(st.steps for st in self.stages)

    @staticmethod
    def progressive(target: Sequence[int], dim: int, total_steps: int) -> "Schedule":
        """Schedule::progressive (schedule.cpp:27-54): target/4, /2, /1 floored
        at 4 vertices (capped at the target), equal split, duplicates
        collapsed, remainder to the last stage."""
        sch = Schedule()
        for d in (4, 2, 1):
            res = [2, 2, 2]
            same_as_target = True
            for a in range(dim):
                res[a] = min(max(4, int(target[a]) // d), int(target[a]))
                same_as_target &= res[a] == int(target[a])
            if sch.stages and all(res[a] == sch.stages[-1].resolution[a] for a in range(dim)):
                continue
            sch.stages.append(Stage(tuple(res), total_steps // 3))
            if same_as_target:
                break
        sch.stages[-1].steps += total_steps - sch.total_steps()
        return sch

    @staticmethod
    def single(target: Sequence[int], steps: int) -> "Schedule":
        return Schedule([Stage(tuple(target), steps)])


@dataclass
class TraceRow:
    """tg::TraceRow (schedule.hpp:50-56)."""
    step: int
    stage: int
    resolution: tuple
    loss: LossTerms
    wall_ms: float


@dataclass
class ScheduleResult:
    """tg::ScheduleResult (schedule.hpp:68-72)."""
    grid: TaylorGrid
    trace: List[TraceRow]
    stage_seconds: List[float]


class TrainProblem:
    """tg::TrainProblem (schedule.hpp:60-66); see the module docstring."""
    fused = True
    loss: LossConfig = LossConfig()

    def batch(self, grid: TaylorGrid, step: int):
        """Samples (n, 4) of global step `step` (host array or CUDA tensor)."""
        raise NotImplementedError

    def compute(self, grid: TaylorGrid, step: int = 0, asynchronous: bool = False) -> Optional[LossTerms]:
        return train_step(grid, self.batch(grid, step), self.loss, asynchronous=asynchronous,
                          rng=getattr(self, "rng", None))

    def on_stage_start(self, grid: TaylorGrid, stage: int) -> None:
        pass


class BatchProblem(TrainProblem):
    """Feeds a fixed list of batches in order (the parity harness / cmd_bench shape)."""

    def __init__(self, batches, loss: LossConfig = LossConfig()):
        self.batches = batches
        self.loss = loss

    def batch(self, grid, step):
        return self.batches[step]


class SdfProblem(TrainProblem):
    """SdfProblem (sdf_fit.cpp:14-32): each step draws min(batch_size, pool)
    samples with replacement from the training pool.

    exact_stream=True draws the indices with the reference Rng (mt19937_64
    seeded with `seed`, Rng::index, sdf_fit.cpp:22) on the host, so the batches
    equal the reference's; otherwise the draw is a device kernel over the
    device-resident pool (tgcu_draw_batch; hashed stream, same distribution)."""

    def __init__(self, train: np.ndarray, loss: LossConfig, seed: int, exact_stream: bool = False, device: int = 0):
        self.loss = loss
        self.train = np.ascontiguousarray(np.asarray(train, dtype=np.float32)).reshape(-1, 4)
        self.n = min(int(loss.batch_size), self.train.shape[0])
        self.seed = seed
        self.exact = exact_stream
        # the reference Rng: with exact_stream one stream serves the batch
        # draws and (FreshUniform) the eikonal points, in the reference's order
        # (sdf_fit.cpp:21-24); with device draws it serves the eikonal points
        self.rng = Rng(seed)
        if not exact_stream:
            import torch
            self.pool = torch.from_numpy(self.train).to(f"cuda:{device}")
            self.out = torch.empty((self.n, 4), dtype=torch.float32, device=self.pool.device)

    def batch(self, grid, step):
        if self.exact:
            return self.train[self.rng.index(self.train.shape[0], self.n)]
        import torch
        return draw_batch(self.pool, self.n, self.seed, step, self.out,
                          stream=torch.cuda.current_stream().cuda_stream)


_STEP_RE = re.compile(r"stage 0 step (\d+)")


def _restage(e: Exception, stage: int, offset: int) -> Exception:
    """Rewrite the library's "stage 0 step <launch index>" with run_schedule's
    stage and per-stage step (schedule.cpp:88-91)."""
    msg = str(e)
    m = _STEP_RE.search(msg)
    if m:
        msg = msg[:m.start()] + f"stage {stage} step {int(m.group(1)) - offset}" + msg[m.end():]
    return type(e)(msg)


def run_schedule(problem: TrainProblem, schedule: Schedule, grid: TaylorGrid, adam: AdamConfig = AdamConfig(),
                 asynchronous: bool = False) -> ScheduleResult:
    """run_schedule (schedule.cpp:62-108) on the device.

    asynchronous=True (fused problems) issues a stage's steps without a host
    round trip per step and reads the loss trace back at the end of the stage
    (or every 4096 steps); wall_ms is then the stage's mean step time."""
    schedule.validate(grid.spec.dim)
    trace: List[TraceRow] = []
    stage_seconds: List[float] = []
    gstep = 0
    dim = grid.spec.dim
    for si, st in enumerate(schedule.stages):
        if any(int(st.resolution[a]) != int(grid.spec.resolution[a]) for a in range(dim)):
            grid = upsample(grid, st.resolution)
        grid.adam_reset(adam)  # moments reset with each stage
        problem.on_stage_start(grid, si)
        res = tuple(int(r) for r in st.resolution[:3])
        t_stage = time.perf_counter()
        if asynchronous and problem.fused and st.steps > 0:
            k = 0
            while k < st.steps:
                w = min(4096, st.steps - k)
                off = grid.steps_launched - k
                t0 = time.perf_counter()
                try:
                    for j in range(w):
                        problem.compute(grid, gstep + k + j, asynchronous=True)
                    grid.sync()
                    rows = grid.trace(w)
                except (NumericalError, ValueError) as e:
                    raise _restage(e, si, off) from e
                ms = (time.perf_counter() - t0) * 1e3 / w
                for j in range(w):
                    r = rows[j]
                    trace.append(TraceRow(gstep + k + j, si, res, LossTerms(*r), ms))
                k += w
            gstep += st.steps
        else:
            for k in range(st.steps):
                t0 = time.perf_counter()
                off = grid.steps_launched - k
                try:
                    if problem.fused:
                        terms = problem.compute(grid, gstep)
                    else:
                        grid.zero_grad()
                        terms = problem.compute(grid, gstep)
                except (NumericalError, ValueError) as e:
                    raise _restage(e, si, off) from e
                if not np.isfinite(terms.total):
                    raise NumericalError(f"run_schedule: non-finite loss at stage {si} step {k}")
                if not problem.fused:
                    try:
                        adam_step(grid)
                    except NumericalError as e:
                        raise NumericalError(f"{e} (stage {si} step {k})") from e
                trace.append(TraceRow(gstep, si, res, terms, (time.perf_counter() - t0) * 1e3))
                gstep += 1
        stage_seconds.append(time.perf_counter() - t_stage)
    return ScheduleResult(grid, trace, stage_seconds)


def trace_csv_string(trace: List[TraceRow], fit_label: str = "recon") -> str:
    """trace_csv_string (schedule.cpp:110-120), same columns and formats."""
    out = io.StringIO()
    out.write(f"step,stage,resolution,total_loss,{fit_label},eik,tv,wall_ms\n")
    for r in trace:
        rz = tuple(r.resolution) + (0, 0, 0)
        out.write(f"{r.step},{r.stage},{rz[0]}x{rz[1]}x{rz[2]},{r.loss.total:.17g},{r.loss.fit:.17g},"
                  f"{r.loss.eik:.17g},{r.loss.tv:.17g},{r.wall_ms:.3f}\n")
    return out.getvalue()


def write_trace_csv(path, trace: List[TraceRow], fit_label: str = "recon") -> None:
    with open(path, "w") as f:
        f.write(trace_csv_string(trace, fit_label))


# ---- fit_sdf (sdf_fit.hpp / sdf_fit.cpp) ---------------------------------------------


@dataclass
class FitOptions:
    """tg::FitOptions (sdf_fit.hpp:11-21)."""
    loss: LossConfig = field(default_factory=LossConfig)
    adam: AdamConfig = field(default_factory=AdamConfig)
    schedule: Schedule = field(default_factory=Schedule)  # empty -> default progressive plan
    total_steps: int = 3000
    holdout_fraction: float = 0.0
    seed: int = 1
    metric_hook: Optional[Callable[[TaylorGrid], dict]] = None
    exact_stream: bool = False  # reference batch-index stream (host) instead of the device draw
    asynchronous: bool = True


@dataclass
class FitReport:
    """tg::FitReport (sdf_fit.hpp:23-35)."""
    final_loss: LossTerms = field(default_factory=LossTerms)
    stage_seconds: List[float] = field(default_factory=list)
    total_seconds: float = 0.0
    total_steps: int = 0
    train_samples: int = 0
    holdout_samples: int = 0
    holdout_mae: float = 0.0
    metrics: dict = field(default_factory=dict)

    def to_json(self) -> dict:
        f = self.final_loss
        return {"final_loss": {"total": f.total, "recon": f.fit, "eik": f.eik, "tv": f.tv},
                "stage_seconds": list(self.stage_seconds), "total_seconds": self.total_seconds,
                "total_steps": self.total_steps, "train_samples": self.train_samples,
                "holdout_samples": self.holdout_samples, "holdout_mae": self.holdout_mae,
                "metrics": dict(self.metrics), "config": {}}


@dataclass
class FitResult:
    grid: TaylorGrid
    report: FitReport
    trace: List[TraceRow]


def mean_abs_error(grid: TaylorGrid, samples) -> float:
    """mean_abs_error (sdf_fit.cpp:36-50): mean |eval - gt| (device query)."""
    s = np.asarray(samples, dtype=np.float64).reshape(-1, 4)
    if s.shape[0] == 0:
        return 0.0
    v = tg_eval(grid, s[:, :3])
    return float(np.mean(np.abs(v - s[:, 3])))


def fit_sdf(samples, spec: GridSpec, options: FitOptions = FitOptions(), device: int = 0) -> FitResult:
    """fit_sdf (sdf_fit.cpp:52-105): seeded shuffle + holdout split
    (sdf_fit.cpp:58-74, reference Rng), progressive schedule by default,
    SdfProblem batches, run_schedule on the device, holdout MAE."""
    import ctypes as C
    s = np.ascontiguousarray(np.asarray(samples, dtype=np.float64)).reshape(-1, 4)
    if s.shape[0] == 0:
        raise ValueError("fit_sdf: sample set is empty")
    if options.loss.k <= 0 or options.loss.lambda1 < 0 or options.loss.lambda2 < 0:
        raise ValueError("LossConfig: invalid weights")
    n = s.shape[0]
    order = np.empty(n, dtype=np.uint32)
    _check(lib().tgcu_shuffle_order((options.seed ^ 0x5DEECE66D) & (2 ** 64 - 1), n, _ptr(order)))
    holdout_n = min(n - 1, int(options.holdout_fraction * n))
    train = s[order[:n - holdout_n]]
    holdout = s[order[n - holdout_n:]]
    schedule = options.schedule if options.schedule.stages else Schedule.progressive(spec.resolution, spec.dim,
                                                                                       options.total_steps)
    start = GridSpec(dim=spec.dim, resolution=tuple(schedule.stages[0].resolution[:spec.dim]),
                     origin=tuple(spec.origin), extent=tuple(spec.extent), order=spec.order)
    grid = init_grid(start, device=device)
    problem = SdfProblem(train, options.loss, options.seed, options.exact_stream, device)
    t0 = time.perf_counter()
    sr = run_schedule(problem, schedule, grid, options.adam, asynchronous=options.asynchronous)
    t1 = time.perf_counter()
    rep = FitReport(stage_seconds=sr.stage_seconds, total_seconds=t1 - t0, total_steps=schedule.total_steps(),
                    train_samples=n - holdout_n, holdout_samples=holdout_n)
    if sr.trace:
        rep.final_loss = sr.trace[-1].loss
    if holdout_n > 0:
        rep.holdout_mae = mean_abs_error(sr.grid, holdout)
    if options.metric_hook:
        rep.metrics = options.metric_hook(sr.grid)
    return FitResult(sr.grid, rep, sr.trace)
