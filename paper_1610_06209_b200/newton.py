"""Sketched Newton for logistic regression on the device — Python mirror of
proj/include/spinners/newton_sketch.hpp / proj/src/newton_sketch.cpp.

=====================  ==========================================================
this module            reference
=====================  ==========================================================
``LogisticProblem``    ``LogisticProblem`` (newton_sketch.hpp:13-21; .cpp:28-37)
``SketchConfig``       ``SketchConfig`` (newton_sketch.hpp:23-33; .cpp:39-43)
``NewtonTrace``        ``NewtonTrace`` (newton_sketch.hpp:35-42)
``loss``/``gradient``  ``loss``/``gradient`` (.cpp:45-61) — one fused pass over A
``hessian_sqrt``       ``hessian_sqrt`` (.cpp:63-72)
``sketched_step``      ``sketched_step`` (.cpp:103-122)
``solve``              ``solve`` (.cpp:124-183)
``generate_ar1_problem``  ``generate_ar1_problem`` (.cpp:185-204)
=====================  ==========================================================

Features and labels live on the device in fp32 (the reference's fp64 features
rounded once); iterates, steps, gradients, losses and every reduction are fp64.
The sketch is the spinner SketchOperator of this package with the Hessian row
scales folded into its first pass; the d x d system is solved by a blocked fp64
Cholesky with the reference's ridge retry.  No CPU fallback: every numeric step
runs in the sm_100a library.
"""
from __future__ import annotations

import concurrent.futures
import ctypes as C
import dataclasses
import time
from typing import List, Optional

import numpy as np

from . import (DimensionError, DomainError, SingularSystemError, SketchOperator, SpinnerVariant, _check, _i32, _i64,
               _lib, _sig, _stream_ptr, _torch, _u64, _vp, mix_seed)

_dbl = C.c_double
_newton_create = _sig("spn_newton_create", C.c_int, [C.POINTER(_vp), _i64, _i64, _i64, _i32])
_newton_destroy = _sig("spn_newton_destroy", C.c_int, [_vp])
_eval = _sig("spn_logistic_eval_f32", C.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp])
_hsqrt = _sig("spn_hessian_sqrt_f32", C.c_int, [_vp, _vp, _i64, _vp, _vp, _i64, _vp])
_step = _sig("spn_sketched_step_f32", C.c_int, [_vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp])
_line = _sig("spn_logistic_line_f32", C.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, _dbl, _i64, _vp, _vp])
_ar1 = _sig("spn_ar1_problem", C.c_int, [_i64, _i64, _u64, _vp, _vp])

_MAX_BACKTRACK = 41  # s = 2^-k for k = 0..39 are tested; 2^-40 <= 1e-12 ends the loop (.cpp:142,164)


class _Workspace:
    def __init__(self, n, d, rows, device):
        h = _vp()
        _check(_newton_create(C.byref(h), n, d, rows, device))
        self.h, self.rows = h, rows

    def __del__(self):
        h = getattr(self, "h", None)
        destroy = _newton_destroy
        if h is not None and h.value and destroy is not None:
            destroy(h)
            self.h = None


class LogisticProblem:
    """Rows a_i of A (n x d) and labels y_i in {-1, +1}, held on the device (fp32)."""

    def __init__(self, features, labels, device: int = 0):
        torch = _torch()
        self.device = device
        f = features if isinstance(features, torch.Tensor) else torch.from_numpy(np.asarray(features))
        y = labels if isinstance(labels, torch.Tensor) else torch.from_numpy(np.asarray(labels))
        if f.dim() != 2:
            raise DimensionError("LogisticProblem: features must be n x d")
        self.features = f.to(device=f"cuda:{device}", dtype=torch.float32).contiguous()
        self.labels = y.reshape(-1).to(device=f"cuda:{device}", dtype=torch.float32).contiguous()
        self._ws: Optional[_Workspace] = None

    def observations(self) -> int:
        return int(self.features.shape[0])

    def dim(self) -> int:
        return int(self.features.shape[1])

    def validate(self) -> None:  # newton_sketch.cpp:28-37
        torch = _torch()
        if self.features.shape[0] < 1 or self.features.shape[1] < 1:
            raise DimensionError("LogisticProblem: empty data")
        if self.labels.numel() != self.features.shape[0]:
            raise DimensionError("LogisticProblem: label count mismatch")
        if not bool(torch.isfinite(self.features).all()):
            raise DomainError("LogisticProblem: non-finite features")
        if not bool(((self.labels == 1.0) | (self.labels == -1.0)).all()):
            raise DomainError("LogisticProblem: labels must be +-1")

    def workspace(self, rows: int = 0) -> _Workspace:
        if self._ws is None or self._ws.rows < rows:
            self._ws = _Workspace(self.observations(), self.dim(), max(rows, 0), self.device)
        return self._ws


@dataclasses.dataclass
class SketchConfig:
    """newton_sketch.hpp:23-33 (sketch_variant None = exact Newton)."""
    sketch_variant: Optional[SpinnerVariant] = None
    sketch_rows: int = 0
    max_iters: int = 50
    gap_tolerance: float = 1e-10
    line_search: bool = True
    seed: int = 0

    def validate(self, p: LogisticProblem) -> None:  # newton_sketch.cpp:39-43
        if self.sketch_variant is not None and self.sketch_rows < p.dim():
            raise DimensionError("SketchConfig: sketch_rows must be >= d")
        if self.max_iters < 1:
            raise DimensionError("SketchConfig: max_iters must be >= 1")


@dataclasses.dataclass
class NewtonTrace:
    """newton_sketch.hpp:35-42."""
    iterates: List[np.ndarray] = dataclasses.field(default_factory=list)
    losses: List[float] = dataclasses.field(default_factory=list)
    gaps: List[float] = dataclasses.field(default_factory=list)
    seconds: List[float] = dataclasses.field(default_factory=list)
    f_star: float = 0.0
    converged: bool = False


def _dvec(p, x):
    torch = _torch()
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    t = t.reshape(-1).to(device=f"cuda:{p.device}", dtype=torch.float64).contiguous()
    if t.numel() != p.dim():
        raise DimensionError("dimension mismatch")
    return t


def _eval_dev(p, x, stream=None):
    torch = _torch()
    ws = p.workspace()
    f = torch.empty(1, dtype=torch.float64, device=x.device)
    g = torch.empty(p.dim(), dtype=torch.float64, device=x.device)
    _check(_eval(ws.h, p.features.data_ptr(), p.features.stride(0), p.labels.data_ptr(), x.data_ptr(),
                 f.data_ptr(), g.data_ptr(), _stream_ptr(stream)))
    return f, g


def loss(p: LogisticProblem, x, stream=None) -> float:
    """newton_sketch.cpp:45-52."""
    f, _ = _eval_dev(p, _dvec(p, x), stream)
    return float(f.item())


def gradient(p: LogisticProblem, x, stream=None) -> np.ndarray:
    """newton_sketch.cpp:54-61."""
    _, g = _eval_dev(p, _dvec(p, x), stream)
    return g.cpu().numpy()


def hessian_sqrt(p: LogisticProblem, x, stream=None):
    """newton_sketch.cpp:63-72 (device fp32 [n][d])."""
    torch = _torch()
    ws = p.workspace()
    xd = _dvec(p, x)
    out = torch.empty_like(p.features)
    _check(_hsqrt(ws.h, p.features.data_ptr(), p.features.stride(0), xd.data_ptr(), out.data_ptr(), out.stride(0),
                  _stream_ptr(stream)))
    return out


def _step_dev(p, x, sketch: Optional[SketchOperator], stream=None):
    torch = _torch()
    exact = sketch is None or sketch.is_exact()
    rows = 0 if exact else sketch.m
    if not exact and sketch.row_list is not None:
        raise DomainError("sketched_step uses the reference's first-m SketchOperator")
    if not exact and sketch.input_dim != p.observations():
        raise DimensionError("SketchOperator::apply: row count mismatch")
    ws = p.workspace(rows)
    step = torch.empty(p.dim(), dtype=torch.float64, device=x.device)
    g = torch.empty_like(step)
    f = torch.empty(1, dtype=torch.float64, device=x.device)
    plan = None if exact else sketch.plan._h
    _check(_step(ws.h, plan, rows, p.features.data_ptr(), p.features.stride(0), p.labels.data_ptr(), x.data_ptr(),
                 step.data_ptr(), g.data_ptr(), f.data_ptr(), _stream_ptr(stream)))
    return step, g, f


def sketched_step(p: LogisticProblem, x, sketch: Optional[SketchOperator] = None, stream=None) -> np.ndarray:
    """newton_sketch.cpp:103-122: solve ((S B)^T (S B)) delta = -gradient, B = hessian_sqrt.
    Raises SingularSystemError when the ridge retry fails too."""
    step, _, _ = _step_dev(p, _dvec(p, x), sketch, stream)
    return step.cpu().numpy()


def _line_losses(p, x, step, s0, count, stream=None):
    torch = _torch()
    ws = p.workspace()
    out = torch.empty(count, dtype=torch.float64, device=x.device)
    _check(_line(ws.h, p.features.data_ptr(), p.features.stride(0), p.labels.data_ptr(), x.data_ptr(),
                 step.data_ptr(), float(s0), count, out.data_ptr(), _stream_ptr(stream)))
    return out.cpu().numpy()


def _backtrack(p, x, step, f0, slope, stream=None):
    """Backtracking Armijo (alpha 0.1, beta 0.5) of newton_sketch.cpp:140-142 / 163-164:
    returns (s, loss(x + s step)).  The first 4 candidates s = 2^-k come from one pass over
    A (one transcendental per lane per 8 rows); deeper backtracking evaluates all 41."""
    losses = _line_losses(p, x, step, 1.0, 4, stream)
    if not any(losses[k] <= f0 + 0.1 * 2.0 ** -k * slope for k in range(4)):
        losses = _line_losses(p, x, step, 1.0, _MAX_BACKTRACK, stream)
    s = 1.0
    for k in range(_MAX_BACKTRACK):
        if not (s > 1e-12):
            return s, float(losses[k])
        if not (losses[k] > f0 + 0.1 * s * slope):
            return s, float(losses[k])
        s *= 0.5
    return s, float(_line_losses(p, x, step, s, 1, stream)[0])  # pragma: no cover


def solve(p: LogisticProblem, cfg: SketchConfig, stream=None) -> NewtonTrace:
    """newton_sketch.cpp:124-183."""
    torch = _torch()
    p.validate()
    cfg.validate(p)
    d, n = p.dim(), p.observations()
    # reference optimum: exact Newton to a decrement below round-off (.cpp:130-147)
    x = torch.zeros(d, dtype=torch.float64, device=f"cuda:{p.device}")
    for _ in range(200):
        step, g, f = _step_dev(p, x, None, stream)
        decrement = -float(torch.dot(g, step).item())
        f0 = float(f.item())
        s, _ = _backtrack(p, x, step, f0, -decrement, stream)
        x = x + s * step
        if decrement / 2.0 < 1e-13:
            break
    f_star = float(_eval_dev(p, x, stream)[0].item())

    trace = NewtonTrace(f_star=f_star)
    x = torch.zeros(d, dtype=torch.float64, device=f"cuda:{p.device}")
    # fresh sketch every iteration (.cpp:155-157); its seed is known in advance, so the next
    # iteration's operator is realised on a host thread while this one runs on the GPU
    pool = concurrent.futures.ThreadPoolExecutor(1) if cfg.sketch_variant is not None else None
    make = lambda it: SketchOperator(cfg.sketch_variant, n, cfg.sketch_rows, mix_seed(cfg.seed, it),  # noqa: E731
                                     device=p.device)
    pending = pool.submit(make, 0) if pool else None
    for t in range(cfg.max_iters):
        tic = time.perf_counter()
        sketch = None
        if pool is not None:
            sketch = pending.result()
            if t + 1 < cfg.max_iters:
                pending = pool.submit(make, t + 1)
        step, g, f = _step_dev(p, x, sketch, stream)
        f0 = float(f.item())
        if cfg.line_search:
            slope = float(torch.dot(g, step).item())
            s, f_next = _backtrack(p, x, step, f0, slope, stream)
        else:
            s, f_next = 1.0, float(_line_losses(p, x, step, 1.0, 1, stream)[0])
        x_next = x + s * step
        if not cfg.line_search and f_next > f0:
            raise SingularSystemError("solve: loss increased under a full step (divergence)")
        x = x_next
        torch.cuda.synchronize(p.device)
        toc = time.perf_counter()
        trace.iterates.append(x.cpu().numpy())
        trace.losses.append(f_next)
        trace.gaps.append(f_next - f_star)
        trace.seconds.append(toc - tic)
        if f_next - f_star <= cfg.gap_tolerance:
            trace.converged = True
            break
    if pool is not None:
        pool.shutdown(wait=True)
    return trace


def generate_ar1_problem(n: int, d: int, seed: int, device: int = 0) -> LogisticProblem:
    """newton_sketch.cpp:185-204 (reference generator on the host, fp32 features)."""
    if n < 1 or d < 1:
        raise DimensionError("generate_ar1_problem: n, d must be >= 1")
    f = np.zeros((n, d), dtype=np.float32)
    y = np.zeros(n, dtype=np.float32)
    _check(_ar1(n, d, seed & (2**64 - 1), f.ctypes.data, y.ctypes.data))
    return LogisticProblem(f, y, device=device)


__all__ = ["LogisticProblem", "SketchConfig", "NewtonTrace", "loss", "gradient", "hessian_sqrt", "sketched_step",
           "solve", "generate_ar1_problem"]
