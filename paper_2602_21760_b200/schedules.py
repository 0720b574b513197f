"""Noise schedules and the single-step denoising updates, on the GPU.

Host side: the VP schedule tables are fp64 numpy arrays built exactly as the
reference builds them (schedules.py:88-118: ``np.linspace`` then
``np.cumprod``), with the t = 0 accessor convention (alpha_bar = 1,
sigma = 0, schedules.py:31-41). The engine folds them into per-step fp64
scalars (``StepCoefficients``) that the fused kernel consumes.

Device side: ``cfg_combine`` (schedules.py:128-133), ``ddim_step``
(:152-168), ``fm_euler_step`` (:171-182) and ``ddpm_posterior_mean``
(:136-149) each run as one ``hp_sampler_step`` launch. Arguments may be torch
tensors (results stay on the GPU) or array-likes (results come back as
numpy float64, like the reference). The fp64 instantiation keeps the
reference's operation order without FMA contraction, so its output equals the
numpy reference bit for bit.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _kernels as K
from . import _native as N
from .errors import NumericError, ParameterError, ShapeError, StepUnderflowError  # noqa: F401

SCHEDULE_KINDS = ("linear", "scaled-linear")


@dataclass(frozen=True)
class NoiseSchedule:
    """Discrete VP schedule, tables stored for t = 1..T (read-only)."""

    kind: str
    T: int
    beta_start: float
    beta_end: float
    betas: np.ndarray = field(repr=False)
    alphas: np.ndarray = field(repr=False)
    alpha_bars: np.ndarray = field(repr=False)
    sigmas: np.ndarray = field(repr=False)

    def _idx(self, t: int) -> int:
        if t < 1 or t > self.T:
            raise ParameterError(f"timestep t={t} outside [1, {self.T}]")
        return t - 1

    def alpha_bar(self, t: int) -> float:
        return 1.0 if t == 0 else float(self.alpha_bars[self._idx(t)])

    def sigma(self, t: int) -> float:
        return 0.0 if t == 0 else float(self.sigmas[self._idx(t)])

    def beta(self, t: int) -> float:
        return float(self.betas[self._idx(t)])

    def alpha(self, t: int) -> float:
        return float(self.alphas[self._idx(t)])

    def to_config(self) -> dict:
        return {"kind": self.kind, "T": self.T, "beta_start": self.beta_start,
                "beta_end": self.beta_end}


@dataclass(frozen=True)
class GuidanceParams:
    """Classifier-free guidance weight w >= 0 (e = eps_c + w (eps_c - eps_u))."""

    w: float

    def __post_init__(self):
        if not (math.isfinite(self.w) and self.w >= 0):
            raise ParameterError(f"guidance w must be finite and >= 0, got {self.w}")


@dataclass(frozen=True)
class LatentState:
    """Latent (torch tensor or array) at integer timestep t."""

    x: object
    t: int

    def __post_init__(self):
        if self.t < 0:
            raise ParameterError(f"latent timestep must be >= 0, got {self.t}")


def build_schedule(kind: str, T: int, beta_start: float, beta_end: float) -> NoiseSchedule:
    if kind not in SCHEDULE_KINDS:
        raise ParameterError(f"unknown schedule kind {kind!r}; expected one of {SCHEDULE_KINDS}")
    if not isinstance(T, int) or T < 1:
        raise ParameterError(f"T must be an integer >= 1, got {T!r}")
    for name, b in (("beta_start", beta_start), ("beta_end", beta_end)):
        if not 0.0 < b < 1.0:
            raise ParameterError(f"{name} must lie in (0, 1), got {b}")
    if beta_start > beta_end:
        raise ParameterError(f"beta_start={beta_start} exceeds beta_end={beta_end}")
    if kind == "linear":
        betas = np.linspace(beta_start, beta_end, T)
    else:
        betas = np.linspace(np.sqrt(beta_start), np.sqrt(beta_end), T) ** 2
    alphas = 1.0 - betas
    alpha_bars = np.cumprod(alphas)
    sigmas = np.sqrt(1.0 - alpha_bars)
    for a in (betas, alphas, alpha_bars, sigmas):
        a.setflags(write=False)
    return NoiseSchedule(kind, T, float(beta_start), float(beta_end), betas, alphas,
                         alpha_bars, sigmas)


@dataclass(frozen=True)
class StepCoefficients:
    """Per-step fp64 scalars folded on the host for hp_sampler_step (DDIM)."""

    c_sigma: float
    c_sqrt_ab: float
    c_sqrt_ab_prev: float
    c_sqrt_1m_ab_prev: float

    @classmethod
    def ddim(cls, sched: NoiseSchedule, t: int) -> "StepCoefficients":
        ab_t = sched.alpha_bar(t)
        ab_prev = sched.alpha_bar(t - 1)
        # the exact scalars numpy forms in ddim_step (schedules.py:164-167)
        return cls(sched.sigma(t), float(np.sqrt(ab_t)), float(np.sqrt(ab_prev)),
                   float(np.sqrt(1.0 - ab_prev)))


def _common_dtype(*ts):
    if any(t.dtype == torch.float64 for t in ts):
        return torch.float64
    return torch.float32


def _pair(eps_c, eps_u):
    a, ia = K.ensure_cuda_tensor(eps_c)
    b, ib = K.ensure_cuda_tensor(eps_u)
    if tuple(a.shape) != tuple(b.shape):
        raise ShapeError(f"branch outputs disagree: {tuple(a.shape)} vs {tuple(b.shape)}")
    if a.dtype != b.dtype:
        dt = _common_dtype(a, b)
        a, b = a.to(dt), b.to(dt)
    return a, b, (ia or ib)


def _out(t: torch.Tensor, to_numpy: bool):
    return t.cpu().numpy() if to_numpy else t


def cfg_combine(eps_c, eps_u, g: GuidanceParams):
    """Guided estimate eps_c + w (eps_c - eps_u) (schedules.py:128-133)."""
    a, b, np_out = _pair(eps_c, eps_u)
    out_dtype = torch.float64 if a.dtype == torch.float64 else torch.float32
    out = torch.empty(a.shape, dtype=out_dtype, device=a.device)
    ws = K.workspace(a.device)
    K.sampler_step(x=None, eps_c=a, eps_u=b, x_out=out, update=N.HP_UPDATE_NONE, w=g.w, ws=ws)
    K.read_status(ws, "non-finite values in branch outputs")
    return _out(out, np_out)


def _x_and_eps(x, eps):
    xt, ix = K.ensure_cuda_tensor(x)
    et, ie = K.ensure_cuda_tensor(eps)
    if tuple(xt.shape) != tuple(et.shape):
        raise ShapeError(f"branch outputs disagree: {tuple(xt.shape)} vs {tuple(et.shape)}")
    if xt.dtype == torch.bfloat16:
        xt = xt.float()
    if xt.dtype == torch.float64 and et.dtype != torch.float64:
        et = et.double()
    if et.dtype == torch.float64 and xt.dtype != torch.float64:
        xt = xt.double()
    return xt, et, (ix or ie)


def ddpm_posterior_mean(x_t, t: int, eps_cfg, sched: NoiseSchedule):
    """(x_t - beta_t / sqrt(1 - ab_t) eps) / sqrt(alpha_t)  (schedules.py:136-149)."""
    if t == 0:
        raise StepUnderflowError("no update exists below t = 1")
    xt, et, np_out = _x_and_eps(x_t, eps_cfg)
    coeff = sched.beta(t) / np.sqrt(1.0 - sched.alpha_bar(t))
    out = torch.empty_like(xt)
    ws = K.workspace(xt.device)
    # DDIM form with c_sqrt_ab_prev = 1, c_sqrt_1m_ab_prev = 0 is exactly (x - c e) / s
    K.sampler_step(x=xt, eps_c=et, eps_u=None, x_out=out, update=N.HP_UPDATE_DDIM,
                   c_sigma=float(coeff), c_sqrt_ab=float(np.sqrt(sched.alpha(t))),
                   c_sqrt_ab_prev=1.0, c_sqrt_1m_ab_prev=0.0, ws=ws)
    K.read_status(ws, "non-finite values in branch outputs")
    return _out(out, np_out)


def ddim_step(state: LatentState, eps, sched: NoiseSchedule) -> LatentState:
    """Deterministic eta = 0 update t -> t-1 (schedules.py:152-168)."""
    if state.t == 0:
        raise StepUnderflowError("cannot step below t = 1")
    xt, et, np_out = _x_and_eps(state.x, eps)
    c = StepCoefficients.ddim(sched, state.t)
    out = torch.empty_like(xt)
    ws = K.workspace(xt.device)
    K.sampler_step(x=xt, eps_c=et, eps_u=None, x_out=out, update=N.HP_UPDATE_DDIM, t=state.t,
                   c_sigma=c.c_sigma, c_sqrt_ab=c.c_sqrt_ab, c_sqrt_ab_prev=c.c_sqrt_ab_prev,
                   c_sqrt_1m_ab_prev=c.c_sqrt_1m_ab_prev, ws=ws)
    K.read_status(ws, "non-finite values in branch outputs")
    return LatentState(x=_out(out, np_out), t=state.t - 1)


def check_euler(t_cont: float, dt: float) -> None:
    if not 0.0 < t_cont <= 1.0:
        raise ParameterError(f"continuous time must lie in (0, 1], got {t_cont}")
    if dt <= 0:
        raise ParameterError(f"dt must be positive, got {dt}")
    if t_cont - dt < -1e-12:
        raise StepUnderflowError(f"step dt={dt} would overshoot t = 0 from t = {t_cont}")


def fm_euler_step(x, t_cont: float, v, dt: float):
    """x - v dt, integrating dx/dt = v from t toward 0 (schedules.py:171-182)."""
    check_euler(t_cont, dt)
    xt, vt, np_out = _x_and_eps(x, v)
    out = torch.empty_like(xt)
    ws = K.workspace(xt.device)
    K.sampler_step(x=xt, eps_c=vt, eps_u=None, x_out=out, update=N.HP_UPDATE_EULER, dt=dt, ws=ws)
    K.read_status(ws, "non-finite values in branch outputs")
    return _out(out, np_out)

