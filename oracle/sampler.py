"""ORACLE (test infrastructure only): numpy fp64 sampler numerics.

Restates /root/reference/pkg/src/hybridpar/schedules.py and monitor.py:103-118.
"""
from __future__ import annotations

import numpy as np


def schedule_tables(kind: str, T: int, b0: float, b1: float):
    """schedules.py:88-118 — betas, alphas, cumulative alpha_bar, sigma."""
    if kind == "linear":
        betas = np.linspace(b0, b1, T)
    elif kind == "scaled-linear":
        betas = np.square(np.linspace(np.sqrt(b0), np.sqrt(b1), T))
    else:
        raise ValueError(kind)
    alphas = 1.0 - betas
    abar = np.cumprod(alphas)
    return betas, alphas, abar, np.sqrt(1.0 - abar)


def ab_at(abar, t):       # schedules.py:31-35 (t = 0 is the clean sample)
    return 1.0 if t == 0 else float(abar[t - 1])


def sig_at(sig, t):       # schedules.py:37-41
    return 0.0 if t == 0 else float(sig[t - 1])


def cfg(eps_c, eps_u, w):  # schedules.py:128-133
    eps_c = np.asarray(eps_c, float)
    eps_u = np.asarray(eps_u, float)
    return eps_c + w * (eps_c - eps_u)


def ddim(x, eps, t, abar, sig):  # schedules.py:152-168
    x = np.asarray(x, float)
    eps = np.asarray(eps, float)
    a_t = ab_at(abar, t)
    x0_hat = (x - sig_at(sig, t) * eps) / np.sqrt(a_t)
    a_p = ab_at(abar, t - 1)
    return np.sqrt(a_p) * x0_hat + np.sqrt(1.0 - a_p) * eps


def euler(x, v, dt):  # schedules.py:171-182
    return np.asarray(x, float) - np.asarray(v, float) * dt


def rel_mae(eps_c, eps_u):  # monitor.py:103-118
    eps_c = np.asarray(eps_c, float)
    eps_u = np.asarray(eps_u, float)
    return float(np.abs(eps_c - eps_u).sum() / np.abs(eps_u).sum())
