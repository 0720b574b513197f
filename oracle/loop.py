"""ORACLE (test infrastructure only): the staged denoising loop on the CPU.

Restates /root/reference/pkg/src/hybridpar/engine.py:147-304 (initial
latents, branch fan-out, exact update, pipelined blend, staged loop) and the
analytic GMM branch output of mixture.py:101-158, in numpy fp64, with the
denoiser pluggable so a CPU torch network can stand in (the reference's
``eps_prediction`` seam, engine.py:28).

``branches(x, t) -> (eps_c, eps_u)`` and ``conditional(x, t) -> eps_c`` are
the two callables a denoiser provides.
"""
from __future__ import annotations

import numpy as np

from . import controller as ctl
from . import sampler as smp


# ---- analytic GMM (mixture.py:101-158) ---------------------------------------

def gmm_eps(weights, means, variances, sub, ab, sig, x):
    """-sigma_t * score of the noised (sub-)mixture at x (mixture.py:152-158)."""
    w = np.asarray(weights, float)
    w = w / w.sum()
    mu = np.asarray(means, float)
    var = np.asarray(variances, float)
    if sub is not None:
        idx = np.asarray(sub, int)
        w, mu, var = w[idx] / w[idx].sum(), mu[idx], var[idx]
    mu_t = np.sqrt(ab) * mu                                   # noised_mixture :101-110
    var_t = ab * var + (1.0 - ab)
    x = np.atleast_2d(np.asarray(x, float))
    diff = x[:, None, :] - mu_t[None]
    lj = np.log(w)[None] - 0.5 * np.sum(diff * diff / var_t[None] + np.log(2 * np.pi * var_t[None]), axis=2)
    mx = lj.max(axis=1, keepdims=True)
    ld = mx[:, 0] + np.log(np.exp(lj - mx).sum(axis=1))        # _log_resp :125-133
    r = np.exp(lj - ld[:, None])
    s = np.einsum("bk,bkd->bd", r, (mu_t[None] - x[:, None, :]) / var_t[None])
    return -sig * s


class GMMDenoiser:
    """_branches / _conditional_branch (engine.py:164-184) over the analytic GMM."""

    def __init__(self, weights, means, variances, cond_rows, abar, sig):
        self.p = (weights, means, variances)
        self.abar, self.sig = abar, sig
        groups: dict = {}
        for row, c in enumerate(cond_rows):
            groups.setdefault(tuple(c), []).append(row)
        self.groups = [(idx, np.asarray(rows)) for idx, rows in groups.items()]

    def _at(self, sub, x, t):
        return gmm_eps(*self.p, sub, smp.ab_at(self.abar, t), smp.sig_at(self.sig, t), x)

    def conditional(self, x, t):
        out = np.empty_like(x)
        for idx, rows in self.groups:
            out[rows] = self._at(idx, x[rows], t)
        return out

    def branches(self, x, t):
        return self.conditional(x, t), self._at(None, x, t)


def initial_latents(weights, means, variances, cond_rows, seed, ab_T):
    """engine.py:147-161 with mixture.sample_x0 (:194-202), same RNG call order."""
    rng = np.random.default_rng(seed)
    w = np.asarray(weights, float)
    w = w / w.sum()
    mu, var = np.asarray(means, float), np.asarray(variances, float)
    b, d = len(cond_rows), mu.shape[1]
    x0 = np.empty((b, d))
    for i, c in enumerate(cond_rows):
        idx = np.asarray(c, int)
        wi = w[idx] / w[idx].sum()
        comp = rng.choice(len(idx), size=1, p=wi)
        z = rng.standard_normal((1, d))
        x0[i] = (mu[idx][comp] + np.sqrt(var[idx][comp]) * z)[0]
    e = rng.standard_normal((b, d))
    return np.sqrt(ab_T) * x0 + np.sqrt(1.0 - ab_T) * e


def _update(x, e, t, T, abar, sig, update):
    """ddim_step (schedules.py:152-168) or fm_euler_step (schedules.py:171-182)
    at t_cont = t/T, dt = 1/T (the engine's FM parameterisation)."""
    if update == "euler":
        return smp.euler(x, e, 1.0 / T)
    return smp.ddim(x, e, t, abar, sig)


def run_exact(den, x, T, w, abar, sig, update="ddim"):
    """Serial / full condition partitioning (engine.py:195-251): every step exact."""
    series = []
    for t in range(T, 0, -1):
        ec, eu = den.branches(x, t)
        series.append((t, smp.rel_mae(ec, eu)))
        x = _update(x, smp.cfg(ec, eu, w), t, T, abar, sig, update)
    return x, series


def run_staged(den, x, T, w, abar, sig, L, g, tau_cap, k, fractions, update="ddim",
               pipeline="reference_blend"):
    """_run_staged (engine.py:264-304): warm-up, pipelined window, reconnect.

    ``update="euler"``: the same loop with fm_euler_step (schedules.py:171-182) in
    place of ddim_step -- BASELINE config 3's flow-matching staged loop, which the
    reference engine (DDIM-only, engine.py:31) composes from its public pieces.
    ``pipeline="stage_split"``: the window runs the network split into
    len(fractions) stages (``den`` is an ``oracle.stage_ref.StagedNet``), stage j
    on the boundary state stage j-1 produced at the previous step, filled from
    the conditional forward of the last measured step (paper_2602_21760_b200/
    stages.py states the convention); ``reference_blend`` is engine.py:254-261."""
    n = len(fractions)
    state = {"steps": 0, "tau1": None, "tau2": None}
    series: dict = {}
    history: list = []
    labels = []
    prev = None
    bstate = None
    for s in range(1, T + 1):
        t = T - s + 1
        history = [x] + history[:n - 1]
        if state["tau1"] is None:
            ec, eu = den.branches(x, t)
            series[t] = smp.rel_mae(ec, eu)
            label = ctl.step(state, series, t, L, g, tau_cap, k)
            x = _update(x, smp.cfg(ec, eu, w), t, T, abar, sig, update)
        else:
            label = ctl.step(state, series, t, L, g, tau_cap, k)
            if label == ctl.PAR and pipeline == "stage_split":
                if prev != ctl.PAR:
                    bstate = den.recorded()                      # fill from the last exact forward
                est, bstate = den.window_step(x, bstate, t)
                x = _update(x, est, t, T, abar, sig, update)
            elif label == ctl.PAR:
                est = np.zeros_like(history[0])                   # _pipelined_estimate :254-261
                for d, f in enumerate(fractions):
                    est += f * den.conditional(history[min(d, len(history) - 1)], t)
                x = _update(x, est, t, T, abar, sig, update)
            else:
                ec, eu = den.branches(x, t)
                series[t] = smp.rel_mae(ec, eu)
                x = _update(x, smp.cfg(ec, eu, w), t, T, abar, sig, update)
        labels.append(label)
        prev = label
    ser = sorted(series.items(), key=lambda kv: -kv[0])
    return x, ser, state["tau1"], state["tau2"], labels
