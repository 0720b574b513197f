"""ORACLE (test infrastructure only): the stage-split pipeline window restated
over the plain-torch reference networks (``UNetRef`` / ``MMDiTRef`` in fp32).

The reference has no stage split -- its window is the segment blend of
engine.py:254-261 -- so this restates the convention written down in
``paper_2602_21760_b200/stages.py`` (AsyncDiff-style stale boundary states,
PAPER.md:45, :395) independently of the product: its own unit lists
(``ref_units`` / [embed, blocks, out]), its own boundary states (NCHW skips),
its own time embedding per stage. The cuts are passed in (test
infrastructure takes them from the plan and pins them separately).

Protocol used by ``oracle.loop.run_staged(pipeline="stage_split")``:
``branches(x, t)`` (records the conditional forward's boundary states at the
cuts), ``conditional(x, t)``, ``recorded()`` and ``window_step(x, bstate, t)``.
x is the engine's flat (B, N) fp64 latent (NHWC order per image).
"""
from __future__ import annotations

import numpy as np
import torch

from .unet_ref import ref_units


class StagedNet:
    def __init__(self, net, kind, cond, spec, T, cuts, device="cpu", timestep=None):
        """kind: "unet" (UNetRef, NCHW) or "mmdit" (MMDiTRef, NHWC); cond: a
        Conditioning (rows = prompts); ``timestep(t, T)`` -> network timestep."""
        self.net, self.kind, self.c, self.s, self.T = net, kind, cond, spec, T
        self.cuts = tuple(cuts)
        self.dev = device
        self.ts = timestep
        self.units = len(ref_units(spec)) if kind == "unet" else spec.depth + 2
        self.edges = (0,) + self.cuts + (self.units,)
        self._rec = None

    # ---- layout -------------------------------------------------------------------
    def _to_net(self, x):
        B = x.shape[0]
        hw, ch = self.s.latent_hw, self.s.in_channels
        xt = torch.from_numpy(np.asarray(x)).to(self.dev).float().view(B, hw, hw, ch)
        return xt.permute(0, 3, 1, 2) if self.kind == "unet" else xt

    def _from_net(self, e):
        if self.kind == "unet":
            e = e.permute(0, 2, 3, 1)
        return e.reshape(e.shape[0], -1).double().cpu().numpy()

    def _ctx(self, B, cond: bool):
        if cond:
            return self.c.context[:B].to(self.dev), self.c.pooled[:B].to(self.dev)
        return (self.c.null_context.expand(B, -1, -1).to(self.dev), self.c.null_pooled.expand(B, -1).to(self.dev))

    def _t(self, t, B):
        return torch.full((B,), float(self.ts(t, self.T)), device=self.dev)

    def _run(self, state, t, B, cond, a, b):
        ctx, pooled = self._ctx(B, cond)
        with torch.no_grad():
            return self.net.run_units(state, self._t(t, B), ctx, pooled, a, b)

    # ---- loop protocol -------------------------------------------------------------
    def cond(self, x, t):
        """The conditional branch, run stage by stage so its boundary states at
        the cuts are kept (the window's fill)."""
        B = x.shape[0]
        st = {"x": self._to_net(x)}
        rec = []
        for j in range(len(self.edges) - 1):
            st = self._run(st, t, B, True, self.edges[j], self.edges[j + 1])
            if j < len(self.edges) - 2:
                rec.append(st)
        self._rec = rec
        return self._from_net(st["eps"])

    def uncond(self, x, t):
        B = x.shape[0]
        with torch.no_grad():
            ctx, pooled = self._ctx(B, False)
            return self._from_net(self.net(self._to_net(x), self._t(t, B), ctx, pooled))

    def branches(self, x, t):
        """Exact CFG branches (eps_c, eps_u); records the conditional boundary states."""
        return self.cond(x, t), self.uncond(x, t)

    def stage(self, j, inp, t, B):
        """Network stage j on its input (``{"x": net-layout latent}`` for j = 0)."""
        return self._run(inp, t, B, True, self.edges[j], self.edges[j + 1])

    def conditional(self, x, t):
        B = x.shape[0]
        return self._from_net(self._run({"x": self._to_net(x)}, t, B, True, 0, self.units)["eps"])

    def recorded(self):
        return list(self._rec)

    def window_step(self, x, bstate, t):
        """Stage 0 on x_t, stage j >= 1 on bstate[j-1] (previous step's output of
        stage j-1); returns (eps estimate, the new boundary states)."""
        B = x.shape[0]
        n_st = len(self.edges) - 1
        new = []
        st = self._run({"x": self._to_net(x)}, t, B, True, self.edges[0], self.edges[1])
        new.append(st)
        for j in range(1, n_st):
            st = self._run(bstate[j - 1], t, B, True, self.edges[j], self.edges[j + 1])
            if j < n_st - 1:
                new.append(st)
        return self._from_net(st["eps"]), new
