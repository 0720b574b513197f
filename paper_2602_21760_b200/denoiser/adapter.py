"""Seam adapter: a neural denoiser as the engine's branch evaluator.

Replaces the reference's per-condition-group ``eps_prediction`` fan-out
(engine.py:164-184) for neural networks:

* ``branches(x, t)`` runs ONE batched forward over [uncond rows; cond rows]
  (classifier-free guidance batched on one GPU; the rows are independent, so
  the result is bit-identical to two separate forwards) and returns
  (eps_c, eps_u) as views of the graph's static output;
* ``conditional(x, t)`` runs the conditional rows only (pipelined window).

Each distinct batch layout is captured once into a CUDA graph; a step is then
``t`` upload + graph replay. The fused sampler kernel writes the next bf16
latent straight into the graph's static input (``input_slot``), so no copy
sits between two steps.
"""
from __future__ import annotations

import torch

from .. import _native as N
from ..stages import Boundary, stage_bounds, state_rows
from . import kernels as K


def net_timestep(t: int, T: int) -> float:
    return float(round(t * 1000 / T) - 1)


class _Graphed:
    def __init__(self, fn, x_static, t_static, use_graph: bool):
        self.fn, self.x, self.t = fn, x_static, t_static
        self.graph = None
        self.out = None
        self.use_graph = use_graph
        self.launches = 0

    def run(self):
        if self.graph is not None:
            self.graph.replay()
            return self.out
        if not self.use_graph:
            self.out = self.fn(self.x, self.t)
            return self.out
        # warm-up eagerly (kernel attributes, TMA encoder, allocator), then capture
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.fn(self.x, self.t)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        before = K.LAUNCHES
        with torch.cuda.graph(g):
            self.out = self.fn(self.x, self.t)
        self.launches = K.LAUNCHES - before
        self.graph = g
        g.replay()
        return self.out


class NetDenoiser:
    """Neural branch evaluator behind the seam (UNet or MMDiT)."""

    latent_dtype = torch.float32
    eps_dtype = torch.bfloat16
    wants_bf16_input = True

    def __init__(self, net, conditioning, conditions, schedule, latent_shape, use_graph=True):
        N.require_cuda()
        self.net, self.sched = net, schedule
        self.shape = tuple(latent_shape)             # (H, W, C) NHWC per image
        self.numel = self.shape[0] * self.shape[1] * self.shape[2]
        self.B = len(conditions)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        prompts = [c.indices[0] for c in conditions]
        ctx_c = conditioning.context[prompts]
        pool_c = conditioning.pooled[prompts]
        ctx_u = conditioning.null_context.expand(self.B, -1, -1)
        pool_u = conditioning.null_pooled.expand(self.B, -1)
        self._ctx_u, self._pool_u = ctx_u.to(dev), pool_u.to(dev)
        net.prepare(torch.cat([ctx_u, ctx_c]).to(dev), torch.cat([pool_u, pool_c]).to(dev), key="both")
        net.prepare(ctx_c.to(dev), pool_c.to(dev), key="cond")
        B2 = 2 * self.B
        self.x_both = torch.zeros((B2,) + self.shape, dtype=torch.bfloat16, device=dev)
        self.t_both = torch.zeros(B2, dtype=torch.float32, device=dev)
        self.x_cond = torch.zeros((self.B,) + self.shape, dtype=torch.bfloat16, device=dev)
        self.t_cond = torch.zeros(self.B, dtype=torch.float32, device=dev)
        half = self.x_both[: self.B]

        def both(x, t):
            x[self.B:].copy_(x[: self.B])
            return net.forward(x, t, key="both")

        def cond(x, t):
            return net.forward(x, t, key="cond")

        self.g_both = _Graphed(both, self.x_both, self.t_both, use_graph)
        self.g_cond = _Graphed(cond, self.x_cond, self.t_cond, use_graph)
        self._slot = half.view(self.B, self.numel)
        self.use_graph = use_graph
        self.cuts = None

    def input_slot(self):
        """bf16 [B, N] buffer the sampler kernel writes the next latent into."""
        return self._slot

    def load_input(self, x: torch.Tensor) -> None:
        self._slot.copy_(x.to(torch.bfloat16).view(self.B, self.numel))

    def _set_t(self, buf, t):
        tf = getattr(self.net, "timestep_for", None)
        buf.fill_(tf(t, self.sched.T) if tf is not None else net_timestep(t, self.sched.T))

    def branches(self, x, t, x_bf16=None):
        if x_bf16 is None or x_bf16.data_ptr() != self._slot.data_ptr():
            self.load_input(x)
        self._set_t(self.t_both, t)
        self._last = "both"
        out = self.g_both.run().reshape(2 * self.B, self.numel)
        return out[self.B:], out[: self.B]            # eps_c, eps_u

    def conditional(self, x, t, x_bf16=None):
        self.x_cond.view(self.B, self.numel).copy_(x.to(torch.bfloat16).view(self.B, self.numel))
        self._set_t(self.t_cond, t)
        self._last = "cond"
        return self.g_cond.run().reshape(self.B, self.numel)

    def unconditional(self, x, t, x_bf16=None):
        """Unconditional rows only (the uncond rank of a condition-partitioned pair)."""
        if not hasattr(self, "g_uncond"):
            self.net.prepare(self._ctx_u, self._pool_u, key="uncond")
            self.x_unc = torch.zeros((self.B,) + self.shape, dtype=torch.bfloat16, device=self.dev)
            self.t_unc = torch.zeros(self.B, dtype=torch.float32, device=self.dev)
            self.g_uncond = _Graphed(lambda xx, tt: self.net.forward(xx, tt, key="uncond"), self.x_unc,
                                     self.t_unc, self.g_cond.use_graph)
        self.x_unc.view(self.B, self.numel).copy_(x.to(torch.bfloat16).view(self.B, self.numel))
        self._set_t(self.t_unc, t)
        return self.g_uncond.run().reshape(self.B, self.numel)

    # ---- stage-split pipeline window (stages.py) -------------------------------------
    def enable_stage_split(self, cuts) -> None:
        """Split the network at unit indices ``cuts`` (network order). The CFG
        forward is re-captured so it keeps the boundary states at the cuts (its
        conditional rows fill the window's first step); one graph per stage runs
        the conditional rows of that stage on static boundary buffers."""
        cuts = tuple(int(c) for c in cuts)
        if cuts == self.cuts:
            return
        net, B = self.net, self.B
        U = len(net.units)
        self.cuts = cuts
        self.bounds = stage_bounds(cuts, U)
        self._rec = {}

        def both(x, t):
            x[B:].copy_(x[:B])
            rec = {c: None for c in cuts}
            out = net.run_units({"x": x}, t, "both", 0, U, record=rec)["eps"]
            self._rec["both"] = rec
            return out

        def cond(x, t):
            rec = {c: None for c in cuts}
            out = net.run_units({"x": x}, t, "cond", 0, U, record=rec)["eps"]
            self._rec["cond"] = rec
            return out
        self.g_both = _Graphed(both, self.x_both, self.t_both, self.use_graph)
        self.g_cond = _Graphed(cond, self.x_cond, self.t_cond, self.use_graph)
        self.g_both.run()                                    # capture; defines the recorded states
        self.g_cond.run()
        self._last = "both"
        # boundary j (input of stage j >= 1): the conditional rows of a forward
        self.bnd = [None] + [Boundary(state_rows(self._rec["cond"][c], 0, B), self.dev) for c in cuts]
        self.x_stage = torch.zeros((B,) + self.shape, dtype=torch.bfloat16, device=self.dev)
        self.t_stage = torch.zeros(B, dtype=torch.float32, device=self.dev)
        self.g_stage = [None] * len(self.bounds)

    @property
    def n_stages(self) -> int:
        return len(self.bounds)

    def _stage_fn(self, j):
        a, b = self.bounds[j]
        last = j == len(self.bounds) - 1

        def fn(_x, t):
            st = {"x": self.x_stage} if j == 0 else self.bnd[j].state()
            out = self.net.run_units(st, t, "cond", a, b)
            if last:
                return out["eps"]
            self.bnd[j + 1].load(out)                        # hand-off buffer (one message)
            return self.bnd[j + 1].buf
        return fn

    def stage_run(self, j: int, t: int):
        """Run network stage j at timestep t on its static input (``stage_input``);
        the last stage returns eps [B, N] bf16, the others fill ``bnd[j+1]``."""
        if self.g_stage[j] is None:
            self.g_stage[j] = _Graphed(self._stage_fn(j), None, self.t_stage, self.use_graph)
        self._set_t(self.t_stage, t)
        out = self.g_stage[j].run()
        return out.reshape(self.B, self.numel) if j == len(self.bounds) - 1 else out

    def stage_input(self, j: int):
        """The static input buffer of stage j: the bf16 latent for j = 0, else the
        contiguous boundary buffer (what an upstream rank pushes into)."""
        return self.x_stage if j == 0 else self.bnd[j].buf

    def load_stage_x(self, x) -> None:
        self.x_stage.view(self.B, self.numel).copy_(x.to(torch.bfloat16).view(self.B, self.numel))

    def window_fill(self) -> None:
        """Boundary states of the conditional rows of the last exact forward (the
        CFG batch on one device, or the conditional-only forward of dev0 in a
        condition-partitioned pair) -> stage inputs."""
        lo = self.B if self._last == "both" else 0
        for j, c in enumerate(self.cuts, start=1):
            self.bnd[j].load(state_rows(self._rec[self._last][c], lo, lo + self.B))

    def window_step(self, x, t, steps_left=None):
        """One pipelined step on one device: every stage on its stale input, last
        stage first so each stage reads its input before the upstream stage
        overwrites it. ``steps_left`` (window steps after this one): stage j is
        skipped when its output could no longer reach the last stage (the
        pipeline's drain; numerically irrelevant). Returns the unguided eps
        estimate [B, N]."""
        n = len(self.bounds)
        eps = None
        for j in reversed(range(n)):
            if steps_left is not None and j < n - 1 and steps_left < n - 1 - j:
                continue
            if j == 0:
                self.load_stage_x(x)
            out = self.stage_run(j, t)
            if j == n - 1:
                eps = out
        return eps
