"""ORACLE (test infrastructure only): plain-torch fp32 NCHW reference of the
SDXL-shaped U-Net, consuming the canonical weights of
paper_2602_21760_b200.denoiser.weights. Written directly from the
architecture (diffusers-style UNet2DConditionModel semantics: resnets with
time-embedding bias, linear-projection transformers with self/cross
attention and GEGLU feed-forward, text-time additional embedding) with
stock torch.nn.functional ops only — none of the package's kernels.

Also serves as the CPU baseline denoiser (bench.py cpu_baseline) and, through
``SeamAdapter``, as the network behind the reference engine's monkey-patched
``eps_prediction`` seam (engine.py:28, mixture.py:152-158).
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F


def _sinus(t, dim, max_period=10000.0):
    half = dim // 2
    fr = torch.exp(-math.log(max_period) * torch.arange(half, dtype=torch.float32, device=t.device) / half)
    arg = t.float()[:, None] * fr[None]
    return torch.cat([torch.cos(arg), torch.sin(arg)], dim=1)


class UNetRef:
    """``dtype=torch.bfloat16`` gives the same network as a stock-torch bf16 model
    (cuBLAS/cuDNN bf16 with fp32 accumulation): the yardstick for how much error
    bf16 itself costs, against which our kernels' error is judged."""

    def __init__(self, spec, W: dict, dtype=torch.float32):
        self.s = spec
        self.dt = dtype
        self.W = {k: v.to(dtype) for k, v in W.items()}

    def _lin(self, x, name, bias=True):
        b = self.W.get(name + ".bias") if bias else None
        return F.linear(x, self.W[name + ".weight"], b)

    def _conv(self, x, name, stride=1):
        w = self.W[name + ".weight"]
        return F.conv2d(x, w, self.W[name + ".bias"], stride=stride, padding=w.shape[-1] // 2)

    def _gn(self, x, name, eps=1e-5):
        return F.group_norm(x, self.s.groups, self.W[name + ".weight"], self.W[name + ".bias"], eps=eps)

    def _res(self, x, name, emb):
        h = self._conv(F.silu(self._gn(x, name + ".norm1")), name + ".conv1")
        h = h + self._lin(F.silu(emb), name + ".time_emb_proj")[:, :, None, None]
        h = self._conv(F.silu(self._gn(h, name + ".norm2")), name + ".conv2")
        sc = self._conv(x, name + ".conv_shortcut") if (name + ".conv_shortcut.weight") in self.W else x
        return sc + h

    def _attn(self, x, ctx, name, heads):
        q = self._lin(x, name + ".to_q", False)
        k = self._lin(ctx, name + ".to_k", False)
        v = self._lin(ctx, name + ".to_v", False)
        B, S, C = q.shape
        d = C // heads
        q, k, v = (t.view(B, -1, heads, d).transpose(1, 2) for t in (q, k, v))
        o = F.scaled_dot_product_attention(q, k, v)
        return self._lin(o.transpose(1, 2).reshape(B, S, C), name + ".to_out.0")

    def _transformer(self, x, ctx, name, depth):
        B, C, H, Wd = x.shape
        heads = C // self.s.head_dim
        h = self._gn(x, name + ".norm", eps=1e-6).permute(0, 2, 3, 1).reshape(B, H * Wd, C)
        h = self._lin(h, name + ".proj_in")
        for d in range(depth):
            b = f"{name}.transformer_blocks.{d}"
            n1 = F.layer_norm(h, (C,), self.W[b + ".norm1.weight"], self.W[b + ".norm1.bias"], eps=1e-5)
            h = h + self._attn(n1, n1, b + ".attn1", heads)
            n2 = F.layer_norm(h, (C,), self.W[b + ".norm2.weight"], self.W[b + ".norm2.bias"], eps=1e-5)
            h = h + self._attn(n2, ctx, b + ".attn2", heads)
            n3 = F.layer_norm(h, (C,), self.W[b + ".norm3.weight"], self.W[b + ".norm3.bias"], eps=1e-5)
            a, gate = self._lin(n3, b + ".ff.net.0.proj").chunk(2, dim=-1)
            h = h + self._lin(a * F.gelu(gate), b + ".ff.net.2")
        h = self._lin(h, name + ".proj_out")
        return h.reshape(B, H, Wd, C).permute(0, 3, 1, 2) + x

    def _emb(self, t, pooled, B, device):
        s = self.s
        temb = self._lin(F.silu(self._lin(_sinus(t, s.block_out[0]).to(self.dt), "time_embedding.linear_1")),
                         "time_embedding.linear_2")
        size = 8.0 * s.latent_hw
        ids = torch.tensor([size, size, 0.0, 0.0, size, size], device=device).repeat(B, 1).reshape(-1)
        tid = _sinus(ids, s.time_id_dim).reshape(B, -1)
        a = torch.cat([pooled.float(), tid], dim=1).to(self.dt)
        return temb + self._lin(F.silu(self._lin(a, "add_embedding.linear_1")), "add_embedding.linear_2")

    def run_units(self, state, t, context, pooled, a, b):
        """Units [a, b) of ``ref_units(spec)`` on a boundary state: ``{"x": NCHW
        latent}`` before unit 0, ``{"eps": NCHW}`` after the last, else ``{"h":
        NCHW activation, "skips": [pushed skips]}`` (the stage-split pipeline's
        unit of hand-off; every stage embeds the current step's t)."""
        s = self.s
        units = ref_units(s)
        if a == 0:
            x = state["x"].to(self.dt)
            h, skips = None, []
        else:
            h, skips = state["h"], list(state["skips"])
        B = (x if a == 0 else h).shape[0]
        emb = self._emb(t, pooled, B, (x if a == 0 else h).device)
        ctx = context.to(self.dt)
        depth = {"down": s.transformer_depth, "up": s.transformer_depth[::-1]}
        for u in units[a:b]:
            kind = u[0]
            if kind == "conv_in":
                h = self._conv(x, "conv_in")
                skips.append(h)
            elif kind == "res":
                _, where, lvl, j, push = u
                name = f"mid_block.resnets.{j}" if where == "mid" else f"{where}_blocks.{lvl}.resnets.{j}"
                if where == "up":
                    h = torch.cat([h, skips.pop()], dim=1)
                h = self._res(h, name, emb)
                if push:
                    skips.append(h)
            elif kind == "attn":
                _, where, lvl, j, push = u
                if where == "mid":
                    h = self._transformer(h, ctx, "mid_block.attentions.0", s.mid_depth)
                else:
                    h = self._transformer(h, ctx, f"{where}_blocks.{lvl}.attentions.{j}", depth[where][lvl])
                if push:
                    skips.append(h)
            elif kind == "ds":
                h = self._conv(h, f"down_blocks.{u[1]}.downsamplers.0.conv", stride=2)
                skips.append(h)
            elif kind == "us":
                h = F.interpolate(h, scale_factor=2.0, mode="nearest")
                h = self._conv(h, f"up_blocks.{u[1]}.upsamplers.0.conv")
            elif kind == "out":
                h = F.silu(self._gn(h, "conv_norm_out"))
                return {"eps": self._conv(h, "conv_out").float()}
        return {"h": h, "skips": skips}

    def __call__(self, x_nchw, t, context, pooled):
        """x [B, C, H, W] fp32, t [B] timesteps, context [B, L, D], pooled [B, P] -> eps NCHW."""
        return self.run_units({"x": x_nchw}, t, context, pooled, 0, len(ref_units(self.s)))["eps"]


def ref_units(s) -> list:
    """The forward's units in execution order (diffusers UNet2DConditionModel
    order): conv_in; per down level (resnet[, transformer]) x layers, then the
    downsampler; mid resnet, transformer, resnet; per up level (resnet[,
    transformer]) x (layers + 1), then the upsampler; norm_out + conv_out.
    ``push``: the unit's output is pushed as a skip."""
    ch = s.block_out
    out = [("conv_in",)]
    for lvl in range(len(ch)):
        d = s.transformer_depth[lvl]
        for j in range(s.layers_per_block):
            out.append(("res", "down", lvl, j, not d))
            if d:
                out.append(("attn", "down", lvl, j, True))
        if lvl < len(ch) - 1:
            out.append(("ds", lvl))
    out += [("res", "mid", 0, 0, False), ("attn", "mid", 0, 0, False), ("res", "mid", 0, 1, False)]
    for u in range(len(ch)):
        d = s.transformer_depth[len(ch) - 1 - u]
        for j in range(s.layers_per_block + 1):
            out.append(("res", "up", u, j, False))
            if d:
                out.append(("attn", "up", u, j, False))
        if u < len(ch) - 1:
            out.append(("us", u))
    out.append(("out",))
    return out


def net_timestep(t: int, T: int) -> float:
    """Discrete step t of a T-step schedule -> the network's 1000-step timestep."""
    return float(round(t * 1000 / T) - 1)


class SeamAdapter:
    """Reference-engine seam: ``eps_prediction(gm, cond, sched, x, t)`` backed by
    UNetRef on the CPU. x is the reference's flat (B, N) fp64 latent in NHWC
    order; cond None = unconditional (null prompt), else prompt cond.indices[0]."""

    def __init__(self, net: UNetRef, conditioning, hw: int, channels: int):
        self.net, self.c, self.hw, self.ch = net, conditioning, hw, channels
        self.calls = 0

    def __call__(self, gm, cond, sched, x, t):
        import numpy as np
        self.calls += 1
        xb = torch.from_numpy(np.asarray(x, dtype=np.float64)).float()
        B = xb.shape[0]
        xn = xb.view(B, self.hw, self.hw, self.ch).permute(0, 3, 1, 2)
        if cond is None:
            ctx = self.c.null_context.expand(B, -1, -1)
            pooled = self.c.null_pooled.expand(B, -1)
        else:
            i = cond.indices[0]
            ctx = self.c.context[i:i + 1].expand(B, -1, -1)
            pooled = self.c.pooled[i:i + 1].expand(B, -1)
        tt = torch.full((B,), net_timestep(t, sched.T))
        with torch.no_grad():
            eps = self.net(xn, tt, ctx, pooled)
        return eps.permute(0, 2, 3, 1).reshape(B, -1).double().numpy()
