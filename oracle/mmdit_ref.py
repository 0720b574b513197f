"""ORACLE (test infrastructure only): plain-torch fp32 reference of the SD3-shaped
MMDiT consuming the canonical weights of paper_2602_21760_b200.denoiser.weights.

Written from the architecture (SD3 joint transformer: patch embedding with a
cropped positional table, adaLN-Zero modulated joint attention over
[image tokens; text tokens], GELU MLPs, context-pre-only last block,
AdaLayerNormContinuous output) with stock torch ops only.
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


class MMDiTRef:
    """``dtype=torch.bfloat16``: the same network as a stock-torch bf16 model (the
    yardstick for the error bf16 itself costs)."""

    def __init__(self, spec, W: dict, dtype=torch.float32):
        self.s = spec
        self.dt = dtype
        self.W = {k: v.to(dtype) for k, v in W.items()}

    def _lin(self, x, name):
        return F.linear(x, self.W[name + ".weight"], self.W.get(name + ".bias"))

    def __call__(self, x_nhwc, t, context, pooled):
        """x [n, H, W, C] fp32 latent (NHWC), t [n] network timesteps -> velocity NHWC."""
        s, W = self.s, self.W
        n, Hl, Wl, C = x_nhwc.shape
        P, H = s.patch, s.hidden
        gh, gw = Hl // P, Wl // P
        tok = x_nhwc.to(self.dt).view(n, gh, P, gw, P, C).permute(0, 1, 3, 2, 4, 5).reshape(n, gh * gw, P * P * C)
        off = (s.pos_max - gh) // 2
        pos = W["pos_embed.pos"].view(s.pos_max, s.pos_max, H)[off:off + gh, off:off + gw].reshape(gh * gw, H)
        xi = self._lin(tok, "pos_embed.proj") + pos
        xc = self._lin(context.to(self.dt), "context_embedder")
        te = F.silu(self._lin(_sinus(t, s.freq_dim).to(self.dt), "time_text_embed.timestep_embedder.linear_1"))
        te = self._lin(te, "time_text_embed.timestep_embedder.linear_2")
        pe = F.silu(self._lin(pooled.to(self.dt), "time_text_embed.text_embedder.linear_1"))
        c = te + self._lin(pe, "time_text_embed.text_embedder.linear_2")
        sc = F.silu(c)
        heads = s.heads
        Ti = xi.shape[1]
        for d in range(s.depth):
            b = f"transformer_blocks.{d}"
            last = d == s.depth - 1
            mi = self._lin(sc, f"{b}.norm1.linear").chunk(6, dim=1)
            mc_raw = self._lin(sc, f"{b}.norm1_context.linear")
            ni = F.layer_norm(xi, (H,), eps=1e-6) * (1 + mi[1][:, None]) + mi[0][:, None]
            if last:
                c_scale, c_shift = mc_raw.chunk(2, dim=1)
                nc = F.layer_norm(xc, (H,), eps=1e-6) * (1 + c_scale[:, None]) + c_shift[:, None]
            else:
                mc = mc_raw.chunk(6, dim=1)
                nc = F.layer_norm(xc, (H,), eps=1e-6) * (1 + mc[1][:, None]) + mc[0][:, None]
            q = torch.cat([self._lin(ni, f"{b}.attn.to_q"), self._lin(nc, f"{b}.attn.add_q_proj")], 1)
            k = torch.cat([self._lin(ni, f"{b}.attn.to_k"), self._lin(nc, f"{b}.attn.add_k_proj")], 1)
            v = torch.cat([self._lin(ni, f"{b}.attn.to_v"), self._lin(nc, f"{b}.attn.add_v_proj")], 1)
            T = q.shape[1]
            q, k, v = (z.view(n, T, heads, H // heads).transpose(1, 2) for z in (q, k, v))
            o = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(n, T, H)
            oi, oc = o[:, :Ti], o[:, Ti:]
            xi = xi + mi[2][:, None] * self._lin(oi, f"{b}.attn.to_out.0")
            ni = F.layer_norm(xi, (H,), eps=1e-6) * (1 + mi[4][:, None]) + mi[3][:, None]
            xi = xi + mi[5][:, None] * self._lin(F.gelu(self._lin(ni, f"{b}.ff.net.0.proj")), f"{b}.ff.net.2")
            if not last:
                xc = xc + mc[2][:, None] * self._lin(oc, f"{b}.attn.to_add_out")
                nc = F.layer_norm(xc, (H,), eps=1e-6) * (1 + mc[4][:, None]) + mc[3][:, None]
                xc = xc + mc[5][:, None] * self._lin(F.gelu(self._lin(nc, f"{b}.ff_context.net.0.proj")),
                                                       f"{b}.ff_context.net.2")
        scale, shift = self._lin(sc, "norm_out.linear").chunk(2, dim=1)
        y = F.layer_norm(xi, (H,), eps=1e-6) * (1 + scale[:, None]) + shift[:, None]
        o = self._lin(y, "proj_out")
        return o.float().view(n, gh, gw, P, P, C).permute(0, 1, 3, 2, 4, 5).reshape(n, Hl, Wl, C)
