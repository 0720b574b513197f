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

    def run_units(self, state, t, context, pooled, a, b):
        """Units [a, b) of [embed, block 0..depth-1, out] on a boundary state:
        ``{"x": NHWC latent}`` before unit 0, ``{"eps": NHWC}`` after the last,
        else ``{"xi": image tokens, "xc": text tokens, "hw": (Hl, Wl)}``; the
        conditioning vector is recomputed from t in every stage."""
        s, W = self.s, self.W
        P, H = s.patch, s.hidden
        C = s.in_channels
        if a == 0:
            x_nhwc = state["x"]
            n, Hl, Wl, _ = x_nhwc.shape
        else:
            xi, xc = state["xi"], state["xc"]
            n = xi.shape[0]
            Hl, Wl = state["hw"]
        gh, gw = Hl // P, Wl // P
        te = F.silu(self._lin(_sinus(t, s.freq_dim).to(self.dt), "time_text_embed.timestep_embedder.linear_1"))
        te = self._lin(te, "time_text_embed.timestep_embedder.linear_2")
        pe = F.silu(self._lin(pooled.to(self.dt), "time_text_embed.text_embedder.linear_1"))
        c = te + self._lin(pe, "time_text_embed.text_embedder.linear_2")
        sc = F.silu(c)
        heads = s.heads
        units = ["embed"] + [d for d in range(s.depth)] + ["out"]
        for u in units[a:b]:
            if u == "embed":
                tok = x_nhwc.to(self.dt).view(n, gh, P, gw, P, C).permute(0, 1, 3, 2, 4, 5).reshape(n, gh * gw, P * P * C)
                off = (s.pos_max - gh) // 2
                pos = W["pos_embed.pos"].view(s.pos_max, s.pos_max, H)[off:off + gh, off:off + gw].reshape(gh * gw, H)
                xi = self._lin(tok, "pos_embed.proj") + pos
                xc = self._lin(context.to(self.dt), "context_embedder")
                continue
            if u == "out":
                scale, shift = self._lin(sc, "norm_out.linear").chunk(2, dim=1)
                y = F.layer_norm(xi, (H,), eps=1e-6) * (1 + scale[:, None]) + shift[:, None]
                o = self._lin(y, "proj_out")
                return {"eps": o.float().view(n, gh, gw, P, P, C).permute(0, 1, 3, 2, 4, 5).reshape(n, Hl, Wl, C)}
            d = u
            Ti = xi.shape[1]
            b_ = f"transformer_blocks.{d}"
            last = d == s.depth - 1
            mi = self._lin(sc, f"{b_}.norm1.linear").chunk(6, dim=1)
            mc_raw = self._lin(sc, f"{b_}.norm1_context.linear")
            ni = F.layer_norm(xi, (H,), eps=1e-6) * (1 + mi[1][:, None]) + mi[0][:, None]
            if last:
                c_scale, c_shift = mc_raw.chunk(2, dim=1)
                nc = F.layer_norm(xc, (H,), eps=1e-6) * (1 + c_scale[:, None]) + c_shift[:, None]
            else:
                mc = mc_raw.chunk(6, dim=1)
                nc = F.layer_norm(xc, (H,), eps=1e-6) * (1 + mc[1][:, None]) + mc[0][:, None]
            q = torch.cat([self._lin(ni, f"{b_}.attn.to_q"), self._lin(nc, f"{b_}.attn.add_q_proj")], 1)
            k = torch.cat([self._lin(ni, f"{b_}.attn.to_k"), self._lin(nc, f"{b_}.attn.add_k_proj")], 1)
            v = torch.cat([self._lin(ni, f"{b_}.attn.to_v"), self._lin(nc, f"{b_}.attn.add_v_proj")], 1)
            T = q.shape[1]
            q, k, v = (z.view(n, T, heads, H // heads).transpose(1, 2) for z in (q, k, v))
            o = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(n, T, H)
            oi, oc = o[:, :Ti], o[:, Ti:]
            xi = xi + mi[2][:, None] * self._lin(oi, f"{b_}.attn.to_out.0")
            ni = F.layer_norm(xi, (H,), eps=1e-6) * (1 + mi[4][:, None]) + mi[3][:, None]
            xi = xi + mi[5][:, None] * self._lin(F.gelu(self._lin(ni, f"{b_}.ff.net.0.proj")), f"{b_}.ff.net.2")
            if not last:
                xc = xc + mc[2][:, None] * self._lin(oc, f"{b_}.attn.to_add_out")
                nc = F.layer_norm(xc, (H,), eps=1e-6) * (1 + mc[4][:, None]) + mc[3][:, None]
                xc = xc + mc[5][:, None] * self._lin(F.gelu(self._lin(nc, f"{b_}.ff_context.net.0.proj")),
                                                       f"{b_}.ff_context.net.2")
        return {"xi": xi, "xc": xc, "hw": (Hl, Wl)}

    def __call__(self, x_nhwc, t, context, pooled):
        """x [n, H, W, C] fp32 latent (NHWC), t [n] network timesteps -> velocity NHWC."""
        return self.run_units({"x": x_nhwc}, t, context, pooled, 0, self.s.depth + 2)["eps"]
