"""SDXL-style VAE decoder (AutoencoderKL decoder half) on this package's kernels.

The step right after the denoising loop: x0 latents
[n, h, w, 4] -> pixels [n, 8h, 8w, 3]. The reference has no decoder (its loop
ends at x0), so parity is against the plain-torch fp32
restatement ``oracle/vae_ref.py`` of the same architecture and weights.

Layout and kernels are the U-Net's: NHWC bf16 activations, 3x3 convolutions as
tensor-core implicit GEMMs (the 4 latent channels and the 3 pixel channels are
zero-padded to 64 by ``copy_cols``), GroupNorm(+SiLU) single-launch kernels,
nearest-2x upsampling fused with the following 3x3 conv (four sub-pixel 2x2
convs in one launch, ``kernels.upsample_conv``). The mid-block attention is one head of width 512 over
all (h*w) latent positions; it runs as Q K^T (GEMM, bf16 scores) -> row
softmax -> P V (GEMM against V^T, which a GEMM produces directly as
W_v . x^T; the V bias folds into the output projection because softmax rows
sum to one).
"""
from __future__ import annotations

import math

import torch

from . import kernels as K
from .weights import VAESpec, init_weights, vae_decoder_param_specs


def _bf(t):
    return t.to(torch.bfloat16).contiguous()


def _f32(t):
    return t.to(torch.float32).contiguous()


class _Conv:
    def __init__(self, W, name, dev, cin_pad=None, cout_pad=None, scale=1.0):
        w = W[name + ".weight"].to(dev).float() * scale          # [co, ci, k, k]
        b = W[name + ".bias"].to(dev).float()
        co, ci, kh, _ = w.shape
        ci_p = cin_pad or ci
        co_p = cout_pad or co
        wp = torch.zeros(co_p, kh, kh, ci_p, device=dev)
        wp[:co, :, :, :ci] = w.permute(0, 2, 3, 1)
        bp = torch.zeros(co_p, device=dev)
        bp[:co] = b
        self.k, self.ci, self.co = kh, ci_p, co_p
        self.w = _bf(wp.reshape(co_p, kh * kh * ci_p))
        self.b = _f32(bp)

    def __call__(self, x, n, h, w, **kw):
        if self.k == 1:
            return K.gemm(x, self.w, bias=self.b, **kw)
        return K.gemm(x, self.w, bias=self.b, conv=(n, h, w, self.ci, 1), **kw)


class _Norm:
    def __init__(self, W, name, dev):
        self.g = _f32(W[name + ".weight"].to(dev))
        self.b = _f32(W[name + ".bias"].to(dev))


class _Resnet:
    def __init__(self, W, name, dev):
        self.n1, self.n2 = _Norm(W, name + ".norm1", dev), _Norm(W, name + ".norm2", dev)
        self.c1, self.c2 = _Conv(W, name + ".conv1", dev), _Conv(W, name + ".conv2", dev)
        self.short = _Conv(W, name + ".conv_shortcut", dev) if (name + ".conv_shortcut.weight") in W else None

    def __call__(self, x, n, h, w, groups, stats):
        ci, co = self.c1.ci, self.c1.co
        y = K.group_norm(x, n, h * w, ci, self.n1.g, self.n1.b, groups=groups, eps=1e-6, silu=True, stats=stats)
        y = self.c1(y, n, h, w)
        y = K.group_norm(y, n, h * w, co, self.n2.g, self.n2.b, groups=groups, eps=1e-6, silu=True, stats=stats)
        res = self.short(x, n, h, w) if self.short is not None else x
        return self.c2(y, n, h, w, residual=res)


class _MidAttention:
    def __init__(self, W, name, c, dev):
        self.c = c
        self.norm = _Norm(W, name + ".group_norm", dev)
        self.wq, self.bq = _bf(W[name + ".to_q.weight"].to(dev)), _f32(W[name + ".to_q.bias"].to(dev))
        self.wk, self.bk = _bf(W[name + ".to_k.weight"].to(dev)), _f32(W[name + ".to_k.bias"].to(dev))
        self.wv = _bf(W[name + ".to_v.weight"].to(dev))
        wo = W[name + ".to_out.0.weight"].to(dev).float()
        self.wo = _bf(wo)
        # softmax rows sum to 1: P (V + 1 b_v^T) W_o^T + b_o = P V W_o^T + (W_o b_v + b_o)
        self.bo = _f32(W[name + ".to_out.0.bias"].to(dev).float() + wo @ W[name + ".to_v.bias"].to(dev).float())

    def __call__(self, x, n, hw, groups, stats):
        c = self.c
        xn = K.group_norm(x, n, hw, c, self.norm.g, self.norm.b, groups=groups, eps=1e-6, stats=stats)
        q = K.gemm(xn, self.wq, bias=self.bq)
        k = K.gemm(xn, self.wk, bias=self.bk)
        o = torch.empty_like(xn)
        scale = 1.0 / math.sqrt(c)
        for i in range(n):                       # one image at a time: scores are hw x hw
            rows = slice(i * hw, (i + 1) * hw)
            vt = K.gemm(self.wv, xn[rows])                       # V^T [c, hw] = W_v . x^T
            s = K.gemm(q[rows], k[rows])                         # [hw, hw] bf16 scores
            p = K.softmax_rows(s, scale=scale)
            K.gemm(p, vt, out=o[rows])                           # P V
        return K.gemm(o, self.wo, bias=self.bo, residual=x)


class VAEDecoder:
    """``decode(latents)``: latents [n, h, w, 4] (the loop's x0, NHWC, any float
    dtype) -> images [n, 8h, 8w, 3] fp32 in roughly [-1, 1]."""

    PAD = 64

    def __init__(self, spec: VAESpec, W: dict, device="cuda"):
        self.spec = s = spec
        dev = torch.device(device)
        self.dev = dev
        rev = list(reversed(s.block_out))
        # 1 / scaling_factor folded into post_quant_conv; 4 latent channels padded to 64
        self.pq = _Conv(W, "post_quant_conv", dev, cin_pad=self.PAD, cout_pad=self.PAD, scale=1.0 / s.scaling_factor)
        self.conv_in = _Conv(W, "decoder.conv_in", dev, cin_pad=self.PAD)
        self.mid = (_Resnet(W, "decoder.mid_block.resnets.0", dev),
                    _MidAttention(W, "decoder.mid_block.attentions.0", rev[0], dev),
                    _Resnet(W, "decoder.mid_block.resnets.1", dev))
        self.up = []
        for u in range(len(rev)):
            res = [_Resnet(W, f"decoder.up_blocks.{u}.resnets.{j}", dev) for j in range(s.layers_per_block + 1)]
            us = None
            if u < len(rev) - 1:     # nearest-2x + 3x3 conv as one sub-pixel launch (HP_A_UPCONV)
                name = f"decoder.up_blocks.{u}.upsamplers.0.conv"
                us = (_Conv(W, name, dev), K.upconv_weights(W[name + ".weight"].to(dev).permute(0, 2, 3, 1)))
            self.up.append((res, us))
        self.norm_out = _Norm(W, "decoder.conv_norm_out", dev)
        self.conv_out = _Conv(W, "decoder.conv_out", dev, cout_pad=self.PAD)
        self.stats = torch.empty(2 * 64 * 64 * 32, dtype=torch.float32, device=dev)

    def decode(self, latents: torch.Tensor) -> torch.Tensor:
        s = self.spec
        n, h, w, c = latents.shape
        if c != s.latent_channels:
            raise ValueError(f"expected {s.latent_channels} latent channels, got {c}")
        g, st = s.groups, self.stats
        z = K.copy_cols(_bf(latents.to(self.dev)).view(n * h * w, c), self.PAD)
        z = self.pq(z, n, h, w)
        x = self.conv_in(z, n, h, w)
        r0, att, r1 = self.mid
        x = r0(x, n, h, w, g, st)
        x = att(x, n, h * w, g, st)
        x = r1(x, n, h, w, g, st)
        for res, us in self.up:
            for r in res:
                x = r(x, n, h, w, g, st)
            if us is not None:
                conv, w4 = us
                if n * h * w > 128:                    # CTA-pair kernel (M > 128 rows)
                    x = K.upsample_conv(x, n, h, w, conv.ci, w4, conv.b)
                else:
                    x = conv(K.upsample2x(x, n, h, w, x.shape[1]), n, 2 * h, 2 * w)
                h, w = 2 * h, 2 * w
        y = K.group_norm(x, n, h * w, x.shape[1], self.norm_out.g, self.norm_out.b, groups=g, eps=1e-6, silu=True,
                         stats=st)
        img = K.copy_cols(self.conv_out(y, n, h, w), s.out_channels)
        return img.float().view(n, h, w, s.out_channels)


def build_vae(spec: VAESpec, seed: int = 0, device="cuda", weights: dict | None = None) -> VAEDecoder:
    if weights is None:
        weights = init_weights(vae_decoder_param_specs(spec), seed=seed, device=device)
    return VAEDecoder(spec, weights, device=device)


def vae_decoder_flops(spec: VAESpec, n: int) -> float:
    """Analytic multiply-add count x2 of the decoder (convolutions + attention)."""
    rev = list(reversed(spec.block_out))
    h = w = spec.latent_hw
    fl = 0.0

    def conv(px, ci, co, k=3):
        return 2.0 * px * co * k * k * ci

    px = h * w
    fl += conv(px, spec.latent_channels, rev[0])
    fl += 4 * conv(px, rev[0], rev[0])                                   # mid resnets
    fl += 2.0 * px * rev[0] * rev[0] * 4 + 4.0 * px * px * rev[0]         # mid attention projections + QK^T, PV
    prev = rev[0]
    for u, co in enumerate(rev):
        for j in range(spec.layers_per_block + 1):
            ci = prev if j == 0 else co
            fl += conv(px, ci, co) + conv(px, co, co) + (conv(px, ci, co, k=1) if ci != co else 0.0)
        prev = co
        if u < len(rev) - 1:
            px *= 4
            fl += conv(px, co, co) * 4 / 9                               # sub-pixel upsampler (HP_A_UPCONV)
    fl += conv(px, rev[-1], spec.out_channels)
    return n * fl
