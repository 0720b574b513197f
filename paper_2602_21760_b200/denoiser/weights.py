"""Architecture specs and deterministic random-init weights for the denoisers.

There are no checkpoints (no network); every denoiser is random-init with a
fixed seed. Weights are produced in a canonical fp32 PyTorch layout
(conv [co, ci, 3, 3], linear [out, in]) so the CPU fp32 reference in
``oracle/`` and the B200 modules (which re-lay them out as bf16 NHWC/K-major
tensors) consume the identical values. Each tensor is drawn from its own
generator seeded by (seed, index), so generation is order-independent and can
run on the CPU (parity) or directly on the GPU (benchmarks, faster).

Shapes follow the public SDXL U-Net (block channels 320/640/1280, transformer
depth 0/2/10, head dim 64, cross-attention dim 2048, text-time additional
embedding 2816) and SD3-medium MMDiT (24 joint blocks, hidden 1536, 24 heads,
patch 2, 16 latent channels) configurations.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch


@dataclass(frozen=True)
class UNetSpec:
    name: str = "sdxl"
    in_channels: int = 4
    out_channels: int = 4
    block_out: tuple = (320, 640, 1280)
    layers_per_block: int = 2
    transformer_depth: tuple = (0, 2, 10)
    mid_depth: int = 10
    cross_dim: int = 2048
    pooled_dim: int = 1280
    time_ids: int = 6
    time_id_dim: int = 256
    groups: int = 32
    head_dim: int = 64
    context_len: int = 77
    latent_hw: int = 128

    @property
    def temb_dim(self) -> int:
        return 4 * self.block_out[0]

    @property
    def add_in_dim(self) -> int:
        return self.pooled_dim + self.time_ids * self.time_id_dim


SDXL = UNetSpec()
SDXL_2048 = UNetSpec(name="sdxl-2048", latent_hw=256)
TINY = UNetSpec(name="tiny", block_out=(64, 128, 128), transformer_depth=(0, 1, 1), mid_depth=1,
                cross_dim=128, pooled_dim=128, time_id_dim=32, context_len=77, latent_hw=64)


@dataclass(frozen=True)
class MMDiTSpec:
    name: str = "sd3"
    in_channels: int = 16
    patch: int = 2
    hidden: int = 1536
    depth: int = 24
    heads: int = 24
    mlp_ratio: int = 4
    ctx_dim: int = 4096
    pooled_dim: int = 2048
    ctx_len: int = 333
    latent_hw: int = 128
    pos_max: int = 192
    freq_dim: int = 256


SD3 = MMDiTSpec()
TINY_DIT = MMDiTSpec(name="tiny-dit", in_channels=16, hidden=128, depth=2, heads=2, ctx_dim=128,
                     pooled_dim=128, ctx_len=77, latent_hw=32, pos_max=32, freq_dim=64)


# ---------------------------------------------------------------------------------
def unet_param_specs(s: UNetSpec) -> list:
    """(name, shape, kind) for every parameter, in a fixed order."""
    P = []

    def lin(name, o, i, bias=True, scale=1.0):
        P.append((name + ".weight", (o, i), ("lin", scale)))
        if bias:
            P.append((name + ".bias", (o,), ("bias", 0.0)))

    def conv(name, o, i, k=3, scale=1.0):
        P.append((name + ".weight", (o, i, k, k), ("lin", scale)))
        P.append((name + ".bias", (o,), ("bias", 0.0)))

    def norm(name, c):
        P.append((name + ".weight", (c,), ("one", 0.0)))
        P.append((name + ".bias", (c,), ("zero", 0.0)))

    def resnet(name, ci, co):
        norm(name + ".norm1", ci)
        conv(name + ".conv1", co, ci)
        lin(name + ".time_emb_proj", co, s.temb_dim)
        norm(name + ".norm2", co)
        conv(name + ".conv2", co, co, scale=0.5)
        if ci != co:
            conv(name + ".conv_shortcut", co, ci, k=1)

    def transformer(name, c, depth):
        norm(name + ".norm", c)
        lin(name + ".proj_in", c, c)
        for d in range(depth):
            b = f"{name}.transformer_blocks.{d}"
            for ln in ("norm1", "norm2", "norm3"):
                norm(f"{b}.{ln}", c)
            for a, kv_in in (("attn1", c), ("attn2", s.cross_dim)):
                lin(f"{b}.{a}.to_q", c, c, bias=False)
                lin(f"{b}.{a}.to_k", c, kv_in, bias=False)
                lin(f"{b}.{a}.to_v", c, kv_in, bias=False)
                lin(f"{b}.{a}.to_out.0", c, c, scale=0.5)
            lin(f"{b}.ff.net.0.proj", 8 * c, c)
            lin(f"{b}.ff.net.2", c, 4 * c, scale=0.5)
        lin(name + ".proj_out", c, c, scale=0.5)

    ch = s.block_out
    conv("conv_in", ch[0], s.in_channels)
    lin("time_embedding.linear_1", s.temb_dim, ch[0])
    lin("time_embedding.linear_2", s.temb_dim, s.temb_dim)
    lin("add_embedding.linear_1", s.temb_dim, s.add_in_dim)
    lin("add_embedding.linear_2", s.temb_dim, s.temb_dim)
    prev = ch[0]
    for lvl, co in enumerate(ch):
        for j in range(s.layers_per_block):
            ci = prev if j == 0 else co
            resnet(f"down_blocks.{lvl}.resnets.{j}", ci, co)
            if s.transformer_depth[lvl]:
                transformer(f"down_blocks.{lvl}.attentions.{j}", co, s.transformer_depth[lvl])
        if lvl < len(ch) - 1:
            conv(f"down_blocks.{lvl}.downsamplers.0.conv", co, co)
        prev = co
    resnet("mid_block.resnets.0", ch[-1], ch[-1])
    transformer("mid_block.attentions.0", ch[-1], s.mid_depth)
    resnet("mid_block.resnets.1", ch[-1], ch[-1])
    skips = unet_skip_channels(s)
    rev = list(reversed(ch))
    prev = ch[-1]
    for u, co in enumerate(rev):
        lvl = len(ch) - 1 - u
        for j in range(s.layers_per_block + 1):
            sk = skips.pop()
            resnet(f"up_blocks.{u}.resnets.{j}", prev + sk, co)
            prev = co
            if s.transformer_depth[lvl]:
                transformer(f"up_blocks.{u}.attentions.{j}", co, s.transformer_depth[lvl])
        if u < len(ch) - 1:
            conv(f"up_blocks.{u}.upsamplers.0.conv", co, co)
    norm("conv_norm_out", ch[0])
    conv("conv_out", s.out_channels, ch[0], scale=0.5)
    return P


def unet_skip_channels(s: UNetSpec) -> list:
    ch = s.block_out
    skips = [ch[0]]
    for lvl, co in enumerate(ch):
        skips += [co] * s.layers_per_block
        if lvl < len(ch) - 1:
            skips.append(co)
    return skips


def mmdit_param_specs(s: MMDiTSpec) -> list:
    P = []
    H = s.hidden

    def lin(name, o, i, bias=True, scale=1.0):
        P.append((name + ".weight", (o, i), ("lin", scale)))
        if bias:
            P.append((name + ".bias", (o,), ("bias", 0.0)))

    pdim = s.patch * s.patch * s.in_channels
    lin("pos_embed.proj", H, pdim)
    P.append(("pos_embed.pos", (s.pos_max * s.pos_max, H), ("pos", 0.0)))
    lin("context_embedder", H, s.ctx_dim)
    lin("time_text_embed.timestep_embedder.linear_1", H, s.freq_dim)
    lin("time_text_embed.timestep_embedder.linear_2", H, H)
    lin("time_text_embed.text_embedder.linear_1", H, s.pooled_dim)
    lin("time_text_embed.text_embedder.linear_2", H, H)
    for d in range(s.depth):
        b = f"transformer_blocks.{d}"
        last = d == s.depth - 1
        lin(f"{b}.norm1.linear", 6 * H, H, scale=0.2)
        lin(f"{b}.norm1_context.linear", (2 if last else 6) * H, H, scale=0.2)
        for nm in ("to_q", "to_k", "to_v"):
            lin(f"{b}.attn.{nm}", H, H)
            lin(f"{b}.attn.add_{nm[3]}_proj", H, H)
        lin(f"{b}.attn.to_out.0", H, H, scale=0.5)
        if not last:
            lin(f"{b}.attn.to_add_out", H, H, scale=0.5)
        lin(f"{b}.ff.net.0.proj", s.mlp_ratio * H, H)
        lin(f"{b}.ff.net.2", H, s.mlp_ratio * H, scale=0.5)
        if not last:
            lin(f"{b}.ff_context.net.0.proj", s.mlp_ratio * H, H)
            lin(f"{b}.ff_context.net.2", H, s.mlp_ratio * H, scale=0.5)
    lin("norm_out.linear", 2 * H, H, scale=0.2)
    lin("proj_out", pdim, H, scale=0.5)
    return P


def _fan_in(shape):
    return int(math.prod(shape[1:])) if len(shape) > 1 else 1


@dataclass(frozen=True)
class VAESpec:
    """SDXL-style AutoencoderKL decoder (latent -> pixels): the step after the
    denoising loop."""
    name: str = "sdxl-vae"
    latent_channels: int = 4
    out_channels: int = 3
    block_out: tuple = (128, 256, 512, 512)
    layers_per_block: int = 2
    groups: int = 32
    scaling_factor: float = 0.13025
    latent_hw: int = 128


VAE_SDXL = VAESpec()
VAE_TINY = VAESpec(name="vae-tiny", block_out=(64, 64, 128, 128), latent_hw=16)


def vae_decoder_param_specs(s: VAESpec) -> list:
    """(name, shape, kind) of the decoder half of AutoencoderKL (diffusers naming)."""
    P = []

    def lin(name, o, i):
        P.append((name + ".weight", (o, i), ("lin", 1.0)))
        P.append((name + ".bias", (o,), ("bias", 0.0)))

    def conv(name, o, i, k=3, scale=1.0):
        P.append((name + ".weight", (o, i, k, k), ("lin", scale)))
        P.append((name + ".bias", (o,), ("bias", 0.0)))

    def norm(name, c):
        P.append((name + ".weight", (c,), ("one", 0.0)))
        P.append((name + ".bias", (c,), ("zero", 0.0)))

    def resnet(name, ci, co):
        norm(name + ".norm1", ci)
        conv(name + ".conv1", co, ci)
        norm(name + ".norm2", co)
        conv(name + ".conv2", co, co, scale=0.5)
        if ci != co:
            conv(name + ".conv_shortcut", co, ci, k=1)

    rev = list(reversed(s.block_out))
    conv("post_quant_conv", s.latent_channels, s.latent_channels, k=1)
    conv("decoder.conv_in", rev[0], s.latent_channels)
    resnet("decoder.mid_block.resnets.0", rev[0], rev[0])
    a = "decoder.mid_block.attentions.0"
    norm(a + ".group_norm", rev[0])
    for nm in ("to_q", "to_k", "to_v"):
        lin(f"{a}.{nm}", rev[0], rev[0])
    lin(f"{a}.to_out.0", rev[0], rev[0])
    resnet("decoder.mid_block.resnets.1", rev[0], rev[0])
    prev = rev[0]
    for u, co in enumerate(rev):
        for j in range(s.layers_per_block + 1):
            resnet(f"decoder.up_blocks.{u}.resnets.{j}", prev if j == 0 else co, co)
        prev = co
        if u < len(rev) - 1:
            conv(f"decoder.up_blocks.{u}.upsamplers.0.conv", co, co)
    norm("decoder.conv_norm_out", rev[-1])
    conv("decoder.conv_out", s.out_channels, rev[-1])
    return P


def init_weights(specs, seed: int = 0, device="cpu", dtype=torch.float32) -> dict:
    """Deterministic random init; identical values for a given (seed, device type)."""
    out = {}
    dev = torch.device(device)
    for i, (name, shape, (kind, scale)) in enumerate(specs):
        g = torch.Generator(device=dev)
        g.manual_seed(seed * 1_000_003 + i)
        if kind == "lin":
            t = torch.randn(shape, generator=g, device=dev, dtype=torch.float32) * (scale / math.sqrt(_fan_in(shape)))
        elif kind == "bias":
            t = torch.randn(shape, generator=g, device=dev, dtype=torch.float32) * 0.02
        elif kind == "pos":
            t = torch.randn(shape, generator=g, device=dev, dtype=torch.float32) * 0.02
        elif kind == "one":
            t = torch.ones(shape, device=dev)
        else:
            t = torch.zeros(shape, device=dev)
        out[name] = t.to(dtype)
    return out


def count_params(specs) -> int:
    return sum(int(math.prod(s)) for _, s, _ in specs)


@dataclass
class Conditioning:
    """Synthetic prompt conditioning (no text encoders exist in this scope)."""

    context: torch.Tensor          # [rows, L, D]
    pooled: torch.Tensor           # [rows, P]
    null_context: torch.Tensor     # [1, L, D]  unconditional branch
    null_pooled: torch.Tensor      # [1, P]
    extra: dict = field(default_factory=dict)


def synthetic_conditioning(n_prompts: int, ctx_len: int, ctx_dim: int, pooled_dim: int, seed: int = 1234,
                           device="cpu") -> Conditioning:
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    ctx = torch.randn(n_prompts, ctx_len, ctx_dim, generator=g)
    pooled = torch.randn(n_prompts, pooled_dim, generator=g)
    null_ctx = torch.randn(1, ctx_len, ctx_dim, generator=g) * 0.1
    null_pooled = torch.randn(1, pooled_dim, generator=g) * 0.1
    return Conditioning(ctx.to(device), pooled.to(device), null_ctx.to(device), null_pooled.to(device))
