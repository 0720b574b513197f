"""SDXL's two CLIP text encoders on this package's kernels (the step before the
loop).

ViT-L/14 (12 layers, width 768, quick-GELU) and OpenCLIP ViT-bigG/14 (32
layers, width 1280, GELU, text projection) with causal self-attention over 77
tokens. SDXL conditions on the concatenated penultimate hidden states
([n, 77, 768 + 1280]) and on bigG's projected, final-layer-normed EOS token
([n, 1280]) — exactly the Conditioning the U-Net denoiser consumes. There is
no tokenizer (no vocabulary files in this scope): inputs are token ids. The
reference has no text encoders; parity is against the plain-torch
restatement ``oracle/text_ref.py``.

Kernels: token+position embedding gather, LayerNorm, fused-QKV / out / MLP
GEMMs (tcgen05 CTA pairs; GELU and residual adds fused in the epilogue;
quick-GELU as a separate elementwise pass), single-block causal attention
(head_dim 64).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import kernels as K
from .weights import Conditioning, init_weights


@dataclass(frozen=True)
class CLIPTextSpec:
    name: str
    vocab: int = 49408
    seq: int = 77
    hidden: int = 768
    heads: int = 12
    layers: int = 12
    mlp: int = 3072
    act: str = "quick_gelu"
    proj: int = 0            # text_projection width (0 = none)


CLIP_L = CLIPTextSpec("clip-vit-l-14")
CLIP_BIGG = CLIPTextSpec("openclip-vit-bigg-14", hidden=1280, heads=20, layers=32, mlp=5120, act="gelu", proj=1280)
CLIP_TINY_A = CLIPTextSpec("clip-tiny-a", vocab=1000, hidden=128, heads=2, layers=3, mlp=512)
CLIP_TINY_B = CLIPTextSpec("clip-tiny-b", vocab=1000, hidden=192, heads=3, layers=3, mlp=768, act="gelu", proj=128)


def clip_text_param_specs(s: CLIPTextSpec) -> list:
    """(name, shape, kind) in HF CLIPTextModel(WithProjection) naming."""
    P = []

    def lin(name, o, i, bias=True, scale=1.0):
        P.append((name + ".weight", (o, i), ("lin", scale)))
        if bias:
            P.append((name + ".bias", (o,), ("bias", 0.0)))

    def norm(name, c):
        P.append((name + ".weight", (c,), ("one", 0.0)))
        P.append((name + ".bias", (c,), ("zero", 0.0)))

    t = "text_model"
    P.append((f"{t}.embeddings.token_embedding.weight", (s.vocab, s.hidden), ("pos", 0.0)))
    P.append((f"{t}.embeddings.position_embedding.weight", (s.seq, s.hidden), ("pos", 0.0)))
    for i in range(s.layers):
        b = f"{t}.encoder.layers.{i}"
        norm(b + ".layer_norm1", s.hidden)
        for nm in ("q_proj", "k_proj", "v_proj"):
            lin(f"{b}.self_attn.{nm}", s.hidden, s.hidden)
        lin(f"{b}.self_attn.out_proj", s.hidden, s.hidden, scale=0.5)
        norm(b + ".layer_norm2", s.hidden)
        lin(f"{b}.mlp.fc1", s.mlp, s.hidden)
        lin(f"{b}.mlp.fc2", s.hidden, s.mlp, scale=0.5)
    norm(f"{t}.final_layer_norm", s.hidden)
    if s.proj:
        lin("text_projection", s.proj, s.hidden, bias=False)
    return P


class CLIPTextEncoder:
    def __init__(self, spec: CLIPTextSpec, W: dict, device="cuda"):
        self.s = s = spec
        dev = torch.device(device)
        t = "text_model"
        self.tok = W[f"{t}.embeddings.token_embedding.weight"].to(dev).float().contiguous()
        self.pos = W[f"{t}.embeddings.position_embedding.weight"].to(dev).float().contiguous()
        self.layers = []
        for i in range(s.layers):
            b = f"{t}.encoder.layers.{i}"
            g = lambda n: W[f"{b}.{n}"].to(dev)   # noqa: E731
            self.layers.append(dict(
                ln1=(g("layer_norm1.weight").float().contiguous(), g("layer_norm1.bias").float().contiguous()),
                qkv_w=torch.cat([g("self_attn.q_proj.weight"), g("self_attn.k_proj.weight"),
                                 g("self_attn.v_proj.weight")]).to(torch.bfloat16).contiguous(),
                qkv_b=torch.cat([g("self_attn.q_proj.bias"), g("self_attn.k_proj.bias"),
                                 g("self_attn.v_proj.bias")]).float().contiguous(),
                o_w=g("self_attn.out_proj.weight").to(torch.bfloat16).contiguous(),
                o_b=g("self_attn.out_proj.bias").float().contiguous(),
                ln2=(g("layer_norm2.weight").float().contiguous(), g("layer_norm2.bias").float().contiguous()),
                fc1_w=g("mlp.fc1.weight").to(torch.bfloat16).contiguous(), fc1_b=g("mlp.fc1.bias").float().contiguous(),
                fc2_w=g("mlp.fc2.weight").to(torch.bfloat16).contiguous(), fc2_b=g("mlp.fc2.bias").float().contiguous(),
            ))
        self.lnf = (W[f"{t}.final_layer_norm.weight"].to(dev).float().contiguous(),
                    W[f"{t}.final_layer_norm.bias"].to(dev).float().contiguous())
        self.proj = W["text_projection.weight"].to(dev).to(torch.bfloat16).contiguous() if s.proj else None
        self.quick = s.act == "quick_gelu"

    def _layer(self, x, n, L):
        s = self.s
        H = s.hidden
        y = K.layer_norm(x, H, gamma=L["ln1"][0], beta=L["ln1"][1], eps=1e-5)
        qkv = K.gemm(y, L["qkv_w"], bias=L["qkv_b"])
        att = torch.empty_like(y)
        K.attention(qkv, qkv, qkv, att, batch=n, heads=s.heads, sq=s.seq, skv=s.seq, scale=1.0 / math.sqrt(H // s.heads),
                    q_col0=0, k_col0=H, v_col0=2 * H, causal=True)
        x = K.gemm(att, L["o_w"], bias=L["o_b"], residual=x)
        y = K.layer_norm(x, H, gamma=L["ln2"][0], beta=L["ln2"][1], eps=1e-5)
        if self.quick:                        # quick GELU as its own pass (keeps the GEMM epilogue lean)
            h = K.quick_gelu(K.gemm(y, L["fc1_w"], bias=L["fc1_b"]))
        else:
            h = K.gemm(y, L["fc1_w"], bias=L["fc1_b"], act=K.ACT_GELU)
        return K.gemm(h, L["fc2_w"], bias=L["fc2_b"], residual=x)

    def encode(self, ids: torch.Tensor):
        """ids [n, seq] int64 -> (penultimate hidden states [n, seq, hidden] bf16,
        pooled [n, proj or hidden] fp32: final-layer-normed EOS token (argmax id),
        projected when the encoder has a projection)."""
        s = self.s
        ids = ids.to(self.tok.device, torch.int64).contiguous()
        n = ids.shape[0]
        x = K.embed_tokens(ids, self.tok, self.pos)
        penult = None
        for i, L in enumerate(self.layers):
            if i == s.layers - 1:
                penult = x
            x = self._layer(x, n, L)
        eos = ids.argmax(dim=1) + torch.arange(n, device=ids.device) * s.seq
        xe = x.index_select(0, eos).contiguous()
        pooled = K.layer_norm(xe, s.hidden, gamma=self.lnf[0], beta=self.lnf[1], eps=1e-5)
        if self.proj is not None:
            pooled = K.linear_small(pooled.float().contiguous(), self.proj)
        return penult.view(n, s.seq, s.hidden), pooled.float()


class SDXLTextEncoders:
    """Both encoders: token ids -> the U-Net's Conditioning (context ViT-L ++ bigG
    penultimate states, pooled = bigG projected EOS)."""

    def __init__(self, enc_l: CLIPTextEncoder, enc_g: CLIPTextEncoder):
        self.l, self.g = enc_l, enc_g

    def encode(self, ids: torch.Tensor):
        hl, _ = self.l.encode(ids)
        hg, pooled = self.g.encode(ids)
        n, L = ids.shape
        ctx = K.concat_channels(hl.reshape(n * L, -1), hl.shape[-1], hg.reshape(n * L, -1), hg.shape[-1], n * L)
        return ctx.view(n, L, -1), pooled

    def conditioning(self, prompt_ids: torch.Tensor, null_ids: torch.Tensor) -> Conditioning:
        ctx, pooled = self.encode(prompt_ids)
        nctx, npooled = self.encode(null_ids)
        return Conditioning(ctx.float(), pooled, nctx.float(), npooled)


def build_text_encoders(spec_l=CLIP_L, spec_g=CLIP_BIGG, seed: int = 0, device="cuda") -> SDXLTextEncoders:
    wl = init_weights(clip_text_param_specs(spec_l), seed=seed, device=device)
    wg = init_weights(clip_text_param_specs(spec_g), seed=seed + 1, device=device)
    return SDXLTextEncoders(CLIPTextEncoder(spec_l, wl, device), CLIPTextEncoder(spec_g, wg, device))
