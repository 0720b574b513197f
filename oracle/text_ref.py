"""ORACLE (test infrastructure only): plain-torch fp32 restatement of a CLIP
text transformer (HF CLIPTextModel(WithProjection) semantics: token + position
embedding, pre-LN blocks with causal multi-head self-attention and a quick-GELU
or GELU MLP, final LayerNorm; SDXL reads the penultimate hidden states and the
projected final-normed EOS token), consuming the weights of
``paper_2602_21760_b200.denoiser.text_encoders.clip_text_param_specs``. Stock
torch ops only. The reference has no text encoders.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F


class CLIPTextRef:
    def __init__(self, spec, W: dict):
        self.s = spec
        self.W = {k: v.float() for k, v in W.items()}

    def _lin(self, x, name, bias=True):
        return F.linear(x, self.W[name + ".weight"], self.W.get(name + ".bias") if bias else None)

    def _ln(self, x, name):
        return F.layer_norm(x, (x.shape[-1],), self.W[name + ".weight"], self.W[name + ".bias"], eps=1e-5)

    @torch.no_grad()
    def encode(self, ids: torch.Tensor):
        s, W = self.s, self.W
        t = "text_model"
        n, L = ids.shape
        x = W[f"{t}.embeddings.token_embedding.weight"][ids] + W[f"{t}.embeddings.position_embedding.weight"][:L]
        hd = s.hidden // s.heads
        mask = torch.full((L, L), float("-inf"), device=ids.device).triu(1)
        penult = None
        for i in range(s.layers):
            if i == s.layers - 1:
                penult = x
            b = f"{t}.encoder.layers.{i}"
            y = self._ln(x, b + ".layer_norm1")
            q = self._lin(y, b + ".self_attn.q_proj").view(n, L, s.heads, hd).transpose(1, 2)
            k = self._lin(y, b + ".self_attn.k_proj").view(n, L, s.heads, hd).transpose(1, 2)
            v = self._lin(y, b + ".self_attn.v_proj").view(n, L, s.heads, hd).transpose(1, 2)
            p = torch.softmax(q @ k.transpose(-1, -2) / hd ** 0.5 + mask, dim=-1)
            o = (p @ v).transpose(1, 2).reshape(n, L, s.hidden)
            x = x + self._lin(o, b + ".self_attn.out_proj")
            y = self._ln(x, b + ".layer_norm2")
            h = self._lin(y, b + ".mlp.fc1")
            h = h * torch.sigmoid(1.702 * h) if s.act == "quick_gelu" else F.gelu(h)
            x = x + self._lin(h, b + ".mlp.fc2")
        xe = x[torch.arange(n), ids.argmax(dim=1)]
        pooled = self._ln(xe, f"{t}.final_layer_norm")
        if s.proj:
            pooled = F.linear(pooled, W["text_projection.weight"])
        return penult, pooled
