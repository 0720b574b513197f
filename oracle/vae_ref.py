"""ORACLE (test infrastructure only): plain-torch fp32 NCHW restatement of the
SDXL-style VAE decoder (diffusers AutoencoderKL.decode semantics:
post_quant_conv on latents / scaling_factor, conv_in, mid block = resnet,
single-head self-attention with group norm and residual, resnet; up blocks
of (layers_per_block + 1) resnets with nearest-2x + conv upsamplers; group
norm, SiLU, conv_out), consuming the canonical weights of
``paper_2602_21760_b200.denoiser.weights.vae_decoder_param_specs``. Stock
torch.nn.functional ops only — none of the package's kernels. The reference
has no decoder: parity for this row is against this restatement.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F


class VAEDecoderRef:
    def __init__(self, spec, W: dict):
        self.s = spec
        self.W = {k: v.float() for k, v in W.items()}

    def _conv(self, x, name):
        w = self.W[name + ".weight"]
        return F.conv2d(x, w, self.W[name + ".bias"], padding=w.shape[-1] // 2)

    def _gn(self, x, name, silu):
        y = F.group_norm(x, self.s.groups, self.W[name + ".weight"], self.W[name + ".bias"], eps=1e-6)
        return F.silu(y) if silu else y

    def _resnet(self, x, name):
        y = self._conv(self._gn(x, name + ".norm1", True), name + ".conv1")
        y = self._conv(self._gn(y, name + ".norm2", True), name + ".conv2")
        res = self._conv(x, name + ".conv_shortcut") if (name + ".conv_shortcut.weight") in self.W else x
        return res + y

    def _attention(self, x, name):
        n, c, h, w = x.shape
        t = self._gn(x, name + ".group_norm", False).reshape(n, c, h * w).transpose(1, 2)   # [n, hw, c]
        q = F.linear(t, self.W[name + ".to_q.weight"], self.W[name + ".to_q.bias"])
        k = F.linear(t, self.W[name + ".to_k.weight"], self.W[name + ".to_k.bias"])
        v = F.linear(t, self.W[name + ".to_v.weight"], self.W[name + ".to_v.bias"])
        p = torch.softmax(q @ k.transpose(1, 2) / c ** 0.5, dim=-1)
        o = F.linear(p @ v, self.W[name + ".to_out.0.weight"], self.W[name + ".to_out.0.bias"])
        return x + o.transpose(1, 2).reshape(n, c, h, w)

    @torch.no_grad()
    def decode(self, latents_nhwc: torch.Tensor) -> torch.Tensor:
        s = self.s
        z = latents_nhwc.float().permute(0, 3, 1, 2) / s.scaling_factor
        z = self._conv(z, "post_quant_conv")
        x = self._conv(z, "decoder.conv_in")
        x = self._resnet(x, "decoder.mid_block.resnets.0")
        x = self._attention(x, "decoder.mid_block.attentions.0")
        x = self._resnet(x, "decoder.mid_block.resnets.1")
        for u in range(len(s.block_out)):
            for j in range(s.layers_per_block + 1):
                x = self._resnet(x, f"decoder.up_blocks.{u}.resnets.{j}")
            if u < len(s.block_out) - 1:
                x = F.interpolate(x, scale_factor=2.0, mode="nearest")
                x = self._conv(x, f"decoder.up_blocks.{u}.upsamplers.0.conv")
        x = self._conv(self._gn(x, "decoder.conv_norm_out", True), "decoder.conv_out")
        return x.permute(0, 2, 3, 1).contiguous()                                       # NHWC
