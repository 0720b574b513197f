"""SD3-shaped MMDiT (joint-attention diffusion transformer) on our kernels.

Token buffer X is [n, T_img + T_ctx, H] bf16 (image tokens first, then text
tokens, per image), so the joint attention reads one contiguous sequence per
image while the per-stream weights run as batched GEMMs over row ranges
(3-D TMA maps, no copies). Per block:

  joint modulated LayerNorm (one launch, image / text rows pick their own
  adaLN shift/scale) -> batched QKV GEMMs per stream -> joint attention over
  T = 4096 + 333 tokens -> output GEMMs with the adaLN-Zero gate and the
  residual fused in the epilogue (d = x + gate * (o W^T + b)) -> joint
  modulated LayerNorm -> GELU MLP GEMM -> gated-residual MLP GEMM.

The modulation vectors of both streams come from one small GEMV over SiLU(c)
(weights concatenated), the patch embedding adds the positional table in the
GEMM epilogue, and the text-context projection and pooled-text embedding are
per-run (``prepare``). The last block is context-pre-only (no text output
projection / MLP), as in SD3.
"""
from __future__ import annotations

import math

import torch

from . import kernels as K
from .weights import MMDiTSpec, mmdit_param_specs


def _bf(t):
    return t.to(torch.bfloat16).contiguous()


def _f32(t):
    return t.to(torch.float32).contiguous()


class MMDiT:
    """Random-init SD3-shaped MMDiT; ``forward`` maps bf16 NHWC latents to velocity."""

    def __init__(self, spec: MMDiTSpec, W: dict, device="cuda"):
        self.spec = s = spec
        dev = torch.device(device)
        self.dev = dev
        H = s.hidden
        g = lambda n: W[n].to(dev)  # noqa: E731
        self.patch_w, self.patch_b = _bf(g("pos_embed.proj.weight")), _f32(g("pos_embed.proj.bias"))
        grid = s.latent_hw // s.patch
        off = (s.pos_max - grid) // 2
        pos = g("pos_embed.pos").view(s.pos_max, s.pos_max, H)[off:off + grid, off:off + grid]
        self.pos = _bf(pos.reshape(grid * grid, H))
        self.ctx_w, self.ctx_b = _bf(g("context_embedder.weight")), _f32(g("context_embedder.bias"))
        tt = "time_text_embed"
        self.t1w, self.t1b = _bf(g(f"{tt}.timestep_embedder.linear_1.weight")), _f32(g(f"{tt}.timestep_embedder.linear_1.bias"))
        self.t2w, self.t2b = _bf(g(f"{tt}.timestep_embedder.linear_2.weight")), _f32(g(f"{tt}.timestep_embedder.linear_2.bias"))
        self.p1w, self.p1b = _bf(g(f"{tt}.text_embedder.linear_1.weight")), _f32(g(f"{tt}.text_embedder.linear_1.bias"))
        self.p2w, self.p2b = _bf(g(f"{tt}.text_embedder.linear_2.weight")), _f32(g(f"{tt}.text_embedder.linear_2.bias"))
        self.blocks = []
        for d in range(s.depth):
            b = f"transformer_blocks.{d}"
            last = d == s.depth - 1
            blk = {"last": last}
            blk["mod_w"] = _bf(torch.cat([g(f"{b}.norm1.linear.weight"), g(f"{b}.norm1_context.linear.weight")]))
            blk["mod_b"] = _f32(torch.cat([g(f"{b}.norm1.linear.bias"), g(f"{b}.norm1_context.linear.bias")]))
            blk["qkv_i_w"] = _bf(torch.cat([g(f"{b}.attn.to_{c}.weight") for c in "qkv"]))
            blk["qkv_i_b"] = _f32(torch.cat([g(f"{b}.attn.to_{c}.bias") for c in "qkv"]))
            blk["qkv_c_w"] = _bf(torch.cat([g(f"{b}.attn.add_{c}_proj.weight") for c in "qkv"]))
            blk["qkv_c_b"] = _f32(torch.cat([g(f"{b}.attn.add_{c}_proj.bias") for c in "qkv"]))
            blk["o_i_w"], blk["o_i_b"] = _bf(g(f"{b}.attn.to_out.0.weight")), _f32(g(f"{b}.attn.to_out.0.bias"))
            blk["m1_i_w"], blk["m1_i_b"] = _bf(g(f"{b}.ff.net.0.proj.weight")), _f32(g(f"{b}.ff.net.0.proj.bias"))
            blk["m2_i_w"], blk["m2_i_b"] = _bf(g(f"{b}.ff.net.2.weight")), _f32(g(f"{b}.ff.net.2.bias"))
            if not last:
                blk["o_c_w"], blk["o_c_b"] = _bf(g(f"{b}.attn.to_add_out.weight")), _f32(g(f"{b}.attn.to_add_out.bias"))
                blk["m1_c_w"], blk["m1_c_b"] = _bf(g(f"{b}.ff_context.net.0.proj.weight")), _f32(g(f"{b}.ff_context.net.0.proj.bias"))
                blk["m2_c_w"], blk["m2_c_b"] = _bf(g(f"{b}.ff_context.net.2.weight")), _f32(g(f"{b}.ff_context.net.2.bias"))
            self.blocks.append(blk)
        self.nout_w, self.nout_b = _bf(g("norm_out.linear.weight")), _f32(g("norm_out.linear.bias"))
        self.out_w, self.out_b = _bf(g("proj_out.weight")), _f32(g("proj_out.bias"))
        # every block's adaLN modulation weights (and norm_out's) stacked in forward order,
        # so one GEMV per stage computes all of them at the HBM rate (they depend on the
        # step's conditioning vector only); the per-block entries are row views into it
        mw = torch.cat([blk["mod_w"] for blk in self.blocks] + [self.nout_w])
        mb = torch.cat([blk["mod_b"] for blk in self.blocks] + [self.nout_b])
        self.mod_w_all, self.mod_b_all = mw.contiguous(), mb.contiguous()
        self.mod_rows = [0]
        for blk in self.blocks:
            self.mod_rows.append(self.mod_rows[-1] + blk["mod_w"].shape[0])
        self.mod_rows.append(self.mod_rows[-1] + self.nout_w.shape[0])
        for d, blk in enumerate(self.blocks):
            blk["mod_w"] = self.mod_w_all[self.mod_rows[d]:self.mod_rows[d + 1]]
            blk["mod_b"] = self.mod_b_all[self.mod_rows[d]:self.mod_rows[d + 1]]
        self.ctx_cache, self.pemb = {}, {}

    @staticmethod
    def timestep_for(t: int, T: int) -> float:
        return 1000.0 * t / T                      # flow-matching sigma * 1000

    def prepare(self, context: torch.Tensor, pooled: torch.Tensor, key="default"):
        s = self.spec
        n = context.shape[0]
        ctx = _bf(context.to(self.dev).reshape(n * s.ctx_len, s.ctx_dim))
        self.ctx_cache[key] = K.gemm(ctx, self.ctx_w, bias=self.ctx_b).view(n, s.ctx_len, s.hidden)
        p = K.linear_small(_f32(pooled.to(self.dev)), self.p1w, self.p1b, act_out=K.ACT_SILU)
        self.pemb[key] = K.linear_small(p, self.p2w, self.p2b)

    @property
    def units(self):
        """Forward units (stage-split granularity): patch + context embedding, the
        joint blocks, the output head."""
        return [("embed",)] + [("block", d) for d in range(self.spec.depth)] + [("out",)]

    @property
    def unit_flops(self):
        return [f for _, f in mmdit_units(self.spec)]

    def run_units(self, state: dict, t: torch.Tensor, key: str, a: int, b: int, record=None) -> dict:
        """Units [a, b) on a boundary state: ``{"x": latent}`` before unit 0,
        ``{"eps": velocity}`` after the last, else ``{"X": joint token buffer
        [n, Ti + L, H], "hw": (Hl, Wl)}``. The conditioning vector is recomputed
        from the current step's t in every stage. ``record``: {unit index: None}
        filled with a COPY of the token buffer entering each listed unit (the
        blocks update it in place)."""
        s = self.spec
        H, P = s.hidden, s.patch
        L = s.ctx_len
        heads = s.heads
        if a == 0:
            x = state["x"]
            n, Hl, Wl, C = x.shape
        else:
            X = state["X"]
            n = X.shape[0]
            Hl, Wl = state["hw"]
            C = s.in_channels
        Ti = (Hl // P) * (Wl // P)
        T = Ti + L
        dev = self.dev
        te = K.timestep_embedding(t, s.freq_dim)
        te = K.linear_small(te, self.t1w, self.t1b, act_out=K.ACT_SILU)
        c = K.linear_small(te, self.t2w, self.t2b) + self.pemb[key]
        qkv = torch.empty((n, T, 3 * H), dtype=torch.bfloat16, device=dev)
        att = torch.empty((n, T, H), dtype=torch.bfloat16, device=dev)
        hid_i = torch.empty((n, Ti, s.mlp_ratio * H), dtype=torch.bfloat16, device=dev)
        hid_c = torch.empty((n, L, s.mlp_ratio * H), dtype=torch.bfloat16, device=dev)
        scale = 1.0 / math.sqrt(H // heads)
        units = self.units
        # modulation vectors of the blocks (and output norm) this stage runs: one GEMV over
        # the stacked weight rows [r0, r1)
        d0 = max(a, 1) - 1
        d1 = min(b - 1, s.depth)                   # blocks [d0, d1); unit depth+1 is the output head
        r0 = self.mod_rows[d0]
        r1 = self.mod_rows[d1 + 1] if b == len(units) else self.mod_rows[d1]
        mods = (K.linear_small(c, self.mod_w_all[r0:r1], self.mod_b_all[r0:r1], act_in=K.ACT_SILU)
                if r1 > r0 else None)
        for i in range(a, b):
            u = units[i]
            if record is not None and i in record:
                record[i] = {"X": X.clone(), "hw": (Hl, Wl)}
            if u[0] == "embed":
                X = torch.empty((n, T, H), dtype=torch.bfloat16, device=dev)
                tok = K.patchify(x, n, Hl, Wl, C, P).view(n, Ti, P * P * C)
                K.gemm(tok, self.patch_w, bias=self.patch_b, residual=self.pos, out=X[:, :Ti])
                X[:, Ti:].copy_(self.ctx_cache[key])
                continue
            if u[0] == "out":
                nf = mods[:, self.mod_rows[s.depth] - r0:self.mod_rows[s.depth + 1] - r0]   # [n, 2H]: scale, shift
                Y = K.layer_norm_joint(X, H, T, Ti, nf[:, H:2 * H], nf[:, 0:H], nf[:, H:2 * H], nf[:, 0:H],
                                       mods.shape[1])
                o = K.gemm(Y[:, :Ti], self.out_w, bias=self.out_b)                       # [n, Ti, P*P*C]
                v = K.patchify(o, n, Hl, Wl, C, P, inverse=True)
                return {"eps": v.view(n, Hl, Wl, C)}
            blk = self.blocks[u[1]]
            last = blk["last"]
            d = u[1]
            mod = mods[:, self.mod_rows[d] - r0:self.mod_rows[d + 1] - r0]      # [n, 12H] (8H last)
            ldm = mods.shape[1]
            mi = mod[:, :6 * H]
            mc = mod[:, 6 * H:]
            # image: shift_msa, scale_msa, gate_msa, shift_mlp, scale_mlp, gate_mlp
            # text (last block: AdaLayerNormContinuous -> scale, shift)
            if last:
                c_shift, c_scale = mc[:, H:2 * H], mc[:, 0:H]
            else:
                c_shift, c_scale = mc[:, 0:H], mc[:, H:2 * H]
            Y = K.layer_norm_joint(X, H, T, Ti, mi[:, 0:H], mi[:, H:2 * H], c_shift, c_scale, ldm)
            K.gemm(Y[:, :Ti], blk["qkv_i_w"], bias=blk["qkv_i_b"], out=qkv[:, :Ti])
            K.gemm(Y[:, Ti:], blk["qkv_c_w"], bias=blk["qkv_c_b"], out=qkv[:, Ti:])
            q2 = qkv.view(n * T, 3 * H)
            K.attention(q2, q2, q2, att.view(n * T, H), batch=n, heads=heads, sq=T, skv=T, scale=scale,
                        q_col0=0, k_col0=H, v_col0=2 * H)
            K.gemm(att[:, :Ti], blk["o_i_w"], bias=blk["o_i_b"], residual=X[:, :Ti], colscale=mi[:, 2 * H:3 * H],
                   out=X[:, :Ti])
            if not last:
                K.gemm(att[:, Ti:], blk["o_c_w"], bias=blk["o_c_b"], residual=X[:, Ti:],
                       colscale=mc[:, 2 * H:3 * H], out=X[:, Ti:])
                Y = K.layer_norm_joint(X, H, T, Ti, mi[:, 3 * H:4 * H], mi[:, 4 * H:5 * H],
                                       mc[:, 3 * H:4 * H], mc[:, 4 * H:5 * H], ldm)
            else:
                Y = K.layer_norm_joint(X, H, T, Ti, mi[:, 3 * H:4 * H], mi[:, 4 * H:5 * H],
                                       mi[:, 3 * H:4 * H], mi[:, 4 * H:5 * H], ldm)
            K.gemm(Y[:, :Ti], blk["m1_i_w"], bias=blk["m1_i_b"], act=K.ACT_GELU, out=hid_i)
            K.gemm(hid_i, blk["m2_i_w"], bias=blk["m2_i_b"], residual=X[:, :Ti], colscale=mi[:, 5 * H:6 * H],
                   out=X[:, :Ti])
            if not last:
                K.gemm(Y[:, Ti:], blk["m1_c_w"], bias=blk["m1_c_b"], act=K.ACT_GELU, out=hid_c)
                K.gemm(hid_c, blk["m2_c_w"], bias=blk["m2_c_b"], residual=X[:, Ti:], colscale=mc[:, 5 * H:6 * H],
                       out=X[:, Ti:])
        return {"X": X, "hw": (Hl, Wl)}

    def forward(self, x: torch.Tensor, t: torch.Tensor, key="default") -> torch.Tensor:
        return self.run_units({"x": x}, t, key, 0, len(self.units))["eps"]


def mmdit_units(spec: MMDiTSpec) -> list:
    """(unit, FLOPs for one image) in forward order; sums to ``mmdit_flops(spec, 1)``."""
    s = spec
    H = s.hidden
    Ti = (s.latent_hw // s.patch) ** 2
    T = Ti + s.ctx_len
    out = [(("embed",), 2.0 * Ti * (s.patch ** 2 * s.in_channels) * H)]
    for d in range(s.depth):
        rows_out = Ti if d == s.depth - 1 else T
        f = 2.0 * T * H * 3 * H + 4.0 * T * T * H + 2.0 * rows_out * H * H + 2 * 2.0 * rows_out * H * s.mlp_ratio * H
        out.append((("block", d), f))
    out.append((("out",), 2.0 * Ti * H * s.patch ** 2 * s.in_channels))
    return out


def build_mmdit(spec: MMDiTSpec, seed: int = 0, device="cuda", weights: dict | None = None) -> MMDiT:
    if weights is None:
        from .weights import init_weights
        weights = init_weights(mmdit_param_specs(spec), seed=seed, device=device)
    return MMDiT(spec, weights, device=device)


def mmdit_flops(spec: MMDiTSpec, n: int) -> float:
    s = spec
    H = s.hidden
    Ti = (s.latent_hw // s.patch) ** 2
    L = s.ctx_len
    T = Ti + L
    f = 2.0 * n * Ti * (s.patch ** 2 * s.in_channels) * H            # patch embed
    for d in range(s.depth):
        last = d == s.depth - 1
        f += 2.0 * n * T * H * 3 * H                                 # qkv both streams
        f += 4.0 * n * T * T * H                                     # joint attention
        rows_out = Ti if last else T
        f += 2.0 * n * rows_out * H * H                              # output projections
        f += 2 * 2.0 * n * rows_out * H * s.mlp_ratio * H            # MLP
    f += 2.0 * n * Ti * H * s.patch ** 2 * s.in_channels             # proj_out
    return f
