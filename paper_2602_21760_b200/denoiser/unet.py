"""SDXL-shaped U-Net on the package's sm_100a kernels (the denoiser seam).

Activations are bf16 NHWC (pixels x channels, row-major), weights bf16 in the
kernels' layouts, accumulation fp32 in TMEM. Every op is one of our kernels:

  ResBlock      GN+SiLU -> conv3x3 (implicit GEMM; epilogue: bias + per-image
                time-embedding bias) -> GN+SiLU -> conv3x3 (epilogue: bias +
                residual = identity or 1x1-conv shortcut)
  GroupNorm     statistics come from the producing GEMM's epilogue (per 128-row
                block and 10-channel segment partials, ``gemm(gn_hw=)``), so a
                GroupNorm is one normalise pass (``hp_group_norm_parts``); tensors
                without partials (stage boundaries) take the two-pass path
  Transformer   GN -> proj_in GEMM -> [LN -> fused QKV GEMM -> attention ->
                out GEMM(+residual) -> LN -> Q GEMM -> cross-attention over
                per-run cached K/V -> out GEMM(+residual) -> LN -> GEGLU GEMM
                (gate fused in the epilogue) -> GEMM(+residual)] -> proj_out
                GEMM(+residual)
  Down / Up     stride-2 conv3x3 via TMA element strides / nearest 2x + conv3x3

Step-invariant work (text-time embedding, cross-attention K/V of the fixed
prompt context) is computed once per run in ``prepare``; ``forward`` is pure
kernel launches on fixed buffers, so it is captured in a CUDA graph.
Batch-invariant by construction (per-row GEMM tiles, per-image norms,
per-(image, head) attention): image b's output never depends on the other
rows of the batch, which makes serial (batched CFG), condition-partitioned
and empty-window hybrid runs bit-identical.
"""
from __future__ import annotations

import math

import torch

from . import kernels as K
from .weights import UNetSpec, unet_param_specs, unet_skip_channels


def _bf(t):
    return t.to(torch.bfloat16).contiguous()


def _f32(t):
    return t.to(torch.float32).contiguous()


class _Lin:
    def __init__(self, W, name, bias=True, dev="cuda"):
        self.w = _bf(W[name + ".weight"].to(dev))
        self.b = _f32(W[name + ".bias"].to(dev)) if bias and (name + ".bias") in W else None

    def __call__(self, x, **kw):
        return K.gemm(x, self.w, bias=self.b, **kw)


class _Conv:
    def __init__(self, W, name, dev="cuda"):
        w = W[name + ".weight"].to(dev)
        co, ci, kh, kw = w.shape
        self.co, self.ci, self.k = co, ci, kh
        self.w = _bf(w.permute(0, 2, 3, 1).reshape(co, kh * kw * ci))
        self.b = _f32(W[name + ".bias"].to(dev))

    def __call__(self, x, n, h, w, stride=1, **kw):
        if self.k == 1:
            return K.gemm(x, self.w, bias=self.b, **kw)
        return K.gemm(x, self.w, bias=self.b, conv=(n, h, w, self.ci, stride), **kw)


class _UpConv(_Conv):
    """Upsampler: nearest 2x then 3x3 conv, as one sub-pixel launch (HP_A_UPCONV:
    16 instead of 36 taps of MMA work per output pixel; no upsampled tensor)."""

    def __init__(self, W, name, dev="cuda"):
        super().__init__(W, name, dev)
        self.w4 = K.upconv_weights(W[name + ".weight"].to(dev).permute(0, 2, 3, 1))

    def up(self, x, n, h, w):
        """x: [n*h*w, ci] low-res -> [n*2h*2w, co]"""
        if n * h * w > 128:                    # CTA-pair kernel (M > 128 rows)
            return K.upsample_conv(x, n, h, w, self.ci, self.w4, self.b, gn=True)
        return self(K.upsample2x(x, n, h, w, self.ci), n, 2 * h, 2 * w)


class _Norm:
    def __init__(self, W, name, dev="cuda"):
        self.g = _f32(W[name + ".weight"].to(dev))
        self.b = _f32(W[name + ".bias"].to(dev))


class _ResBlock:
    def __init__(self, W, name, temb_dim, dev):
        self.n1, self.n2 = _Norm(W, name + ".norm1", dev), _Norm(W, name + ".norm2", dev)
        self.c1, self.c2 = _Conv(W, name + ".conv1", dev), _Conv(W, name + ".conv2", dev)
        self.tproj = _Lin(W, name + ".time_emb_proj", dev=dev)
        self.short = _Conv(W, name + ".conv_shortcut", dev) if (name + ".conv_shortcut.weight") in W else None

    def __call__(self, x, n, h, w, tb, groups, stats):
        """tb: this block's time-embedding bias [n, co] (a column slice of the
        UNet's single batched projection of SiLU(temb))."""
        ci, co = self.c1.ci, self.c1.co
        hw = h * w
        y = K.group_norm(x, n, hw, ci, self.n1.g, self.n1.b, groups=groups, silu=True, stats=stats)
        y = self.c1(y, n, h, w, bias2=tb, bias2_div=hw, gn_hw=hw)
        y = K.group_norm(y, n, hw, co, self.n2.g, self.n2.b, groups=groups, silu=True, stats=stats)
        res = self.short(x, n, h, w) if self.short is not None else x
        return self.c2(y, n, h, w, residual=res, gn_hw=hw)


class _Block:
    def __init__(self, W, name, c, heads, dev):
        self.c, self.heads = c, heads
        self.n1, self.n2, self.n3 = (_Norm(W, f"{name}.norm{i}", dev) for i in (1, 2, 3))
        # each LayerNorm feeds exactly one GEMM: fold gamma/beta into that GEMM's
        # weights/bias; the producing GEMM's epilogue records the row statistics
        a1 = f"{name}.attn1"
        qkv = torch.cat([W[f"{a1}.to_q.weight"], W[f"{a1}.to_k.weight"], W[f"{a1}.to_v.weight"]]).to(dev)
        self.f1 = K.FoldedLN(qkv, self.n1.g, self.n1.b, eps=1e-5)
        self.o1 = _Lin(W, f"{a1}.to_out.0", dev=dev)
        a2 = f"{name}.attn2"
        self.f2 = K.FoldedLN(W[f"{a2}.to_q.weight"].to(dev), self.n2.g, self.n2.b, eps=1e-5)
        self.kv2 = _bf(torch.cat([W[f"{a2}.to_k.weight"], W[f"{a2}.to_v.weight"]]).to(dev))
        self.o2 = _Lin(W, f"{a2}.to_out.0", dev=dev)
        # GEGLU: interleave hidden/gate rows per 256-wide output tile (128 + 128)
        pw, pb = W[f"{name}.ff.net.0.proj.weight"].to(dev), W[f"{name}.ff.net.0.proj.bias"].to(dev)
        F_ = pw.shape[0] // 2
        half = 128
        idx = torch.cat([torch.cat([torch.arange(i, i + half), torch.arange(F_ + i, F_ + i + half)])
                         for i in range(0, F_, half)]).to(dev)
        self.f3 = K.FoldedLN(pw[idx], self.n3.g, self.n3.b, bias=pb[idx], eps=1e-5)
        self.ff2 = _Lin(W, f"{name}.ff.net.2", dev=dev)
        self.kv_cache = {}

    def prepare(self, ctx2d, key):
        self.kv_cache[key] = K.gemm(ctx2d, self.kv2)        # [rows*L, 2C]

    def __call__(self, h, n, S, ctx_len, key, rs):
        """h: residual stream whose row statistics the producing GEMM left in rs."""
        c = self.c
        scale = 1.0 / math.sqrt(64)
        f1, f2, f3 = self.f1, self.f2, self.f3
        qkv = K.gemm(h, f1.w, bias=f1.bias, ln_fold=(rs, f1))                 # norm1 folded
        att = torch.empty_like(h)
        K.attention(qkv, qkv, qkv, att, batch=n, heads=self.heads, sq=S, skv=S, scale=scale,
                    q_col0=0, k_col0=c, v_col0=2 * c)
        h = self.o1(att, residual=h, out=h, stats_out=rs)
        q = K.gemm(h, f2.w, bias=f2.bias, ln_fold=(rs, f2))                   # norm2 folded
        kv = self.kv_cache[key]
        K.attention(q, kv, kv, att, batch=n, heads=self.heads, sq=S, skv=ctx_len, scale=scale,
                    q_col0=0, k_col0=0, v_col0=c)
        h = self.o2(att, residual=h, out=h, stats_out=rs)
        f = K.gemm(h, f3.w, bias=f3.bias, act=K.ACT_GEGLU, block_n=256, ln_fold=(rs, f3))   # norm3 folded
        return self.ff2(f, residual=h, out=h, stats_out=rs)


class _Transformer:
    def __init__(self, W, name, c, depth, head_dim, dev):
        self.c = c
        self.norm = _Norm(W, name + ".norm", dev)
        self.pin, self.pout = _Lin(W, name + ".proj_in", dev=dev), _Lin(W, name + ".proj_out", dev=dev)
        self.blocks = [_Block(W, f"{name}.transformer_blocks.{d}", c, c // head_dim, dev) for d in range(depth)]

    def prepare(self, ctx2d, key):
        for b in self.blocks:
            b.prepare(ctx2d, key)

    def __call__(self, x, n, hw, groups, stats, ctx_len, key, rs):
        y = K.group_norm(x, n, hw, self.c, self.norm.g, self.norm.b, groups=groups, eps=1e-6, stats=stats)
        h = self.pin(y, stats_out=rs)
        for b in self.blocks:
            h = b(h, n, hw, ctx_len, key, rs)
        return self.pout(h, residual=x, gn_hw=hw)


class UNet:
    """Random-init SDXL-shaped U-Net; ``forward`` maps bf16 NHWC latents to eps."""

    def __init__(self, spec: UNetSpec, W: dict, device="cuda"):
        self.spec = s = spec
        dev = torch.device(device)
        self.dev = dev
        ch = s.block_out
        # conv_in / conv_out on the tensor-core implicit-GEMM conv: the 4 latent
        # channels are zero-padded to 64 (conv_in's input, conv_out's output)
        wi = W["conv_in.weight"].to(dev)                                   # [320, 4, 3, 3]
        self.cin_pad = 64
        wpad = torch.zeros(wi.shape[0], 3, 3, self.cin_pad, device=dev)
        wpad[..., :wi.shape[1]] = wi.permute(0, 2, 3, 1)
        self.conv_in_w = _bf(wpad.reshape(wi.shape[0], 9 * self.cin_pad))
        self.conv_in_b = _f32(W["conv_in.bias"].to(dev))
        self.t1, self.t2 = _Lin(W, "time_embedding.linear_1", dev=dev), _Lin(W, "time_embedding.linear_2", dev=dev)
        self.a1, self.a2 = _Lin(W, "add_embedding.linear_1", dev=dev), _Lin(W, "add_embedding.linear_2", dev=dev)
        self.down = []
        for lvl, co in enumerate(ch):
            res = [_ResBlock(W, f"down_blocks.{lvl}.resnets.{j}", s.temb_dim, dev) for j in range(s.layers_per_block)]
            att = [(_Transformer(W, f"down_blocks.{lvl}.attentions.{j}", co, s.transformer_depth[lvl], s.head_dim, dev)
                    if s.transformer_depth[lvl] else None) for j in range(s.layers_per_block)]
            ds = _Conv(W, f"down_blocks.{lvl}.downsamplers.0.conv", dev) if lvl < len(ch) - 1 else None
            self.down.append((res, att, ds))
        self.mid = (_ResBlock(W, "mid_block.resnets.0", s.temb_dim, dev),
                    _Transformer(W, "mid_block.attentions.0", ch[-1], s.mid_depth, s.head_dim, dev),
                    _ResBlock(W, "mid_block.resnets.1", s.temb_dim, dev))
        self.up = []
        for u in range(len(ch)):
            lvl = len(ch) - 1 - u
            co = ch[lvl]
            res = [_ResBlock(W, f"up_blocks.{u}.resnets.{j}", s.temb_dim, dev) for j in range(s.layers_per_block + 1)]
            att = [(_Transformer(W, f"up_blocks.{u}.attentions.{j}", co, s.transformer_depth[lvl], s.head_dim, dev)
                    if s.transformer_depth[lvl] else None) for j in range(s.layers_per_block + 1)]
            us = _UpConv(W, f"up_blocks.{u}.upsamplers.0.conv", dev) if u < len(ch) - 1 else None
            self.up.append((res, att, us))
        self.norm_out = _Norm(W, "conv_norm_out", dev)
        wo = W["conv_out.weight"].to(dev)                                  # [4, 320, 3, 3]
        self.cout_pad = 64
        wpad = torch.zeros(self.cout_pad, 3, 3, wo.shape[1], device=dev)
        wpad[:wo.shape[0]] = wo.permute(0, 2, 3, 1)
        self.conv_out_w = _bf(wpad.reshape(self.cout_pad, 9 * wo.shape[1]))
        bpad = torch.zeros(self.cout_pad, device=dev)
        bpad[:wo.shape[0]] = W["conv_out.bias"].to(dev)
        self.conv_out_b = _f32(bpad)
        self.stats = torch.empty(2 * 64 * 64 * 32, dtype=torch.float32, device=dev)
        self.aug = {}
        self.ctx_len = s.context_len
        # every ResBlock's time_emb_proj(SiLU(temb)) as ONE small GEMV per forward
        blocks = [r for res, _, _ in self.down for r in res] + [self.mid[0], self.mid[2]] + \
                 [r for res, _, _ in self.up for r in res]
        offs, o = [], 0
        for r in blocks:
            offs.append(o)
            o += r.c1.co
        self.tproj_w = torch.cat([r.tproj.w for r in blocks]).contiguous()
        self.tproj_b = torch.cat([r.tproj.b for r in blocks]).contiguous()
        self.tproj_slot = {id(r): (off, r.c1.co) for r, off in zip(blocks, offs)}
        for r in blocks:
            r.tproj = None
        spec_units = unet_units(s)
        self.units = [u for u, _, _ in spec_units]
        self.unit_flops = [f for _, f, _ in spec_units]
        self._levels = [lv for _, _, lv in spec_units]

    def _row_stats(self, floats: int) -> "K.RowStats":
        rs = getattr(self, "_rs", None)
        if rs is None or rs.buf.numel() < floats:
            rs = self._rs = K.RowStats(floats, self.dev)
        return rs

    def _transformers(self):
        for res, att, _ in self.down + self.up:
            for a in att:
                if a is not None:
                    yield a
        yield self.mid[1]

    def prepare(self, context: torch.Tensor, pooled: torch.Tensor, key="default"):
        """Per-run, step-invariant work: text-time embedding and cross-attention K/V.

        context [n, L, cross_dim], pooled [n, pooled_dim] (fp32 or bf16), one row per
        image of the forward batch."""
        s = self.spec
        n = context.shape[0]
        ctx2d = _bf(context.to(self.dev).reshape(n * s.context_len, s.cross_dim))
        for t in self._transformers():
            t.prepare(ctx2d, key)
        # add_embedding(text_embeds ++ time_ids embedding); SDXL time ids for 1024^2
        size = 8.0 * s.latent_hw
        ids = torch.tensor([size, size, 0.0, 0.0, size, size], device=self.dev).repeat(n, 1)
        tid = K.timestep_embedding(ids.reshape(-1).contiguous(), s.time_id_dim).reshape(n, -1)
        add_in = torch.cat([_f32(pooled.to(self.dev)), tid], dim=1).contiguous()
        a = K.linear_small(add_in, self.a1.w, self.a1.b, act_out=K.ACT_SILU)
        self.aug[key] = K.linear_small(a, self.a2.w, self.a2.b)

    def _prologue(self, t: torch.Tensor, key: str) -> torch.Tensor:
        """Per-step embeddings: every ResBlock's time-embedding bias for timestep t
        (one batched GEMV over all blocks) -> [n, sum(co)] fp32."""
        s = self.spec
        te = K.timestep_embedding(t, s.block_out[0])
        te = K.linear_small(te, self.t1.w, self.t1.b, act_out=K.ACT_SILU)
        temb = K.linear_small(te, self.t2.w, self.t2.b)
        temb = temb + self.aug[key]                    # tiny [n, 1280] add
        return K.linear_small(temb, self.tproj_w, self.tproj_b, act_in=K.ACT_SILU)

    def run_units(self, state: dict, t: torch.Tensor, key: str, a: int, b: int, record=None) -> dict:
        """Execute units [a, b) of the forward (``unet_units`` order) on a boundary
        state and return the boundary state after unit b-1.

        A boundary state is ``{"x": latent}`` before unit 0, ``{"eps": eps}``
        after the last unit, else ``{"h": activation [n*hh*ww, c], "skips":
        [pushed, not yet popped skip tensors], "hw": (hh, ww), "n": n}``. The
        per-step time embedding is recomputed from t (stage-split pipelining runs
        every stage at the current step's t, SPEC.md:390 / PAPER.md:45).

        ``record``: {unit index: None} filled with the boundary state entering
        each listed unit (tensor references: no unit writes a tensor it did
        not create, so they stay valid until the next forward)."""
        s = self.spec
        st, g = self.stats, s.groups
        units = self.units
        if a == 0:
            x = state["x"]
            n, H, Wd = x.shape[0], x.shape[1], x.shape[2]
            h, skips, (hh, ww) = None, [], (H, Wd)
        else:
            n, h, skips, (hh, ww) = state["n"], state["h"], list(state["skips"]), state["hw"]
            # a stage entry: boundary tensors arrive without their producers' GroupNorm
            # partials when they crossed GPUs, so drop them here too (fresh views) and the
            # GroupNorms at every stage entry take the same two-pass path in-process or not
            h = h.view(h.shape)
            skips = [t.view(t.shape) for t in skips]
        full_hw = hh * (2 ** self._levels[a]) if a else hh       # latent side length
        rs = self._row_stats(2 * n * full_hw * full_hw * max(c // 4 ** l for l, c in enumerate(s.block_out)) // 64)
        tb_all = self._prologue(t, key) if any(u[0] in ("res",) for u in units[a:b]) else None

        def tb(r):
            off, co = self.tproj_slot[id(r)]
            return tb_all[:, off:off + co]             # row stride sum(co): GEMM bias2_ld
        for i in range(a, b):
            u = units[i]
            kind = u[0]
            if record is not None and i in record:
                record[i] = {"h": h, "skips": list(skips), "hw": (hh, ww), "n": n}
            if kind == "conv_in":
                xp = K.copy_cols(x.view(n * hh * ww, s.in_channels), self.cin_pad)
                h = K.gemm(xp, self.conv_in_w, bias=self.conv_in_b, conv=(n, hh, ww, self.cin_pad, 1),
                           gn_hw=hh * ww)
                skips.append(h)
            elif kind == "res":
                _, where, lvl, j, push = u
                r = self._res_of(where, lvl, j)
                if where == "up":
                    sk = skips.pop()
                    h = K.concat_channels(h, h.shape[1], sk, sk.shape[1], n * hh * ww)
                h = r(h, n, hh, ww, tb(r), g, st)
                if push:
                    skips.append(h)
            elif kind == "attn":
                _, where, lvl, j, push = u
                h = self._attn_of(where, lvl, j)(h, n, hh * ww, g, st, self.ctx_len, key, rs)
                if push:
                    skips.append(h)
            elif kind == "ds":
                h = self.down[u[1]][2](h, n, hh, ww, stride=2, gn_hw=(hh // 2) * (ww // 2))
                hh, ww = hh // 2, ww // 2
                skips.append(h)
            elif kind == "us":
                h = self.up[u[1]][2].up(h, n, hh, ww)
                hh, ww = hh * 2, ww * 2
            elif kind == "out":
                y = K.group_norm(h, n, hh * ww, s.block_out[0], self.norm_out.g, self.norm_out.b, groups=g,
                                 silu=True, stats=st)
                e64 = K.gemm(y, self.conv_out_w, bias=self.conv_out_b, conv=(n, hh, ww, s.block_out[0], 1))
                eps = K.copy_cols(e64, s.out_channels)
                return {"eps": eps.view(n, hh, ww, s.out_channels)}
        return {"h": h, "skips": skips, "hw": (hh, ww), "n": n}

    def _res_of(self, where, lvl, j):
        if where == "mid":
            return self.mid[0] if j == 0 else self.mid[2]
        return (self.down if where == "down" else self.up)[lvl][0][j]

    def _attn_of(self, where, lvl, j):
        if where == "mid":
            return self.mid[1]
        return (self.down if where == "down" else self.up)[lvl][1][j]

    def forward(self, x: torch.Tensor, t: torch.Tensor, key="default") -> torch.Tensor:
        """x: [n, H, W, in_ch] bf16 NHWC; t: [n] fp32 timesteps -> eps [n, H, W, out_ch] bf16."""
        return self.run_units({"x": x}, t, key, 0, len(self.units))["eps"]


def unet_units(spec: UNetSpec) -> list:
    """The U-Net forward as a list of units, the granularity at which it can be
    cut into pipeline stages, with each unit's FLOPs for ONE image (same
    counting as ``unet_flops``) and the resolution level of its input.

    Units: ("conv_in",), ("res", where, lvl, j, push), ("attn", where, lvl, j,
    push), ("ds", lvl), ("us", u), ("out",); ``push`` = the unit ends a
    (res[, attn]) group whose output is pushed as a skip."""
    s = spec
    ch = s.block_out
    H = s.latent_hw
    L = s.context_len
    out = []

    def conv(hw, ci, co, k=3):
        return 2.0 * hw * ci * co * k * k

    def res(hw, ci, co):
        f = conv(hw, ci, co) + conv(hw, co, co)
        if ci != co:
            f += conv(hw, ci, co, 1)
        return f

    def tr(hw, c, depth):
        f = 2 * 2.0 * hw * c * c
        per = (2.0 * hw * c * 3 * c + 2.0 * hw * c * c + 4.0 * hw * hw * c + 2.0 * hw * c * c * 2
               + 4.0 * hw * L * c + 2.0 * hw * c * 8 * c + 2.0 * hw * 4 * c * c)
        return f + depth * per

    out.append((("conv_in",), 2.0 * H * H * s.in_channels * ch[0] * 9, 0))
    hw, lv, prev = H * H, 0, ch[0]
    for lvl, co in enumerate(ch):
        d = s.transformer_depth[lvl]
        for j in range(s.layers_per_block):
            out.append((("res", "down", lvl, j, not d), res(hw, prev if j == 0 else co, co), lv))
            if d:
                out.append((("attn", "down", lvl, j, True), tr(hw, co, d), lv))
        prev = co
        if lvl < len(ch) - 1:
            out.append((("ds", lvl), conv(hw // 4, co, co), lv))
            hw //= 4
            lv += 1
    out.append((("res", "mid", 0, 0, False), res(hw, ch[-1], ch[-1]), lv))
    out.append((("attn", "mid", 0, 0, False), tr(hw, ch[-1], s.mid_depth), lv))
    out.append((("res", "mid", 0, 1, False), res(hw, ch[-1], ch[-1]), lv))
    skips = unet_skip_channels(s)
    prev = ch[-1]
    for u in range(len(ch)):
        lvl = len(ch) - 1 - u
        co = ch[lvl]
        d = s.transformer_depth[lvl]
        for j in range(s.layers_per_block + 1):
            out.append((("res", "up", u, j, False), res(hw, prev + skips.pop(), co), lv))
            prev = co
            if d:
                out.append((("attn", "up", u, j, False), tr(hw, co, d), lv))
        if u < len(ch) - 1:
            out.append((("us", u), conv(hw * 4, co, co) * 4 / 9, lv))
            hw *= 4
            lv -= 1
    out.append((("out",), 2.0 * H * H * ch[0] * s.out_channels * 9, 0))
    return out


def build_unet(spec: UNetSpec, seed: int = 0, device="cuda", weights: dict | None = None) -> UNet:
    if weights is None:
        from .weights import init_weights
        weights = init_weights(unet_param_specs(spec), seed=seed, device=device)
    return UNet(spec, weights, device=device)


def unet_flops(spec: UNetSpec, n: int) -> float:
    """Analytic forward FLOPs (2*MACs of every GEMM/conv + 4*S*S*C attention) for n images."""
    s = spec
    ch = s.block_out
    H = s.latent_hw
    fl = 0.0
    L = s.context_len

    def conv(hw, ci, co, k=3):
        return 2.0 * n * hw * ci * co * k * k

    def res(hw, ci, co):
        f = conv(hw, ci, co) + conv(hw, co, co)
        if ci != co:
            f += conv(hw, ci, co, 1)
        return f

    def tr(hw, c, depth):
        f = 2 * 2.0 * n * hw * c * c                        # proj in/out
        per = (2.0 * n * hw * c * 3 * c + 2.0 * n * hw * c * c      # qkv + out
               + 4.0 * n * hw * hw * c                              # self attention
               + 2.0 * n * hw * c * c * 2                           # q2 + out2
               + 4.0 * n * hw * L * c                               # cross attention
               + 2.0 * n * hw * c * 8 * c + 2.0 * n * hw * 4 * c * c)  # GEGLU + ff2
        return f + depth * per

    fl += 2.0 * n * H * H * s.in_channels * ch[0] * 9
    hw = H * H
    prev = ch[0]
    for lvl, co in enumerate(ch):
        for j in range(s.layers_per_block):
            fl += res(hw, prev if j == 0 else co, co)
            if s.transformer_depth[lvl]:
                fl += tr(hw, co, s.transformer_depth[lvl])
        prev = co
        if lvl < len(ch) - 1:
            fl += conv(hw // 4, co, co)
            hw //= 4
    fl += 2 * res(hw, ch[-1], ch[-1]) + tr(hw, ch[-1], s.mid_depth)
    skips = unet_skip_channels(s)
    prev = ch[-1]
    for u in range(len(ch)):
        lvl = len(ch) - 1 - u
        co = ch[lvl]
        for j in range(s.layers_per_block + 1):
            fl += res(hw, prev + skips.pop(), co)
            prev = co
            if s.transformer_depth[lvl]:
                fl += tr(hw, co, s.transformer_depth[lvl])
        if u < len(ch) - 1:
            hw *= 4
            fl += conv(hw, co, co) * 4 / 9        # upsampler: sub-pixel, 4 of the 9 taps (HP_A_UPCONV)
    fl += 2.0 * n * H * H * ch[0] * s.out_channels * 9
    return fl
