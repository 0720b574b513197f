"""ctypes bindings of the denoiser kernels (include/hybridpar_b200_denoiser.h).

Thin torch-tensor wrappers: shapes/dtypes are checked here, pointers and the
current stream cross the C ABI, results are written into caller-provided or
freshly allocated bf16 tensors (the caching allocator makes the latter free
inside captured CUDA graphs). No computation happens in Python.
"""
from __future__ import annotations

import ctypes as C

import torch

from .. import _native as N
from ..errors import ShapeError
from ..errors import check as _check

# number of our kernel launches issued through these wrappers (the engine and
# bench read it around graph capture to report launches per forward)
LAUNCHES = 0
# wrappers whose C entry issues more than one kernel (hp_group_norm is one launch on its
# single-launch path, which every denoiser shape takes; two only for batches too large
# for all statistics CTAs to be resident)
_KERNELS_PER_CALL: dict = {}


def check(rc, what):
    global LAUNCHES
    LAUNCHES += _KERNELS_PER_CALL.get(what.split()[0], 1)
    _check(rc, what)

_VP, _I32, _I64, _F32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float

HP_A_PLAIN, HP_A_CONV3X3, HP_A_CONV3X3_S2, HP_A_UPCONV = 0, 1, 2, 3
ACT_NONE, ACT_GELU, ACT_SILU, ACT_GEGLU = 0, 1, 2, 3


class HpGemmDesc(C.Structure):
    _fields_ = [
        ("a", _VP), ("lda", _I64), ("a_mode", _I32),
        ("img_n", _I32), ("img_h", _I32), ("img_w", _I32), ("img_c", _I32),
        ("b", _VP), ("ldb", _I64),
        ("d", _VP), ("ldd", _I64),
        ("M", _I64), ("N", _I64), ("K", _I64),
        ("bias", _VP),
        ("bias2", _VP), ("bias2_div", _I64),
        ("residual", _VP), ("ldr", _I64),
        ("act", _I32), ("block_n", _I32), ("alpha", _F32),
        ("colscale", _VP),
        ("batch", _I32),
        ("a_bstride", _I64), ("d_bstride", _I64), ("r_bstride", _I64), ("cs_bstride", _I64),
        ("bias2_ld", _I64),
        ("ln_gamma", _VP), ("ln_beta", _VP), ("ln_eps", _F32), ("ln_y", _VP), ("ldy", _I64),
        ("stats_out", _VP),
        ("ln_stats", _VP), ("ln_parts", _I32), ("ln_part_n", _I32), ("ln_colsum", _VP), ("ln_fold_eps", _F32),
        ("gn_part", _VP), ("gn_rows", _I64), ("gn_parts", _I32),
    ]


class HpAttnDesc(C.Structure):
    _fields_ = [
        ("q", _VP), ("ldq", _I64), ("q_col0", _I64),
        ("k", _VP), ("ldk", _I64), ("k_col0", _I64),
        ("v", _VP), ("ldv", _I64), ("v_col0", _I64),
        ("o", _VP), ("ldo", _I64),
        ("batch", _I32), ("heads", _I32), ("sq", _I32), ("skv", _I32),
        ("scale", _F32), ("causal", _I32),
    ]


SIGNATURES = {
    "hp_gemm": (C.c_int, [C.POINTER(HpGemmDesc), _VP]),
    "hp_gemm_pick_block_n": (_I32, [_I64, _I64, _I64, _I32]),
    "hp_gemm_stats_block_n": (_I32, [_I64, _I64, _I64]),
    "hp_attention": (C.c_int, [C.POINTER(HpAttnDesc), _VP]),
    "hp_group_norm": (C.c_int, [_VP, _I32, _VP, _I32, _I32, _I64, _I32, _F32, _VP, _VP, _I32, _VP, _VP, _VP]),
    "hp_group_norm_parts": (C.c_int, [_VP, _I32, _I32, _I64, _VP, _I32, _VP, _I32, _F32, _VP, _VP, _I32, _VP, _VP]),
    "hp_layer_norm": (C.c_int, [_VP, _I64, _I32, _F32, _VP, _VP, _VP, _VP, _I64, _I64, _VP, _VP]),
    "hp_layer_norm_joint": (C.c_int, [_VP, _I64, _I32, _F32, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _VP, _VP]),
    "hp_silu": (C.c_int, [_VP, _VP, _I64, _VP]),
    "hp_upsample2x": (C.c_int, [_VP, _I32, _I32, _I32, _I32, _VP, _VP]),
    "hp_concat_channels": (C.c_int, [_VP, _I32, _VP, _I32, _I64, _VP, _VP]),
    "hp_copy_cols": (C.c_int, [_VP, _I64, _I32, _I64, _VP, _I64, _I32, _VP]),
    "hp_softmax_rows": (C.c_int, [_VP, _I64, _I64, _I32, _F32, _VP, _I64, _VP]),
    "hp_embed_tokens": (C.c_int, [_VP, _I64, _I32, _VP, _VP, _I32, _VP, _VP]),
    "hp_quick_gelu": (C.c_int, [_VP, _VP, _I64, _VP]),
    "hp_conv3x3_small": (C.c_int, [_VP, _I32, _I32, _I32, _I32, _VP, _VP, _I32, _VP, _I32, _VP]),
    "hp_timestep_embedding": (C.c_int, [_VP, _I32, _I32, _F32, _VP, _VP]),
    "hp_linear_small": (C.c_int, [_VP, _I32, _I32, _VP, _VP, _I32, _I32, _I32, _VP, _VP]),
    "hp_patchify": (C.c_int, [_VP, _I32, _I32, _I32, _I32, _I32, _I32, _VP, _VP]),
    "hp_add_rows": (C.c_int, [_VP, _VP, _I64, _I64, _I32, _VP, _VP]),
    "hp_gated_residual": (C.c_int, [_VP, _VP, _VP, _I64, _I64, _I32, _I64, _VP]),
    "hp_cast_bf16_f32": (C.c_int, [_VP, _VP, _I64, _VP]),
}
N.register_signatures(SIGNATURES)


def _p(t):
    return None if t is None else t.data_ptr()


def _s():
    return C.c_void_p(N.stream_ptr())


def _bf16(t, name):
    if t.dtype != torch.bfloat16 or not t.is_cuda:
        raise ShapeError(f"{name} must be a bf16 CUDA tensor, got {t.dtype} on {t.device}")


class RowStats:
    """Per-(row, N tile) (mean, M2) of a GEMM's stored output (``gemm(stats_out=)``),
    consumed by the next GEMM's folded LayerNorm (``gemm(ln_fold=)``)."""

    def __init__(self, capacity_floats: int, device):
        self.buf = torch.empty(capacity_floats, dtype=torch.float32, device=device)
        self.parts = 0
        self.part_n = 0


class FoldedLN:
    """LayerNorm(gamma, beta) folded into the weights of the GEMM it feeds:
    W' = bf16(W * gamma), colsum = sum_k W', bias' = bias + W beta (all on the
    host once). ``gemm(x, fold.w, bias=fold.bias, ln_fold=(stats, fold))``
    equals ``gemm(layer_norm(x), W, bias=bias)`` up to bf16 rounding."""

    def __init__(self, w, gamma, beta, bias=None, eps=1e-5):
        wf = w.float()
        self.w = (wf * gamma.float()[None, :]).to(torch.bfloat16).contiguous()
        self.colsum = self.w.float().sum(1).contiguous()
        b = wf @ beta.float()
        self.bias = (b if bias is None else b + bias.float()).contiguous()
        self.eps = float(eps)


GN_SEG, GN_ROWS = 10, 128      # GroupNorm partial: 10 columns x 128 rows (hp_gemm gn_part)


class GnParts:
    """GroupNorm partials a GEMM left for its output (``gemm(gn_hw=...)``): (sum, sum of
    squares) per 128-row block and 10-column segment; ``group_norm`` folds them instead
    of re-reading the tensor for statistics. ``parts2`` / ``c1``: a channel concat whose
    second input carries its own partials."""

    def __init__(self, buf, hw, c, parts2=None, c1=None):
        self.buf, self.hw, self.c = buf, hw, c
        self.parts2, self.c1 = parts2, c if c1 is None else c1


def gn_parts_ok(M, N, hw):
    """Shapes whose producing GEMM can record GroupNorm partials."""
    return N % 160 == 0 and hw % GN_ROWS == 0 and M % hw == 0 and M > GN_ROWS


def _gn_buf(M, N, dev):
    return torch.empty((M // GN_ROWS) * (N // GN_SEG) * 2, dtype=torch.float32, device=dev)


def gemm(a, w, *, out=None, bias=None, bias2=None, bias2_div=1, residual=None, act=ACT_NONE,
         alpha=1.0, block_n=0, conv=None, colscale=None, ln=None, stats_out=None, ln_fold=None, gn_hw=None):
    """out[M, N'] = residual + colscale * act(alpha * A @ W^T + bias).
    ``conv=(n, h, w, c, stride)`` reads A as NHWC. ``stats_out`` (RowStats):
    also record the output rows' LayerNorm partials; ``ln_fold=(RowStats,
    FoldedLN)``: A is un-normalised, LN applied in the epilogue (w, bias must
    be the FoldedLN's). ``gn_hw``: rows per image; also record GroupNorm
    partials of the output (``out.hp_gn``, a GnParts) when the shape allows."""
    lib = N.load()
    _bf16(a, "A")
    _bf16(w, "W")
    Nn, K = w.shape
    d = HpGemmDesc()
    d.a = _p(a)
    if conv is None and a.dim() == 3:
        # batched: a [batch, M, K] (any batch stride), out [batch, M, N'], residual
        # [batch, M, N'] or [M, N'] (shared), colscale [batch, N] or [N] (shared)
        nb, M, _ = a.shape
        if a.shape[2] != K:
            raise ShapeError(f"gemm K mismatch: A {tuple(a.shape)} vs W {tuple(w.shape)}")
        n_out = Nn // 2 if act == ACT_GEGLU else Nn
        if out is None:
            out = torch.empty((nb, M, n_out), dtype=torch.bfloat16, device=a.device)
        d.lda, d.a_mode, d.batch, d.a_bstride = a.stride(1), HP_A_PLAIN, nb, a.stride(0)
        d.b, d.ldb = _p(w), w.stride(0)
        d.d, d.ldd, d.d_bstride = _p(out), out.stride(1), out.stride(0)
        d.M, d.N, d.K = M, Nn, K
        d.bias = _p(bias)
        d.bias2, d.bias2_div = _p(bias2), 1
        d.residual = _p(residual)
        if residual is not None:
            d.ldr = residual.stride(-2)
            d.r_bstride = residual.stride(0) if residual.dim() == 3 else 0
        d.act, d.block_n, d.alpha = int(act), int(block_n), float(alpha)
        d.colscale = _p(colscale)
        if colscale is not None:
            d.cs_bstride = colscale.stride(0) if colscale.dim() == 2 else 0
        check(lib.hp_gemm(C.byref(d), _s()), f"hp_gemm batched {nb}x M={M} N={Nn} K={K}")
        return out
    if conv is None:
        M = a.numel() // a.shape[-1]
        if a.shape[-1] != K:
            raise ShapeError(f"gemm K mismatch: A {tuple(a.shape)} vs W {tuple(w.shape)}")
        d.lda = a.stride(-2) if a.dim() >= 2 else K
        d.a_mode = HP_A_PLAIN
    else:
        n, h, wd, c, stride = conv
        if K != 9 * c:
            raise ShapeError(f"conv weight K={K} != 9*{c}")
        M = n * (h // stride) * (wd // stride)
        d.lda = c
        d.a_mode = HP_A_CONV3X3 if stride == 1 else HP_A_CONV3X3_S2
        d.img_n, d.img_h, d.img_w, d.img_c = n, h, wd, c
    n_out = Nn // 2 if act == ACT_GEGLU else Nn
    if out is None:
        out = torch.empty((M, n_out), dtype=torch.bfloat16, device=a.device)
    d.b, d.ldb = _p(w), w.stride(0)
    d.d, d.ldd = _p(out), out.stride(-2) if out.dim() >= 2 else n_out
    d.M, d.N, d.K = M, Nn, K
    d.bias = _p(bias)
    d.bias2, d.bias2_div = _p(bias2), int(bias2_div)
    d.bias2_ld = bias2.stride(0) if (bias2 is not None and bias2.dim() == 2) else 0
    d.residual = _p(residual)
    d.ldr = residual.stride(-2) if residual is not None else 0
    d.act, d.block_n, d.alpha = int(act), int(block_n), float(alpha)
    d.colscale = _p(colscale)
    if ln is not None:
        # ln = (gamma, beta, eps, y_out): also write y_out = LayerNorm(out) (fused epilogue)
        g, b_, eps, y = ln
        d.ln_gamma, d.ln_beta, d.ln_eps, d.ln_y, d.ldy = _p(g), _p(b_), float(eps), _p(y), y.stride(-2)
    if stats_out is not None:
        # the statistics layout must not depend on M (batch invariance of the folded LayerNorm)
        bn = int(block_n) or int(lib.hp_gemm_stats_block_n(M, Nn, K))
        seg = bn // 2 if bn > 256 else bn            # statistics segment width (hp_gemm.cu StatW)
        if bn == 0 or Nn % bn or stats_out.buf.numel() < 2 * M * (Nn // seg):
            raise ShapeError(f"row stats: N={Nn} block_n={bn} capacity {stats_out.buf.numel()}")
        d.block_n = bn
        d.stats_out = _p(stats_out.buf)
        stats_out.parts, stats_out.part_n = Nn // seg, seg
    if ln_fold is not None:
        st, fold = ln_fold
        d.ln_stats, d.ln_parts, d.ln_part_n = _p(st.buf), st.parts, st.part_n
        d.ln_colsum, d.ln_fold_eps = _p(fold.colsum), fold.eps
    gp = None
    if gn_hw is not None and act == ACT_NONE and gn_parts_ok(M, Nn, gn_hw):
        gp = GnParts(_gn_buf(M, Nn, a.device), gn_hw, Nn)
        d.gn_part, d.gn_rows, d.gn_parts = _p(gp.buf), gn_hw, gn_hw // GN_ROWS
    check(lib.hp_gemm(C.byref(d), _s()), f"hp_gemm M={M} N={Nn} K={K}")
    if gp is not None:
        out.hp_gn = gp
    elif getattr(out, "hp_gn", None) is not None:
        del out.hp_gn                                # overwritten in place: its partials are stale
    return out


def attention(q, k, v, out, *, batch, heads, sq, skv, scale, q_col0=0, k_col0=0, v_col0=0, causal=False):
    """Multi-head attention, head_dim 64; q/k/v/out are 2-D [batch*rows, ld] views."""
    lib = N.load()
    d = HpAttnDesc()
    d.q, d.ldq, d.q_col0 = _p(q), q.stride(0), q_col0
    d.k, d.ldk, d.k_col0 = _p(k), k.stride(0), k_col0
    d.v, d.ldv, d.v_col0 = _p(v), v.stride(0), v_col0
    d.o, d.ldo = _p(out), out.stride(0)
    d.batch, d.heads, d.sq, d.skv, d.scale = batch, heads, sq, skv, float(scale)
    d.causal = 1 if causal else 0
    check(lib.hp_attention(C.byref(d), _s()), f"hp_attention B={batch} H={heads} Sq={sq} Skv={skv}")
    return out


def group_norm(x, n, hw, c, gamma, beta, *, groups=32, eps=1e-5, silu=False, x2=None, c2=0, out=None,
               stats=None):
    """GroupNorm(+SiLU) over NHWC rows. When x carries its producer's GroupNorm partials
    (``x.hp_gn``) for this very shape, one launch folds them (no statistics pass);
    otherwise the statistics are computed here (hp_group_norm)."""
    lib = N.load()
    C_ = c + (c2 if x2 is not None else 0)
    if out is None:
        out = torch.empty((n * hw, C_), dtype=torch.bfloat16, device=x.device)
    gp = getattr(x, "hp_gn", None)
    if (gp is not None and x2 is None and gp.hw == hw and gp.c == c and x.shape[0] == n * hw
            and (c // groups) % GN_SEG == 0 and x.is_contiguous()):
        check(lib.hp_group_norm_parts(_p(x), c, n, hw, _p(gp.buf), gp.c1,
                                      _p(gp.parts2.buf) if gp.parts2 is not None else None, groups, eps,
                                      _p(gamma), _p(beta), int(silu), _p(out), _s()),
              f"hp_group_norm_parts n={n} hw={hw} C={c}")
        return out
    if stats is None:
        stats = torch.empty(2 * n * groups * 256, dtype=torch.float32, device=x.device)
    check(lib.hp_group_norm(_p(x), c, _p(x2), c2, n, hw, groups, eps, _p(gamma), _p(beta), int(silu),
                            _p(out), _p(stats), _s()), f"hp_group_norm n={n} hw={hw} C={C_}")
    return out


def layer_norm(x, c, *, eps=1e-6, gamma=None, beta=None, shift=None, scale=None, ldm=0, rows_per_batch=0,
               out=None):
    lib = N.load()
    rows = x.numel() // c
    if out is None:
        out = torch.empty((rows, c), dtype=torch.bfloat16, device=x.device)
    check(lib.hp_layer_norm(_p(x), rows, c, eps, _p(gamma), _p(beta), _p(shift), _p(scale), int(ldm),
                            int(rows_per_batch), _p(out), _s()), "hp_layer_norm")
    return out


def layer_norm_joint(x, c, rows_per_batch, split, shift, scale, shift2, scale2, ldm, *, eps=1e-6, out=None):
    """Two-stream modulated LayerNorm over a [batch, rows_per_batch, c] token buffer."""
    lib = N.load()
    rows = x.numel() // c
    if out is None:
        out = torch.empty_like(x)
    check(lib.hp_layer_norm_joint(_p(x), rows, c, eps, _p(shift), _p(scale), _p(shift2), _p(scale2), int(ldm),
                                  int(rows_per_batch), int(split), _p(out), _s()), "hp_layer_norm_joint")
    return out


def quick_gelu(x, out=None):
    lib = N.load()
    out = torch.empty_like(x) if out is None else out
    check(lib.hp_quick_gelu(_p(x), _p(out), x.numel(), _s()), "hp_quick_gelu")
    return out


def silu(x, out=None):
    lib = N.load()
    out = torch.empty_like(x) if out is None else out
    check(lib.hp_silu(_p(x), _p(out), x.numel(), _s()), "hp_silu")
    return out


# sub-pixel decomposition of nearest-2x upsample + 3x3 conv: for output phase p (row or
# column parity) the 2x2 taps t = 0, 1 read input offsets p - 1 + t, and collect the 3x3
# taps k that land on the same input pixel
_UP_TAPS = {0: ((0,), (1, 2)), 1: ((0, 1), (2,))}


def upconv_weights(w3):
    """3x3 conv weights [co, 3, 3, ci] (any float dtype) -> the HP_A_UPCONV operand
    [4 * co, 4 * ci] bf16: phase-major (py, px), then tap (ty, tx), channel-minor."""
    w3 = w3.float()
    co, _, _, ci = w3.shape
    ph = []
    for py in (0, 1):
        for px in (0, 1):
            taps = []
            for ty in (0, 1):
                for tx in (0, 1):
                    t = torch.zeros(co, ci, device=w3.device)
                    for ky in _UP_TAPS[py][ty]:
                        for kx in _UP_TAPS[px][tx]:
                            t = t + w3[:, ky, kx, :]
                    taps.append(t)
            ph.append(torch.stack(taps, dim=1).reshape(co, 4 * ci))
    return torch.cat(ph, dim=0).to(torch.bfloat16).contiguous()


def upsample_conv(x, n, h, w, c, w4, bias=None, out=None, gn=False):
    """conv3x3(nearest_upsample_2x(x)) in one tensor-core launch (HP_A_UPCONV):
    x [n*h*w, c] NHWC low-res, w4 = upconv_weights(...) -> [n*2h*2w, co].
    ``gn``: also record the output's GroupNorm partials (``out.hp_gn``)."""
    lib = N.load()
    _bf16(x, "A")
    _bf16(w4, "W")
    co = w4.shape[0] // 4
    if w4.shape[1] != 4 * c:
        raise ShapeError(f"upconv weight K={w4.shape[1]} != 4*{c}")
    if out is None:
        out = torch.empty((n * 4 * h * w, co), dtype=torch.bfloat16, device=x.device)
    d = HpGemmDesc()
    d.a, d.lda, d.a_mode = _p(x), c, HP_A_UPCONV
    d.img_n, d.img_h, d.img_w, d.img_c = n, h, w, c
    d.b, d.ldb = _p(w4), w4.stride(0)
    d.d, d.ldd = _p(out), out.stride(0)
    d.M, d.N, d.K = n * h * w, co, 4 * c
    d.bias = _p(bias)
    d.alpha = 1.0
    gp = None
    if gn and gn_parts_ok(n * 4 * h * w, co, 4 * h * w) and (h * w) % GN_ROWS == 0:
        # partials per output image: 4 phases x (h*w / 128) blocks, phase-major
        gp = GnParts(_gn_buf(n * 4 * h * w, co, x.device), 4 * h * w, co)
        d.gn_part, d.gn_rows, d.gn_parts = _p(gp.buf), h * w, 4 * h * w // GN_ROWS
    check(lib.hp_gemm(C.byref(d), _s()), f"hp_gemm upconv n={n} {h}x{w} {c}->{co}")
    if gp is not None:
        out.hp_gn = gp
    return out


def upsample2x(x, n, h, w, c):
    lib = N.load()
    out = torch.empty((n * 4 * h * w, c), dtype=torch.bfloat16, device=x.device)
    check(lib.hp_upsample2x(_p(x), n, h, w, c, _p(out), _s()), "hp_upsample2x")
    return out


def concat_channels(a, c1, b, c2, pixels):
    """[a | b] along channels; when both inputs carry GroupNorm partials of the same
    image size, the result carries both (``out.hp_gn``: channels [0, c1) from a's)."""
    lib = N.load()
    out = torch.empty((pixels, c1 + c2), dtype=torch.bfloat16, device=a.device)
    check(lib.hp_concat_channels(_p(a), c1, _p(b), c2, pixels, _p(out), _s()), "hp_concat_channels")
    ga, gb = getattr(a, "hp_gn", None), getattr(b, "hp_gn", None)
    if (ga is not None and gb is not None and ga.parts2 is None and gb.parts2 is None and ga.hw == gb.hw
            and ga.c == c1 and gb.c == c2):
        out.hp_gn = GnParts(ga.buf, ga.hw, c1 + c2, parts2=gb, c1=c1)
    return out


def embed_tokens(ids, tok, pos, out=None):
    """ids [n, seq] int64 -> [n*seq, dim] bf16 = tok[ids] + pos[position]."""
    lib = N.load()
    n, seq = ids.shape
    dim = tok.shape[1]
    if out is None:
        out = torch.empty((n * seq, dim), dtype=torch.bfloat16, device=ids.device)
    check(lib.hp_embed_tokens(_p(ids), n * seq, seq, _p(tok), _p(pos), dim, _p(out), _s()), "hp_embed_tokens")
    return out


def softmax_rows(x, scale=1.0, out=None):
    """Row softmax of a 2-D bf16 matrix (fp32 math), e.g. attention scores."""
    lib = N.load()
    rows, cols = x.shape
    if out is None:
        out = torch.empty((rows, cols), dtype=torch.bfloat16, device=x.device)
    check(lib.hp_softmax_rows(_p(x), x.stride(0), rows, cols, float(scale), _p(out), out.stride(0), _s()),
          "hp_softmax_rows")
    return out


def copy_cols(x, c_dst, *, c_src=None, out=None):
    """Per-row channel window: zero-pad or slice the last dim of a 2-D bf16 view."""
    lib = N.load()
    rows, ldx = x.shape[0], x.stride(0)
    c_src = x.shape[1] if c_src is None else c_src
    if out is None:
        out = torch.empty((rows, c_dst), dtype=torch.bfloat16, device=x.device)
    check(lib.hp_copy_cols(_p(x), ldx, c_src, rows, _p(out), out.stride(0), c_dst, _s()), "hp_copy_cols")
    return out


def conv3x3_small(x, n, h, w, cin, wgt, bias, cout, *, out=None, out_f32=False):
    lib = N.load()
    if out is None:
        out = torch.empty((n * h * w, cout), dtype=torch.float32 if out_f32 else torch.bfloat16,
                          device=x.device)
    check(lib.hp_conv3x3_small(_p(x), n, h, w, cin, _p(wgt), _p(bias), cout, _p(out), int(out_f32), _s()),
          "hp_conv3x3_small")
    return out


def timestep_embedding(t, dim, max_period=10000.0):
    lib = N.load()
    out = torch.empty((t.numel(), dim), dtype=torch.float32, device=t.device)
    check(lib.hp_timestep_embedding(_p(t), t.numel(), dim, float(max_period), _p(out), _s()),
          "hp_timestep_embedding")
    return out


SMALL_MAX_M = 8      # csrc/hp_norm.cu kSmallMaxM


def linear_small(x, w, bias=None, *, act_in=ACT_NONE, act_out=ACT_NONE, out=None):
    lib = N.load()
    M, K = x.shape
    Nn = w.shape[0]
    if out is None:
        out = torch.empty((M, Nn), dtype=torch.float32, device=x.device)
    # the kernel keeps up to SMALL_MAX_M input rows in shared memory; larger batches
    # (e.g. 8 prompts x 2 CFG branches) run as row chunks (rows are independent)
    for r0 in range(0, M, SMALL_MAX_M):
        m = min(SMALL_MAX_M, M - r0)
        xs, ys = x[r0:r0 + m], out[r0:r0 + m]
        check(lib.hp_linear_small(_p(xs), m, K, _p(w), _p(bias), Nn, act_in, act_out, _p(ys), _s()),
              "hp_linear_small")
    return out


def patchify(x, n, h, w, c, p, inverse=False, out=None):
    lib = N.load()
    if out is None:
        out = torch.empty(n * h * w * c, dtype=torch.bfloat16, device=x.device)
    check(lib.hp_patchify(_p(x), n, h, w, c, p, int(inverse), _p(out), _s()), "hp_patchify")
    return out


def add_rows(x, add, c, out=None):
    lib = N.load()
    rows = x.numel() // c
    out = torch.empty_like(x) if out is None else out
    check(lib.hp_add_rows(_p(x), _p(add), rows, add.numel() // c, c, _p(out), _s()), "hp_add_rows")
    return out


def gated_residual(x, y, gate, ldg, c, rows_per_batch):
    lib = N.load()
    check(lib.hp_gated_residual(_p(x), _p(y), _p(gate), ldg, x.numel() // c, c, rows_per_batch, _s()),
          "hp_gated_residual")
    return x


def cast_bf16_f32(x, out):
    lib = N.load()
    check(lib.hp_cast_bf16_f32(_p(x), _p(out), x.numel(), _s()), "hp_cast_bf16_f32")
    return out
