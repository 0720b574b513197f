"""GPU: denoiser kernels (tcgen05 GEMM / conv, attention, norms) vs plain torch fp32.

Tolerances: outputs are bf16, so each check is max-abs error <= tol * max|ref|
with tol = 1e-2 (one bf16 ulp is 2^-8 = 3.9e-3 relative) unless stated.
"""
import math

import pytest
import torch
import torch.nn.functional as F

from paper_2602_21760_b200.denoiser import kernels as K

pytestmark = pytest.mark.gpu
TOL = 1e-2


def close(out, ref, tol=TOL):
    out = out.float()
    err = (out - ref).abs().max().item()
    scale = ref.abs().max().item() + 1e-6
    assert err <= tol * scale, f"max err {err:.4g} vs scale {scale:.4g} ({err / scale:.3g})"


def rnd(*shape, s=1.0):
    return (torch.randn(*shape, device="cuda") * s).bfloat16()


@pytest.mark.parametrize("M,N,Kd,bn", [(128, 64, 64, 0), (256, 256, 128, 0), (2048, 1280, 1280, 0),
                                       (154, 640, 2048, 0), (8192, 320, 640, 0), (300, 128, 72, 0),
                                       (1024, 512, 256, 64), (1024, 512, 256, 128), (1024, 512, 256, 256),
                                       (640, 320, 320, 160), (2048, 640, 640, 320), (8192, 1280, 640, 320),
                                       (300, 640, 192, 320)])
def test_gemm_plain(M, N, Kd, bn):
    torch.manual_seed(M + N + Kd)
    a, w = rnd(M, Kd), rnd(N, Kd, s=Kd ** -0.5)
    bias = torch.randn(N, device="cuda")
    out = K.gemm(a, w, bias=bias, block_n=bn)
    ref = a.float() @ w.float().t() + bias
    close(out, ref)


def test_gemm_epilogues():
    torch.manual_seed(1)
    M, N, Kd = 512, 256, 320
    a, w = rnd(M, Kd), rnd(N, Kd, s=Kd ** -0.5)
    bias = torch.randn(N, device="cuda")
    res = rnd(M, N)
    b2 = torch.randn(2, N, device="cuda")
    close(K.gemm(a, w, bias=bias, act=K.ACT_GELU), F.gelu(a.float() @ w.float().t() + bias))
    close(K.gemm(a, w, bias=bias, act=K.ACT_SILU), F.silu(a.float() @ w.float().t() + bias))
    close(K.gemm(a, w, bias=bias, residual=res), a.float() @ w.float().t() + bias + res.float())
    close(K.gemm(a, w, bias=bias, bias2=b2, bias2_div=M // 2),
          a.float() @ w.float().t() + bias + b2.repeat_interleave(M // 2, 0))
    close(K.gemm(a, w, alpha=0.5), 0.5 * (a.float() @ w.float().t()))


@pytest.mark.parametrize("bn", [128, 256])
def test_gemm_geglu(bn):
    torch.manual_seed(2)
    M, F_, Kd = 256, 512, 320
    a = rnd(M, Kd)
    w = rnd(2 * F_, Kd, s=Kd ** -0.5)
    bias = torch.randn(2 * F_, device="cuda")
    # interleave: each tile of bn rows = bn/2 "a" rows followed by the matching bn/2 gate rows
    h = bn // 2
    idx = torch.cat([torch.cat([torch.arange(i, i + h), torch.arange(F_ + i, F_ + i + h)])
                     for i in range(0, F_, h)]).cuda()
    out = K.gemm(a, w[idx].contiguous(), bias=bias[idx].contiguous(), act=K.ACT_GEGLU, block_n=bn)
    full = a.float() @ w.float().t() + bias
    ref = full[:, :F_] * F.gelu(full[:, F_:])
    close(out, ref)


@pytest.mark.parametrize("n,h,w,c,co,stride", [(2, 32, 32, 64, 128, 1), (1, 128, 128, 64, 64, 1),
                                               (2, 64, 64, 128, 256, 1), (1, 256, 256, 64, 64, 1),
                                               (2, 64, 64, 64, 64, 2), (2, 128, 128, 64, 128, 2),
                                               (1, 16, 16, 192, 320, 1), (2, 64, 64, 128, 640, 1),
                                               (2, 128, 128, 64, 320, 1), (2, 32, 32, 1280, 1280, 1)])
def test_conv3x3_implicit_gemm(n, h, w, c, co, stride):
    torch.manual_seed(h + c)
    x = rnd(n, h, w, c)
    wt = rnd(co, c, 3, 3, s=(9 * c) ** -0.5)
    bias = torch.randn(co, device="cuda")
    wk = wt.permute(0, 2, 3, 1).reshape(co, 9 * c).contiguous()
    out = K.gemm(x, wk, bias=bias, conv=(n, h, w, c, stride))
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), wt.float(), bias, stride=stride, padding=1)
    close(out.view(n, h // stride, w // stride, co), ref.permute(0, 2, 3, 1))


# dispatch (csrc/hp_attn.cu hp_attention): one key block -> single-block CTAs;
# up to 32 key blocks -> persistent split-KV units; beyond -> persistent two-tile
# units sharing K/V. Each path with and without the partial-key-block mask
# (S_kv % 128 != 0):
ATTN_SHAPES = [
    (1, 1, 128, 128), (2, 4, 256, 77),                    # single block
    (2, 20, 1024, 77), (1, 3, 200, 16), (1, 2, 130, 100),  # single block: SDXL cross-attention, one 16-key
                                                          # unit (second softmax half idle), odd unit count
    (2, 3, 256, 256), (1, 2, 1024, 1024),                 # split-KV, unmasked
    (2, 2, 333, 333), (2, 1, 130, 500),                   # split-KV, masked
    (2, 10, 4096, 4096), (2, 20, 1024, 1024),             # split-KV at the SDXL-1024 shapes (B=2)
    (1, 37, 1024, 1024), (1, 20, 1024, 1024),             # split-KV, B=1 (one branch per GPU)
    (2, 24, 4429, 4429),                                  # two-tile, masked: SD3-1024 joint attention
    (1, 24, 4429, 4429),                                  # SD3 at B=1 (one branch per GPU)
    (1, 2, 16384, 16384),                                 # two-tile, unmasked: SDXL-2048 level 1
]


@pytest.mark.parametrize("H,S,SKV", [(20, 1024, 1024), (10, 4096, 4096), (24, 4429, 4429), (20, 1024, 77)])
def test_attention_batch_invariant(H, S, SKV):
    """Image 1's rows of a B=2 launch equal a B=1 launch on image 1 bit for bit (the unit
    kind and split points depend on the key count only)."""
    torch.manual_seed(S + H + SKV)
    q, k, v = rnd(2 * S, H * 64), rnd(2 * SKV, H * 64), rnd(2 * SKV, H * 64)
    o2 = torch.empty_like(q)
    K.attention(q, k, v, o2, batch=2, heads=H, sq=S, skv=SKV, scale=0.125)
    o1 = torch.empty(S, H * 64, dtype=torch.bfloat16, device="cuda")
    K.attention(q[S:].contiguous(), k[SKV:].contiguous(), v[SKV:].contiguous(), o1, batch=1, heads=H, sq=S,
                skv=SKV, scale=0.125)
    assert torch.equal(o2[S:], o1)


@pytest.mark.parametrize("B,H,sq,skv", ATTN_SHAPES)
def test_attention(B, H, sq, skv):
    torch.manual_seed(sq + skv)
    q = rnd(B * sq, H * 64)
    k = rnd(B * skv, H * 64)
    v = rnd(B * skv, H * 64)
    o = torch.empty_like(q)
    K.attention(q, k, v, o, batch=B, heads=H, sq=sq, skv=skv, scale=1 / 8)
    qf = q.float().view(B, sq, H, 64).transpose(1, 2)
    kf = k.float().view(B, skv, H, 64).transpose(1, 2)
    vf = v.float().view(B, skv, H, 64).transpose(1, 2)
    ref = F.scaled_dot_product_attention(qf, kf, vf, scale=1 / 8).transpose(1, 2).reshape(B * sq, H * 64)
    close(o, ref, tol=2e-2)


def test_attention_fused_qkv_columns():
    B, S, H = 2, 256, 2
    qkv = rnd(B * S, 3 * H * 64)
    o = torch.empty(B * S, H * 64, dtype=torch.bfloat16, device="cuda")
    K.attention(qkv, qkv, qkv, o, batch=B, heads=H, sq=S, skv=S, scale=0.125, q_col0=0, k_col0=H * 64,
                v_col0=2 * H * 64)
    q, k, v = qkv.float().view(B, S, 3, H, 64).unbind(2)
    ref = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), scale=0.125)
    close(o, ref.transpose(1, 2).reshape(B * S, H * 64), tol=2e-2)


@pytest.mark.parametrize("n,hw,c,c2,silu", [(2, 4096, 320, 0, True), (2, 1024, 1280, 640, False),
                                            (1, 256, 960, 0, True),
                                            # >= 16 KB pixel chunks: staged in shared memory
                                            (2, 16384, 320, 0, True), (2, 4096, 640, 640, True),
                                            (2, 1024, 1280, 1280, False)])
def test_group_norm(n, hw, c, c2, silu):
    x = rnd(n * hw, c, s=2.0) + 0.5
    x2 = rnd(n * hw, c2) if c2 else None
    C = c + c2
    g, b = torch.randn(C, device="cuda"), torch.randn(C, device="cuda")
    out = K.group_norm(x, n, hw, c, g, b, silu=silu, x2=x2, c2=c2)
    full = x.float() if x2 is None else torch.cat([x.float(), x2.float()], 1)
    ref = F.group_norm(full.view(n, hw, C).permute(0, 2, 1), 32, g, b, eps=1e-5).permute(0, 2, 1).reshape(n * hw, C)
    if silu:
        ref = F.silu(ref)
    close(out, ref)


@pytest.mark.parametrize("hw,c", [(1024, 640), (16384, 320)])
def test_group_norm_batch_invariant(hw, c):
    """Image 1's output does not depend on image 0 (also on the shared-memory staged path)."""
    x = rnd(2 * hw, c)
    g, b = torch.ones(c, device="cuda"), torch.zeros(c, device="cuda")
    both = K.group_norm(x, 2, hw, c, g, b)
    one = K.group_norm(x[hw:].contiguous(), 1, hw, c, g, b)
    assert torch.equal(both[hw:], one)


def test_group_norm_concurrent_streams_and_graphs():
    """Single-launch GroupNorms in flight at once on two streams, and inside two CUDA
    graphs replayed on two streams, each with its own barrier slot: every output
    matches the reference (a shared barrier would mix the images' arrivals)."""
    n, hw, c = 2, 4096, 640
    xs = [rnd(n * hw, c, s=2.0) + 0.5 * i for i in range(2)]
    g, b = torch.randn(c, device="cuda"), torch.randn(c, device="cuda")
    refs = [F.group_norm(x.float().view(n, hw, c).permute(0, 2, 1), 32, g, b, eps=1e-5).permute(0, 2, 1)
            .reshape(n * hw, c) for x in xs]
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [torch.empty(n * hw, c, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    torch.cuda.synchronize()
    for _ in range(20):
        for i in range(2):
            with torch.cuda.stream(streams[i]):
                K.group_norm(xs[i], n, hw, c, g, b, out=outs[i])
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        close(o, r)
    graphs = []
    for i in range(2):
        K.group_norm(xs[i], n, hw, c, g, b, out=outs[i])        # warm (attributes, pool)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            K.group_norm(xs[i], n, hw, c, g, b, out=outs[i])
        graphs.append(gr)
    for o in outs:
        o.zero_()
    torch.cuda.synchronize()
    for _ in range(20):
        for i in range(2):
            with torch.cuda.stream(streams[i]):
                graphs[i].replay()
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        close(o, r)


@pytest.mark.parametrize("c", [640, 1280, 1536])
def test_layer_norm(c):
    x = rnd(700, c) + 1.0
    g, b = torch.randn(c, device="cuda"), torch.randn(c, device="cuda")
    close(K.layer_norm(x, c, gamma=g, beta=b, eps=1e-5), F.layer_norm(x.float(), (c,), g, b, eps=1e-5))
    sh, sc = torch.randn(2, c, device="cuda"), torch.randn(2, c, device="cuda") * 0.3
    out = K.layer_norm(x[:600], c, shift=sh, scale=sc, ldm=c, rows_per_batch=300)
    ref = F.layer_norm(x[:600].float(), (c,), eps=1e-6)
    ref = ref * (1 + sc.repeat_interleave(300, 0)) + sh.repeat_interleave(300, 0)
    close(out, ref)


def test_gemm_colscale_gate():
    """adaLN-Zero gated residual fused in the epilogue: d = res + gate[col] * (A W^T + b)."""
    M, N, Kd = 384, 256, 192
    a, w = rnd(M, Kd), rnd(N, Kd, s=Kd ** -0.5)
    b, g = torch.randn(N, device="cuda"), torch.randn(N, device="cuda")
    res = rnd(M, N)
    close(K.gemm(a, w, bias=b, colscale=g, residual=res),
          res.float() + g * (a.float() @ w.float().t() + b))


def test_small_ops():
    n, h, w = 2, 16, 16
    x4 = rnd(n, h, w, 4)
    wt = torch.randn(320, 4, 3, 3, device="cuda") * 0.3
    bias = torch.randn(320, device="cuda")
    out = K.conv3x3_small(x4, n, h, w, 4, wt.permute(0, 2, 3, 1).contiguous(), bias, 320)
    ref = F.conv2d(x4.float().permute(0, 3, 1, 2), wt, bias, padding=1).permute(0, 2, 3, 1)
    close(out.view(n, h, w, 320), ref)
    x320 = rnd(n, h, w, 320)
    wo = torch.randn(4, 320, 3, 3, device="cuda") * 0.05
    bo = torch.randn(4, device="cuda")
    out = K.conv3x3_small(x320, n, h, w, 320, wo.permute(0, 2, 3, 1).contiguous(), bo, 4)
    ref = F.conv2d(x320.float().permute(0, 3, 1, 2), wo, bo, padding=1).permute(0, 2, 3, 1)
    close(out.view(n, h, w, 4), ref)
    up = K.upsample2x(x320, n, h, w, 320)
    assert torch.equal(up.view(n, 2 * h, 2 * w, 320),
                       x320.repeat_interleave(2, 1).repeat_interleave(2, 2))
    cat = K.concat_channels(x320.view(-1, 320), 320, x4.view(-1, 4).repeat(1, 2), 8, n * h * w)
    assert torch.equal(cat[:, :320], x320.view(-1, 320))
    t = torch.tensor([999.0, 1.0], device="cuda")
    emb = K.timestep_embedding(t, 320)
    half = 160
    fr = torch.exp(-math.log(10000.0) * torch.arange(half, device="cuda") / half)
    ref = torch.cat([torch.cos(t[:, None] * fr), torch.sin(t[:, None] * fr)], 1)
    assert (emb - ref).abs().max().item() < 2e-3
    xs = torch.randn(2, 320, device="cuda")
    ws = rnd(1280, 320, s=0.05)
    bs = torch.randn(1280, device="cuda")
    ys = K.linear_small(xs, ws, bs, act_in=K.ACT_SILU)
    assert (ys - (F.silu(xs) @ ws.float().t() + bs)).abs().max().item() < 1e-3
    xb = torch.randn(19, 320, device="cuda")               # > 8 rows: chunked (8 prompts x CFG)
    yb = K.linear_small(xb, ws, bs, act_out=K.ACT_SILU)
    assert (yb - F.silu(xb @ ws.float().t() + bs)).abs().max().item() < 1e-3
    lat = rnd(2, 8, 8, 16)
    tok = K.patchify(lat, 2, 8, 8, 16, 2)
    ref = lat.view(2, 4, 2, 4, 2, 16).permute(0, 1, 3, 2, 4, 5).reshape(-1)
    assert torch.equal(tok, ref)
    assert torch.equal(K.patchify(tok, 2, 8, 8, 16, 2, inverse=True), lat.reshape(-1))


@pytest.mark.parametrize("M,N,Kd,bn", [(2048, 1280, 1280, 160), (2048, 1280, 1280, 256), (8192, 640, 640, 160),
                                       (300, 640, 320, 128), (256, 1536, 256, 256)])
def test_gemm_fused_layernorm_cluster(M, N, Kd, bn):
    """Residual GEMM + LayerNorm of its output rows in one launch (cluster DSMEM row sums)."""
    torch.manual_seed(M + N)
    a, w = rnd(M, Kd), rnd(N, Kd, s=Kd ** -0.5)
    b = torch.randn(N, device="cuda")
    h = rnd(M, N, s=2.0) + 0.3
    h_ref = h.float() + a.float() @ w.float().t() + b
    g, be = torch.randn(N, device="cuda"), torch.randn(N, device="cuda")
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    out = K.gemm(a, w, bias=b, residual=h, out=h, block_n=bn, ln=(g, be, 1e-5, y))
    close(out, h_ref)
    ref_y = F.layer_norm(out.float(), (N,), g, be, eps=1e-5)      # LN of the stored bf16 rows
    close(y, ref_y, tol=2e-2)


@pytest.mark.parametrize("M,C,Nc,act", [(2048, 1280, 3840, K.ACT_NONE), (8192, 640, 640, K.ACT_NONE),
                                        (300, 320, 512, K.ACT_GEGLU), (2048, 1280, 2560, K.ACT_GEGLU)])
def test_gemm_layernorm_fold(M, C, Nc, act):
    """Producer GEMM (+residual) records row (mean, M2) per N tile; the consumer
    GEMM applies LayerNorm(gamma, beta) in its epilogue from those partials
    with gamma folded into its weights == GEMM(LayerNorm(h)) in fp32."""
    torch.manual_seed(M + C)
    a, w0 = rnd(M, C), rnd(C, C, s=C ** -0.5)
    res = (torch.randn(M, C, device="cuda") * 3 + 1.5).bfloat16()      # off-centre residual stream
    rs = K.RowStats(2 * M * C // 64, "cuda")
    h = K.gemm(a, w0, residual=res, stats_out=rs)
    # partials are exact statistics of the stored bf16 tile segments
    seg = h.float().view(M, rs.parts, rs.part_n)
    st = rs.buf[:2 * M * rs.parts].view(M, rs.parts, 2)
    torch.testing.assert_close(st[..., 0], seg.mean(-1), rtol=1e-5, atol=1e-5)
    m2 = ((seg - seg.mean(-1, keepdim=True)) ** 2).sum(-1)
    torch.testing.assert_close(st[..., 1], m2, rtol=1e-4, atol=1e-3)
    gamma = 1.0 + 0.2 * torch.randn(C, device="cuda")
    beta = 0.1 * torch.randn(C, device="cuda")
    w = torch.randn(Nc, C, device="cuda") * C ** -0.5
    bias = torch.randn(Nc, device="cuda")
    fold = K.FoldedLN(w, gamma, beta, bias=bias, eps=1e-5)
    out = K.gemm(h, fold.w, bias=fold.bias, act=act, block_n=256 if act == K.ACT_GEGLU else 0, ln_fold=(rs, fold))
    y = F.layer_norm(h.float(), (C,), gamma, beta, eps=1e-5)
    pre = y @ w.t() + bias
    if act == K.ACT_GEGLU:
        # host interleaving convention of the GEGLU epilogue: per 256-wide tile, 128 hidden + 128 gate
        pre = pre.view(M, Nc // 256, 2, 128)
        ref = (pre[:, :, 0] * F.gelu(pre[:, :, 1])).reshape(M, Nc // 2)
    else:
        ref = pre
    close(out, ref, tol=2e-2)


@pytest.mark.parametrize("N,Kd,stats", [(1280, 1280, False), (1280, 5120, True), (640, 640, True)])
def test_gemm_rows_batch_invariant(N, Kd, stats):
    """An image's rows come out bit-identical whatever else is in the batch: tile width,
    split-K and the statistics layout depend on N and K only (serial CFG-batched and
    condition-partitioned runs then produce the same latents)."""
    torch.manual_seed(N + Kd)
    a, w = rnd(2048, Kd), rnd(N, Kd, s=Kd ** -0.5)
    res = rnd(2048, N)
    kw = {}
    outs = []
    for rows in (2048, 1024):
        rs = K.RowStats(2 * rows * N // 64, "cuda") if stats else None
        out = K.gemm(a[:rows], w, residual=res[:rows], stats_out=rs)
        outs.append((out, rs))
    (o2, r2), (o1, r1) = outs
    assert torch.equal(o2[:1024], o1)
    if stats:
        assert r2.parts == r1.parts and r2.part_n == r1.part_n
        assert torch.equal(r2.buf[:2 * 1024 * r1.parts], r1.buf[:2 * 1024 * r1.parts])


@pytest.mark.parametrize("n,h,w,c,co", [(2, 32, 32, 1280, 1280), (2, 64, 64, 640, 640), (1, 16, 16, 64, 128),
                                        (1, 8, 32, 128, 320)])
def test_upsample_conv_subpixel(n, h, w, c, co):
    """nearest-2x upsample + 3x3 conv as four sub-pixel 2x2 convs in one launch
    (HP_A_UPCONV) vs torch fp32 on the same bf16 input and weights."""
    torch.manual_seed(n * h + c)
    x = rnd(n * h * w, c)
    w3 = torch.randn(co, 3, 3, c, device="cuda") * (9 * c) ** -0.5
    bias = torch.randn(co, device="cuda")
    out = K.upsample_conv(x, n, h, w, c, K.upconv_weights(w3), bias)
    xi = x.float().view(n, h, w, c).permute(0, 3, 1, 2)
    ref = F.conv2d(F.interpolate(xi, scale_factor=2, mode="nearest"), w3.permute(0, 3, 1, 2), bias, padding=1)
    close(out.view(n, 2 * h, 2 * w, co), ref.permute(0, 2, 3, 1))


def _gn_ref(full, n, hw, C, g, b, silu):
    ref = F.group_norm(full.view(n, hw, C).permute(0, 2, 1), 32, g, b, eps=1e-5).permute(0, 2, 1).reshape(n * hw, C)
    return F.silu(ref) if silu else ref


# GroupNorm statistics from the producing GEMM's epilogue (gemm(gn_hw=), hp_group_norm_parts):
# plain (with residual and per-image bias), split-K (K >= 4096 at N = 1280), 3x3 conv
# (pair 160 / 320 wide), against torch GroupNorm of the GEMM's own output
@pytest.mark.parametrize("kind,n,hw,Kd,N", [("plain", 2, 1024, 1280, 1280), ("splitk", 2, 1024, 5120, 1280),
                                            ("plain", 1, 4096, 640, 640), ("conv", 2, 1024, 640, 1280),
                                            ("conv", 2, 4096, 320, 640), ("conv", 1, 16384, 320, 320)])
def test_gemm_groupnorm_partials(kind, n, hw, Kd, N):
    torch.manual_seed(hw + N + Kd)
    side = int(math.isqrt(hw))
    if kind == "conv":
        x = rnd(n * hw, Kd)
        w = rnd(N, 9 * Kd, s=(9 * Kd) ** -0.5)
        kw = dict(conv=(n, side, side, Kd, 1))
    else:
        x = rnd(n * hw, Kd)
        w = rnd(N, Kd, s=Kd ** -0.5)
        kw = dict(residual=rnd(n * hw, N, s=0.5) + 0.25)
    bias, b2 = torch.randn(N, device="cuda"), torch.randn(n, N, device="cuda")
    y = K.gemm(x, w, bias=bias, bias2=b2, bias2_div=hw, gn_hw=hw, **kw)
    assert getattr(y, "hp_gn", None) is not None
    g, b = torch.randn(N, device="cuda"), torch.randn(N, device="cuda")
    out = K.group_norm(y, n, hw, N, g, b, silu=True)
    close(out, _gn_ref(y.float(), n, hw, N, g, b, True))
    y.hp_gn = None                                   # the two-pass path on the same tensor
    close(out, K.group_norm(y, n, hw, N, g, b, silu=True).float(), tol=8e-3)


def test_gemm_groupnorm_partials_batch_invariant():
    """Image 1's partials and normalised output from a B=2 GEMM equal a B=1 GEMM on image 1
    bit for bit, although M changes (and with it the tile width the GEMM picks)."""
    torch.manual_seed(7)
    hw, Kd, N = 1024, 1280, 1280
    x, w = rnd(2 * hw, Kd), rnd(N, Kd, s=Kd ** -0.5)
    res = rnd(2 * hw, N)
    g, b = torch.randn(N, device="cuda"), torch.randn(N, device="cuda")
    y2 = K.gemm(x, w, residual=res, gn_hw=hw)
    y1 = K.gemm(x[hw:].contiguous(), w, residual=res[hw:].contiguous(), gn_hw=hw)
    assert torch.equal(y2[hw:], y1)
    half = y2.hp_gn.buf.numel() // 2
    assert torch.equal(y2.hp_gn.buf[half:], y1.hp_gn.buf)
    assert torch.equal(K.group_norm(y2, 2, hw, N, g, b, silu=True)[hw:], K.group_norm(y1, 1, hw, N, g, b, silu=True))


@pytest.mark.parametrize("n,h,w,c,co,c2", [(2, 32, 32, 1280, 1280, 640), (2, 64, 64, 640, 640, 320)])
def test_groupnorm_partials_upconv_concat(n, h, w, c, co, c2):
    """Upsampler output (phase-major partials) concatenated with a skip that carries its own
    partials: one GroupNorm over the concat (groups straddle the two inputs) vs torch."""
    torch.manual_seed(h + c)
    x = rnd(n * h * w, c)
    w3 = torch.randn(co, 3, 3, c, device="cuda") * (9 * c) ** -0.5
    up = K.upsample_conv(x, n, h, w, c, K.upconv_weights(w3), torch.randn(co, device="cuda"), gn=True)
    hw = 4 * h * w
    sk = K.gemm(rnd(n * hw, 320), rnd(c2, 320, s=320 ** -0.5), gn_hw=hw)
    assert up.hp_gn is not None and sk.hp_gn is not None
    cat = K.concat_channels(up, co, sk, c2, n * hw)
    assert cat.hp_gn.parts2 is not None
    C = co + c2
    g, b = torch.randn(C, device="cuda"), torch.randn(C, device="cuda")
    out = K.group_norm(cat, n, hw, C, g, b, silu=True)
    close(out, _gn_ref(cat.float(), n, hw, C, g, b, True))


@pytest.mark.parametrize("M", [2048, 1024])
def test_gemm_geglu_halfwidth_tail(M):
    """SDXL level-3 GEGLU (N = 2 x 5120 interleaved, K = 1280): 320 (M=2048) / 160 (M=1024)
    256-wide pair tiles leave a partial last wave on 74 CTA pairs, which runs as half-width
    tiles. Against torch fp32 with the LayerNorm fold, and bit-identical rows between the
    two batch sizes (and with the tail split switched off)."""
    import os
    import subprocess
    import sys
    torch.manual_seed(11)
    C, F_ = 1280, 5120
    h = rnd(2048, C)
    rs = K.RowStats(2 * 2048 * C // 64, "cuda")
    h = K.gemm(h, rnd(C, C, s=C ** -0.5), residual=rnd(2048, C), stats_out=rs)
    gamma, beta = 1.0 + 0.2 * torch.randn(C, device="cuda"), 0.1 * torch.randn(C, device="cuda")
    w, bias = torch.randn(2 * F_, C, device="cuda") * C ** -0.5, torch.randn(2 * F_, device="cuda")
    fold = K.FoldedLN(w, gamma, beta, bias=bias, eps=1e-5)
    out = K.gemm(h[:M], fold.w, bias=fold.bias, act=K.ACT_GEGLU, block_n=256, ln_fold=(rs, fold))
    pre = (F.layer_norm(h[:M].float(), (C,), gamma, beta, eps=1e-5) @ w.t() + bias).view(M, 2 * F_ // 256, 2, 128)
    close(out, (pre[:, :, 0] * F.gelu(pre[:, :, 1])).reshape(M, F_), tol=2e-2)
    if M == 1024:
        full = K.gemm(h, fold.w, bias=fold.bias, act=K.ACT_GEGLU, block_n=256, ln_fold=(rs, fold))
        assert torch.equal(full[:1024], out)


def test_groupnorm_partials_dropped_when_overwritten():
    """A GEMM that writes in place into a tensor carrying GroupNorm partials without
    recording new ones drops them (stale statistics must never be folded)."""
    torch.manual_seed(5)
    hw, C = 1024, 640
    y = K.gemm(rnd(2 * hw, 320), rnd(C, 320, s=320 ** -0.5), gn_hw=hw)
    assert y.hp_gn is not None
    K.gemm(rnd(2 * hw, 320), rnd(C, 320, s=320 ** -0.5), out=y)        # no gn_hw: partials now stale
    assert getattr(y, "hp_gn", None) is None
    g, b = torch.randn(C, device="cuda"), torch.randn(C, device="cuda")
    close(K.group_norm(y, 2, hw, C, g, b), _gn_ref(y.float(), 2, hw, C, g, b, False))
