"""GPU: the SD3-shaped MMDiT on our kernels (batched GEMMs, joint LayerNorm,
gated-residual epilogues, joint attention) vs the plain-torch fp32 reference,
and a flow-matching Euler CFG run through the engine vs the oracle loop.

Tolerances (bf16 compute): forward max-abs <= 5e-2 of max|ref|, mean-abs <=
1e-2 of mean|ref|; 28-step x0 max-abs <= 5e-2, mean-abs <= 1e-2.
"""
import numpy as np
import pytest
import torch

import paper_2602_21760_b200 as hp
from paper_2602_21760_b200 import pipelines
from paper_2602_21760_b200.denoiser.mmdit import MMDiT
from paper_2602_21760_b200.denoiser.weights import TINY_DIT, init_weights, mmdit_param_specs, synthetic_conditioning

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    W = init_weights(mmdit_param_specs(TINY_DIT), seed=0, device="cpu")
    cond = synthetic_conditioning(2, TINY_DIT.ctx_len, TINY_DIT.ctx_dim, TINY_DIT.pooled_dim)
    return W, cond


def _ref(W):
    from oracle.mmdit_ref import MMDiTRef
    return MMDiTRef(TINY_DIT, {k: v.cuda() for k, v in W.items()})


def test_forward_matches_fp32_reference(tiny):
    W, cond = tiny
    s = TINY_DIT
    net = MMDiT(s, W)
    ctx = torch.cat([cond.null_context, cond.context[:1]]).cuda()
    pooled = torch.cat([cond.null_pooled, cond.pooled[:1]]).cuda()
    net.prepare(ctx, pooled, key="k")
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(2, s.latent_hw, s.latent_hw, s.in_channels, device="cuda", generator=g)
    t = torch.tensor([750.0, 750.0], device="cuda")
    v = net.forward(x.bfloat16(), t, key="k").float()
    ref = _ref(W)(x, t, ctx, pooled)
    err = (v - ref).abs()
    assert err.max().item() <= 5e-2 * ref.abs().max().item(), err.max().item()
    assert err.mean().item() <= 1e-2 * ref.abs().mean().item()


def test_batch_invariance_bitwise(tiny):
    W, cond = tiny
    s = TINY_DIT
    net = MMDiT(s, W)
    ctx = torch.cat([cond.null_context, cond.context[:1]]).cuda()
    pooled = torch.cat([cond.null_pooled, cond.pooled[:1]]).cuda()
    net.prepare(ctx, pooled, key="both")
    net.prepare(ctx[1:], pooled[1:], key="one")
    x = torch.randn(2, s.latent_hw, s.latent_hw, s.in_channels, device="cuda").bfloat16()
    t = torch.tensor([500.0, 500.0], device="cuda")
    both = net.forward(x, t, key="both")
    one = net.forward(x[1:].contiguous(), t[1:].contiguous(), key="one")
    assert torch.equal(both[1:], one)


def test_euler_cfg_run_matches_oracle_loop(tiny):
    W, cond = tiny
    s = TINY_DIT
    T, w = 12, 4.0
    den = pipelines.build_sd3_denoiser(s, n_prompts=2, steps=T, weights=W, conditioning=cond)
    plan = pipelines.sd3_plan(s, variant="serial", steps=T, n_prompts=2, seed=5, guidance=w, denoiser=den,
                              clock="model")
    res = hp.run_plan(plan)
    ref = _ref(W)
    x = torch.from_numpy(hp.initial_latents(plan)).cuda().float()
    shape = (2, s.latent_hw, s.latent_hw, s.in_channels)
    with torch.no_grad():
        for t in range(T, 0, -1):
            tt = torch.full((2,), 1000.0 * t / T, device="cuda")
            xv = x.view(shape)
            vc = ref(xv, tt, cond.context.cuda(), cond.pooled.cuda()).reshape(2, -1)
            vu = ref(xv, tt, cond.null_context.expand(2, -1, -1).cuda(),
                     cond.null_pooled.expand(2, -1).cuda()).reshape(2, -1)
            x = x - (vc + w * (vc - vu)) / T
    err = np.abs(res.x0 - x.double().cpu().numpy())
    assert err.max() <= 5e-2, err.max()
    assert err.mean() <= 1e-2, err.mean()
    assert len(res.series) == T


def test_gemm_batched_matches_loop():
    from paper_2602_21760_b200.denoiser import kernels as K
    n, T, Ti, H = 3, 333, 256, 128
    X = torch.randn(n, T, H, device="cuda").bfloat16()
    w = (torch.randn(3 * H, H, device="cuda") * H ** -0.5).bfloat16()
    b = torch.randn(3 * H, device="cuda")
    out = torch.zeros(n, T, 3 * H, device="cuda", dtype=torch.bfloat16)
    K.gemm(X[:, Ti:], w, bias=b, out=out[:, Ti:])
    ref = X[:, Ti:].float() @ w.float().t() + b
    assert (out[:, Ti:].float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()
    assert out[:, :Ti].abs().max().item() == 0.0              # untouched rows
    gate = torch.randn(n, 2 * H, device="cuda")[:, H:]          # strided per-batch gate view
    res = torch.randn(n, Ti, H, device="cuda").bfloat16()
    o2 = K.gemm(X[:, :Ti], w[:H].contiguous(), bias=b[:H].contiguous(), residual=res, colscale=gate)
    ref2 = res.float() + gate[:, None, :] * (X[:, :Ti].float() @ w[:H].float().t() + b[:H])
    assert (o2.float() - ref2).abs().max().item() <= 1e-2 * ref2.abs().max().item()
