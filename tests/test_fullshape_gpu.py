"""GPU: the shipped configurations at FULL shape against the fp32 oracle networks.

* SDXL-1024 (BASELINE config 2): one B=2 CFG forward of the SDXL-shaped U-Net
  on our kernels vs ``oracle.unet_ref.UNetRef`` (plain torch fp32 on CUDA, TF32
  off), and a complete 50-step CFG DDIM generation through ``run_plan`` vs
  ``oracle.loop.run_exact`` (engine.py:195-214 restated, fp64 sampler) driven
  by UNetRef.
* SD3-1024 (config 3): one B=2 forward of the SD3-shaped MMDiT (S = 4096 image
  + 333 text tokens, 24 heads: the joint attention runs the two-tile kernel
  with the partial-key mask) vs ``oracle.mmdit_ref.MMDiTRef``.
* SDXL-2048 (config 4): one B=1 forward at a 256^2 latent (S = 16384 at the
  640-channel level) vs UNetRef.

Tolerances. The yardstick is the SAME network run as a stock-torch bf16 model
(``UNetRef``/``MMDiTRef`` with ``dtype=bfloat16``: cuBLAS/cuDNN bf16 with fp32
accumulation), compared with the fp32 oracle: that error is what bf16 itself
costs on a ~100-layer random-init network (about 1% mean-relative). Our
kernels must be no worse than 1.5x that yardstick (mean) / 2x (max), and
inside absolute sanity bounds (max-abs <= 3e-2 * max|ref|, mean-abs <= 2e-2 *
mean|ref|). Every measured error is printed as a ``PARITY`` line (recorded in
DESIGN.md section 4).
"""
import numpy as np
import pytest
import torch

import paper_2602_21760_b200 as hp
from paper_2602_21760_b200 import pipelines
from paper_2602_21760_b200.denoiser.weights import (SD3, SDXL, SDXL_2048, init_weights, mmdit_param_specs,
                                                    synthetic_conditioning, unet_param_specs)

pytestmark = pytest.mark.gpu

FWD_MAX, FWD_MEAN = 3e-2, 2e-2          # absolute sanity bounds, relative to |ref|
YARD_MAX, YARD_MEAN = 2.0, 1.5           # vs the stock-torch bf16 network's own error


@pytest.fixture(autouse=True)
def _fp32_exact():
    prev = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = prev
    torch.cuda.empty_cache()


def _report(name, out, ref):
    err = (out.float() - ref.float()).abs()
    mx, mean = err.max().item(), err.mean().item()
    rmx, rmean = ref.abs().max().item(), ref.abs().mean().item()
    print(f"PARITY {name}: max_abs={mx:.4g} ({mx / rmx:.3g} of max|ref|={rmx:.4g}) "
          f"mean_abs={mean:.4g} ({mean / rmean:.3g} of mean|ref|={rmean:.4g})")
    return mx, mean, rmx, rmean


def _check_forward(name, out, ref, yard):
    mx, mean, rmx, rmean = _report(name, out, ref)
    ymx, ymean, _, _ = _report(name + " [torch bf16 yardstick]", yard, ref)
    assert mx <= FWD_MAX * rmx, (name, mx, rmx)
    assert mean <= FWD_MEAN * rmean, (name, mean, rmean)
    assert mx <= YARD_MAX * ymx, (name, mx, ymx)
    assert mean <= YARD_MEAN * ymean, (name, mean, ymean)


def _unet_pair(spec, n_prompts=1):
    W = init_weights(unet_param_specs(spec), seed=0, device="cuda")
    cond = synthetic_conditioning(n_prompts, spec.context_len, spec.cross_dim, spec.pooled_dim, device="cuda")
    return W, cond


def _unet_forward_case(spec, n, t_net):
    from oracle.unet_ref import UNetRef
    from paper_2602_21760_b200.denoiser.unet import UNet
    W, cond = _unet_pair(spec)
    net = UNet(spec, W)
    ctx = torch.cat([cond.null_context, cond.context])[-n:].contiguous()
    pooled = torch.cat([cond.null_pooled, cond.pooled])[-n:].contiguous()
    net.prepare(ctx, pooled, key="k")
    g = torch.Generator(device="cuda").manual_seed(0)
    hw = spec.latent_hw
    x = torch.randn(n, hw, hw, spec.in_channels, device="cuda", generator=g)
    t = torch.full((n,), t_net, device="cuda")
    eps = net.forward(x.bfloat16(), t, key="k").float()
    del net
    torch.cuda.empty_cache()
    with torch.no_grad():
        ref = UNetRef(spec, W)(x.permute(0, 3, 1, 2), t, ctx, pooled).permute(0, 2, 3, 1)
        torch.cuda.empty_cache()
        yard = UNetRef(spec, W, torch.bfloat16)(x.permute(0, 3, 1, 2), t, ctx, pooled).permute(0, 2, 3, 1)
    return eps, ref, yard


@pytest.mark.parametrize("t_net", [979.0, 499.0, 19.0])
def test_sdxl1024_forward_vs_fp32(t_net):
    eps, ref, yard = _unet_forward_case(SDXL, 2, t_net)
    _check_forward(f"sdxl1024 B=2 forward t={t_net:g}", eps, ref, yard)


def test_sdxl2048_forward_vs_fp32():
    eps, ref, yard = _unet_forward_case(SDXL_2048, 1, 499.0)
    _check_forward("sdxl2048 B=1 forward t=499", eps, ref, yard)


def test_sd3_forward_vs_fp32():
    from oracle.mmdit_ref import MMDiTRef
    from paper_2602_21760_b200.denoiser.mmdit import MMDiT
    s = SD3
    W = init_weights(mmdit_param_specs(s), seed=0, device="cuda")
    cond = synthetic_conditioning(1, s.ctx_len, s.ctx_dim, s.pooled_dim, device="cuda")
    net = MMDiT(s, W)
    ctx = torch.cat([cond.null_context, cond.context]).contiguous()
    pooled = torch.cat([cond.null_pooled, cond.pooled]).contiguous()
    net.prepare(ctx, pooled, key="k")
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(2, s.latent_hw, s.latent_hw, s.in_channels, device="cuda", generator=g)
    t = torch.tensor([750.0, 750.0], device="cuda")
    v = net.forward(x.bfloat16(), t, key="k").float()
    del net
    torch.cuda.empty_cache()
    with torch.no_grad():
        ref = MMDiTRef(s, W)(x, t, ctx, pooled)
        yard = MMDiTRef(s, W, torch.bfloat16)(x, t, ctx, pooled)
    _check_forward("sd3 B=2 forward t=750", v, ref, yard)


class _RefBranches:
    """oracle.loop denoiser protocol over UNetRef on CUDA (fp32, TF32 off):
    (B, N) fp64 numpy in -> (eps_c, eps_u) fp64 numpy, one B=2B forward."""

    def __init__(self, net, cond, spec, T):
        self.net, self.c, self.s, self.T = net, cond, spec, T

    def branches(self, x, t):
        from oracle.unet_ref import net_timestep
        B = x.shape[0]
        hw, ch = self.s.latent_hw, self.s.in_channels
        xt = torch.from_numpy(np.asarray(x)).cuda().float().view(B, hw, hw, ch).permute(0, 3, 1, 2)
        xt = torch.cat([xt, xt])
        ctx = torch.cat([self.c.context[:B], self.c.null_context.expand(B, -1, -1)])
        pooled = torch.cat([self.c.pooled[:B], self.c.null_pooled.expand(B, -1)])
        tt = torch.full((2 * B,), net_timestep(t, self.T), device="cuda")
        with torch.no_grad():
            e = self.net(xt, tt, ctx, pooled).permute(0, 2, 3, 1).reshape(2 * B, -1).double().cpu().numpy()
        return e[:B], e[B:]


def test_sdxl1024_50step_generation_vs_oracle_loop():
    """BASELINE config 2's workload end to end: 50 CFG DDIM steps (w as the
    bench), x_T from the host seed path; serial == the shipped bench loop."""
    from oracle import loop as oloop
    from oracle.unet_ref import UNetRef
    T, seed, w = 50, 0, 5.0
    W, cond = _unet_pair(SDXL)
    den = pipelines.build_sdxl_denoiser(SDXL, n_prompts=1, steps=T, weights=W, conditioning=cond)
    plan = pipelines.sdxl_plan(SDXL, variant="serial", steps=T, seed=seed, guidance=w, denoiser=den,
                               clock="model")
    res = hp.run_plan(plan)
    del den, plan
    torch.cuda.empty_cache()
    sch = pipelines.sdxl_schedule(T)
    x_T = hp.initial_latents(pipelines.sdxl_plan(SDXL, variant="serial", steps=T, seed=seed, guidance=w,
                                                 denoiser=object(), clock="model"))
    ref = _RefBranches(UNetRef(SDXL, W), cond, SDXL, T)
    xo, series = oloop.run_exact(ref, x_T, T, w, sch.alpha_bars, sch.sigmas)
    ybr = _RefBranches(UNetRef(SDXL, W, torch.bfloat16), cond, SDXL, T)
    xy, _ = oloop.run_exact(ybr, x_T, T, w, sch.alpha_bars, sch.sigmas)
    mx, mean, _, _ = _report("sdxl1024 50-step x0 (serial, w=5)", torch.from_numpy(res.x0), torch.from_numpy(xo))
    ymx, ymean, _, _ = _report("sdxl1024 50-step x0 [torch bf16 yardstick]", torch.from_numpy(xy),
                               torch.from_numpy(xo))
    m_gpu = np.array([m for _, m in res.series])
    m_ref = np.array([m for _, m in series])
    rel = np.abs(m_gpu - m_ref) / np.abs(m_ref)
    print(f"PARITY sdxl1024 50-step M_t: max rel err {rel.max():.3g}")
    assert [t for t, _ in res.series] == [t for t, _ in series]
    assert mx <= YARD_MAX * ymx and mean <= YARD_MEAN * ymean, (mx, ymx, mean, ymean)
    assert rel.max() <= 2e-2


def test_sdxl1024_hybrid_stage_split_natural_switch_vs_oracle():
    """BASELINE config 2's hybrid plan at full shape with NATURAL slope detection
    (L=12, g=4e-4, k=5, tau_cap=32: the cap calibrated from the network's own
    discrepancy curves, profiles/r02/calibration) and the stage-split window
    (north_star iii), against the CPU-side staged loop (oracle.loop.run_staged,
    pipeline="stage_split") over the fp32 oracle U-Net: the switch schedule (tau1,
    tau2, every step's label, the recorded series keys) must match exactly, and
    the slope margin at the firing step is printed next to the M_t error."""
    from dataclasses import replace
    from oracle import loop as oloop
    from oracle.stage_ref import StagedNet
    from oracle.unet_ref import UNetRef, net_timestep
    from paper_2602_21760_b200.stages import network_fractions, stage_cuts
    T, seed, w = 50, 0, 5.0
    sw = dict(L=12, g_slope=4e-4, tau_cap=32, k=5)
    W, cond = _unet_pair(SDXL)
    den = pipelines.build_sdxl_denoiser(SDXL, n_prompts=1, steps=T, weights=W, conditioning=cond)
    plan = pipelines.sdxl_plan(SDXL, variant="hybrid", steps=T, seed=seed, guidance=w, denoiser=den,
                               clock="model", switch=sw)
    plan = replace(plan, pipeline_numerics="stage_split")
    res = hp.run_plan(plan)
    cuts = stage_cuts(den.net.unit_flops, network_fractions(plan.segment_fractions))
    x_T = hp.initial_latents(plan)
    fr = plan.segment_fractions
    del den, plan
    torch.cuda.empty_cache()
    sch = pipelines.sdxl_schedule(T)
    net = StagedNet(UNetRef(SDXL, W), "unet", cond, SDXL, T, cuts, device="cuda", timestep=net_timestep)
    xo, series, t1, t2, labels = oloop.run_staged(net, x_T, T, w, sch.alpha_bars, sch.sigmas, sw["L"],
                                                  sw["g_slope"], sw["tau_cap"], sw["k"], fr,
                                                  pipeline="stage_split")
    assert t1 is not None and t1 < sw["tau_cap"], "the detector must fire by itself here"
    assert (res.tau1, res.tau2) == (t1, t2), ((res.tau1, res.tau2), (t1, t2))
    assert [s.value for s in res.stages] == labels
    assert [t for t, _ in res.series] == [t for t, _ in series]
    ms = dict(series)
    t_fire = T - t1 + 1
    g = (ms[t_fire] - ms[t_fire + sw["L"]]) / sw["L"]
    m_gpu = np.array([m for _, m in res.series])
    m_ref = np.array([m for _, m in series])
    rel = np.abs(m_gpu - m_ref) / np.abs(m_ref)
    mx, mean, _, _ = _report(f"sdxl1024 hybrid stage_split x0 (tau1={t1}, tau2={t2})", torch.from_numpy(res.x0),
                             torch.from_numpy(xo))
    print(f"PARITY sdxl1024 hybrid natural switch: slope at firing {g:.4g} (g_slope {sw['g_slope']}, "
          f"margin {sw['g_slope'] - g:.3g}), M_t max rel err {rel.max():.3g}")
    assert rel.max() <= 2e-2
    assert mx <= 2.5e-2 and mean <= 5e-3, (mx, mean)


class _RefBranchesDiT:
    """oracle.loop denoiser protocol over MMDiTRef on CUDA (NHWC latents, FM timestep)."""

    def __init__(self, net, cond, spec, T):
        self.net, self.c, self.s, self.T = net, cond, spec, T

    def branches(self, x, t):
        B = x.shape[0]
        hw, ch = self.s.latent_hw, self.s.in_channels
        xt = torch.from_numpy(np.asarray(x)).cuda().float().view(B, hw, hw, ch)
        xt = torch.cat([xt, xt])
        ctx = torch.cat([self.c.context[:B], self.c.null_context.expand(B, -1, -1)])
        pooled = torch.cat([self.c.pooled[:B], self.c.null_pooled.expand(B, -1)])
        tt = torch.full((2 * B,), 1000.0 * t / self.T, device="cuda")
        with torch.no_grad():
            e = self.net(xt, tt, ctx, pooled).reshape(2 * B, -1).double().cpu().numpy()
        return e[:B], e[B:]


def test_sd3_28step_euler_generation_vs_oracle_loop():
    """BASELINE config 3's sampler end to end at full shape: 28 flow-matching Euler steps
    with CFG through run_plan (serial) vs oracle.loop.run_exact(update="euler") over the
    fp32 MMDiT, with the stock-torch bf16 network as the yardstick."""
    from oracle import loop as oloop
    from oracle.mmdit_ref import MMDiTRef
    T, seed, w = 28, 0, 5.0
    s = SD3
    W = init_weights(mmdit_param_specs(s), seed=0, device="cuda")
    cond = synthetic_conditioning(1, s.ctx_len, s.ctx_dim, s.pooled_dim, device="cuda")
    den = pipelines.build_sd3_denoiser(s, n_prompts=1, steps=T, weights=W, conditioning=cond)
    plan = pipelines.sd3_plan(s, variant="serial", steps=T, seed=seed, guidance=w, denoiser=den, clock="model")
    res = hp.run_plan(plan)
    x_T = hp.initial_latents(plan)
    del den, plan
    torch.cuda.empty_cache()
    sch = pipelines.sd3_schedule(T)
    xo, series = oloop.run_exact(_RefBranchesDiT(MMDiTRef(s, W), cond, s, T), x_T, T, w, sch.alpha_bars,
                                 sch.sigmas, update="euler")
    xy, _ = oloop.run_exact(_RefBranchesDiT(MMDiTRef(s, W, torch.bfloat16), cond, s, T), x_T, T, w,
                            sch.alpha_bars, sch.sigmas, update="euler")
    mx, mean, _, _ = _report("sd3 28-step x0 (serial, FM Euler, w=5)", torch.from_numpy(res.x0),
                             torch.from_numpy(xo))
    ymx, ymean, _, _ = _report("sd3 28-step x0 [torch bf16 yardstick]", torch.from_numpy(xy), torch.from_numpy(xo))
    m_gpu = np.array([m for _, m in res.series])
    m_ref = np.array([m for _, m in series])
    rel = np.abs(m_gpu - m_ref) / np.abs(m_ref)
    print(f"PARITY sd3 28-step M_t: max rel err {rel.max():.3g}")
    assert [t for t, _ in res.series] == [t for t, _ in series]
    assert mx <= YARD_MAX * ymx and mean <= YARD_MEAN * ymean, (mx, ymx, mean, ymean)
    assert rel.max() <= 2e-2


def test_sd3_hybrid_stage_split_switch_vs_oracle():
    """BASELINE config 3 at full shape: the SD3 hybrid plan (flow-matching Euler, CFG)
    with the switch calibrated from the network's own discrepancy curves (L=15,
    g=1e-4, k=5, tau_cap=22: profiles/r02/calibration/calibration_sd3.json) and the
    stage-split window, against oracle.loop.run_staged(update="euler",
    pipeline="stage_split") over the fp32 MMDiT: the switch schedule (tau1, tau2,
    every step's label, the recorded series keys) must match exactly."""
    from dataclasses import replace
    from oracle import loop as oloop
    from oracle.mmdit_ref import MMDiTRef
    from oracle.stage_ref import StagedNet
    from paper_2602_21760_b200.stages import network_fractions, stage_cuts
    T, seed, w = 28, 0, 5.0
    sw = dict(L=15, g_slope=1e-4, tau_cap=22, k=5)
    s = SD3
    W = init_weights(mmdit_param_specs(s), seed=0, device="cuda")
    cond = synthetic_conditioning(1, s.ctx_len, s.ctx_dim, s.pooled_dim, device="cuda")
    den = pipelines.build_sd3_denoiser(s, n_prompts=1, steps=T, weights=W, conditioning=cond)
    plan = pipelines.sd3_plan(s, variant="hybrid", steps=T, seed=seed, guidance=w, denoiser=den, clock="model",
                              switch=sw)
    plan = replace(plan, pipeline_numerics="stage_split")
    res = hp.run_plan(plan)
    cuts = stage_cuts(den.net.unit_flops, network_fractions(plan.segment_fractions))
    x_T = hp.initial_latents(plan)
    fr = plan.segment_fractions
    del den, plan
    torch.cuda.empty_cache()
    sch = pipelines.sd3_schedule(T)
    net = StagedNet(MMDiTRef(s, W), "mmdit", cond, s, T, cuts, device="cuda", timestep=lambda t, T_: 1000.0 * t / T_)
    xo, series, t1, t2, labels = oloop.run_staged(net, x_T, T, w, sch.alpha_bars, sch.sigmas, sw["L"],
                                                  sw["g_slope"], sw["tau_cap"], sw["k"], fr, update="euler",
                                                  pipeline="stage_split")
    assert t1 is not None
    assert (res.tau1, res.tau2) == (t1, t2), ((res.tau1, res.tau2), (t1, t2))
    assert [s_.value for s_ in res.stages] == labels
    assert [t for t, _ in res.series] == [t for t, _ in series]
    m_gpu = np.array([m for _, m in res.series])
    m_ref = np.array([m for _, m in series])
    rel = np.abs(m_gpu - m_ref) / np.abs(m_ref)
    mx, mean, _, _ = _report(f"sd3 hybrid stage_split x0 (tau1={t1}, tau2={t2}, "
                             f"{'natural' if t1 < sw['tau_cap'] else 'cap'})", torch.from_numpy(res.x0),
                             torch.from_numpy(xo))
    print(f"PARITY sd3 hybrid: M_t max rel err {rel.max():.3g}")
    assert rel.max() <= 2e-2
    assert mx <= 8e-2 and mean <= 1.5e-2, (mx, mean)
