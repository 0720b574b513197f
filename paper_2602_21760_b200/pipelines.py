"""Ready-made plans for the north-star workloads (BASELINE.json configs).

Each builder returns an ``ExecutionPlan`` whose denoiser is a random-init
network on this package's kernels, plugged in at the reference's seam:

* ``sdxl_plan``  — SDXL-shaped U-Net, 50-step DDIM (scaled-linear VP
  schedule), CFG; configs 1 (tiny, 64^2 latent, 20 steps), 2 (1024^2) and
  4 (2048^2);
* ``sd3_plan``   — SD3-shaped MMDiT, 28-step flow-matching Euler, CFG;
  configs 3 and 5;
* ``build_sdxl_vae`` / ``decode_latents`` — the step after the loop: x0
  latents to 1024^2 pixels with an SDXL-style VAE decoder (no reference
  counterpart; parity against ``oracle/vae_ref.py``).

The latent prior is a mixture with one zero-mean unit-variance component per
prompt (dimension = latent numel), so ``initial_latents`` (engine.py:147-161
semantics, host numpy, seeded) produces x_T exactly as the reference would for
the same plan, and plan validation is the reference's.
"""
from __future__ import annotations

import numpy as np

from .engine import ExecutionPlan, PlanVariant
from .mixture import Condition, GaussianMixture
from .monitor import SwitchConfig
from .schedules import GuidanceParams, build_schedule
from .trace import DeviceSpec, LinkSpec

# per-paper switch parameters, with the stated overrides where
# the preset is infeasible at the config's T
SWITCH = {
    "sdxl": dict(L=12, g_slope=4e-4, tau_cap=15, k=5),
    "tiny": dict(L=4, g_slope=4e-4, tau_cap=8, k=5),
    "sd3": dict(L=15, g_slope=1e-4, tau_cap=22, k=5),
}


def latent_prior(n_prompts: int, numel: int) -> GaussianMixture:
    return GaussianMixture(np.full(n_prompts, 1.0), np.zeros((n_prompts, numel)),
                           np.ones((n_prompts, numel)))


def _devices(variant: PlanVariant, n: int | None, cost: float):
    if n is None:
        n = 1 if variant is PlanVariant.SERIAL else 2
    return tuple(DeviceSpec(f"dev{i}", cost) for i in range(n))


def make_plan(*, variant="serial", denoiser=None, schedule, numel: int, n_prompts=1, seed=0,
              guidance=5.0, switch=None, n_devices=None, clock="device", sampler="ddim",
              branch_cost=0.1649, link=None) -> ExecutionPlan:
    v = PlanVariant(variant)
    staged = v in (PlanVariant.HYBRID, PlanVariant.LAYER_WISE, PlanVariant.BATCH_LEVEL)
    link = link or LinkSpec(float("inf"), 0.0, 4096, 16384)
    sw = SwitchConfig(**switch) if (staged and switch is not None) else None
    return ExecutionPlan(variant=v, schedule=schedule, mixture=latent_prior(n_prompts, numel),
                         conditions=tuple(Condition((i,)) for i in range(n_prompts)),
                         guidance=GuidanceParams(guidance), devices=_devices(v, n_devices, branch_cost),
                         link=link, seed=seed, switch=sw, denoiser=denoiser, clock=clock,
                         sampler=sampler)


def sdxl_schedule(steps: int = 50):
    return build_schedule("scaled-linear", steps, 0.00085, 0.012)


def sd3_schedule(steps: int = 28):
    # the FM Euler loop only consumes t/T; the VP table is carried for the API
    return build_schedule("linear", steps, 0.0005, 0.05)


def build_sdxl_denoiser(spec, n_prompts=1, steps=50, seed=0, use_graph=True, weights=None,
                        conditioning=None):
    import torch
    from .denoiser.adapter import NetDenoiser
    from .denoiser.unet import build_unet
    from .denoiser.weights import synthetic_conditioning
    unet = build_unet(spec, seed=seed, device="cuda", weights=weights)
    cond = conditioning or synthetic_conditioning(n_prompts, spec.context_len, spec.cross_dim,
                                                  spec.pooled_dim)
    conditions = tuple(Condition((i,)) for i in range(n_prompts))
    den = NetDenoiser(unet, cond, conditions, sdxl_schedule(steps),
                      (spec.latent_hw, spec.latent_hw, spec.in_channels), use_graph=use_graph)
    torch.cuda.synchronize()
    return den


def build_sd3_denoiser(spec, n_prompts=1, steps=28, seed=0, use_graph=True, weights=None, conditioning=None):
    import torch
    from .denoiser.adapter import NetDenoiser
    from .denoiser.mmdit import build_mmdit
    from .denoiser.weights import synthetic_conditioning
    net = build_mmdit(spec, seed=seed, device="cuda", weights=weights)
    cond = conditioning or synthetic_conditioning(n_prompts, spec.ctx_len, spec.ctx_dim, spec.pooled_dim)
    conditions = tuple(Condition((i,)) for i in range(n_prompts))
    den = NetDenoiser(net, cond, conditions, sd3_schedule(steps),
                      (spec.latent_hw, spec.latent_hw, spec.in_channels), use_graph=use_graph)
    torch.cuda.synchronize()
    return den


def sd3_plan(spec, *, variant="serial", steps=28, n_prompts=1, seed=0, guidance=5.0, denoiser=None,
             switch_key="sd3", switch=None, **kw) -> ExecutionPlan:
    """SD3-shaped MMDiT, flow-matching Euler (x_1 = x0 + e straight path, engine
    ``sampler="euler"``), CFG; BASELINE configs 3 and 5."""
    if denoiser is None:
        denoiser = build_sd3_denoiser(spec, n_prompts=n_prompts, steps=steps)
    numel = spec.latent_hw * spec.latent_hw * spec.in_channels
    return make_plan(variant=variant, denoiser=denoiser, schedule=sd3_schedule(steps), numel=numel,
                     n_prompts=n_prompts, seed=seed, guidance=guidance, switch=switch or SWITCH[switch_key],
                     sampler="euler", **kw)


def sdxl_plan(spec, *, variant="serial", steps=50, n_prompts=1, seed=0, guidance=5.0,
              denoiser=None, switch_key=None, switch=None, **kw) -> ExecutionPlan:
    if denoiser is None:
        denoiser = build_sdxl_denoiser(spec, n_prompts=n_prompts, steps=steps)
    numel = spec.latent_hw * spec.latent_hw * spec.in_channels
    key = switch_key or ("tiny" if spec.name == "tiny" else "sdxl")
    return make_plan(variant=variant, denoiser=denoiser, schedule=sdxl_schedule(steps), numel=numel,
                     n_prompts=n_prompts, seed=seed, guidance=guidance, switch=switch or SWITCH[key], **kw)


def build_sdxl_vae(spec=None, seed: int = 0, weights=None):
    """Random-init SDXL-style VAE decoder on this package's kernels (the step
    after the loop)."""
    from .denoiser.vae import build_vae
    from .denoiser.weights import VAE_SDXL
    return build_vae(spec or VAE_SDXL, seed=seed, weights=weights)


def decode_latents(vae, x0, latent_hw: int, channels: int = 4):
    """x0 of a RunResult (flat [B, h*w*C] NHWC latents, numpy or torch) -> images
    [B, 8h, 8w, 3] fp32 torch tensor on the GPU."""
    import torch
    x = torch.as_tensor(np.asarray(x0) if not isinstance(x0, torch.Tensor) else x0)
    return vae.decode(x.reshape(-1, latent_hw, latent_hw, channels))
