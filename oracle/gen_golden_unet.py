"""Golden runs of the REFERENCE engine with the tiny random-init U-Net at its seam.

    PYTHONPATH=/root/reference/pkg/src python -m oracle.gen_golden_unet

BASELINE config 1: tiny U-Net, 64x64x4 latent, 20-step DDIM with CFG, two
simulated ranks. ``hybridpar.engine.eps_prediction`` (imported by name at
engine.py:28) is replaced by ``oracle.unet_ref.SeamAdapter`` (CPU fp32
torch, canonical weights from paper_2602_21760_b200.denoiser.weights with
seed 0), the plan gets a latent-prior mixture (one zero-mean unit-variance
component per prompt, d = 16384) so ``initial_latents`` and validation run
unchanged, and the reference's own ``run_plan`` produces x0 / series / tau.
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"
REF = Path(os.environ.get("HYBRIDPAR_REF", "/root/reference/pkg/src"))

CASES = {
    "serial": dict(variant="serial"),
    "hybrid_cap": dict(variant="hybrid", switch=dict(L=4, g_slope=1e-12, tau_cap=8, k=5)),
    "hybrid_k0": dict(variant="hybrid", switch=dict(L=4, g_slope=1e-12, tau_cap=8, k=0)),
    # natural slope detection on the network's own M_t: fires at s=5 (G=2.2e-3 in [0, 4e-3))
    "hybrid_natural": dict(variant="hybrid", switch=dict(L=4, g_slope=4e-3, tau_cap=8, k=5)),
    # SURVEY 8(d) config-1 parameters: the detector runs every step from s=5 and must NOT
    # fire (G is negative or >= 4e-4 at s=5..7), the cap forces tau1=8
    "hybrid_survey": dict(variant="hybrid", switch=dict(L=4, g_slope=4e-4, tau_cap=8, k=5)),
}
T, GUIDANCE, SEED, PROMPTS = 20, 5.0, 3, 1


def reference_plan(hp, case):
    from paper_2602_21760_b200.denoiser.weights import TINY
    numel = TINY.latent_hw * TINY.latent_hw * TINY.in_channels
    gm = hp.GaussianMixture(np.ones(PROMPTS), np.zeros((PROMPTS, numel)), np.ones((PROMPTS, numel)))
    v = hp.PlanVariant(case["variant"])
    nd = 1 if v is hp.PlanVariant.SERIAL else 2
    sw = hp.SwitchConfig(**case["switch"]) if "switch" in case else None
    return hp.ExecutionPlan(variant=v, schedule=hp.build_schedule("scaled-linear", T, 0.00085, 0.012),
                            mixture=gm, conditions=tuple(hp.Condition((i,)) for i in range(PROMPTS)),
                            guidance=hp.GuidanceParams(GUIDANCE),
                            devices=tuple(hp.DeviceSpec(f"dev{i}", 0.1) for i in range(nd)),
                            link=hp.LinkSpec(float("inf"), 0.0, 4096, 16384), seed=SEED, switch=sw)


def main():
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(ROOT))
    import torch
    import hybridpar as hp
    import hybridpar.engine as eng
    from paper_2602_21760_b200.denoiser.weights import TINY, init_weights, synthetic_conditioning, unet_param_specs
    from oracle.unet_ref import SeamAdapter, UNetRef

    torch.set_num_threads(os.cpu_count() or 8)
    W = init_weights(unet_param_specs(TINY), seed=0, device="cpu")
    cond = synthetic_conditioning(PROMPTS, TINY.context_len, TINY.cross_dim, TINY.pooled_dim)
    adapter = SeamAdapter(UNetRef(TINY, W), cond, TINY.latent_hw, TINY.in_channels)
    eng.eps_prediction = adapter             # the reference's seam (engine.py:28)
    meta, arrays = {}, {}
    for name, case in CASES.items():
        adapter.calls = 0
        res = hp.run_plan(reference_plan(hp, case))
        arrays[name] = res.x0
        meta[name] = {"tau1": res.tau1, "tau2": res.tau2, "calls": adapter.calls,
                      "series": [[int(t), float(m)] for t, m in res.series], **case}
        print(name, res.tau1, res.tau2, adapter.calls, float(np.abs(res.x0).mean()))
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / "unet_tiny.npz", **arrays)
    (OUT / "unet_tiny.json").write_text(json.dumps({"T": T, "guidance": GUIDANCE, "seed": SEED,
                                                     "prompts": PROMPTS, "cases": meta}, indent=1))


if __name__ == "__main__":
    main()
