"""Quick timing of one SDXL-shaped U-Net forward (B=2) and the 50-step serial loop.

Development tool (not the bench): prints per-forward ms, achieved TFLOP/s,
and the top-level time split.
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200 import pipelines  # noqa: E402
from paper_2602_21760_b200.denoiser.unet import unet_flops  # noqa: E402
from paper_2602_21760_b200.denoiser import weights as Wm  # noqa: E402
import paper_2602_21760_b200 as hp  # noqa: E402


def main():
    spec = Wm.TINY if "tiny" in sys.argv else Wm.SDXL
    t0 = time.time()
    den = pipelines.build_sdxl_denoiser(spec, n_prompts=1, steps=50)
    print(f"build {time.time() - t0:.1f}s params {Wm.count_params(Wm.unet_param_specs(spec)) / 1e9:.3f}B")
    x = torch.randn(1, spec.latent_hw * spec.latent_hw * 4, device="cuda")
    den.load_input(x)
    for _ in range(3):
        den.branches(x, 30, den.input_slot())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 10
    for _ in range(n):
        den.branches(x, 30, den.input_slot())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    fl = unet_flops(spec, 2)
    print(f"forward B=2: {ms:.2f} ms, {fl / 1e12:.2f} TFLOP, {fl / ms / 1e9:.1f} TFLOP/s")
    plan = pipelines.sdxl_plan(spec, variant="serial", steps=50, denoiser=den)
    hp.run_plan(plan)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = hp.run_plan(plan)
    torch.cuda.synchronize()
    print(f"50-step serial: {time.perf_counter() - t0:.3f} s wall, latency_s {res.latency_s:.3f}")


if __name__ == "__main__":
    main()
