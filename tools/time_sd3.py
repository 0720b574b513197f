"""Timing of the SD3-shaped MMDiT forward (B=2 CFG) and a 28-step Euler run."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_21760_b200 as hp  # noqa: E402
from paper_2602_21760_b200 import pipelines  # noqa: E402
from paper_2602_21760_b200.denoiser import weights as Wm  # noqa: E402
from paper_2602_21760_b200.denoiser.mmdit import mmdit_flops  # noqa: E402


def main():
    prompts = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    spec = Wm.SD3
    t0 = time.time()
    den = pipelines.build_sd3_denoiser(spec, n_prompts=prompts, steps=28)
    print(f"build {time.time() - t0:.1f}s params {Wm.count_params(Wm.mmdit_param_specs(spec)) / 1e9:.3f}B")
    x = torch.randn(prompts, spec.latent_hw * spec.latent_hw * spec.in_channels, device="cuda")
    den.load_input(x)
    for _ in range(3):
        den.branches(x, 20, den.input_slot())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        den.branches(x, 20, den.input_slot())
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    fl = mmdit_flops(spec, 2 * prompts)
    print(f"forward B={2 * prompts}: {ms:.2f} ms, {fl / 1e12:.2f} TFLOP, {fl / ms / 1e9:.1f} TFLOP/s")
    plan = pipelines.sd3_plan(spec, variant="serial", steps=28, n_prompts=prompts, denoiser=den, clock="device")
    hp.run_plan(plan)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hp.run_plan(plan)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"28-step Euler serial, {prompts} prompt(s): {dt:.3f} s, {prompts / dt:.3f} images/s")


if __name__ == "__main__":
    main()
