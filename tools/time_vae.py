"""Timing of the SDXL VAE decoder (128x128x4 latent -> 1024x1024 RGB) on our kernels."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser.vae import build_vae, vae_decoder_flops  # noqa: E402
from paper_2602_21760_b200.denoiser.weights import VAE_SDXL, count_params, vae_decoder_param_specs  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    t0 = time.time()
    vae = build_vae(VAE_SDXL)
    print(f"build {time.time() - t0:.1f}s params {count_params(vae_decoder_param_specs(VAE_SDXL)) / 1e6:.1f}M")
    z = torch.randn(n, 128, 128, 4, device="cuda") * 0.5
    for _ in range(2):
        vae.decode(z)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    reps = 5
    for _ in range(reps):
        img = vae.decode(z)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    fl = vae_decoder_flops(VAE_SDXL, n)
    print(f"decode n={n} -> {tuple(img.shape)}: {ms:.2f} ms, {fl / 1e12:.2f} TFLOP, {fl / ms / 1e9:.1f} TFLOP/s "
          f"(eager launches)")


if __name__ == "__main__":
    main()
