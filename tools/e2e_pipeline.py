"""End to end on one B200: token ids -> SDXL text encoders -> 50-step CFG loop
(U-Net, hybrid-capable plan) -> VAE decoder -> 1024^2 pixels. Random-init
weights everywhere (no checkpoints in this environment); times each stage.

    python tools/e2e_pipeline.py [n_prompts]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_21760_b200 as hp  # noqa: E402
from paper_2602_21760_b200 import pipelines  # noqa: E402
from paper_2602_21760_b200.denoiser.text_encoders import build_text_encoders  # noqa: E402
from paper_2602_21760_b200.denoiser.weights import SDXL  # noqa: E402


def timed(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    print(f"{label}: {1e3 * (time.perf_counter() - t0):.1f} ms")
    return out


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    enc = build_text_encoders()
    vae = pipelines.build_sdxl_vae()
    g = torch.Generator().manual_seed(0)
    ids = torch.randint(1, 49406, (n, 77), generator=g)
    ids[:, 20:] = 0
    ids[:, 20] = 49407                                             # EOS
    null = torch.zeros(1, 77, dtype=torch.int64)
    null[0, 0], null[0, 1] = 49406, 49407                          # BOS, EOS
    enc.conditioning(ids, null)                                    # warm-up
    cond = timed("text encoders (ViT-L + bigG, prompts + null)", lambda: enc.conditioning(ids, null))
    den = pipelines.build_sdxl_denoiser(SDXL, n_prompts=n, steps=50, conditioning=cond)
    plan = pipelines.sdxl_plan(SDXL, variant="serial", steps=50, n_prompts=n, denoiser=den, clock="device")
    hp.run_plan(plan)
    res = timed("50-step CFG loop", lambda: hp.run_plan(plan))
    pipelines.decode_latents(vae, res.x0, SDXL.latent_hw)
    img = timed("VAE decode", lambda: pipelines.decode_latents(vae, res.x0, SDXL.latent_hw))
    print(f"images {tuple(img.shape)}, mean {img.mean().item():.4f}, std {img.std().item():.4f}")


if __name__ == "__main__":
    main()
