"""Run SDXL-shaped U-Net forwards eagerly (no CUDA graph) for ncu launch lists.

    python tools/prof_forward.py [n_forwards] [tiny] [b1]

``b1``: the B=1 conditional-branch forward (one GPU of a condition-partitioned
pair) instead of the B=2 CFG batch.

Prints the number of our kernel launches per forward so ncu's -s can skip the
warm-up forward.
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200 import pipelines  # noqa: E402
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402
from paper_2602_21760_b200.denoiser import weights as Wm  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    spec = Wm.TINY if "tiny" in sys.argv else Wm.SDXL
    den = pipelines.build_sdxl_denoiser(spec, n_prompts=1, steps=50, use_graph=False)
    x = torch.randn(1, spec.latent_hw * spec.latent_hw * 4, device="cuda")
    den.load_input(x)
    for i in range(n):
        before = K.LAUNCHES
        if "b1" in sys.argv:
            den.conditional(x, 30)
        else:
            den.branches(x, 30, den.input_slot())
        torch.cuda.synchronize()
        print(f"forward {i}: {K.LAUNCHES - before} launches", flush=True)


if __name__ == "__main__":
    main()
