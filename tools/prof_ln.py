"""Joint (two-stream) modulated LayerNorm at SD3's shape: graph-timed, for ncu.

    python tools/prof_ln.py [reps]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    n, Ti, L, H = 2, 4096, 333, 1536
    T = Ti + L
    X = torch.randn(n, T, H, device="cuda").bfloat16()
    mods = torch.randn(n, 12 * H, device="cuda")
    ldm = mods.shape[1]
    fn = lambda: K.layer_norm_joint(X, H, T, Ti, mods[:, 0:H], mods[:, H:2 * H], mods[:, 6 * H:7 * H],  # noqa
                                    mods[:, 7 * H:8 * H], ldm)
    fn()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / reps * 1e3
    gb = 2 * X.numel() * 2 / 1e9
    print(f"layer_norm_joint {n}x{T}x{H}: {us:.1f} us, {gb / us * 1e6 / 1e3:.2f} TB/s")


if __name__ == "__main__":
    main()
