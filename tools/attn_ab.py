"""Attention A/B: max error vs fp32 SDPA and graph-timed microseconds per shape.

    HP_ATTN_MODE=0|1|2 python tools/attn_ab.py [reps]

Shapes: the SDXL/SD3 self-attention shapes plus a rescale stress case (key
magnitudes growing along the sequence, so the running max moves often).
"""
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402

SHAPES = [(2, 10, 4096, 4096), (2, 20, 1024, 1024), (2, 24, 4429, 4429), (1, 24, 4429, 4429),
          (1, 10, 4096, 4096), (1, 20, 1024, 1024), (2, 3, 333, 333), (2, 2, 256, 256), (1, 2, 16384, 16384)]


def run(B, H, S, SKV, reps, stress=False):
    g = torch.Generator(device="cuda").manual_seed(S + H)
    q = torch.randn(B * S, H * 64, device="cuda", generator=g)
    k = torch.randn(B * SKV, H * 64, device="cuda", generator=g)
    v = torch.randn(B * SKV, H * 64, device="cuda", generator=g)
    if stress:
        k = k * torch.linspace(0.2, 6.0, SKV, device="cuda").repeat(B)[:, None]
    q, k, v = q.bfloat16(), k.bfloat16(), v.bfloat16()
    o = torch.empty_like(q)
    fn = lambda: K.attention(q, k, v, o, batch=B, heads=H, sq=S, skv=SKV, scale=0.125)  # noqa: E731
    fn()
    torch.cuda.synchronize()
    qf = q.float().view(B, S, H, 64).transpose(1, 2)
    kf = k.float().view(B, SKV, H, 64).transpose(1, 2)
    vf = v.float().view(B, SKV, H, 64).transpose(1, 2)
    ref = F.scaled_dot_product_attention(qf, kf, vf, scale=0.125).transpose(1, 2).reshape(B * S, H * 64)
    err = (o.float() - ref).abs().max().item() / (ref.abs().max().item() + 1e-6)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    gr.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / reps * 1e3
    fl = 4.0 * B * H * S * SKV * 64
    return err, us, fl / us / 1e6


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    tag = f"mode={os.environ.get('HP_ATTN_MODE', '0')}"
    for sh in SHAPES:
        err, us, tf = run(*sh, reps)
        print(f"{tag} B={sh[0]} H={sh[1]} S={sh[2]}: err {err:.2e}  {us:8.1f} us  {tf:6.1f} TFLOP/s", flush=True)
    err, us, tf = run(2, 4, 2048, 2048, reps, stress=True)
    print(f"{tag} stress B=2 H=4 S=2048: err {err:.2e}  {us:8.1f} us", flush=True)


if __name__ == "__main__":
    main()
