"""Micro-timings of the memory-bound denoiser kernels at SDXL shapes (and an ncu target).

    python tools/prof_misc.py [ln|gn|xattn|all]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402


def bench(name, fn, nbytes=None, flops=None, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / reps * 1e3
    extra = ""
    if nbytes:
        extra += f" {nbytes / us / 1e3:.2f} TB/s"
    if flops:
        extra += f" {flops / us / 1e6:.1f} TFLOP/s"
    print(f"{name:40s} {us:8.2f} us{extra}")


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("ln", "all"):
        for rows, c in ((2048, 1280), (8192, 640)):
            x = torch.randn(rows, c, device="cuda").bfloat16()
            g, b = torch.ones(c, device="cuda"), torch.zeros(c, device="cuda")
            out = torch.empty_like(x)
            bench(f"layernorm {rows}x{c}", lambda: K.layer_norm(x, c, gamma=g, beta=b, out=out), nbytes=4 * x.numel())
    if what in ("gn", "all"):
        for n, hw, c in ((2, 1024, 1280), (2, 16384, 320), (2, 4096, 640)):
            x = torch.randn(n * hw, c, device="cuda").bfloat16()
            g, b = torch.ones(c, device="cuda"), torch.zeros(c, device="cuda")
            out = torch.empty_like(x)
            st = torch.empty(2 * 64 * 64 * 32, device="cuda")
            bench(f"groupnorm n={n} hw={hw} c={c}", lambda: K.group_norm(x, n, hw, c, g, b, silu=True, out=out, stats=st),
                  nbytes=6 * x.numel())
    if what in ("xattn", "all"):
        for S, H, C in ((1024, 20, 1280), (4096, 10, 640)):
            q = torch.randn(2 * S, C, device="cuda").bfloat16()
            kv = torch.randn(2 * 77, 2 * C, device="cuda").bfloat16()
            o = torch.empty_like(q)
            bench(f"xattn S={S} H={H}", lambda: K.attention(q, kv, kv, o, batch=2, heads=H, sq=S, skv=77, scale=0.125,
                                                            k_col0=0, v_col0=C), flops=4.0 * 2 * H * S * 77 * 64)


if __name__ == "__main__":
    main()
