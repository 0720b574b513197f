"""Sweep block_n over the SDXL GEMM / conv shapes; prints the best per shape."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402

SHAPES = [  # (M, N, K, conv(n,h,w,c,stride) or None)
    (2048, 1280, 1280, None), (2048, 3840, 1280, None), (2048, 1280, 5120, None), (154, 2560, 2048, None),
    (8192, 640, 640, None), (8192, 1920, 640, None), (8192, 640, 2560, None), (32768, 320, 640, None),
    (None, 320, None, (2, 128, 128, 320, 1)), (None, 640, None, (2, 64, 64, 640, 1)),
    (None, 1280, None, (2, 32, 32, 1280, 1)), (None, 640, None, (2, 64, 64, 320, 1)),
    (None, 320, None, (2, 128, 128, 640, 1)), (None, 1280, None, (2, 32, 32, 2560, 1)),
    (None, 320, None, (2, 128, 128, 320, 2)), (None, 640, None, (2, 64, 64, 640, 2)),
]


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main():
    for M, N, Kd, conv in SHAPES:
        if conv is not None:
            n, h, w, c, st = conv
            x = torch.randn(n, h, w, c, device="cuda").bfloat16()
            Kd = 9 * c
            M = n * (h // st) * (w // st)
        else:
            x = torch.randn(M, Kd, device="cuda").bfloat16()
        wt = (torch.randn(N, Kd, device="cuda") * Kd ** -0.5).bfloat16()
        b = torch.randn(N, device="cuda")
        res = []
        for bn in (64, 128, 160, 256):
            if N % bn:
                continue
            us = t(lambda: K.gemm(x, wt, bias=b, block_n=bn, conv=conv))
            res.append((us, bn))
        auto = int(K.N.load().hp_gemm_pick_block_n(M, N, 0))
        best = min(res)
        fl = 2.0 * M * N * Kd
        print(f"M={M:6d} N={N:5d} K={Kd:6d} conv={conv is not None} best bn={best[1]:3d} {best[0]:7.1f} us "
              f"{fl / best[0] / 1e6:7.1f} TF/s | auto={auto} | " + " ".join(f"{bn}:{us:.1f}" for us, bn in res))


if __name__ == "__main__":
    main()
