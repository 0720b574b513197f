"""Sweep block_n over the SDXL U-Net's GEMM / conv shapes (B=2) and compare with the
automatic choice (`pick_bn`); CUDA-graph timing of back-to-back launches.

    python tools/sweep_gemm.py
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402
from tools.floor_probe import graph_time  # noqa: E402

# (label, M, N, K) plain GEMMs and (label, N, (n, h, w, cin, stride)) 3x3 convs of one forward
PLAIN = [
    ("L2 o/q/o-proj", 2048, 1280, 1280), ("L2 qkv", 2048, 3840, 1280), ("L2 ff2", 2048, 1280, 5120),
    ("L2 shortcut", 2048, 1280, 2560), ("L2 shortcut", 2048, 1280, 1920),
    ("L1 proj/o", 8192, 640, 640), ("L1 qkv", 8192, 1920, 640), ("L1 ff2", 8192, 640, 2560),
    ("L1 shortcut", 8192, 640, 1920), ("L1 shortcut", 8192, 640, 1280), ("L1 shortcut", 8192, 640, 960),
    ("L1 shortcut", 8192, 640, 320),
    ("L0 shortcut", 32768, 320, 960), ("L0 shortcut", 32768, 320, 640),
]
CONV = [
    ("L0 conv", 320, (2, 128, 128, 320, 1)), ("L0 conv cat", 320, (2, 128, 128, 640, 1)),
    ("L0 conv cat", 320, (2, 128, 128, 960, 1)), ("L0 down", 320, (2, 128, 128, 320, 2)),
    ("L1 conv", 640, (2, 64, 64, 640, 1)), ("L1 conv in", 640, (2, 64, 64, 320, 1)),
    ("L1 conv cat", 640, (2, 64, 64, 1920, 1)), ("L1 conv cat", 640, (2, 64, 64, 1280, 1)),
    ("L1 conv cat", 640, (2, 64, 64, 960, 1)), ("L1 down", 640, (2, 64, 64, 640, 2)),
    ("L2 conv", 1280, (2, 32, 32, 1280, 1)), ("L2 conv in", 1280, (2, 32, 32, 640, 1)),
    ("L2 conv cat", 1280, (2, 32, 32, 2560, 1)), ("L2 conv cat", 1280, (2, 32, 32, 1920, 1)),
]


def run(label, M, N, Kd, x, conv):
    wt = (torch.randn(N, Kd, device="cuda") * Kd ** -0.5).bfloat16()
    b = torch.randn(N, device="cuda")
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    res = {}
    for bn in (0, 320, 256, 160, 128, 64):
        if bn and N % bn:
            continue
        res[bn] = graph_time(lambda: K.gemm(x, wt, bias=b, out=out, block_n=bn, conv=conv), reps=20)
    best = min((us, bn) for bn, us in res.items() if bn)
    fl = 2.0 * M * N * Kd
    flag = " <-- auto loses {:.0%}".format(res[0] / best[0] - 1) if res[0] > 1.03 * best[0] else ""
    print(f"{label:13s} M={M:6d} N={N:5d} K={Kd:6d} auto {res[0]:7.1f} us {fl / res[0] / 1e6:6.0f} TF/s | best "
          f"bn={best[1]:3d} {best[0]:7.1f} us | " + " ".join(f"{bn}:{us:.1f}" for bn, us in res.items() if bn) + flag)


def main():
    for label, M, N, Kd in PLAIN:
        run(label, M, N, Kd, torch.randn(M, Kd, device="cuda").bfloat16(), None)
    for label, N, conv in CONV:
        n, h, w, c, st = conv
        run(label, n * (h // st) * (w // st), N, 9 * c, torch.randn(n * h * w, c, device="cuda").bfloat16(), conv)


if __name__ == "__main__":
    main()
