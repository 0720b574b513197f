"""GroupNorm from producer partials (hp_group_norm_parts) vs the statistics-pass GroupNorm
(hp_group_norm) at the SDXL shapes, warm, in CUDA graphs of 20 launches (us per launch).

    python tools/gn_parts_time.py
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402

SHAPES = [(2, 1024, 1280), (2, 4096, 640), (2, 16384, 320), (2, 16384, 960), (2, 1024, 2560), (1, 1024, 1280)]


def graph_us(fn, reps=20):
    fn()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (5 * reps)


def main():
    for n, hw, c in SHAPES:
        x = torch.randn(n * hw, 320, device="cuda").bfloat16()
        w = (torch.randn(c, 320, device="cuda") * 320 ** -0.5).bfloat16()
        y = K.gemm(x, w, gn_hw=hw)
        gp = y.hp_gn
        g, b = torch.randn(c, device="cuda"), torch.randn(c, device="cuda")
        out = torch.empty_like(y)
        st = torch.empty(2 * 64 * 64 * 32, dtype=torch.float32, device="cuda")
        t_parts = graph_us(lambda: K.group_norm(y, n, hw, c, g, b, silu=True, out=out, stats=st))
        y.hp_gn = None
        t_two = graph_us(lambda: K.group_norm(y, n, hw, c, g, b, silu=True, out=out, stats=st))
        y.hp_gn = gp
        mb = 2 * n * hw * c * 2 / 1e6
        print(f"n={n} hw={hw} C={c}: parts {t_parts:6.2f} us ({mb / t_parts:5.2f} TB/s)   stats-pass {t_two:6.2f} us")


if __name__ == "__main__":
    main()
