"""GroupNorm(+SiLU) at the SDXL shapes, back to back inside a CUDA graph."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402
from tools.floor_probe import graph_time  # noqa: E402

for hw, c, c2 in [(16384, 320, 0), (4096, 640, 0), (1024, 1280, 0), (1024, 1280, 1280), (16384, 320, 320)]:
    n = 2
    x = torch.randn(n * hw, c, device="cuda").bfloat16()
    x2 = torch.randn(n * hw, c2, device="cuda").bfloat16() if c2 else None
    g, b = torch.ones(c + c2, device="cuda"), torch.zeros(c + c2, device="cuda")
    out = torch.empty(n * hw, c + c2, device="cuda", dtype=torch.bfloat16)
    st = torch.empty(2 * n * 32 * 256, device="cuda")
    us = graph_time(lambda: K.group_norm(x, n, hw, c, g, b, groups=32, silu=True, x2=x2, c2=c2, out=out, stats=st),
                    reps=20)
    mb = n * hw * (c + c2) * 2 * 3 / 1e6
    print(f"GN n={n} hw={hw} c={c}+{c2}: {us:.1f} us, {mb / us * 1e-3 * 1e3:.2f} TB/s (3 passes of {mb / 3:.1f} MB)")

# the per-step embedding GEMV (all resnets' time-embedding projections in one launch)
xe = torch.randn(2, 1280, device="cuda")
we = (torch.randn(13824, 1280, device="cuda") * 0.03).bfloat16()
ye = torch.empty(2, 13824, device="cuda")
us = graph_time(lambda: K.linear_small(xe, we, None, act_in=K.ACT_SILU, out=ye), reps=20)
print(f"linear_small 2x1280 -> 13824 (silu in): {us:.1f} us, {we.numel() * 2 / us / 1e6:.2f} TB/s")
