"""Per-launch floor of back-to-back PDL kernels inside one CUDA graph."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402


def graph_time(fn, reps=100):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


if __name__ == "__main__":
    x = torch.randn(256, device="cuda").bfloat16()
    print(f"silu 256 elems: {graph_time(lambda: K.silu(x, out=x)):.2f} us/launch")
    a = torch.randn(128, 64, device="cuda").bfloat16()
    w = torch.randn(64, 64, device="cuda").bfloat16()
    o = torch.empty(128, 64, device="cuda", dtype=torch.bfloat16)
    print(f"gemm 128x64x64: {graph_time(lambda: K.gemm(a, w, out=o)):.2f} us/launch")
    a2 = torch.randn(2048, 64, device="cuda").bfloat16()
    w2 = torch.randn(1280, 64, device="cuda").bfloat16()
    o2 = torch.empty(2048, 1280, device="cuda", dtype=torch.bfloat16)
    print(f"gemm 2048x1280x64: {graph_time(lambda: K.gemm(a2, w2, out=o2)):.2f} us/launch")
