"""Run the attention kernel at SDXL shapes (for ncu captures and quick timing).

    python tools/prof_attn.py [S] [H] [reps] [SKV]

Timed inside a CUDA graph of ``reps`` launches (no host launch overhead).
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    SKV = int(sys.argv[4]) if len(sys.argv) > 4 else S
    B = 2
    q = torch.randn(B * S, H * 64, device="cuda").bfloat16()
    kv = torch.randn(B * SKV, 2 * H * 64, device="cuda").bfloat16()
    o = torch.empty(B * S, H * 64, device="cuda", dtype=torch.bfloat16)
    run = lambda: K.attention(q, kv, kv, o, batch=B, heads=H, sq=S, skv=SKV, scale=0.125,  # noqa: E731
                              q_col0=0, k_col0=0, v_col0=H * 64)
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            run()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    fl = 4.0 * B * H * S * SKV * 64
    print(f"attn B={B} H={H} S={S} SKV={SKV}: {ms * 1e3:.1f} us  {fl / ms / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
