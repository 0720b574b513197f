"""Run the attention kernel at SDXL shapes (for ncu captures and quick timing).

    python tools/prof_attn.py [S] [H] [reps]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    B = 2
    qkv = torch.randn(B * S, 3 * H * 64, device="cuda").bfloat16()
    o = torch.empty(B * S, H * 64, device="cuda", dtype=torch.bfloat16)
    run = lambda: K.attention(qkv, qkv, qkv, o, batch=B, heads=H, sq=S, skv=S, scale=0.125,  # noqa: E731
                              q_col0=0, k_col0=H * 64, v_col0=2 * H * 64)
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    fl = 4.0 * B * H * S * S * 64
    print(f"attn B={B} H={H} S={S}: {ms * 1e3:.1f} us  {fl / ms / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
