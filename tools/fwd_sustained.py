"""Back-to-back SDXL forward replays: per-forward time over 10 / 50 / 150 / 10 replays, showing
the burst -> sustained (power-capped) clock transition.

    python tools/fwd_sustained.py
"""
import sys, time, torch
sys.path.insert(0, ".")
from paper_2602_21760_b200 import pipelines
from paper_2602_21760_b200.denoiser import weights as Wm
spec = Wm.SDXL
den = pipelines.build_sdxl_denoiser(spec, n_prompts=1, steps=50)
x = torch.randn(1, spec.latent_hw * spec.latent_hw * 4, device="cuda")
den.load_input(x)
for _ in range(3):
    den.branches(x, 30, den.input_slot())
torch.cuda.synchronize()
for n in (10, 50, 150, 10):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    evs[0].record()
    for i in range(n):
        den.branches(x, 30, den.input_slot())
        evs[i + 1].record()
    torch.cuda.synchronize()
    ts = [evs[i].elapsed_time(evs[i + 1]) for i in range(n)]
    print(f"n={n}: mean {sum(ts)/n:.2f} ms, first5 {[round(t,2) for t in ts[:5]]}, last5 {[round(t,2) for t in ts[-5:]]}")
