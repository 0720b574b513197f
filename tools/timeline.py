"""In-graph kernel timeline of the SDXL U-Net forward (B=2) via torch.profiler (CUPTI):
warm per-kernel durations as they run inside the CUDA graph with PDL overlap, unlike
ncu's serialised cold replays. Prints the per-kernel share and the gap (idle) time.

    python tools/timeline.py [out.txt]
"""
import collections
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2602_21760_b200 import pipelines  # noqa: E402
from paper_2602_21760_b200.denoiser import weights as Wm  # noqa: E402


def short(name):
    name = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    return name.split("(")[0][:60]


def main():
    spec = Wm.SDXL
    den = pipelines.build_sdxl_denoiser(spec, n_prompts=1, steps=50)
    x = torch.randn(1, spec.latent_hw * spec.latent_hw * 4, device="cuda")
    den.load_input(x)
    for _ in range(3):
        den.branches(x, 30, den.input_slot())
    torch.cuda.synchronize()
    reps = 3
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            den.branches(x, 30, den.input_slot())
        torch.cuda.synchronize()
    evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
                  and e.name and "Memcpy" not in e.name and "Memset" not in e.name),
                 key=lambda e: e.time_range.start)
    if not evs:
        print("no CUDA kernel events recorded")
        return
    span = (evs[-1].time_range.end - evs[0].time_range.start) / reps
    # exclusive time: a kernel owns [max(its start, the previous kernel's end), its end] -- with
    # PDL a kernel's CTAs start (and wait) while its predecessor drains, so raw durations overlap
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    busy_end, busy = evs[0].time_range.start, 0.0
    for e in evs:
        k = short(e.name)
        s, t = e.time_range.start, e.time_range.end
        excl = max(0.0, t - max(s, busy_end))
        agg[k][0] += 1
        agg[k][1] += excl
        agg[k][2] += e.time_range.elapsed_us()
        busy += excl
        busy_end = max(busy_end, t)
    lines = [f"{len(evs) // reps} kernels per forward, {span / 1e3:.2f} ms per forward (first start to last end), "
             f"GPU busy {busy / reps / 1e3:.2f} ms ({100 * busy / reps / span:.1f}%; the rest is idle between "
             f"kernels)", f"{'kernel':62s} {'n':>5s} {'exclusive':>12s} {'share':>6s} {'raw (overlapping)':>18s}"]
    for k, (c, ex, raw) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:62s} {c // reps:5d} {ex / reps:9.1f} us {100 * ex / busy:5.1f}% {raw / reps:12.1f} us")
    text = "\n".join(lines)
    print(text)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(text + "\n")


if __name__ == "__main__":
    main()
