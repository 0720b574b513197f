"""In-graph time per call SHAPE of one denoiser forward (B=2 CFG batch, or B=1 with
``b1``): the kernel sequence of the captured forward (torch.profiler / CUPTI,
exclusive time as in tools/timeline.py) zipped with the sequence of C-ABI calls
of one eager forward (kernels.check records each call's descriptor), then
aggregated per (call, shape) with FLOPs and achieved TFLOP/s for GEMMs and
attention, sorted by time.

    python tools/timeline_shapes.py [b1] [sd3] [out.txt]
"""
import collections
import re
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2602_21760_b200 import pipelines  # noqa: E402
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402
from paper_2602_21760_b200.denoiser import weights as Wm  # noqa: E402


def flops(desc):
    m = re.match(r"hp_gemm (?:batched (\d+)x )?M=(\d+) N=(\d+) K=(\d+)", desc)
    if m:
        nb = int(m.group(1) or 1)
        return 2.0 * nb * int(m.group(2)) * int(m.group(3)) * int(m.group(4))
    m = re.match(r"hp_gemm upconv n=(\d+) (\d+)x(\d+) (\d+)->(\d+)", desc)
    if m:
        n, h, w, c, co = (int(v) for v in m.groups())
        return 2.0 * n * 4 * h * w * co * 4 * c        # four 2x2 sub-pixel convs at low resolution
    m = re.match(r"hp_attention B=(\d+) H=(\d+) Sq=(\d+) Skv=(\d+)", desc)
    if m:
        b, h, sq, skv = (int(v) for v in m.groups())
        return 4.0 * b * h * sq * skv * 64
    return 0.0


def main():
    b1 = "b1" in sys.argv
    sd3 = "sd3" in sys.argv
    out = [a for a in sys.argv[1:] if a not in ("b1", "sd3")]
    spec = Wm.SD3 if sd3 else Wm.SDXL
    den = (pipelines.build_sd3_denoiser(spec, n_prompts=1, steps=28) if sd3
           else pipelines.build_sdxl_denoiser(spec, n_prompts=1, steps=50))
    x = torch.randn(1, spec.latent_hw * spec.latent_hw * spec.in_channels, device="cuda")
    den.load_input(x)
    run = (lambda: den.conditional(x, 20)) if b1 else (lambda: den.branches(x, 20, den.input_slot()))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    # the call sequence of one forward, eagerly (same kernels in the same order as the graph)
    calls = []
    orig = K.check

    def rec(rc, what):
        calls.append(what)
        return orig(rc, what)
    K.check = rec
    g = den.g_cond if b1 else den.g_both
    g.fn(g.x, g.t)
    torch.cuda.synchronize()
    K.check = orig
    reps = 3
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            run()
        torch.cuda.synchronize()
    evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
                  and e.name and "Memcpy" not in e.name and "Memset" not in e.name
                  and "at::native" not in e.name and "elementwise" not in e.name and "memcpy" not in e.name),
                 key=lambda e: e.time_range.start)
    per = len(evs) // reps
    if per != len(calls):
        print(f"kernel count {per} != call count {len(calls)}: cannot zip")
        print(collections.Counter(e.name[:70] for e in evs[:per]).most_common())
        return
    busy_end = evs[0].time_range.start
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    total = 0.0
    for i, e in enumerate(evs):
        s, t = e.time_range.start, e.time_range.end
        excl = max(0.0, t - max(s, busy_end))
        busy_end = max(busy_end, t)
        d = calls[i % per]
        agg[d][0] += 1
        agg[d][1] += excl
        agg[d][2] = flops(d)
        total += excl
    lines = [f"{'B=1 branch' if b1 else 'B=2 CFG'} forward: {per} calls, busy {total / reps / 1e3:.2f} ms",
             f"{'call':56s} {'n':>4s} {'us each':>8s} {'total us':>9s} {'share':>6s} {'TFLOP/s':>8s}"]
    for d, (c, ex, fl) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        n = c // reps
        each = ex / reps / n
        tf = fl / each / 1e6 if fl else 0.0
        lines.append(f"{d[:56]:56s} {n:4d} {each:8.1f} {ex / reps:9.1f} {100 * ex / total:5.1f}% {tf:8.0f}")
    text = "\n".join(lines)
    print(text)
    if out:
        with open(out[0], "w") as fh:
            fh.write(text + "\n")


if __name__ == "__main__":
    main()
