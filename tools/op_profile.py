"""Per-call timing of the denoiser's kernels (CUDA events around each wrapper
call, eager forward, warm). Prints per-shape achieved TFLOP/s / GB/s and the
time share, to pick the next kernel to optimise.

    python tools/op_profile.py [tiny|sd3]
"""
import collections
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200 import pipelines  # noqa: E402
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402
from paper_2602_21760_b200.denoiser import weights as Wm  # noqa: E402

RECS = []


def wrap(name, fn, flops_fn):
    def inner(*a, **kw):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out = fn(*a, **kw)
        e.record()
        RECS.append((name, s, e, flops_fn(*a, **kw)))
        return out
    return inner


def gemm_key(a, w, **kw):
    conv = kw.get("conv")
    Nn, Kd = w.shape
    if conv is None:
        M = a.numel() // a.shape[-1]
        tag = "lin"
    else:
        n, h, wd, c, st = conv
        M = n * (h // st) * (wd // st)
        tag = f"conv{st}"
    act = kw.get("act", 0)
    return (f"gemm {tag} M={M} N={Nn} K={Kd} act={act}", 2.0 * M * Nn * Kd)


def attn_key(q, k, v, o, **kw):
    B, H, sq, skv = kw["batch"], kw["heads"], kw["sq"], kw["skv"]
    return (f"attn B={B} H={H} sq={sq} skv={skv}", 4.0 * B * H * sq * skv * 64)


def ln_key(x, c, **kw):
    return (f"layernorm rows={x.numel() // c} c={c}", 4.0 * x.numel())   # bytes r+w


def gn_key(x, n, hw, c, *a, **kw):
    return (f"groupnorm n={n} hw={hw} c={c}", 2 * 2.0 * n * hw * c)


def ljoint_key(*a, **kw):
    return ("layer_norm_joint", 0.0)


def main():
    sd3 = "sd3" in sys.argv
    if sd3:
        spec = Wm.SD3
        den = pipelines.build_sd3_denoiser(spec, n_prompts=1, steps=28, use_graph=False)
    else:
        spec = Wm.TINY if "tiny" in sys.argv else Wm.SDXL
        den = pipelines.build_sdxl_denoiser(spec, n_prompts=1, steps=50, use_graph=False)
    K.gemm = wrap("gemm", K.gemm, gemm_key)
    K.attention = wrap("attn", K.attention, attn_key)
    K.layer_norm = wrap("ln", K.layer_norm, ln_key)
    K.group_norm = wrap("gn", K.group_norm, gn_key)
    if hasattr(K, "layer_norm_joint"):
        K.layer_norm_joint = wrap("lnj", K.layer_norm_joint, ljoint_key)
    import paper_2602_21760_b200.denoiser.mmdit as D
    import paper_2602_21760_b200.denoiser.unet as U
    U.K = K
    D.K = K
    x = torch.randn(1, spec.latent_hw * spec.latent_hw * spec.in_channels, device="cuda")
    den.load_input(x)
    for _ in range(2):
        RECS.clear()
        den.branches(x, 30, den.input_slot())
        torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for name, s, e, (key, fl) in RECS:
        ms = s.elapsed_time(e)
        agg[key][0] += 1
        agg[key][1] += ms
        agg[key][2] += fl
    tot = sum(v[1] for v in agg.values())
    print(f"profiled ops: {tot:.2f} ms")
    for key, (c, ms, fl) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        rate = fl / (ms / 1e3) / 1e12
        unit = "TB/s" if key.startswith(("layernorm", "groupnorm")) else "TFLOP/s"
        print(f"{key:58s} x{c:3d} {ms:8.3f} ms {100 * ms / tot:5.1f}%  {rate:7.1f} {unit}")
    _ = (t0, t1)


if __name__ == "__main__":
    main()
