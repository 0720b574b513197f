"""Fused sampler kernel (K1) timings: bench.sampler_roofline (one launch after an L2
flush, device time) and back-to-back launches in a CUDA graph (warm).

    python tools/sampler_time.py
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2602_21760_b200 as hp  # noqa: E402
from paper_2602_21760_b200 import _kernels as K, _native as N  # noqa: E402


def graph_us(n, reps=50):
    s = hp.build_schedule("scaled-linear", 50, 0.00085, 0.012)
    c = hp.StepCoefficients.ddim(s, 30)
    x = torch.randn(n, device="cuda")
    ec, eu = torch.randn(n, device="cuda").bfloat16(), torch.randn(n, device="cuda").bfloat16()
    out, ob = torch.empty_like(x), torch.empty(n, dtype=torch.bfloat16, device="cuda")
    ws = K.workspace()
    fn = lambda: K.sampler_step(x=x, eps_c=ec, eps_u=eu, x_out=out, x_out_bf16=ob, update=N.HP_UPDATE_DDIM,  # noqa
                                t=30, w=5.0, c_sigma=c.c_sigma, c_sqrt_ab=c.c_sqrt_ab,
                                c_sqrt_ab_prev=c.c_sqrt_ab_prev, c_sqrt_1m_ab_prev=c.c_sqrt_1m_ab_prev, ws=ws)
    fn()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    for v in bench.sampler_roofline(6542.1).values():
        v["graph_warm_us"] = graph_us(v["elements"])
        print(json.dumps({k: round(x, 3) if isinstance(x, float) else x for k, x in v.items()}), flush=True)


if __name__ == "__main__":
    main()
