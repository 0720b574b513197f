"""cross-check the measured makespan against the reference
``Timeline`` cost model (trace.py:95-124, engine.py:217-337) fed with costs
measured on this B200.

    python tools/makespan_check.py [out.json]

Measured on one GPU (CUDA events, graph replays): C1 = one branch forward at B=1,
C2 = the CFG-batched B=2 forward, the fused sampler kernel, each stage of the
stage-split network (segment fractions of the layer-wise plans) and the bytes of
each stage boundary. Then:
  * the serial plan runs with ``clock="device"`` (real makespan of 50 steps) and
    with ``clock="model"`` fed C = C1 and the CFG-batching factor rho = C2 / C1:
    the model must reproduce the measured makespan up to the sampler kernels
    and launch gaps it does not model;
  * FCP / hybrid (N=2) and layer-wise stage-split (N=3, 4) makespans are
    predicted by the same model with C = C1 and the NVLink link (770 GB/s
    measured peer copy, an assumed 5 us flag round trip, latent message = the
    bf16 eps, activation message = the measured boundary bytes). A multi-GPU box
    is needed to measure those; the prediction is what the scaling run checks.
"""
import json
import sys
from dataclasses import replace

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200 import engine, pipelines  # noqa: E402
from paper_2602_21760_b200.denoiser.weights import SDXL  # noqa: E402
from paper_2602_21760_b200.stages import network_fractions, stage_cuts  # noqa: E402
from paper_2602_21760_b200.trace import LinkSpec  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/makespan_check.json"
    spec, T = SDXL, 50
    den = pipelines.build_sdxl_denoiser(spec, n_prompts=1, steps=T)
    numel = spec.latent_hw * spec.latent_hw * spec.in_channels
    x = torch.randn(1, numel, device="cuda")
    den.load_input(x)
    c2 = timed(lambda: den.branches(x, 30, den.input_slot()))
    c1 = timed(lambda: den.conditional(x, 30))
    res = {"C1_branch_forward_s": c1, "C2_cfg_batched_forward_s": c2, "rho_measured": c2 / c1}

    # serial: real makespan vs model fed rho = C2 / C1
    dev = engine.run_plan(pipelines.sdxl_plan(spec, variant="serial", steps=T, denoiser=den, clock="device"))
    dev = engine.run_plan(pipelines.sdxl_plan(spec, variant="serial", steps=T, denoiser=den, clock="device"))
    model = engine.run_plan(replace(pipelines.sdxl_plan(spec, variant="serial", steps=T, denoiser=den,
                                                        clock="model", branch_cost=c1),
                                    cfg_batching_factor=c2 / c1))
    res["serial"] = {"measured_makespan_s": dev.latency_s, "model_makespan_s": model.latency_s,
                     "measured_over_model": dev.latency_s / model.latency_s,
                     "unmodelled_per_step_s": (dev.latency_s - model.latency_s) / T}

    # stage-split boundaries: measured per-stage times and message bytes
    stages = {}
    for n in (2, 3, 4):
        fr = tuple([1.0 / n] * n)
        cuts = stage_cuts(den.net.unit_flops, network_fractions(fr))
        den.enable_stage_split(cuts)
        den.window_fill()
        st = [timed(lambda j=j: den.stage_run(j, 30)) for j in range(den.n_stages)]
        nbytes = [int(den.bnd[j].buf.numel() * den.bnd[j].buf.element_size()) for j in range(1, den.n_stages)]
        stages[n] = {"fractions": fr, "cuts": list(cuts), "stage_s": st, "stage_sum_over_C1": sum(st) / c1,
                     "boundary_bytes": nbytes}
    res["stage_split"] = stages

    latent_bytes = numel * 2
    preds = {}
    for name, variant, n in (("fcp_2", "full_condition_partition", 2), ("hybrid_2", "hybrid", 2),
                             ("layer_wise_3", "layer_wise", 3), ("layer_wise_4", "layer_wise", 4)):
        act = max(stages[n]["boundary_bytes"]) if n in stages else latent_bytes
        link = LinkSpec(770e9, 5e-6, latent_bytes, act)
        plan = pipelines.sdxl_plan(spec, variant=variant, steps=T, denoiser=den, clock="model", branch_cost=c1,
                                   n_devices=n, link=link)
        r = engine.run_plan(plan)
        preds[name] = {"model_makespan_s": r.latency_s, "tau1": r.tau1, "tau2": r.tau2,
                       "comm_bytes": r.comm_bytes, "speedup_vs_measured_serial": dev.latency_s / r.latency_s,
                       "link": {"GBps": 770, "base_latency_us": 5, "latent_bytes": latent_bytes,
                                "activation_bytes": act}}
    res["predicted"] = preds
    with open(out, "w") as fh:
        json.dump(res, fh, indent=2)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
