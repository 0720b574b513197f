"""Benchmark: SDXL 1024^2 50-step CFG latency (s/image) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One bench "step" is one complete 50-step classifier-free-guided generation of
one 1024^2 image (128x128x4 latent) with a random-init SDXL-shaped U-Net
(2.57 B parameters) on this package's sm_100a kernels, driven through the
drop-in ``run_plan`` API. At N=1 the plan is ``serial`` (both guidance
branches on one GPU, batched); at N>1 each GPU pair runs one image with the
hybrid plan (``--mode pairs``, the default: condition partitioning with the
branch exchange fused into the sampler kernel over NVLink) or every GPU runs
its own image (``--mode replicas``). A failed run on any rank makes every rank
agree and exit non-zero with an ``error`` line (no silent change of mode).

Printed JSON (rank 0, one line): ``value`` = device-resident seconds per image
(latency: each group generates one image per bench step, so the timed region /
K; max over ranks); ``throughput_images_per_s`` = all images / timed region;
``e2e`` = the same latency through the public API with host x_T in and host x0
out each run; ``roofline`` = the denoiser forward the GPU runs (B=2 at N=1, B=1
per GPU in pairs) against MEASURED_PEAKS.json; ``forward_b1`` = the B=1 branch
forward, the reference's sequential rho=2 one-GPU latency built from it and the
predicted pair latency; ``sampler_roofline`` = the fused exchange+CFG+DDIM
kernel (HBM-bound); ``cpu_baseline`` = the oracle CPU path (fp32 torch U-Net +
numpy sampler) on this host over whole denoising steps, x50.

``--impl reference`` times the reference's CPU implementation of the path
(the oracle port: numpy fp64 sampler trio of schedules.py / monitor.py plus the
fp32 torch network at the seam, all host threads) on the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SDXL 1024^2 50-step latency (s/image)"
UNIT = "s/image"
STEPS_T = 50


class Workload:
    """One BASELINE.json config as a bench workload (``--spec``): the network spec,
    steps, builders and analytic FLOPs."""

    def __init__(self, key):
        from paper_2602_21760_b200 import pipelines
        from paper_2602_21760_b200.denoiser import weights as Wm
        self.key = key
        self.dit = key == "sd3"
        self.spec = {"sdxl": Wm.SDXL, "sdxl2048": Wm.SDXL_2048, "tiny": Wm.TINY, "sd3": Wm.SD3}[key]
        self.T = {"sdxl": 50, "sdxl2048": 50, "tiny": 20, "sd3": 28}[key]
        self.build = pipelines.build_sd3_denoiser if self.dit else pipelines.build_sdxl_denoiser
        self.plan = pipelines.sd3_plan if self.dit else pipelines.sdxl_plan
        px = {"sdxl": "1024^2", "sdxl2048": "2048^2", "tiny": "tiny 64x64-latent", "sd3": "1024^2"}[key]
        net = "SD3" if self.dit else "SDXL"
        self.metric = METRIC if key == "sdxl" else f"{net} {px} {self.T}-step latency (s/image)"
        self.name = {"sdxl": "sdxl-1024-50step-cfg", "sdxl2048": "sdxl-2048-50step-cfg", "tiny": "tiny-unet-20step-cfg",
                     "sd3": "sd3-1024-28step-fm-euler-cfg"}[key]
        self.sampler = "flow-matching Euler" if self.dit else "DDIM"

    @property
    def params(self) -> int:
        """Parameter count of the network (analytic, from its parameter specs)."""
        import math
        from paper_2602_21760_b200.denoiser.weights import mmdit_param_specs, unet_param_specs
        specs = mmdit_param_specs(self.spec) if self.dit else unet_param_specs(self.spec)
        return sum(math.prod(shape) for _, shape, _ in specs)

    def flops(self, n):
        if self.dit:
            from paper_2602_21760_b200.denoiser.mmdit import mmdit_flops
            return mmdit_flops(self.spec, n)
        from paper_2602_21760_b200.denoiser.unet import unet_flops
        return unet_flops(self.spec, n)

    @property
    def latent(self):
        return [self.spec.latent_hw, self.spec.latent_hw, self.spec.in_channels]


def _forward_traffic():
    """DRAM bytes of one forward from the committed ncu launch list (profiles/):
    dram__bytes_read.sum + dram__bytes_write.sum summed over the forward's kernels."""
    path = os.path.join(ROOT, "profiles", "r02", "bench_r2d_traffic.json")   # ncu pass over bench.py itself
    try:
        with open(path) as fh:
            t = json.load(fh)
        return {"traffic": t["dram_bytes"], "traffic_unit": "bytes per forward",
                "traffic_source": os.path.relpath(path, ROOT) + " (ncu replay, cold caches per kernel: upper bound)"}
    except Exception:
        return {"traffic": None}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([s.strip() for s in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def _max_over_ranks(ws, v):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------------
def cpu_reference_sample(wl, n_steps: int = 2, threads: int | None = None, weights=None):
    """Oracle CPU path on this host, timed over ``n_steps`` whole denoising steps of the
    reference's serial runner (engine.py:195-214 with config.py:174 rho=2): per step the
    fp32 torch network (U-Net or MMDiT restatement) evaluates the conditional and then
    the unconditional branch (B=1 each, sequentially) and the numpy fp64 trio (rel_mae,
    cfg, ddim / fm-euler) updates the latent. Returns (s/image = T x the measured mean
    step, details)."""
    import torch
    from oracle import sampler as osmp
    from paper_2602_21760_b200.denoiser.weights import (init_weights, mmdit_param_specs, synthetic_conditioning,
                                                         unet_param_specs)
    spec, T = wl.spec, wl.T
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    t0 = time.perf_counter()
    if weights is None:
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        specs = mmdit_param_specs(spec) if wl.dit else unet_param_specs(spec)
        weights = {k: v.cpu() for k, v in init_weights(specs, seed=0, device=dev).items()}
    init_s = time.perf_counter() - t0
    hw, c = spec.latent_hw, spec.in_channels
    if wl.dit:
        from oracle.mmdit_ref import MMDiTRef
        net = MMDiTRef(spec, weights)
        cond = synthetic_conditioning(1, spec.ctx_len, spec.ctx_dim, spec.pooled_dim)
        fwd_in = lambda xn, tt, ctx, pool: net(xn.reshape(1, hw, hw, c), tt, ctx, pool)  # noqa: E731
    else:
        from oracle.unet_ref import UNetRef
        net = UNetRef(spec, weights)
        cond = synthetic_conditioning(1, spec.context_len, spec.cross_dim, spec.pooled_dim)
        fwd_in = lambda xn, tt, ctx, pool: net(xn.reshape(1, c, hw, hw), tt, ctx, pool)  # noqa: E731
    _, _, abar, sig = osmp.schedule_tables("scaled-linear", T, 0.00085, 0.012)
    g = torch.Generator().manual_seed(0)
    x = torch.randn(1, hw * hw * c, generator=g).double().numpy()
    steps, fwd = [], []
    with torch.no_grad():
        for i in range(n_steps):
            t = T - i
            t1 = time.perf_counter()
            xt = torch.from_numpy(x).float()
            tt = torch.tensor([float(t * (1000 // T))])
            ec = fwd_in(xt, tt, cond.context, cond.pooled).double().numpy().reshape(1, -1)
            t2 = time.perf_counter()
            eu = fwd_in(xt, tt, cond.null_context, cond.null_pooled).double().numpy().reshape(1, -1)
            fwd.append(time.perf_counter() - t2)
            fwd.append(t2 - t1)
            m = osmp.rel_mae(ec, eu)
            e = osmp.cfg(ec, eu, 5.0)
            x = osmp.euler(x, e, 1.0 / T) if wl.dit else osmp.ddim(x, e, t, abar, sig)
            steps.append(time.perf_counter() - t1)
    step = sum(steps) / len(steps)
    return T * step, {"step_s": step, "forward_s": min(fwd), "steps_measured": n_steps, "threads": threads,
                      "weight_init_s": init_s, "m": float(np.asarray(m).ravel()[0])}


def run_reference_arm(args):
    ws, rank, local = _dist()
    if rank != 0:
        return 0
    import torch
    wl = Workload("sdxl")
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    from paper_2602_21760_b200.denoiser.weights import init_weights, unet_param_specs
    weights = {k: v.cpu() for k, v in init_weights(unet_param_specs(wl.spec), seed=0, device=dev).items()}
    vals = []
    for i in range(args.warmup + args.steps):
        v, det = cpu_reference_sample(wl, 1, weights=weights)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    sample = (f"per bench step: one whole denoising step of the reference serial runner on the host cores "
              f"(fp32 SDXL-shaped U-Net, conditional then unconditional branch at B=1, numpy fp64 "
              f"rel_mae/cfg/ddim at N=65536), x{STEPS_T} steps per image")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": {"workload": "sdxl-1024-50step-cfg", "latent": [128, 128, 4], "T": STEPS_T,
                       "parallelism": "cpu"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": det["threads"], "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------
def sampler_roofline(hbm_peak):
    """Time the fused CFG+DDIM+rel-MAE kernel at the SDXL latent size (both
    branches of one image: 65,536 elements) and at 2^26 elements."""
    import torch
    import paper_2602_21760_b200 as hp
    from paper_2602_21760_b200 import _kernels as K, _native as N
    s = hp.build_schedule("scaled-linear", 50, 0.00085, 0.012)
    c = hp.StepCoefficients.ddim(s, 30)
    res = {}
    for n in (65536, 1 << 22, 1 << 26):
        x = torch.randn(n, device="cuda")
        ec = torch.randn(n, device="cuda").bfloat16()
        eu = torch.randn(n, device="cuda").bfloat16()
        out = torch.empty_like(x)
        ob = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        ws = K.workspace()

        # the exchange-fused form: eps_u sits behind a flag word (system-scope acquire
        # by one thread per CTA before any CTA reads it). On one GPU the flag is
        # pre-released and eps_u is local, so this times the acquire + the fused read
        # path; the NVLink leg is bounded by the model below.
        flag = torch.ones(1, dtype=torch.int32, device="cuda")

        def launch(fused=False):
            K.sampler_step(x=x, eps_c=ec, eps_u=eu, x_out=out, x_out_bf16=ob, update=N.HP_UPDATE_DDIM, t=30,
                           w=5.0, c_sigma=c.c_sigma, c_sqrt_ab=c.c_sqrt_ab, c_sqrt_ab_prev=c.c_sqrt_ab_prev,
                           c_sqrt_1m_ab_prev=c.c_sqrt_1m_ab_prev, ws=ws,
                           wait_flag=flag if fused else None, wait_value=1 if fused else 0)
        for _ in range(5):
            launch()
            launch(True)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

        def cold(fused):
            times = []
            for _ in range(20):
                flush.zero_()                                # evict L2 (> 126 MB)
                torch.cuda._sleep(100000)                    # GPU busy while the host enqueues: device time only
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                launch(fused)
                b.record()
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b) / 1e3)
            return statistics.median(times)
        t, tf = cold(False), cold(True)
        bytes_ = 14 * n       # x f32 in + eps_c, eps_u bf16 + x f32 out + x bf16 out
        # fused over NVLink: 12 n local HBM bytes + 2 n peer bytes
        nvl_bound = max(12 * n / (hbm_peak * 1e9), 2 * n / 900e9)
        res[n] = {"elements": n, "us": t * 1e6, "algorithmic_bytes": bytes_, "gbs": bytes_ / t / 1e9,
                  "frac": bytes_ / t / 1e9 / hbm_peak,
                  "fused_flag_us": tf * 1e6, "fused_flag_frac": bytes_ / tf / 1e9 / hbm_peak,
                  "fused_nvlink_bound_us": nvl_bound * 1e6}
    return res


def _graph_time(run, reps):
    import torch
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        run()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def forward_roofline(den, wl, reps=20):
    """Back-to-back replays of the CFG-batched (both branches, all prompts) forward graph."""
    import torch
    spec = wl.spec
    x = torch.randn(den.B, spec.latent_hw * spec.latent_hw * spec.in_channels, device="cuda")
    den.load_input(x)
    t = _graph_time(lambda: den.branches(x, min(wl.T - 1, 30), den.input_slot()), reps)
    return t, wl.flops(2 * den.B)


def forward_b1(den, wl, reps=20):
    """Back-to-back replays of the B=1 conditional-branch forward graph: the work one GPU
    of a condition-partitioned pair does per step, and half of the reference serial
    runner's rho=2 step (engine.py:195-214, config.py:174: branches evaluated in turn)."""
    import torch
    spec = wl.spec
    x = torch.randn(den.B, spec.latent_hw * spec.latent_hw * spec.in_channels, device="cuda")
    t = _graph_time(lambda: den.conditional(x, min(wl.T - 1, 30)), reps)
    return t, wl.flops(den.B)


def top_kernel_rooflines(bf16_peak, reps=20):
    """The step's dominant kernels (profiles/r02/timeline_shapes_b2.txt: GEGLU GEMM 15%,
    self-attention S=1024 9% + S=4096 8%) at their SDXL shapes, each timed live with CUDA
    events around a CUDA graph of `reps` back-to-back launches on the launching stream
    (inputs L2-resident between launches: a per-kernel ceiling, not the in-step rate)."""
    import torch
    from paper_2602_21760_b200.denoiser import kernels as K

    def graph_us(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
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

    out = []
    for S, H, n in ((4096, 10, 10), (1024, 20, 60)):       # level 1 / level 2 self-attention, launches per step
        q = torch.randn(2 * S, H * 64, device="cuda").bfloat16()
        kv = torch.randn(2 * S, 2 * H * 64, device="cuda").bfloat16()
        o = torch.empty_like(q)
        us = graph_us(lambda: K.attention(q, kv, kv, o, batch=2, heads=H, sq=S, skv=S, scale=0.125,
                                          q_col0=0, k_col0=0, v_col0=H * 64))
        fl = 4.0 * 2 * H * S * S * 64
        scores = 2.0 * H * S * S
        # MUFU bound: 6 of 8 exp2 pairs on MUFU.EX2 (16 / clk / SM at 1965 MHz); softmax bound:
        # the kernel's softmax instruction stream alone, 13.2 scores / clk / SM measured on B200
        # (tools/micro/softmax_rate.cu), with perfect balance over the 148 SMs
        mufu_us = scores * 6 / 8 / (16 * 148 * 1.965e9) * 1e6
        soft_us = scores / (13.2 * 148 * 1.965e9) * 1e6
        out.append({"kernel": f"attn_stream S={S} H={H} B=2 (x{n} per step)", "flops_per_launch": fl,
                    "us": us, "achieved": fl / us / 1e6, "frac": fl / us / 1e6 / bf16_peak,
                    "mufu_bound_us": mufu_us, "frac_of_mufu_bound": mufu_us / us,
                    "softmax_bound_us": soft_us, "frac_of_softmax_bound": soft_us / us})
    M, N, Kd = 2048, 10240, 1280                                # level-2 GEGLU (x60 per step)
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    w = (torch.randn(N, Kd, device="cuda") * Kd ** -0.5).bfloat16()
    y = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
    us = graph_us(lambda: K.gemm(a, w, out=y, act=K.ACT_GEGLU))
    fl = 2.0 * M * N * Kd
    out.append({"kernel": f"gemm_pair GEGLU {M}x{N}x{Kd} (x60 per step)", "flops_per_launch": fl, "us": us,
                "achieved": fl / us / 1e6, "frac": fl / us / 1e6 / bf16_peak})
    return out


def time_replicas(args, wl, ws, rank, local):
    """Every GPU generates its own images (``--prompts`` per run, one CFG batch) with
    the serial plan."""
    import torch
    import paper_2602_21760_b200 as hp
    den = wl.build(wl.spec, n_prompts=args.prompts, steps=wl.T, seed=rank)
    plan = wl.plan(wl.spec, variant="serial", steps=wl.T, n_prompts=args.prompts, seed=rank, denoiser=den,
                   clock="device")
    for _ in range(args.warmup):
        hp.run_plan(plan)
    torch.cuda.synchronize()
    x_host = hp.initial_latents(plan)
    x_dev = torch.from_numpy(x_host).cuda()
    clocks = ClockSampler(local)
    with clocks:
        _barrier(ws)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            hp.engine.run_plan_resident(plan, x_dev)
        b.record()
        torch.cuda.synchronize()
        _barrier(ws)
    dev_s = _max_over_ranks(ws, a.elapsed_time(b) / 1e3)
    _barrier(ws)
    torch.cuda.synchronize()
    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2.record()
    last = None
    for _ in range(args.steps):
        last = hp.run_plan(plan)
    b2.record()
    torch.cuda.synchronize()
    _barrier(ws)
    e2e_s = _max_over_ranks(ws, a2.elapsed_time(b2) / 1e3)
    h2d = int(x_host.nbytes)
    d2h = int(last.x0.nbytes) + 16 * len(last.series)
    return den, dev_s, args.steps * ws * args.prompts, e2e_s, h2d, d2h, clocks, 1


def time_pairs(args, wl, ws, rank, local):
    """Condition-partitioned pairs over NVLink: ranks (2p, 2p+1) generate one image
    together with the hybrid plan (cond / uncond branch per GPU, fused exchange)."""
    import torch
    import torch.distributed as dist
    import paper_2602_21760_b200 as hp
    from paper_2602_21760_b200 import parallel, pipelines
    if ws % 2:
        raise RuntimeError(f"pairs mode needs an even GPU count, got {ws}")
    groups = [dist.new_group([2 * p, 2 * p + 1]) for p in range(ws // 2)]
    role = parallel.pair_role(rank)
    den = wl.build(wl.spec, n_prompts=args.prompts, steps=wl.T, seed=0)   # same weights in a pair
    plan = wl.plan(wl.spec, variant="hybrid", steps=wl.T, n_prompts=args.prompts, seed=role.pair, denoiser=den,
                   clock="device")
    # HP_BENCH_SHARED_GPU=1 (validation only): every rank on GPU 0 over gloo with host-side
    # flag waits, so the multi-process pair path runs end to end on a one-GPU box
    shared = os.environ.get("HP_BENCH_SHARED_GPU") == "1"
    sess = parallel.GroupSession(plan, groups[role.pair], wait="host" if shared else "device")
    for _ in range(args.warmup):
        sess.run()
    x_host = hp.initial_latents(plan)
    x_dev = torch.from_numpy(x_host).cuda()
    clocks = ClockSampler(local)
    with clocks:
        _barrier(ws)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            sess.run(x_dev)
        b.record()
        torch.cuda.synchronize()
        _barrier(ws)
    dev_s = _max_over_ranks(ws, a.elapsed_time(b) / 1e3)
    _barrier(ws)
    torch.cuda.synchronize()
    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2.record()
    last = None
    for _ in range(args.steps):
        last = sess.run()
    b2.record()
    torch.cuda.synchronize()
    _barrier(ws)
    e2e_s = _max_over_ranks(ws, a2.elapsed_time(b2) / 1e3)
    h2d = int(x_host.nbytes)
    d2h = int(last.x0.nbytes) + 16 * len(last.series)
    return den, dev_s, args.steps * (ws // 2) * args.prompts, e2e_s, h2d, d2h, clocks, 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="pairs", choices=["replicas", "pairs"])
    ap.add_argument("--spec", default="sdxl", choices=["sdxl", "sdxl2048", "sd3", "tiny"],
                    help="BASELINE config: sdxl (config 2, the headline), sdxl2048 (config 4), sd3 (configs 3/5), "
                         "tiny (config 1 network)")
    ap.add_argument("--prompts", type=int, default=1, help="prompts (images) per generation (config 5: 8)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    ws, rank, local = _dist()
    shared = os.environ.get("HP_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        # a bounded collective timeout: a rank that fails inside a collective (e.g. while
        # the pair exchanges IPC handles) turns its partner's wait into an error, not a hang
        from datetime import timedelta
        if shared:
            dist.init_process_group("gloo", timeout=timedelta(minutes=10))
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=timedelta(minutes=10))
    import paper_2602_21760_b200 as hp  # noqa: F401
    wl = Workload(args.spec)
    spec = wl.spec
    hbm_peak, bf16_burst, bf16_sus, peak_src = _peaks()

    mode = "single" if ws == 1 else args.mode
    err = None
    try:
        res = time_pairs(args, wl, ws, rank, local) if mode == "pairs" else time_replicas(args, wl, ws, rank, local)
    except Exception as exc:   # agreed across ranks below; never silently re-measured another way
        err = f"{mode} run failed on rank {rank}: {type(exc).__name__}: {exc}"
        res = None
    if ws > 1:
        import torch.distributed as dist
        flag = torch.tensor([1.0 if err else 0.0], device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        if flag.item() and not err:
            err = "another rank failed"
    if err:
        if rank == 0 or "rank" in err:
            print(json.dumps({"metric": wl.metric, "unit": UNIT, "n_gpus": ws, "error": err}), flush=True)
        return 1
    den, dev_s, images, e2e_s, h2d, d2h, clocks, _ = res
    # latency per image: every step each group (pair / replica) generates one image
    # concurrently, so the per-image latency is the timed region over the K steps
    value = dev_s / args.steps / args.prompts
    e2e_value = e2e_s / args.steps / args.prompts

    fwd_s, fwd_flops = forward_roofline(den, wl) if mode != "pairs" else (None, None)
    b1_s, b1_flops = forward_b1(den, wl)
    launches_fwd = (den.g_both.launches if mode != "pairs"
                    else max(den.g_cond.launches, getattr(getattr(den, "g_uncond", None), "launches", 0)))
    samp = sampler_roofline(hbm_peak) if rank == 0 else {}
    top = top_kernel_rooflines(bf16_burst) if rank == 0 and wl.key == "sdxl" else []

    if rank != 0:
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return 0
    k1_s = samp[65536]["us"] * 1e-6 if samp else 0.0
    den_weight_gb = wl.params * 2 / 1e9
    if mode != "pairs":
        # per GPU over the timed region itself: each rank ran K generations of 50 steps, each
        # step one B=2 forward (+ one sampler launch, counted in the time, not the FLOPs)
        achieved = fwd_flops * wl.T * args.steps / dev_s / 1e12
        achieved_src = "timed region: K x 50 denoiser forwards / CUDA-event time of the K generations"
        roof_flops, roof_kernel = fwd_flops, (f"denoiser forward (tcgen05 GEMM/conv + attention), "
                                              f"B={2 * args.prompts} (both branches)")
    else:
        achieved = b1_flops / b1_s / 1e12
        achieved_src = "isolated B=1 branch-forward graph replays (the per-GPU work of a pair)"
        roof_flops, roof_kernel = b1_flops, f"denoiser forward, B={args.prompts} (one branch per GPU)"
    # what a condition-partitioned pair would take on this clock: one B=1 forward per GPU
    # per step + the eps exchange (bf16 latent over NVLink: bytes / 770 GB/s measured peer
    # copy + an assumed 5 us flag round trip) + the fused sampler kernel
    numel = spec.latent_hw * spec.latent_hw * spec.in_channels
    xch_s = args.prompts * numel * 2 / 770e9 + 5e-6
    pair_pred = wl.T * (b1_s + xch_s + k1_s) / args.prompts
    seq_rho2 = wl.T * (2 * b1_s + k1_s) / args.prompts
    line = {
        "metric": wl.metric, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": wl.name, "latent": wl.latent, "T": wl.T, "sampler": wl.sampler,
                   "guidance_w": 5.0, "images": images, "prompts_per_generation": args.prompts,
                   "plan": ("hybrid on condition-partitioned pairs" if mode == "pairs"
                            else f"serial (CFG batched B={2 * args.prompts})"),
                   "parallelism": f"{mode}x{ws}" if ws > 1 else "single",
                   "params_b": round(wl.params / 1e9, 3),
                   "l2": (f"working set ({den_weight_gb:.1f} GB of bf16 weights per step) >> 126 MB L2"
                          if den_weight_gb > 0.126 else "weights fit in L2 (small network)")},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(args.steps * wl.T * (launches_fwd + 1)),
        "roofline": {"bound": "tensor", "kernel": roof_kernel,
                     "achieved": achieved, "achieved_source": achieved_src,
                     "peak": bf16_sus, "unit": "TFLOP/s", "frac": achieved / bf16_sus,
                     "peak_kind": f"{peak_src} sustained", "frac_of_burst": achieved / bf16_burst,
                     "flops_per_launch": roof_flops,
                     "forward_ms": fwd_s * 1e3 if fwd_s else None,
                     **(_forward_traffic() if wl.key == "sdxl" else {"traffic": None}),
                     "top_kernels": top, "top_kernels_peak": f"{peak_src} burst bf16 {bf16_burst}"},
        "forward_b1": {"ms": b1_s * 1e3, "tflops": b1_flops / b1_s / 1e12,
                       "frac_of_sustained": b1_flops / b1_s / 1e12 / bf16_sus, "flops": b1_flops,
                       "sequential_rho2_s_per_image": seq_rho2,
                       "predicted_pair_latency_s": pair_pred,
                       "predicted_pair_speedup_vs_batched": (value / pair_pred) if mode == "single" else None,
                       "predicted_pair_speedup_vs_sequential": seq_rho2 / pair_pred,
                       "model": f"{wl.T} x (B=1 forward + exchange (numel*2 B / 770 GB/s + 5 us) + sampler kernel)"},
        "sampler_roofline": {"bound": "hbm", "peak": hbm_peak, "unit": "GB/s", "peak_kind": peak_src,
                             "sizes": list(samp.values())},
        "clocks": clocks.summary(),
        "throughput_images_per_s": images / dev_s,
    }
    if ws == 1 and not args.no_cpu_baseline:
        try:
            v, det = cpu_reference_sample(wl, 2)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": det["threads"], "kind": "port",
                                    "sample": f"{det['steps_measured']} whole denoising steps of the serial runner "
                                              f"(fp32 CPU {'MMDiT' if wl.dit else 'U-Net'}, cond then uncond branch "
                                              f"at B=1, numpy fp64 rel_mae/cfg/{'euler' if wl.dit else 'ddim'} at "
                                              f"the latent size), mean step x{wl.T} (one prompt)",
                                    "step_s": det["step_s"], "forward_s": det["forward_s"]}
        except Exception as exc:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                                    "sample": f"failed: {exc}"}
    print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
