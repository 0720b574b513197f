"""Command-line harness on the GPU path: simulate, curve, detect, sweep.

Same subcommands, file formats (CURVE / SWEEP / TRACE headers, 17-significant-
digit floats, metrics.json keys) and failure contract (one JSON object on
stderr, exit 1) as the reference harness (cli.py:25-281), so its files
round-trip between the two implementations. Differences: every trajectory runs
on the GPU through the fused sampler; ``--denoiser`` swaps the analytic GMM
for a neural network at the seam (then the curve's score_ratio column repeats
the measured rel-MAE, the identity the reference's criterion 01 pins for
exact scores); ``--clock device`` exports CUDA-event timings in trace.csv /
trace.json instead of the model clock; ``calibrate`` (no reference
counterpart) derives tau_cap from measured curves.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

from .config import ExperimentConfig, load_config
from .engine import PlanVariant, RunResult, condition_groups, initial_latents, run_plan, run_serial
from .errors import HybridparError, PlanError, SeriesParseError
from .metrics import compare_runs
from .monitor import replay_series

CURVE_HEADER = "t,rel_mae,score_ratio,band_lo,band_hi,is_argmin"
SWEEP_HEADER = "k,status,latency_s,speedup,fidelity_l1,psnr_analog"
TRACE_HEADER = "event,step,stage,device,src,dst,label,kind,start,end,nbytes"


def _g17(v: float) -> str:
    return format(v, ".17g")


def _dump(obj) -> str:
    return json.dumps(obj, sort_keys=True, indent=2) + "\n"


def _config(path) -> ExperimentConfig:
    return ExperimentConfig.from_dict({}) if path is None else load_config(path)


def _denoiser_for(name, cfg, plan):
    if name in (None, "gmm"):
        return None
    from . import pipelines
    from .denoiser.weights import SD3, SDXL, TINY, TINY_DIT
    n = len(plan.conditions)
    if name in ("sdxl", "tiny"):
        spec = SDXL if name == "sdxl" else TINY
        return pipelines.build_sdxl_denoiser(spec, n_prompts=n, steps=plan.schedule.T)
    spec = SD3 if name == "sd3" else TINY_DIT
    return pipelines.build_sd3_denoiser(spec, n_prompts=n, steps=plan.schedule.T)


def _net_plan_fields(name, plan):
    """Schedule, sampler, latent prior and conditions of a network at the seam: the
    config keeps T, seeds, variant, switch, devices and link; the network brings its
    own noise schedule (SDXL scaled-linear DDIM, SD3 flow-matching Euler) and a
    latent-shaped prior with one component per prompt (pipelines.latent_prior)."""
    from . import pipelines
    from .denoiser.weights import SD3, SDXL, TINY, TINY_DIT
    from .mixture import Condition
    spec = {"sdxl": SDXL, "tiny": TINY, "sd3": SD3, "tiny-dit": TINY_DIT}[name]
    dit = name in ("sd3", "tiny-dit")
    T, n = plan.schedule.T, len(plan.conditions)
    return dict(schedule=pipelines.sd3_schedule(T) if dit else pipelines.sdxl_schedule(T),
                sampler="euler" if dit else "ddim",
                mixture=pipelines.latent_prior(n, spec.latent_hw * spec.latent_hw * spec.in_channels),
                conditions=tuple(Condition((i,)) for i in range(n)))


def _plan(cfg, args, **kw):
    from dataclasses import replace
    plan = cfg.to_plan(**kw)
    den = getattr(args, "_den", None)
    if getattr(args, "denoiser", None) not in (None, "gmm"):
        if den is None:
            den = args._den = _denoiser_for(args.denoiser, cfg, plan)
        plan = replace(plan, denoiser=den, **_net_plan_fields(args.denoiser, plan))
    if getattr(args, "clock", None):
        plan = replace(plan, clock=args.clock)
    if getattr(args, "pipeline_numerics", None):
        plan = replace(plan, pipeline_numerics=args.pipeline_numerics)
    return plan


def trace_rows(result: RunResult) -> list:
    rows = [TRACE_HEADER]
    for b in result.trace.busy:
        rows.append(f"busy,{b.step},{b.stage},{b.device},,,{b.label},,{_g17(b.start)},{_g17(b.end)},")
    for m in result.trace.messages:
        rows.append(f"message,{m.step},,,{m.src},{m.dst},,{m.kind},{_g17(m.depart)},{_g17(m.arrive)},{m.nbytes}")
    return rows


def write_trace(result: RunResult, out_dir: str) -> None:
    with open(os.path.join(out_dir, "trace.csv"), "w", encoding="utf-8") as fh:
        fh.write("\n".join(trace_rows(result)) + "\n")
    doc = {"busy": [dict(device=b.device, start=b.start, end=b.end, step=b.step, stage=b.stage, label=b.label)
                    for b in result.trace.busy],
           "messages": [dict(src=m.src, dst=m.dst, kind=m.kind, nbytes=m.nbytes, depart=m.depart,
                             arrive=m.arrive, step=m.step) for m in result.trace.messages]}
    with open(os.path.join(out_dir, "trace.json"), "w", encoding="utf-8") as fh:
        fh.write(_dump(doc))


def simulate(args) -> int:
    cfg = _config(args.config)
    plan = _plan(cfg, args, seed=args.seed, variant=PlanVariant(args.variant) if args.variant else None)
    result = run_plan(plan)
    baseline = result if plan.variant is PlanVariant.SERIAL else run_serial(
        _plan(cfg, args, seed=plan.seed, variant=PlanVariant.SERIAL))
    text = _dump(compare_runs(result, baseline).to_dict())
    out_dir = args.out or cfg.out_dir
    if out_dir is None:
        raise PlanError("simulate needs an output directory (--out or config out_dir)")
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "metrics.json"), "w", encoding="utf-8") as fh:
        fh.write(text)
    write_trace(result, out_dir)
    sys.stdout.write(text)
    return 0


def curve_rows(cfg: ExperimentConfig, args=None) -> list:
    """Serial-trajectory discrepancy curve on the GPU: (t, rel_mae, score_ratio,
    band_lo, band_hi) per step; band = mean +/- 2 sample sd of per-row ratios."""
    from . import _kernels as K, _native as N
    from .engine import _StepRunner
    from .mixture import conditional_grad, noised_mixture, score
    plan = _plan(cfg, args, variant=PlanVariant.SERIAL) if args is not None else cfg.to_plan(variant=PlanVariant.SERIAL)
    st = _StepRunner(plan)
    x, xb = st.upload(initial_latents(plan))
    gmm = plan.denoiser is None
    groups = condition_groups(plan.conditions)
    out = []
    for t in range(plan.schedule.T, 0, -1):
        eps_c, eps_u = st.den.branches(x, t, xb)
        ec, eu = eps_c.double(), eps_u.double()
        ws = K.rel_mae_dev(eps_c, eps_u)
        m = float(ws.m.item())
        K.read_status(ws, "rel_mae")
        if gmm:
            s_u = score(noised_mixture(plan.mixture, plan.schedule.alpha_bar(t)), x).score
            num = sum(float(conditional_grad(plan.mixture, c, plan.schedule, x[torch.as_tensor(r, device=x.device)],
                                             t).abs().sum()) for c, r in groups)
            ratio = num / float(s_u.abs().sum())
        else:
            ratio = m
        per_row = (ec - eu).abs().sum(dim=1) / eu.abs().sum(dim=1)
        sd = float(per_row.std(unbiased=True)) if per_row.numel() > 1 else 0.0
        out.append((t, m, ratio, m - 2.0 * sd, m + 2.0 * sd))
        x, xb = st._advance(x, xb, eps_c, eps_u, t, N.HP_CTRL_NONE)
    return out


def curve(args) -> int:
    rows = curve_rows(_config(args.config), args)
    lowest = min(range(len(rows)), key=lambda i: rows[i][1])
    lines = [CURVE_HEADER] + [f"{t},{_g17(m)},{_g17(r)},{_g17(lo)},{_g17(hi)},{int(i == lowest)}"
                              for i, (t, m, r, lo, hi) in enumerate(rows)]
    with open(args.out, "w", encoding="utf-8") as fh:
        fh.write("\n".join(lines) + "\n")
    return 0


def read_series_csv(path: str) -> list:
    """(t, M) pairs from a curve CSV (columns t, rel_mae) or a bare two-column file."""
    with open(path, encoding="utf-8") as fh:
        numbered = [(i + 1, ln.strip()) for i, ln in enumerate(fh) if ln.strip()]
    if not numbered:
        raise SeriesParseError("series file is empty")
    head = [f.strip() for f in numbered[0][1].split(",")]
    cols = (0, 1)
    try:
        float(head[0])
    except ValueError:
        if "t" not in head or "rel_mae" not in head:
            raise SeriesParseError(f"header must name columns t and rel_mae, got {head}", line=1) from None
        cols = (head.index("t"), head.index("rel_mae"))
        numbered = numbered[1:]
    pairs = []
    for lineno, text in numbered:
        f = [v.strip() for v in text.split(",")]
        if len(f) <= max(cols):
            raise SeriesParseError(f"expected at least {max(cols) + 1} columns, got {len(f)}", line=lineno)
        try:
            pairs.append((int(f[cols[0]]), float(f[cols[1]])))
        except ValueError:
            raise SeriesParseError(f"bad numeric fields {f[cols[0]]!r}, {f[cols[1]]!r}", line=lineno) from None
    return pairs


def detect(args) -> int:
    cfg = _config(args.config)
    state, labels = replay_series(read_series_csv(args.series), cfg.switch)
    sys.stdout.write(_dump({"tau1": state.tau1, "tau2": state.tau2, "stages": [s.value for s in labels]}))
    return 0


def calibrate_tau_cap(curves, switch, T: int, margin: int = 1) -> dict:
    """tau_cap from measured discrepancy curves: replay each
    curve through the controller with the cap out of the way (tau_cap = T - k - 1)
    to find the step at which the slope detector fires by itself (natural tau1),
    then cap one ``margin`` past the latest natural firing so the cap never
    pre-empts detection on these trajectories. Curves on which the detector never
    fires keep the configured cap (reported as ``binding``)."""
    from .monitor import SwitchConfig
    loose = SwitchConfig(L=switch.L, g_slope=switch.g_slope, tau_cap=max(1, T - switch.k - 1), k=switch.k)
    per = []
    for name, pairs in curves:
        state, _ = replay_series(pairs, loose)
        fired = state.tau1 is not None and state.tau1 < loose.tau_cap
        ms = dict(pairs)
        t_fire = T - state.tau1 + 1 if fired else None
        g = ((ms[t_fire] - ms[t_fire + switch.L]) / switch.L
             if fired and t_fire + switch.L in ms else None)
        per.append({"curve": name, "natural_tau1": state.tau1 if fired else None,
                    "t_at_firing": t_fire, "slope_at_firing": g,
                    "slope_margin": None if g is None else switch.g_slope - g})
    natural = [c["natural_tau1"] for c in per if c["natural_tau1"] is not None]
    binding = len(natural) < len(per)
    tau_cap = switch.tau_cap if binding else min(max(natural) + margin, T - switch.k - 1)
    cal = SwitchConfig(L=switch.L, g_slope=switch.g_slope, tau_cap=tau_cap, k=switch.k)
    for c, (_, pairs) in zip(per, curves):
        st, labels = replay_series(pairs, cal)
        c["detect"] = {"tau1": st.tau1, "tau2": st.tau2, "stages": [x.value for x in labels]}
    return {"L": switch.L, "g_slope": switch.g_slope, "k": switch.k, "T": T, "margin": margin,
            "configured_tau_cap": switch.tau_cap, "tau_cap": tau_cap, "cap_binding": binding, "curves": per}


def calibrate(args) -> int:
    cfg = _config(args.config)
    curves = [(path, read_series_csv(path)) for path in args.series]
    T = max(t for _, pairs in curves for t, _ in pairs)
    sys.stdout.write(_dump(calibrate_tau_cap(curves, cfg.switch, T, args.margin)))
    return 0


def _k_values(text: str) -> list:
    try:
        return sorted({int(tok) for tok in text.replace(" ", "").split(",") if tok})
    except ValueError:
        raise SeriesParseError(f"bad k list {text!r}; expected comma-separated integers") from None


def sweep(args) -> int:
    cfg = _config(args.config)
    serial = {s: run_serial(_plan(cfg, args, seed=s, variant=PlanVariant.SERIAL)) for s in cfg.seeds}
    lines = [SWEEP_HEADER]
    for k in _k_values(args.k):
        try:
            plans = [_plan(cfg, args, seed=s, variant=PlanVariant.HYBRID, k=k) for s in cfg.seeds]
        except PlanError:
            lines.append(f"{k},infeasible,,,,")
            continue
        ms = [compare_runs(run_plan(p), serial[p.seed]) for p in plans]
        psnr = [m.psnr_analog for m in ms if m.psnr_analog is not None]
        lines.append(",".join([str(k), "ok", _g17(float(np.mean([m.latency_s for m in ms]))),
                               _g17(float(np.mean([m.speedup for m in ms]))),
                               _g17(float(np.mean([m.fidelity_l1 for m in ms]))),
                               _g17(float(np.mean(psnr))) if psnr else ""]))
    text = "\n".join(lines) + "\n"
    if args.out:
        with open(args.out, "w", encoding="utf-8") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="hybridpar-b200",
                                 description="Adaptive hybrid-parallel diffusion sampling on B200.")
    sub = ap.add_subparsers(dest="command", required=True)
    common = dict(config=dict(help="experiment JSON; defaults apply if omitted"),
                  denoiser=dict(choices=["gmm", "tiny", "sdxl", "tiny-dit", "sd3"], default="gmm",
                                help="branch evaluator at the seam"),
                  clock=dict(choices=["model", "device"], default=None, help="trace clock"),
                  **{"pipeline-numerics": dict(choices=["reference_blend", "stage_split"], default=None,
                                               help="window numerics (stage_split needs a network denoiser)")})
    specs = {
        "simulate": (simulate, "run one plan and write metrics + trace",
                     [("--variant", dict(choices=[v.value for v in PlanVariant])), ("--seed", dict(type=int)),
                      ("--out", dict(help="output directory"))]),
        "curve": (curve, "emit the discrepancy curve CSV", [("--out", dict(required=True))]),
        "detect": (detect, "replay switch detection over a series CSV", [("--series", dict(required=True))]),
        "calibrate": (calibrate, "tau_cap from measured discrepancy curves (natural slope detection)",
                      [("--series", dict(required=True, nargs="+")), ("--margin", dict(type=int, default=1))]),
        "sweep": (sweep, "sweep the pipelined-window width k",
                  [("--k", dict(required=True)), ("--out", dict(help="destination CSV; stdout if omitted"))]),
    }
    for name, (fn, helptext, extra) in specs.items():
        p = sub.add_parser(name, help=helptext)
        for flag, kw in [(f"--{k}", v) for k, v in common.items()] + extra:
            p.add_argument(flag, **kw)
        p.set_defaults(func=fn)
    return ap


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    try:
        return args.func(args)
    except HybridparError as exc:
        err = {"error": type(exc).__name__, "message": str(exc)}
        if isinstance(exc, SeriesParseError) and exc.line is not None:
            err["line"] = exc.line
        sys.stderr.write(json.dumps(err, sort_keys=True) + "\n")
        return 1
    except (json.JSONDecodeError, OSError) as exc:
        sys.stderr.write(json.dumps({"error": type(exc).__name__, "message": str(exc)}, sort_keys=True) + "\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
