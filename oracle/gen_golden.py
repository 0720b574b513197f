"""Generate tests/golden/* by running the REFERENCE itself (read-only import).

Run in the build container (the GPU box has no /root/reference):

    PYTHONPATH=/root/reference/pkg/src python -m oracle.gen_golden

Writes small fixtures only; every value comes from the reference package's
public API (hybridpar 0.1.0). The script also checks the oracle restatement
against those values before writing, so a fixture is never produced by a
disagreeing oracle.
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"
REF = Path(os.environ.get("HYBRIDPAR_REF", "/root/reference/pkg/src"))


def _ref():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import hybridpar  # noqa: F401  (the reference package)
    return hybridpar


def gen_sampler(hp):
    from . import sampler as smp
    rng = np.random.default_rng(20260218)
    out = {}
    for name, (kind, T, b0, b1) in {
        "default": ("linear", 50, 0.01, 0.12),
        "sdxl": ("scaled-linear", 50, 0.00085, 0.012),
        "sd3": ("linear", 28, 0.0005, 0.05),
        "t20": ("linear", 20, 0.01, 0.2),
    }.items():
        s = hp.build_schedule(kind, T, b0, b1)
        out[f"sched_{name}_abar"] = np.asarray(s.alpha_bars)
        out[f"sched_{name}_sigma"] = np.asarray(s.sigmas)
        o = smp.schedule_tables(kind, T, b0, b1)
        assert np.array_equal(o[2], s.alpha_bars) and np.array_equal(o[3], s.sigmas)
    s = hp.build_schedule("linear", 20, 0.01, 0.2)
    for tag, shape in (("small", (3, 7)), ("med", (2, 2048)), ("odd", (1, 1001))):
        ec = rng.standard_normal(shape)
        eu = rng.standard_normal(shape) + 0.25
        x = rng.standard_normal(shape) * 2.0
        w = float(rng.uniform(0.5, 8.0))
        out[f"{tag}_eps_c"], out[f"{tag}_eps_u"], out[f"{tag}_x"] = ec, eu, x
        out[f"{tag}_w"] = np.array(w)
        e = hp.cfg_combine(ec, eu, hp.GuidanceParams(w))
        out[f"{tag}_cfg"] = e
        assert np.array_equal(e, smp.cfg(ec, eu, w))
        out[f"{tag}_rel_mae"] = np.array(hp.rel_mae(ec, eu))
        assert smp.rel_mae(ec, eu) == float(out[f"{tag}_rel_mae"])
        for t in (20, 11, 1):
            r = hp.ddim_step(hp.LatentState(x, t), e, s).x
            out[f"{tag}_ddim_t{t}"] = r
            assert np.array_equal(r, smp.ddim(x, e, t, s.alpha_bars, s.sigmas))
        out[f"{tag}_euler"] = hp.fm_euler_step(x, 0.75, e, 0.05)
        assert np.array_equal(out[f"{tag}_euler"], smp.euler(x, e, 0.05))
        out[f"{tag}_ddpm_t7"] = hp.ddpm_posterior_mean(x, 7, e, s)
    np.savez_compressed(OUT / "sampler.npz", **out)


def gen_controller(hp):
    from . import controller as ctl
    cases = []

    def add(name, pairs, L, g, cap, k):
        st, labels = hp.replay_series(pairs, hp.SwitchConfig(L=L, g_slope=g, tau_cap=cap, k=k))
        lab = [x.value for x in labels]
        o = ctl.replay(pairs, L, g, cap, k)
        assert (o[0], o[1], o[2]) == (st.tau1, st.tau2, lab), name
        cases.append({"name": name, "pairs": [[int(t), float(m)] for t, m in pairs], "L": L,
                      "g_slope": g, "tau_cap": cap, "k": k, "tau1": st.tau1, "tau2": st.tau2,
                      "labels": lab})

    parab = [(t, 0.02 * (t - 25.0) ** 2 / 25.0 ** 2 + 0.05) for t in range(50, 0, -1)]
    add("parabola", parab, 12, 4e-4, 50, 5)
    add("cap_decay", [(t, 0.1 + 0.01 * t) for t in range(50, 0, -1)], 12, 4e-4, 15, 5)
    add("flat", [(t, 0.25) for t in range(50, 0, -1)], 12, 4e-4, 50, 5)
    add("flat_clamped", [(t, 0.25) for t in range(50, 0, -1)], 12, 4e-4, 8, 3)
    add("k_zero", [(t, 0.1 + 0.01 * t) for t in range(30, 0, -1)], 12, 4e-4, 10, 0)
    rng = np.random.default_rng(404)
    for i in range(50):
        amp, t0, floor = float(rng.uniform(0.005, 0.05)), float(rng.uniform(10, 40)), float(rng.uniform(0.01, 0.2))
        pairs = [(t, amp * (t - t0) ** 2 / t0 ** 2 + floor) for t in range(50, 0, -1)]
        add(f"ucurve_{i}", pairs, int(rng.integers(1, 16)), float(rng.uniform(1e-5, 1e-3)),
            int(rng.integers(1, 51)), int(rng.integers(0, 8)))
    rng = np.random.default_rng(17)
    for i in range(40):
        T = int(rng.integers(10, 80))
        L, g, cap, k = int(rng.integers(1, 15)), float(rng.uniform(1e-5, 1e-2)), int(rng.integers(1, T + 1)), int(rng.integers(0, 10))
        add(f"random_{i}", [(t, float(rng.uniform(0.0, 1.0))) for t in range(T, 0, -1)], L, g, cap, k)
    (OUT / "controller.json").write_text(json.dumps(cases))


def gen_loops(hp):
    """Default testbed runs (config.py defaults) through the reference runners."""
    from . import loop, sampler as smp
    runs, arrays = [], {}
    spec = [
        ("serial", {}, [0, 3, 5]),
        ("full_condition_partition", {}, [0, 3]),
        ("hybrid", {}, [0, 1, 4, 5]),
        ("hybrid", {"switch": {"k": 0}}, [5]),
        ("hybrid", {"switch": {"k": 10}}, [0]),
        ("layer_wise", {"devices": 4}, [0]),
        ("layer_wise", {"devices": 2}, [4]),
        ("batch_level", {"devices": 4}, [10]),
        ("hybrid", {"condition_batch": 4, "schedule": {"T": 10},
                    "switch": {"L": 2, "tau_cap": 3, "k": 4}}, [2]),
        ("full_condition_partition", {"link": {"base_latency_s": 0.00995}}, [0]),
        ("layer_wise", {"devices": 3}, [7]),
    ]
    for variant, over, seeds in spec:
        for seed in seeds:
            raw = {"variant": variant, "seeds": [seed], **over}
            cfg = hp.ExperimentConfig.from_dict(raw)
            plan = cfg.to_plan()
            res = hp.run_plan(plan)
            key = f"run{len(runs)}"
            arrays[key] = res.x0
            runs.append({"key": key, "raw": raw, "variant": variant, "seed": seed,
                         "latency_s": res.latency_s, "comm_bytes": res.comm_bytes,
                         "speedup": res.speedup, "tau1": res.tau1, "tau2": res.tau2,
                         "series": [[int(t), float(m)] for t, m in res.series],
                         "throughput": res.throughput_samples_per_s,
                         "n_messages": len(res.trace.messages)})
            # oracle restatement must agree bit for bit with the reference runner
            gm = plan.mixture
            rows = [c.indices for c in plan.conditions]
            s = plan.schedule
            if variant == "batch_level":
                continue
            x = loop.initial_latents(gm.weights, gm.means, gm.variances, rows, seed, s.alpha_bar(s.T))
            assert np.array_equal(x, hp.initial_latents(plan))
            den = loop.GMMDenoiser(gm.weights, gm.means, gm.variances, rows, s.alpha_bars, s.sigmas)
            if variant in ("serial", "full_condition_partition"):
                xo, ser = loop.run_exact(den, x, s.T, plan.guidance.w, s.alpha_bars, s.sigmas)
            else:
                sw = plan.switch
                xo, ser, t1, t2, _ = loop.run_staged(den, x, s.T, plan.guidance.w, s.alpha_bars,
                                                     s.sigmas, sw.L, sw.g_slope, sw.tau_cap, sw.k,
                                                     plan.segment_fractions)
                assert (t1, t2) == (res.tau1, res.tau2)
            assert np.array_equal(xo, res.x0), (variant, seed)
            assert [t for t, _ in ser] == [t for t, _ in res.series]
            np.testing.assert_allclose([m for _, m in ser], [m for _, m in res.series], rtol=1e-12)
    np.savez_compressed(OUT / "loops.npz", **arrays)
    (OUT / "loops.json").write_text(json.dumps(runs, indent=1))
    _ = smp


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    hp = _ref()
    gen_sampler(hp)
    gen_controller(hp)
    gen_loops(hp)
    print(f"golden fixtures written to {OUT}")


if __name__ == "__main__":
    main()


def gen_cli():
    """Reference CLI outputs (cli.py:44-228) for the harness parity tests."""
    import contextlib
    import io
    import shutil
    hp = _ref()
    from hybridpar import cli
    d = OUT / "cli"
    if d.exists():
        shutil.rmtree(d)
    d.mkdir(parents=True)
    small = {"condition_batch": 4, "seeds": [0, 1], "schedule": {"T": 12}, "switch": {"L": 2, "tau_cap": 3, "k": 4}}
    (d / "small.json").write_text(json.dumps(small))
    runs = {
        "simulate": ["simulate", "--out", str(d / "sim")],
        "curve": ["curve", "--out", str(d / "curve.csv")],
        "sweep": ["sweep", "--k", "0,5,10,40", "--out", str(d / "sweep.csv")],
        "sweep_small": ["sweep", "--config", str(d / "small.json"), "--k", "0,2,4,9"],
    }
    outs = {}
    for name, argv in runs.items():
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert cli.main(argv) == 0, name
        outs[name] = buf.getvalue()
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        assert cli.main(["detect", "--series", str(d / "curve.csv")]) == 0
    outs["detect"] = buf.getvalue()
    (d / "stdout.json").write_text(json.dumps(outs, indent=1))
    _ = hp


if __name__ == "__main__" and "--cli" in sys.argv:
    gen_cli()
