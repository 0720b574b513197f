"""CPU: the oracle restatement against golden vectors produced by the reference.

Pins the oracle (oracle/) before it is trusted as the checker of the CUDA
path; the fixtures come from running hybridpar 0.1.0 itself
(oracle/gen_golden.py).
"""
import json
import os

import numpy as np
import pytest

from oracle import controller as ctl
from oracle import loop
from oracle import sampler as smp


@pytest.fixture(scope="module")
def sampler_golden(golden_dir):
    return np.load(os.path.join(golden_dir, "sampler.npz"))


@pytest.fixture(scope="module")
def controller_cases(golden_dir):
    with open(os.path.join(golden_dir, "controller.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def loop_runs(golden_dir):
    with open(os.path.join(golden_dir, "loops.json")) as fh:
        runs = json.load(fh)
    return runs, np.load(os.path.join(golden_dir, "loops.npz"))


@pytest.mark.parametrize("name,spec", [
    ("default", ("linear", 50, 0.01, 0.12)),
    ("sdxl", ("scaled-linear", 50, 0.00085, 0.012)),
    ("sd3", ("linear", 28, 0.0005, 0.05)),
    ("t20", ("linear", 20, 0.01, 0.2)),
])
def test_schedule_tables_bit_exact(sampler_golden, name, spec):
    _, _, abar, sig = smp.schedule_tables(*spec)
    assert np.array_equal(abar, sampler_golden[f"sched_{name}_abar"])
    assert np.array_equal(sig, sampler_golden[f"sched_{name}_sigma"])


def test_scaled_linear_kat():
    # tests/test_schedules.py:14 in the reference
    _, _, abar, _ = smp.schedule_tables("scaled-linear", 50, 0.00085, 0.012)
    assert abs(abar[-1] - 0.763763285673763) <= 1e-12 * 0.763763285673763


@pytest.mark.parametrize("tag", ["small", "med", "odd"])
def test_sampler_primitives_bit_exact(sampler_golden, tag):
    g = sampler_golden
    ec, eu, x, w = g[f"{tag}_eps_c"], g[f"{tag}_eps_u"], g[f"{tag}_x"], float(g[f"{tag}_w"])
    e = smp.cfg(ec, eu, w)
    assert np.array_equal(e, g[f"{tag}_cfg"])
    assert smp.rel_mae(ec, eu) == float(g[f"{tag}_rel_mae"])
    _, _, abar, sig = smp.schedule_tables("linear", 20, 0.01, 0.2)
    for t in (20, 11, 1):
        assert np.array_equal(smp.ddim(x, e, t, abar, sig), g[f"{tag}_ddim_t{t}"])
    assert np.array_equal(smp.euler(x, e, 0.05), g[f"{tag}_euler"])


def test_hand_values():
    assert np.array_equal(smp.cfg([2.0], [1.0], 3.0), [5.0])        # test_schedules.py:92
    assert smp.rel_mae([2.0, 0.0], [1.0, 1.0]) == 1.0                 # test_monitor.py:34
    assert np.array_equal(smp.euler([1.0], [2.0], 0.5), [0.0])        # test_schedules.py:197


def test_controller_replays(controller_cases):
    assert len(controller_cases) == 95
    for c in controller_cases:
        t1, t2, labels = ctl.replay([tuple(p) for p in c["pairs"]], c["L"], c["g_slope"],
                                    c["tau_cap"], c["k"])
        assert (t1, t2) == (c["tau1"], c["tau2"]), c["name"]
        assert labels == c["labels"], c["name"]


def test_controller_kats(controller_cases):
    by = {c["name"]: c for c in controller_cases}
    assert (by["parabola"]["tau1"], by["parabola"]["tau2"]) == (32, 37)
    assert (by["cap_decay"]["tau1"], by["cap_decay"]["tau2"]) == (15, 20)
    assert by["flat"]["tau1"] == 13 and by["flat_clamped"]["tau1"] == 8
    assert by["k_zero"]["tau1"] == by["k_zero"]["tau2"] == 10


def _plan_inputs(run):
    from paper_2602_21760_b200.config import ExperimentConfig
    cfg = ExperimentConfig.from_dict(run["raw"])
    plan = cfg.to_plan()
    gm, s = plan.mixture, plan.schedule
    rows = [c.indices for c in plan.conditions]
    return plan, gm, s, rows


def test_oracle_loops_reproduce_reference(loop_runs):
    runs, arrays = loop_runs
    checked = 0
    for run in runs:
        if run["variant"] == "batch_level":
            continue
        plan, gm, s, rows = _plan_inputs(run)
        x = loop.initial_latents(gm.weights, gm.means, gm.variances, rows, run["seed"],
                                 s.alpha_bar(s.T))
        den = loop.GMMDenoiser(gm.weights, gm.means, gm.variances, rows, s.alpha_bars, s.sigmas)
        if run["variant"] in ("serial", "full_condition_partition"):
            xo, ser = loop.run_exact(den, x, s.T, plan.guidance.w, s.alpha_bars, s.sigmas)
        else:
            sw = plan.switch
            xo, ser, t1, t2, _ = loop.run_staged(den, x, s.T, plan.guidance.w, s.alpha_bars,
                                                 s.sigmas, sw.L, sw.g_slope, sw.tau_cap, sw.k,
                                                 plan.segment_fractions)
            assert (t1, t2) == (run["tau1"], run["tau2"])
        assert np.array_equal(xo, arrays[run["key"]]), run
        assert [t for t, _ in ser] == [t for t, _ in run["series"]]
        checked += 1
    assert checked >= 10


def test_default_hybrid_kat(loop_runs):
    runs, arrays = loop_runs
    r = next(r for r in runs if r["variant"] == "hybrid" and r["seed"] == 0 and r["raw"].keys() == {"variant", "seeds"})
    assert (r["tau1"], r["tau2"]) == (15, 20)
    assert r["comm_bytes"] == 450560
    assert [t for t, _ in r["series"]] == list(range(50, 35, -1)) + list(range(30, 0, -1))
    assert abs(float(arrays[r["key"]].sum()) - (-17.873421572221)) < 1e-9
