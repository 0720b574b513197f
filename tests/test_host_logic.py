"""CPU: host-side logic of the drop-in API (no kernels launched)."""
import json
import os

import numpy as np
import pytest

import paper_2602_21760_b200 as hp


def test_controller_host_mirror_matches_reference_cases(golden_dir):
    with open(os.path.join(golden_dir, "controller.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        cfg = hp.SwitchConfig(L=c["L"], g_slope=c["g_slope"], tau_cap=c["tau_cap"], k=c["k"])
        st, labels = hp.replay_series([tuple(p) for p in c["pairs"]], cfg)
        assert (st.tau1, st.tau2) == (c["tau1"], c["tau2"]), c["name"]
        assert [l.value for l in labels] == c["labels"], c["name"]


def test_series_rules():
    s = hp.DiscrepancySeries()
    s.record(10, 0.5)
    s.record(8, 0.25)
    with pytest.raises(hp.SequencingError):
        s.record(9, 0.1)
    with pytest.raises(hp.NumericError):
        s.record(7, float("nan"))
    with pytest.raises(hp.HistoryError):
        s.get(9)
    assert s.items() == [(10, 0.5), (8, 0.25)]
    assert hp.slope(s, 8, 2) == -0.125
    with pytest.raises(hp.HistoryError):
        hp.slope(s, 8, 5)
    with pytest.raises(hp.ParameterError):
        hp.slope(s, 8, 0)


def test_controller_sequencing():
    cfg = hp.SwitchConfig(L=2, g_slope=1e-3, tau_cap=5, k=2)
    series, state = hp.DiscrepancySeries(), hp.StageState()
    series.record(10, 0.5)
    hp.update_controller(state, series, 10, cfg)
    with pytest.raises(hp.SequencingError):
        hp.update_controller(state, series, 8, cfg)


@pytest.mark.parametrize("bad", [dict(L=0, g_slope=1e-4, tau_cap=10, k=5),
                                 dict(L=5, g_slope=0.0, tau_cap=10, k=5),
                                 dict(L=5, g_slope=1e-4, tau_cap=-1, k=5),
                                 dict(L=5, g_slope=1e-4, tau_cap=10, k=-1)])
def test_switch_config_validation(bad):
    with pytest.raises(hp.ParameterError):
        hp.SwitchConfig(**bad)


def _plan(variant, seed=0, **over):
    return hp.ExperimentConfig.from_dict({"variant": variant, "seeds": [seed], **over}).to_plan()


def test_plan_validation_mirrors_reference():
    with pytest.raises(hp.PlanError):
        _plan("hybrid", switch={"k": 40})
    with pytest.raises(hp.PlanError):
        _plan("hybrid", switch={"L": 50})
    with pytest.raises(hp.PlanError):
        _plan("hybrid", switch={"tau_cap": 60})
    with pytest.raises(hp.PlanError):
        _plan("hybrid", switch={"tau_cap": 0})
    with pytest.raises(hp.PlanError):
        _plan("layer_wise", devices=4, segment_fractions=[0.5, 0.5])
    with pytest.raises(hp.PlanError):
        _plan("layer_wise", devices=2, segment_fractions=[0.9, 0.3])
    with pytest.raises(hp.PlanError):
        _plan("batch_level", devices=3)
    from dataclasses import replace
    p = _plan("hybrid")
    with pytest.raises(hp.PlanError):
        replace(p, seed=-1)
    with pytest.raises(hp.PlanError):
        replace(p, cfg_batching_factor=2.5)
    with pytest.raises(hp.PlanError):
        replace(p, clock="wall")


def test_config_rejects_unknown_keys_and_bad_values():
    with pytest.raises(hp.ParameterError):
        hp.ExperimentConfig.from_dict({"bogus": 1})
    with pytest.raises(hp.ParameterError):
        hp.ExperimentConfig.from_dict({"preset": "nope"})
    with pytest.raises(hp.ParameterError):
        hp.ExperimentConfig.from_dict({"condition_batch": 0})
    with pytest.raises(hp.ParameterError):
        hp.ExperimentConfig.from_dict({"seeds": [-1]})


def test_initial_latents_match_reference_generator(golden_dir):
    # x_T is host numpy with the reference's exact RNG call order
    from oracle import loop
    for seed in (0, 7, 12):
        plan = _plan("serial", seed, condition_batch=8)
        gm, s = plan.mixture, plan.schedule
        rows = [c.indices for c in plan.conditions]
        ref = loop.initial_latents(gm.weights, gm.means, gm.variances, rows, seed, s.alpha_bar(s.T))
        assert np.array_equal(hp.initial_latents(plan), ref)


def test_schedule_host_tables_match_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "sampler.npz"))
    s = hp.build_schedule("scaled-linear", 50, 0.00085, 0.012)
    assert np.array_equal(s.alpha_bars, g["sched_sdxl_abar"])
    assert s.alpha_bar(0) == 1.0 and s.sigma(0) == 0.0
    with pytest.raises(ValueError):
        s.betas[0] = 0.5
    with pytest.raises(hp.ParameterError):
        hp.build_schedule("cosine", 10, 0.1, 0.2)


def test_serial_latency_ref_and_hoeffding():
    assert abs(hp.serial_latency_ref(_plan("serial")) - 16.49) < 1e-12 * 16.49
    m = hp.SlopeNoiseModel(delta=1.0 / np.sqrt(2.0), range_lo=0.0, range_hi=1.0)
    assert abs(hp.hoeffding_false_alarm(1, m) - 0.7357588823428847) < 1e-15
