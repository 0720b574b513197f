"""GPU: the drop-in runners on the reference's default testbed.

Every run's schedule (tau1, tau2, stage labels, series keys), comm bytes and
model-clock latency must equal the reference's exactly; latents match to
1e-10 (the GMM denoiser runs as torch fp64 on the GPU, whose exp/log differ
from numpy's in the last ulp; the sampler update itself is bit-exact).
"""
import json
import os

import numpy as np
import pytest

import paper_2602_21760_b200 as hp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def runs(golden_dir):
    with open(os.path.join(golden_dir, "loops.json")) as fh:
        r = json.load(fh)
    return r, np.load(os.path.join(golden_dir, "loops.npz"))


def test_all_reference_runs(runs):
    rs, arrays = runs
    for r in rs:
        plan = hp.ExperimentConfig.from_dict(r["raw"]).to_plan()
        res = hp.run_plan(plan)
        assert (res.tau1, res.tau2) == (r["tau1"], r["tau2"]), r
        assert res.comm_bytes == r["comm_bytes"], r
        assert abs(res.latency_s - r["latency_s"]) <= 1e-12 * r["latency_s"], r
        assert len(res.trace.messages) == r["n_messages"]
        assert [t for t, _ in res.series] == [t for t, _ in r["series"]], r
        np.testing.assert_allclose([m for _, m in res.series], [m for _, m in r["series"]],
                                   rtol=1e-9, atol=1e-13)
        np.testing.assert_allclose(res.x0, arrays[r["key"]], rtol=0, atol=1e-10)


def test_empty_window_and_fcp_bitwise_equal_serial():
    for seed in (0, 5):
        base = {"seeds": [seed]}
        s = hp.run_plan(hp.ExperimentConfig.from_dict({**base, "variant": "serial"}).to_plan())
        f = hp.run_plan(hp.ExperimentConfig.from_dict({**base, "variant": "full_condition_partition"}).to_plan())
        h = hp.run_plan(hp.ExperimentConfig.from_dict({**base, "variant": "hybrid", "switch": {"k": 0}}).to_plan())
        assert np.array_equal(s.x0, f.x0)
        assert np.array_equal(s.x0, h.x0)
        assert s.series == f.series


def test_hybrid_stage_labels_and_device_clock():
    plan = hp.ExperimentConfig.from_dict({"variant": "hybrid", "clock": "device"}).to_plan()
    res = hp.run_plan(plan)
    labels = [s.value for s in res.stages]
    assert labels == ["warm_up"] * 15 + ["parallelism"] * 5 + ["fully_connecting"] * 30
    assert res.latency_s > 0 and len(res.trace.busy) == 50


def test_layer_wise_two_equals_hybrid():
    hy = hp.run_plan(hp.ExperimentConfig.from_dict({"variant": "hybrid", "seeds": [4]}).to_plan())
    lw = hp.run_plan(hp.ExperimentConfig.from_dict({"variant": "layer_wise", "devices": 2, "seeds": [4]}).to_plan())
    assert np.array_equal(hy.x0, lw.x0)
    assert hy.latency_s == lw.latency_s and hy.comm_bytes == lw.comm_bytes


def test_euler_sampler_runs_with_gmm_velocity():
    from oracle import sampler as smp
    plan = hp.ExperimentConfig.from_dict({"variant": "serial", "sampler": "euler",
                                          "condition_batch": 8, "schedule": {"T": 28}}).to_plan()
    res = hp.run_plan(plan)
    # restated on the host: x_{t-1} = x_t - v_cfg dt with v from mixture.fm_velocity
    x = hp.initial_latents(plan)
    T = plan.schedule.T
    for t in range(T, 0, -1):
        vu = hp.fm_velocity(plan.mixture, None, x, t / T)
        vc = np.empty_like(x)
        for i, c in enumerate(plan.conditions):
            vc[i] = hp.fm_velocity(plan.mixture, c, x[i:i + 1], t / T)[0]
        x = smp.euler(x, smp.cfg(vc, vu, plan.guidance.w), 1.0 / T)
    np.testing.assert_allclose(res.x0, x, atol=1e-10)
