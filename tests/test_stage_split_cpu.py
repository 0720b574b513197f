"""CPU: stage-split plumbing (stages.py) and its oracle restatement.

* cut selection: each stage's FLOP share tracks its device's segment fraction,
  every stage owns >= 1 unit, and the cuts for the shipped networks are pinned;
* the product's unit lists equal the oracle's own (``oracle.unet_ref.ref_units``);
* the oracle's stage-split loop with k = 0 is bit-identical to the exact loop,
  and a window step fed with FRESH boundary states (all from x_t) reproduces
  the plain conditional forward bit for bit (the split itself loses nothing;
  only staleness changes numbers);
* a stage-split plan with the analytic GMM (no layers) is a PlanError.
"""
import numpy as np
import pytest
import torch

import paper_2602_21760_b200 as hp
from paper_2602_21760_b200.denoiser.mmdit import mmdit_units
from paper_2602_21760_b200.denoiser.unet import unet_units
from paper_2602_21760_b200.denoiser.weights import SD3, SDXL, TINY, init_weights, synthetic_conditioning, unet_param_specs
from paper_2602_21760_b200.errors import PlanError
from paper_2602_21760_b200.stages import network_fractions, stage_bounds, stage_cuts


def _flops(spec):
    return [f for _, f, _ in unet_units(spec)] if hasattr(spec, "block_out") else [f for _, f in mmdit_units(spec)]


@pytest.mark.parametrize("spec", [SDXL, TINY, SD3])
@pytest.mark.parametrize("fr", [(0.5, 0.5), (0.3, 0.7), (0.25,) * 4, (0.1, 0.2, 0.3, 0.4)])
def test_cuts_track_fractions(spec, fr):
    fl = _flops(spec)
    cuts = stage_cuts(fl, network_fractions(fr))
    assert list(cuts) == sorted(set(cuts)) and 0 < cuts[0] and cuts[-1] < len(fl)
    tot = sum(fl)
    shares = [sum(fl[a:b]) / tot for a, b in stage_bounds(cuts, len(fl))]
    biggest = max(fl) / tot
    for share, want in zip(shares, network_fractions(fr)):
        assert abs(share - want) <= biggest + 1e-9          # within one unit's FLOPs


def test_pinned_cuts():
    # SDXL-1024, 2 GPUs: dev1 runs units [0, 17) (conv_in .. the first up resnet,
    # 45.7% of the FLOPs), dev0 units [17, 34) (up path + conv_out) and the sampler
    assert stage_cuts(_flops(SDXL), network_fractions((0.5, 0.5))) == (17,)
    assert stage_cuts(_flops(SD3), network_fractions((0.5, 0.5))) == (13,)       # 12 joint blocks each
    assert stage_cuts(_flops(SDXL), network_fractions((0.25,) * 4)) == (12, 17, 22)


@pytest.mark.parametrize("spec", [SDXL, TINY])
def test_unit_lists_equal_oracle(spec):
    from oracle.unet_ref import ref_units
    assert ref_units(spec) == [u for u, _, _ in unet_units(spec)]


@pytest.fixture(scope="module")
def tiny_ref():
    from oracle.stage_ref import StagedNet
    from oracle.unet_ref import UNetRef, net_timestep
    torch.manual_seed(0)
    W = init_weights(unet_param_specs(TINY), seed=0)
    cond = synthetic_conditioning(1, TINY.context_len, TINY.cross_dim, TINY.pooled_dim)
    cuts = stage_cuts(_flops(TINY), network_fractions((0.5, 0.5)))
    return StagedNet(UNetRef(TINY, W), "unet", cond, TINY, 6, cuts, timestep=net_timestep)


def test_oracle_k0_equals_exact(tiny_ref):
    from oracle import loop as oloop
    from oracle import sampler as osmp
    T = 6
    _, _, ab, sig = osmp.schedule_tables("scaled-linear", T, 0.00085, 0.012)
    x = np.random.default_rng(0).standard_normal((1, 64 * 64 * 4))
    xe, _ = oloop.run_exact(tiny_ref, x, T, 5.0, ab, sig)
    xs, _, t1, t2, _ = oloop.run_staged(tiny_ref, x, T, 5.0, ab, sig, 2, 1e-12, 3, 0, (0.5, 0.5),
                                        pipeline="stage_split")
    assert (t1, t2) == (3, 3)
    assert np.array_equal(xe, xs)


def test_oracle_fresh_window_equals_forward(tiny_ref):
    x = np.random.default_rng(1).standard_normal((1, 64 * 64 * 4))
    ec, _ = tiny_ref.branches(x, 4)
    fresh = tiny_ref.recorded()                      # boundary states of the forward at (x, t=4)
    est, _ = tiny_ref.window_step(x, fresh, 4)
    assert np.array_equal(est, ec)


def test_stage_split_with_gmm_is_plan_error():
    cfg = hp.ExperimentConfig.from_dict({"variant": "hybrid", "seeds": [0]})
    from dataclasses import replace
    with pytest.raises(PlanError):
        replace(cfg.to_plan(), pipeline_numerics="stage_split")
