"""GPU: the fused sampler kernel and device controller against the reference.

fp64: bit-exact against the reference's own outputs (golden fixtures).
fp32 latent + bf16 eps: within the stated tolerance of the fp64 oracle.
"""
import json
import os

import numpy as np
import pytest
import torch

import paper_2602_21760_b200 as hp
from oracle import controller as ctl
from oracle import sampler as smp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g(golden_dir):
    return np.load(os.path.join(golden_dir, "sampler.npz"))


@pytest.mark.parametrize("tag", ["small", "med", "odd"])
def test_fp64_primitives_bit_exact_vs_reference(g, tag):
    ec, eu, x, w = g[f"{tag}_eps_c"], g[f"{tag}_eps_u"], g[f"{tag}_x"], float(g[f"{tag}_w"])
    e = hp.cfg_combine(ec, eu, hp.GuidanceParams(w))
    assert isinstance(e, np.ndarray)
    assert np.array_equal(e, g[f"{tag}_cfg"])
    s = hp.build_schedule("linear", 20, 0.01, 0.2)
    for t in (20, 11, 1):
        out = hp.ddim_step(hp.LatentState(x, t), e, s)
        assert out.t == t - 1
        assert np.array_equal(out.x, g[f"{tag}_ddim_t{t}"]), t
    assert np.array_equal(hp.fm_euler_step(x, 0.75, e, 0.05), g[f"{tag}_euler"])
    assert np.array_equal(hp.ddpm_posterior_mean(x, 7, e, s), g[f"{tag}_ddpm_t7"])
    m = hp.rel_mae(ec, eu)
    assert abs(m - float(g[f"{tag}_rel_mae"])) <= 1e-14 * abs(m)


def test_torch_tensors_stay_on_device(g):
    ec = torch.from_numpy(g["med_eps_c"]).cuda()
    eu = torch.from_numpy(g["med_eps_u"]).cuda()
    e = hp.cfg_combine(ec, eu, hp.GuidanceParams(float(g["med_w"])))
    assert e.is_cuda and e.dtype == torch.float64
    assert np.array_equal(e.cpu().numpy(), g["med_cfg"])


def test_errors_map_to_reference_taxonomy():
    s = hp.build_schedule("linear", 10, 0.02, 0.1)
    with pytest.raises(hp.NumericError):
        hp.ddim_step(hp.LatentState(np.array([1.0, np.inf]), 5), np.zeros(2), s)
    with pytest.raises(hp.NumericError):
        hp.cfg_combine(np.array([np.nan]), np.array([1.0]), hp.GuidanceParams(1.0))
    with pytest.raises(hp.ShapeError):
        hp.cfg_combine(np.zeros(3), np.zeros(4), hp.GuidanceParams(1.0))
    with pytest.raises(hp.StepUnderflowError):
        hp.ddim_step(hp.LatentState(np.zeros(2), 0), np.zeros(2), s)
    with pytest.raises(hp.DegenerateInputError):
        hp.rel_mae(np.array([1.0]), np.array([0.0]))
    with pytest.raises(hp.NumericError):
        hp.rel_mae(np.array([np.inf]), np.array([1.0]))
    with pytest.raises(hp.ParameterError):
        hp.fm_euler_step(np.zeros(2), 1.5, np.zeros(2), 0.1)
    with pytest.raises(hp.StepUnderflowError):
        hp.fm_euler_step(np.zeros(2), 0.1, np.zeros(2), 0.2)
    # workspace recovers after an error
    assert np.array_equal(hp.cfg_combine(np.array([2.0]), np.array([1.0]), hp.GuidanceParams(3.0)), [5.0])


@pytest.mark.parametrize("n", [1, 3, 1000, 65536, 65536 * 4 + 7, 1 << 22])
def test_fp32_bf16_fused_step_within_tolerance(n):
    """fp32 master latent, bf16 branch outputs (the neural path's dtypes):
    max-abs <= 1e-5 relative to the fp64 oracle on the same bf16-rounded inputs."""
    from paper_2602_21760_b200 import _kernels as K, _native as N
    gen = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randn(n, device="cuda", generator=gen)
    ec = torch.randn(n, device="cuda", generator=gen).bfloat16()
    eu = (torch.randn(n, device="cuda", generator=gen) * 0.9).bfloat16()
    s = hp.build_schedule("scaled-linear", 50, 0.00085, 0.012)
    t = 37
    c = hp.StepCoefficients.ddim(s, t)
    out = torch.empty_like(x)
    outb = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    ws = K.workspace()
    K.sampler_step(x=x, eps_c=ec, eps_u=eu, x_out=out, x_out_bf16=outb, update=N.HP_UPDATE_DDIM,
                   t=t, w=6.5, c_sigma=c.c_sigma, c_sqrt_ab=c.c_sqrt_ab,
                   c_sqrt_ab_prev=c.c_sqrt_ab_prev, c_sqrt_1m_ab_prev=c.c_sqrt_1m_ab_prev, ws=ws)
    m = float(ws.m.item())
    xd, ecd, eud = (v.double().cpu().numpy() for v in (x, ec, eu))
    ref = smp.ddim(xd, smp.cfg(ecd, eud, 6.5), t, s.alpha_bars, s.sigmas)
    err = np.abs(out.double().cpu().numpy() - ref).max()
    assert err <= 1e-5 * max(1.0, np.abs(ref).max()), err
    assert torch.equal(outb, out.bfloat16())
    assert abs(m - smp.rel_mae(ecd, eud)) <= 1e-6 * smp.rel_mae(ecd, eud)
    assert int(ws.status.item()) == 0


def test_discrepancy_is_deterministic():
    from paper_2602_21760_b200 import _kernels as K
    n = 3 << 20
    a = torch.randn(n, device="cuda")
    b = torch.randn(n, device="cuda")
    vals = set()
    for _ in range(5):
        ws = K.rel_mae_dev(a, b)
        vals.add(float(ws.m.item()))
    assert len(vals) == 1


def test_device_controller_matches_reference_replays(golden_dir):
    with open(os.path.join(golden_dir, "controller.json")) as fh:
        cases = json.load(fh)
    for c in cases[:60]:
        cfg = hp.SwitchConfig(L=c["L"], g_slope=c["g_slope"], tau_cap=c["tau_cap"], k=c["k"])
        st, labels = hp.replay_series_device([tuple(p) for p in c["pairs"]], cfg)
        assert (st.tau1, st.tau2) == (c["tau1"], c["tau2"]), c["name"]
        assert [l.value for l in labels] == c["labels"], c["name"]


def test_device_controller_sequencing_error():
    cfg = hp.SwitchConfig(L=2, g_slope=1e-3, tau_cap=5, k=2)
    with pytest.raises(hp.SequencingError):
        hp.replay_series_device([(10, 0.5), (8, 0.4)], cfg)


def test_blend_matches_reference_accumulation():
    from paper_2602_21760_b200 import _kernels as K
    rng = np.random.default_rng(3)
    es = [rng.standard_normal(4097) for _ in range(3)]
    fr = (0.5, 0.3, 0.2)
    acc = torch.empty(4097, dtype=torch.float64, device="cuda")
    for d, (f, e) in enumerate(zip(fr, es)):
        K.blend_accumulate(acc, torch.from_numpy(e).cuda(), f, first=d == 0)
    ref = np.zeros(4097)
    for f, e in zip(fr, es):
        ref += f * e
    assert np.array_equal(acc.cpu().numpy(), ref)
