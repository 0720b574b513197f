"""The harness (paper_2602_21760_b200.cli) against outputs of the reference's
own CLI (tests/golden/cli, produced by oracle/gen_golden.py --cli)."""
import json
import os

import numpy as np
import pytest

from paper_2602_21760_b200 import cli
from paper_2602_21760_b200.errors import SeriesParseError


@pytest.fixture(scope="module")
def gold(golden_dir):
    d = os.path.join(golden_dir, "cli")
    with open(os.path.join(d, "stdout.json")) as fh:
        return d, json.load(fh)


def test_headers_match_reference():
    assert cli.CURVE_HEADER == "t,rel_mae,score_ratio,band_lo,band_hi,is_argmin"
    assert cli.SWEEP_HEADER == "k,status,latency_s,speedup,fidelity_l1,psnr_analog"
    assert cli.TRACE_HEADER == "event,step,stage,device,src,dst,label,kind,start,end,nbytes"


def test_detect_on_reference_curve_is_byte_identical(gold, capsys):
    d, out = gold
    assert cli.main(["detect", "--series", os.path.join(d, "curve.csv")]) == 0
    assert capsys.readouterr().out == out["detect"]


def test_series_parse_errors(tmp_path, capsys):
    p = tmp_path / "bad.csv"
    p.write_text("t,rel_mae\n50,0.1\n49,abc\n")
    with pytest.raises(SeriesParseError) as e:
        cli.read_series_csv(str(p))
    assert e.value.line == 3
    p.write_text("")
    assert cli.main(["detect", "--series", str(p)]) == 1
    err = json.loads(capsys.readouterr().err)
    assert err["error"] == "SeriesParseError"
    p.write_text("x,y\n1,2\n")
    with pytest.raises(SeriesParseError) as e:
        cli.read_series_csv(str(p))
    assert e.value.line == 1


def _rows(path):
    with open(path) as fh:
        return [ln.rstrip("\n") for ln in fh]


@pytest.mark.gpu
def test_simulate_matches_reference(gold, tmp_path, capsys):
    d, out = gold
    assert cli.main(["simulate", "--out", str(tmp_path)]) == 0
    mine = json.loads(capsys.readouterr().out)
    ref = json.loads(out["simulate"])
    assert set(mine) == set(ref)
    for k in ("latency_s", "speedup", "comm_bytes", "tau1", "tau2"):
        assert mine[k] == ref[k], k
    for k in ("fidelity_l1", "fidelity_l2", "psnr_analog"):
        assert abs(mine[k] - ref[k]) <= 1e-9 * max(1.0, abs(ref[k])), k
    # model-clock trace: byte-identical rows
    assert _rows(tmp_path / "trace.csv") == _rows(os.path.join(d, "sim", "trace.csv"))


@pytest.mark.gpu
def test_curve_matches_reference(gold, tmp_path):
    d, _ = gold
    assert cli.main(["curve", "--out", str(tmp_path / "c.csv")]) == 0
    mine = np.genfromtxt(tmp_path / "c.csv", delimiter=",", names=True)
    ref = np.genfromtxt(os.path.join(d, "curve.csv"), delimiter=",", names=True)
    assert np.array_equal(mine["t"], ref["t"]) and np.array_equal(mine["is_argmin"], ref["is_argmin"])
    for col in ("rel_mae", "score_ratio", "band_lo", "band_hi"):
        np.testing.assert_allclose(mine[col], ref[col], rtol=1e-9, atol=1e-12)


@pytest.mark.gpu
def test_sweep_matches_reference(gold, tmp_path, capsys):
    d, out = gold
    assert cli.main(["sweep", "--config", os.path.join(d, "small.json"), "--k", "0,2,4,9"]) == 0
    mine = capsys.readouterr().out.splitlines()
    ref = out["sweep_small"].splitlines()
    assert mine[0] == ref[0] and len(mine) == len(ref)
    for a, b in zip(mine[1:], ref[1:]):
        fa, fb = a.split(","), b.split(",")
        assert fa[:2] == fb[:2]
        for x, y in zip(fa[2:], fb[2:]):
            if x or y:
                assert abs(float(x) - float(y)) <= 1e-9 * max(1.0, abs(float(y))), (a, b)


def test_calibrate_on_reference_curve(gold, capsys):
    """tau_cap calibration on the reference's own curve: the cap
    lands one step past the natural firing, and the detect replay under it fires
    naturally at the same step (the cap is not what switches)."""
    d, out = gold
    path = os.path.join(d, "curve.csv")
    assert cli.main(["calibrate", "--series", path, path]) == 0
    cal = json.loads(capsys.readouterr().out)
    c = cal["curves"][0]
    if cal["cap_binding"]:
        assert c["natural_tau1"] is None and cal["tau_cap"] == cal["configured_tau_cap"]
        return
    assert cal["tau_cap"] == min(c["natural_tau1"] + 1, cal["T"] - cal["k"] - 1)
    assert c["detect"]["tau1"] == c["natural_tau1"]
    assert c["detect"]["tau2"] == c["natural_tau1"] + cal["k"]
    assert 0.0 <= c["slope_at_firing"] < cal["g_slope"] and c["slope_margin"] > 0


def test_calibrate_cap_binding_on_flat_start(tmp_path, capsys):
    """A curve whose slope never enters [0, g) keeps the configured cap."""
    p = tmp_path / "c.csv"
    p.write_text("t,rel_mae\n" + "".join(f"{t},{0.5 + 0.01 * t}\n" for t in range(50, 0, -1)))
    assert cli.main(["calibrate", "--series", str(p)]) == 0
    cal = json.loads(capsys.readouterr().out)
    assert cal["cap_binding"] and cal["tau_cap"] == cal["configured_tau_cap"]
    assert cal["curves"][0]["detect"]["tau1"] == cal["configured_tau_cap"]


@pytest.mark.gpu
def test_curve_and_calibrate_on_tiny_unet(tmp_path, capsys):
    """`curve --denoiser tiny` (BASELINE config 1 network at the seam, latent-shaped
    prior and the network's own schedule) then `calibrate` over two seeds."""
    paths = []
    for s in (0, 1):
        cfg = tmp_path / f"c{s}.json"
        cfg.write_text(json.dumps({"variant": "serial", "schedule": {"T": 20}, "seeds": [s],
                                   "condition_batch": 1, "switch": {"L": 4, "g_slope": 4e-4, "tau_cap": 8, "k": 5}}))
        out = tmp_path / f"curve{s}.csv"
        assert cli.main(["curve", "--config", str(cfg), "--denoiser", "tiny", "--out", str(out)]) == 0
        rows = out.read_text().splitlines()
        assert rows[0] == cli.CURVE_HEADER and len(rows) == 21
        ts = [int(r.split(",")[0]) for r in rows[1:]]
        assert ts == list(range(20, 0, -1))
        assert all(float(r.split(",")[1]) > 0 for r in rows[1:])
        paths.append(str(out))
    capsys.readouterr()
    assert cli.main(["calibrate", "--config", str(cfg), "--series", *paths]) == 0
    cal = json.loads(capsys.readouterr().out)
    assert cal["T"] == 20 and 1 <= cal["tau_cap"] <= 20 - 5 - 1
    for c in cal["curves"]:
        assert c["detect"]["tau1"] <= cal["tau_cap"]
