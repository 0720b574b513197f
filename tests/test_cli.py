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
