"""GPU-measured discrepancy curves of the random-init networks in
the reference's CURVE format, and tau_cap calibrated from them (``calibrate``), with
the reference ``detect`` replay of each curve under the calibrated cap.

    python tools/switch_calibration.py [out_dir] [seeds]

Writes <out_dir>/curve_{sdxl,sd3}_seed{s}.csv (cli ``curve --denoiser ...``),
calibration_{sdxl,sd3}.json (cli ``calibrate``) and detect_{...}.json (cli ``detect``
with the calibrated config). SDXL: T=50, L=12, g=4e-4, k=5; SD3: T=28, L=15,
g=1e-4, k=5 (pipelines.SWITCH).
"""
import contextlib
import io
import json
import os
import sys

sys.path.insert(0, ".")
from paper_2602_21760_b200 import cli, pipelines  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/calibration"
    seeds = [int(s) for s in (sys.argv[2] if len(sys.argv) > 2 else "0,1,2").split(",")]
    os.makedirs(out, exist_ok=True)
    for name, T, key in (("sdxl", 50, "sdxl"), ("sd3", 28, "sd3")):
        sw = pipelines.SWITCH[key]
        paths = []
        den = None
        for s in seeds:
            cfg = {"variant": "serial", "schedule": {"T": T}, "seeds": [s], "condition_batch": 1,
                   "switch": sw}
            cpath = os.path.join(out, f"config_{name}_seed{s}.json")
            with open(cpath, "w") as fh:
                json.dump(cfg, fh)
            csv = os.path.join(out, f"curve_{name}_seed{s}.csv")
            args = cli._parser().parse_args(["curve", "--config", cpath, "--denoiser", name, "--out", csv])
            args._den = den                       # one network per spec (same random-init weights)
            assert args.func(args) == 0
            den = args._den
            paths.append(csv)
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert cli.main(["calibrate", "--config", cpath, "--series", *paths]) == 0
        cal = json.loads(buf.getvalue())
        with open(os.path.join(out, f"calibration_{name}.json"), "w") as fh:
            fh.write(buf.getvalue())
        # the reference detect replay under the calibrated cap
        cfg["switch"] = dict(sw, tau_cap=cal["tau_cap"])
        ccal = os.path.join(out, f"config_{name}_calibrated.json")
        with open(ccal, "w") as fh:
            json.dump(cfg, fh)
        for pth in paths:
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                assert cli.main(["detect", "--config", ccal, "--series", pth]) == 0
            with open(pth.replace("curve_", "detect_").replace(".csv", ".json"), "w") as fh:
                fh.write(buf.getvalue())
        print(name, json.dumps({k: cal[k] for k in ("tau_cap", "configured_tau_cap", "cap_binding")}),
              [c["natural_tau1"] for c in cal["curves"]], flush=True)
        del den


if __name__ == "__main__":
    main()
