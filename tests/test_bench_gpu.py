"""GPU: bench.py's own code paths run end to end (the driver runs them on other boxes):
the one-GPU line carries every contract key, and the multi-process pairs path runs as two
ranks sharing GPU 0 (gloo, host-side flag waits: HP_BENCH_SHARED_GPU=1) and prints one
line with no error."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"}


def _line(out):
    return json.loads(out.strip().splitlines()[-1])


def test_bench_single_gpu_tiny():
    r = subprocess.run([sys.executable, "bench.py", "--spec", "tiny", "--steps", "2", "--no-cpu-baseline"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _line(r.stdout)
    assert KEYS <= set(line), KEYS - set(line)
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    assert line["forward_b1"]["predicted_pair_latency_s"] > 0


def test_bench_pairs_two_ranks_shared_gpu():
    env = dict(os.environ, HP_BENCH_SHARED_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
                        "--steps", "1", "--warmup", "3", "--spec", "tiny"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _line(r.stdout)
    assert "error" not in line, line
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "pairsx2"
    assert line["config"]["images"] == 1 and line["value"] > 0
