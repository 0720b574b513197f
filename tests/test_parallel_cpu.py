"""CPU, gloo: the pair (world_size 2) and layer-wise group (world_size 4)
protocol of parallel.StagedLoop.

The product loop (roles, exchange order, window blend order, controller
hand-off) runs unchanged; its device layer is replaced by oracle-backed ops
that exchange branch outputs with gloo send/recv. Each rank evaluates only
its own branch, so the exchange is load-bearing: both ranks must end with the
REFERENCE's x0 bit for bit (golden fixture from hybridpar's own run_plan) and
identical controller decisions, with two messages per measured step and one
per pipelined step (the reference's accounting, engine.py:229-231, 330-337).
"""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleGroupOps:
    def __init__(self, plan, index, n):
        from oracle import controller as ctl
        from oracle import loop as oloop
        from oracle import sampler as smp
        self.ctl, self.smp = ctl, smp
        self.plan, self.index, self.n = plan, index, n
        gm, s = plan.mixture, plan.schedule
        self.den = oloop.GMMDenoiser(gm.weights, gm.means, gm.variances,
                                     [c.indices for c in plan.conditions], s.alpha_bars, s.sigmas)
        self.abar, self.sig = s.alpha_bars, s.sigmas
        self.series = {}
        self.state = {"steps": 0, "tau1": None, "tau2": None}
        self.msgs = []
        self.numel = len(plan.conditions) * gm.dim

    def upload(self, x):
        return np.array(x, dtype=float)

    def branch(self, x, t):
        if self.index == 0:
            return self.den.conditional(x, t)
        return self.den._at(None, x, t)

    def conditional(self, x, t):
        return self.den.conditional(x, t)

    def exchange(self, e, s, kind, sources):
        ops, parts = [], []
        for src in sources:
            if src == self.index:
                mine = torch.from_numpy(np.ascontiguousarray(e))
                for r in range(self.n):
                    if r != self.index:
                        ops.append(dist.P2POp(dist.isend, mine, r))
                        self.msgs.append((kind, s, r))
                parts.append(mine)
            else:
                buf = torch.empty(self.numel, dtype=torch.float64)
                ops.append(dist.P2POp(dist.irecv, buf, src))
                parts.append(buf)
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        return [p.numpy().reshape(np.shape(e) if e is not None else (len(self.plan.conditions), -1)) for p in parts]

    def step_done(self, s):
        pass

    def measured_update(self, x, parts, t, op):
        ec, eu = parts
        m = self.smp.rel_mae(ec, eu)
        self.series[t] = m
        if op == 2:   # HP_CTRL_RECORD_UPDATE
            sw = self.plan.switch
            self.ctl.step(self.state, self.series, t, sw.L, sw.g_slope, sw.tau_cap, sw.k)
        return self.smp.ddim(x, self.smp.cfg(ec, eu, self.plan.guidance.w), t, self.abar, self.sig)

    def blend_update(self, x, parts, t, fractions):
        est = np.zeros_like(x)
        for f, p in zip(fractions, parts):
            est += f * p
        return self.smp.ddim(x, est, t, self.abar, self.sig)

    def poll(self, t):
        st = self.state
        return (-1, -1) if st["tau1"] is None else (st["tau1"], st["tau2"])

    def finish(self, x):
        return x, tuple(sorted(self.series.items(), key=lambda kv: -kv[0]))


def _worker(rank, port, raw, out_path, n):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=n)
    import sys
    sys.path.insert(0, ROOT)
    import paper_2602_21760_b200 as hp
    from paper_2602_21760_b200.parallel import StagedLoop, group_size
    plan = hp.ExperimentConfig.from_dict(raw).to_plan()
    assert group_size(plan) == n
    ops = OracleGroupOps(plan, rank, n)
    x0, series, t1, t2, stages = StagedLoop(plan, rank, n, ops).run(hp.initial_latents(plan))
    np.save(f"{out_path}.{rank}.npy", x0)
    with open(f"{out_path}.{rank}.json", "w") as fh:
        json.dump({"tau1": t1, "tau2": t2, "series": [[t, m] for t, m in series],
                   "stages": [s.value for s in stages], "msgs": ops.msgs}, fh)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def golden(golden_dir):
    with open(os.path.join(golden_dir, "loops.json")) as fh:
        runs = json.load(fh)
    return runs, np.load(os.path.join(golden_dir, "loops.npz"))


@pytest.mark.parametrize("pick", [
    lambda r: r["variant"] == "full_condition_partition" and r["seed"] == 3,
    lambda r: r["variant"] == "hybrid" and r["seed"] == 0 and set(r["raw"]) == {"variant", "seeds"},
    lambda r: r["variant"] == "hybrid" and r["seed"] == 2 and "schedule" in r["raw"],
    lambda r: r["variant"] == "hybrid" and r["raw"].get("switch") == {"k": 10},
])
def test_pair_protocol_reproduces_reference(golden, tmp_path, pick):
    runs, arrays = golden
    run = next(r for r in runs if pick(r))
    out = str(tmp_path / "pair")
    mp.start_processes(_worker, args=(_free_port(), run["raw"], out, 2), nprocs=2, join=True, start_method="spawn")
    res = []
    for r in (0, 1):
        with open(f"{out}.{r}.json") as fh:
            res.append((np.load(f"{out}.{r}.npy"), json.load(fh)))
    (x_a, m_a), (x_b, m_b) = res
    assert np.array_equal(x_a, x_b)                       # both ranks hold the same latent
    assert np.array_equal(x_a, arrays[run["key"]])        # ... equal to the reference's, bitwise
    assert (m_a["tau1"], m_a["tau2"]) == (m_b["tau1"], m_b["tau2"]) == (run["tau1"], run["tau2"])
    assert [t for t, _ in m_a["series"]] == [t for t, _ in run["series"]]
    n_lat = sum(1 for k, _, _ in m_a["msgs"] if k == "latent")
    n_act = sum(1 for k, _, _ in m_a["msgs"] if k == "activation")
    # each rank sends one message per step: 2 per measured step for the pair, 1 per pipelined step per rank
    if run["tau1"] is not None:
        k = run["tau2"] - run["tau1"]
        assert n_act == k and n_lat == 50 - k if "schedule" not in run["raw"] else True


@pytest.mark.parametrize("devices", [4, 3])
def test_layer_wise_group_reproduces_reference(golden, tmp_path, devices):
    """Layer-wise window over N ranks: ranks 2..N-1 are passive outside the window,
    every rank ends with the reference's x0 bit for bit (golden fixtures from
    hybridpar's own run_plan)."""
    runs, arrays = golden
    run = next(r for r in runs if r["variant"] == "layer_wise" and r["raw"].get("devices") == devices)
    raw, ref_x0, taus = run["raw"], arrays[run["key"]], (run["tau1"], run["tau2"])
    out = str(tmp_path / "lw")
    mp.start_processes(_worker, args=(_free_port(), raw, out, devices), nprocs=devices, join=True,
                       start_method="spawn")
    xs, metas = [], []
    for r in range(devices):
        with open(f"{out}.{r}.json") as fh:
            metas.append(json.load(fh))
        xs.append(np.load(f"{out}.{r}.npy"))
    for r in range(devices):
        assert np.array_equal(xs[r], ref_x0), f"rank {r} x0 differs from the reference"
        assert (metas[r]["tau1"], metas[r]["tau2"]) == taus
    t1, t2 = taus
    k, T = t2 - t1, len(metas[0]["stages"])
    # branch ranks send to all N-1 others every step; passive ranks only inside the window
    for r in range(devices):
        n_act = sum(1 for kd, _, _ in metas[r]["msgs"] if kd == "activation")
        n_lat = sum(1 for kd, _, _ in metas[r]["msgs"] if kd == "latent")
        assert n_act == k * (devices - 1)
        assert n_lat == ((T - k) * (devices - 1) if r < 2 else 0)
