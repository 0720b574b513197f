"""GPU (one device, 2-3 processes): the multi-GPU product loop for real.

``parallel.GroupSession`` with ``CudaGroupOps`` (our kernels, IPC-mapped
receive slots, vector-store pushes with system-scope flag releases) runs the
tiny U-Net (BASELINE config 1) as a condition-partitioned pair, as a hybrid
pair (reference-blend and stage-split windows) and as a 3-rank stage-split
layer-wise group, every rank a separate process on cuda:0. Waits are
``wait="host"``: the host polls each flag before enqueueing the consumer, so no
kernel ever waits on another process's kernel (B200_PROFILING.md: such waits on
a shared GPU can hit Xid 109); the multi-GPU mode fuses the same waits into
the kernels.

Each run must reproduce the single-process ``run_plan`` x0 BIT FOR BIT (the
kernels are batch-invariant, so a B=1 branch forward per rank equals the rows
of the B=2 CFG forward) with the same switch schedule, and send exactly the
messages of the protocol: 2 latent messages per measured step; per
steady-state stage-split window step N-1 activations plus one latent.
"""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
T = 20
SW = dict(L=4, g_slope=1e-12, tau_cap=6, k=5)


def _plan(hp, pipelines, den, variant, numerics, n):
    from dataclasses import replace
    from paper_2602_21760_b200.denoiser.weights import TINY
    plan = pipelines.sdxl_plan(TINY, variant=variant, steps=T, seed=3, guidance=5.0, denoiser=den, clock="model",
                               n_devices=n, switch=SW)
    return replace(plan, pipeline_numerics=numerics)


def _denoiser(pipelines):
    from paper_2602_21760_b200.denoiser.weights import TINY, init_weights, synthetic_conditioning, unet_param_specs
    W = init_weights(unet_param_specs(TINY), seed=0, device="cpu")
    cond = synthetic_conditioning(1, TINY.context_len, TINY.cross_dim, TINY.pooled_dim)
    return pipelines.build_sdxl_denoiser(TINY, n_prompts=1, steps=T, weights=W, conditioning=cond)


def _worker(rank, port, n, variant, numerics, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=n)
    torch.cuda.set_device(0)
    try:
        import paper_2602_21760_b200 as hp
        from paper_2602_21760_b200 import pipelines
        from paper_2602_21760_b200.parallel import GroupSession
        den = _denoiser(pipelines)
        plan = _plan(hp, pipelines, den, variant, numerics, n)
        sess = GroupSession(plan, wait="host")
        res = sess.run()
        res2 = sess.run()                          # a second run on the same session (monotonic counters)
        meta = {"tau1": res.tau1, "tau2": res.tau2, "stages": [s.value for s in res.stages],
                "msgs": [[k, nb, s, d] for k, nb, s, d in
                         [(m.kind, m.nbytes, m.step, int(m.dst[3:])) for m in res.trace.messages]],
                "has_x0": res.x0 is not None, "comm": res.comm_bytes}
        if res.x0 is not None:
            np.save(f"{out}.{rank}.npy", res.x0)
            meta["rerun_equal"] = bool(np.array_equal(res.x0, res2.x0))
        if rank == 0:                               # the single-process reference run
            single = hp.run_plan(_plan(hp, pipelines, _denoiser(pipelines), variant, numerics, n))
            np.save(f"{out}.single.npy", single.x0)
            meta["single"] = {"tau1": single.tau1, "tau2": single.tau2,
                              "stages": [s.value for s in single.stages]}
        with open(f"{out}.{rank}.json", "w") as fh:
            json.dump(meta, fh)
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("variant,numerics,n", [("full_condition_partition", "reference_blend", 2),
                                                ("hybrid", "reference_blend", 2),
                                                ("hybrid", "stage_split", 2),
                                                ("layer_wise", "stage_split", 3)])
def test_group_session_bitwise_equals_single_process(tmp_path, variant, numerics, n):
    out = str(tmp_path / "g")
    mp.start_processes(_worker, args=(_port(), n, variant, numerics, out), nprocs=n, join=True,
                       start_method="spawn")
    metas = []
    for r in range(n):
        with open(f"{out}.{r}.json") as fh:
            metas.append(json.load(fh))
    single = np.load(f"{out}.single.npy")
    ref = metas[0]["single"]
    for r in (0, 1):
        x = np.load(f"{out}.{r}.npy")
        assert np.array_equal(x, single), f"rank {r}: max diff {np.abs(x - single).max()}"
        assert metas[r]["rerun_equal"]
        assert (metas[r]["tau1"], metas[r]["tau2"]) == (ref["tau1"], ref["tau2"])
        if variant != "full_condition_partition":          # run_plan keeps no labels for FCP
            assert metas[r]["stages"] == ref["stages"]
    for r in range(2, n):
        assert not metas[r]["has_x0"] and metas[r]["stages"] == ref["stages"]
    t1, t2 = ref["tau1"], ref["tau2"]
    window = range(t1 + 1, t2 + 1) if t1 is not None else range(0)
    for s in range(1, T + 1):
        sent = [(k, r, d) for r in range(n) for k, _, ss, d in metas[r]["msgs"] if ss == s]
        acts = [m for m in sent if m[0] == "activation"]
        lats = sorted((r, d) for k, r, d in sent if k == "latent")
        if s not in window:
            assert not acts and lats == [(0, 1), (1, 0)], (s, sent)       # engine.py:229-231
        elif numerics == "stage_split" and s + n - 1 <= t2 and s > t1 + 1:
            assert len(acts) == n - 1 and all(d == r - 1 for _, r, d in acts), (s, acts)
            # dev0 hands x_{t-1} to stage 0's rank while stage 0 still runs next step
            want = [(0, n - 1)] if (n == 2 or s + 1 + n - 1 <= t2) else []
            assert lats == want, (s, lats)
