"""Stage-split pipeline numerics (``pipeline_numerics="stage_split"``).

north_star (iii): in the switched-in pipeline window the denoiser is split
into N consecutive stages, one per GPU of the group, and each stage runs on
the boundary state its upstream stage produced at the PREVIOUS step, so all
stages work concurrently (AsyncDiff-style asynchronous denoising, PAPER.md:45;
layer-wise extension PAPER.md:395, :673). The reference's own window is a
surrogate (engine.py:254-261: full-network evaluations at stale latents,
blended) whose timing nevertheless charges f_d * C per device and
N-1 activation hops (engine.py:307-337) -- i.e. it models exactly this split.

Conventions (shared by the engine, ``parallel.py`` and the CPU restatement
in ``oracle/stage_ref.py``):

* the network is a list of units (``UNet.units`` / ``MMDiT.units``); stage j
  (network order, j = 0 is the input side) owns units [cuts[j], cuts[j+1]);
* group index d hosts network stage j = N-1-d: dev0 runs the LAST stage and
  the sampler update (the reference's assembler, the end of its fill chain
  engine.py:339-344), dev N-1 the first stage;
* a device's compute share is ``segment_fractions[d]`` (engine.py:325/332),
  so network stage j gets fraction ``segment_fractions[N-1-j]`` and the cuts
  are the unit boundaries whose cumulative FLOPs come closest to the
  cumulative fractions;
* boundary state j (the input of stage j >= 1) = the activation plus every
  U-Net skip tensor pushed but not yet popped at cut j (the MMDiT: the joint
  token buffer);
* window step at timestep t: stage 0 runs on x_t; stage j >= 1 on boundary
  state j produced at the previous step; every stage embeds the current t;
  the last stage's output is the (unguided) eps estimate;
* fill: on the first window step boundary state j comes from the conditional
  branch of the last measured step's forward (the exact forward at x_{t+1}),
  recorded at the cuts -- AsyncDiff's warm-up hand-over;
* k = 0 (no window) is bit-identical to full condition partitioning.
"""
from __future__ import annotations

import torch

from .errors import PlanError


def network_fractions(segment_fractions) -> tuple:
    """Per-network-stage compute fractions (stage j on group index N-1-j)."""
    return tuple(reversed(tuple(segment_fractions)))


def stage_cuts(unit_flops, fractions) -> tuple:
    """Unit indices (c_1 < ... < c_{N-1}) splitting the forward into N stages whose
    FLOP shares approximate ``fractions`` (network order). Each stage gets >= 1 unit."""
    U = len(unit_flops)
    N = len(fractions)
    if N < 2:
        raise PlanError("a stage split needs >= 2 stages")
    if U < N:
        raise PlanError(f"network has {U} units, cannot split into {N} stages")
    total = float(sum(unit_flops))
    cum = [0.0]
    for f in unit_flops:
        cum.append(cum[-1] + f)
    cuts = []
    target = 0.0
    prev = 0
    for j in range(1, N):
        target += fractions[j - 1] * total
        lo, hi = prev + 1, U - (N - j)          # leave >= 1 unit for every later stage
        best = min(range(lo, hi + 1), key=lambda c: (abs(cum[c] - target), c))
        cuts.append(best)
        prev = best
    return tuple(cuts)


def stage_bounds(cuts, n_units) -> list:
    edges = (0,) + tuple(cuts) + (n_units,)
    return [(edges[j], edges[j + 1]) for j in range(len(edges) - 1)]


# ---- boundary states -------------------------------------------------------------

def state_tensors(state: dict) -> list:
    """The tensors of a boundary state in a fixed order (U-Net: h then the skip
    stack bottom-up; MMDiT: X)."""
    if "X" in state:
        return [state["X"]]
    return [state["h"]] + list(state["skips"])


def state_rows(state: dict, lo: int, hi: int) -> dict:
    """The rows of images [lo, hi) of a batched boundary state (views)."""
    n = state["n"] if "n" in state else state["X"].shape[0]
    if "X" in state:
        return {"X": state["X"][lo:hi], "hw": state["hw"]}

    def rows(t):
        per = t.shape[0] // n
        return t[lo * per:hi * per]
    return {"h": rows(state["h"]), "skips": [rows(s) for s in state["skips"]], "hw": state["hw"], "n": hi - lo}


class Boundary:
    """One boundary state in ONE contiguous bf16 buffer (the unit of hand-off: a
    single message over NVLink), with views shaped like the recorded state."""

    def __init__(self, like: dict, device):
        self.kind = "X" if "X" in like else "unet"
        self.meta = {k: v for k, v in like.items() if k in ("hw", "n")}
        tens = state_tensors(like)
        self.shapes = [tuple(t.shape) for t in tens]
        sizes = [t.numel() for t in tens]
        padded = [n + (-n) % 8 for n in sizes]      # every view 16-byte aligned (vector copies)
        self.buf = torch.zeros(sum(padded), dtype=torch.bfloat16, device=device)
        self.views, o = [], 0
        for shp, n, p in zip(self.shapes, sizes, padded):
            self.views.append(self.buf[o:o + n].view(shp))
            o += p
        self.nbytes = self.buf.numel() * 2

    def state(self) -> dict:
        if self.kind == "X":
            return {"X": self.views[0], **self.meta}
        return {"h": self.views[0], "skips": list(self.views[1:]), **self.meta}

    def load(self, state: dict) -> None:
        """Copy a (same-shaped) boundary state into the buffer (stream-ordered)."""
        for v, t in zip(self.views, state_tensors(state)):
            v.copy_(t)
