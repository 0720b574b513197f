"""Execution plans and their runners on B200.

Drop-in for the reference engine (engine.py:35-396): same ``PlanVariant``,
``ExecutionPlan`` validation, ``RunResult`` fields, runner names and
``run_plan`` dispatch. What changes is where the numbers come from:

* every step's numerics run on the GPU — the denoiser seam produces both
  branch outputs, then ONE fused launch (``hp_sampler_step``: CFG combine,
  DDIM/Euler update, rel-MAE partials, fixed-order finalize, series record and
  the Algorithm-1 controller in the last CTA) advances the latent;
* the host learns the switch point by polling a mapped pinned mirror the
  kernel publishes, and only on steps where the decision can change
  (s in [min(L+1, tau_cap), tau1]); every other step is launch-and-go;
* timing comes from either the reference's model clock (``clock="model"``,
  the affine link of trace.py, so closed-form latencies match the reference)
  or CUDA events (``clock="device"``). Real multi-GPU execution of the pair,
  layer-wise and batch-level plans lives in ``parallel.py``.

Numeric contract (engine.py:1-20): measured steps are exact guided steps, so
serial, full condition partitioning and an empty-window hybrid produce the
same latents bit for bit; pipelined steps use the segment-blended conditional
estimate of engine.py:254-261 (``pipeline_numerics="reference_blend"``), or
the network split into stages fed with previous-step boundary states
(``"stage_split"``, stages.py; north_star iii).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _kernels as K
from . import _native as N
from .errors import PlanError, from_status
from .mixture import Condition, GaussianMixture, eps_prediction, fm_velocity, sample_x0
from .monitor import DiscrepancySeries, Stage, StageState, SwitchConfig, update_controller
from .schedules import GuidanceParams, NoiseSchedule, StepCoefficients, check_euler
from .trace import LinkSpec, RunTrace, Timeline, account_comm


class PlanVariant(enum.Enum):
    SERIAL = "serial"
    FULL_CONDITION_PARTITION = "full_condition_partition"
    HYBRID = "hybrid"
    BATCH_LEVEL = "batch_level"
    LAYER_WISE = "layer_wise"


STAGED = (PlanVariant.HYBRID, PlanVariant.BATCH_LEVEL, PlanVariant.LAYER_WISE)
CLOCKS = ("model", "device")
SAMPLERS = ("ddim", "euler")
PIPELINE_NUMERICS = ("reference_blend", "stage_split")


@dataclass(frozen=True)
class ExecutionPlan:
    """Model, schedule, devices and strategy of one run.

    Fields up to ``cfg_batching_factor`` are the reference's (engine.py:46-59);
    the rest are B200 extensions with defaults that keep reference behaviour.
    """

    variant: PlanVariant
    schedule: NoiseSchedule
    mixture: GaussianMixture
    conditions: tuple
    guidance: GuidanceParams
    devices: tuple
    link: LinkSpec
    seed: int
    switch: SwitchConfig | None = None
    segment_fractions: tuple | None = None
    cfg_batching_factor: float = 2.0
    denoiser: object | None = None        # None -> analytic GMM on the GPU
    clock: str = "model"
    sampler: str = "ddim"
    pipeline_numerics: str = "reference_blend"

    def __post_init__(self):
        if not self.conditions:
            raise PlanError("plan needs at least one condition")
        K_ = self.mixture.n_components
        for c in self.conditions:
            if max(c.indices) >= K_:
                raise PlanError(f"condition {c.indices} exceeds mixture components")
        if not isinstance(self.seed, int) or self.seed < 0:
            raise PlanError(f"seed must be an integer >= 0, got {self.seed!r}")
        if not 1.0 <= self.cfg_batching_factor <= 2.0:
            raise PlanError(f"cfg_batching_factor must lie in [1, 2], got {self.cfg_batching_factor}")
        if self.clock not in CLOCKS:
            raise PlanError(f"clock must be one of {CLOCKS}, got {self.clock!r}")
        if self.sampler not in SAMPLERS:
            raise PlanError(f"sampler must be one of {SAMPLERS}, got {self.sampler!r}")
        if self.pipeline_numerics not in PIPELINE_NUMERICS:
            raise PlanError(f"unknown pipeline_numerics {self.pipeline_numerics!r}")
        if (self.pipeline_numerics == "stage_split" and self.variant in STAGED
                and not hasattr(self.denoiser, "enable_stage_split")):
            raise PlanError("pipeline_numerics='stage_split' needs a layered network denoiser "
                            "(the analytic GMM has no stages)")
        nd = len(self.devices)
        v = self.variant
        if v is PlanVariant.SERIAL:
            if nd < 1:
                raise PlanError("serial plan needs one device")
        elif v is PlanVariant.FULL_CONDITION_PARTITION:
            if nd != 2:
                raise PlanError(f"condition partitioning needs exactly 2 devices, got {nd}")
        elif v in (PlanVariant.HYBRID, PlanVariant.LAYER_WISE):
            if v is PlanVariant.HYBRID and nd != 2:
                raise PlanError(f"hybrid plan needs exactly 2 devices, got {nd}")
            if v is PlanVariant.LAYER_WISE and nd < 2:
                raise PlanError(f"layer-wise plan needs >= 2 devices, got {nd}")
            self._validate_switch()
            segs = 2 if v is PlanVariant.HYBRID else nd
            fr = self.segment_fractions
            if fr is None:
                fr = tuple(1.0 / segs for _ in range(segs))
                object.__setattr__(self, "segment_fractions", fr)
            if len(fr) != segs:
                raise PlanError(f"segment_fractions must have {segs} entries, got {len(fr)}")
            if min(fr) <= 0 or abs(sum(fr) - 1.0) > 1e-9:
                raise PlanError(f"segment_fractions must be positive and sum to 1, got {fr}")
        elif v is PlanVariant.BATCH_LEVEL:
            if nd < 2 or nd % 2:
                raise PlanError(f"batch-level plan needs an even device count >= 2, got {nd}")
            self._validate_switch()

    def _validate_switch(self):
        sw, T = self.switch, self.schedule.T
        if sw is None:
            raise PlanError("staged plan needs a switch config")
        if sw.tau_cap < 1:
            raise PlanError("staged plan needs tau_cap >= 1 (at least one measured step)")
        if sw.L >= T:
            raise PlanError(f"slope window L={sw.L} must be < T={T}")
        if sw.tau_cap > T:
            raise PlanError(f"tau_cap={sw.tau_cap} exceeds T={T}")
        if sw.k >= 1 and sw.k >= T - sw.tau_cap:
            raise PlanError(f"window k={sw.k} infeasible: need k < T - tau_cap = {T - sw.tau_cap}")


@dataclass(frozen=True)
class RunResult:
    x0: np.ndarray
    latency_s: float
    comm_bytes: int
    speedup: float
    throughput_samples_per_s: float
    tau1: int | None
    tau2: int | None
    trace: RunTrace
    series: tuple
    per_sample: tuple | None = None
    stages: tuple = ()                     # per-step stage labels (extension)
    x0_device: object = field(default=None, repr=False, compare=False)


def serial_latency_ref(plan: ExecutionPlan) -> float:
    """T steps of rho * C accumulated one by one (engine.py:134-144)."""
    per_step = plan.cfg_batching_factor * plan.devices[0].branch_step_cost
    total = 0.0
    for _ in range(plan.schedule.T):
        total += per_step
    return total


def initial_latents(plan: ExecutionPlan) -> np.ndarray:
    """Seeded x_T, one row per condition, bit-identical to engine.py:147-161.

    For the Euler (flow-matching) sampler the same draws are combined on the
    straight path x_1 = x0 + e used by mixture.fm_velocity.
    """
    rng = np.random.default_rng(plan.seed)
    gm, sched = plan.mixture, plan.schedule
    rows = len(plan.conditions)
    x0 = np.empty((rows, gm.dim))
    for i, c in enumerate(plan.conditions):
        x0[i] = sample_x0(gm, c, rng, 1)[0]
    noise = rng.standard_normal((rows, gm.dim))
    if plan.sampler == "euler":
        return x0 + noise
    ab = sched.alpha_bar(sched.T)
    return np.sqrt(ab) * x0 + np.sqrt(1.0 - ab) * noise


def condition_groups(conditions) -> list:
    """Distinct conditions with the batch rows they own, in first-seen order."""
    order: dict = {}
    for row, c in enumerate(conditions):
        order.setdefault(c.indices, []).append(row)
    return [(Condition(idx), np.asarray(rs)) for idx, rs in order.items()]


class MixtureDenoiser:
    """Seam adapter for the analytic GMM (the reference's only denoiser)."""

    latent_dtype = torch.float64
    eps_dtype = torch.float64
    wants_bf16_input = False

    def __init__(self, plan: ExecutionPlan):
        self.gm, self.sched, self.sampler = plan.mixture, plan.schedule, plan.sampler
        self.groups = [(c, torch.as_tensor(r)) for c, r in condition_groups(plan.conditions)]

    def input_slot(self):
        return None

    def load_input(self, x):
        return None

    def _one(self, cond, x, t):
        if self.sampler == "euler":
            return fm_velocity(self.gm, cond, x, t / self.sched.T)
        return eps_prediction(self.gm, cond, self.sched, x, t)

    def conditional(self, x, t, x_bf16=None):
        out = torch.empty_like(x)
        for cond, rows in self.groups:
            r = rows.to(x.device)
            out[r] = self._one(cond, x[r], t)
        return out

    def branches(self, x, t, x_bf16=None):
        eps_u = self._one(None, x, t)
        return self.conditional(x, t), eps_u

    def unconditional(self, x, t, x_bf16=None):
        return self._one(None, x, t)


class _StepRunner:
    """Per-run GPU state: coefficient table, workspace, controller, mirror."""

    def __init__(self, plan: ExecutionPlan):
        N.require_cuda()
        self.plan = plan
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.den = plan.denoiser if plan.denoiser is not None else MixtureDenoiser(plan)
        self.ws = K.workspace(self.dev)
        self.ctrl = K.ctrl_alloc(self.dev)
        sw = plan.switch
        if sw is not None:
            K.ctrl_init(self.ctrl, sw.L, sw.g_slope, sw.tau_cap, sw.k, plan.schedule.T)
        else:
            K.ctrl_init(self.ctrl, 1, 1.0, plan.schedule.T, 0, plan.schedule.T)
        self.mirror = K.PinnedMirror()
        self._sw = sw
        T = plan.schedule.T
        if plan.sampler == "euler":
            self.coef = {t: None for t in range(1, T + 1)}
            for t in range(1, T + 1):
                check_euler(t / T, 1.0 / T)
        else:
            self.coef = {t: StepCoefficients.ddim(plan.schedule, t) for t in range(1, T + 1)}
        self.update = N.HP_UPDATE_EULER if plan.sampler == "euler" else N.HP_UPDATE_DDIM
        self.split = plan.pipeline_numerics == "stage_split" and plan.variant in STAGED
        if self.split:
            from .stages import network_fractions, stage_cuts
            fr = plan.segment_fractions or (0.5, 0.5)
            self.den.enable_stage_split(stage_cuts(self.den.net.unit_flops, network_fractions(fr)))

    def reset(self):
        """Fresh controller + mirror for another run on the same runner."""
        torch.cuda.synchronize()
        T = self.plan.schedule.T
        sw = self._sw
        if sw is not None:
            K.ctrl_init(self.ctrl, sw.L, sw.g_slope, sw.tau_cap, sw.k, T)
        else:
            K.ctrl_init(self.ctrl, 1, 1.0, T, 0, T)
        self.mirror.view.seq = -1
        torch.cuda.synchronize()

    def upload(self, x_host):
        if isinstance(x_host, torch.Tensor):
            x = x_host.to(self.dev, non_blocking=True)
        else:
            x = torch.from_numpy(np.ascontiguousarray(x_host)).to(self.dev, non_blocking=True)
        x = x.to(self.den.latent_dtype)
        xb = None
        if self.den.wants_bf16_input:
            self.den.load_input(x)
            xb = self.den.input_slot()
        return x, xb

    def _advance(self, x, xb, eps_c, eps_u, t, ctrl_op, discrepancy=True):
        out = torch.empty_like(x)
        # the next bf16 latent goes straight into the denoiser's (graph) input
        outb = self.den.input_slot() if self.den.wants_bf16_input else None
        c = self.coef[t]
        kw = {}
        if c is not None:
            kw = dict(c_sigma=c.c_sigma, c_sqrt_ab=c.c_sqrt_ab, c_sqrt_ab_prev=c.c_sqrt_ab_prev,
                      c_sqrt_1m_ab_prev=c.c_sqrt_1m_ab_prev)
        K.sampler_step(x=x, eps_c=eps_c, eps_u=eps_u, x_out=out, x_out_bf16=outb,
                       update=self.update, t=t, w=self.plan.guidance.w,
                       dt=1.0 / self.plan.schedule.T, ws=self.ws, discrepancy=discrepancy,
                       ctrl=self.ctrl, ctrl_op=ctrl_op, mirror_ptr=self.mirror.ptr, **kw)
        return out, outb

    def measured(self, x, xb, t, ctrl_op):
        eps_c, eps_u = self.den.branches(x, t, xb)
        return self._advance(x, xb, eps_c, eps_u, t, ctrl_op)

    def pipelined(self, history, fractions, t):
        """Blend sum_d f_d eps_c(history[min(d, len-1)], t) then an unguided step."""
        x, xb = history[0]
        acc = None
        for d, f in enumerate(fractions):
            hx, _ = history[min(d, len(history) - 1)]
            e = self.den.conditional(hx, t)
            if acc is None:
                acc = torch.empty(e.shape, dtype=x.dtype, device=x.device)
            K.blend_accumulate(acc, e, f, first=(d == 0))
        return self._advance(x, xb, acc, None, t, N.HP_CTRL_NONE)

    def pipelined_split(self, x, xb, t, fill, steps_left=None):
        """Stage-split window step on one device (stages.py): every stage on its
        previous-step input, then an unguided update."""
        if fill:
            self.den.window_fill()
        eps = self.den.window_step(x, t, steps_left)
        return self._advance(x, xb, eps, None, t, N.HP_CTRL_NONE)

    def poll(self, t):
        mr = self.mirror.wait_step(t)
        if mr.status != 0:
            raise from_status(mr.status, f"step at t={t}")
        return mr

    def finish(self, x, to_host=True):
        host = K.ctrl_read(self.ctrl)
        if host.status != 0:
            raise from_status(host.status, "denoising loop")
        series = tuple((t, float(host.m[t])) for t in range(self.plan.schedule.T, -1, -1)
                       if host.has[t])
        x0 = x.to(torch.float64).cpu().numpy() if to_host else None
        return x0, series


# ---- model-clock timing (reference cost model, engine.py:217-231, 307-337) ----

def _model_measured(plan, tl: Timeline, s, stage, a_clock, b_avail):
    d0, d1 = plan.devices[0], plan.devices[1]
    a_done = tl.busy(d0.name, a_clock, d0.branch_step_cost, s, stage, "eps_c")
    b_done = tl.busy(d1.name, b_avail, d1.branch_step_cost, s, stage, "eps_u")
    eps_u_at_a = tl.send(d1.name, d0.name, "latent", b_done, s)
    combined = max(a_done, eps_u_at_a)
    return combined, tl.send(d0.name, d1.name, "latent", combined, s)


def _model_pipelined(plan, tl: Timeline, s, fill, a_clock, b_avail):
    devs, fr = plan.devices, plan.segment_fractions
    n = len(devs)
    tag = Stage.PARALLELISM.value
    if fill:
        # sequential chain from the last segment down to the assembler
        t_cur = b_avail if n == 2 else a_clock   # only segment 1 waits for the partner
        for d in range(n - 1, 0, -1):
            done = tl.busy(devs[d].name, t_cur, fr[d] * devs[d].branch_step_cost, s, tag, f"segment_{d}")
            t_cur = tl.send(devs[d].name, devs[d - 1].name, "activation", done, s)
        return tl.busy(devs[0].name, t_cur, fr[0] * devs[0].branch_step_cost, s, tag, "segment_0")
    ends = []
    for d in range(1, n):
        start = max(b_avail, a_clock) if d == 1 else a_clock
        done = tl.busy(devs[d].name, start, fr[d] * devs[d].branch_step_cost, s, tag, f"segment_{d}")
        ends.append(tl.send(devs[d].name, devs[0].name, "activation", done, s))
    ends.insert(0, tl.busy(devs[0].name, a_clock, fr[0] * devs[0].branch_step_cost, s, tag, "segment_0"))
    return max(ends)


class _Clock:
    """Either the model Timeline or CUDA events on this device."""

    def __init__(self, plan: ExecutionPlan):
        self.plan = plan
        self.model = plan.clock == "model"
        self.tl = Timeline(plan.link)
        self.a, self.b = 0.0, 0.0
        if not self.model:
            self.ev0 = torch.cuda.Event(enable_timing=True)
            self.ev0.record()
            self.events = []

    def serial_step(self, s):
        if self.model:
            d = self.plan.devices[0]
            self.a = self.tl.busy(d.name, self.a, self.plan.cfg_batching_factor * d.branch_step_cost,
                                  s, "", "cfg_branches")
        else:
            self._mark(s, "", "cfg_branches")

    def measured_step(self, s, stage):
        if self.model:
            self.a, self.b = _model_measured(self.plan, self.tl, s, stage, self.a, self.b)
        else:
            self._mark(s, stage, "measured")

    def pipelined_step(self, s, fill):
        if self.model:
            self.a = _model_pipelined(self.plan, self.tl, s, fill, self.a, self.b)
            self.b = self.a
        else:
            self._mark(s, Stage.PARALLELISM.value, "pipelined")

    def _mark(self, s, stage, label):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.append((ev, s, stage, label))

    def result(self):
        if self.model:
            return self.tl.trace
        from .trace import BusyInterval
        torch.cuda.synchronize()
        tr = RunTrace()
        prev = 0.0
        name = self.plan.devices[0].name
        for ev, s, stage, label in self.events:
            end = self.ev0.elapsed_time(ev) / 1e3
            tr.busy.append(BusyInterval(name, prev, end, s, stage, label))
            prev = end
        return tr


def _result(plan, x0, trace, series, tau1=None, tau2=None, stages=(), x_dev=None):
    latency = trace.makespan()
    ref = serial_latency_ref(plan)
    speed = ref / latency if latency > 0 else float("inf")
    return RunResult(x0=x0, latency_s=latency, comm_bytes=account_comm(trace), speedup=speed,
                     throughput_samples_per_s=1.0 / latency if latency > 0 else float("inf"),
                     tau1=tau1, tau2=tau2, trace=trace, series=series, stages=tuple(stages),
                     x0_device=x_dev)


def _run_exact(plan: ExecutionPlan, serial: bool, x_init=None, to_host=True) -> RunResult:
    st = _StepRunner(plan)
    clock = _Clock(plan)
    x, xb = st.upload(initial_latents(plan) if x_init is None else x_init)
    T = plan.schedule.T
    for s in range(1, T + 1):
        t = T - s + 1
        x, xb = st.measured(x, xb, t, N.HP_CTRL_RECORD)
        if serial:
            clock.serial_step(s)
        else:
            clock.measured_step(s, "")
    x0, series = st.finish(x, to_host)
    return _result(plan, x0, clock.result(), series, x_dev=x)


def run_serial(plan: ExecutionPlan) -> RunResult:
    """Both branches on one device, every step exact (engine.py:195-214)."""
    if plan.variant is not PlanVariant.SERIAL:
        raise PlanError(f"run_serial got a {plan.variant.value} plan")
    return _run_exact(plan, serial=True)


def run_full_condition_partition(plan: ExecutionPlan) -> RunResult:
    """Condition-partitioned numerics (identical to serial) on one process.

    For the real two-GPU execution see ``parallel.run_pair``.
    """
    if plan.variant is not PlanVariant.FULL_CONDITION_PARTITION:
        raise PlanError(f"run_full_condition_partition got a {plan.variant.value} plan")
    return _run_exact(plan, serial=False)


def _run_staged(plan: ExecutionPlan, fractions, x_init=None, to_host=True) -> RunResult:
    st = _StepRunner(plan)
    clock = _Clock(plan)
    sw = plan.switch
    T = plan.schedule.T
    n = len(plan.devices)
    x, xb = st.upload(initial_latents(plan) if x_init is None else x_init)
    host = StageState()
    no_series = DiscrepancySeries()
    first_poll = min(sw.L + 1, sw.tau_cap)   # the slope cannot fire earlier
    history: list = []
    prev = Stage.WARM_UP
    stages = []
    for s in range(1, T + 1):
        t = T - s + 1
        history.insert(0, (x, xb))
        del history[n:]
        if host.tau1 is None:
            x, xb = st.measured(x, xb, t, N.HP_CTRL_RECORD_UPDATE)
            if s >= first_poll:
                mr = st.poll(t)
                if mr.tau1 >= 0:
                    host.tau1, host.tau2 = mr.tau1, mr.tau2
            host.steps_done, host.last_t, host.stage = s, t, Stage.WARM_UP
            clock.measured_step(s, host.stage.value)
        else:
            update_controller(host, no_series, t, sw)
            if host.stage is Stage.PARALLELISM:
                fill = prev is not Stage.PARALLELISM
                if st.split:
                    x, xb = st.pipelined_split(x, xb, t, fill, host.tau2 - s)
                else:
                    x, xb = st.pipelined(history, fractions, t)
                clock.pipelined_step(s, fill=fill)
            else:
                x, xb = st.measured(x, xb, t, N.HP_CTRL_RECORD)
                clock.measured_step(s, host.stage.value)
        stages.append(host.stage)
        prev = host.stage
    x0, series = st.finish(x, to_host)
    return _result(plan, x0, clock.result(), series, host.tau1, host.tau2, stages, x_dev=x)


def run_hybrid(plan: ExecutionPlan) -> RunResult:
    """Adaptive three-stage run on two devices (engine.py:340-344)."""
    if plan.variant is not PlanVariant.HYBRID:
        raise PlanError(f"run_hybrid got a {plan.variant.value} plan")
    return _run_staged(plan, plan.segment_fractions)


def run_layer_wise(plan: ExecutionPlan) -> RunResult:
    """Staged run with the window split over N segment devices (engine.py:347-355)."""
    if plan.variant is not PlanVariant.LAYER_WISE:
        raise PlanError(f"run_layer_wise got a {plan.variant.value} plan")
    return _run_staged(plan, plan.segment_fractions)


def run_batch_level(plan: ExecutionPlan) -> RunResult:
    """N/2 independent hybrid pairs, pair i seeded seed + i (engine.py:358-383)."""
    if plan.variant is not PlanVariant.BATCH_LEVEL:
        raise PlanError(f"run_batch_level got a {plan.variant.value} plan")
    pairs = len(plan.devices) // 2
    results, merged = [], RunTrace()
    for i in range(pairs):
        sub = replace(plan, variant=PlanVariant.HYBRID, devices=plan.devices[2 * i:2 * i + 2],
                      segment_fractions=None, seed=plan.seed + i)
        r = run_hybrid(sub)
        results.append(r)
        merged.merge(r.trace)
    latency = max(r.latency_s for r in results)
    first = results[0]
    return RunResult(x0=first.x0, latency_s=latency, comm_bytes=sum(r.comm_bytes for r in results),
                     speedup=pairs * serial_latency_ref(plan) / latency,
                     throughput_samples_per_s=pairs / latency, tau1=first.tau1, tau2=first.tau2,
                     trace=merged, series=first.series, per_sample=tuple(results),
                     stages=first.stages, x0_device=first.x0_device)


_RUNNERS = {
    PlanVariant.SERIAL: run_serial,
    PlanVariant.FULL_CONDITION_PARTITION: run_full_condition_partition,
    PlanVariant.HYBRID: run_hybrid,
    PlanVariant.LAYER_WISE: run_layer_wise,
    PlanVariant.BATCH_LEVEL: run_batch_level,
}


def run_plan(plan: ExecutionPlan) -> RunResult:
    return _RUNNERS[plan.variant](plan)


def run_plan_resident(plan: ExecutionPlan, x_init: torch.Tensor) -> RunResult:
    """``run_plan`` with x_T already resident on the device and x0 left there
    (``RunResult.x0`` is None, ``x0_device`` holds it): the device-side cost of
    a run with no host<->device traffic. Serial / FCP / hybrid / layer-wise."""
    v = plan.variant
    if v in (PlanVariant.SERIAL, PlanVariant.FULL_CONDITION_PARTITION):
        return _run_exact(plan, serial=v is PlanVariant.SERIAL, x_init=x_init, to_host=False)
    if v in (PlanVariant.HYBRID, PlanVariant.LAYER_WISE):
        return _run_staged(plan, plan.segment_fractions, x_init=x_init, to_host=False)
    raise PlanError(f"run_plan_resident does not run {v.value} plans")
