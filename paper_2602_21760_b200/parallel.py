"""Real multi-GPU execution: condition-partitioned pairs, hybrid windows,
batch-level pairs (one process per GPU, torch.distributed for set-up only).

Pair roles (engine.py:217-231): rank 2p is ``dev0`` and evaluates the
conditional branch, rank 2p+1 is ``dev1`` and evaluates the unconditional
branch. Per measured step each rank pushes its branch output into the
partner's receive buffer over NVLink (``hp_stage_send``: 16-byte vector
stores to the IPC-mapped peer buffer, then a system-scope release of the step
number into the partner's flag word) — the reference's two latent messages per
step, one per direction. Each rank then runs the fused sampler kernel with the
partner's output as its second operand; the kernel's CTAs acquire the flag
before loading it. Both ranks therefore compute the identical x_{t-1} and
M_t (same inputs, deterministic kernel), so the switch controller agrees on
both sides without any further message: the only data-path traffic is the
branch exchange. Receive buffers are double-buffered by step parity, which is
sufficient because a rank cannot reach step s+2 before its partner finished
step s (it waits on the partner's step-(s+1) flag).

Pipelined window (``pipeline_numerics="reference_blend"``, engine.py:254-261):
rank d evaluates the conditional branch on the d-steps-stale latent, the two
estimates are exchanged the same way and blended in d order on both ranks.

The loop itself (``PairLoop``) is device-agnostic: it talks to a ``PairOps``
object. ``CudaPairOps`` is the product (kernels + NVLink); the CPU test-suite
drives the same loop with gloo and the oracle.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import torch

from . import _kernels as K
from . import _native as N
from .engine import ExecutionPlan, PlanVariant, RunResult, initial_latents, serial_latency_ref
from .errors import PlanError, check
from .monitor import DiscrepancySeries, Stage, StageState, update_controller
from .trace import BusyInterval, MessageEvent, RunTrace


@dataclass(frozen=True)
class PairRole:
    pair: int
    role: int          # 0 = dev0 / conditional branch, 1 = dev1 / unconditional branch
    peer_rank: int


def pair_role(rank: int) -> PairRole:
    return PairRole(rank // 2, rank % 2, rank ^ 1)


class PairLoop:
    """The staged / exact loop of one condition-partitioned pair, seen from one rank."""

    def __init__(self, plan: ExecutionPlan, role: PairRole, ops):
        self.plan, self.role, self.ops = plan, role, ops

    def run(self, x_init):
        plan, ops, role = self.plan, self.ops, self.role.role
        T = plan.schedule.T
        staged = plan.variant in (PlanVariant.HYBRID, PlanVariant.LAYER_WISE)
        sw = plan.switch
        fr = plan.segment_fractions if staged else None
        host = StageState()
        no_series = DiscrepancySeries()
        first_poll = min(sw.L + 1, sw.tau_cap) if staged else T + 1
        x = ops.upload(x_init)
        history: list = []
        stages = []
        for s in range(1, T + 1):
            t = T - s + 1
            history.insert(0, x)
            del history[2:]
            if staged and host.tau1 is not None:
                update_controller(host, no_series, t, sw)
            if staged and host.stage is Stage.PARALLELISM:
                # segment `role` of the blend: conditional branch at the role-stale latent
                e = ops.conditional(history[min(role, len(history) - 1)], t)
                h = ops.exchange(e, s, kind="activation")
                x = ops.blend_update(x, e, h, t, fr)
            else:
                e = ops.my_branch(x, t)
                h = ops.exchange(e, s, kind="latent")
                op = N.HP_CTRL_RECORD_UPDATE if (staged and host.tau1 is None) else N.HP_CTRL_RECORD
                x = ops.measured_update(x, e, h, t, op)
                if staged and host.tau1 is None:
                    if s >= first_poll:
                        t1, t2 = ops.poll(t)
                        if t1 >= 0:
                            host.tau1, host.tau2 = t1, t2
                    host.steps_done, host.last_t, host.stage = s, t, Stage.WARM_UP
            stages.append(host.stage)
        x0, series = ops.finish(x)
        return x0, series, host.tau1, host.tau2, stages


class _Raw:
    """Minimal tensor-like view of a raw device pointer for the kernel wrappers."""

    def __init__(self, ptr: int, numel: int, dtype: torch.dtype, device):
        self._ptr, self._n, self.dtype, self.device = int(ptr), int(numel), dtype, device

    def data_ptr(self):
        return self._ptr

    def numel(self):
        return self._n


class PeerBuffers:
    """Receive buffers (2 x [B, N] bf16, step-parity double buffer) and flag words
    in this rank's HBM, exported by IPC handle; the partner's opened likewise."""

    def __init__(self, numel: int, elem_bytes: int, group, peer_rank: int):
        import torch.distributed as dist
        lib = N.require_cuda()
        self.numel, self.bytes = numel, numel * elem_bytes
        p = C.c_void_p()
        check(lib.hp_alloc(2 * self.bytes, C.byref(p)), "hp_alloc rbuf")
        self.rbuf = p.value
        f = C.c_void_p()
        check(lib.hp_alloc(64, C.byref(f)), "hp_alloc flags")
        self.flags = f.value
        h1 = C.create_string_buffer(64)
        h2 = C.create_string_buffer(64)
        check(lib.hp_ipc_get_handle(C.c_void_p(self.rbuf), h1), "ipc handle rbuf")
        check(lib.hp_ipc_get_handle(C.c_void_p(self.flags), h2), "ipc handle flags")
        mine = (bytes(h1.raw), bytes(h2.raw))
        got = [None] * dist.get_world_size(group)
        dist.all_gather_object(got, mine, group=group)
        peer_local = dist.get_group_rank(group, peer_rank) if group is not None else peer_rank
        ph1, ph2 = got[peer_local]
        q1, q2 = C.c_void_p(), C.c_void_p()
        check(lib.hp_ipc_open(C.create_string_buffer(ph1, 64), C.byref(q1)), "ipc open rbuf")
        check(lib.hp_ipc_open(C.create_string_buffer(ph2, 64), C.byref(q2)), "ipc open flags")
        self.peer_rbuf, self.peer_flags = q1.value, q2.value

    def local_slot(self, s):
        return self.rbuf + (s & 1) * self.bytes

    def peer_slot(self, s):
        return self.peer_rbuf + (s & 1) * self.bytes


class CudaPairOps:
    """Product PairOps: our kernels, NVLink pushes, device controller."""

    def __init__(self, plan: ExecutionPlan, role: PairRole, group, exchange: str = "p2p"):
        from .engine import _StepRunner
        self.plan, self.role, self.group, self.kind = plan, role, group, exchange
        self.st = _StepRunner(plan)
        self.den = self.st.den
        self.dev = self.st.dev
        self.numel = len(plan.conditions) * plan.mixture.dim
        self.edtype = getattr(self.den, "eps_dtype", torch.float64)
        esz = torch.tensor([], dtype=self.edtype).element_size()
        self.buf = PeerBuffers(self.numel, esz, group, role.peer_rank) if exchange == "p2p" else None
        self.msgs = []        # (kind, nbytes, step)
        self.lib = N.load()
        self.seq0 = 0         # flag value offset of the current run

    def begin_run(self, seq0: int):
        self.seq0 = seq0
        self.msgs = []
        self.st.reset()

    # ---- branch evaluation ----
    def upload(self, x_init):
        x, _ = self.st.upload(x_init)
        return x

    def my_branch(self, x, t):
        if self.role.role == 0:
            return self.den.conditional(x, t)
        return self.den.unconditional(x, t)

    def conditional(self, x, t):
        return self.den.conditional(x, t)

    # ---- exchange ----
    def exchange(self, e, s, kind):
        nbytes = e.numel() * e.element_size()
        self.msgs.append((kind, nbytes, s))
        if self.kind == "p2p":
            flag_idx = self.role.role            # my slot in the partner's flag words
            q = self.seq0 + s                     # global message sequence number
            check(self.lib.hp_stage_send(C.c_void_p(self.buf.peer_slot(q)), C.c_void_p(e.data_ptr()), nbytes,
                                         C.c_void_p(self.buf.peer_flags + 4 * flag_idx), q,
                                         C.c_void_p(N.stream_ptr())), "hp_stage_send")
            peer = _Raw(self.buf.local_slot(q), e.numel(), e.dtype, e.device)
            wait = self.buf.flags + 4 * (1 - self.role.role)
            return (peer, wait, q)
        import torch.distributed as dist
        other = torch.empty_like(e)
        ops = [dist.P2POp(dist.isend, e.contiguous(), self.role.peer_rank, self.group),
               dist.P2POp(dist.irecv, other, self.role.peer_rank, self.group)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        return (other, None, 0)

    # ---- fused updates ----
    def measured_update(self, x, e, h, t, ctrl_op):
        peer, wait, val = h
        ec, eu = (e, peer) if self.role.role == 0 else (peer, e)
        st = self.st
        out = torch.empty_like(x)
        outb = self.den.input_slot() if self.den.wants_bf16_input else None
        c = st.coef[t]
        kw = {} if c is None else dict(c_sigma=c.c_sigma, c_sqrt_ab=c.c_sqrt_ab,
                                       c_sqrt_ab_prev=c.c_sqrt_ab_prev, c_sqrt_1m_ab_prev=c.c_sqrt_1m_ab_prev)
        K.sampler_step(x=x, eps_c=ec, eps_u=eu, x_out=out, x_out_bf16=outb, update=st.update, t=t,
                       w=self.plan.guidance.w, dt=1.0 / self.plan.schedule.T, ws=st.ws, ctrl=st.ctrl,
                       ctrl_op=ctrl_op, mirror_ptr=st.mirror.ptr, wait_flag=wait, wait_value=val, **kw)
        return out

    def blend_update(self, x, e, h, t, fractions):
        peer, wait, val = h
        if wait is not None:
            check(self.lib.hp_flag_wait(C.c_void_p(wait), val, None, 0, C.c_void_p(N.stream_ptr())), "hp_flag_wait")
        parts = (e, peer) if self.role.role == 0 else (peer, e)
        acc = torch.empty(x.shape, dtype=x.dtype, device=x.device)
        for d, (f, part) in enumerate(zip(fractions, parts)):
            K.blend_accumulate(acc, part, f, first=(d == 0))
        xb, _ = self.st._advance(x, None, acc, None, t, N.HP_CTRL_NONE)
        return xb

    def poll(self, t):
        mr = self.st.poll(t)
        return mr.tau1, mr.tau2

    def finish(self, x):
        return self.st.finish(x)


class PairSession:
    """Set up a pair once (IPC buffers, graphs, controller) and run it repeatedly.

    Flag values are a monotonically increasing message sequence across runs
    (run r, step s -> r*T + s), so a new run can never consume a flag left
    over from the previous one."""

    def __init__(self, plan: ExecutionPlan, group=None, exchange: str = "p2p"):
        import torch.distributed as dist
        if plan.variant not in (PlanVariant.FULL_CONDITION_PARTITION, PlanVariant.HYBRID):
            raise PlanError(f"a pair runs condition-partitioned plans, got {plan.variant.value}")
        self.plan, self.group = plan, group
        self.role = pair_role(dist.get_rank())
        self.ops = CudaPairOps(plan, self.role, group, exchange)
        self.runs = 0

    def run(self, x_init=None) -> RunResult:
        import torch.distributed as dist
        plan, ops, role = self.plan, self.ops, self.role
        ops.begin_run(self.runs * plan.schedule.T)
        self.runs += 1
        loop = PairLoop(plan, role, ops)
        dist.barrier(self.group)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        x0, series, tau1, tau2, stages = loop.run(initial_latents(plan) if x_init is None else x_init)
        b.record()
        torch.cuda.synchronize()
        mine = torch.tensor([a.elapsed_time(b) / 1e3], dtype=torch.float64, device="cuda")
        dist.all_reduce(mine, op=dist.ReduceOp.MAX, group=self.group)
        latency = float(mine.item())
        trace = RunTrace()
        me = plan.devices[role.role].name
        trace.busy.append(BusyInterval(me, 0.0, latency, plan.schedule.T, "", "run"))
        peer_name = plan.devices[1 - role.role].name
        for kind, nb, s in ops.msgs:
            trace.messages.append(MessageEvent(me, peer_name, kind, nb, 0.0, 0.0, s))
        comm = 2 * sum(nb for _, nb, _ in ops.msgs)     # both directions of the pair
        ref = serial_latency_ref(plan)
        return RunResult(x0=x0, latency_s=latency, comm_bytes=comm, speedup=ref / latency,
                         throughput_samples_per_s=1.0 / latency, tau1=tau1, tau2=tau2, trace=trace,
                         series=series, stages=tuple(stages))


def run_pair(plan: ExecutionPlan, group=None, exchange: str = "p2p") -> RunResult:
    """Execute a FULL_CONDITION_PARTITION or HYBRID plan on this rank's pair.

    Every rank of the pair calls this with the same plan; both return the same
    x0 and series. latency_s is the max over the pair of the device time."""
    return PairSession(plan, group, exchange).run()


def run_batch_level_distributed(plan: ExecutionPlan, exchange: str = "p2p") -> RunResult:
    """N/2 pairs, pair p runs seed + p (engine.py:358-383); one process per GPU."""
    import torch.distributed as dist
    ws = dist.get_world_size()
    if ws % 2:
        raise PlanError(f"batch-level needs an even number of ranks, got {ws}")
    rank = dist.get_rank()
    role = pair_role(rank)
    groups = [dist.new_group([2 * p, 2 * p + 1]) for p in range(ws // 2)]
    sub = replace(plan, variant=PlanVariant.HYBRID, devices=plan.devices[:2], segment_fractions=None,
                  seed=plan.seed + role.pair)
    res = run_pair(sub, groups[role.pair], exchange)
    lat = torch.tensor([res.latency_s], dtype=torch.float64, device="cuda")
    dist.all_reduce(lat, op=dist.ReduceOp.MAX)
    pairs = ws // 2
    latency = float(lat.item())
    return replace(res, latency_s=latency, throughput_samples_per_s=pairs / latency,
                   speedup=pairs * serial_latency_ref(plan) / latency)

