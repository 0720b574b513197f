"""Real multi-GPU execution: condition-partitioned pairs, hybrid windows,
layer-wise windows over N ranks, batch-level pairs (one process per GPU,
torch.distributed for set-up only).

Roles (engine.py:217-231, 330-337): a sample runs on a group of n ranks; group
index 0 is ``dev0`` and evaluates the conditional branch, index 1 is ``dev1``
and evaluates the unconditional branch, indices 2..n-1 (layer-wise only) idle
outside the window like the reference's extra segment devices
(engine.py:350-351). Per measured step ranks 0 and 1 push their branch output
into every other rank's receive buffer over NVLink (``hp_stage_broadcast``:
16-byte vector stores to the IPC-mapped peer buffers, then a system-scope
release of the message number into each destination's flag word) — for a
pair exactly the reference's two latent messages per step, one per direction.
Every rank then runs the fused sampler kernel on (eps_c, eps_u), the remote
operand(s) read from its receive buffer after the kernel's CTAs acquire the
flag. All ranks therefore compute the identical x_{t-1} and M_t (same inputs,
deterministic kernel), so the switch controller agrees everywhere without any
further message: the only data-path traffic is the branch exchange.

Pipelined window (``pipeline_numerics="reference_blend"``, engine.py:254-261):
rank d evaluates the conditional branch on the d-steps-stale latent (each rank
keeps its own history, identical on all ranks), every rank hands its
contribution to all others and all blend in d order.

Receive buffers are double-buffered by message parity. Within a pair (and in
the window, where every rank waits on every rank) that suffices: nobody can
send message q+2 before its consumer finished with q. Ranks 2..n-1 are passive
in measured steps, so they acknowledge every step to ranks 0 and 1, which wait
for the acknowledgement of q-2 before sending q.

The loop itself (``StagedLoop``) is device-agnostic: it talks to an ops
object. ``CudaGroupOps`` is the product (kernels + NVLink); the CPU test-suite
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

BRANCH_SOURCES = (0, 1)     # group indices that evaluate the two CFG branches
WAIT_TIMEOUT_NS = 20_000_000_000


@dataclass(frozen=True)
class PairRole:
    pair: int
    role: int          # 0 = dev0 / conditional branch, 1 = dev1 / unconditional branch
    peer_rank: int


def pair_role(rank: int) -> PairRole:
    return PairRole(rank // 2, rank % 2, rank ^ 1)


def group_size(plan: ExecutionPlan) -> int:
    """Ranks one sample runs on: the plan's devices for layer-wise, else a pair."""
    return len(plan.devices) if plan.variant is PlanVariant.LAYER_WISE else 2


class StagedLoop:
    """The exact / staged loop of one sample, seen from group index ``index`` of ``n``."""

    def __init__(self, plan: ExecutionPlan, index: int, n: int, ops):
        if not 0 <= index < n:
            raise PlanError(f"group index {index} outside [0, {n})")
        self.plan, self.index, self.n, self.ops = plan, index, n, ops

    def run(self, x_init):
        plan, ops, d, n = self.plan, self.ops, self.index, self.n
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
        everyone = tuple(range(n))
        for s in range(1, T + 1):
            t = T - s + 1
            history.insert(0, x)
            del history[n:]
            if staged and host.tau1 is not None:
                update_controller(host, no_series, t, sw)
            if staged and host.stage is Stage.PARALLELISM:
                # segment d of the blend: conditional branch at the d-stale latent
                e = ops.conditional(history[min(d, len(history) - 1)], t)
                parts = ops.exchange(e, s, "activation", everyone)
                x = ops.blend_update(x, parts, t, fr)
            else:
                e = ops.branch(x, t) if d in BRANCH_SOURCES else None
                parts = ops.exchange(e, s, "latent", BRANCH_SOURCES)
                op = N.HP_CTRL_RECORD_UPDATE if (staged and host.tau1 is None) else N.HP_CTRL_RECORD
                x = ops.measured_update(x, parts, t, op)
                if staged and host.tau1 is None:
                    if s >= first_poll:
                        t1, t2 = ops.poll(t)
                        if t1 >= 0:
                            host.tau1, host.tau2 = t1, t2
                    host.steps_done, host.last_t, host.stage = s, t, Stage.WARM_UP
            ops.step_done(s)
            stages.append(host.stage)
        x0, series = ops.finish(x)
        return x0, series, host.tau1, host.tau2, stages


class PairLoop(StagedLoop):
    """A condition-partitioned pair (n = 2) — kept for the pair-centred callers."""

    def __init__(self, plan: ExecutionPlan, role: PairRole, ops):
        super().__init__(plan, role.role, 2, ops)


class _Raw:
    """Minimal tensor-like view of a raw device pointer for the kernel wrappers."""

    def __init__(self, ptr: int, numel: int, dtype: torch.dtype, device):
        self._ptr, self._n, self.dtype, self.device = int(ptr), int(numel), dtype, device

    def data_ptr(self):
        return self._ptr

    def numel(self):
        return self._n


class GroupBuffers:
    """Receive buffers and flag words of one rank, exported by CUDA IPC; the other
    group members' are opened likewise.

    Layout in this rank's HBM: ``rbuf[src][parity]`` (n x 2 x numel x elem)
    and ``flags[0:n]`` = last message number received from src,
    ``flags[n:2n]`` = last step acknowledged by passive rank r (on ranks 0, 1)."""

    def __init__(self, numel: int, elem_bytes: int, group, index: int, n: int):
        import torch.distributed as dist
        lib = N.require_cuda()
        if n > N.HP_MAX_PEERS + 1:
            raise PlanError(f"a group spans at most {N.HP_MAX_PEERS + 1} GPUs, got {n}")
        self.numel, self.bytes, self.index, self.n = numel, numel * elem_bytes, index, n
        p = C.c_void_p()
        check(lib.hp_alloc(2 * n * self.bytes, C.byref(p)), "hp_alloc rbuf")
        self.rbuf = p.value
        f = C.c_void_p()
        check(lib.hp_alloc(max(64, 8 * n), C.byref(f)), "hp_alloc flags")
        self.flags = f.value
        h1 = C.create_string_buffer(N.HP_IPC_HANDLE_BYTES)
        h2 = C.create_string_buffer(N.HP_IPC_HANDLE_BYTES)
        check(lib.hp_ipc_get_handle(C.c_void_p(self.rbuf), h1), "ipc handle rbuf")
        check(lib.hp_ipc_get_handle(C.c_void_p(self.flags), h2), "ipc handle flags")
        got = [None] * n
        dist.all_gather_object(got, (index, bytes(h1.raw), bytes(h2.raw)), group=group)
        self.peer_rbuf, self.peer_flags = {}, {}
        for idx, ph1, ph2 in got:
            if idx == index:
                continue
            q1, q2 = C.c_void_p(), C.c_void_p()
            check(lib.hp_ipc_open(C.create_string_buffer(ph1, N.HP_IPC_HANDLE_BYTES), C.byref(q1)), "ipc open rbuf")
            check(lib.hp_ipc_open(C.create_string_buffer(ph2, N.HP_IPC_HANDLE_BYTES), C.byref(q2)), "ipc open flags")
            self.peer_rbuf[idx], self.peer_flags[idx] = q1.value, q2.value

    def local_slot(self, src: int, q: int) -> int:
        return self.rbuf + (2 * src + (q & 1)) * self.bytes

    def peer_slot(self, dst: int, q: int) -> int:
        """Where this rank's message q lands in rank dst's buffer."""
        return self.peer_rbuf[dst] + (2 * self.index + (q & 1)) * self.bytes

    def data_flag(self, src: int) -> int:
        return self.flags + 4 * src

    def peer_data_flag(self, dst: int) -> int:
        return self.peer_flags[dst] + 4 * self.index

    def ack_flag(self, r: int) -> int:
        return self.flags + 4 * (self.n + r)

    def peer_ack_flag(self, dst: int) -> int:
        return self.peer_flags[dst] + 4 * (self.n + self.index)


class CudaGroupOps:
    """Product ops: our kernels, NVLink pushes, device controller."""

    def __init__(self, plan: ExecutionPlan, index: int, n: int, group, exchange: str = "p2p"):
        from .engine import _StepRunner
        if exchange not in ("p2p", "nccl"):
            raise PlanError(f"exchange must be 'p2p' or 'nccl', got {exchange!r}")
        self.plan, self.index, self.n, self.group, self.kind = plan, index, n, group, exchange
        self.st = _StepRunner(plan)
        self.den = self.st.den
        self.dev = self.st.dev
        self.numel = len(plan.conditions) * plan.mixture.dim
        self.edtype = getattr(self.den, "eps_dtype", torch.float64)
        esz = torch.tensor([], dtype=self.edtype).element_size()
        self.buf = GroupBuffers(self.numel, esz, group, index, n) if exchange == "p2p" else None
        self.msgs = []        # (kind, nbytes, step, dst index)
        self.lib = N.load()
        self.seq0 = 0         # message number offset of the current run
        self.others = [r for r in range(n) if r != index]
        self.passive = list(range(2, n))
        if exchange == "nccl":
            import torch.distributed as dist
            self._ranks = [dist.get_global_rank(group, r) if group is not None else r for r in range(n)]

    def begin_run(self, seq0: int):
        self.seq0 = seq0
        self.msgs = []
        self.st.reset()

    # ---- branch evaluation ----
    def upload(self, x_init):
        x, _ = self.st.upload(x_init)
        return x

    def branch(self, x, t):
        if self.index == 0:
            return self.den.conditional(x, t)
        return self.den.unconditional(x, t)

    def conditional(self, x, t):
        return self.den.conditional(x, t)

    # ---- exchange ----
    def _wait(self, flag: int, value: int):
        # a peer that never arrives ends the wait after WAIT_TIMEOUT_NS with HP_ERR_TIMEOUT in
        # the device controller's status word, raised by the next poll / finish
        status = C.c_void_p(self.st.ctrl.data_ptr() + N.HpCtrl.status.offset)
        check(self.lib.hp_flag_wait(C.c_void_p(flag), value, status, WAIT_TIMEOUT_NS, C.c_void_p(N.stream_ptr())),
              "hp_flag_wait")

    def exchange(self, e, s, kind, sources):
        q = self.seq0 + s
        me = self.index
        if self.kind == "nccl":
            return self._exchange_nccl(e, s, kind, sources)
        if me in sources:
            nbytes = e.numel() * e.element_size()
            if me in BRANCH_SOURCES and q > 2:
                for r in self.passive:          # passive ranks finished message q-2
                    self._wait(self.buf.ack_flag(r), q - 2)
            dsts = (C.c_void_p * len(self.others))(*[self.buf.peer_slot(r, q) for r in self.others])
            flags = (C.c_void_p * len(self.others))(*[self.buf.peer_data_flag(r) for r in self.others])
            check(self.lib.hp_stage_broadcast(dsts, flags, len(self.others), C.c_void_p(e.data_ptr()), nbytes, q,
                                              C.c_void_p(N.stream_ptr())), "hp_stage_broadcast")
            self.msgs.extend((kind, nbytes, s, r) for r in self.others)
        parts = []
        for src in sources:
            if src == me:
                parts.append((e, None, 0))
            else:
                parts.append((_Raw(self.buf.local_slot(src, q), self.numel, self.edtype, self.dev),
                              self.buf.data_flag(src), q))
        return parts

    def _exchange_nccl(self, e, s, kind, sources):
        import torch.distributed as dist
        me = self.index
        ops, parts = [], []
        for src in sources:
            if src == me:
                for r in self.others:
                    ops.append(dist.P2POp(dist.isend, e.contiguous(), self._ranks[r], self.group))
                    self.msgs.append((kind, e.numel() * e.element_size(), s, r))
                parts.append((e, None, 0))
            else:
                buf = torch.empty(self.numel, dtype=self.edtype, device=self.dev)
                ops.append(dist.P2POp(dist.irecv, buf, self._ranks[src], self.group))
                parts.append((buf, None, 0))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        return parts

    def step_done(self, s):
        # passive ranks release their receive slots of message q to the branch ranks
        if self.kind == "p2p" and self.index >= 2:
            flags = (C.c_void_p * 2)(*[self.buf.peer_ack_flag(r) for r in BRANCH_SOURCES])
            dsts = (C.c_void_p * 2)(0, 0)
            check(self.lib.hp_stage_broadcast(dsts, flags, 2, None, 0, self.seq0 + s, C.c_void_p(N.stream_ptr())),
                  "hp_stage_broadcast ack")

    # ---- fused updates ----
    def measured_update(self, x, parts, t, ctrl_op):
        (ec, wc, vc), (eu, wu, vu) = parts
        if wc is not None and wu is not None:     # passive rank: both operands remote
            self._wait(wc, vc)
            wc = None
        wait, val = (wu, vu) if wu is not None else (wc, vc)
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

    def blend_update(self, x, parts, t, fractions):
        acc = torch.empty(x.shape, dtype=x.dtype, device=x.device)
        for d, (f, (part, wait, val)) in enumerate(zip(fractions, parts)):
            if wait is not None:
                self._wait(wait, val)
            K.blend_accumulate(acc, part, f, first=(d == 0))
        xb, _ = self.st._advance(x, None, acc, None, t, N.HP_CTRL_NONE)
        return xb

    def poll(self, t):
        mr = self.st.poll(t)
        return mr.tau1, mr.tau2

    def finish(self, x):
        return self.st.finish(x)


def CudaPairOps(plan: ExecutionPlan, role: PairRole, group, exchange: str = "p2p") -> CudaGroupOps:
    return CudaGroupOps(plan, role.role, 2, group, exchange)


class GroupSession:
    """Set up one sample's group once (IPC buffers, graphs, controller) and run it
    repeatedly. FCP / hybrid plans run on a pair; layer-wise on len(devices) ranks.

    Message numbers increase monotonically across runs (run r, step s -> r*T + s),
    so a new run can never consume a flag left over from the previous one."""

    def __init__(self, plan: ExecutionPlan, group=None, exchange: str = "p2p"):
        import torch.distributed as dist
        if plan.variant not in (PlanVariant.FULL_CONDITION_PARTITION, PlanVariant.HYBRID, PlanVariant.LAYER_WISE):
            raise PlanError(f"a group runs FCP, hybrid or layer-wise plans, got {plan.variant.value}")
        n = group_size(plan)
        size = dist.get_world_size(group)
        if size != n:
            raise PlanError(f"{plan.variant.value} plan needs a group of {n} ranks, got {size}")
        self.plan, self.group, self.n = plan, group, n
        self.index = dist.get_group_rank(group, dist.get_rank()) if group is not None else dist.get_rank()
        self.ops = CudaGroupOps(plan, self.index, n, group, exchange)
        self.runs = 0

    def run(self, x_init=None) -> RunResult:
        import torch.distributed as dist
        plan, ops = self.plan, self.ops
        ops.begin_run(self.runs * plan.schedule.T)
        self.runs += 1
        loop = StagedLoop(plan, self.index, self.n, ops)
        dist.barrier(self.group)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        x0, series, tau1, tau2, stages = loop.run(initial_latents(plan) if x_init is None else x_init)
        b.record()
        torch.cuda.synchronize()
        sent = sum(nb for _, nb, _, _ in ops.msgs)
        red = torch.tensor([a.elapsed_time(b) / 1e3, float(sent)], dtype=torch.float64, device="cuda")
        mx, tot = red[:1].clone(), red[1:].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=self.group)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM, group=self.group)
        latency, comm = float(mx.item()), int(tot.item())
        trace = RunTrace()
        me = plan.devices[self.index].name
        trace.busy.append(BusyInterval(me, 0.0, latency, plan.schedule.T, "", "run"))
        for kind, nb, s, dst in ops.msgs:
            trace.messages.append(MessageEvent(me, plan.devices[dst].name, kind, nb, 0.0, 0.0, s))
        ref = serial_latency_ref(plan)
        return RunResult(x0=x0, latency_s=latency, comm_bytes=comm, speedup=ref / latency,
                         throughput_samples_per_s=1.0 / latency, tau1=tau1, tau2=tau2, trace=trace,
                         series=series, stages=tuple(stages))


PairSession = GroupSession


def run_pair(plan: ExecutionPlan, group=None, exchange: str = "p2p") -> RunResult:
    """Execute a FULL_CONDITION_PARTITION or HYBRID plan on this rank's pair.

    Every rank of the pair calls this with the same plan; both return the same
    x0 and series. latency_s is the max over the pair of the device time."""
    return GroupSession(plan, group, exchange).run()


def run_layer_wise_distributed(plan: ExecutionPlan, group=None, exchange: str = "p2p") -> RunResult:
    """A LAYER_WISE plan on len(plan.devices) ranks (engine.py:340-348): group
    index d is plan.devices[d]; every rank returns the same x0 and series."""
    if plan.variant is not PlanVariant.LAYER_WISE:
        raise PlanError(f"run_layer_wise_distributed got a {plan.variant.value} plan")
    return GroupSession(plan, group, exchange).run()


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
