"""Real multi-GPU execution: condition-partitioned pairs, hybrid windows,
layer-wise windows over N ranks, batch-level pairs (one process per GPU,
torch.distributed for set-up only).

Roles (engine.py:217-231, 330-337): a sample runs on a group of n ranks; group
index 0 is ``dev0`` and evaluates the conditional branch, index 1 is ``dev1``
and evaluates the unconditional branch, indices 2..n-1 (layer-wise only) idle
outside the window like the reference's extra segment devices
(engine.py:350-351).

Messages travel on per-(src, dst) links (``LinkBuffers``): the producer pushes
its payload with 16-byte vector stores into the consumer's receive slot over
NVLink (IPC-mapped peer pointer) and releases the link's message count into the
consumer's flag word (system scope); the consumer acquires the flag -- inside
the fused sampler kernel, in a wait kernel, or (``wait="host"``) by polling
from the host -- reads the slot and acknowledges; slots are double-buffered by
message parity and a producer waits for the acknowledgement of message q-2
before it sends q.

Measured step (every plan): ranks 0 and 1 evaluate their branch and exchange
the outputs -- the reference's two latent messages per step, one per direction
(engine.py:229-231). Both run the fused CFG + sampler + discrepancy kernel on
the same inputs, so they hold the identical x_{t-1} and M_t and take the same
switch decision with no further message.

Window, ``pipeline_numerics="stage_split"`` (stages.py, north_star iii): group
index d runs network stage j = N-1-d on the boundary state stage j-1 produced
at the previous step, so the N stages run concurrently; per step N-1
activation messages hop d -> d-1 (the reference's N-1 activations,
engine.py:330-337) and dev0, which runs the last stage and the unguided
update, hands x_{t-1} to the first stage's rank (one latent message: the loop
closing hop a real pipeline needs and the reference's cost model leaves out).
The fill comes from the conditional branch of the last measured step's
forward on dev0 (recorded at the cuts); for N > 2 dev0 ships those boundary
states and x_t to the passive ranks, which learn the window's first step from
a control word and idle before and after it.

Window, ``reference_blend`` (engine.py:254-261): rank d evaluates the
conditional branch at its d-stale latent and every rank blends every
contribution in d order (so every rank needs every contribution; for N > 2
the passive ranks also receive both branch outputs in measured steps to keep
their latent history). This is the reference's numerics surrogate, kept for
parity; ``stage_split`` is the mode with the reference's message contract.

The loop (``StagedLoop``) is device-agnostic and talks to an ops object:
``CudaGroupOps`` is the product (kernels + NVLink); the CPU test-suite drives
the same loop with gloo and the oracle.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import torch

from . import _kernels as K
from . import _native as N
from .engine import ExecutionPlan, PlanVariant, RunResult, initial_latents, serial_latency_ref
from .errors import NativeError, PlanError, check, from_status
from .monitor import DiscrepancySeries, Stage, StageState, update_controller
from .trace import BusyInterval, MessageEvent, RunTrace

BRANCH_SOURCES = (0, 1)     # group indices that evaluate the two CFG branches
WAIT_TIMEOUT_NS = 20_000_000_000
WAIT_MODES = ("device", "host")


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


@dataclass
class Part:
    """A received (or local) operand: ``data`` plus, while the consumer has not
    waited yet, the flag word and message count that publish it."""
    data: object
    src: int = -1
    flag: int | None = None
    value: int = 0


class StagedLoop:
    """The exact / staged loop of one sample, seen from group index ``index`` of ``n``."""

    def __init__(self, plan: ExecutionPlan, index: int, n: int, ops):
        if not 0 <= index < n:
            raise PlanError(f"group index {index} outside [0, {n})")
        self.plan, self.index, self.n, self.ops = plan, index, n, ops
        v = plan.variant
        self.staged = v in (PlanVariant.HYBRID, PlanVariant.LAYER_WISE)
        self.split = self.staged and plan.pipeline_numerics == "stage_split"
        self.blend_all = self.staged and not self.split and n > 2

    # ---- measured step -------------------------------------------------------------
    def _measured(self, x, s, t, op):
        ops, d, n = self.ops, self.index, self.n
        if d >= 2:
            dsts = []                                  # passive rank (blend layer-wise): receives only
        else:
            dsts = [r for r in range(n) if r != d] if self.blend_all else [d ^ 1]
        e = ops.branch(x, t) if d < 2 else None
        for dst in dsts:
            ops.send(dst, e, "latent", s)
        parts = [Part(e) if src == d else ops.recv(src, "eps") for src in BRANCH_SOURCES]
        return ops.measured_update(x, parts, t, op)

    # ---- stage-split window ----------------------------------------------------------
    def _stage_runs(self, j, s, tau2):
        """Stage j's output at window step s reaches the last stage at step
        s + (N-1-j); it is computed only if that is still inside the window
        (the pipeline drains at the end of the window)."""
        return s + (self.n - 1 - j) <= tau2

    def _split_step(self, x, s, t, fill, tau2):
        ops, d, n = self.ops, self.index, self.n
        j = n - 1 - d
        if d == 0:
            if fill:
                ops.stage_fill_local()
                if n > 2:
                    ops.signal_control(range(2, n), s)   # passive ranks learn the first window step
                    for jj in range(1, n - 1):
                        ops.send(n - 1 - jj, ops.stage_input(jj), "activation", s)
                    ops.send(n - 1, x, "latent", s)
            else:
                ops.stage_load(j, ops.recv(1, "activation"))
            eps = ops.stage_run(j, t)
            x = ops.unguided_update(x, eps, t)
            if n == 2:
                ops.send(1, x, "latent", s)              # next stage-0 input / dev1's x after the window
            else:
                if s + 1 <= tau2 and self._stage_runs(0, s + 1, tau2):
                    ops.send(n - 1, x, "latent", s)
                if s == tau2:
                    ops.send(1, x, "latent", s)          # dev1 resumes the measured steps
            return x
        # d == 1 (n == 2: stage 0 on x_t; n > 2: stage n-2)
        if n > 2 and (fill or self._stage_runs(j, s, tau2)):
            ops.stage_load(j, ops.recv(0 if fill else 2, "activation"))
        if self._stage_runs(j, s, tau2):
            if n == 2:
                ops.load_stage_x(x)
            ops.send(0, ops.stage_run(j, t), "activation", s)
        return x

    def _run_passive_split(self):
        """Ranks 2..n-1 of a stage-split layer-wise group: idle until dev0's fill,
        then run stage j = n-1-d while its output can still reach the last stage."""
        plan, ops, d, n = self.plan, self.ops, self.index, self.n
        T, k = plan.schedule.T, plan.switch.k
        j = n - 1 - d
        if k < 1:
            return None, (), None, None, []
        s_fill = ops.wait_control()
        tau1, tau2 = s_fill - 1, s_fill - 1 + k
        for s in range(s_fill, tau2 + 1):
            t = T - s + 1
            if s == s_fill or self._stage_runs(j, s, tau2):
                if d == n - 1:
                    ops.load_stage_x(ops.take_latent(ops.recv(0, "latent")))
                else:
                    ops.stage_load(j, ops.recv(0 if s == s_fill else d + 1, "activation"))
            if self._stage_runs(j, s, tau2):
                ops.send(d - 1, ops.stage_run(j, t), "activation", s)
        ops.drain()
        stages = [Stage.WARM_UP] * tau1 + [Stage.PARALLELISM] * k + [Stage.FULLY_CONNECTING] * (T - tau2)
        return None, (), tau1, tau2, stages

    def run(self, x_init):
        plan, ops, d, n = self.plan, self.ops, self.index, self.n
        if self.split and d >= 2:
            return self._run_passive_split()
        T = plan.schedule.T
        staged, sw = self.staged, plan.switch
        fr = plan.segment_fractions if staged else None
        host = StageState()
        no_series = DiscrepancySeries()
        first_poll = min(sw.L + 1, sw.tau_cap) if staged else T + 1
        x = ops.upload(x_init)
        history: list = []
        stages = []
        prev = Stage.WARM_UP
        for s in range(1, T + 1):
            t = T - s + 1
            history.insert(0, x)
            del history[n:]
            if staged and host.tau1 is not None:
                update_controller(host, no_series, t, sw)
            window = staged and host.stage is Stage.PARALLELISM
            if self.split and d == 1 and prev is Stage.PARALLELISM and (n == 2 or not window):
                x = ops.take_latent(ops.recv(0, "latent"))      # x_t from dev0's last window step
            if window and self.split:
                x = self._split_step(x, s, t, fill=prev is not Stage.PARALLELISM, tau2=host.tau2)
            elif window:
                e = ops.conditional(history[min(d, len(history) - 1)], t)
                for dst in range(n):
                    if dst != d:
                        ops.send(dst, e, "activation", s)
                parts = [Part(e) if src == d else ops.recv(src, "eps") for src in range(n)]
                x = ops.blend_update(x, parts, t, fr)
            elif d < 2 or self.blend_all:
                op = N.HP_CTRL_RECORD_UPDATE if (staged and host.tau1 is None) else N.HP_CTRL_RECORD
                x = self._measured(x, s, t, op)
                if staged and host.tau1 is None:
                    if s >= first_poll:
                        t1, t2 = ops.poll(t)
                        if t1 >= 0:
                            host.tau1, host.tau2 = t1, t2
                    host.steps_done, host.last_t, host.stage = s, t, Stage.WARM_UP
            stages.append(host.stage)
            prev = host.stage
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

    def element_size(self):
        return torch.tensor([], dtype=self.dtype).element_size()


class LinkBuffers:
    """Receive slots and flag words of one rank, exported by CUDA IPC; the other
    group members' are opened likewise.

    Layout in this rank's HBM: ``rbuf[src][parity]`` (n x 2 x slot_bytes) and
    u32 words ``flags[0:n]`` = messages received from src, ``flags[n:2n]`` =
    messages of mine that dst has consumed (its acknowledgement),
    ``flags[2n]`` = control word (the stage-split window's first step)."""

    def __init__(self, slot_bytes: int, group, index: int, n: int):
        import torch.distributed as dist
        lib = N.require_cuda()
        if n > N.HP_MAX_PEERS + 1:
            raise PlanError(f"a group spans at most {N.HP_MAX_PEERS + 1} GPUs, got {n}")
        self.bytes = (int(slot_bytes) + 255) // 256 * 256
        self.index, self.n = index, n
        p = C.c_void_p()
        check(lib.hp_alloc(2 * n * self.bytes, C.byref(p)), "hp_alloc rbuf")
        self.rbuf = p.value
        f = C.c_void_p()
        check(lib.hp_alloc(max(64, 4 * (2 * n + 1)), C.byref(f)), "hp_alloc flags")
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
        """Where my message q lands in rank dst's buffer."""
        return self.peer_rbuf[dst] + (2 * self.index + (q & 1)) * self.bytes

    def data_flag(self, src: int) -> int:
        return self.flags + 4 * src

    def peer_data_flag(self, dst: int) -> int:
        return self.peer_flags[dst] + 4 * self.index

    def ack_flag(self, dst: int) -> int:
        return self.flags + 4 * (self.n + dst)

    def peer_ack_flag(self, src: int) -> int:
        return self.peer_flags[src] + 4 * (self.n + self.index)

    def control(self) -> int:
        return self.flags + 4 * 2 * self.n

    def peer_control(self, dst: int) -> int:
        return self.peer_flags[dst] + 4 * 2 * self.n


class CudaGroupOps:
    """Product ops: our kernels, NVLink pushes, device controller.

    ``wait="device"``: consumers acquire flags on the GPU (inside the fused
    sampler kernel or a one-thread wait kernel), the host never blocks -- the
    multi-GPU mode. ``wait="host"``: the host polls each flag (``hp_flag_poll``)
    before it enqueues the consumer, so no kernel ever waits on another
    process: ranks may then share ONE GPU (tests; B200_PROFILING.md forbids
    cross-process GPU-side waits on a shared device)."""

    def __init__(self, plan: ExecutionPlan, index: int, n: int, group, exchange: str = "p2p",
                 wait: str = "device"):
        from .engine import _StepRunner
        if exchange not in ("p2p", "nccl"):
            raise PlanError(f"exchange must be 'p2p' or 'nccl', got {exchange!r}")
        if wait not in WAIT_MODES:
            raise PlanError(f"wait must be one of {WAIT_MODES}, got {wait!r}")
        self.plan, self.index, self.n, self.group, self.kind, self.wait_mode = plan, index, n, group, exchange, wait
        self.st = _StepRunner(plan)
        self.den = self.st.den
        self.dev = self.st.dev
        self.numel = len(plan.conditions) * plan.mixture.dim
        self.edtype = getattr(self.den, "eps_dtype", torch.float64)
        self.xdtype = getattr(self.den, "latent_dtype", torch.float64)
        esz = torch.tensor([], dtype=self.edtype).element_size()
        xsz = torch.tensor([], dtype=self.xdtype).element_size()
        slot = self.numel * max(esz, xsz)
        if self.st.split:
            slot = max([slot] + [b.nbytes for b in self.den.bnd[1:]])
        self.buf = LinkBuffers(slot, group, index, n) if exchange == "p2p" else None
        self.msgs = []        # (kind, nbytes, step, dst index)
        self.lib = N.load()
        self.sent = [0] * n   # per-link message counters (monotonic across runs)
        self.recvd = [0] * n
        self.ctrl_base = 0
        self._nccl_work = []
        if exchange == "nccl":
            import torch.distributed as dist
            self._ranks = [dist.get_global_rank(group, r) if group is not None else r for r in range(n)]

    def begin_run(self, run_index: int):
        self.msgs = []
        self.ctrl_base = run_index * (self.plan.schedule.T + 1)
        self.st.reset()

    # ---- compute ----
    def upload(self, x_init):
        x, _ = self.st.upload(x_init)
        return x

    def branch(self, x, t):
        if self.index == 0:
            return self.den.conditional(x, t)
        return self.den.unconditional(x, t)

    def conditional(self, x, t):
        return self.den.conditional(x, t)

    # ---- links ----
    def _status_ptr(self):
        return C.c_void_p(self.st.ctrl.data_ptr() + N.HpCtrl.status.offset)

    def _wait_value(self, flag: int, value: int):
        if self.wait_mode == "host":
            rc = self.lib.hp_flag_poll(C.c_void_p(flag), value, WAIT_TIMEOUT_NS, None)
            if rc != 0:
                raise from_status(rc, f"peer message {value} never arrived")
            return
        # a peer that never arrives ends the wait after WAIT_TIMEOUT_NS with HP_ERR_TIMEOUT in
        # the device controller's status word, raised by the next poll / finish
        check(self.lib.hp_flag_wait(C.c_void_p(flag), value, self._status_ptr(), WAIT_TIMEOUT_NS,
                                    C.c_void_p(N.stream_ptr())), "hp_flag_wait")

    def send(self, dst: int, payload, kind: str, s: int):
        nbytes = payload.numel() * payload.element_size()
        self.msgs.append((kind, nbytes, s, dst))
        if self.kind == "nccl":
            import torch.distributed as dist
            self._nccl_work.append(dist.isend(payload.contiguous(), self._ranks[dst], self.group))
            return
        if nbytes > self.buf.bytes:
            raise PlanError(f"message of {nbytes} B exceeds the {self.buf.bytes} B link slot")
        q = self.sent[dst] + 1
        if q > 2:
            self._wait_value(self.buf.ack_flag(dst), q - 2)     # dst released the slot of q-2
        dsts = (C.c_void_p * 1)(self.buf.peer_slot(dst, q))
        flags = (C.c_void_p * 1)(self.buf.peer_data_flag(dst))
        check(self.lib.hp_stage_broadcast(dsts, flags, 1, C.c_void_p(payload.data_ptr()), nbytes, q,
                                          C.c_void_p(N.stream_ptr())), "hp_stage_broadcast")
        self.sent[dst] = q

    def recv(self, src: int, what: str) -> Part:
        """Next message on link src -> me; ``what``: "eps" (branch output / blend
        part), "latent" (fp32 x) or "activation" (a stage-split boundary)."""
        dt = {"eps": self.edtype, "latent": self.xdtype, "activation": torch.bfloat16}[what]
        numel = self.numel if what != "activation" else self.buf.bytes // 2 if self.buf else 0
        if self.kind == "nccl":
            import torch.distributed as dist
            if what == "activation":
                buf = torch.empty(self.den.bnd[self.n - 1 - self.index].buf.numel(), dtype=dt, device=self.dev)
            else:
                buf = torch.empty(self.numel, dtype=dt, device=self.dev)
            dist.irecv(buf, self._ranks[src], self.group).wait()
            return Part(buf, src)
        q = self.recvd[src] + 1
        self.recvd[src] = q
        return Part(_Raw(self.buf.local_slot(src, q), numel, dt, self.dev), src, self.buf.data_flag(src), q)

    def wait(self, part: Part):
        if part.flag is not None:
            self._wait_value(part.flag, part.value)
            part.flag = None

    def done(self, part: Part):
        """Acknowledge (stream-ordered) that the slot of ``part`` may be reused."""
        if self.kind == "nccl" or part.src < 0:
            return
        flags = (C.c_void_p * 1)(self.buf.peer_ack_flag(part.src))
        check(self.lib.hp_stage_broadcast(None, flags, 1, None, 0, self.recvd[part.src], C.c_void_p(N.stream_ptr())),
              "hp_stage_broadcast ack")

    def _copy(self, dst_ptr: int, src_ptr: int, nbytes: int):
        check(self.lib.hp_stage_send(C.c_void_p(dst_ptr), C.c_void_p(src_ptr), nbytes, None, 0,
                                     C.c_void_p(N.stream_ptr())), "hp_stage_send copy")

    def take_latent(self, part: Part):
        """x from a latent message, copied out of the slot (then released)."""
        self.wait(part)
        x = torch.empty((len(self.plan.conditions), self.plan.mixture.dim), dtype=self.xdtype, device=self.dev)
        self._copy(x.data_ptr(), part.data.data_ptr(), x.numel() * x.element_size())
        self.done(part)
        return x

    def signal_control(self, dsts, s: int):
        if self.kind == "nccl":
            import torch.distributed as dist
            for dst in dsts:
                self._nccl_work.append(dist.isend(torch.tensor([s], dtype=torch.int64, device=self.dev),
                                                  self._ranks[dst], self.group))
            return
        ptrs = list(dsts)
        flags = (C.c_void_p * len(ptrs))(*[self.buf.peer_control(r) for r in ptrs])
        check(self.lib.hp_stage_broadcast(None, flags, len(ptrs), None, 0, self.ctrl_base + s,
                                          C.c_void_p(N.stream_ptr())), "hp_stage_broadcast control")

    def wait_control(self) -> int:
        if self.kind == "nccl":
            import torch.distributed as dist
            v = torch.empty(1, dtype=torch.int64, device=self.dev)
            dist.recv(v, self._ranks[0], self.group)
            return int(v.item())
        got = C.c_uint32()
        rc = self.lib.hp_flag_poll(C.c_void_p(self.buf.control()), self.ctrl_base + 1, 6 * WAIT_TIMEOUT_NS,
                                   C.byref(got))
        if rc != 0:
            raise from_status(rc, "stage-split control word")
        return int(got.value) - self.ctrl_base

    # ---- stage split ----
    def stage_fill_local(self):
        self.den.window_fill()

    def stage_input(self, j: int):
        return self.den.stage_input(j)

    def stage_load(self, j: int, part: Part):
        self.wait(part)
        dst = self.den.stage_input(j)
        if part.data.data_ptr() != dst.data_ptr():
            self._copy(dst.data_ptr(), part.data.data_ptr(), dst.numel() * dst.element_size())
        self.done(part)

    def load_stage_x(self, x):
        self.den.load_stage_x(x)

    def stage_run(self, j: int, t: int):
        return self.den.stage_run(j, t)

    def unguided_update(self, x, eps, t):
        out, _ = self.st._advance(x, None, eps, None, t, N.HP_CTRL_NONE)
        return out

    # ---- fused updates ----
    def measured_update(self, x, parts, t, ctrl_op):
        pc, pu = parts
        remote = [p for p in parts if p.flag is not None]
        if self.wait_mode == "host":
            for p in remote:
                self.wait(p)
            fused = None
        else:
            for p in remote[:-1]:                 # a passive rank: both operands remote
                self.wait(p)
            fused = remote[-1] if remote else None    # acquired inside the sampler kernel
        st = self.st
        out = torch.empty_like(x)
        outb = self.den.input_slot() if self.den.wants_bf16_input else None
        c = st.coef[t]
        kw = {} if c is None else dict(c_sigma=c.c_sigma, c_sqrt_ab=c.c_sqrt_ab,
                                       c_sqrt_ab_prev=c.c_sqrt_ab_prev, c_sqrt_1m_ab_prev=c.c_sqrt_1m_ab_prev)
        K.sampler_step(x=x, eps_c=pc.data, eps_u=pu.data, x_out=out, x_out_bf16=outb, update=st.update, t=t,
                       w=self.plan.guidance.w, dt=1.0 / self.plan.schedule.T, ws=st.ws, ctrl=st.ctrl,
                       ctrl_op=ctrl_op, mirror_ptr=st.mirror.ptr,
                       wait_flag=None if fused is None else fused.flag,
                       wait_value=0 if fused is None else fused.value, **kw)
        if fused is not None:
            fused.flag = None
        for p in parts:
            self.done(p)
        return out

    def blend_update(self, x, parts, t, fractions):
        acc = torch.empty(x.shape, dtype=x.dtype, device=x.device)
        for d, (f, p) in enumerate(zip(fractions, parts)):
            self.wait(p)
            K.blend_accumulate(acc, p.data, f, first=(d == 0))
            self.done(p)
        xb, _ = self.st._advance(x, None, acc, None, t, N.HP_CTRL_NONE)
        return xb

    def poll(self, t):
        mr = self.st.poll(t)
        return mr.tau1, mr.tau2

    def drain(self):
        """Complete this rank's outstanding sends (NCCL work handles)."""
        for w in self._nccl_work:
            w.wait()
        self._nccl_work = []

    def finish(self, x):
        self.drain()
        return self.st.finish(x)


class GroupSession:
    """Set up one sample's group once (IPC buffers, graphs, controller) and run it
    repeatedly. FCP / hybrid plans run on a pair; layer-wise on len(devices) ranks.

    Per-link message counters and the control word increase monotonically
    across runs, so a new run can never consume a flag left over from the
    previous one."""

    def __init__(self, plan: ExecutionPlan, group=None, exchange: str = "p2p", wait: str = "device"):
        import torch.distributed as dist
        if plan.variant not in (PlanVariant.FULL_CONDITION_PARTITION, PlanVariant.HYBRID, PlanVariant.LAYER_WISE):
            raise PlanError(f"a group runs FCP, hybrid or layer-wise plans, got {plan.variant.value}")
        n = group_size(plan)
        size = dist.get_world_size(group)
        if size != n:
            raise PlanError(f"{plan.variant.value} plan needs a group of {n} ranks, got {size}")
        self.plan, self.group, self.n = plan, group, n
        self.index = dist.get_group_rank(group, dist.get_rank()) if group is not None else dist.get_rank()
        self.ops = CudaGroupOps(plan, self.index, n, group, exchange, wait)
        self.runs = 0

    def run(self, x_init=None) -> RunResult:
        import torch.distributed as dist
        plan, ops = self.plan, self.ops
        ops.begin_run(self.runs)
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
        # NCCL reduces device tensors only; gloo (CPU tests) host tensors
        on = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        red = torch.tensor([a.elapsed_time(b) / 1e3, float(sent)], dtype=torch.float64, device=on)
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


def run_pair(plan: ExecutionPlan, group=None, exchange: str = "p2p", wait: str = "device") -> RunResult:
    """Execute a FULL_CONDITION_PARTITION or HYBRID plan on this rank's pair.

    Every rank of the pair calls this with the same plan; both return the same
    x0 and series. latency_s is the max over the pair of the device time;
    comm_bytes the bytes both ranks pushed (trace.messages lists them)."""
    return GroupSession(plan, group, exchange, wait).run()


def run_layer_wise_distributed(plan: ExecutionPlan, group=None, exchange: str = "p2p",
                               wait: str = "device") -> RunResult:
    """A LAYER_WISE plan on len(plan.devices) ranks (engine.py:340-348): group
    index d is plan.devices[d]; ranks 0 and 1 return x0 and the series (the
    passive ranks of a stage-split group return x0 None)."""
    if plan.variant is not PlanVariant.LAYER_WISE:
        raise PlanError(f"run_layer_wise_distributed got a {plan.variant.value} plan")
    return GroupSession(plan, group, exchange, wait).run()


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
    lat = torch.tensor([res.latency_s], dtype=torch.float64,
                       device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(lat, op=dist.ReduceOp.MAX)
    pairs = ws // 2
    latency = float(lat.item())
    return replace(res, latency_s=latency, throughput_samples_per_s=pairs / latency,
                   speedup=pairs * serial_latency_ref(plan) / latency)


def message_counts(msgs) -> dict:
    """{(kind, step): count} of a rank's sent messages (for the contract tests)."""
    out: dict = {}
    for kind, _, s, _ in msgs:
        out[(kind, s)] = out.get((kind, s), 0) + 1
    return out


__all__ = ["StagedLoop", "CudaGroupOps", "GroupSession", "LinkBuffers", "Part", "run_pair",
           "run_layer_wise_distributed", "run_batch_level_distributed", "pair_role", "group_size",
           "message_counts", "NativeError"]
