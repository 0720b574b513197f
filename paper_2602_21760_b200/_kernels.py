"""Typed wrappers that launch the sampler / monitor kernels on torch tensors.

Only device pointers, sizes and the current CUDA stream cross into the C ABI
(``hp_sampler_step`` and friends, include/hybridpar_b200.h). Workspaces are
allocated once per device and reused, so the hot loop never allocates and
every launch is CUDA-graph capturable.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from .errors import NativeError, ShapeError, check, from_status

_DT = {torch.float64: N.HP_F64, torch.float32: N.HP_F32, torch.bfloat16: N.HP_BF16}


def hp_dtype(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ShapeError(f"unsupported dtype {t.dtype}") from None


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class StepWorkspace:
    """Per-device scratch for the fused step: partials, ticket, counters."""

    def __init__(self, device: torch.device):
        lib = N.require_cuda()
        nblk = int(lib.hp_step_blocks(1 << 40))
        self.device = device
        self.partials = torch.zeros(2 * nblk, dtype=torch.float64, device=device)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=device)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=device)
        self.m = torch.zeros(1, dtype=torch.float64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)


_WS: dict = {}


def workspace(device=None) -> StepWorkspace:
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    ws = _WS.get(dev)
    if ws is None:
        ws = _WS[dev] = StepWorkspace(dev)
    return ws


def sampler_step(*, x, eps_c, eps_u, x_out, update, t=0, w=0.0, c_sigma=0.0, c_sqrt_ab=1.0,
                 c_sqrt_ab_prev=1.0, c_sqrt_1m_ab_prev=0.0, dt=0.0, x_out_bf16=None,
                 ws: StepWorkspace | None = None, discrepancy=True, m_out=None, status=None,
                 ctrl=None, ctrl_op=N.HP_CTRL_NONE, mirror_ptr=None, wait_flag=None,
                 wait_value=0, stream=None) -> None:
    """Launch one hp_sampler_step (K1 + K2 tail). Asynchronous."""
    lib = N.load()
    d = N.HpStepDesc()
    d.x = None if x is None else x.data_ptr()
    d.x_dtype = hp_dtype(x_out)
    d.eps_c = eps_c.data_ptr()
    d.eps_u = None if eps_u is None else eps_u.data_ptr()
    d.eps_dtype = hp_dtype(eps_c)
    d.x_out = x_out.data_ptr()
    d.x_out_bf16 = None if x_out_bf16 is None else x_out_bf16.data_ptr()
    d.n = eps_c.numel()
    d.update = update
    d.t = int(t)
    d.w = float(w)
    d.c_sigma, d.c_sqrt_ab = float(c_sigma), float(c_sqrt_ab)
    d.c_sqrt_ab_prev, d.c_sqrt_1m_ab_prev, d.dt = float(c_sqrt_ab_prev), float(c_sqrt_1m_ab_prev), float(dt)
    if discrepancy:
        ws = ws or workspace(eps_c.device)
        d.partials = ws.partials.data_ptr()
        d.ticket = ws.ticket.data_ptr()
        d.nonfinite = ws.nonfinite.data_ptr()
        d.m_out = (m_out if m_out is not None else ws.m).data_ptr()
        d.status = (status if status is not None else ws.status).data_ptr()
    d.ctrl = None if ctrl is None else ctrl.data_ptr()
    d.ctrl_op = int(ctrl_op)
    d.mirror = mirror_ptr
    d.wait_flag = None if wait_flag is None else (wait_flag if isinstance(wait_flag, int) else wait_flag.data_ptr())
    d.wait_value = int(wait_value)
    rc = lib.hp_sampler_step(C.byref(d), C.c_void_p(N.stream_ptr(stream)))
    check(rc, "hp_sampler_step")


def read_status(ws: StepWorkspace, what: str) -> None:
    """Synchronising status check used by the reference-shaped primitives."""
    code = int(ws.status.item())
    if code != 0:
        ws.status.zero_()
        raise from_status(code, what)


def rel_mae_dev(eps_c: torch.Tensor, eps_u: torch.Tensor, ws: StepWorkspace | None = None):
    lib = N.load()
    ws = ws or workspace(eps_c.device)
    rc = lib.hp_rel_mae(_ptr(eps_c), _ptr(eps_u), hp_dtype(eps_c), eps_c.numel(), _ptr(ws.partials),
                        _ptr(ws.ticket), _ptr(ws.nonfinite), _ptr(ws.m), _ptr(ws.status),
                        C.c_void_p(N.stream_ptr()))
    check(rc, "hp_rel_mae")
    return ws


def blend_accumulate(acc: torch.Tensor, eps: torch.Tensor, f: float, first: bool) -> None:
    lib = N.load()
    rc = lib.hp_blend_accumulate(_ptr(acc), hp_dtype(acc), _ptr(eps), hp_dtype(eps), float(f),
                                 1 if first else 0, acc.numel(), C.c_void_p(N.stream_ptr()))
    check(rc, "hp_blend_accumulate")


CTRL_BYTES = C.sizeof(N.HpCtrl)


def ctrl_alloc(device) -> torch.Tensor:
    # raw bytes, 8-byte aligned (torch allocations are 512-byte aligned)
    return torch.zeros(CTRL_BYTES, dtype=torch.uint8, device=device)


def ctrl_init(ctrl: torch.Tensor, L: int, g_slope: float, tau_cap: int, k: int, T: int) -> None:
    lib = N.load()
    check(lib.hp_ctrl_init(_ptr(ctrl), int(L), float(g_slope), int(tau_cap), int(k), int(T),
                           C.c_void_p(N.stream_ptr())), "hp_ctrl_init")


def ctrl_step(ctrl: torch.Tensor, t: int, m: torch.Tensor | None, op: int, mirror_ptr=None) -> None:
    lib = N.load()
    check(lib.hp_ctrl_step(_ptr(ctrl), int(t), _ptr(m), int(op), mirror_ptr,
                           C.c_void_p(N.stream_ptr())), "hp_ctrl_step")


def ctrl_read(ctrl: torch.Tensor) -> N.HpCtrl:
    host = ctrl.detach().cpu().numpy().tobytes()
    return N.HpCtrl.from_buffer_copy(host)


class PinnedMirror:
    """Mapped pinned host memory the sampler tail publishes the switch into."""

    def __init__(self):
        self._buf = torch.zeros(C.sizeof(N.HpCtrlMirror), dtype=torch.uint8).pin_memory()
        self.view = N.HpCtrlMirror.from_address(self._buf.data_ptr())
        self.view.seq = -1

    @property
    def ptr(self) -> int:
        # pinned host memory allocated by torch is portable+mapped under UVA:
        # the host address is also the device address
        return self._buf.data_ptr()

    def wait_step(self, t: int, timeout_s: float = 60.0):
        import time
        want = N.HP_MAX_T + 1 - int(t)
        t0 = time.perf_counter()
        while C.c_int32.from_address(self._buf.data_ptr()).value < want:
            if time.perf_counter() - t0 > timeout_s:
                raise NativeError(f"controller mirror for t={t} never arrived")
        return self.view


def ensure_cuda_tensor(a, dtype=None):
    """(tensor on the current CUDA device, came_from_numpy) for array-likes."""
    import numpy as np
    if isinstance(a, torch.Tensor):
        t = a
        if t.dtype not in _DT:
            t = t.to(torch.float64)
        if dtype is not None:
            t = t.to(dtype)
        if not t.is_cuda:
            N.require_cuda()
            t = t.cuda()
        return t.contiguous(), False
    arr = np.asarray(a, dtype=np.float64)
    N.require_cuda()
    t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
    if dtype is not None:
        t = t.to(dtype)
    return t, True
