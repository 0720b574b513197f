"""ctypes binding of the C-ABI extension (include/hybridpar_b200.h).

The library is built in-tree by ``_build.py`` into ``lib/libhybridpar_b200.so``.
There is no fallback: if the library is missing or no CUDA device is visible,
every compute entry point raises ``NativeError``. Loading the library itself
(symbol resolution) works without a GPU so the CPU test-suite can check the
exported surface.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import NativeError, check

_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libhybridpar_b200.so"
if os.environ.get("HP_LIB_VARIANT"):          # A/B kernel experiments (tools/): lib/<variant>.so
    _LIB_PATH = _LIB_PATH.parent / (os.environ["HP_LIB_VARIANT"] + ".so")
_lock = threading.Lock()
_lib = None

# ---- constants mirrored from the header -------------------------------------
HP_F64, HP_F32, HP_BF16 = 0, 1, 2
HP_UPDATE_DDIM, HP_UPDATE_EULER, HP_UPDATE_NONE = 0, 1, 2
HP_CTRL_NONE, HP_CTRL_RECORD, HP_CTRL_RECORD_UPDATE = 0, 1, 2
HP_STAGE_WARM_UP, HP_STAGE_PARALLELISM, HP_STAGE_FULLY_CONNECTING = 0, 1, 2
HP_MAX_T = 1024
HP_MAX_PEERS = 8
HP_IPC_HANDLE_BYTES = 64


class HpCtrl(C.Structure):
    _fields_ = [
        ("L", C.c_int32), ("tau_cap", C.c_int32), ("k", C.c_int32), ("T", C.c_int32),
        ("g_slope", C.c_double),
        ("tau1", C.c_int32), ("tau2", C.c_int32), ("stage", C.c_int32),
        ("steps_done", C.c_int32), ("last_t", C.c_int32), ("last_recorded_t", C.c_int32),
        ("status", C.c_int32), ("n_recorded", C.c_int32),
        ("m", C.c_double * (HP_MAX_T + 1)),
        ("has", C.c_uint8 * (HP_MAX_T + 1)),
    ]


class HpCtrlMirror(C.Structure):
    _fields_ = [
        ("seq", C.c_int32), ("tau1", C.c_int32), ("tau2", C.c_int32), ("stage", C.c_int32),
        ("status", C.c_int32), ("t", C.c_int32), ("m", C.c_double),
    ]


class HpStepDesc(C.Structure):
    _fields_ = [
        ("x", C.c_void_p), ("x_dtype", C.c_int32),
        ("eps_c", C.c_void_p),
        ("eps_u", C.c_void_p), ("eps_dtype", C.c_int32),
        ("x_out", C.c_void_p),
        ("x_out_bf16", C.c_void_p),
        ("n", C.c_int64),
        ("update", C.c_int32),
        ("t", C.c_int32),
        ("w", C.c_double),
        ("c_sigma", C.c_double), ("c_sqrt_ab", C.c_double), ("c_sqrt_ab_prev", C.c_double),
        ("c_sqrt_1m_ab_prev", C.c_double), ("dt", C.c_double),
        ("partials", C.c_void_p), ("ticket", C.c_void_p), ("nonfinite", C.c_void_p),
        ("m_out", C.c_void_p), ("status", C.c_void_p),
        ("ctrl", C.c_void_p), ("ctrl_op", C.c_int32),
        ("mirror", C.c_void_p),
        ("wait_flag", C.c_void_p), ("wait_value", C.c_uint32),
    ]


_VP, _I32, _I64, _U32, _F64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_double

# name -> (restype, argtypes); every symbol include/*.h declares
SIGNATURES = {
    "hp_step_blocks": (_I64, [_I64]),
    "hp_sampler_step": (C.c_int, [C.POINTER(HpStepDesc), _VP]),
    "hp_rel_mae": (C.c_int, [_VP, _VP, _I32, _I64, _VP, _VP, _VP, _VP, _VP, _VP]),
    "hp_blend_accumulate": (C.c_int, [_VP, _I32, _VP, _I32, _F64, _I32, _I64, _VP]),
    "hp_ctrl_init": (C.c_int, [_VP, _I32, _F64, _I32, _I32, _I32, _VP]),
    "hp_ctrl_step": (C.c_int, [_VP, _I32, _VP, _I32, _VP, _VP]),
    "hp_ipc_get_handle": (C.c_int, [_VP, C.c_char_p]),
    "hp_ipc_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "hp_ipc_close": (C.c_int, [_VP]),
    "hp_enable_peer": (C.c_int, [_I32]),
    "hp_signal": (C.c_int, [_VP, _U32, _VP]),
    "hp_flag_wait": (C.c_int, [_VP, _U32, _VP, C.c_uint64, _VP]),
    "hp_flag_poll": (C.c_int, [_VP, _U32, C.c_uint64, C.POINTER(C.c_uint32)]),
    "hp_stage_send": (C.c_int, [_VP, _VP, _I64, _VP, _U32, _VP]),
    "hp_stage_broadcast": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int32, _VP, _I64, _U32, _VP]),
    "hp_alloc": (C.c_int, [_I64, C.POINTER(C.c_void_p)]),
    "hp_free": (C.c_int, [_VP]),
    "hp_version": (C.c_char_p, []),
    "hp_device_sm_count": (C.c_int, [_VP]),
}

# optional extra signature tables registered by the denoiser-kernel bindings
_EXTRA: dict = {}


def register_signatures(table: dict) -> None:
    _EXTRA.update(table)
    if _lib is not None:
        _bind(_lib, table)


def _bind(lib, table):
    for name, (res, args) in table.items():
        fn = getattr(lib, name)  # AttributeError -> missing export, loud
        fn.restype = res
        fn.argtypes = args


def library_path() -> Path:
    return _LIB_PATH


def load():
    """Load (once) and return the ctypes library handle; raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not _LIB_PATH.exists():
            raise NativeError(
                f"CUDA extension not built: {_LIB_PATH} is missing "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
        lib = C.CDLL(str(_LIB_PATH), mode=os.RTLD_GLOBAL if hasattr(os, "RTLD_GLOBAL") else 0)
        _bind(lib, SIGNATURES)
        _bind(lib, _EXTRA)
        _lib = lib
    return _lib


def require_cuda():
    """The compute path: library + a visible CUDA device, or a loud error."""
    import torch
    lib = load()
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device visible: hybridpar_b200 has no CPU path")
    return lib


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def call(name: str, *args, what: str | None = None) -> int:
    lib = load()
    rc = getattr(lib, name)(*args)
    check(rc, what or name)
    return rc
