"""CPU: the C-ABI library loads and exports every symbol include/*.h declares."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = h.read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(hp_\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


def test_header_declares_entry_points():
    names = _declared()
    for must in ("hp_sampler_step", "hp_rel_mae", "hp_ctrl_step", "hp_ipc_open", "hp_signal",
                 "hp_stage_send", "hp_blend_accumulate"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2602_21760_b200 import _native as N
    lib = N.load()
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_every_declared_symbol():
    from paper_2602_21760_b200 import _native as N
    import paper_2602_21760_b200.denoiser.kernels  # noqa: F401  registers the denoiser table
    bound = set(N.SIGNATURES) | set(N._EXTRA)
    missing = sorted(_declared() - bound)
    assert not missing, missing


def test_struct_layouts_match_header():
    from paper_2602_21760_b200 import _native as N
    # hp_ctrl: 4 int + double + 8 int + (T+1) doubles + (T+1) bytes, padded to 8
    base = 4 * 4 + 8 + 8 * 4 + 8 * (N.HP_MAX_T + 1) + (N.HP_MAX_T + 1)
    assert ctypes.sizeof(N.HpCtrl) == (base + 7) // 8 * 8
    assert ctypes.sizeof(N.HpCtrlMirror) == 32


def test_version_string_without_gpu():
    from paper_2602_21760_b200 import _native as N
    assert b"sm_100a" in N.load().hp_version()


def test_compute_path_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    from paper_2602_21760_b200 import GuidanceParams, NativeError, cfg_combine
    with pytest.raises(NativeError):
        cfg_combine(np.ones(4), np.zeros(4), GuidanceParams(1.0))
