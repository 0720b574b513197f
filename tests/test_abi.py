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


def _c_layout(tmp_path, structs):
    """sizeof / offsetof of the header's structs, from gcc on the real headers."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "hybridpar_b200_denoiser.h"', "int main(void) {"]
    for cname, fields in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f in fields:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    out = {}
    for line in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines():
        cname, key, val = line.split()
        out[(cname, key)] = int(val)
    return out


def test_ctypes_structs_match_c_layout(tmp_path):
    """Every ctypes mirror of a header struct has the C compiler's size and field offsets."""
    from paper_2602_21760_b200 import _native as N
    from paper_2602_21760_b200.denoiser import kernels as K
    mirrors = {"hp_ctrl": N.HpCtrl, "hp_ctrl_mirror": N.HpCtrlMirror, "hp_step_desc": N.HpStepDesc,
               "hp_gemm_desc": K.HpGemmDesc, "hp_attn_desc": K.HpAttnDesc}
    fields = {c: [f[0] for f in py._fields_] for c, py in mirrors.items()}
    lay = _c_layout(tmp_path, fields)
    for cname, py in mirrors.items():
        assert ctypes.sizeof(py) == lay[(cname, "size")], cname
        for f in fields[cname]:
            assert getattr(py, f).offset == lay[(cname, f)], (cname, f)


def test_integer_constants_match_python_mirrors():
    """#define HP_* integers in include/*.h equal the same-named Python constants."""
    from paper_2602_21760_b200 import _native as N
    from paper_2602_21760_b200.denoiser import kernels as K
    from paper_2602_21760_b200 import errors as E
    status = {"HP_ERR_PARAMETER": E.ParameterError, "HP_ERR_SHAPE": E.ShapeError, "HP_ERR_NUMERIC": E.NumericError,
              "HP_ERR_STEP_UNDERFLOW": E.StepUnderflowError, "HP_ERR_HISTORY": E.HistoryError,
              "HP_ERR_SEQUENCING": E.SequencingError, "HP_ERR_DEGENERATE": E.DegenerateInputError,
              "HP_ERR_PLAN": E.PlanError}
    checked = 0
    for h in (ROOT / "include").glob("*.h"):
        for m in re.finditer(r"^#define\s+(HP_\w+)\s+(-?\d+)\b", h.read_text(), flags=re.M):
            name, val = m.group(1), int(m.group(2))
            for mod in (N, K):
                for alias in (name, name[3:] if name.startswith("HP_ACT_") else None):
                    if alias and hasattr(mod, alias):
                        assert getattr(mod, alias) == val, (name, getattr(mod, alias), val)
                        checked += 1
            if name in status:                       # status code -> the reference's exception class
                assert isinstance(E.from_status(val, "x"), status[name]), name
                checked += 1
            elif name.startswith("HP_ERR_"):          # CUDA / unsupported / timeout: NativeError
                assert isinstance(E.from_status(val, "x"), E.NativeError), name
                checked += 1
    assert checked >= 30
