"""Build lib/<name>.so from the current sources with extra nvcc defines, for A/B runs
with HP_LIB_VARIANT=<name> (tools/ab_var.sh, tools/gn_parts_time.py ...).

    python tools/build_variant.py gnd2 -DHP_GN_PARTS_DEPTH=2
"""
import subprocess
import sys

sys.path.insert(0, ".")
from paper_2602_21760_b200 import _build  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    objs = []
    _build.OBJDIR.mkdir(parents=True, exist_ok=True)
    for src in sorted(_build.CSRC.glob("*.cu")):
        obj = _build.OBJDIR / f"{name}_{src.stem}.o"
        cmd = [_build._nvcc(), *_build.ARCH, *_build.NVCC_FLAGS, *defs, f"-I{_build.INCLUDE}",
               f"-I{_build.CSRC}", "-c", str(src), "-o", str(obj)]
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    out = _build.LIBDIR / f"{name}.so"
    subprocess.run([_build._nvcc(), *_build.ARCH, "-shared", "-o", str(out), *objs, "-lcuda"], check=True)
    print(f"built {out}")


if __name__ == "__main__":
    main()
