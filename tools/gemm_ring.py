"""Per-launch GEMM timeline inside the SDXL forward graph: builds nothing itself; run
with HP_LIB_VARIANT=trace after `python tools/gemm_ring.py build` (compiles
lib/trace.so with -DHP_GEMM_TRACE). For every CTA-pair GEMM launch of one forward
(cluster 0 leader, globaltimer ns): the wait for the previous kernel (entry -> PDL
wait passed), first-load latency (PDL passed -> first stage landed), main loop
(first stage -> all MMAs of tile 0 issued), epilogue of tile 0, and the tail to the
kernel's final barrier; then totals per (M, N, K).

    python tools/gemm_ring.py build
    HP_LIB_VARIANT=trace python tools/gemm_ring.py [b1] [out.txt]
"""
import collections
import ctypes as C
import os
import subprocess
import sys

sys.path.insert(0, ".")


def build():
    from paper_2602_21760_b200 import _build
    objs = []
    for src in sorted(_build.CSRC.glob("*.cu")):
        obj = _build.OBJDIR / f"trace_{src.stem}.o"
        cmd = [_build._nvcc(), *_build.ARCH, *_build.NVCC_FLAGS, "-DHP_GEMM_TRACE", f"-I{_build.INCLUDE}",
               f"-I{_build.CSRC}", "-c", str(src), "-o", str(obj)]
        _build.OBJDIR.mkdir(parents=True, exist_ok=True)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    out = _build.LIBDIR / "trace.so"
    subprocess.run([_build._nvcc(), *_build.ARCH, "-shared", "-o", str(out), *objs, "-lcuda"], check=True)
    print("built", out)


def main():
    if "build" in sys.argv:
        return build()
    import torch
    from paper_2602_21760_b200 import _native as N, pipelines
    from paper_2602_21760_b200.denoiser import weights as Wm
    assert os.environ.get("HP_LIB_VARIANT") == "trace", "run with HP_LIB_VARIANT=trace"
    b1 = "b1" in sys.argv
    outp = [a for a in sys.argv[1:] if a != "b1"]
    spec = Wm.SDXL
    den = pipelines.build_sdxl_denoiser(spec, n_prompts=1, steps=50)
    x = torch.randn(1, spec.latent_hw * spec.latent_hw * 4, device="cuda")
    den.load_input(x)
    run = (lambda: den.conditional(x, 30)) if b1 else (lambda: den.branches(x, 30, den.input_slot()))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    lib = N.load()
    run()
    torch.cuda.synchronize()
    import numpy as np
    ring = np.zeros((4096, 13), dtype=np.uint64)
    ctr = np.zeros(1, dtype=np.uint32)
    f = lib.hp_debug_symbol
    f.restype = C.c_int
    f.argtypes = [C.c_char_p, C.c_void_p, C.c_size_t]
    for name, arr in (("g_gemm_ring", ring), ("g_gemm_ctr", ctr)):
        rc = f(name.encode(), arr.ctypes.data, arr.nbytes)
        assert rc == 0, (name, rc)
    n = int(ctr[0])
    lines = []
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0])
    # one forward = the launches after the last but one run(); find it by M,N,K of the first launch
    first = tuple(ring[(n - 1) % 4096][9:12])
    idx = [i for i in range(max(0, n - 2000), n) if tuple(ring[i % 4096][9:12]) == first]
    per = n - 1 - idx[-2] if len(idx) >= 2 else None
    start = n - per if per else max(0, n - 700)
    prev_end = None
    for i in range(start, n):
        r = ring[i % 4096].astype(np.int64)
        key = (f"M={r[9]} N={r[10]} K={r[11]} splitK bn={r[12] - 1000}" if r[12] >= 1000
               else f"M={r[9]} N={r[10]} K={r[11]} bn={r[12]}")
        # split-K: event 3 = partials exchanged (between acc ready and the epilogue)
        wait = (r[2] - r[0]) / 1e3
        gap = (r[2] - prev_end) / 1e3 if prev_end is not None else 0.0
        first_land = (r[4] - r[2]) / 1e3
        loop = (r[5] - r[4]) / 1e3
        epi = (r[7] - r[6]) / 1e3
        tail = (r[8] - r[7]) / 1e3
        total = (r[8] - r[2]) / 1e3
        if r[12] >= 1000:   # split-K: 'epi' split into exchange (acc ready -> partials in) + epilogue
            key += f" [xch {(r[3] - r[6]) / 1e3:.2f} epi {(r[7] - r[3]) / 1e3:.2f}]"
        a = agg[key]
        a[0] += 1
        for j, v in enumerate((gap, first_land, loop, epi, tail, total)):
            a[1 + j] += v
        prev_end = r[8]
    lines.append(f"{'B=1' if b1 else 'B=2'} forward: {n - start} pair-GEMM launches (cluster 0 leader, us)")
    lines.append(f"{'shape':36s} {'n':>4s} {'gap':>6s} {'1st ld':>6s} {'loop':>6s} {'epi':>6s} {'tail':>6s} "
                 f"{'pdl->end':>8s} {'x n':>8s}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][6]):
        c = a[0]
        lines.append(f"{k:36s} {c:4d} {a[1] / c:6.2f} {a[2] / c:6.2f} {a[3] / c:6.2f} {a[4] / c:6.2f} "
                     f"{a[5] / c:6.2f} {a[6] / c:8.2f} {a[6]:8.1f}")
    text = "\n".join(lines)
    print(text)
    if outp:
        open(outp[0], "w").write(text + "\n")


if __name__ == "__main__":
    main()
