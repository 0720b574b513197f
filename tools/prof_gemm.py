"""Time one GEMM shape through hp_gemm, back-to-back inside a CUDA graph (no host
overhead, PDL between launches), for quick sweeps and ncu targets.

    python tools/prof_gemm.py M N K [block_n] [act] [reps] [eager]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21760_b200.denoiser import kernels as K  # noqa: E402


def main():
    if sys.argv[1] == "conv":      # conv n h w cin cout stride [bn] [reps]
        n, h, w, ci, co, st = (int(v) for v in sys.argv[2:8])
        bn = int(sys.argv[8]) if len(sys.argv) > 8 else 0
        reps = int(sys.argv[9]) if len(sys.argv) > 9 else 20
        x = torch.randn(n * h * w, ci, device="cuda").bfloat16()
        wt = (torch.randn(co, 9 * ci, device="cuda") * (9 * ci) ** -0.5).bfloat16()
        bias = torch.randn(co, device="cuda")
        M = n * (h // st) * (w // st)
        out = torch.empty(M, co, device="cuda", dtype=torch.bfloat16)
        run = lambda: K.gemm(x, wt, bias=bias, out=out, block_n=bn, conv=(n, h, w, ci, st))  # noqa: E731
        for _ in range(3):
            run()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                run()
        g.replay()
        torch.cuda.synchronize()
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record()
        g.replay()
        e_.record()
        torch.cuda.synchronize()
        ms = s_.elapsed_time(e_) / reps
        print(f"conv n={n} {h}x{w} {ci}->{co} s{st} bn={bn} graph: {ms * 1e3:.1f} us "
              f"{2.0 * M * co * 9 * ci / ms / 1e9:.1f} TFLOP/s")
        return
    M, N, Kd = (int(v) for v in sys.argv[1:4])
    bn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    act = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    reps = int(sys.argv[6]) if len(sys.argv) > 6 else 20
    eager = "eager" in sys.argv[7:]
    use_ln = "ln" in sys.argv[7:]
    use_stats = "stats" in sys.argv[7:]
    use_fold = "fold" in sys.argv[7:]
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    w = (torch.randn(N, Kd, device="cuda") * Kd ** -0.5).bfloat16()
    bias = torch.randn(N, device="cuda")
    out = torch.empty(M, N // 2 if act == 3 else N, device="cuda", dtype=torch.bfloat16)
    ln = None
    if use_ln:
        ln = (torch.ones(N, device="cuda"), torch.zeros(N, device="cuda"), 1e-5,
              torch.empty(M, N, device="cuda", dtype=torch.bfloat16))
    res = torch.randn(M, N, device="cuda").bfloat16() if use_ln else None
    kw = {}
    if use_stats or use_fold:
        rs = K.RowStats(2 * M * max(N, Kd) // 64, "cuda")
        if use_stats:
            kw["stats_out"] = rs
        else:
            rs.parts, rs.part_n = Kd // 160 if Kd % 160 == 0 else Kd // 128, 160 if Kd % 160 == 0 else 128
            rs.buf[:2 * M * rs.parts].view(-1, 2)[:, 0] = 0.1
            rs.buf[:2 * M * rs.parts].view(-1, 2)[:, 1] = float(rs.part_n)
            fold = K.FoldedLN(w.float(), torch.ones(Kd, device="cuda"), torch.zeros(Kd, device="cuda"), bias=bias)
            w, bias = fold.w, fold.bias
            kw["ln_fold"] = (rs, fold)
    run = lambda: K.gemm(a, w, bias=bias, out=out, act=act, block_n=bn, residual=res, ln=ln, **kw)  # noqa: E731
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    if eager:
        body = lambda: [run() for _ in range(reps)]  # noqa: E731
    else:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                run()
        body = g.replay
    body()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    body()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"gemm M={M} N={N} K={Kd} bn={bn} act={act} {'eager' if eager else 'graph'}: "
          f"{' +LN' if use_ln else ''}{' +stats' if use_stats else ''}{' +fold' if use_fold else ''} {ms * 1e3:.1f} us {2.0 * M * N * Kd / ms / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
