"""Isolated timing of f3d_gemm_gelu vs cuBLAS GEMM + f3d_bias_gelu at several
row counts (d=96): python tools/gemm_gelu_bench.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2412_16481_b200 import _lib as L  # noqa: E402


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


d = 96
for n in (50_000, 100_000, 400_000, 1_000_000):
    x = torch.randn((n, d), device="cuda").to(torch.bfloat16)
    w = (torch.randn((d, 4 * d), device="cuda") / d ** 0.5).to(torch.bfloat16)
    wt = w.t().contiguous()
    b = torch.randn((4 * d,), device="cuda") * 0.1
    u = torch.empty((n, 4 * d), device="cuda", dtype=torch.bfloat16)

    def fused():
        L.call("f3d_gemm_gelu", L.ptr(x), d, n, d, L.ptr(wt), L.ptr(b), L.ptr(u), 4 * d, None,
               L.stream())

    def unfused():
        torch.mm(x, w, out=u)
        L.call("f3d_bias_gelu", L.ptr(u), n, 4 * d, L.ptr(b), L.stream())

    def gemm_only():
        torch.mm(x, w, out=u)
    tf, tu, tg = timeit(fused), timeit(unfused), timeit(gemm_only)
    gb = n * d * 2 + n * 4 * d * 2
    print(f"n={n}: fused {tf:.1f} us ({gb / tf / 1e3:.0f} GB/s)  cublas+bias_gelu {tu:.1f} us "
          f"(gemm alone {tg:.1f})")
