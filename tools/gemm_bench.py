"""f3d_gemm vs the library GEMM (cuBLAS via torch) at the stage shapes.

    python tools/gemm_bench.py [--d 96]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_16481_b200 import _lib as L  # noqa: E402


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=96)
ap.add_argument("--n", type=int, default=100_000)
a = ap.parse_args()
d, n = a.d, a.n
for name, K, N, gelu in (("qkv", d, 3 * d, 0), ("o", d, d, 0), ("mlp_in", d, 4 * d, 1),
                         ("mlp_out", 4 * d, d, 0)):
    x = torch.randn((n, K), device="cuda").to(torch.bfloat16)
    w = torch.randn((K, N), device="cuda").to(torch.bfloat16)
    wt = w.t().contiguous()
    b = torch.zeros(N, device="cuda")
    y = torch.empty((n, N), device="cuda", dtype=torch.bfloat16)
    ours = timeit(lambda: L.call("f3d_gemm", L.ptr(x), K, n, K, L.ptr(wt), N, L.ptr(b), gelu,
                                 L.ptr(y), N, None, L.stream()))
    lib = timeit(lambda: torch.mm(x, w, out=y))
    nbytes = 2 * n * (K + N)
    print(f"{name:8s} n={n} K={K} N={N} gelu={gelu}: f3d_gemm {ours:7.1f} us "
          f"({nbytes / ours / 1e3:6.0f} GB/s)  cuBLAS mm {lib:7.1f} us", flush=True)
