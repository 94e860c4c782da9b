"""GPU: f3d_gemm (csrc/gemm_tc.cu, tcgen05 + TMA) against an fp32 torch
reference of the same op, y = x W (+ b) (GELU-erf), at the stage shapes of
configs B-D (d = 96, 192, 384, 512; bw/stage.py:135-138, 146-158), with the
bf16 output rounding as the only error source (tolerance 1e-2 relative
Frobenius, measured ~2e-3)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2412_16481_b200 import _lib as L  # noqa: E402

SHAPES = [(100_000, 96, 288), (50_000, 96, 96), (100_000, 384, 96), (4096, 96, 384),
          (30_000, 384, 1152), (20_000, 384, 384), (12_000, 1536, 384), (9_000, 512, 1536),
          (7_000, 2048, 512), (777, 192, 576), (129, 192, 768), (1, 96, 96), (255, 32, 16)]


def _run(n, K, N, gelu, bias=True, n_dev=None, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((n, K), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((K, N), device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g) if bias else None
    y = torch.full((n, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    wt = w.t().contiguous()
    nd = None if n_dev is None else torch.tensor([n_dev], dtype=torch.int32, device="cuda")
    L.call("f3d_gemm", L.ptr(x), x.stride(0), n, K, L.ptr(wt), N, L.ptr(b), int(gelu), L.ptr(y),
           y.stride(0), L.ptr(nd), L.stream())
    ref = x.float() @ w.float()
    if bias:
        ref = ref + b
    if gelu:
        ref = torch.nn.functional.gelu(ref)
    return y, ref


@pytest.mark.parametrize("n,K,N", SHAPES)
@pytest.mark.parametrize("gelu", [False, True])
def test_gemm_matches_fp32_reference(n, K, N, gelu):
    assert L.load().f3d_gemm_supported(K, N)
    y, ref = _run(n, K, N, gelu)
    assert torch.isfinite(y).all()
    rel = float((y.float() - ref).norm() / ref.norm())
    assert rel < 1e-2, rel


def test_gemm_device_row_count_leaves_tail_untouched():
    n, K, N = 5000, 96, 288
    y, ref = _run(n, K, N, False, n_dev=3333)
    assert torch.isnan(y[3333:].float()).all()
    rel = float((y[:3333].float() - ref[:3333]).norm() / ref[:3333].norm())
    assert rel < 1e-2, rel


def test_gemm_no_bias_and_strided_rows():
    n, K, N = 3000, 96, 96
    g = torch.Generator(device="cuda").manual_seed(5)
    big = torch.randn((n, 3 * K), device="cuda", generator=g).to(torch.bfloat16)
    x = big[:, K:2 * K]                                  # row stride 3K
    w = torch.randn((K, N), device="cuda", generator=g).to(torch.bfloat16)
    out = torch.zeros((n, 2 * N), device="cuda", dtype=torch.bfloat16)
    y = out[:, N:]
    L.call("f3d_gemm", L.ptr(x), x.stride(0), n, K, L.ptr(w.t().contiguous()), N, None, 0,
           L.ptr(y), y.stride(0), None, L.stream())
    ref = x.float() @ w.float()
    assert float((y.float() - ref).norm() / ref.norm()) < 1e-2
    assert (out[:, :N] == 0).all()


def test_gemm_rejects_unsupported_shapes():
    lib = L.load()
    assert not lib.f3d_gemm_supported(40, 96)       # K % 32
    assert not lib.f3d_gemm_supported(96, 40)       # N % 16
