"""GPU parity for bucket-swin attention, positional encoding and the stage
against golden fixtures (reference output) and the CPU oracle.

Tolerances (measured bf16 emulation): attention per scope
<= 1e-2 relative Frobenius, stage <= 2e-2."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import restated as O

pytestmark = pytest.mark.gpu

import paper_2412_16481_b200 as F  # noqa: E402
from paper_2412_16481_b200.errors import ConfigError, NumericError  # noqa: E402

ATT_TOL = 1e-2
STAGE_TOL = 2e-2


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def test_attention_golden():
    g = load_golden("attention.npz")
    for i, (m, d, H) in enumerate(((16, 64, 4), (100, 64, 4), (300, 96, 4), (200, 48, 2),
                                   (130, 128, 1), (64, 32, 2))):
        p = F.AttentionParams(d_model=d, n_heads=H)
        out = F.tiled_attention(g[f"a{i}_Q"], g[f"a{i}_K"], g[f"a{i}_V"], p, ranges=[(0, m)])
        assert out.shape == (m, d)
        assert rel(out, g[f"a{i}_out"]) < ATT_TOL, (i, rel(out, g[f"a{i}_out"]))
        dense = F.reference_attention(g[f"a{i}_Q"], g[f"a{i}_K"], g[f"a{i}_V"], p)
        assert rel(dense, g[f"a{i}_out"]) < ATT_TOL


def test_attention_ranges_and_mask_golden():
    g = load_golden("attention.npz")
    rg = [tuple(r) for r in g["rg_ranges"]]
    out = F.tiled_attention(g["rg_Q"], g["rg_K"], g["rg_V"], F.AttentionParams(64, 4), ranges=rg,
                            mask=g["rg_mask"])
    ref = g["rg_out"]
    assert out.shape == ref.shape
    assert rel(out, ref) < ATT_TOL
    # masked query rows are exactly zero
    rows = np.concatenate([np.arange(a, b) for a, b in rg])
    assert np.all(out[~g["rg_mask"][rows]] == 0)


def test_positional_encoding_golden():
    g = load_golden("attention.npz")
    np.testing.assert_allclose(F.positional_encoding(g["pe_coords"], 96), g["pe_96"], atol=1e-12)
    np.testing.assert_allclose(F.positional_encoding(g["pe_coords"], 12), g["pe_12"], atol=1e-12)
    with pytest.raises(ConfigError):
        F.positional_encoding(g["pe_coords"], 64)


@pytest.mark.parametrize("d,H", [(64, 4), (96, 4), (384, 4), (512, 4), (12, 2), (40, 5), (256, 2)])
def test_attention_random_scopes_vs_oracle(d, H):
    """Multi-segment scopes (two disjoint ranges) and ragged lengths."""
    r = np.random.default_rng(d * 7 + H)
    for m in (16, 77, 200, 1000):
        N = m + 50
        Q, K, V = (r.normal(size=(N, d)) for _ in range(3))
        cut = m // 2
        ranges = [(3, 3 + cut), (3 + cut + 40, 3 + m + 40)]
        out = F.tiled_attention(Q, K, V, F.AttentionParams(d, H), ranges=ranges)
        ref = O.attention_ranges(Q, K, V, H, ranges)
        assert rel(out, ref) < ATT_TOL, (d, H, m, rel(out, ref))


@pytest.mark.parametrize("nseg", [8, 9, 13])
@pytest.mark.parametrize("d,H", [(96, 4), (64, 2), (512, 4)])
def test_attention_many_segment_scope(nseg, d, H):
    """A scope made of many disjoint row ranges: the kernel keeps up to 8
    segments per item in its shared-memory item record and maps rows of
    longer scopes through the global segment arrays."""
    r = np.random.default_rng(nseg * 31 + d)
    lens = r.integers(1, 160, size=nseg)
    lens[nseg // 2] = 1                      # a one-row segment
    ranges, at = [], 5
    for ln in lens:
        ranges.append((at, at + int(ln)))
        at += int(ln) + int(r.integers(1, 30))
    N = at + 7
    Q, K, V = (r.normal(size=(N, d)) for _ in range(3))
    out = F.tiled_attention(Q, K, V, F.AttentionParams(d, H), ranges=ranges)
    ref = O.attention_ranges(Q, K, V, H, ranges)
    assert rel(out, ref) < ATT_TOL, (nseg, d, H, rel(out, ref))


def test_attention_extreme_logits_and_errors():
    r = np.random.default_rng(0)
    Q = r.normal(size=(128, 32)) * 30
    K = r.normal(size=(128, 32)) * 30
    V = r.normal(size=(128, 32))
    out = F.tiled_attention(Q, K, V, F.AttentionParams(32, 2))
    ref = O.attention_dense(Q, K, V, 2)
    assert np.isfinite(out).all()
    assert rel(out, ref) < 5e-2   # near-one-hot softmax: bf16 logits dominate the error
    Q[3, 1] = np.nan
    with pytest.raises(NumericError):
        F.tiled_attention(Q, K, V, F.AttentionParams(32, 2))
    with pytest.raises(ConfigError):
        F.tiled_attention(K, K, V[:, :16], F.AttentionParams(32, 2))


def test_all_masked_scope_warns():
    r = np.random.default_rng(1)
    Q = r.normal(size=(40, 16))
    with pytest.warns(RuntimeWarning):
        out = F.tiled_attention(Q, Q, Q, F.AttentionParams(16, 2), ranges=[(0, 40)],
                                mask=np.zeros(40, dtype=bool))
    assert np.all(out == 0)


def test_zero_gather_bytes():
    F.copy_meter.reset()
    r = np.random.default_rng(2)
    Q = r.normal(size=(300, 32))
    F.tiled_attention(Q, Q, Q, F.AttentionParams(32, 2), ranges=[(0, 100), (150, 300)])
    assert F.copy_meter.bytes["gather"] == 0
    assert F.copy_meter.bytes["attention"] > 0


# -------------------------------------------------------------------- stage

@pytest.mark.parametrize("tag", ["s0", "s1"])
def test_stage_golden(tag):
    g = load_golden("stage.npz")
    seed, n, K, S, d, H, W, shift, rounds = g[f"{tag}_meta"].tolist()
    counts = g[f"{tag}_counts"]
    base = O.exclusive_scan(counts)
    a = F.BucketAssignment(np.zeros(n, np.int64), np.zeros(n, np.int64), counts, base, S, K)
    table = O.bucket_table(counts, base, K, S)
    sched = F.build_schedule(len(table[0]), W, 1, shift, rounds)
    p = F.init_params(seed, d, n_heads=H)
    out = F.stage_forward(g[f"{tag}_feats"], g[f"{tag}_coords"], a, sched, p)
    assert rel(out, g[f"{tag}_out"]) < STAGE_TOL, rel(out, g[f"{tag}_out"])


def _config_a(n=4096, seed=7, d=96):
    coords = O.synth_cloud(seed, n, "uniform-box")
    vox = O.remap_nonnegative(O.voxelize(coords, (0, 0, 0), 1 / 64))
    a = F.assign_buckets(vox, None, F.HashConfig("zorder-div", K=40, S_div=6554), 128)
    feats = np.random.default_rng(1).normal(size=(n, d))
    sf, _ = F.scatter(feats, a)
    sc, _ = F.scatter(coords, a)
    return a, sf, sc


@pytest.mark.parametrize("d,H", [(96, 4), (384, 4), (48, 2)])
def test_stage_config_a_vs_oracle(d, H):
    a, sf, sc = _config_a(d=d)
    table = a.bucket_table()
    sched = F.build_schedule(len(table[0]), 2, 1, 1, 2)
    p = F.init_params(0, d, n_heads=H)
    out = F.stage_forward(sf, sc, a, sched, p)
    ref = O.stage_forward(sf, sc, table, O.build_schedule(len(table[0]), 2, 1, 1, 2),
                          O.init_params(0, d, n_heads=H), threads=8)
    assert rel(out, ref) < STAGE_TOL, rel(out, ref)


def test_stage_residual_identity_is_exact():
    a, sf, sc = _config_a(n=1024, d=12)
    sched = F.build_schedule(len(a.bucket_table()[0]), 2)
    p = F.init_params(1, 12, n_heads=2)
    p.w_v[:] = 0
    p.b_v[:] = 0
    p.w_out[:] = 0
    p.b_out[:] = 0
    out = F.stage_forward(sf, sc, a, sched, p)
    assert np.array_equal(out, sf)


def test_stage_cross_scope_flow_needs_second_round():
    """pkg/tests/test_stage.py:107-126 on the GPU: round 0 cannot leak across
    scopes (bit-identical rows), round 1 does."""
    sizes = [512, 512, 512, 512]
    n = sum(sizes)
    r = np.random.default_rng(3)
    counts = np.array(sizes + [0])
    base = O.exclusive_scan(counts)
    ids = np.repeat(np.arange(4), sizes)
    offs = np.concatenate([np.arange(s) for s in sizes])
    a = F.BucketAssignment(ids, offs, counts, base, 512, 4)
    feats = r.normal(size=(n, 12))
    coords = r.uniform(size=(n, 3))
    p = F.init_params(2, 12, n_heads=2)
    zeroed = feats.copy()
    zeroed[1024:1536] = 0.0
    one = F.build_schedule(4, 2, shift=1, rounds=1)
    np.testing.assert_array_equal(F.stage_forward(feats, coords, a, one, p)[512:1024],
                                  F.stage_forward(zeroed, coords, a, one, p)[512:1024])
    two = F.build_schedule(4, 2, shift=1, rounds=2)
    diff = np.linalg.norm(F.stage_forward(feats, coords, a, two, p)[512:1024]
                          - F.stage_forward(zeroed, coords, a, two, p)[512:1024])
    assert diff > 0


def test_stage_errors():
    a, sf, sc = _config_a(n=512, d=12)
    p = F.init_params(0, 12, n_heads=2)
    with pytest.raises(ConfigError):
        F.stage_forward(sf, sc, a, F.build_schedule(3, 2), p)      # wrong bucket count
    p64 = F.init_params(0, 64, n_heads=4)
    with pytest.raises(ConfigError):
        F.stage_forward(np.zeros((512, 64)), sc, a, F.build_schedule(len(a.bucket_table()[0]), 2), p64)


def test_layer_norm_and_gelu_f64():
    r = np.random.default_rng(4)
    x = r.normal(size=(50, 24))
    g, b = r.normal(size=24), r.normal(size=24)
    np.testing.assert_allclose(F.layer_norm(x, g, b), O.layer_norm(x, g, b), rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(F.gelu(x), O.gelu(x), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("d,H", [(96, 4), (512, 4), (64, 4)])
def test_attention_growing_max_rescales(d, H):
    """Logits that grow along the key order move every row's running max
    tile after tile (the kernel rescales O in TMEM only when the max grows
    by more than 2^8), over a 3000-row two-segment scope."""
    r = np.random.default_rng(d + H)
    m = 3000
    N = m + 64
    Q = r.normal(size=(N, d))
    Q[:, :] = np.abs(Q) * 0.5
    K = np.abs(r.normal(size=(N, d))) * np.linspace(0.0, 3.0, N)[:, None]
    V = r.normal(size=(N, d))
    ranges = [(0, 1700), (1764, 1764 + m - 1700)]
    out = F.tiled_attention(Q, K, V, F.AttentionParams(d, H), ranges=ranges)
    ref = O.attention_ranges(Q, K, V, H, ranges)
    assert np.isfinite(out).all()
    assert rel(out, ref) < 3e-2, rel(out, ref)


@pytest.mark.parametrize("n,k,ln,pe,ndev", [(3001, 96, True, False, None),
                                            (3001, 384, True, True, 2900),
                                            (4096, 384, False, False, None),
                                            (100_000, 96, True, True, 99_900),
                                            (257, 96, True, True, None)])
def test_gemm_res_ln_matches_torch(n, k, ln, pe, ndev):
    """f3d_gemm_res_ln (the opt-in O-projection / MLP-output epilogue):
    F += x W + b in place, y = LN(F) g + b (+PE) against torch fp32 on the same
    bf16 operands; rows past the device count are never written."""
    import ctypes

    import torch

    from paper_2412_16481_b200 import _lib as L
    d = 96
    g = torch.Generator(device="cuda").manual_seed(k + n)
    x = torch.randn((n, k), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((k, d), device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)
    bias = torch.randn((d,), device="cuda", generator=g) * 0.1
    F0 = torch.randn((n, d), device="cuda", generator=g)
    lg = 1 + 0.1 * torch.randn((d,), device="cuda", generator=g)
    lb = 0.1 * torch.randn((d,), device="cuda", generator=g)
    coords = torch.rand((n, 3), device="cuda", dtype=torch.float64, generator=g)
    lo_ext = torch.tensor([0, 0, 0, 1, 1, 1], device="cuda", dtype=torch.float64)
    Fg = F0.clone()
    xn = torch.full((n, d), 3.0, device="cuda", dtype=torch.bfloat16)
    nd = None if ndev is None else torch.tensor([ndev], dtype=torch.int32, device="cuda")
    wt = w.t().contiguous()
    assert L.load().f3d_gemm_res_ln_supported(k, d) == 1
    rc = L.load().f3d_gemm_res_ln(L.ptr(x), x.stride(0), n, k, L.ptr(wt), d, L.ptr(bias),
                                  L.ptr(Fg), Fg.stride(0), L.ptr(lg) if ln else None,
                                  L.ptr(lb) if ln else None, L.ptr(coords) if pe else None,
                                  L.ptr(lo_ext) if pe else None, ctypes.c_double(10000.0),
                                  ctypes.c_double(1e-12), L.ptr(xn), xn.stride(0), L.ptr(nd),
                                  L.stream())
    assert rc == 0
    torch.cuda.synchronize()
    m = n if ndev is None else ndev
    Fr = F0 + (x.float() @ w.float() + bias)
    assert float(((Fg[:m] - Fr[:m]).norm() / Fr[:m].norm()).item()) < 1e-4
    assert torch.equal(Fg[m:], F0[m:])
    if ln:
        xr = torch.nn.functional.layer_norm(Fr, (d,), lg, lb, eps=1e-12)
        if pe:
            xr = xr + torch.tensor(F.positional_encoding(coords.cpu().numpy(), d),
                                   device="cuda", dtype=torch.float32)
        got = xn[:m].float()
        assert float(((got - xr[:m]).norm() / xr[:m].norm()).item()) < 1e-2
    assert bool((xn[m:] == 3.0).all())
    if not ln:
        assert bool((xn == 3.0).all())


def test_stage_gemm_res_ln_matches_row_ln_path():
    """The stage with the fused residual + LN epilogue (opt-in) against the
    GEMM + f3d_row_ln two-kernel path (default)."""
    import torch

    from paper_2412_16481_b200 import stage as ST
    a, sf, sc = _config_a(n=3000, d=96)
    sched = F.build_schedule(len(a.bucket_table()[0]), 2, 1, 1, 2)
    p = F.init_params(0, 96, n_heads=4)
    X = torch.tensor(sf, dtype=torch.float32, device="cuda")
    C = torch.tensor(sc, device="cuda")
    old = ST.GEMM_RES_LN
    try:
        ST.GEMM_RES_LN = False
        ref = F.stage_forward(X, C, a, sched, p)
        ST.GEMM_RES_LN = True
        out = F.stage_forward(X, C, a, sched, p)
    finally:
        ST.GEMM_RES_LN = old
    rr = ((out.double() - ref.double()).norm() / ref.double().norm()).item()
    assert rr < 1e-2, rr
