"""GPU parity for in-bucket pooling: sub-bucket partitions bit-exact against the
reference golden fixtures and the oracle; pooled float64 features/centroids
exact (sequential index-order reduction)."""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import restated as O

pytestmark = pytest.mark.gpu

import paper_2412_16481_b200 as F  # noqa: E402
from paper_2412_16481_b200.errors import ConfigError, EmptyInputError  # noqa: E402


def test_subbuckets_golden():
    g = load_golden("pooling.npz")
    for i in range(30):
        sub = F.build_subbuckets(g[f"t{i}_coords"], int(g[f"t{i}_rho"]))
        np.testing.assert_array_equal(sub.subbucket_id, g[f"t{i}_sub"], err_msg=f"tile {i}")
        np.testing.assert_array_equal(sub.seeds, g[f"t{i}_seeds"], err_msg=f"tile {i}")
        sub.validate()


def test_subbuckets_random_vs_oracle():
    r = np.random.default_rng(31)
    for i in range(200):
        m = int(r.integers(1, 1025))
        rho = int(r.choice((1, 2, 3, 4, 7, 8, 16)))
        scale = float(r.choice((1e-3, 1.0, 50.0)))
        c = r.uniform(0, scale, size=(m, 3))
        if i % 3 == 1:
            piles = r.uniform(0, scale, size=(max(1, m // 50), 3))
            c[: m // 2] = piles[r.integers(0, len(piles), size=m // 2)]
        if i % 5 == 2:
            c[:, 1] = 0.25   # a degenerate axis (extent 0)
        if i % 7 == 3:       # lattice: many exactly / nearly equal step-3 distances
            c = r.integers(0, 6, size=(m, 3)) * 0.1 * scale
        sub = F.build_subbuckets(c, rho)
        osub, osizes, oseeds = O.subbuckets(c, rho)
        np.testing.assert_array_equal(sub.subbucket_id, osub, err_msg=f"case {i}")
        np.testing.assert_array_equal(sub.sizes, osizes, err_msg=f"case {i}")
        assert sub.num_subbuckets == math.ceil(m / rho)


def test_subbucket_kats():
    sub = F.build_subbuckets(np.full((4, 3), 0.5), rho=2)
    assert sub.num_subbuckets == 2 and sorted(sub.sizes.tolist()) == [2, 2]
    sub = F.build_subbuckets(np.random.default_rng(0).uniform(size=(5, 3)), rho=2)
    assert sorted(sub.sizes.tolist()) == [1, 2, 2]
    with pytest.raises(EmptyInputError):
        F.build_subbuckets(np.zeros((0, 3)), 2)
    with pytest.raises(ConfigError):
        F.build_subbuckets(np.zeros((1025, 3)), 2)


def test_pool_stage_golden():
    g = load_golden("pooling.npz")
    counts = g["ps_counts"]
    base = O.exclusive_scan(counts)
    a = F.BucketAssignment(np.zeros(len(g["ps_feats"]), np.int64), np.zeros(len(g["ps_feats"]), np.int64),
                           counts, base, 1500, 8)
    for rho, red in ((3, "sum"), (2, "mean"), (4, "max"), (5, "min")):
        pf, pc, na = F.pool_stage(g["ps_feats"], g["ps_coords"], a, rho, red)
        np.testing.assert_array_equal(na.counts, g[f"ps_{rho}_{red}_counts"])
        assert na.S == int(g[f"ps_{rho}_{red}_S"])
        np.testing.assert_array_equal(pc, g[f"ps_{rho}_{red}_coords"])
        np.testing.assert_array_equal(pf, g[f"ps_{rho}_{red}_feats"])
        na.validate()


def test_pool_stage_config_b_vs_oracle():
    coords = O.synth_cloud(7, 100_000, "surface-shell")
    vox = O.remap_nonnegative(O.voxelize(coords, (0, 0, 0), 1 / 64))
    a = F.assign_buckets(vox, None, F.HashConfig("zorder-div", K=256, S_div=1024), 512)
    feats = np.random.default_rng(1).normal(size=(100_000, 8))
    sf, _ = F.scatter(feats, a)
    sc, _ = F.scatter(coords, a)
    pf, pc, na = F.pool_stage(sf, sc, a, 2, "mean")
    of, oc, onc, oS, _ = O.pool_stage(sf, sc, a.counts, a.bucket_base, 256, 512, 1, 2, "mean")
    np.testing.assert_array_equal(na.counts, onc)
    np.testing.assert_array_equal(pc, oc)
    np.testing.assert_array_equal(pf, of)


def test_pool_features_matches_oracle_and_bf16_path():
    import torch
    r = np.random.default_rng(5)
    c = r.uniform(size=(700, 3))
    x = r.normal(size=(700, 16))
    sub = F.build_subbuckets(c, 3)
    for red in ("sum", "mean", "min", "max"):
        got = F.pool_features(x, sub, red)
        ref = O.pool_reduce(x, np.asarray(sub.subbucket_id), np.asarray(sub.sizes), red)
        np.testing.assert_array_equal(got, ref)
    xb = torch.tensor(x, device="cuda", dtype=torch.bfloat16)
    got = F.pool_features(xb, sub, "mean")
    ref = O.pool_reduce(xb.float().cpu().numpy(), np.asarray(sub.subbucket_id), np.asarray(sub.sizes), "mean")
    np.testing.assert_allclose(got.float().cpu().numpy(), ref, rtol=1e-2, atol=1e-2)


def test_pool_stage_map_and_unpool_vs_oracle():
    """parent[i] names the pooled row of scattered row i (tile-local sub id +
    first pooled row of its tile, oracle-side); unpool gathers by it."""
    coords = O.synth_cloud(9, 6000, "uniform-box")
    vox = O.remap_nonnegative(O.voxelize(coords, (0, 0, 0), 1 / 32))
    K, S = 24, 512
    ids, offs, counts, base = O.psh_assign(vox, None, "zorder-div", K, S, 2048)
    a = F.assign_buckets(vox, None, F.HashConfig("zorder-div", K=K, S_div=2048), S)
    dest = O.dest_index(ids, offs, base, K)
    Cs = np.empty_like(coords)
    Cs[dest] = coords
    feats = np.random.default_rng(2).normal(size=(6000, 8))
    Fs = np.empty_like(feats)
    Fs[dest] = feats
    pf, pc, na, parent = F.pool_stage_map(Fs, Cs, a, 2, "mean")
    of, oc, onc, _, sub_all = O.pool_stage(Fs, Cs, counts, base, K, S, 1, 2)
    # oracle parent: pooled rows are laid out slot by slot, tile by tile
    opar = np.empty(len(Fs), dtype=np.int64)
    out0 = 0
    for slot in range(K + 1):
        st, cnt = int(base[slot]), int(counts[slot])
        for t0 in range(0, cnt, 1024):
            lo, hi = st + t0, st + min(t0 + 1024, cnt)
            opar[lo:hi] = out0 + sub_all[lo:hi]
            out0 += int(sub_all[lo:hi].max()) + 1
    np.testing.assert_array_equal(parent, opar)
    np.testing.assert_array_equal(pc, oc)
    up = F.unpool(pc, parent)
    np.testing.assert_array_equal(up, oc[opar])
    with pytest.raises(ConfigError):
        F.unpool(pc, np.array([len(pc)]))


@pytest.mark.parametrize("rho", [2, 8, 11, 64])
@pytest.mark.parametrize("reduce", ["sum", "mean", "min", "max"])
def test_pool_features_fp32_vector_path_bit_exact(rho, reduce):
    """fp32 rows with d % 4 == 0 take the float4 reduce kernel; per column it
    must reproduce numpy's float32 add.reduceat order (and min/max/mean) bit
    for bit."""
    import torch
    r = np.random.default_rng(rho)
    m = 1000
    c = r.uniform(size=(m, 3))
    x = r.normal(size=(m, 96)).astype(np.float32)
    sub = F.build_subbuckets(c, rho)
    got = F.pool_features(torch.tensor(x, device="cuda"), sub, reduce).cpu().numpy()
    sid, sizes = np.asarray(sub.subbucket_id), np.asarray(sub.sizes)
    order = np.argsort(sid, kind="stable")
    bounds = np.r_[0, np.cumsum(sizes)[:-1]]
    g = x[order]
    if reduce in ("sum", "mean"):
        ref = np.add.reduceat(g, bounds, axis=0)
        if reduce == "mean":
            ref = ref / sizes[:, None].astype(np.float32)
    elif reduce == "min":
        ref = np.minimum.reduceat(g, bounds, axis=0)
    else:
        ref = np.maximum.reduceat(g, bounds, axis=0)
    assert got.dtype == np.float32
    np.testing.assert_array_equal(got, ref.astype(np.float32))
