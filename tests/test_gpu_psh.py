"""GPU parity for voxelize / remap / hash / PSH / validate / scatter against
the golden fixtures (reference output) and the CPU oracle.  Bit-exact."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle import restated as O

pytestmark = pytest.mark.gpu

import paper_2412_16481_b200 as F  # noqa: E402
from paper_2412_16481_b200 import bucketing as FB  # noqa: E402
from paper_2412_16481_b200.errors import (ConfigError, EmptyInputError,  # noqa: E402
                                          IntegrityError, RangeError)

KINDS = ("xor-mod", "xor-div", "zorder-mod", "zorder-div")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a), dtype=np.int64).tobytes()).hexdigest()


def recipes():
    with open(os.path.join(GOLDEN, "recipes.json")) as fh:
        return json.load(fh)


# ------------------------------------------------------------------ hashing

def test_hashing_golden():
    g = load_golden("hashing.npz")
    np.testing.assert_array_equal(F.morton_encode(g["vox"], 10), g["morton10"])
    np.testing.assert_array_equal(F.morton_encode(g["vox21"], 21), g["morton21"])
    for kind in KINDS:
        for K, S_div in ((16, 4), (256, 1024), (40, 6554), (1280, 1639), (7, 1)):
            got = F.hash_bucket(g["vox"], F.HashConfig(kind, K=K, S_div=S_div))
            np.testing.assert_array_equal(got, g[f"{kind}_{K}_{S_div}"], err_msg=kind)
    np.testing.assert_array_equal(F.remap_nonnegative(g["remap_in"], g["remap_batch"]), g["remap_out"])
    np.testing.assert_array_equal(F.remap_nonnegative(g["remap_in"]), g["remap_out_nobatch"])
    np.testing.assert_array_equal(F.voxelize(F.PointCloud(g["voxA_coords"]), F.VoxelGrid(1 / 64)), g["voxA"])
    np.testing.assert_array_equal(
        F.voxelize(F.PointCloud(g["vox_gc_coords"]), F.VoxelGrid(0.037, origin=(0.1, -0.2, 0.3))),
        g["vox_gc"])


def test_hashing_kats_and_errors():
    assert F.morton_encode((1, 2, 3), bits_per_axis=2) == 53
    assert F.morton_encode((0, 0, 0)) == 0
    top = (1 << 21) - 1
    assert F.morton_encode((top, top, top), bits_per_axis=21) == 2 ** 63 - 1
    assert F.hash_bucket((5, 3, 6), F.HashConfig("xor-mod", K=4)) == 0
    for bad, axis in (((-1, 0, 0), "x"), ((0, -2, 0), "y"), ((0, 0, -9), "z"),
                      ((1024, 0, 0), "x"), ((0, 1024, 0), "y"), ((0, 0, 1024), "z")):
        with pytest.raises(RangeError, match=axis):
            F.morton_encode(bad, bits_per_axis=10)
    # wrap vs error on div overflow (pkg/tests/test_hashing.py:112-129)
    v = np.array([[2047, 0, 0]])
    assert F.hash_bucket(v, F.HashConfig("xor-div", K=16, S_div=1, bits_per_axis=11))[0] == 2047 % 16
    with pytest.raises(RangeError):
        F.hash_bucket(v, F.HashConfig("xor-div", K=16, S_div=1, bits_per_axis=11, div_overflow="error"))
    with pytest.raises(ConfigError):
        F.HashConfig("nope", K=4)


# ---------------------------------------------------------------------- PSH

@pytest.mark.parametrize("case", recipes()["cases"], ids=lambda c: c["name"])
def test_psh_golden_cases(case):
    g = load_golden("psh.npz")
    nm = case["name"]
    vox = g[f"{nm}__vox"].astype(np.int64)
    batch = g[f"{nm}__batch"].astype(np.int64) if case["batched"] else None
    cfg = F.HashConfig(case["kind"], K=case["K"], S_div=case["S_div"],
                       div_overflow="error" if case["strict"] else "wrap")
    probes = F.default_probe_schedule(seed=case["seed"], max_probes=case["max_probes"])
    a = F.assign_buckets(vox, batch, cfg, case["S"], probes=probes)
    np.testing.assert_array_equal(a.bucket_id, g[f"{nm}__id"])
    np.testing.assert_array_equal(a.bucket_offset, g[f"{nm}__off"])
    np.testing.assert_array_equal(a.counts, g[f"{nm}__counts"])
    a.validate()


@pytest.mark.parametrize("name", ["A", "B_uniform", "B_shell", "C_uniform", "C_clusters", "D"])
def test_psh_recipe_digests(name):
    rc = recipes()["recipes"][name]
    coords, batch = [], []
    for b, s in enumerate(rc["seeds"]):
        c = O.synth_cloud(s, rc["n"], rc["dist"])
        coords.append(c)
        batch.append(np.full(len(c), b))
    coords = np.vstack(coords)
    multi = len(rc["seeds"]) > 1
    batch = np.concatenate(batch) if multi else None
    vox = F.remap_nonnegative(F.voxelize(F.PointCloud(coords, batch), F.VoxelGrid(rc["voxel"])), batch)
    assert sha(vox) == rc["vox_sha"]
    a = F.assign_buckets(vox, batch, F.HashConfig("zorder-div", K=rc["K"], S_div=rc["S_div"]), rc["S"])
    assert sha(a.bucket_id) == rc["id_sha"]
    assert sha(a.bucket_offset) == rc["off_sha"]
    assert a.counts.tolist() == rc["counts"]
    assert sha(a.dest_index()) == rc["dest_sha"]


def test_psh_random_vs_oracle():
    """Acceptance-suite style instances (pkg/tests/test_acceptance.py:27-76)."""
    r = np.random.default_rng(20240502)
    for i in range(120):
        n = 200_000 if i == 0 else int(r.integers(1, 15_001))
        side = int(r.choice((4, 8, 16, 32, 64)))
        vox = r.integers(0, side, size=(n, 3))
        if i % 3 == 1:
            vox[r.random(n) < 0.4] = r.integers(0, side, size=3)
        kind = KINDS[i % 4]
        S = (16, 32, 512, 1, 4)[(i // 4) % 5]
        K = (64, 256, 3, 1000)[(i // 12) % 4]
        S_div = int(r.choice((8, 64, 1024)))
        batch = None
        if i % 5 == 2 and n >= 3:
            batch = r.integers(0, 3, size=n)
            batch[:3] = [0, 1, 2]
        cfg = F.HashConfig(kind, K=K, S_div=S_div)
        a = F.assign_buckets(vox, batch, cfg, S)
        ids, offs, counts, _ = O.psh_assign(vox, batch, kind, K, S, S_div)
        np.testing.assert_array_equal(a.bucket_id, ids, err_msg=f"instance {i}")
        np.testing.assert_array_equal(a.bucket_offset, offs, err_msg=f"instance {i}")
        np.testing.assert_array_equal(a.counts, counts, err_msg=f"instance {i}")
        dest = a.dest_index()
        assert np.array_equal(np.sort(dest), np.arange(n))


def test_psh_hotspot_and_kats():
    vox = np.tile(np.array([5, 9, 14]), (1000, 1))
    a = F.assign_buckets(vox, None, F.HashConfig("zorder-mod", K=256), S=16)
    assert a.recycle_fraction() == 0.488
    a = F.assign_buckets(np.zeros((3, 3), np.int64), None, F.HashConfig("xor-mod", K=2), S=2)
    assert a.bucket_id.tolist() == [0, 0, 1] and a.bucket_offset.tolist() == [0, 1, 0]
    vox = np.zeros((4, 3), dtype=np.int64)
    a = F.assign_buckets(vox, np.array([0, 0, 1, 1]), F.HashConfig("xor-mod", K=2), S=4)
    d = a.dest_index()
    assert set(d[:2]) == {0, 1} and set(d[2:]) == {2, 3}
    a = F.assign_buckets(np.zeros((40, 3), np.int64), None, F.HashConfig("xor-mod", K=1), S=4)
    assert a.counts[0] == 4 and a.counts[1] == 36


def test_psh_sweep_cap_fallback_is_exact():
    """Force the in-kernel sequential fallback (max_sweeps=1) on a hotspot."""
    vox = np.tile(np.array([5, 9, 14]), (1000, 1))
    cfg = F.HashConfig("zorder-mod", K=256)
    a = FB._assign(vox, None, cfg, 16, None, max_sweeps=1)
    assert int(a._dev["info"][1]) == 1
    ids, offs, counts, _ = O.psh_assign(vox, None, "zorder-mod", 256, 16)
    np.testing.assert_array_equal(a.bucket_id, ids)
    np.testing.assert_array_equal(a.bucket_offset, offs)


def test_psh_large_k_sequential_path():
    r = np.random.default_rng(5)
    vox = r.integers(0, 64, size=(3000, 3))
    a = F.assign_buckets(vox, None, F.HashConfig("zorder-mod", K=20000), S=1)
    ids, offs, counts, _ = O.psh_assign(vox, None, "zorder-mod", 20000, 1)
    np.testing.assert_array_equal(a.bucket_id, ids)
    np.testing.assert_array_equal(a.bucket_offset, offs)


def test_psh_warp_exact_fallback_is_fast_and_exact():
    """Past max_sweeps (here 1) the exact path is one warp per batch over
    32-point windows: a 4-batch shell-like instance
    with heavy recycling finishes in milliseconds and equals the oracle."""
    import time
    import torch
    r = np.random.default_rng(11)
    n = 200_000
    vox = r.integers(0, 24, size=(n, 3))          # dense: many full buckets, recycling
    batch = np.sort(r.integers(0, 4, size=n))
    cfg = F.HashConfig("zorder-div", K=512, S_div=64)
    FB._assign(vox[:4000], batch[:4000] * 0, cfg, 64, None, max_sweeps=1)   # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a = FB._assign(vox, batch, cfg, 64, None, max_sweeps=1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    assert int(a._dev["info"][1]) == 1
    ids, offs, counts, base = O.psh_assign(vox, batch, "zorder-div", 512, 64, S_div=64)
    np.testing.assert_array_equal(a.bucket_id, ids)
    np.testing.assert_array_equal(a.bucket_offset, offs)
    np.testing.assert_array_equal(a.counts, counts)
    assert (counts.reshape(4, -1)[:, -1] > 0).all()   # recycling happened
    assert dt < 2.0, dt


def test_psh_large_k_multibatch_exact():
    """K + 1 beyond the shared-memory histogram: one warp per batch over the
    original order (unsorted batch ids), then the base / dest pass."""
    r = np.random.default_rng(6)
    n = 50_000
    vox = r.integers(0, 40, size=(n, 3))
    batch = r.integers(0, 3, size=n)
    cfg = F.HashConfig("zorder-mod", K=20000)
    a = F.assign_buckets(vox, batch, cfg, S=2)
    ids, offs, counts, base = O.psh_assign(vox, batch, "zorder-mod", 20000, 2)
    np.testing.assert_array_equal(a.bucket_id, ids)
    np.testing.assert_array_equal(a.bucket_offset, offs)
    np.testing.assert_array_equal(a.counts, counts)
    np.testing.assert_array_equal(a.dest_index(), base[batch * 20001 + ids] + offs)


def test_two_stage_equals_one_stage():
    r = np.random.default_rng(777)
    for i in range(10):
        vox = r.integers(0, 40, size=(int(r.integers(200, 5001)), 3))
        cfg = F.HashConfig(KINDS[i % 4], K=64, S_div=64)
        one = F.assign_buckets(vox, None, cfg, 16)
        two = F.assign_buckets_two_stage(vox, None, cfg, 16, block_size=64, threads=2)
        np.testing.assert_array_equal(one.bucket_id, two.bucket_id)
        np.testing.assert_array_equal(one.bucket_offset, two.bucket_offset)
    with pytest.raises(ConfigError):
        F.assign_buckets_two_stage(vox, None, cfg, 16, block_size=0)


def test_psh_errors():
    cfg = F.HashConfig("xor-mod", K=4)
    with pytest.raises(RangeError):
        F.assign_buckets(np.array([[0, -1, 0]]), None, cfg, S=4)
    with pytest.raises(ConfigError):
        F.assign_buckets(np.zeros((3, 2), np.int64), None, cfg, S=4)
    with pytest.raises(ConfigError):
        F.assign_buckets(np.zeros((3, 3), np.int64), None, cfg, S=0)
    with pytest.raises(EmptyInputError):
        F.assign_buckets(np.zeros((0, 3), np.int64), None, cfg, S=4)
    with pytest.raises(ConfigError):
        F.assign_buckets(np.zeros((3, 3), np.int64), np.array([0, 2, 2]), cfg, S=4)
    with pytest.raises(ConfigError):
        F.assign_buckets(np.zeros((3, 3), np.int64), None, cfg, S=4, trace=[])


def test_validate_catches_corruption(rng):
    vox = rng.integers(0, 16, size=(200, 3))
    a = F.assign_buckets(vox, None, F.HashConfig("xor-mod", K=8), S=64)
    a.validate()
    c = F.BucketAssignment(a.bucket_id, a.bucket_offset, a.counts.copy(), a.bucket_base, a.S, a.K)
    c.counts[0] += 1
    with pytest.raises(IntegrityError, match="sum"):
        c.validate()
    d = F.BucketAssignment(a.bucket_id, a.bucket_offset, a.counts, a.bucket_base.copy(), a.S, a.K)
    d.bucket_base[2] += 1
    with pytest.raises(IntegrityError, match="prefix"):
        d.validate()
    b = F.BucketAssignment(a.bucket_id.copy(), a.bucket_offset.copy(), a.counts, a.bucket_base, a.S, a.K)
    i, j = np.flatnonzero(b.bucket_id == b.bucket_id[0])[:2]
    b.bucket_offset[i] = b.bucket_offset[j]
    with pytest.raises(IntegrityError, match="bijection"):
        b.validate()


# ------------------------------------------------------------------ scatter

def test_scatter_kats_and_roundtrip(rng):
    vox = np.array([[1, 0, 0], [0, 0, 0]], dtype=np.int64)
    a = F.assign_buckets(vox, None, F.HashConfig("xor-mod", K=2), S=1)
    out, perm = F.scatter(np.array([[10.0], [20.0]]), a)
    np.testing.assert_array_equal(perm, [1, 0])
    np.testing.assert_array_equal(out, [[20.0], [10.0]])
    vox = rng.integers(0, 20, size=(3000, 3))
    a = F.assign_buckets(vox, None, F.HashConfig("zorder-mod", K=8), S=512)
    for dt, d in ((np.float64, 5), (np.float32, 64), (np.float32, 3), (np.int64, 3)):
        feats = rng.normal(size=(3000, d)).astype(dt)
        out, perm = F.scatter(feats, a)
        np.testing.assert_array_equal(out[perm], feats)
        np.testing.assert_array_equal(F.gather(out, a), feats)
    ids_in_layout = np.empty(3000, dtype=np.int64)
    ids_in_layout[perm] = a.bucket_id
    assert (np.diff(ids_in_layout) >= 0).all()


def test_device_tensors_stay_on_device():
    import torch
    vox = torch.randint(0, 30, (5000, 3), device="cuda")
    a = F.assign_buckets(vox, None, F.HashConfig("zorder-div", K=32, S_div=64), 256)
    assert a.bucket_id.is_cuda and a.counts.is_cuda
    ids, offs, counts, _ = O.psh_assign(vox.cpu().numpy(), None, "zorder-div", 32, 256, 64)
    np.testing.assert_array_equal(a.bucket_id.cpu().numpy(), ids)
    f = torch.randn(5000, 96, device="cuda", dtype=torch.bfloat16)
    s, perm = F.scatter(f, a)
    assert s.is_cuda and torch.equal(s[perm], f)


def _boundary_cloud(vs, org, n=60_000, seed=0):
    """Coordinates on and next to voxel boundaries: c = o + k*vs, and the
    neighbouring doubles, so (c - o) / vs rounds onto or next to an integer."""
    r = np.random.default_rng(seed)
    k = r.integers(-3000, 3000, size=(n, 3)).astype(np.float64)
    c = np.asarray(org)[None, :] + k * vs
    step = r.integers(-2, 3, size=(n, 3))
    for s in (-2, -1, 1, 2):
        m = step == s
        c[m] = np.nextafter(c[m], np.inf if s > 0 else -np.inf)
        if abs(s) == 2:
            c[m] = np.nextafter(c[m], np.inf if s > 0 else -np.inf)
    c[::7] = r.uniform(-60, 60, size=c[::7].shape)          # plus generic points
    return c


@pytest.mark.parametrize("vs,org", [(1 / 128, (0.0, 0.0, 0.0)), (0.02, (0.1, -0.3, 7.25)),
                                    (0.05, (0.0, 0.0, 0.0)), (1 / 3, (1e-3, 2.0, -5.0)),
                                    (0.1, (-12.7, 3.3, 0.0))])
def test_voxelize_boundaries_exact(vs, org):
    """floor((c - o) / vs) with numpy's rounded division, exactly, where the
    quotient lands on or next to an integer (the kernels multiply by the
    reciprocal and fall back to the IEEE division near integers): the plain
    voxelize and the fused voxel-hash pass (remapped voxels)."""
    import torch
    from paper_2412_16481_b200 import _lib as L
    c = _boundary_cloud(vs, org, seed=int(vs * 1e4))
    want = np.floor((c - np.asarray(org)[None, :]) / vs).astype(np.int64)
    got = F.voxelize(F.PointCloud(c), F.VoxelGrid(vs, org))
    np.testing.assert_array_equal(got, want)
    n = c.shape[0]
    cd = torch.tensor(c, device="cuda")
    vox32 = torch.empty((n, 3), dtype=torch.int32, device="cuda")
    home = torch.empty(n, dtype=torch.int32, device="cuda")
    stats = torch.empty(8, dtype=torch.int64, device="cuda")
    ws = torch.empty(8, dtype=torch.int64, device="cuda")
    o3 = (L._F64 * 3)(*org)
    L.call("f3d_voxel_hash", L.ptr(cd), None, n, 1, o3, float(vs), 3, 256, 1024, 21,
           L.ptr(vox32), L.ptr(home), L.ptr(stats), L.ptr(ws), None, L.stream())
    np.testing.assert_array_equal(vox32.cpu().numpy().astype(np.int64), want - want.min(axis=0))
