"""GPU: the fused voxelize + remap + hash + PSH launch (f3d_psh_assign_coords)
returns exactly what the separate launches (f3d_voxel_hash + f3d_psh_assign)
and the oracle return: bucket ids, offsets, counts, bases, destinations,
sweep counts and the 7 range words (bw/geometry.py:69-72,
bw/hashing.py:60-149, bw/bucketing.py:275-320)."""

import numpy as np
import pytest
import torch

from oracle import restated as O

pytestmark = pytest.mark.gpu

from paper_2412_16481_b200 import _lib as L  # noqa: E402
from paper_2412_16481_b200 import backbone as B  # noqa: E402
from paper_2412_16481_b200.backbone import Backbone, StageConfig  # noqa: E402
from paper_2412_16481_b200.bucketing import default_probe_schedule  # noqa: E402
from paper_2412_16481_b200.hashing import HashConfig  # noqa: E402

CASES = [
    ("uniform-box", 100_000, StageConfig(K=256, S=512, S_div=1024)),
    ("surface-shell", 100_000, StageConfig(K=256, S=512, S_div=1024)),
    ("gaussian-clusters", 200_000, StageConfig(K=512, S=512, S_div=512)),
    ("uniform-box", 1_000_000, StageConfig(voxel=1 / 128, K=1280, S=1024, S_div=1639)),
    ("surface-shell", 50_000, StageConfig(K=128, S=512, S_div=2048, kind="xor-mod")),
    ("uniform-box", 4096, StageConfig(K=40, S=128, S_div=6554)),
    ("uniform-box", 1, StageConfig(K=8, S=16, S_div=64)),
    ("gaussian-clusters", 7, StageConfig(K=3, S=2, S_div=64, kind="xor-div")),
]


def _both(C, cfg, n_cap=None, n_dev=None):
    bb = Backbone.__new__(Backbone)
    out = []
    old = B.FUSED_PSH
    try:
        for fused in (True, False):
            B.FUSED_PSH = fused
            a, stats, info = bb.bucketize(C, cfg, n_cap, n_dev)
            d = a._dev
            out.append({k: d[k].clone() for k in ("id", "off", "counts", "base", "dest")}
                       | {"stats": stats.clone(), "info": info.clone()})
    finally:
        B.FUSED_PSH = old
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("dist,n,cfg", CASES)
def test_fused_psh_equals_separate_launches_and_oracle(dist, n, cfg):
    coords = O.synth_cloud(7, n, dist)
    C = torch.tensor(coords, device="cuda")
    f, s = _both(C, cfg)
    for k in ("id", "off", "counts", "base", "dest", "stats"):
        assert torch.equal(f[k], s[k]), k
    assert torch.equal(f["info"][:3], s["info"][:3])
    vox = O.remap_nonnegative(O.voxelize(coords, (0, 0, 0), cfg.voxel))
    ids, offs, counts, base = O.psh_assign(vox, None, cfg.kind, cfg.K, cfg.S, cfg.S_div)
    np.testing.assert_array_equal(f["id"].cpu().numpy(), ids)
    np.testing.assert_array_equal(f["off"].cpu().numpy(), offs)
    np.testing.assert_array_equal(f["counts"].cpu().numpy(), counts)
    np.testing.assert_array_equal(f["base"].cpu().numpy(), base)


def test_fused_psh_device_row_count():
    coords = O.synth_cloud(3, 60_000, "surface-shell")
    C = torch.tensor(coords, device="cuda")
    nd = torch.tensor([41_234], dtype=torch.int32, device="cuda")
    cfg = StageConfig(K=128, S=512, S_div=2048)
    f, s = _both(C, cfg, 60_000, nd)
    for k in ("counts", "base", "stats"):
        assert torch.equal(f[k], s[k]), k
    for k in ("id", "off", "dest"):
        assert torch.equal(f[k][:41_234], s[k][:41_234]), k
    vox = O.remap_nonnegative(O.voxelize(coords[:41_234], (0, 0, 0), cfg.voxel))
    ids, offs, _, _ = O.psh_assign(vox, None, cfg.kind, cfg.K, cfg.S, cfg.S_div)
    np.testing.assert_array_equal(f["id"][:41_234].cpu().numpy(), ids)


def test_fused_psh_range_words():
    """Coordinates beyond 2^bits voxels: the same range words (and thus the
    same RangeError) as the separate launches."""
    coords = O.synth_cloud(5, 20_000, "uniform-box") * 40.0
    C = torch.tensor(coords, device="cuda")
    f, s = _both(C, StageConfig(K=64, S=512, S_div=4096))
    assert torch.equal(f["stats"], s["stats"])
    assert int(f["stats"][3]) >= 1024


def _coords_call(coords, cfg, max_sweeps):
    n = coords.shape[0]
    hc = HashConfig(cfg.kind, K=cfg.K, S_div=cfg.S_div)
    table, P = default_probe_schedule().device_table()
    t = {k: L.empty((m,), torch.int32) for k, m in
         (("id", n), ("off", n), ("counts", cfg.K + 1), ("base", cfg.K + 1), ("dest", n),
          ("info", 4))}
    stats = L.empty((7,), torch.int64)
    wsb = L.load().f3d_psh_coords_workspace_size(n, cfg.K)
    ws = L.empty((wsb,), torch.uint8)
    org = (L._F64 * 3)(0.0, 0.0, 0.0)
    L.call("f3d_psh_assign_coords", L.ptr(coords), n, org, float(cfg.voxel), hc.kind_code,
           cfg.K, cfg.S, cfg.S_div, hc.bits_per_axis, 0, table.ctypes.data_as(L._P), P,
           max_sweeps, L.ptr(t["id"]), L.ptr(t["off"]), L.ptr(t["counts"]), L.ptr(t["base"]),
           L.ptr(t["dest"]), L.ptr(t["info"]), L.ptr(stats), L.ptr(ws), wsb, None, L.stream())
    torch.cuda.synchronize()
    return t


@pytest.mark.parametrize("max_sweeps", [1, 2, 3, 128])
def test_fused_psh_sweep_cap_fallback_is_exact(max_sweeps):
    """Past max_sweeps the kernel finishes with the exact sequential path."""
    coords = O.synth_cloud(11, 30_000, "surface-shell")
    cfg = StageConfig(K=64, S=256, S_div=4096)
    t = _coords_call(torch.tensor(coords, device="cuda"), cfg, max_sweeps)
    vox = O.remap_nonnegative(O.voxelize(coords, (0, 0, 0), cfg.voxel))
    ids, offs, counts, _ = O.psh_assign(vox, None, cfg.kind, cfg.K, cfg.S, cfg.S_div)
    np.testing.assert_array_equal(t["id"].cpu().numpy(), ids)
    np.testing.assert_array_equal(t["off"].cpu().numpy(), offs)
    np.testing.assert_array_equal(t["counts"].cpu().numpy(), counts)
    if max_sweeps < 3:
        assert int(t["info"][1]) == 1          # the sequential fallback ran
