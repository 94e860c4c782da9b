"""Small driver for compute-sanitizer (tools/sanitize.sh): one call of each
hot kernel family at config-A-like sizes -- PSH (single batch, multi-batch,
forced exact fallback, large-K warp path, fused coordinates path), pooling
build + reduce, tcgen05 attention, the stage GEMMs -- through the public API."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_16481_b200 as F  # noqa: E402
from paper_2412_16481_b200 import bucketing as FB  # noqa: E402
from paper_2412_16481_b200.backbone import Backbone, StageConfig  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
r = np.random.default_rng(0)
coords = F.synth_cloud(7, 4096, "uniform-box").coords
vox = F.remap_nonnegative(F.voxelize(F.PointCloud(coords), F.VoxelGrid(1 / 64)))
cfg = F.HashConfig("zorder-div", K=40, S_div=6554)
if which in ("all", "psh"):
    a = F.assign_buckets(vox, None, cfg, 128)
    b = np.sort(r.integers(0, 3, size=len(vox)))
    F.assign_buckets(vox, b, cfg, 128)
    FB._assign(np.tile(np.array([5, 9, 14]), (300, 1)), None, F.HashConfig("zorder-mod", K=256), 16,
               None, max_sweeps=1)
    F.assign_buckets(r.integers(0, 30, size=(2000, 3)), r.integers(0, 2, size=2000),
                     F.HashConfig("zorder-mod", K=13000), 2)
if which in ("all", "pool"):
    a = F.assign_buckets(vox, None, cfg, 128)
    sc, _ = F.scatter(coords, a)
    sf, _ = F.scatter(r.normal(size=(len(coords), 96)), a)
    F.pool_stage(sf, sc, a, 2, "mean")
if which in ("all", "backbone"):
    stages = (StageConfig(K=40, S=128, S_div=6554, W=2, d_model=96, pool_rho=2, seed=0),
              StageConfig(K=20, S=128, S_div=13108, W=2, d_model=96, pool_rho=0, seed=1))
    bb = Backbone(stages)
    C = torch.tensor(coords, device="cuda")
    X = torch.tensor(r.normal(size=(len(coords), 96)), dtype=torch.float32, device="cuda")
    bb.forward(C, X)
torch.cuda.synchronize()
print("sanitize drive ok:", which)
