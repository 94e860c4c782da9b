"""Golden text artifacts written by the REFERENCE's own writers
(bw/cli.py:29-78) for tests/test_artifacts*.py.  Build container only:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_artifacts_golden.py

Inputs: synth_cloud(7, 512, uniform-box), voxel 1/16, zorder-div K=8 S=128
S_div=512 (a config-A-shaped instance), features default_rng(3).normal((512, 6)).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

from bucketswin import bucketing, cli, geometry, hashing  # noqa: E402

OUT = os.path.join(HERE, "artifacts")

if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    cloud = geometry.synth_cloud(7, 512, "uniform-box")
    vox = hashing.remap_nonnegative(geometry.voxelize(cloud, geometry.VoxelGrid(1 / 16)))
    a = bucketing.assign_buckets(vox, None, hashing.HashConfig("zorder-div", K=8, S_div=512), 128)
    cli._write_assignment_csv(os.path.join(OUT, "assignment.csv"), a, "zorder-div")
    feats = np.random.default_rng(3).normal(size=(512, 6))
    cli._write_features_csv(os.path.join(OUT, "features.csv"), feats)
    cli._write_coords_csv(os.path.join(OUT, "coords.csv"), cloud.coords)
    print("wrote", sorted(os.listdir(OUT)))
