"""PSH / voxel-hash / pooling throughput at the SURVEY §8(d) sizes.

    python tools/psh_bench.py

Config B (100K), config D (1M, voxel 1/128, K=1280 S=1024) and config C
(16 x 200K multi-batch, K=512 S=512 S_div=512): CUDA-event time per launch,
algorithmic GB/s (36 B/point for hash + PSH; pooling (4d+24)(1+1/rho) B/pt)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_16481_b200 import _lib as L  # noqa: E402
from paper_2412_16481_b200.backbone import Backbone, StageConfig  # noqa: E402
from paper_2412_16481_b200.geometry import synth_cloud  # noqa: E402


def timed(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ms = []
    for _ in range(iters):
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        ms.append(ev[0].elapsed_time(ev[1]))
    return sorted(ms)[len(ms) // 2]


def single(name, n, cfg):
    C = torch.tensor(synth_cloud(7, n, "uniform-box").coords, device="cuda")
    bb = Backbone.__new__(Backbone)
    ms = timed(lambda: Backbone.bucketize(bb, C, cfg))
    with L.Probe(events=True) as pr:
        Backbone.bucketize(bb, C, cfg)
    parts = {k: round(v, 4) for k, v in pr.totals_ms().items()}
    return {"case": name, "n": n, "ms": round(ms, 4), "GB/s": round(36 * n / (ms * 1e-3) / 1e9, 1),
            "parts_ms": parts}


def multi(name, nscene, per, cfg):
    """16 scenes as one multi-batch PSH call (bucketing.assign_buckets with batch ids)."""
    import paper_2412_16481_b200 as F
    pts = np.concatenate([synth_cloud(100 + s, per, "uniform-box").coords for s in range(nscene)])
    bid = np.repeat(np.arange(nscene), per)
    C = torch.tensor(pts, device="cuda")
    B = torch.tensor(bid, device="cuda")
    grid = F.VoxelGrid(cfg.voxel)
    hc = F.HashConfig(cfg.kind, K=cfg.K, S_div=cfg.S_div)

    def run():
        vox = F.remap_nonnegative(F.voxelize(F.PointCloud(C, B), grid), B)
        return F.assign_buckets(vox, B, hc, cfg.S)
    ms = timed(run, 5)
    with L.Probe(events=True) as pr:
        run()
    parts = {k: round(v, 4) for k, v in pr.totals_ms().items()}
    n = nscene * per
    return {"case": name, "n": n, "ms": round(ms, 4), "GB/s": round(44 * n / (ms * 1e-3) / 1e9, 1),
            "note": "public API path (voxelize, remap, assign); 44 B/pt incl. batch id",
            "parts_ms": parts}


if __name__ == "__main__":
    torch.cuda.set_device(0)
    out = [single("config B 100K", 100_000, StageConfig(K=256, S=512, S_div=1024)),
           single("config D 1M", 1_000_000, StageConfig(voxel=1 / 128, K=1280, S=1024, S_div=1639)),
           multi("config C 16x200K", 16, 200_000, StageConfig(K=512, S=512, S_div=512))]
    for o in out:
        print(json.dumps(o))
