"""Backbone forward throughput on the other SURVEY §8(d) workloads.

    python tools/workload_bench.py --workload C   # 16 nuScenes-style scenes x 200K
    python tools/workload_bench.py --workload D   # one 1M-point scene, C=384, W=4
    torchrun --nproc-per-node N tools/workload_bench.py --workload C   # scenes sharded

Config C: synth_cloud(100+s, 200K, uniform-box), s = 0..15, K=512 S=512 S_div=512,
C=96 H=4 W=2, pool rho=2, then K=256 S=512 S_div=1024; the 16 scenes are dealt
round-robin over the ranks (fixed total work: strong scaling of the batch).
Config D: synth_cloud(7, 1M), voxel 1/128, K=1280 S=1024 S_div=1639, W=4 (scopes up
to 4096 rows), C=384 H=4 (dh=96), pool rho=2, then K=640 S=1024 S_div=3278.
Each scene is one CUDA-graph replay of the backbone with its inputs resident in
HBM; the per-rank time is CUDA-event timed and the max over ranks is reported.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2412_16481_b200.backbone import Backbone, StageConfig  # noqa: E402
from paper_2412_16481_b200.geometry import synth_cloud  # noqa: E402

WORKLOADS = {
    "C": dict(scenes=[(100 + s, 200_000) for s in range(16)], d=96,
              stages=(StageConfig(K=512, S=512, S_div=512, W=2, d_model=96, pool_rho=2, seed=0),
                      StageConfig(K=256, S=512, S_div=1024, W=2, d_model=96, pool_rho=0, seed=1))),
    "D": dict(scenes=[(7, 1_000_000)], d=384,
              stages=(StageConfig(voxel=1 / 128, K=1280, S=1024, S_div=1639, W=4, d_model=384,
                                  pool_rho=2, seed=0),
                      StageConfig(voxel=1 / 128, K=640, S=1024, S_div=3278, W=4, d_model=384,
                                  pool_rho=0, seed=1))),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C", choices=sorted(WORKLOADS))
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    W = WORKLOADS[a.workload]
    mine = [sc for i, sc in enumerate(W["scenes"]) if i % world == rank]
    bb = Backbone(W["stages"])
    inputs = []
    for seed, n in mine:
        c = torch.tensor(synth_cloud(seed, n, "uniform-box").coords, device="cuda")
        f = torch.tensor(np.random.default_rng(seed).normal(size=(n, W["d"])),
                         dtype=torch.bfloat16, device="cuda")
        inputs.append((c, f))
    n = mine[0][1]
    bb.capture(n, torch.bfloat16)
    rows = []
    for c, f in inputs:                                    # warm-up + per-scene check
        bb.graph_coords.copy_(c)
        bb.graph_feats.copy_(f)
        bb.replay()
        rows.append(bb.check_graph())
    times = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for c, f in inputs:
            bb.graph_coords.copy_(c)                       # device-resident inputs
            bb.graph_feats.copy_(f)
            bb.replay()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    bb.check_graph()
    t = torch.tensor([min(times)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total = sum(nn for _, nn in W["scenes"])
    if rank == 0:
        print(json.dumps({"workload": a.workload, "n_gpus": world, "scenes": len(W["scenes"]),
                          "points": total, "ms": round(float(t.item()), 3),
                          "points_per_s": total / (float(t.item()) * 1e-3),
                          "rows_out_rank0": rows[:4]}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
