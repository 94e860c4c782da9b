"""Training-step throughput (B recipe scenes, 64 x 100K
over 8 GPUs = 8 scenes per GPU) of the 2-stage config-B backbone
(stage 0 -> mean pool rho=2 -> re-bucketed stage 1), or of stage 0 alone
with --stage0-only.

    python tools/train_bench.py [--scenes 8] [--steps 3]
    torchrun --nproc-per-node N tools/train_bench.py   # scenes per rank fixed (weak)

Per rank: scenes synth_cloud(7 + 8*rank + s, 100K) with the config-B recipe
(stage 0: voxel 1/64, K=256 S=512 S_div=1024, W=2, 2 rounds, C=96 H=4, pool
rho=2; stage 1: K=128 S=512 S_div=2048); per-scene layouts (PSH, scatter maps,
pooling partition, scope plans) are built once (setup, untimed).  One timed
step = for every scene forward with saved activations + loss 0.5*mean(out^2) +
backward, gradients summed over the scenes, one flat NCCL all_reduce(SUM)/world
per stage, SGD on the device fp32 masters with the bf16 operands re-cast in
place.  CUDA-event time, max over ranks.
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

import paper_2412_16481_b200 as F  # noqa: E402
from paper_2412_16481_b200.backbone import StageConfig, scannet_backbone  # noqa: E402
from paper_2412_16481_b200.train import (BackboneTrainer, DeviceWeights,  # noqa: E402
                                         accumulate_grads, allreduce_grads)


def run(scenes=8, points=100_000, steps=3, warmup=1, graph=True, stage0_only=False,
        profile=False, rank=0, world=1, local=0):
    """Config E training throughput on this rank (its process group, if any,
    is already initialised).  Returns the result dict (whole-job points/s,
    max over ranks of the step time)."""
    if stage0_only:
        stages = (StageConfig(K=256, S=512, S_div=1024, W=2, d_model=96, pool_rho=0),)
    else:
        stages = scannet_backbone()
    params = [F.init_params(s.seed, s.d_model, n_heads=s.n_heads) for s in stages]
    wts = [DeviceWeights(p) for p in params]
    trainers, feats = [], []
    for s in range(scenes):
        seed = 7 + rank * scenes + s
        C = torch.tensor(F.synth_cloud(seed, points, "uniform-box").coords, device="cuda")
        X = torch.tensor(np.random.default_rng(seed).normal(size=(points, 96)),
                         dtype=torch.float32, device="cuda")
        trainers.append(BackboneTrainer(C, stages, params, weights=wts))
        feats.append(X)

    def scene_step(tr, X):
        out = tr.forward(X)
        loss = 0.5 * (out * out).mean()
        _, gs = tr.backward(out / out.numel())
        return loss, gs

    graphs = None
    if graph:
        # static per-scene graphs: inputs/weights are resident, the grads and
        # loss are the graph's static outputs (allocations from the graph pool)
        graphs = []
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for tr, X in zip(trainers, feats):
                scene_step(tr, X)                       # warm-up on the side stream
        torch.cuda.current_stream().wait_stream(side)
        for tr, X in zip(trainers, feats):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                loss, gs = scene_step(tr, X)
            graphs.append((g, loss, gs))

    def step():
        acc, loss = [None] * len(stages), 0.0
        if graphs is not None:
            for g, l, gs in graphs:
                g.replay()
                loss = loss + l
                acc = [accumulate_grads(x, gg) for x, gg in zip(acc, gs)]
        else:
            for tr, X in zip(trainers, feats):
                l, gs = scene_step(tr, X)
                loss = loss + l
                acc = [accumulate_grads(x, g) for x, g in zip(acc, gs)]
        for w, g in zip(wts, acc):
            w.sgd(allreduce_grads(g), 1e-3)
        return loss

    for _ in range(warmup):
        step()
    if profile and rank == 0:
        from torch.profiler import ProfilerActivity, profile as tprofile
        torch.cuda.synchronize()
        with tprofile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30,
                                        max_name_column_width=70))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(device_ids=[local])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    losses = [step() for _ in range(steps)]
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / steps], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    pts = scenes * points * world
    res = {"workload": ("config E, stage 0 only" if stage0_only else
                        "config E, 2-stage B-recipe backbone") +
                       ": fwd+bwd+allreduce+SGD" + (" (CUDA graph per scene)" if graph else ""),
           "n_gpus": world, "scenes_per_gpu": scenes, "points_per_scene": points,
           "ms_per_step": round(float(ms.item()), 3),
           "train_points_per_s": pts / (float(ms.item()) * 1e-3),
           "loss": [round(float(x), 5) for x in losses],
           "max_mem_gb": round(torch.cuda.max_memory_allocated() / 2**30, 2)}
    del graphs, trainers, feats
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenes", type=int, default=8)
    ap.add_argument("--points", type=int, default=100_000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--profile", action="store_true", help="print the top kernels of one step")
    ap.add_argument("--stage0-only", action="store_true")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="eager per-scene steps instead of one CUDA graph per scene")
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    res = run(a.scenes, a.points, a.steps, a.warmup, a.graph, a.stage0_only, a.profile, rank,
              world, local)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
