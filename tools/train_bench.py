"""Training-step throughput of one bucket-swin stage (SURVEY.md §8(d) config E:
B recipe scenes, 64 x 100K over 8 GPUs = 8 scenes per GPU).

    python tools/train_bench.py [--scenes 8] [--steps 3]
    torchrun --nproc-per-node N tools/train_bench.py   # scenes per rank fixed (weak)

Per rank: scenes synth_cloud(7 + 64*rank/8 + s, 100K) bucketed on the GPU with
the config-B stage-0 recipe (voxel 1/64, K=256 S=512 S_div=1024, W=2, 2 rounds,
C=96 H=4), scattered once (setup, untimed).  One timed step = for every scene
forward with saved activations + loss 0.5*mean(out^2) + backward, gradients
summed over the scenes, one flat NCCL all_reduce(SUM)/world, SGD on the
device fp32 masters with the bf16 operands re-cast in place.  CUDA-event time,
max over ranks.
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
from paper_2412_16481_b200.backbone import Backbone, StageConfig  # noqa: E402
from paper_2412_16481_b200.train import (DeviceWeights, StageTrainer, accumulate_grads,  # noqa: E402
                                         allreduce_grads)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenes", type=int, default=8)
    ap.add_argument("--points", type=int, default=100_000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--profile", action="store_true", help="print the top kernels of one step")
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = StageConfig(K=256, S=512, S_div=1024, W=2, d_model=96, pool_rho=0)
    bb = Backbone((cfg,))
    p = F.init_params(0, 96, n_heads=4)
    wts = DeviceWeights(p)
    trainers, feats = [], []
    for s in range(a.scenes):
        seed = 7 + rank * a.scenes + s
        C = torch.tensor(F.synth_cloud(seed, a.points, "uniform-box").coords, device="cuda")
        asg, _, _ = bb.bucketize(C, cfg)
        table = asg.bucket_table(split_recycle=True)
        sched = F.build_schedule(len(table[0]), cfg.W, cfg.stride, cfg.shift, cfg.rounds)
        X = torch.tensor(np.random.default_rng(seed).normal(size=(a.points, 96)),
                         dtype=torch.float32, device="cuda")
        Xs = F.scatter(X, asg)[0].contiguous()
        Cs = F.scatter(C, asg)[0].contiguous()
        trainers.append(StageTrainer(Cs, table, sched, p, a.points, weights=wts))
        feats.append(Xs)

    def step():
        acc, loss = None, 0.0
        for tr, X in zip(trainers, feats):
            out = tr.forward(X)
            loss = loss + 0.5 * (out * out).mean()
            _, g = tr.backward(out / out.numel())
            acc = accumulate_grads(acc, g)
        acc = allreduce_grads(acc)
        wts.sgd(acc, 1e-3)
        return loss

    for _ in range(a.warmup):
        step()
    if a.profile and rank == 0:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=70))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(device_ids=[local])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    losses = [step() for _ in range(a.steps)]
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / a.steps], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        pts = a.scenes * a.points * world
        print(json.dumps({"workload": "config E (stage-0 of the B recipe), fwd+bwd+allreduce+SGD",
                          "n_gpus": world, "scenes_per_gpu": a.scenes, "points_per_scene": a.points,
                          "ms_per_step": round(float(ms.item()), 3),
                          "train_points_per_s": pts / (float(ms.item()) * 1e-3),
                          "loss": [round(float(x), 5) for x in losses],
                          "max_mem_gb": round(torch.cuda.max_memory_allocated() / 2**30, 2)}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
