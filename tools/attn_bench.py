"""Attention-only timing on the SURVEY §8(d) scenes (one bucket-swin round).

    python tools/attn_bench.py [--config B|D] [--d 512] [--heads 4] [--iters 20]

Config B: synth_cloud(7, 100K) K=256 S=512 W=2; config D: synth_cloud(7, 1M)
voxel 1/128 K=1280 S=1024 W=4.  Q/K/V are random bf16 rows in the scattered
layout; the plan comes from the PSH counts exactly as in the backbone.
Reports algorithmic TFLOP/s (sum over scopes of 4 m^2 d) per launch, timed
with CUDA events on the launching stream.  Under ncu, wrap with
--profile-from-start off (the timed loop sits inside cudaProfilerStart/Stop).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2412_16481_b200.geometry import synth_cloud  # noqa: E402
from paper_2412_16481_b200.attention import DeviceRoundPlan, attend, qstep_for  # noqa: E402
from paper_2412_16481_b200.backbone import Backbone, StageConfig  # noqa: E402

CONFIGS = {
    "B": dict(n=100_000, cfg=StageConfig(K=256, S=512, S_div=1024, W=2, d_model=96)),
    "D": dict(n=1_000_000, cfg=StageConfig(voxel=1 / 128, K=1280, S=1024, S_div=1639, W=4,
                                           d_model=512)),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="B")
    ap.add_argument("--d", type=int, default=0)
    ap.add_argument("--heads", type=int, default=4)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--round", type=int, default=1)
    ap.add_argument("--stats", action="store_true")
    a = ap.parse_args()
    spec = CONFIGS[a.config]
    cfg = spec["cfg"]
    d = a.d or cfg.d_model
    n = spec["n"]
    torch.cuda.set_device(0)
    C = torch.tensor(synth_cloud(7, n, "uniform-box").coords, device="cuda")
    bb = Backbone.__new__(Backbone)
    asg, _, _ = Backbone.bucketize(bb, C, cfg)
    counts_h = asg._dev["counts"].cpu().numpy()
    nb = cfg.K + -(-int(counts_h[cfg.K]) // cfg.S)
    dh = d // a.heads
    plan = DeviceRoundPlan(asg._dev["counts"], asg._dev["base"], cfg.K, cfg.S, nb, cfg.W,
                           cfg.stride, cfg.shift, a.round, n, qstep=qstep_for(dh))
    g = torch.Generator(device="cuda").manual_seed(0)
    qkv = torch.randn((n, 3 * d), device="cuda", generator=g).to(torch.bfloat16)
    q, k, v = (qkv[:, i * d:(i + 1) * d] for i in range(3))
    out = torch.empty((n, d), device="cuda", dtype=torch.bfloat16)
    lens = plan.scope_len.to(torch.float64)
    flops = 4.0 * float((lens * lens).sum().item()) * d
    for _ in range(3):
        attend(q, k, v, out, plan, a.heads, dh)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.iters)]
    for i in range(a.iters):
        ev[2 * i].record()
        attend(q, k, v, out, plan, a.heads, dh)
        ev[2 * i + 1].record()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ms = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(a.iters))
    med = ms[len(ms) // 2]
    res = {"config": a.config, "n": n, "d": d, "heads": a.heads, "dh": dh, "W": cfg.W, "S": cfg.S,
           "gflop": flops / 1e9, "ms_median": med, "ms_min": ms[0],
           "tflops_median": flops / (med * 1e-3) / 1e12, "tflops_best": flops / (ms[0] * 1e-3) / 1e12,
           "mean_scope_rows": float(lens[lens > 0].mean().item())}
    if a.stats:   # Q tiles per scope / items by live Q tiles (NQ = qstep // 128)
        qs = qstep_for(dh)
        L_ = plan.scope_len[plan.scope_len > 0].cpu().long()
        tiles = (L_ + 127) // 128
        res["tiles_hist"] = {int(t): int((tiles == t).sum()) for t in tiles.unique()}
        nq = qs // 128
        last = tiles - (tiles - 1) // nq * nq
        res["items"] = int(((tiles + nq - 1) // nq).sum())
        res["last_item_nq_hist"] = {int(t): int((last == t).sum()) for t in last.unique()}
        res["len_pctl"] = [int(x) for x in torch.quantile(L_.double(), torch.tensor(
            [0.0, 0.1, 0.5, 0.9, 1.0], dtype=torch.float64)).tolist()]
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
