"""Stress: two cooperative PSH launches in flight at once on two streams
(different scenes), repeated; every result must equal the same launch run
alone.  Used to root-cause the concurrent-g0 corruption."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import restated as O
from paper_2412_16481_b200.backbone import Backbone, StageConfig

cfgs = [StageConfig(K=256, S=512, S_div=1024), StageConfig(K=128, S=512, S_div=2048)]
bb = Backbone.__new__(Backbone)
scenes = [torch.tensor(O.synth_cloud(s, n, d), device="cuda")
          for s, n, d in ((7, 100_000, "uniform-box"), (8, 50_000, "surface-shell"))]
ref = []
for C, cfg in zip(scenes, cfgs):
    a, st, info = bb.bucketize(C, cfg)
    torch.cuda.synchronize()
    ref.append((a._dev["id"].clone(), a._dev["off"].clone(), a._dev["dest"].clone(), info.clone()))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
bad = 0
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for it in range(iters):
    outs = []
    for C, cfg, s in zip(scenes, cfgs, (s1, s2)):
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            outs.append(bb.bucketize(C, cfg))
    torch.cuda.synchronize()
    for (a, st, info), r in zip(outs, ref):
        ok = (torch.equal(a._dev["id"], r[0]) and torch.equal(a._dev["off"], r[1])
              and torch.equal(a._dev["dest"], r[2]) and torch.equal(info, r[3]))
        if not ok:
            bad += 1
            print("MISMATCH it", it, "info", info.tolist(), "ref", r[3].tolist(), flush=True)
print("psh concurrency:", iters, "iterations,", bad, "mismatches")
