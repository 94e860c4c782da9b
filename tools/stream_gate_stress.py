"""Stress of the pipelined host path (Backbone.stream_host) with step i+1's
coordinate-only graph g0 concurrent with step i's g1 -- the configuration that
corrupted results in round 1 when ungated (F3D_PSH_GATE=0 removes the gate).
Every step is compared with the synchronous single call.
    python tools/stream_gate_stress.py [steps] [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import restated as O  # noqa: E402
from paper_2412_16481_b200 import backbone as B  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 24
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
scenes = []
for s in range(6):
    c = torch.tensor(O.synth_cloud(30 + s, n, ("uniform-box", "surface-shell")[s % 2])).pin_memory()
    f = torch.tensor(np.random.default_rng(s).normal(size=(n, 96)),
                     dtype=torch.bfloat16).pin_memory()
    scenes.append((c, f))
seq = [scenes[i % len(scenes)] for i in range(steps)]
single = B.Backbone(B.scannet_backbone())
refs = [single.forward_host(c, f)[0].clone() for c, f in scenes]
bb = B.Backbone(B.scannet_backbone())
bad = []
bb.stream_host(seq, on_result=lambda i, out, n_out: None if torch.equal(out, refs[i % len(scenes)])
               else bad.append(i))
print("stream_host stress: gate", B.PSH_GATE, "steps", steps, "mismatching steps", bad)
