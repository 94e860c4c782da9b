"""Localise the g0-under-g1 corruption (stream_host with F3D_PSH_GATE=0):
two graph slots; for each step i, g1 of step i (compute stream) and g0 of
step i+1 (side stream) run concurrently, then the host syncs and compares
every stage's PSH outputs, stats, pooled coordinates and the final features
of step i with a serial reference of the same scene.
    python tools/g0_overlap_probe.py [steps] [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import restated as O  # noqa: E402
from paper_2412_16481_b200.backbone import Backbone, StageConfig  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000
stages = (StageConfig(K=64, S=512, S_div=4096, pool_rho=2, seed=0),
          StageConfig(K=32, S=512, S_div=8192, pool_rho=0, seed=1))
scenes = [(torch.tensor(O.synth_cloud(s, n, "uniform-box"), device="cuda"),
           torch.tensor(np.random.default_rng(s).normal(size=(n, 96)), dtype=torch.bfloat16,
                        device="cuda")) for s in (3, 4, 5)]
bb = Backbone(stages)
slots = [bb._capture_slot(n, torch.bfloat16) for _ in range(2)]


def snapshot(sl):
    """Real rows only (stage buffers are sized for the capacity; rows past
    the device count hold whatever an earlier scene left there)."""
    out = {}
    m = None
    for si, r in enumerate(sl["runs"]):
        m = r.n_cap if r.n_dev is None else int(r.n_dev.item())
        out[f"s{si}.id"] = r.asg._dev["id"][:m].clone()
        out[f"s{si}.dest"] = r.asg._dev["dest"][:m].clone()
        out[f"s{si}.counts"] = r.asg._dev["counts"].clone()
        out[f"s{si}.stats"] = r.stats.clone()
        out[f"s{si}.info"] = r.info.clone()
        out[f"s{si}.Cs"] = r.Cs[:m].clone()
    out["status"] = sl["status"].clone()
    out["X"] = sl["out_bf16"][:m].clone()
    return out


# serial references, slot 0
refs = []
for C, X in scenes:
    sl = slots[0]
    sl["coords"].copy_(C)
    sl["feats"].copy_(X)
    sl["g0"].replay()
    sl["g1"].replay()
    torch.cuda.synchronize()
    refs.append(snapshot(sl))
side = torch.cuda.Stream()
comp = torch.cuda.current_stream()
sl = slots[0]
sl["coords"].copy_(scenes[0][0])
sl["feats"].copy_(scenes[0][1])
sl["g0"].replay()
torch.cuda.synchronize()
bad = 0
for i in range(steps):
    a, b = slots[i % 2], slots[(i + 1) % 2]
    nc, nx = scenes[(i + 1) % 3]
    b["coords"].copy_(nc)
    b["feats"].copy_(nx)
    torch.cuda.synchronize()
    side.wait_stream(comp)
    a["g1"].replay()                      # step i on the compute stream
    with torch.cuda.stream(side):
        b["g0"].replay()                  # step i+1's g0 concurrently
    torch.cuda.synchronize()
    got, ref = snapshot(a), refs[i % 3]
    diff = [k for k in ref if not torch.equal(got[k], ref[k])]
    if diff:
        bad += 1
        print("step", i, "differs in", diff, flush=True)
print("g0 overlap probe:", steps, "steps,", bad, "with differences")
