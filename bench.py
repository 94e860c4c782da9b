#!/usr/bin/env python
"""Flash3D forward points/sec on B200 (BASELINE.json metric).

Default workload = BASELINE.json configs[1] / SURVEY.md §8(d) config B: a
ScanNet-sized synthetic scene (synth_cloud seed 7+rank, 100K points,
uniform-box) through the full 2-stage backbone forward (PSH -> scatter ->
2-round bucket-swin stage C=96 H=4 -> pool rho=2 -> PSH on the pooled
centroids -> stage), bf16 GEMM/attention operands, fp32 residual stream.
One step = one backbone forward of one scene per GPU (weak scaling: every
rank owns its own scene, no data-path collective; timing is max over ranks).
The ``config_c`` sub-object is BASELINE configs[2]: 16 scenes x 200K points
split contiguously over the ranks (strong scaling of the batch).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

``--gpus N`` without a torchrun environment re-launches this script under
``torch.distributed.run`` with N ranks (one process per GPU, NCCL).
``--impl reference`` times the reference's CPU implementation of the path
(the oracle port in oracle/: numpy float64 + the C claim loop, all host
threads) on rank 0, at the full config-B size, every step.
"""

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Flash3D forward points/sec at 1/2/4/8 B200; bucket-swin attn TFLOPS vs peak"
N_POINTS = 100_000
D_MODEL = 96
C_SCENES = [(100 + s, 200_000) for s in range(16)]      # config C
WORKLOAD = ("config B: 100K-point ScanNet-sized synthetic scene per GPU, full 2-stage backbone "
            "forward (PSH K=256 S=512 S_div=1024 -> 2-round bucket-swin stage C=96 H=4 W=2 -> "
            "pool rho=2 mean -> PSH K=128 S=512 S_div=2048 -> 2-round stage)")
DATA = ("synthetic (synth_cloud uniform-box seed 7+rank; features default_rng(1+rank).normal; "
        "random-init weights from init_params seeds 0/1)")


def bench_config(world):
    """The one config dict both arms print (same workload, same keys)."""
    return {"workload": WORKLOAD, "points_per_gpu": N_POINTS, "d_model": D_MODEL,
            "parallelism": f"scene-sharded x{world}",
            "l2": "GPU arm: L2 flushed (256 MiB write) between timed steps"}


def cpu_affinity():
    try:
        cpus = sorted(os.sched_getaffinity(0))
    except AttributeError:
        cpus = list(range(os.cpu_count() or 1))
    return cpus


def _cpu_ranges(cpus):
    out, i = [], 0
    while i < len(cpus):
        j = i
        while j + 1 < len(cpus) and cpus[j + 1] == cpus[j] + 1:
            j += 1
        out.append(f"{cpus[i]}-{cpus[j]}" if j > i else str(cpus[i]))
        i = j + 1
    return ",".join(out)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            j = json.load(fh)
        return j["hbm_gbs"], j["bf16_tflops"], "measured (MEASURED_PEAKS.json, burst)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def workload(rank):
    from paper_2412_16481_b200.geometry import synth_cloud   # bw/geometry.py:183-212 draws
    coords = synth_cloud(7 + rank, N_POINTS, "uniform-box").coords
    feats = np.random.default_rng(1 + rank).normal(size=(N_POINTS, D_MODEL))
    return coords, feats


class Clocks:
    """Clock / throttle sampling during the timed region (B200_PROFILING.md
    recipe): ONE `nvidia-smi -lms` process is started before the region and
    stopped after it, so no process is forked while steps are being timed."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, period_ms=50):
        self.index = index
        self.period_ms = period_ms
        self.rows = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", f"-lms={self.period_ms}"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)           # first sample lands before the timed region
        except Exception:
            self._p = None
        return self

    def __exit__(self, *exc):
        if self._p is None:
            return
        time.sleep(2 * self.period_ms / 1e3)
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except Exception:
            self._p.kill()
            out, _ = self._p.communicate()
        self.rows = [[x.strip() for x in ln.split(",")] for ln in out.splitlines() if ln.strip()]

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------- launcher

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(n):
    """One process per GPU: re-run this script under torch.distributed.run
    with n ranks on this node (rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def launcher_selftest(args, rank, world):
    """CPU check of the multi-rank plumbing (gloo): every rank times a fixed
    amount of host work, the step time is the max over ranks, and rank 0
    prints the line with the whole-job value, as the GPU arm does."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    x = np.random.default_rng(rank).random((256, 256))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x = np.tanh(x @ x.T / 256.0)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    t = torch.tensor([ms], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ranks = [None] * world
        dist.all_gather_object(ranks, {"rank": rank, "ms": ms, "pid": os.getpid()})
    else:
        ranks = [{"rank": 0, "ms": ms, "pid": os.getpid()}]
    if rank == 0:
        print(json.dumps({"metric": "launcher selftest", "n_gpus": world, "steps": args.steps,
                          "ms_per_step": float(t.item()), "value": world / float(t.item()),
                          "ranks": ranks}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------------- CPU legs

def cpu_forward(coords, feats, threads):
    """One full-size oracle backbone forward (every scope of every round).
    Returns (seconds, per-stage timings)."""
    from oracle import restated as O
    from paper_2412_16481_b200.backbone import scannet_backbone
    tm = []
    t0 = time.perf_counter()
    O.backbone_forward(coords, feats, scannet_backbone(), threads=threads, timings=tm)
    return time.perf_counter() - t0, tm


def cpu_baseline(coords, feats):
    threads = os.cpu_count() or 1
    sec, tm = cpu_forward(coords, feats, threads)
    cpus = cpu_affinity()
    return {"value": N_POINTS / sec, "unit": "points/s", "cores": threads, "kind": "port",
            "affinity": _cpu_ranges(cpus), "affinity_cpus": len(cpus),
            "sample": (f"one full-size config-B oracle backbone forward on the same 100K scene "
                       f"(all {sum(t['scopes'] for t in tm)} scopes, no extrapolation; "
                       f"{sec:.1f}s of CPU work, {threads} threads)")}


def run_reference(args, rank, world):
    if rank != 0:
        return
    coords, feats = workload(0)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_forward(coords, feats, threads)
    times = []
    for _ in range(args.steps):
        sec, tm = cpu_forward(coords, feats, threads)
        times.append(sec)
    ms = 1e3 * sum(times) / len(times)
    value = N_POINTS / (ms / 1e3)
    cpus = cpu_affinity()
    line = {"metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": DATA, "impl": "reference", "config": bench_config(world),
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads, "kind": "port",
                             "affinity": _cpu_ranges(cpus), "affinity_cpus": len(cpus),
                             "sample": ("every step is one full-size config-B backbone forward "
                                        "(oracle port: numpy float64 + C claim loop, attention "
                                        f"over all {sum(t['scopes'] for t in tm)} scopes, "
                                        f"{threads} threads); no sampling or extrapolation")},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU leg

def wide_attention_roofline(tflops_peak, iters=5):
    """Config D attention (BASELINE.json configs[3]): the
    1M-point synth_cloud(7) scene at voxel 1/128, PSH K=1280 S=1024
    S_div=1639, W=4 (scopes up to 4096 rows), C=512, H=4 (dh=128); random
    bf16 Q/K/V rows in the scattered layout, both rounds of the schedule.
    Algorithmic FLOPs = sum over scopes of 4 m^2 C; each launch reads
    ~3 GB of Q/K/V (> L2), so no flush is needed between launches."""
    import torch
    from paper_2412_16481_b200.attention import DeviceRoundPlan, attend, qstep_for
    from paper_2412_16481_b200.backbone import Backbone, StageConfig
    from paper_2412_16481_b200.geometry import synth_cloud
    n, d, H = 1_000_000, 512, 4
    cfg = StageConfig(voxel=1 / 128, K=1280, S=1024, S_div=1639, W=4, d_model=d, n_heads=H)
    C = torch.tensor(synth_cloud(7, n, "uniform-box").coords, device="cuda")
    asg, _, _ = Backbone.bucketize(Backbone.__new__(Backbone), C, cfg)
    nb_cap = cfg.K + -(-n // cfg.S)
    plans = [DeviceRoundPlan(asg._dev["counts"], asg._dev["base"], cfg.K, cfg.S, nb_cap, cfg.W,
                             cfg.stride, cfg.shift, t, n, qstep=qstep_for(d // H)) for t in range(2)]
    g = torch.Generator(device="cuda").manual_seed(0)
    qkv = torch.randn((n, 3 * d), device="cuda", generator=g).to(torch.bfloat16)
    q, k, v = (qkv[:, i * d:(i + 1) * d] for i in range(3))
    out = torch.empty((n, d), device="cuda", dtype=torch.bfloat16)
    flops = 0.0
    for p in plans:
        ln = p.scope_len.to(torch.float64)
        flops += 4.0 * float((ln * ln).sum().item()) * d
    for p in plans:
        attend(q, k, v, out, p, H, d // H)
    torch.cuda.synchronize()
    ms = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for p in plans:
            attend(q, k, v, out, p, H, d // H)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    best = statistics.median(ms)
    tf = flops / (best * 1e-3) / 1e12
    del qkv, out
    torch.cuda.empty_cache()
    return {"kernel": "f3d_bswin_attention_tc", "bound": "tensor", "achieved": round(tf, 1),
            "peak": tflops_peak, "unit": "TFLOP/s", "frac": round(tf / tflops_peak, 4),
            "traffic": None, "workload": "config D: 1M points, K=1280 S=1024 W=4, C=512 H=4 "
                                         "(dh=128), 2 rounds, bf16 operands, fp32 accumulate",
            "flops_per_step": flops, "ms_per_step": round(best, 3),
            "launches_per_step": len(plans)}


def _ncu_traffic():
    """DRAM bytes per attention launch from the committed ncu --set full capture
    (dram__bytes_read.sum + write.sum) next to the algorithmic bytes."""
    for name in ("r2_attn_ncu_traffic.json", "r1_attn_ncu_traffic.json"):
        p = os.path.join(ROOT, "profiles", name)
        try:
            with open(p) as fh:
                t = json.load(fh)
            return {"traffic": t["traffic_bytes_per_launch"],
                    "traffic_algorithmic": t["algorithmic_bytes_per_launch"],
                    "traffic_source": f"profiles/{name} (ncu --set full, per launch)"}
        except (OSError, KeyError, ValueError):
            continue
    return {"traffic": None}


# entry-point families timed alone (their recorded calls re-issued in one
# graph, in step order); each family holds its whole producer chain
FAMILIES = {
    "attention": ("f3d_bswin_attention_tc", "f3d_bswin_attention"),
    "psh": ("f3d_voxel_hash", "f3d_psh_assign"),
    "scatter": ("f3d_scatter_ln_pe", "f3d_scatter_rows", "f3d_scatter_rows_bf16_f32"),
    "pool_build": ("f3d_plan_pool", "f3d_pool_build"),
    "pool_reduce": ("f3d_pool_reduce", "f3d_pool_reduce_res"),
}


def family_times(calls, names, flush, reps=20):
    """Average time of one step's launches of the given entry points, re-issued
    alone as one CUDA graph on the current stream (CUDA events around each
    replay; the L2 is flushed before each replay when ``flush`` is given)."""
    import torch
    from paper_2412_16481_b200 import _lib as L
    sel = [c for c in calls if c[0] in names]
    if not sel:
        return None, 0
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        L.replay_calls(sel, L.stream())          # warm (lazy attributes) outside capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        L.replay_calls(sel, L.stream())
    ms = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return statistics.median(ms), len(sel)


def config_e(world, rank, local, scenes=8, steps=2):
    """BASELINE configs[4]: the training step (forward + fused attention
    backward + gradient all-reduce over the ranks + SGD) on 8 config-B scenes
    per GPU (64 over 8 GPUs); tools/train_bench.run.  Weak scaling."""
    from tools.train_bench import run
    r = run(scenes=scenes, points=N_POINTS, steps=steps, warmup=1, rank=rank, world=world,
            local=local)
    return {"value": r["train_points_per_s"], "unit": "training points/s", "scaling": "weak",
            "ms_per_step": r["ms_per_step"], "scenes_per_gpu": scenes, "n_gpus": world,
            "max_mem_gb": r["max_mem_gb"],
            "workload": ("config E: 8 ScanNet-sized scenes (100K points) per GPU through the "
                         "2-stage backbone, forward with saved activations + backward (fused "
                         "attention backward kernels, no m x m tiles) + one flat NCCL "
                         "all_reduce per stage + SGD, one CUDA graph per scene; CUDA events, "
                         "max over ranks")}


def config_c(world, rank, local, reps=3):
    """BASELINE configs[2]: 16 x 200K-point scenes (synth_cloud 100..115),
    K=512 S=512 S_div=512 then K=256 S_div=1024, C=96; scenes split
    contiguously over the ranks (shard.scenes_for_rank); every scene one graph
    replay with its inputs resident; max over ranks of the pass time."""
    import torch
    import torch.distributed as dist
    from paper_2412_16481_b200.backbone import Backbone, StageConfig
    from paper_2412_16481_b200.geometry import synth_cloud
    from paper_2412_16481_b200.shard import scenes_for_rank
    stages = (StageConfig(K=512, S=512, S_div=512, W=2, d_model=96, pool_rho=2, seed=0),
              StageConfig(K=256, S=512, S_div=1024, W=2, d_model=96, pool_rho=0, seed=1))
    mine = [C_SCENES[i] for i in scenes_for_rank(len(C_SCENES), world, rank)]
    bb = Backbone(stages)
    inputs = []
    for seed, n in mine:
        c = torch.tensor(synth_cloud(seed, n, "uniform-box").coords, device="cuda")
        f = torch.tensor(np.random.default_rng(seed).normal(size=(n, D_MODEL)),
                         dtype=torch.bfloat16, device="cuda")
        inputs.append((c, f))
    flush = torch.empty(64 * 2 ** 20, dtype=torch.int32, device="cuda")
    times = []
    if inputs:
        bb.capture(mine[0][1], torch.bfloat16)
        for c, f in inputs:                                # warm-up + per-scene check
            bb.graph_coords.copy_(c)
            bb.graph_feats.copy_(f)
            bb.replay()
            bb.check_graph()
    for _ in range(reps):
        flush.fill_(1)
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
    if inputs:
        bb.check_graph()
    t = torch.tensor([statistics.median(times)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total = sum(nn for _, nn in C_SCENES)
    ms = float(t.item())
    del bb, inputs, flush
    torch.cuda.empty_cache()
    return {"value": total / (ms * 1e-3), "unit": "points/s", "scaling": "strong",
            "ms_per_pass": round(ms, 3), "scenes": len(C_SCENES), "points": total,
            "scenes_per_rank": len(mine),
            "workload": ("config C: 16 nuScenes-style scenes x 200K points (synth_cloud 100..115 "
                         "uniform-box), K=512 S=512 S_div=512 -> pool rho=2 -> K=256 S_div=1024, "
                         "C=96 H=4 W=2; scenes split contiguously over the ranks; inputs resident, "
                         "L2 flushed before each pass; median of 3 passes, max over ranks")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip config C / config D / per-family timings")
    ap.add_argument("--launcher-selftest", action="store_true",
                    help="CPU/gloo check of the multi-rank launcher and the max-over-ranks timing")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.launcher_selftest:
        launcher_selftest(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    args.warmup = max(3, args.warmup)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2412_16481_b200 import _lib as L
    from paper_2412_16481_b200.backbone import Backbone

    coords, feats = workload(rank)
    dev = torch.device("cuda", local)
    C_d = torch.tensor(coords, device=dev)
    X_d = torch.tensor(feats, dtype=torch.float32, device=dev)
    C_h = torch.tensor(coords).pin_memory()
    X_h32 = torch.tensor(feats, dtype=torch.float32).pin_memory()    # fp32 features in
    flush = torch.empty(64 * 2 ** 20, dtype=torch.int32, device=dev)   # 256 MiB > 126 MB L2
    bb = Backbone()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def max_over_ranks(x):
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        bb.forward(C_d, X_d)
    f_eager, _ = bb.forward(C_d, X_d, keep_trace=True)
    trace = bb.last_trace

    # ---- device-resident throughput (value): the forward captured as CUDA
    # graphs (no host work inside a step), inputs resident in HBM, per-step
    # events, L2 flushed between steps.  The capture records every entry-point
    # call (for the launch count and the per-family timings below).
    with L.Recorder() as rec:
        bb.capture(N_POINTS, torch.float32)
    bb.graph_coords.copy_(C_d)
    bb.graph_feats.copy_(X_d)
    for _ in range(args.warmup):
        bb.replay()
    n_out = bb.check_graph()
    out_ref = bb._graphs["X"][:n_out].clone()
    graph_ok = bool(torch.equal(out_ref, f_eager))
    barrier()
    step_ms = []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            bb.replay()
            s1.record()
            torch.cuda.synchronize()
            step_ms.append(s0.elapsed_time(s1))
    bb.check_graph()
    barrier()
    ms_max = max_over_ranks(sum(step_ms) / len(step_ms))

    # ---- per-family kernel times: each family's recorded launches of one
    # step re-issued alone in a graph and event-timed (serialised, no host gaps)
    fam = {}
    for k, names in FAMILIES.items():
        t_ms, nl = family_times(rec.calls, names, flush)
        if t_ms is not None:
            fam[k] = {"ms_per_step": round(t_ms, 4), "calls": nl}
    # restore the step's state and check it is unchanged
    bb.replay()
    n_out2 = bb.check_graph()
    graph_ok = graph_ok and n_out2 == n_out and bool(torch.equal(bb._graphs["X"][:n_out], out_ref))

    # ---- end to end through the public API with host buffers (e2e)
    out_rows = []
    for _ in range(args.warmup):
        bb.forward_host(C_h, X_h32)
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        res, _ = bb.forward_host(C_h, X_h32)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
        out_rows.append(res.shape[0])
    e2e_single_ms = max_over_ranks(sum(e2e_ms) / len(e2e_ms))

    def pipelined(X_h):
        """Backbone.stream_host: the same per-step copies (inputs H2D from
        pinned host memory, last-stage features + status D2H) on their own
        streams, overlapping the neighbouring steps' compute; timed over all
        steps with events (start before the first upload, end after the last
        read-back), divided by the step count."""
        scenes = [(C_h, X_h)] * args.steps
        bb.stream_host([(C_h, X_h)] * max(2, args.warmup))
        rows_seen = []
        barrier()
        cs = torch.cuda.current_stream()
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        p0.record(cs)
        bb._h2d.wait_event(p0)
        bb.stream_host(scenes, on_result=lambda i, out, n_o: rows_seen.append(n_o))
        cs.wait_stream(bb._d2h)
        p1.record(cs)
        torch.cuda.synchronize()
        slot = bb._slots[0]
        d2h = int(slot["out_bf16"].numel() * 2 + slot["status"].numel() * slot["status"].element_size())
        return max_over_ranks(p0.elapsed_time(p1) / args.steps), rows_seen, d2h

    e2e_ms_max, rows_seen, d2h_bytes = pipelined(X_h32)
    X_h16 = torch.tensor(feats, dtype=torch.bfloat16).pin_memory()
    e2e16_ms, _, _ = pipelined(X_h16)

    # ---- the public host-array call (numpy float64 in, numpy float32 out)
    from paper_2412_16481_b200.backbone import backbone_forward
    for _ in range(2):
        backbone_forward(coords, feats)
    barrier()
    t0 = time.perf_counter()
    for _ in range(min(args.steps, 5)):
        backbone_forward(coords, feats)
    pub_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / min(args.steps, 5))

    cfg_c = cfg_e = None
    if not args.no_extras:
        from paper_2412_16481_b200 import backbone as BBm
        BBm._BACKBONES.clear()
        del bb
        torch.cuda.empty_cache()
        cfg_c = config_c(world, rank, local)
        cfg_e = config_e(world, rank, local)

    if rank == 0:
        hbm, tflops, src = peaks()
        steps = args.steps
        total_pts = N_POINTS * world
        n_tot = sum(s.n for s in trace)
        attn_flops = sum(s.attention_flops for s in trace)
        fa = fam.get("attention", {})
        attn_ms = fa.get("ms_per_step", 0.0)
        attn_tf = attn_flops / (attn_ms * 1e-3) / 1e12 if attn_ms else 0.0
        n_scores = attn_flops // (4 * (D_MODEL // 4))
        sm_mhz = clk.summary().get("sm_mhz") or 1965.0
        exp_ach = n_scores / (attn_ms * 1e-3) / 1e12 if attn_ms else 0.0
        exp_peak = 16 * 148 * sm_mhz * 1e6 / 1e12

        def bw(name, nbytes, note):
            t = fam.get(name, {}).get("ms_per_step")
            if not t:
                return None
            a = nbytes / (t * 1e-3) / 1e9
            return {"bound": "hbm", "achieved": round(a, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(a / hbm, 4), "ms_per_step": t, "bytes_per_step": int(nbytes),
                    "note": note}

        n0, n1 = trace[0].n, trace[1].n
        d = D_MODEL
        rooflines = {
            "psh": bw("psh", 36.0 * n_tot,
                      "f3d_voxel_hash + f3d_psh_assign, both stages; 36 B/point algorithmic "
                      "(24 B f64 coords in, int32 id/offset/dest out; SURVEY §8(d))"),
            "scatter": bw("scatter", (n0 + n1) * (4 * d + 4 + 24 + 4 * d + 2 * d)
                          + (n0 + n1) * (24 + 4 + 24),
                          "f3d_scatter_ln_pe (fp32 features, dest and the unscattered coords "
                          "in -> fp32 F + bf16 LN1(F)+PE out) + f3d_scatter_rows (24-B "
                          "coordinate rows + dest) of both stages"),
            "pool_reduce": bw("pool_reduce", n0 * (4 * d + 2 * d + 24) + n1 * (4 * d + 24),
                              "f3d_pool_reduce_res (fp32 F + bf16 y in, fp32 pooled out) + "
                              "f3d_pool_reduce of the f64 centroids; (6d+24) B/pt in + "
                              "(4d+24)/rho out"),
        }
        pb = fam.get("pool_build")
        if pb:
            rooflines["pool_build"] = {"bound": "latency", "ms_per_step": pb["ms_per_step"],
                                       "note": "sub-bucket partition (sequential step 3 per tile); "
                                               "per-tile latency-bound, no byte roofline"}
        line = {
            "metric": METRIC,
            "value": total_pts / (ms_max / 1e3),
            "unit": "points/s",
            "n_gpus": world,
            "steps": steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": DATA,
            "config": bench_config(world),
            "roofline": {"kernel": "f3d_bswin_attention_tc", "bound": "tensor",
                         "achieved": round(attn_tf, 2), "peak": tflops, "unit": "TFLOP/s",
                         "frac": round(attn_tf / tflops, 4), **_ncu_traffic(),
                         "peak_source": src, "flops_per_step": attn_flops,
                         "ms_per_step": attn_ms, "launches_per_step": fa.get("calls"),
                         "timing": "the step's attention launches re-issued alone as one CUDA "
                                   "graph, CUDA events around each replay, L2 flushed before",
                         "note": "dh=24 (padded 32): exp/MUFU-bound, see roofline_exp"},
            "roofline_exp": {"kernel": "f3d_bswin_attention_tc", "bound": "mufu",
                             "achieved": round(exp_ach, 3), "peak": round(exp_peak, 3),
                             "unit": "T exp/s", "frac": round(exp_ach / exp_peak, 4),
                             "scores_per_step": n_scores,
                             "note": "algorithmic scores (sum over scopes of m^2 x heads) / attention "
                                     "time vs 16 MUFU ex2 per clk per SM x 148 SMs at the sampled "
                                     "SM clock; part of the exponentials run on the FMA pipe, so "
                                     "frac can exceed the pure-MUFU share"},
            "rooflines": {k: v for k, v in rooflines.items() if v is not None},
            "kernel_ms_per_step": {k: v["ms_per_step"] for k, v in fam.items()},
            "psh_sweeps": [s.sweeps for s in trace],
            "gpu_launches": rec.launches(),
            "graph_matches_eager": graph_ok,
            "e2e": {"value": total_pts / (e2e_ms_max / 1e3), "unit": "points/s",
                    "h2d_bytes_per_step": int(C_h.numel() * 8 + X_h32.numel() * 4),
                    "d2h_bytes_per_step": d2h_bytes,
                    "io": "coords f64 + features fp32 in (pinned); last-stage features bf16 "
                          "(capacity rows) + status words out, every step",
                    "mode": "Backbone.stream_host: two CUDA-graph slots, uploads on an H2D stream "
                            "and read-backs on a D2H stream overlap the neighbouring steps' "
                            "compute; events around all steps / steps",
                    "ms_per_step": e2e_ms_max, "rows_out": rows_seen[-1] if rows_seen else None,
                    "bf16_features": {"value": total_pts / (e2e16_ms / 1e3),
                                      "ms_per_step": e2e16_ms,
                                      "h2d_bytes_per_step": int(C_h.numel() * 8 + X_h16.numel() * 2)},
                    "single_call": {"value": total_pts / (e2e_single_ms / 1e3),
                                    "ms_per_step": e2e_single_ms,
                                    "mode": "Backbone.forward_host per step, synchronous "
                                            "(feature upload overlapped with stage-0 PSH)"},
                    "public_call": {"value": total_pts / (pub_ms / 1e3), "ms_per_step": pub_ms,
                                    "mode": "backbone_forward(numpy f64 coords, numpy f64 feats) "
                                            "-> numpy f32, host wall clock (host casts, pageable "
                                            "copies and the read-back included)"}},
            "clocks": clk.summary(),
        }
        if cfg_c is not None:
            line["config_c"] = cfg_c
        if cfg_e is not None:
            line["config_e"] = cfg_e
        if not args.no_extras:
            line["roofline_wide"] = wide_attention_roofline(tflops)
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(coords, feats)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
