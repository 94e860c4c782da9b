"""GPU: device planners equal the host planners; the full backbone forward
matches the oracle composition (layouts bit-exact, features within the stage
tolerance)."""

import numpy as np
import pytest
import torch

from oracle import restated as O

pytestmark = pytest.mark.gpu

from paper_2412_16481_b200 import attention as A  # noqa: E402
from paper_2412_16481_b200.backbone import (Backbone, StageConfig,  # noqa: E402
                                            scannet_backbone, split_table)
from paper_2412_16481_b200.pooling import DeviceTilePlan, TilePlan  # noqa: E402


@pytest.mark.parametrize("seed", range(8))
def test_device_round_plan_equals_host(seed):
    r = np.random.default_rng(seed)
    K, S = int(r.integers(2, 400)), int(r.choice((64, 128, 512)))
    counts = r.integers(0, S + 1, size=K + 1)
    counts[K] = int(r.integers(0, 3 * S))
    base = O.exclusive_scan(counts)
    n = int(counts.sum())
    starts, lens = split_table(counts, base, K, S)
    nb = len(starts)
    W = int(r.integers(1, min(6, nb) + 1))
    stride = int(r.integers(1, 4))
    shift = int(r.integers(0, W))
    cd = torch.tensor(counts, dtype=torch.int32, device="cuda")
    bd = torch.tensor(base, dtype=torch.int32, device="cuda")
    for t in range(3):
        dp = A.DeviceRoundPlan(cd, bd, K, S, nb, W, stride, shift, t, n)
        hp = A.plan_arrays(starts, lens, A.round_members(nb, W, stride, shift, t))
        live = dp.live.cpu().numpy()
        assert live[1] == len(hp["scope_order"])
        assert live[2] == hp["scope_len"].max()
        ns = len(hp["scope_len"])
        np.testing.assert_array_equal(dp.scope_len.cpu().numpy()[:ns], hp["scope_len"])
        np.testing.assert_array_equal(dp.scope_nseg.cpu().numpy()[:ns], hp["scope_nseg"])
        segs = dp.seg_start.cpu().numpy().reshape(-1, W)
        vsts = dp.seg_vstart.cpu().numpy().reshape(-1, W)
        for s in range(ns):
            a, b = hp["scope_seg"][s], hp["scope_seg"][s] + hp["scope_nseg"][s]
            np.testing.assert_array_equal(segs[s, :b - a], hp["seg_start"][a:b])
            np.testing.assert_array_equal(vsts[s, :b - a], hp["seg_vstart"][a:b])
        w = dp.work.cpu().numpy()[:live[0]]
        assert sorted(map(tuple, w)) == sorted(map(tuple, hp["work"]))


def test_device_tile_plan_equals_host():
    r = np.random.default_rng(3)
    counts = r.integers(0, 2600, size=300)
    base = O.exclusive_scan(counts)
    for rho in (1, 2, 3, 7):
        cd = torch.tensor(counts, dtype=torch.int32, device="cuda")
        bd = torch.tensor(base, dtype=torch.int32, device="cuda")
        dp = DeviceTilePlan(counts, cd, bd, rho)
        hp = TilePlan(counts, base, rho, "cuda")
        assert dp.ntiles == hp.ntiles and dp.npool == hp.npool
        for name in ("tile_start", "tile_m", "tile_out"):
            np.testing.assert_array_equal(getattr(dp, name).cpu().numpy()[:dp.ntiles],
                                          getattr(hp, name).cpu().numpy()[:hp.ntiles])
        assert dp.totals.cpu().tolist() == [dp.ntiles, dp.npool]


def test_backbone_matches_oracle_composition():
    n = 20_000
    coords = O.synth_cloud(11, n, "uniform-box")
    feats = np.random.default_rng(2).normal(size=(n, 96))
    stages = (StageConfig(K=64, S=512, S_div=4096, pool_rho=2, seed=0),
              StageConfig(K=32, S=512, S_div=8192, pool_rho=0, seed=1))
    bb = Backbone(stages)
    f, c = bb.forward(torch.tensor(coords, device="cuda"),
                      torch.tensor(feats, dtype=torch.float32, device="cuda"))
    of, oc = O.backbone_forward(coords, feats, stages, threads=8)
    np.testing.assert_array_equal(c.cpu().numpy(), oc)       # layouts + centroids exact
    fr = f.cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(fr - of) / np.linalg.norm(of)
    assert rel < 2e-2, rel


def test_scannet_backbone_runs_and_is_deterministic():
    import bench
    coords, feats = bench.workload(0)
    bb = Backbone(scannet_backbone())
    C = torch.tensor(coords, device="cuda")
    X = torch.tensor(feats, dtype=torch.float32, device="cuda")
    f1, c1 = bb.forward(C, X)
    f2, c2 = bb.forward(C, X)
    assert torch.equal(c1, c2) and torch.equal(f1, f2)
    assert torch.isfinite(f1).all()


def test_graph_replay_matches_eager_and_host_path():
    """The captured CUDA graphs (sync-free, device-side sizes) reproduce the
    eager forward bit for bit, through device inputs and the host e2e path."""
    n = 30_000
    coords = O.synth_cloud(5, n, "uniform-box")
    feats = np.random.default_rng(3).normal(size=(n, 96))
    stages = (StageConfig(K=96, S=512, S_div=2048, pool_rho=2, seed=0),
              StageConfig(K=48, S=512, S_div=4096, pool_rho=0, seed=1))
    bb = Backbone(stages)
    C = torch.tensor(coords, device="cuda")
    X = torch.tensor(feats, dtype=torch.bfloat16, device="cuda")
    f_e, c_e = bb.forward(C, X)
    f_g, c_g = bb.forward_graph(C, X)
    assert torch.equal(c_e, c_g) and torch.equal(f_e, f_g)
    out, n_out = bb.forward_host(torch.tensor(coords).pin_memory(), X.cpu().pin_memory())
    assert n_out == f_e.shape[0]
    assert torch.equal(out, f_e.to(torch.bfloat16).cpu())
    # a second scene through the same graphs (different pooled row count)
    coords2 = O.synth_cloud(6, n, "surface-shell")
    C2 = torch.tensor(coords2, device="cuda")
    f_e2, c_e2 = bb.forward(C2, X)
    f_g2, c_g2 = bb.forward_graph(C2, X)
    assert torch.equal(c_e2, c_g2) and torch.equal(f_e2, f_g2)


def test_stream_host_pipelined_matches_single_calls():
    """Two-slot pipelined host streaming returns each scene's features in
    order, equal to the synchronous host call, with errors checked per step."""
    n = 20_000
    stages = (StageConfig(K=64, S=512, S_div=4096, pool_rho=2, seed=0),
              StageConfig(K=32, S=512, S_div=8192, pool_rho=0, seed=1))
    bb = Backbone(stages)
    scenes = []
    for seed in (3, 4, 5):
        c = torch.tensor(O.synth_cloud(seed, n, "uniform-box")).pin_memory()
        f = torch.tensor(np.random.default_rng(seed).normal(size=(n, 96)),
                         dtype=torch.bfloat16).pin_memory()
        scenes.append((c, f))
    got = {}
    seq = scenes * 3                     # 9 steps: slot reuse + concurrent g0 under g1
    bb.stream_host(seq, on_result=lambda i, out, n_out: got.__setitem__(i, out.clone()))
    assert sorted(got) == list(range(len(seq)))
    single = Backbone(stages)
    for i, (c, f) in enumerate(seq):
        ref, n_ref = single.forward_host(c, f)
        assert got[i].shape[0] == n_ref and torch.equal(got[i], ref), i


def test_backbone_recycle_heavy_matches_oracle():
    """gaussian-clusters at a small K sends most points to the recycle bucket:
    scopes mix regular buckets and S-row recycle chunks, several segments
    each (cp.async fallback tiles); graph, eager and oracle agree."""
    n = 12_000
    coords = O.synth_cloud(21, n, "gaussian-clusters")
    feats = np.random.default_rng(4).normal(size=(n, 96))
    stages = (StageConfig(K=24, S=256, S_div=2048, W=2, stride=2, shift=1, pool_rho=2, seed=0),
              StageConfig(K=12, S=256, S_div=4096, W=2, pool_rho=0, seed=1))
    bb = Backbone(stages)
    C = torch.tensor(coords, device="cuda")
    X = torch.tensor(feats, dtype=torch.float32, device="cuda")
    f, c = bb.forward(C, X)
    assert bb.last_trace == [] and f.shape[0] == c.shape[0]
    fg, cg = bb.forward_graph(C, X.to(torch.bfloat16))
    assert torch.equal(c, cg)
    of, oc = O.backbone_forward(coords, feats, stages, threads=8)
    np.testing.assert_array_equal(c.cpu().numpy(), oc)
    rel = np.linalg.norm(f.cpu().numpy().astype(np.float64) - of) / np.linalg.norm(of)
    assert rel < 2e-2, rel
    relg = np.linalg.norm(fg.cpu().numpy().astype(np.float64) - of) / np.linalg.norm(of)
    assert relg < 2e-2, relg


def test_stream_host_three_stage_backbone():
    """Three stages (two pooled levels, two side-branch PSH launches per step):
    the pipelined path with the next scene's g0 under g1 equals single calls."""
    n = 20_000
    stages = (StageConfig(K=64, S=512, S_div=4096, pool_rho=2, seed=0),
              StageConfig(K=32, S=512, S_div=8192, pool_rho=2, seed=1),
              StageConfig(K=16, S=512, S_div=16384, pool_rho=0, seed=2))
    bb = Backbone(stages)
    scenes = []
    for seed in (6, 7):
        c = torch.tensor(O.synth_cloud(seed, n, "uniform-box")).pin_memory()
        f = torch.tensor(np.random.default_rng(seed).normal(size=(n, 96)),
                         dtype=torch.bfloat16).pin_memory()
        scenes.append((c, f))
    seq = scenes * 3
    got = {}
    bb.stream_host(seq, on_result=lambda i, out, n_out: got.__setitem__(i, out.clone()))
    single = Backbone(stages)
    for i, (c, f) in enumerate(seq):
        ref, n_ref = single.forward_host(c, f)
        assert got[i].shape[0] == n_ref and torch.equal(got[i], ref), i


def test_stream_host_unpooled_intermediate_stage():
    """An unpooled intermediate stage: the next stage's PSH runs on the main
    stream (no side branch) and records the gating event itself, so the
    pipelined path with the next scene's g0 under g1 still equals single calls."""
    n = 16_000
    stages = (StageConfig(K=64, S=512, S_div=4096, pool_rho=0, seed=0),
              StageConfig(K=48, S=512, S_div=4096, pool_rho=2, seed=1),
              StageConfig(K=16, S=512, S_div=16384, pool_rho=0, seed=2))
    bb = Backbone(stages)
    scenes = []
    for seed in (3, 4, 5):
        c = torch.tensor(O.synth_cloud(seed, n, "surface-shell")).pin_memory()
        f = torch.tensor(np.random.default_rng(seed).normal(size=(n, 96)),
                         dtype=torch.bfloat16).pin_memory()
        scenes.append((c, f))
    seq = scenes * 3
    got = {}
    bb.stream_host(seq, on_result=lambda i, out, n_out: got.__setitem__(i, out.clone()))
    single = Backbone(stages)
    for i, (c, f) in enumerate(seq):
        ref, n_ref = single.forward_host(c, f)
        assert got[i].shape[0] == n_ref and torch.equal(got[i], ref), i


def test_stream_host_recovers_after_error():
    """A scene that raises inside stream_host leaves no pending read-back
    behind: the next call on the same slots returns correct results."""
    from paper_2412_16481_b200.errors import RangeError
    n = 8_000
    stages = (StageConfig(K=64, S=512, S_div=4096, pool_rho=2, seed=0),
              StageConfig(K=32, S=512, S_div=8192, pool_rho=0, seed=1))
    bb = Backbone(stages)
    good = torch.tensor(O.synth_cloud(9, n, "uniform-box")).pin_memory()
    bad = (good * 1e4).pin_memory()          # voxels beyond 2^10 per axis -> RangeError
    f = torch.tensor(np.random.default_rng(9).normal(size=(n, 96)),
                     dtype=torch.bfloat16).pin_memory()
    with pytest.raises(RangeError):
        bb.stream_host([(good, f), (bad, f), (good, f)])
    got = {}
    bb.stream_host([(good, f)] * 3,
                   on_result=lambda i, out, n_out: got.__setitem__(i, out.clone()))
    ref, n_ref = Backbone(stages).forward_host(good, f)
    assert sorted(got) == [0, 1, 2]
    for i in range(3):
        assert torch.equal(got[i], ref), i


def test_stage_boundary_fusions_are_bit_identical():
    """f3d_scatter_ln_pe (input scatter + first LN1 + PE) and
    f3d_pool_reduce_res (last residual folded into the pooling) reproduce the
    unfused scatter / row_ln / pool_reduce sequence bit for bit."""
    from paper_2412_16481_b200 import backbone as B
    n = 30_000
    c = torch.tensor(O.synth_cloud(21, n, "uniform-box"), device="cuda")
    f = torch.tensor(np.random.default_rng(21).normal(size=(n, 96)), dtype=torch.bfloat16,
                     device="cuda")
    stages = (StageConfig(K=64, S=512, S_div=4096, pool_rho=2, seed=0),
              StageConfig(K=32, S=512, S_div=8192, pool_rho=0, seed=1))
    old = B.SCATTER_LN, B.POOL_RESIDUAL
    try:
        B.SCATTER_LN, B.POOL_RESIDUAL = True, True
        a, ca = Backbone(stages).forward(c, f)
        B.SCATTER_LN, B.POOL_RESIDUAL = False, False
        b, cb = Backbone(stages).forward(c, f)
    finally:
        B.SCATTER_LN, B.POOL_RESIDUAL = old
    assert torch.equal(a, b) and torch.equal(ca, cb)


def test_attention_dynamic_scheduler_repeats_and_resets():
    """The tcgen05 kernel takes work items from the device plan's counter
    (live[4]); every launch leaves live[4:6] zeroed, repeated launches on one
    plan are bit-identical, and the static schedule (no live words) agrees."""
    from paper_2412_16481_b200.attention import attend, qstep_for
    r = np.random.default_rng(4)
    K, S, W, d, H = 96, 256, 2, 96, 4
    counts = r.integers(S // 2, S + 1, size=K + 1)
    counts[K] = 300
    base = O.exclusive_scan(counts)
    n = int(counts.sum())
    starts, lens = split_table(counts, base, K, S)
    cd = torch.tensor(counts, dtype=torch.int32, device="cuda")
    bd = torch.tensor(base, dtype=torch.int32, device="cuda")
    qs = qstep_for(d // H)
    dp = A.DeviceRoundPlan(cd, bd, K, S, len(starts), W, 1, 1, 0, n, qstep=qs)
    q, k, v = (torch.randn(n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    outs = []
    for _ in range(3):
        o = torch.zeros(n, d, dtype=torch.bfloat16, device="cuda")
        attend(q, k, v, o, dp, H, d // H)
        outs.append(o)
        assert dp.live.cpu().numpy()[4:6].tolist() == [0, 0]
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    hp = A.RoundPlan(A.plan_arrays(starts, lens, A.round_members(len(starts), W, 1, 1, 0), qs),
                     qstep=qs)
    o = torch.zeros(n, d, dtype=torch.bfloat16, device="cuda")
    attend(q, k, v, o, hp, H, d // H)
    assert torch.equal(o, outs[0])


@pytest.mark.parametrize("fused_psh", [False, True])
def test_two_backbones_on_two_streams(fused_psh):
    """Two Backbone objects replayed concurrently on two streams (two
    cooperative PSH grids in flight at once, every kernel family overlapping)
    give exactly their serial results, repeatedly.  The PSH grid barrier lives
    in each call's workspace (cooperative_groups' driver workspace was shared
    by concurrent grids and corrupted results)."""
    from paper_2412_16481_b200 import backbone as B
    old = B.FUSED_PSH
    B.FUSED_PSH = fused_psh
    try:
        n = 40_000
        stages = (StageConfig(K=128, S=512, S_div=2048, pool_rho=2, seed=0),
                  StageConfig(K=64, S=512, S_div=4096, pool_rho=0, seed=1))
        bbs = [Backbone(stages), Backbone(stages)]
        ins = []
        for bb, (seed, dist) in zip(bbs, ((11, "uniform-box"), (12, "surface-shell"))):
            C = torch.tensor(O.synth_cloud(seed, n, dist), device="cuda")
            X = torch.tensor(np.random.default_rng(seed).normal(size=(n, 96)),
                             dtype=torch.bfloat16, device="cuda")
            bb.capture(n, torch.bfloat16)
            bb.graph_coords.copy_(C)
            bb.graph_feats.copy_(X)
            ins.append((C, X))
        ref = []
        for bb in bbs:
            bb.replay()
            n_out = bb.check_graph()
            ref.append((n_out, bb._graphs["X"][:n_out].clone()))
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        for _ in range(12):
            for bb, s in zip(bbs, streams):
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    bb.replay()
            for s in streams:
                torch.cuda.current_stream().wait_stream(s)
            for bb, (n_out, X) in zip(bbs, ref):
                assert bb.check_graph() == n_out
                assert torch.equal(bb._graphs["X"][:n_out], X)
    finally:
        B.FUSED_PSH = old
