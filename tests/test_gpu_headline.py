"""GPU parity at the workloads the bench measures (BASELINE.json configs[1..3],
SURVEY.md §8(d)):

* config B: the full 100K-point 2-stage ``scannet_backbone`` forward against
  the oracle composition (bw/stage.py:99-159 + bw/pooling.py:187-242 composed
  as bw/cli.py:439-529), every scope of every round -- PSH layouts of both
  stages and the final scattered coordinates bit-exact, features within the
  stage tolerance (2e-2 relative Frobenius);
* config C (16 x 200K) and config D (1M points, C=384, W=4): full-size PSH and
  pooling layouts bit-exact per scene, plus 64 sampled scopes per round and
  stage checked against dense float64 attention on the GPU's own bf16 round
  input (1e-2);
* config D attention at C=512 on its real PSH plan: 64 sampled scopes per round.
"""

import os

import numpy as np
import pytest
import torch

from oracle import restated as O

pytestmark = pytest.mark.gpu

from paper_2412_16481_b200 import attention as A  # noqa: E402
from paper_2412_16481_b200.backbone import (Backbone, StageConfig,  # noqa: E402
                                            scannet_backbone, split_table)

THREADS = os.cpu_count() or 1
CONFIG_C = (StageConfig(K=512, S=512, S_div=512, W=2, d_model=96, pool_rho=2, seed=0),
            StageConfig(K=256, S=512, S_div=1024, W=2, d_model=96, pool_rho=0, seed=1))
CONFIG_D = (StageConfig(voxel=1 / 128, K=1280, S=1024, S_div=1639, W=4, d_model=384,
                        pool_rho=2, seed=0),
            StageConfig(voxel=1 / 128, K=640, S=1024, S_div=3278, W=4, d_model=384,
                        pool_rho=0, seed=1))


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _dev_layout(tr):
    """(ids, offs) of one traced stage, real rows only, int64 host."""
    a = tr.assignment
    ids = a._dev["id"][:tr.n].to(torch.int64).cpu().numpy()
    offs = a._dev["off"][:tr.n].to(torch.int64).cpu().numpy()
    return ids, offs


def _forward_with_rounds(bb, C, X):
    """Eager forward that keeps every round's bf16 Q/K/V and attention output
    (clones enqueued right after the round's attention, stream-ordered)."""
    rounds = []
    bb.round_hook = lambda si, t, q, k, v, a: rounds.append(
        (si, t, q.clone(), k.clone(), v.clone(), a.clone()))
    try:
        out = bb.forward(C, X, keep_trace=True)
    finally:
        bb.round_hook = None
    torch.cuda.synchronize()
    return out, rounds


def _check_sampled_scopes(stages, trace, rounds, n_heads=4, per_round=64, tol=1e-2, seed=0):
    """per_round sampled scopes of every (stage, round): dense float64
    attention (bw/attention.py:147-166) on the GPU's own bf16 Q/K/V rows of
    the scope against the GPU's output rows.  Returns the worst error."""
    r = np.random.default_rng(seed)
    worst = 0.0
    for si, t, q, k, v, a in rounds:
        cfg, tr = stages[si], trace[si]
        counts = np.asarray(tr.counts, dtype=np.int64)
        starts, lens = split_table(counts, O.exclusive_scan(counts), cfg.K, cfg.S)
        members = A.round_members(len(starts), cfg.W, cfg.stride, cfg.shift, t)
        scopes = []
        for row in members:
            b = row[row >= 0]
            b = b[lens[b] > 0]
            if len(b):
                scopes.append(b)
        pick = r.choice(len(scopes), size=min(per_round, len(scopes)), replace=False)
        for s in pick:
            rows = np.concatenate([np.arange(starts[b], starts[b] + lens[b]) for b in scopes[s]])
            ri = torch.as_tensor(rows, device=q.device)
            kh, vh = (x[ri].double().cpu().numpy() for x in (k, v))
            # every key of the scope; up to 256 sampled query rows of it (the
            # dense float64 oracle of a 4096-row scope is 4 x 4096^2 scores)
            qi = rows if len(rows) <= 256 else np.sort(r.choice(rows, 256, replace=False))
            qt = torch.as_tensor(qi, device=q.device)
            qh = q[qt].double().cpu().numpy()
            got = a[qt].double().cpu().numpy()
            ref = O.attention_dense(qh, kh, vh, n_heads)
            e = _rel(got, ref)
            worst = max(worst, e)
            assert e < tol, (si, t, int(s), len(rows), e)
    return worst


def _oracle_layouts(coords, stages):
    """Coordinate-only oracle composition: PSH of every stage, scattered
    coordinates, pooled f64 centroids (features do not affect layouts)."""
    out = []
    C = np.asarray(coords, dtype=np.float64)
    for cfg in stages:
        vox = O.remap_nonnegative(O.voxelize(C, (0.0, 0.0, 0.0), cfg.voxel))
        ids, offs, counts, base = O.psh_assign(vox, None, cfg.kind, cfg.K, cfg.S, cfg.S_div)
        dest = O.dest_index(ids, offs, base, cfg.K)
        Cs = np.empty_like(C)
        Cs[dest] = C
        out.append((ids, offs, Cs))
        if cfg.pool_rho:
            _, C, _, _, _ = O.pool_stage(np.zeros((len(C), 1)), Cs, counts, base, cfg.K, cfg.S, 1,
                                         cfg.pool_rho, "mean")
    return out


@pytest.mark.parametrize("dist", ["uniform-box", "surface-shell"])
def test_config_b_full_backbone_matches_oracle(dist):
    """The headline workload itself: synth_cloud(7, 100K), features
    default_rng(1).normal, scannet_backbone(); the oracle runs every scope."""
    n = 100_000
    coords = O.synth_cloud(7, n, dist)
    feats = np.random.default_rng(1).normal(size=(n, 96))
    bb = Backbone(scannet_backbone())
    (X, C), rounds = _forward_with_rounds(bb, torch.tensor(coords, device="cuda"),
                                          torch.tensor(feats, dtype=torch.float32, device="cuda"))
    trace = bb.last_trace
    rec = []
    OX, OC = O.backbone_forward(coords, feats, scannet_backbone(), threads=THREADS, record=rec)
    for si, tr in enumerate(trace):
        ids, offs = _dev_layout(tr)
        assert tr.n == len(rec[si]["ids"])
        np.testing.assert_array_equal(ids, rec[si]["ids"])
        np.testing.assert_array_equal(offs, rec[si]["offs"])
        np.testing.assert_array_equal(np.asarray(tr.counts), rec[si]["counts"])
    # pooled centroids re-bucketed and scattered: the last stage's coordinates
    assert C.shape == OC.shape
    np.testing.assert_array_equal(C.cpu().numpy(), OC)
    e = _rel(X.double().cpu().numpy(), OX)
    assert e < 2e-2, e
    _check_sampled_scopes(scannet_backbone(), trace, rounds)


@pytest.mark.parametrize("variant", ["uniform-box", "gaussian-clusters"])
def test_config_c_layouts_and_sampled_scopes(variant):
    """16 x 200K scenes (seeds 100..115) through the config-C backbone:
    per-scene PSH layouts of both stages and the final (pooled, re-bucketed,
    scattered) coordinates bit-exact; 64 sampled scopes per round and stage."""
    bb = Backbone(CONFIG_C)
    n = 200_000
    seeds = range(100, 116) if variant == "uniform-box" else range(100, 104)
    for seed in seeds:
        coords = O.synth_cloud(seed, n, variant)
        feats = np.random.default_rng(seed).normal(size=(n, 96))
        (X, C), rounds = _forward_with_rounds(
            bb, torch.tensor(coords, device="cuda"),
            torch.tensor(feats, dtype=torch.bfloat16, device="cuda"))
        trace = bb.last_trace
        ref = _oracle_layouts(coords, CONFIG_C)
        for si, tr in enumerate(trace):
            ids, offs = _dev_layout(tr)
            np.testing.assert_array_equal(ids, ref[si][0], err_msg=f"scene {seed} stage {si}")
            np.testing.assert_array_equal(offs, ref[si][1], err_msg=f"scene {seed} stage {si}")
        np.testing.assert_array_equal(C.cpu().numpy(), ref[-1][2])
        assert torch.isfinite(X).all()
        _check_sampled_scopes(CONFIG_C, trace, rounds, seed=seed)
        del rounds


def test_config_d_layouts_and_sampled_scopes():
    """1M points at voxel 1/128, K=1280 S=1024 W=4 (scopes up to 4096 rows),
    C=384 H=4: full-size layouts bit-exact, 64 sampled scopes per round."""
    n = 1_000_000
    coords = O.synth_cloud(7, n, "uniform-box")
    feats = np.random.default_rng(7).normal(size=(n, 384))
    bb = Backbone(CONFIG_D)
    (X, C), rounds = _forward_with_rounds(
        bb, torch.tensor(coords, device="cuda"),
        torch.tensor(feats, dtype=torch.bfloat16, device="cuda"))
    trace = bb.last_trace
    ref = _oracle_layouts(coords, CONFIG_D)
    for si, tr in enumerate(trace):
        ids, offs = _dev_layout(tr)
        np.testing.assert_array_equal(ids, ref[si][0])
        np.testing.assert_array_equal(offs, ref[si][1])
    np.testing.assert_array_equal(C.cpu().numpy(), ref[-1][2])
    assert torch.isfinite(X).all()
    _check_sampled_scopes(CONFIG_D, trace, rounds)


def test_config_d_attention_c512_on_real_plan():
    """The bench's roofline_wide workload: C=512 (dh=128) attention on the
    config-D PSH plan of the 1M-point scene, both rounds, random bf16 Q/K/V;
    64 sampled scopes per round against dense float64 attention."""
    n, d, H = 1_000_000, 512, 4
    cfg = StageConfig(voxel=1 / 128, K=1280, S=1024, S_div=1639, W=4, d_model=d, n_heads=H)
    C = torch.tensor(O.synth_cloud(7, n, "uniform-box"), device="cuda")
    asg, _, _ = Backbone.bucketize(Backbone.__new__(Backbone), C, cfg)
    counts = asg._dev["counts"].to(torch.int64).cpu().numpy()
    nb_cap = cfg.K + -(-n // cfg.S)
    g = torch.Generator(device="cuda").manual_seed(0)
    qkv = torch.randn((n, 3 * d), device="cuda", generator=g).to(torch.bfloat16)
    q, k, v = (qkv[:, i * d:(i + 1) * d] for i in range(3))
    rounds = []
    for t in range(2):
        plan = A.DeviceRoundPlan(asg._dev["counts"], asg._dev["base"], cfg.K, cfg.S, nb_cap, cfg.W,
                                 cfg.stride, cfg.shift, t, n, qstep=A.qstep_for(d // H))
        out = torch.zeros((n, d), device="cuda", dtype=torch.bfloat16)
        A.attend(q, k, v, out, plan, H, d // H)
        rounds.append((0, t, q, k, v, out))

    class _T:
        pass
    tr = _T()
    tr.counts = counts
    _check_sampled_scopes((cfg,), [tr], rounds, n_heads=H)
