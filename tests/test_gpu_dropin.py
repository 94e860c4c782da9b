"""GPU: the drop-in API holes closed in round 2 — reference KATs ported from
pkg/tests (logical_gather ranges, claim_slot / optimistic_race), reference
attention with a key set of its own size, scatter always validating, and the
INTEGRATION.md ctypes stub executed as written."""

import os
import re

import numpy as np
import pytest
import torch

from oracle import restated as O

pytestmark = pytest.mark.gpu

import paper_2412_16481_b200 as F  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _hand_assignment():
    # pkg/tests/test_attention.py:80-84: four single-voxel groups -> xor-mod
    # buckets 0..3 with counts 3/1/2/2
    vox = np.array([[0, 0, 0]] * 3 + [[1, 0, 0]] * 1 +
                   [[2, 0, 0]] * 2 + [[3, 0, 0]] * 2, dtype=np.int64)
    return F.assign_buckets(vox, None, F.HashConfig("xor-mod", K=4), S=4)


def test_logical_gather_strided_scope_kat():
    """pkg/tests/test_attention.py:87-91."""
    a = _hand_assignment()
    ranges = F.logical_gather(a, [1, 3])
    assert ranges == [(3, 4), (6, 8)]
    assert sum(e - s for s, e in ranges) == a.counts[1] + a.counts[3]


def test_claim_slot_kat():
    """Increment-then-verify: the pre-increment value is the offset; a full
    counter is rolled back (bw/bucketing.py:182-200)."""
    c = np.array([0, 2, 0], dtype=np.int64)
    tr = []
    assert F.claim_slot(c, 0, 2, tr) == 0
    assert F.claim_slot(c, 0, 2, tr) == 1
    assert F.claim_slot(c, 0, 2, tr) is None
    assert F.claim_slot(c, 1, 2) is None
    assert c.tolist() == [2, 2, 0]
    assert tr == [("claim", 0, 0), ("claim", 0, 1), ("full", 0, 2)]


def test_optimistic_race_kat():
    """pkg/tests/test_bucketing.py:97-105: home bucket 0 full; probes of
    (0,0,0) clamp until (-1,-1,1) reaches (0,0,1) -> xor 1 -> bucket 1."""
    cfg = F.HashConfig("xor-mod", K=2)
    counters = np.array([2, 0, 0], dtype=np.int64)
    b, off = F.optimistic_race(0, np.zeros(3, dtype=np.int64), counters, 2, cfg,
                               F.default_probe_schedule())
    assert (b, off) == (1, 0)
    assert counters[1] == 1


def test_optimistic_race_recycle_after_exhaustion():
    """pkg/tests/test_bucketing.py:108-116: K=1, every probe hashes back to
    the single full bucket -> recycle."""
    cfg = F.HashConfig("xor-mod", K=1)
    counters = np.array([1, 0], dtype=np.int64)
    trace = []
    b, off = F.optimistic_race(7, np.zeros(3, dtype=np.int64), counters, 1, cfg,
                               F.default_probe_schedule(), trace=trace)
    assert (b, off) == (1, 0)
    failed = [t for t in trace if t[-1] == "full"]
    assert len(failed) == F.default_probe_schedule().max_probes
    assert trace[-1][1] == "recycle"


@pytest.mark.parametrize("kind,strict", [("zorder-div", True), ("xor-div", True),
                                         ("zorder-mod", False), ("xor-mod", False)])
def test_optimistic_race_replays_sequential_psh(kind, strict):
    """Driving optimistic_race point by point (home claims via claim_slot)
    reproduces the oracle's sequential assignment, strict-div skips included."""
    r = np.random.default_rng(11)
    vox = r.integers(0, 24, size=(300, 3))
    K, S = 9, 8
    cfg = F.HashConfig(kind, K=K, S_div=1500 if kind.endswith("div") else 8,
                       div_overflow="error" if strict else "wrap")
    probes = F.default_probe_schedule(max_probes=32)
    home = np.asarray(F.hash_bucket(vox, F.HashConfig(kind, K=K, S_div=cfg.S_div)))
    if strict:
        q = (O.morton(vox, 10) if kind.startswith("zorder")
             else vox[:, 0] ^ vox[:, 1] ^ vox[:, 2]) // cfg.S_div
        keep = q < K
        vox, home = vox[keep], home[keep]
    counters = np.zeros(K + 1, dtype=np.int64)
    ids, offs = [], []
    for i in range(len(vox)):
        off = F.claim_slot(counters, int(home[i]), S)
        if off is not None:
            ids.append(int(home[i]))
            offs.append(off)
        else:
            b, o = F.optimistic_race(i, vox[i], counters, S, cfg, probes)
            ids.append(b)
            offs.append(o)
    a = F.assign_buckets(vox, None, cfg, S, probes)
    assert ids == a.bucket_id.tolist()
    assert offs == a.bucket_offset.tolist()
    assert counters.tolist() == a.counts.tolist()


@pytest.mark.parametrize("m,mk", [(40, 97), (130, 16), (5, 300)])
def test_reference_attention_distinct_key_count(m, mk):
    """bw/attention.py:147-166: the einsum takes any number of keys."""
    r = np.random.default_rng(m + mk)
    p = F.AttentionParams(d_model=64, n_heads=4)
    Q, K, V = r.normal(size=(m, 64)), r.normal(size=(mk, 64)), r.normal(size=(mk, 64))
    out = F.reference_attention(Q, K, V, p)
    assert out.shape == (m, 64)
    ref = O.attention_dense(Q, K, V, 4)
    rel = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    assert rel < 1e-2, rel


def test_scatter_validates_package_assignments():
    """bw/bucketing.py:397: scatter validates every assignment, including one
    this package produced and the caller then corrupted."""
    a = _hand_assignment()
    a.bucket_offset = a.bucket_offset.copy()
    a.bucket_offset[0] = 2                  # collides with point 2
    with pytest.raises(F.IntegrityError):
        F.scatter(np.zeros((8, 4), dtype=np.float32), a)


def _integration_stub():
    txt = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(# bucketswin/_f3d\.py.*?)```", txt, re.S).group(1)
    lib = os.path.join(ROOT, "paper_2412_16481_b200", "libf3d.so")
    block = block.replace("/path/to/paper_2412_16481_b200/libf3d.so", lib)
    ns = {}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    return ns["assign_one_stage"]


@pytest.mark.parametrize("seed", range(4))
def test_integration_stub_assign_one_stage(seed):
    """The reference-side ctypes binding in INTEGRATION.md, executed verbatim,
    fills the reference's output arrays exactly like bw/_kernels.py:69-90."""
    assign_one_stage = _integration_stub()
    r = np.random.default_rng(seed)
    n, K, S = 3000, 37, 64
    vox = r.integers(0, 40, size=(n, 3))
    cfg = F.HashConfig("zorder-div", K=K, S_div=2000)
    h0 = np.asarray(F.hash_bucket(vox, cfg))
    probes = F.default_probe_schedule(seed=seed if seed % 2 else None)
    counters = np.zeros(K + 1, dtype=np.int64)
    bid = np.empty(n, dtype=np.int64)
    boff = np.empty(n, dtype=np.int64)
    assign_one_stage(vox, h0, counters, S, K, cfg.kind_code, cfg.S_div, 10, False,
                     probes.offsets, probes.max_probes, 1023, bid, boff)
    ids, offs, counts, _ = O.psh_assign(vox, None, "zorder-div", K, S, 2000, offsets=probes.offsets)
    assert np.array_equal(bid, ids) and np.array_equal(boff, offs)
    assert np.array_equal(counters, counts)
