"""Pin the CPU oracle (oracle/restated.py + oracle/psh_seq.c) against golden
vectors produced by the reference itself (tests/golden/make_golden.py).

CPU only; runs in the default ``-m "not gpu"`` suite."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle import restated as O


def test_morton_kats():
    assert int(O.morton(np.array([1, 2, 3]), 2)) == 53          # test_hashing.py:24-26
    assert int(O.morton(np.array([1, 1, 1]), 1)) == 7
    top = (1 << 21) - 1
    assert int(O.morton(np.array([top, top, top]), 21)) == 2 ** 63 - 1   # :66-68
    assert int(O.hash_home(np.array([5, 3, 6]), "xor-mod", 4)) == 0      # :73-75


def test_hashing_golden():
    g = load_golden("hashing.npz")
    np.testing.assert_array_equal(O.morton(g["vox"], 10), g["morton10"])
    np.testing.assert_array_equal(O.morton(g["vox21"], 21), g["morton21"])
    for kind in O.KINDS:
        for K, S_div in ((16, 4), (256, 1024), (40, 6554), (1280, 1639), (7, 1)):
            np.testing.assert_array_equal(O.hash_home(g["vox"], kind, K, S_div, 10),
                                          g[f"{kind}_{K}_{S_div}"], err_msg=kind)
    np.testing.assert_array_equal(O.remap_nonnegative(g["remap_in"], g["remap_batch"]), g["remap_out"])
    np.testing.assert_array_equal(O.remap_nonnegative(g["remap_in"]), g["remap_out_nobatch"])
    np.testing.assert_array_equal(O.voxelize(g["voxA_coords"], (0, 0, 0), 1 / 64), g["voxA"])
    np.testing.assert_array_equal(O.voxelize(g["vox_gc_coords"], (0.1, -0.2, 0.3), 0.037), g["vox_gc"])


def _cases():
    with open(os.path.join(GOLDEN, "recipes.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("case", _cases()["cases"], ids=lambda c: c["name"])
def test_psh_golden(case):
    g = load_golden("psh.npz")
    nm = case["name"]
    vox = g[f"{nm}__vox"].astype(np.int64)
    batch = g[f"{nm}__batch"].astype(np.int64) if case["batched"] else None
    ids, offs, counts, base = O.psh_assign(vox, batch, case["kind"], case["K"], case["S"],
                                           case["S_div"], 10, case["strict"],
                                           O.probe_offsets(case["seed"]), case["max_probes"])
    np.testing.assert_array_equal(ids, g[f"{nm}__id"])
    np.testing.assert_array_equal(offs, g[f"{nm}__off"])
    np.testing.assert_array_equal(counts, g[f"{nm}__counts"])


def test_psh_hotspot_recycle_0488():
    vox = np.tile(np.array([[5, 9, 14]]), (1000, 1))
    ids, _, counts, _ = O.psh_assign(vox, None, "zorder-mod", 256, 16)
    assert counts[256] == 488                                   # test_acceptance.py:79-95


@pytest.mark.parametrize("name", ["A", "B_uniform", "B_shell"])
def test_psh_recipe_digests(name):
    import hashlib
    rc = _cases()["recipes"][name]
    coords = O.synth_cloud(rc["seeds"][0], rc["n"], rc["dist"])
    vox = O.remap_nonnegative(O.voxelize(coords, (0, 0, 0), rc["voxel"]))
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()
    assert sha(vox) == rc["vox_sha"]
    ids, offs, counts, base = O.psh_assign(vox, None, "zorder-div", rc["K"], rc["S"], rc["S_div"])
    assert sha(ids) == rc["id_sha"]
    assert sha(offs) == rc["off_sha"]
    assert counts.tolist() == rc["counts"]
    assert sha(O.dest_index(ids, offs, base, rc["K"])) == rc["dest_sha"]


def test_schedule_golden():
    with open(os.path.join(GOLDEN, "schedule.json")) as fh:
        sch = json.load(fh)
    for key, rounds in sch.items():
        nb, W, stride, shift, nr = map(int, key.split("_"))
        got = O.build_schedule(nb, W, stride, shift, nr)
        assert [[s.tolist() for s in r] for r in got] == rounds, key
    # test_attention.py:23-36 KATs
    assert [s.tolist() for s in O.build_schedule(8, 4)[0]] == [[0, 1, 2, 3], [4, 5, 6, 7]]
    assert [s.tolist() for s in O.build_schedule(8, 4, 1, 2, 2)[1]] == [[2, 3, 4, 5], [6, 7, 0, 1]]
    assert [s.tolist() for s in O.build_schedule(8, 2, 2)[0]] == [[0, 2], [1, 3], [4, 6], [5, 7]]


def test_attention_golden():
    g = load_golden("attention.npz")
    for i, (m, d, H) in enumerate(((16, 64, 4), (100, 64, 4), (300, 96, 4), (200, 48, 2), (130, 128, 1), (64, 32, 2))):
        out = O.attention_dense(g[f"a{i}_Q"], g[f"a{i}_K"], g[f"a{i}_V"], H)
        np.testing.assert_allclose(out, g[f"a{i}_out"], rtol=0, atol=1e-12)
    rg = [tuple(r) for r in g["rg_ranges"]]
    out = O.attention_ranges(g["rg_Q"], g["rg_K"], g["rg_V"], 4, rg, g["rg_mask"])
    np.testing.assert_allclose(out, g["rg_out"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(O.positional_encoding(g["pe_coords"], 96), g["pe_96"], rtol=0, atol=0)
    np.testing.assert_allclose(O.positional_encoding(g["pe_coords"], 12), g["pe_12"], rtol=0, atol=0)


@pytest.mark.parametrize("tag", ["s0", "s1"])
def test_stage_golden(tag):
    g = load_golden("stage.npz")
    seed, n, K, S, d, H, W, shift, rounds = g[f"{tag}_meta"].tolist()
    counts = g[f"{tag}_counts"]
    base = O.exclusive_scan(counts)
    table = O.bucket_table(counts, base, K, S)
    sched = O.build_schedule(len(table[0]), W, 1, shift, rounds)
    p = O.init_params(seed, d, n_heads=H)
    np.testing.assert_array_equal(p["w_q"], g[f"{tag}_wq"])
    np.testing.assert_array_equal(p["w_out"], g[f"{tag}_wout"])
    out = O.stage_forward(g[f"{tag}_feats"], g[f"{tag}_coords"], table, sched, p)
    np.testing.assert_allclose(out, g[f"{tag}_out"], rtol=0, atol=1e-10)


def test_subbuckets_golden():
    g = load_golden("pooling.npz")
    for i in range(30):
        sub, sizes, seeds = O.subbuckets(g[f"t{i}_coords"], int(g[f"t{i}_rho"]))
        np.testing.assert_array_equal(sub, g[f"t{i}_sub"], err_msg=f"tile {i}")
        np.testing.assert_array_equal(seeds, g[f"t{i}_seeds"], err_msg=f"tile {i}")


def test_pool_stage_golden():
    g = load_golden("pooling.npz")
    counts = g["ps_counts"]
    base = O.exclusive_scan(counts)
    for rho, red in ((3, "sum"), (2, "mean"), (4, "max"), (5, "min")):
        pf, pc, nc, nS, _ = O.pool_stage(g["ps_feats"], g["ps_coords"], counts, base, 8, 1500, 1, rho, red)
        np.testing.assert_array_equal(pf, g[f"ps_{rho}_{red}_feats"])
        np.testing.assert_array_equal(pc, g[f"ps_{rho}_{red}_coords"])
        np.testing.assert_array_equal(nc, g[f"ps_{rho}_{red}_counts"])
        assert nS == int(g[f"ps_{rho}_{red}_S"])
