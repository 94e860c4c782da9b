"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container only (needs the reference package, which does not
travel to the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [--ref /root/repo/baseline/_ref]

The reference is imported from the git-ignored copy ``baseline/_ref`` (see
SURVEY.md §0: importing /root/reference directly writes numba caches into it).
Everything written here is small: full arrays for instances up to a few
thousand points, and sha256 digests + counts for the full-size configs.
"""

import argparse
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()


def random_voxels(rng, n):
    """Same shape family as pkg/tests/test_acceptance.py:27-40."""
    side = int(rng.choice((4, 8, 16, 32, 64)))
    style = int(rng.integers(3))
    if style == 0:
        return rng.integers(0, side, size=(n, 3))
    if style == 1:
        centers = rng.integers(0, side, size=(int(rng.integers(1, 9)), 3))
        pick = rng.integers(0, len(centers), size=n)
        jitter = rng.normal(0.0, 2.0, size=(n, 3)).astype(np.int64)
        return np.clip(centers[pick] + jitter, 0, side - 1)
    vox = rng.integers(0, side, size=(n, 3))
    vox[rng.random(n) < 0.4] = rng.integers(0, side, size=3)
    return vox


# The §8(d) recipes: name -> (seed(s), n, dist, voxel, K, S, S_div)
RECIPES = {
    "A": dict(seeds=[7], n=4096, dist="uniform-box", voxel=1 / 64, K=40, S=128, S_div=6554),
    "B_uniform": dict(seeds=[7], n=100_000, dist="uniform-box", voxel=1 / 64, K=256, S=512, S_div=1024),
    "B_shell": dict(seeds=[7], n=100_000, dist="surface-shell", voxel=1 / 64, K=256, S=512, S_div=1024),
    "C_uniform": dict(seeds=list(range(100, 116)), n=200_000, dist="uniform-box", voxel=1 / 64, K=512, S=512, S_div=512),
    "C_clusters": dict(seeds=list(range(100, 116)), n=200_000, dist="gaussian-clusters", voxel=1 / 64, K=512, S=512, S_div=512),
    "D": dict(seeds=[7], n=1_000_000, dist="uniform-box", voxel=1 / 128, K=1280, S=1024, S_div=1639),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=os.path.join(HERE, "..", "..", "baseline", "_ref"))
    args = ap.parse_args()
    sys.path.insert(0, os.path.abspath(args.ref))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    from bucketswin import attention as attn
    from bucketswin import bucketing, geometry, hashing, pooling, stage

    out = {}

    # ---------------------------------------------------------------- hashing
    rng = np.random.default_rng(11)
    v = rng.integers(0, 1024, size=(300, 3))
    h = {"vox": v, "morton10": hashing.morton_encode(v, 10)}
    for kind in hashing.HASH_KINDS:
        for K, S_div in ((16, 4), (256, 1024), (40, 6554), (1280, 1639), (7, 1)):
            h[f"{kind}_{K}_{S_div}"] = hashing.hash_bucket(v, hashing.HashConfig(kind, K=K, S_div=S_div))
    v21 = rng.integers(0, 1 << 21, size=(100, 3))
    h["vox21"] = v21
    h["morton21"] = hashing.morton_encode(v21, 21)
    raw = rng.integers(-500, 500, size=(400, 3))
    bat = rng.permutation(np.repeat(np.arange(4), 100))
    h["remap_in"] = raw
    h["remap_batch"] = bat
    h["remap_out"] = hashing.remap_nonnegative(raw, bat)
    h["remap_out_nobatch"] = hashing.remap_nonnegative(raw)
    cl = geometry.synth_cloud(7, 4096, "uniform-box")
    h["voxA_coords"] = cl.coords
    h["voxA"] = geometry.voxelize(cl, geometry.VoxelGrid(1 / 64))
    cl2 = geometry.synth_cloud(3, 2000, "gaussian-clusters")
    h["vox_gc_coords"] = cl2.coords
    h["vox_gc"] = geometry.voxelize(cl2, geometry.VoxelGrid(0.037, origin=(0.1, -0.2, 0.3)))
    np.savez_compressed(os.path.join(HERE, "hashing.npz"), **h)

    # -------------------------------------------------------------------- PSH
    psh = {}
    cases = []

    def add(name, vox, batch, kind, K, S, S_div=8, strict=False, seed=None, max_probes=32):
        cfg = hashing.HashConfig(kind, K=K, S_div=S_div, div_overflow="error" if strict else "wrap")
        probes = bucketing.default_probe_schedule(seed=seed, max_probes=max_probes)
        a = bucketing.assign_buckets(vox, batch, cfg, S, probes=probes)
        psh[f"{name}__vox"] = np.asarray(vox, dtype=np.int32)
        if batch is not None:
            psh[f"{name}__batch"] = np.asarray(batch, dtype=np.int32)
        psh[f"{name}__id"] = a.bucket_id.astype(np.int32)
        psh[f"{name}__off"] = a.bucket_offset.astype(np.int32)
        psh[f"{name}__counts"] = a.counts
        cases.append(dict(name=name, kind=kind, K=K, S=S, S_div=S_div, strict=strict,
                          seed=seed, max_probes=max_probes, batched=batch is not None))

    add("three", np.zeros((3, 3), np.int64), None, "xor-mod", 2, 2)
    add("k1", np.zeros((2, 3), np.int64), None, "xor-mod", 1, 1)
    add("hotspot", np.tile(np.array([[5, 9, 14]]), (1000, 1)), None, "zorder-mod", 256, 16)
    add("batch6", np.zeros((6, 3), np.int64), np.array([0, 0, 0, 1, 1, 1]), "xor-mod", 2, 2)
    add("reversed", np.array([[1, 0, 0], [0, 0, 0]]), None, "xor-mod", 2, 1)
    r = np.random.default_rng(20240501)
    kinds = hashing.HASH_KINDS
    for i in range(40):
        n = int(r.integers(1, 3000))
        vox = random_voxels(r, n)
        kind = kinds[i % 4]
        K = int(r.choice((1, 4, 16, 64, 256)))
        S = int(r.choice((1, 4, 16, 32, 512)))
        S_div = int(r.choice((1, 4, 8, 64, 1024)))
        strict = False
        seed = int(r.integers(0, 1000)) if i % 5 == 1 else None
        mp = int(r.choice((1, 8, 32, 124))) if i % 7 == 3 else 32
        batch = None
        if i % 4 == 2:
            nb = int(r.integers(1, 5))
            batch = r.permutation(np.arange(n) % nb) if n >= nb else np.zeros(n, np.int64)
        add(f"rand{i:02d}", vox, batch, kind, K, S, S_div, strict, seed, mp)
    # strict-div instances whose home quotients fit (probes may still skip)
    for i in range(6):
        n = int(r.integers(200, 2000))
        side = 16
        vox = r.integers(0, side, size=(n, 3))
        kind = ("xor-div", "zorder-div")[i % 2]
        S_div = 64 if kind == "zorder-div" else 2
        key_max = (hashing.morton_encode(np.array([[side - 1] * 3]), 10)[0] if kind == "zorder-div" else 15) // S_div
        # K chosen so every home quotient fits but some clamped probes may not
        K = int(key_max + 1)
        add(f"strict{i}", vox, None, kind, K, int(r.choice((4, 16))), S_div, True, None, 32)
    np.savez_compressed(os.path.join(HERE, "psh.npz"), **psh)

    # full-size recipe digests
    recipes = {}
    for name, rc in RECIPES.items():
        coords, batch = [], []
        for b, s in enumerate(rc["seeds"]):
            c = geometry.synth_cloud(s, rc["n"], rc["dist"]).coords
            coords.append(c)
            batch.append(np.full(len(c), b, dtype=np.int64))
        coords = np.vstack(coords)
        batch = np.concatenate(batch)
        multi = len(rc["seeds"]) > 1
        vox = hashing.remap_nonnegative(
            geometry.voxelize(geometry.PointCloud(coords, batch if multi else None),
                              geometry.VoxelGrid(rc["voxel"])), batch if multi else None)
        cfg = hashing.HashConfig("zorder-div", K=rc["K"], S_div=rc["S_div"])
        a = bucketing.assign_buckets(vox, batch if multi else None, cfg, rc["S"])
        recipes[name] = dict(rc, vox_sha=sha(vox), id_sha=sha(a.bucket_id), off_sha=sha(a.bucket_offset),
                             dest_sha=sha(a.dest_index()), counts=a.counts.tolist(),
                             recycle=a.recycle_fraction())
        print(name, "recycle", a.recycle_fraction(), flush=True)
    with open(os.path.join(HERE, "recipes.json"), "w") as fh:
        json.dump({"cases": cases, "recipes": recipes}, fh, indent=1)

    # --------------------------------------------------------------- schedule
    sch = {}
    for nb, W, stride, shift, rounds in ((8, 4, 1, 0, 1), (8, 4, 1, 2, 2), (8, 2, 2, 0, 1), (8, 4, 4, 1, 3),
                                         (7, 3, 2, 1, 4), (296, 2, 1, 1, 2), (40, 2, 1, 1, 2), (13, 5, 3, 4, 6),
                                         (1, 1, 1, 0, 1)):
        s = attn.build_schedule(nb, W, stride, shift, rounds)
        sch[f"{nb}_{W}_{stride}_{shift}_{rounds}"] = [[sc.tolist() for sc in rd] for rd in s.rounds]
    with open(os.path.join(HERE, "schedule.json"), "w") as fh:
        json.dump(sch, fh)

    # -------------------------------------------------------------- attention
    at = {}
    r = np.random.default_rng(4242)
    acases = []
    for i, (m, d, H) in enumerate(((16, 64, 4), (100, 64, 4), (300, 96, 4), (200, 48, 2), (130, 128, 1), (64, 32, 2))):
        Q, Km, V = (r.normal(size=(m, d)) for _ in range(3))
        params = attn.AttentionParams(d_model=d, n_heads=H)
        at[f"a{i}_Q"], at[f"a{i}_K"], at[f"a{i}_V"] = Q, Km, V
        at[f"a{i}_out"] = attn.tiled_attention(Q, Km, V, params, ranges=[(0, m)])
        acases.append(dict(i=i, m=m, d=d, H=H))
    # two disjoint ranges + a mask
    N, d, H = 400, 64, 4
    Q, Km, V = (r.normal(size=(N, d)) for _ in range(3))
    mask = r.random(N) > 0.1
    rg = [(10, 150), (220, 397)]
    at["rg_Q"], at["rg_K"], at["rg_V"], at["rg_mask"] = Q, Km, V, mask
    at["rg_ranges"] = np.array(rg)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        at["rg_out"] = attn.tiled_attention(Q, Km, V, attn.AttentionParams(d, H), ranges=rg, mask=mask)
    pe_c = r.uniform(size=(50, 3))
    at["pe_coords"] = pe_c
    at["pe_96"] = attn.positional_encoding(pe_c, 96)
    at["pe_12"] = attn.positional_encoding(pe_c, 12)
    np.savez_compressed(os.path.join(HERE, "attention.npz"), **at)

    # ------------------------------------------------------------------ stage
    st = {}
    for tag, (seed, n, dist, vs, K, S, S_div, d, H, W, shift, rounds) in {
        "s0": (7, 600, "uniform-box", 1 / 16, 8, 128, 64, 24, 2, 2, 1, 2),
        "s1": (9, 900, "surface-shell", 1 / 32, 12, 64, 256, 48, 4, 3, 1, 2),
    }.items():
        cl = geometry.synth_cloud(seed, n, dist)
        vox = hashing.remap_nonnegative(geometry.voxelize(cl, geometry.VoxelGrid(vs)))
        a = bucketing.assign_buckets(vox, None, hashing.HashConfig("zorder-div", K=K, S_div=S_div), S)
        F0 = np.random.default_rng(1).normal(size=(n, d))
        feats, _ = bucketing.scatter(F0, a)
        coords, _ = bucketing.scatter(cl.coords, a)
        table = a.bucket_table(split_recycle=True)
        sched = attn.build_schedule(len(table[0]), W, 1, shift, rounds)
        p = stage.init_params(seed, d, n_heads=H)
        st[f"{tag}_feats"] = feats
        st[f"{tag}_coords"] = coords
        st[f"{tag}_counts"] = a.counts
        st[f"{tag}_out"] = stage.stage_forward(feats, coords, a, sched, p)
        st[f"{tag}_meta"] = np.array([seed, n, K, S, d, H, W, shift, rounds])
        st[f"{tag}_wq"] = p.w_q
        st[f"{tag}_wout"] = p.w_out
    np.savez_compressed(os.path.join(HERE, "stage.npz"), **st)

    # ---------------------------------------------------------------- pooling
    pl = {}
    r = np.random.default_rng(999)
    for i in range(30):
        m = int(r.integers(1, 1025)) if i > 2 else (1, 1024, 1000)[i]
        rho = int(r.choice((2, 3, 4, 7, 8))) if i > 2 else (1, 2, 2)[i]
        scale = float(r.choice((1e-3, 1.0, 50.0)))
        c = r.uniform(0, scale, size=(m, 3))
        if i % 2:
            piles = r.uniform(0, scale, size=(max(1, m // 100), 3))
            idx = r.integers(0, len(piles), size=m // 2)
            c[:len(idx)] = piles[idx]
        sub = pooling.build_subbuckets(c, rho)
        pl[f"t{i}_coords"] = c
        pl[f"t{i}_rho"] = np.array(rho)
        pl[f"t{i}_sub"] = sub.subbucket_id.astype(np.int32)
        pl[f"t{i}_seeds"] = sub.seeds
    # pool_stage on a bucketed cloud with a >1024-row bucket and recycle rows
    cl = geometry.synth_cloud(7, 5000, "gaussian-clusters")
    vox = hashing.remap_nonnegative(geometry.voxelize(cl, geometry.VoxelGrid(0.05)))
    a = bucketing.assign_buckets(vox, None, hashing.HashConfig("xor-mod", K=8), 1500)
    feats, _ = bucketing.scatter(np.random.default_rng(2).normal(size=(5000, 8)), a)
    coords, _ = bucketing.scatter(cl.coords, a)
    pl["ps_feats"], pl["ps_coords"], pl["ps_counts"] = feats, coords, a.counts
    for rho, red in ((3, "sum"), (2, "mean"), (4, "max"), (5, "min")):
        pf, pc, na = pooling.pool_stage(feats, coords, a, rho, red)
        pl[f"ps_{rho}_{red}_feats"] = pf
        pl[f"ps_{rho}_{red}_coords"] = pc
        pl[f"ps_{rho}_{red}_counts"] = na.counts
        pl[f"ps_{rho}_{red}_S"] = np.array(na.S)
    np.savez_compressed(os.path.join(HERE, "pooling.npz"), **pl)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
