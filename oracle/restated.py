"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement (numpy float64 / int64, plus the C claim loop in
``psh_seq.c``) of the reference ``bucketswin`` hot path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import this module, and only as the checker or the timed
CPU baseline.  The product package never imports it and has no CPU fallback.

Every function cites the reference file:line it restates (paths relative to
``pkg/src/bucketswin/``).  The restatement is pinned against golden vectors
produced by the reference itself (``tests/golden/make_golden.py``), see
``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

KINDS = ("xor-mod", "xor-div", "zorder-mod", "zorder-div")
POOL_TILE_CAP = 1024

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


# ------------------------------------------------------------------ C helper

def build_c(force: bool = False) -> str:
    """Compile psh_seq.c into oracle/_build/libpsh_oracle.so (gcc -O2)."""
    out_dir = os.path.join(_HERE, "_build")
    os.makedirs(out_dir, exist_ok=True)
    so = os.path.join(out_dir, "libpsh_oracle.so")
    src = os.path.join(_HERE, "psh_seq.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", so, src])
    return so


def _lib():
    global _LIB
    if _LIB is None:
        lib = ctypes.CDLL(build_c())
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        i32 = ctypes.c_int
        lib.oracle_psh_assign.argtypes = [p, p, p, i64, i64, i64, i64, i32, i64, i32,
                                          i32, p, i64, i64, p, p, p]
        lib.oracle_psh_assign.restype = None
        _LIB = lib
    return _LIB


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------------ geometry

def voxelize(coords, origin=(0.0, 0.0, 0.0), voxel_size=1.0):
    """geometry.py:69-72 — floor((c - origin) / size) with a true IEEE divide."""
    c = np.asarray(coords, dtype=np.float64)
    return np.floor((c - np.asarray(origin, dtype=np.float64)) / voxel_size).astype(np.int64)


def synth_cloud(seed: int, n: int, dist: str = "uniform-box"):
    """geometry.py:183-212 — same PCG64 draw order, returns (n,3) f64."""
    rng = np.random.default_rng(seed)
    if dist == "uniform-box":
        return rng.random((n, 3))
    if dist == "gaussian-clusters":
        centers = np.array([[0.2, 0.2, 0.2], [0.8, 0.8, 0.2],
                            [0.2, 0.8, 0.8], [0.8, 0.2, 0.8]])
        which = rng.integers(0, 4, size=n)
        return centers[which] + rng.normal(0.0, 0.03, size=(n, 3))
    if dist == "surface-shell":
        dirs = rng.normal(size=(n, 3))
        nrm = np.linalg.norm(dirs, axis=1, keepdims=True)
        nrm[nrm == 0] = 1.0
        radius = 0.4 + rng.normal(0.0, 0.005, size=(n, 1))
        return 0.5 + dirs / nrm * radius
    raise ValueError(dist)


# ------------------------------------------------------------------- hashing

def remap_nonnegative(vox, batch=None):
    """hashing.py:128-149 — subtract the per-batch, per-axis minimum."""
    v = np.array(vox, dtype=np.int64, copy=True)
    if len(v) == 0:
        return v
    if batch is None:
        return v - v.min(axis=0)
    b = np.asarray(batch, dtype=np.int64)
    for bb in np.unique(b):
        sel = b == bb
        v[sel] -= v[sel].min(axis=0)
    return v


def range_violation(v, bits):
    """hashing.py:60-75 — first (axis, value, 'neg'|'big') violation or None."""
    v = np.asarray(v, dtype=np.int64)
    for ax in range(3):
        comp = v[..., ax]
        if comp.size == 0:
            continue
        lo, hi = int(comp.min()), int(comp.max())
        if lo < 0:
            return ax, lo, "neg"
        if hi >= (1 << bits):
            return ax, hi, "big"
    return None


def _spread3(a):
    """Place bit k of a at bit 3k (a < 2^21): the magic-number bit spread."""
    a = a.astype(np.uint64) & np.uint64(0x1FFFFF)
    a = (a | (a << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    a = (a | (a << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    a = (a | (a << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    a = (a | (a << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    a = (a | (a << np.uint64(2))) & np.uint64(0x1249249249249249)
    return a


def morton(v, bits=10):
    """hashing.py:78-98 / _kernels.py:17-24 — x at 3k, y at 3k+1, z at 3k+2."""
    v = np.asarray(v, dtype=np.int64)
    m = np.int64((1 << bits) - 1)
    code = (_spread3(v[..., 0] & m) | (_spread3(v[..., 1] & m) << np.uint64(1))
            | (_spread3(v[..., 2] & m) << np.uint64(2)))
    return code.astype(np.int64)


def hash_home(v, kind, K, S_div=8, bits=10):
    """hashing.py:101-125 (no range check; see range_violation)."""
    v = np.asarray(v, dtype=np.int64)
    key = (v[..., 0] ^ v[..., 1] ^ v[..., 2]) if kind.startswith("xor") else morton(v, bits)
    if kind.endswith("-div"):
        key = key // S_div
    return key % K


def hash_quotient_max(v, kind, S_div=8, bits=10):
    """Largest key // S_div (hashing.py:116-122 strict-mode check)."""
    v = np.asarray(v, dtype=np.int64)
    key = (v[..., 0] ^ v[..., 1] ^ v[..., 2]) if kind.startswith("xor") else morton(v, bits)
    return int((key // S_div).max()) if key.size else -1


# ---------------------------------------------------------------------- PSH

def probe_offsets(seed=None):
    """bucketing.py:51-66 — radius-1 then radius-2 L-inf shells, lexicographic,
    each shell shuffled by default_rng(seed) when seeded."""
    r1 = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)
          if (a, b, c) != (0, 0, 0)]
    r2 = [(a, b, c) for a in range(-2, 3) for b in range(-2, 3) for c in range(-2, 3)
          if max(abs(a), abs(b), abs(c)) == 2]
    if seed is not None:
        g = np.random.default_rng(seed)
        g.shuffle(r1)
        g.shuffle(r2)
    return np.array(r1 + r2, dtype=np.int64)


def psh_assign(vox, batch, kind, K, S, S_div=8, bits=10, strict=False,
               offsets=None, max_probes=32):
    """bucketing.py:275-320 + _kernels.py:41-90 via the C claim loop.

    Returns (bucket_id, bucket_offset, counts, bucket_base) as int64 arrays.
    """
    vox = np.ascontiguousarray(vox, dtype=np.int64)
    n = len(vox)
    if offsets is None:
        offsets = probe_offsets()
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    if batch is None:
        b = None
        nbatch = 1
    else:
        b = np.ascontiguousarray(batch, dtype=np.int64)
        nbatch = int(b.max()) + 1 if n else 1
    home = np.ascontiguousarray(hash_home(vox, kind, K, S_div, bits), dtype=np.int64)
    ids = np.empty(n, dtype=np.int64)
    offs = np.empty(n, dtype=np.int64)
    counts = np.zeros(nbatch * (K + 1), dtype=np.int64)
    _lib().oracle_psh_assign(_ptr(vox), _ptr(home), _ptr(b), n, nbatch, K, S,
                             KINDS.index(kind), S_div, bits, int(strict), _ptr(offsets),
                             len(offsets), max_probes, _ptr(ids), _ptr(offs), _ptr(counts))
    return ids, offs, counts, exclusive_scan(counts)


def exclusive_scan(counts):
    """bucketing.py:169-179."""
    c = np.asarray(counts, dtype=np.int64)
    out = np.zeros(len(c), dtype=np.int64)
    if len(c) > 1:
        out[1:] = np.cumsum(c[:-1])
    return out


def dest_index(ids, offs, base, K, batch=None):
    """bucketing.py:96-101."""
    b = 0 if batch is None else np.asarray(batch, dtype=np.int64)
    return base[b * (K + 1) + ids] + offs


def bucket_table(counts, base, K, S, split_recycle=True):
    """bucketing.py:147-166 (single batch)."""
    starts = list(base[:K])
    lens = list(counts[:K])
    r, rb = int(counts[K]), int(base[K])
    if split_recycle:
        for j in range(0, r, S):
            starts.append(rb + j)
            lens.append(min(S, r - j))
    else:
        starts.append(rb)
        lens.append(r)
    return np.array(starts, dtype=np.int64), np.array(lens, dtype=np.int64)


# ------------------------------------------------------------------ schedule

def build_schedule(nb, W, stride=1, shift=0, rounds=1):
    """attention.py:84-117 — list (per round) of lists of bucket-id arrays."""
    out = []
    span = W * stride
    for t in range(rounds):
        rot = (np.arange(nb, dtype=np.int64) + (t * shift) % W) % nb
        scopes = []
        for s0 in range(0, nb, span):
            chunk = rot[s0:s0 + span]
            for lane in range(stride):
                sc = chunk[lane::stride]
                if len(sc):
                    scopes.append(sc)
        out.append(scopes)
    return out


def scope_ranges(table, scope):
    """attention.py:120-139 — [(start, stop)] of the non-empty members."""
    starts, lens = table
    return [(int(starts[b]), int(starts[b] + lens[b])) for b in scope if lens[b] > 0]


# ----------------------------------------------------------------- attention

def attention_dense(Q, K, V, n_heads):
    """attention.py:147-166 — per-head max-subtracted softmax in float64."""
    Q, K, V = (np.asarray(a, dtype=np.float64) for a in (Q, K, V))
    m, d = Q.shape
    dh = d // n_heads
    q = Q.reshape(m, n_heads, dh)
    k = K.reshape(K.shape[0], n_heads, dh)
    v = V.reshape(V.shape[0], n_heads, dh)
    s = np.einsum("qhd,khd->hqk", q, k) / math.sqrt(dh)
    s -= s.max(axis=-1, keepdims=True)
    w = np.exp(s)
    w /= w.sum(axis=-1, keepdims=True)
    return np.einsum("hqk,khd->qhd", w, v).reshape(m, d)


def attention_ranges(Q, K, V, n_heads, ranges, mask=None):
    """attention.py:188-268 semantics: rows of the ranges concatenated in range
    order; masked keys excluded; masked / starved query rows give zeros."""
    rows = np.concatenate([np.arange(a, b) for a, b in ranges]) if ranges else np.zeros(0, np.int64)
    if len(rows) == 0:
        return np.zeros((0, Q.shape[1]))
    valid = np.ones(len(rows), dtype=bool) if mask is None else np.asarray(mask, bool)[rows]
    out = np.zeros((len(rows), Q.shape[1]))
    if valid.any():
        kv = rows[valid]
        o = attention_dense(Q[rows], K[kv], V[kv], n_heads)
        out = o * valid[:, None]
    return out


# --------------------------------------------------------------------- stage

def positional_encoding(coords, d, base=10000.0):
    """attention.py:271-288 — d/3 dims per axis, alternating sin/cos."""
    c = np.asarray(coords, dtype=np.float64)
    npair = d // 6
    inv = base ** (-np.arange(npair) / npair)
    pe = np.empty((len(c), d))
    blk = 2 * npair
    for ax in range(3):
        ang = c[:, ax:ax + 1] * inv
        pe[:, ax * blk:(ax + 1) * blk:2] = np.sin(ang)
        pe[:, ax * blk + 1:(ax + 1) * blk:2] = np.cos(ang)
    return pe


def layer_norm(x, g, b, eps=1e-12):
    """stage.py:84-88 — population variance."""
    mu = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def gelu(x):
    """stage.py:91-92 — exact erf GELU."""
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x / np.sqrt(2.0)))


PARAM_ORDER = ("w_q", "w_k", "w_v", "w_o", "w_in", "w_out")


def init_params(seed, d, d_hidden=None, n_heads=4):
    """stage.py:57-81 — U(+-sqrt(3/fan_in)) drawn in the order q,k,v,o,in,out;
    zero biases, unit LN gains.  Returns a dict of float64 arrays."""
    if d_hidden is None:
        d_hidden = 4 * d
    g = np.random.default_rng(seed)
    shapes = {"w_q": (d, d), "w_k": (d, d), "w_v": (d, d), "w_o": (d, d),
              "w_in": (d, d_hidden), "w_out": (d_hidden, d)}
    p = {"n_heads": n_heads}
    for name in PARAM_ORDER:
        fi, fo = shapes[name]
        bound = np.sqrt(3.0 / fi)
        p[name] = g.uniform(-bound, bound, size=(fi, fo))
    for name in ("b_q", "b_k", "b_v", "b_o", "ln1_bias", "ln2_bias", "b_out"):
        p[name] = np.zeros(d)
    p["b_in"] = np.zeros(d_hidden)
    p["ln1_gain"] = np.ones(d)
    p["ln2_gain"] = np.ones(d)
    return p


def stage_forward(F, C, table, rounds, p, threads=1, scope_limit=None, timings=None):
    """stage.py:99-159 — pre-norm block per round over scattered rows.

    ``scope_limit`` (bench sampling only) runs attention on the first
    ``scope_limit`` scopes of each round and leaves the others' rows at zero.
    """
    F = np.array(F, dtype=np.float64, copy=True)
    C = np.asarray(C, dtype=np.float64)
    d = F.shape[1]
    H = p["n_heads"]
    lo = C.min(axis=0)
    ext = C.max(axis=0) - lo
    ext[ext == 0] = 1.0
    pe = positional_encoding((C - lo) / ext, d)
    import time
    for scopes in rounds:
        t0 = time.perf_counter()
        x = layer_norm(F, p["ln1_gain"], p["ln1_bias"]) + pe
        Q = x @ p["w_q"] + p["b_q"]
        K = x @ p["w_k"] + p["b_k"]
        V = x @ p["w_v"] + p["b_v"]
        att = np.zeros_like(F)
        todo = scopes if scope_limit is None else scopes[:scope_limit]

        def one(scope):
            rg = scope_ranges(table, scope)
            if not rg:
                return
            rows = np.concatenate([np.arange(a, b) for a, b in rg])
            att[rows] = attention_dense(Q[rows], K[rows], V[rows], H)

        t1 = time.perf_counter()
        if threads > 1:
            with ThreadPoolExecutor(max_workers=threads) as ex:
                list(ex.map(one, todo))
        else:
            for sc in todo:
                one(sc)
        t2 = time.perf_counter()
        F = F + att @ p["w_o"] + p["b_o"]
        h = layer_norm(F, p["ln2_gain"], p["ln2_bias"])
        F = F + gelu(h @ p["w_in"] + p["b_in"]) @ p["w_out"] + p["b_out"]
        if timings is not None:
            timings.append({"attn": t2 - t1, "rest": time.perf_counter() - t2 + (t1 - t0),
                            "ran": len(todo), "scopes": len(scopes)})
    return F


# ------------------------------------------------------------------- pooling

def tile_voxels(c, bits=10):
    """pooling.py:59-65 — (c-lo)/ext*2^bits, clipped to 2^bits-1, truncated."""
    lo = c.min(axis=0)
    ext = c.max(axis=0) - lo
    ext[ext == 0] = 1.0
    side = (1 << bits) - 1
    return np.minimum((c - lo) / ext * (side + 1), side).astype(np.int64)


def _norm3(diff):
    """np.linalg.norm(axis=1) for (m,3): sqrt((dx*dx + dy*dy) + dz*dz)."""
    return np.sqrt((diff[:, 0] * diff[:, 0] + diff[:, 1] * diff[:, 1]) + diff[:, 2] * diff[:, 2])


def subbuckets(c, rho):
    """pooling.py:68-163 — returns (sub_id, sizes, seeds) for one tile."""
    c = np.asarray(c, dtype=np.float64)
    m = len(c)
    target = -(-m // rho)
    key = morton(tile_voxels(c), 10) % target
    sub = np.full(m, -1, dtype=np.int64)
    sizes = np.zeros(target, dtype=np.int64)
    seeds = np.full(target, -1, dtype=np.int64)
    first = {}
    spill = []
    for i in range(m):                                   # step 1 (:82-102)
        k = int(key[i])
        j = first.get(k)
        if j is None:
            j = first[k] = len(first)
            seeds[j] = i
        if sizes[j] < rho:
            sub[i] = j
            sizes[j] += 1
        else:
            spill.append(i)
    nxt = len(first)
    n_first = nxt
    rest = []
    for i in spill:                                      # step 2 (:104-117)
        if nxt < target:
            seeds[nxt] = i
            sub[i] = nxt
            sizes[nxt] = 1
            nxt += 1
        else:
            rest.append(i)
    fresh = np.arange(n_first, target)
    for i in rest:                                       # step 3 (:119-139)
        cand = fresh[sizes[fresh] < rho]
        if len(cand) == 0:
            cand = np.flatnonzero(sizes < rho)
        dist = _norm3(c[seeds[cand]] - c[i])
        j = int(cand[np.argmin(dist)])
        sub[i] = j
        sizes[j] += 1
    while True:                                          # repair (:141-157)
        under = np.flatnonzero(sizes < rho)
        if len(under) <= 1:
            break
        tgt = int(under[np.argmax(sizes[under])])
        others = under[under != tgt]
        donor = int(others[np.argmin(sizes[others])])
        need = int(rho - sizes[tgt])
        mem = np.flatnonzero(sub == donor)
        dist = _norm3(c[mem] - c[seeds[tgt]])
        mv = mem[np.argsort(dist, kind="stable")[:need]]
        sub[mv] = tgt
        sizes[tgt] += len(mv)
        sizes[donor] -= len(mv)
    return sub, sizes, seeds


def pool_reduce(x, sub, sizes, reduce="mean"):
    """pooling.py:166-184 — members in index order, one row per sub-bucket."""
    x = np.asarray(x, dtype=np.float64)
    order = np.argsort(sub, kind="stable")
    bounds = exclusive_scan(sizes)
    g = x[order]
    if reduce == "sum":
        return np.add.reduceat(g, bounds, axis=0)
    if reduce == "mean":
        return np.add.reduceat(g, bounds, axis=0) / sizes[:, None]
    if reduce == "min":
        return np.minimum.reduceat(g, bounds, axis=0)
    return np.maximum.reduceat(g, bounds, axis=0)


def pool_stage(F, C, counts, base, K, S, nbatch, rho, reduce="mean"):
    """pooling.py:187-242 — returns (feats, coords, new_counts, new_S, sub_ids)
    where sub_ids[i] is the tile-local sub-bucket id of scattered row i."""
    F = np.asarray(F, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    nslots = nbatch * (K + 1)
    of, oc = [], []
    new_counts = np.zeros(nslots, dtype=np.int64)
    sub_all = np.zeros(len(F), dtype=np.int64)
    for slot in range(nslots):
        st, cnt = int(base[slot]), int(counts[slot])
        for t0 in range(0, cnt, POOL_TILE_CAP):
            lo, hi = st + t0, st + min(t0 + POOL_TILE_CAP, cnt)
            sub, sizes, _ = subbuckets(C[lo:hi], rho)
            sub_all[lo:hi] = sub
            of.append(pool_reduce(F[lo:hi], sub, sizes, reduce))
            oc.append(pool_reduce(C[lo:hi], sub, sizes, "mean"))
            new_counts[slot] += len(sizes)
    return (np.vstack(of), np.vstack(oc), new_counts, max(1, -(-S // rho)), sub_all)


# ------------------------------------------------------------------ backbone

def backbone_forward(coords, feats, stages, threads=1, scope_limit=None, timings=None,
                     record=None):
    """Composition of the restated ops in the order of
    paper_2412_16481_b200/backbone.py (voxelize -> remap -> PSH -> scatter ->
    stage_forward -> pool_stage, per stage).  ``stages`` is a sequence of
    objects with the StageConfig fields.  Returns (features, coords)."""
    import time
    C = np.asarray(coords, dtype=np.float64)
    X = np.asarray(feats, dtype=np.float64)
    for cfg in stages:
        t0 = time.perf_counter()
        vox = remap_nonnegative(voxelize(C, (0.0, 0.0, 0.0), cfg.voxel))
        ids, offs, counts, base = psh_assign(vox, None, cfg.kind, cfg.K, cfg.S, cfg.S_div)
        dest = dest_index(ids, offs, base, cfg.K)
        Xs = np.empty_like(X)
        Xs[dest] = X
        Cs = np.empty_like(C)
        Cs[dest] = C
        t1 = time.perf_counter()
        table = bucket_table(counts, base, cfg.K, cfg.S)
        rounds = build_schedule(len(table[0]), cfg.W, cfg.stride, cfg.shift, cfg.rounds)
        p = init_params(cfg.seed, cfg.d_model, n_heads=cfg.n_heads)
        st_t = []
        Xs = stage_forward(Xs, Cs, table, rounds, p, threads=threads, scope_limit=scope_limit,
                           timings=st_t)
        t2 = time.perf_counter()
        if cfg.pool_rho:
            X, C, pcounts, _, _ = pool_stage(Xs, Cs, counts, base, cfg.K, cfg.S, 1, cfg.pool_rho,
                                             "mean")
        else:
            X, C, pcounts = Xs, Cs, None
        t3 = time.perf_counter()
        if record is not None:
            # per-stage intermediates for the parity tests
            record.append({"ids": ids, "offs": offs, "counts": counts, "base": base,
                           "Cs": Cs, "F": Xs, "pooled_C": C if cfg.pool_rho else None,
                           "pooled_counts": pcounts})
        if timings is not None:
            nsc = sum(len(r) for r in rounds)
            # attention time extrapolated linearly in the scope count when sampled
            attn_x = sum(r["attn"] * r["scopes"] / max(1, r["ran"]) for r in st_t)
            rest = sum(r["rest"] for r in st_t)
            timings.append({"psh_scatter": t1 - t0, "stage": t2 - t1, "pool": t3 - t2,
                            "stage_extrapolated": attn_x + rest,
                            "scopes": nsc, "scopes_run": sum(r["ran"] for r in st_t),
                            "n": len(vox)})
    return X, C
