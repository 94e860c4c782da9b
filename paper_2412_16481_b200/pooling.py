"""In-bucket pooling on the GPU.

Drop-in for bw/pooling.py.  ``build_subbuckets`` / ``pool_stage`` run the
one-warp-per-tile partition kernel of csrc/pool.cu (bit-identical sub-bucket
ids, sizes and seeds, float64 distances without contraction) and
``pool_features`` the member-ordered reduce (sequential in index order, so
float64 centroids match the reference bit for bit).
"""

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .bucketing import BucketAssignment
from .errors import ConfigError, EmptyInputError, IntegrityError

TILE_CAP = 1024
REDUCES = ("sum", "mean", "min", "max")
_OP = {"sum": 0, "mean": 1, "min": 2, "max": 3}
_FLAG_MSGS = ((1, "sub-bucket allocation fell short of the target"),
              (2, "step 3 found no under-filled sub-bucket"),
              (4, "a sub-bucket exceeds capacity rho"),
              (8, "empty sub-bucket"),
              (16, "more than one under-filled sub-bucket"),
              (32, "sub-bucket id out of range"))


def _raise_flags(f: int):
    for bit, msg in _FLAG_MSGS:
        if f & bit:
            raise IntegrityError(msg)


@dataclass
class SubBucketAssignment:
    """Partition of one tile (bw/pooling.py:26-56)."""

    subbucket_id: np.ndarray
    rho: int
    num_subbuckets: int
    sizes: np.ndarray
    seeds: np.ndarray
    scan_passes: int = 0
    _members: object = field(default=None, repr=False, compare=False)

    def validate(self) -> None:
        sid = np.asarray(self.subbucket_id.cpu() if isinstance(self.subbucket_id, torch.Tensor)
                         else self.subbucket_id)
        sizes = np.asarray(self.sizes.cpu() if isinstance(self.sizes, torch.Tensor) else self.sizes)
        m = len(sid)
        if sizes.shape != (self.num_subbuckets,):
            raise IntegrityError("sizes shape mismatch")
        if int(sizes.sum()) != m:
            raise IntegrityError("sub-bucket sizes do not sum to the tile size")
        counted = np.bincount(sid, minlength=self.num_subbuckets)
        if not np.array_equal(counted, sizes):
            raise IntegrityError("sizes disagree with subbucket_id")
        if (sizes > self.rho).any():
            raise IntegrityError("a sub-bucket exceeds capacity rho")
        if (sizes < 1).any():
            raise IntegrityError("empty sub-bucket")
        if int((sizes < self.rho).sum()) > 1:
            raise IntegrityError("more than one under-filled sub-bucket")


class TilePlan:
    """<=1024-row tiles of every non-empty slot in scatter order, with the
    first pooled row of each tile (bw/pooling.py:211-225)."""

    def __init__(self, counts, base, rho, dev):
        counts = np.asarray(counts, dtype=np.int64)
        base = np.asarray(base, dtype=np.int64)
        reps = -(-counts // TILE_CAP)
        slot_of_tile = np.repeat(np.arange(len(counts)), reps)
        first_tile = np.cumsum(reps) - reps
        k = np.arange(len(slot_of_tile)) - np.repeat(first_tile, reps)
        starts = base[slot_of_tile] + k * TILE_CAP
        m = np.minimum(TILE_CAP, counts[slot_of_tile] - k * TILE_CAP)
        targets = -(-m // rho)
        out = np.cumsum(targets) - targets
        self.ntiles = len(m)
        self.npool = int(targets.sum())
        self.slot_of_tile = slot_of_tile
        self.targets = targets
        self.new_counts = np.bincount(slot_of_tile, weights=targets, minlength=len(counts)).astype(np.int64)
        up = L.upload({"tile_start": starts if self.ntiles else [0],
                       "tile_m": m if self.ntiles else [0],
                       "tile_out": out if self.ntiles else [0]})
        self.tile_start = up["tile_start"]
        self.tile_m = up["tile_m"]
        self.tile_out = up["tile_out"]


class DeviceTilePlan:
    """TilePlan built on the device by f3d_plan_pool from the PSH counts/base;
    only the totals (tile and pooled-row counts, needed for allocation) are
    computed on the host from the counts already read back."""

    def __init__(self, counts_h, counts_dev, base_dev, rho):
        c = np.asarray(counts_h, dtype=np.int64)
        full, rem = c // TILE_CAP, c % TILE_CAP
        self.ntiles = int((-(-c // TILE_CAP)).sum())
        self.npool = int((full * (-(-TILE_CAP // rho)) + (-(-rem // rho))).sum())
        buf = L.empty((3 * max(1, self.ntiles) + 2,), torch.int32)
        k = max(1, self.ntiles)
        self.tile_start, self.tile_m, self.tile_out = buf[:k], buf[k:2 * k], buf[2 * k:3 * k]
        self.totals = buf[3 * k:]
        L.call("f3d_plan_pool", L.ptr(counts_dev), L.ptr(base_dev), len(c), TILE_CAP, rho,
               L.ptr(self.tile_start), L.ptr(self.tile_m), L.ptr(self.tile_out),
               L.ptr(self.totals), L.stream())


def _build(coords_dev, plan: TilePlan, rho: int, want_sub=False, want_seeds=False,
           ntiles_dev=None):
    n = coords_dev.shape[0]
    members = L.empty((max(1, plan.npool), rho), torch.int32)
    sizes = L.empty((max(1, plan.npool),), torch.int32)
    seeds = L.empty((max(1, plan.npool),), torch.int32) if want_seeds else None
    sub = L.empty((max(1, n),), torch.int32) if want_sub else None
    passes = L.empty((max(1, plan.ntiles),), torch.int32) if want_seeds else None
    flags = L.empty((1,), torch.int32)
    L.call("f3d_pool_build", L.ptr(coords_dev), L.ptr(plan.tile_start), L.ptr(plan.tile_m),
           L.ptr(plan.tile_out), plan.ntiles, rho, L.ptr(sub), L.ptr(members), L.ptr(sizes),
           L.ptr(seeds), L.ptr(passes), L.ptr(flags), L.ptr(ntiles_dev), L.stream())
    return members, sizes, seeds, sub, passes, flags


def _reduce(x, members, sizes, npool, rho, reduce, npool_dev=None, out=None):
    if x.dtype == torch.float64:
        dt = 2
    elif x.dtype == torch.float32:
        dt = 1
    elif x.dtype == torch.bfloat16:
        dt = 0
    else:
        x = x.to(torch.float64)
        dt = 2
    x = x.contiguous()
    if out is None:
        out = torch.empty((npool, x.shape[1]), dtype=x.dtype, device=x.device)
    L.call("f3d_pool_reduce", L.ptr(x), dt, x.stride(0), x.shape[1], L.ptr(members),
           L.ptr(sizes), npool, rho, _OP[reduce], L.ptr(out), out.stride(0), L.ptr(npool_dev),
           L.stream())
    return out


def build_subbuckets(coords, rho: int) -> SubBucketAssignment:
    """Partition one tile of m <= 1024 points into ceil(m / rho) sub-buckets
    (bw/pooling.py:68-163)."""
    host = L.is_host(coords)
    c = L.to_dev(coords, torch.float64)
    if c.ndim != 2 or c.shape[1] != 3:
        raise ConfigError(f"coords must be (m, 3), got {tuple(c.shape)}")
    m = c.shape[0]
    if m == 0:
        raise EmptyInputError("build_subbuckets needs at least one point")
    if m > TILE_CAP:
        raise ConfigError(f"tile holds {m} points; the cap is {TILE_CAP}")
    if rho < 1:
        raise ConfigError(f"rho must be >= 1, got {rho}")
    if rho > 64:
        raise ConfigError("the GPU partition kernel supports rho <= 64")
    plan = TilePlan([m], [0], rho, c.device)
    members, sizes, seeds, sub, passes, flags = _build(c.contiguous(), plan, rho, True, True)
    _raise_flags(int(flags.item()))
    target = plan.npool
    res = SubBucketAssignment(
        subbucket_id=L.out(sub[:m].to(torch.int64), host), rho=rho, num_subbuckets=target,
        sizes=L.out(sizes[:target].to(torch.int64), host),
        seeds=L.out(seeds[:target].to(torch.int64), host), scan_passes=int(passes[0].item()),
        _members=(members, sizes))
    return res


def pool_features(features, sub: SubBucketAssignment, reduce: str = "mean"):
    """Reduce each sub-bucket's rows to one row, in sub-bucket id order
    (bw/pooling.py:166-184)."""
    if reduce not in REDUCES:
        raise ConfigError(f"reduce must be one of {REDUCES}, got {reduce!r}")
    host = L.is_host(features)
    x = L.to_dev(features, torch.float64) if host else features.to(L.device())
    if x.ndim == 1:
        x = x[:, None]
    if x.shape[0] != len(sub.subbucket_id):
        raise ConfigError("features rows do not match the sub-bucket assignment")
    sub.validate()
    if sub._members is not None:
        members, sizes = sub._members
    else:
        sid = np.asarray(sub.subbucket_id.cpu() if isinstance(sub.subbucket_id, torch.Tensor)
                         else sub.subbucket_id, dtype=np.int64)
        order = np.argsort(sid, kind="stable")
        sz = np.bincount(sid, minlength=sub.num_subbuckets)
        mem = np.full((sub.num_subbuckets, sub.rho), -1, dtype=np.int32)
        pos = np.arange(len(sid)) - np.repeat(np.cumsum(sz) - sz, sz)
        mem[sid[order], pos] = order
        members = L.to_dev(mem, torch.int32)
        sizes = L.to_dev(sz, torch.int32)
    out = _reduce(x, members, sizes, sub.num_subbuckets, sub.rho, reduce)
    return L.out(out, host)


def pool_stage(features, coords, assignment: BucketAssignment, rho: int, reduce: str = "mean"):
    """Pool every bucket slot by rho (bw/pooling.py:187-242).  Returns
    (pooled_features, pooled_coords, new_assignment)."""
    host = L.is_host(features)
    if isinstance(features, torch.Tensor):
        x = features.to(L.device())
    else:
        x = L.to_dev(np.asarray(features, dtype=np.float64), torch.float64)
    C = L.to_dev(coords, torch.float64).contiguous()
    if x.shape[0] != len(assignment) or tuple(C.shape) != (x.shape[0], 3):
        raise ConfigError("features/coords must match the assignment size")
    if rho < 1:
        raise ConfigError(f"rho must be >= 1, got {rho}")
    if rho > 64:
        raise ConfigError("the GPU partition kernel supports rho <= 64")
    if reduce not in REDUCES:
        raise ConfigError(f"reduce must be one of {REDUCES}, got {reduce!r}")
    K, S = assignment.K, assignment.S
    m = assignment._mirrors()
    counts = m["counts"].cpu().numpy().astype(np.int64)
    base = m["base"].cpu().numpy().astype(np.int64)
    res = pool_device(x, C, counts, base, K, S, assignment.num_batches, rho, reduce)
    pf, pc, na = res
    if host:
        return pf.cpu().numpy(), pc.cpu().numpy(), na.to_host()
    return pf, pc, na


def pool_device(x, C, counts, base, K, S, nbatch, rho, reduce, check=True, assignment=True,
                dev_counts=None, want_parent=False):
    """Device path of pool_stage given host counts/base; returns device
    tensors and (optionally) a device-resident BucketAssignment.
    dev_counts = (counts_dev, base_dev) builds the tile table on the device."""
    if dev_counts is not None:
        plan = DeviceTilePlan(counts, dev_counts[0], dev_counts[1], rho)
    else:
        plan = TilePlan(counts, base, rho, x.device)
    members, sizes, _, _, _, flags = _build(C, plan, rho)
    if check:
        _raise_flags(int(flags.item()))
    pf = _reduce(x, members, sizes, plan.npool, rho, reduce)
    pc = _reduce(C, members, sizes, plan.npool, rho, "mean")
    na = None
    if assignment:
        if not hasattr(plan, "new_counts"):
            plan = TilePlan(counts, base, rho, x.device)
        na = new_assignment(plan.new_counts, K, max(1, math.ceil(S / rho)), nbatch, x.device)
    if want_parent:
        parent = L.empty((max(1, C.shape[0]),), torch.int32)
        L.call("f3d_pool_parent", L.ptr(members), L.ptr(sizes), plan.npool, rho, L.ptr(parent),
               None, L.stream())
        return pf, pc, na, parent[:C.shape[0]]
    return pf, pc, na


def pool_stage_map(features, coords, assignment: BucketAssignment, rho: int,
                   reduce: str = "mean"):
    """pool_stage plus the pooling map: parent[i] = pooled row of scattered
    row i (the input of ``unpool``).  Returns
    (pooled_features, pooled_coords, new_assignment, parent int64)."""
    host = L.is_host(features)
    x = features.to(L.device()) if isinstance(features, torch.Tensor) else \
        L.to_dev(np.asarray(features, dtype=np.float64), torch.float64)
    C = L.to_dev(coords, torch.float64).contiguous()
    if x.shape[0] != len(assignment) or tuple(C.shape) != (x.shape[0], 3):
        raise ConfigError("features/coords must match the assignment size")
    if rho < 1 or rho > 64:
        raise ConfigError(f"rho must be in [1, 64] on the GPU, got {rho}")
    if reduce not in REDUCES:
        raise ConfigError(f"reduce must be one of {REDUCES}, got {reduce!r}")
    m = assignment._mirrors()
    counts = m["counts"].cpu().numpy().astype(np.int64)
    base = m["base"].cpu().numpy().astype(np.int64)
    pf, pc, na, parent = pool_device(x, C, counts, base, assignment.K, assignment.S,
                                     assignment.num_batches, rho, reduce, want_parent=True)
    parent = parent.to(torch.int64)
    if host:
        return pf.cpu().numpy(), pc.cpu().numpy(), na.to_host(), parent.cpu().numpy()
    return pf, pc, na, parent


def unpool(pooled, parent):
    """Unpooling of a pooled level back onto its finer rows: out[i] =
    pooled[parent[i]] (f3d_gather_rows).  The reference has no unpooling
    (SPEC.md:488); this is the builder-defined inverse of pool_stage's map."""
    host = L.is_host(pooled)
    p = pooled.to(L.device()) if isinstance(pooled, torch.Tensor) else \
        L.to_dev(np.asarray(pooled), torch.float64)
    if p.ndim == 1:
        p = p[:, None]
    p = p.contiguous()
    idx = L.to_dev(parent, torch.int32)
    n = idx.shape[0]
    if n and (int(idx.min()) < 0 or int(idx.max()) >= p.shape[0]):
        raise ConfigError("parent indices outside the pooled rows")
    out = torch.empty((n, p.shape[1]), dtype=p.dtype, device=p.device)
    rb = p.shape[1] * p.element_size()
    if rb % 4:
        raise ConfigError("row size must be a multiple of 4 bytes on the GPU")
    if n:
        L.call("f3d_gather_rows", L.ptr(p), L.ptr(idx), n, rb, L.ptr(out), None, L.stream())
    return L.out(out, host)


def new_assignment(new_counts, K, S_new, nbatch, dev) -> BucketAssignment:
    """Assignment of the pooled rows: bucket identity kept, offsets 0..c-1 in
    slot order, so the pooled rows are already in scattered order."""
    new_counts = np.asarray(new_counts, dtype=np.int64)
    nslots = len(new_counts)
    slots_h = np.repeat(np.arange(nslots), new_counts)
    base_h = np.cumsum(new_counts) - new_counts
    npool = int(new_counts.sum())
    offs_h = np.arange(npool) - base_h[slots_h]
    up = L.upload({"counts": new_counts, "base": base_h, "bid": slots_h % (K + 1),
                   "bat": slots_h // (K + 1), "off": offs_h, "dest": np.arange(npool)})
    nc, base = up["counts"].to(torch.int64), up["base"].to(torch.int64)
    bid, bat, offs = up["bid"].to(torch.int64), up["bat"].to(torch.int64), up["off"].to(torch.int64)
    a = BucketAssignment(bucket_id=bid, bucket_offset=offs, counts=nc, bucket_base=base, S=S_new,
                         K=K, batch_id=bat, num_batches=nbatch,
                         _dev={"id": up["bid"], "off": up["off"], "counts": up["counts"],
                               "base": up["base"], "batch": up["bat"] if nbatch > 1 else None,
                               "dest": up["dest"]})
    return a
