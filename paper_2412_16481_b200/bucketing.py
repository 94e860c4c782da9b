"""Perfect spatial hashing (PSH) bucket assignment on the GPU.

Drop-in for bw/bucketing.py.  ``assign_buckets`` and
``assign_buckets_two_stage`` (which the reference proves bit-identical,
pkg/tests/test_bucketing.py:305-359) both run the exact parallel fixed point
of csrc/psh.cu in one cooperative launch and return the reference's
bucket ids, offsets, counts and bases bit for bit.  ``scatter`` packs rows
with csrc/rows.cu; ``gather`` is its inverse (pkg/tests/test_stage.py:165).

Array types follow the caller: host inputs give numpy int64 fields like the
reference; CUDA-tensor inputs give CUDA int64 tensors and never leave the
device.  The instrumented ``trace=`` path of the reference is pure Python and
is not offered on the GPU (ConfigError).
"""

import itertools
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .errors import ConfigError, EmptyInputError, IntegrityError, RangeError
from .hashing import HashConfig, check_hash_stats, dense_batch, hash_device

DEFAULT_MAX_PROBES = 32
DEFAULT_MAX_SWEEPS = 128


_ZERO_BATCH = {}


def _zero_batch_ids(n, device):
    """Single-batch ids for the backbone's internal assignments: one cached
    int64 zero vector per (size, device), so an assignment built inside a
    captured graph adds no fill kernel (the backbone never writes it; public
    assignments keep a private zeros tensor)."""
    key = (int(n), str(device))
    z = _ZERO_BATCH.get(key)
    if z is None:
        z = _ZERO_BATCH[key] = torch.zeros(int(n), dtype=torch.int64, device=device)
    return z


@dataclass(frozen=True)
class ProbeSchedule:
    """Probe offsets, nearest shell first (bw/bucketing.py:28-48)."""

    offsets: np.ndarray
    max_probes: int = DEFAULT_MAX_PROBES
    seed: int = None

    def __post_init__(self):
        arr = np.asarray(self.offsets, dtype=np.int64)
        if arr.ndim != 2 or arr.shape[1] != 3 or arr.shape[0] == 0:
            raise ConfigError(f"offsets must be a non-empty (P, 3) array, got {arr.shape}")
        if (np.abs(arr).max(axis=1) == 0).any():
            raise ConfigError("probe offsets must exclude (0, 0, 0)")
        if self.max_probes < 1:
            raise ConfigError(f"max_probes must be >= 1, got {self.max_probes}")
        object.__setattr__(self, "offsets", arr)

    def device_table(self):
        """(P, 3) int8 host table cut to min(max_probes, len), for the kernel."""
        P = min(self.max_probes, len(self.offsets))
        if P > 128:
            raise ConfigError("the GPU probe table holds at most 128 offsets")
        cut = self.offsets[:P]
        if np.abs(cut).max() > 127:
            raise ConfigError("GPU probe offsets must fit in int8")
        return np.ascontiguousarray(cut.astype(np.int8)), P


def default_probe_schedule(seed=None, max_probes: int = DEFAULT_MAX_PROBES) -> ProbeSchedule:
    """26 radius-1 then 98 radius-2 L-inf offsets, lexicographic; each shell
    shuffled with default_rng(seed) when seeded (bw/bucketing.py:51-66)."""
    shell1 = [d for d in itertools.product((-1, 0, 1), repeat=3) if d != (0, 0, 0)]
    shell2 = [d for d in itertools.product(range(-2, 3), repeat=3) if max(abs(c) for c in d) == 2]
    if seed is not None:
        rng = np.random.default_rng(seed)
        rng.shuffle(shell1)
        rng.shuffle(shell2)
    return ProbeSchedule(np.array(shell1 + shell2, dtype=np.int64), max_probes=max_probes, seed=seed)


_INTEGRITY_MSGS = (
    (1, "counts do not sum to the point count"),
    (2, "a non-recycle bucket exceeds capacity S"),
    (4, "negative bucket count"),
    (8, "bucket_base is not the exclusive prefix sum of counts"),
    (16, "bucket_id outside [0, K]"),
    (32, "bucket_offset outside [0, count)"),
    (64, "destination map is not a bijection onto [0, N)"),
)


def _to_np(x):
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


@dataclass
class BucketAssignment:
    """Result of PSH bucketing (bw/bucketing.py:69-166).

    Public fields hold int64 arrays of the caller's type.  Assignments made by
    this package also carry int32 device mirrors (``_dev``) that downstream
    kernels use without re-uploading; user-built ones are converted on use.
    """

    bucket_id: object
    bucket_offset: object
    counts: object
    bucket_base: object
    S: int
    K: int
    batch_id: object = field(default=None)
    num_batches: int = 1
    _dev: dict = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if self.batch_id is None:
            if isinstance(self.bucket_id, torch.Tensor):
                self.batch_id = torch.zeros_like(self.bucket_id, dtype=torch.int64)
            else:
                self.batch_id = np.zeros(len(self.bucket_id), dtype=np.int64)

    # -------------------------------------------------------------- helpers
    @property
    def on_device(self) -> bool:
        return isinstance(self.bucket_id, torch.Tensor) and self.bucket_id.is_cuda

    def _mirrors(self):
        """int32 device copies of (id, offset, counts, base, batch, dest?)."""
        if self._dev is not None:
            return self._dev
        return {
            "id": L.to_dev(self.bucket_id, torch.int32),
            "off": L.to_dev(self.bucket_offset, torch.int32),
            "counts": L.to_dev(self.counts, torch.int32),
            "base": L.to_dev(self.bucket_base, torch.int32),
            "batch": L.to_dev(self.batch_id, torch.int32) if self.num_batches > 1 else None,
            "dest": None,
        }

    def to_host(self) -> "BucketAssignment":
        """Public fields as numpy int64 (device mirrors kept)."""
        for name in ("bucket_id", "bucket_offset", "counts", "bucket_base", "batch_id"):
            v = getattr(self, name)
            if isinstance(v, torch.Tensor):
                setattr(self, name, v.detach().cpu().numpy())
        return self

    def _wrap(self, t):
        return t if self.on_device else t.cpu().numpy()

    def __len__(self) -> int:
        return len(self.bucket_id)

    def slot_id(self):
        """Global counter slot per point: batch * (K + 1) + local id."""
        return self.batch_id * (self.K + 1) + self.bucket_id

    def dest_index(self):
        m = self._mirrors()
        if m.get("dest") is not None:
            return self._wrap(m["dest"].to(torch.int64))
        slot = m["id"].to(torch.int64)
        if m["batch"] is not None:
            slot = slot + m["batch"].to(torch.int64) * (self.K + 1)
        return self._wrap(m["base"].to(torch.int64)[slot] + m["off"].to(torch.int64))

    def dest_device(self) -> torch.Tensor:
        """int32 destination rows on the device (kernel input)."""
        m = self._mirrors()
        if m.get("dest") is None:
            m["dest"] = L.to_dev(self.dest_index(), torch.int32)
        return m["dest"]

    def recycle_fraction(self) -> float:
        n = len(self)
        if n == 0:
            return 0.0
        if self.on_device:
            return float(int((self.bucket_id == self.K).sum())) / n
        return float(np.count_nonzero(np.asarray(self.bucket_id) == self.K)) / n

    def counts_of_batch(self, batch: int):
        if not 0 <= batch < self.num_batches:
            raise ConfigError(f"batch {batch} out of range")
        w = self.K + 1
        return self.counts[batch * w:(batch + 1) * w]

    def validate(self) -> None:
        """Raise IntegrityError unless every structural invariant holds
        (bw/bucketing.py:116-145), checked by f3d_validate_assignment."""
        n = len(self)
        nslots = self.num_batches * (self.K + 1)
        if tuple(self.counts.shape) != (nslots,) or tuple(self.bucket_base.shape) != (nslots,):
            raise IntegrityError("counts/bucket_base have the wrong shape")
        self._dev_validate(self._mirrors_fresh())

    def _mirrors_fresh(self):
        self_dev, self._dev = self._dev, None
        try:
            return self._mirrors()
        finally:
            self._dev = self_dev

    def _dev_validate(self, m, sync=True):
        n = len(self)
        flags = L.empty((1,), torch.int32)
        ws = L.empty((max(1, n),), torch.int32)
        L.call("f3d_validate_assignment", L.ptr(m["id"]), L.ptr(m["off"]), L.ptr(m["batch"]),
               L.ptr(m["counts"]), L.ptr(m["base"]), n, self.num_batches, self.K, self.S,
               L.ptr(flags), L.ptr(ws), L.stream())
        if sync:
            raise_integrity(int(flags.item()), n)
        return flags

    def bucket_table(self, split_recycle: bool = True):
        """(starts, lengths) of each contiguous bucket range in the scattered
        layout (bw/bucketing.py:147-166); single batch only."""
        if self.num_batches != 1:
            raise ConfigError("bucket_table requires a single-batch assignment")
        counts = _to_np(self.counts).astype(np.int64)
        base = _to_np(self.bucket_base).astype(np.int64)
        K, S = self.K, self.S
        starts = list(base[:K])
        lengths = list(counts[:K])
        r = int(counts[K])
        b0 = int(base[K])
        if split_recycle:
            for j in range(0, r, S):
                starts.append(b0 + j)
                lengths.append(min(S, r - j))
        else:
            starts.append(b0)
            lengths.append(r)
        st = np.array(starts, dtype=np.int64)
        ln = np.array(lengths, dtype=np.int64)
        if self.on_device:
            return torch.from_numpy(st).to(self.bucket_id.device), torch.from_numpy(ln).to(
                self.bucket_id.device)
        return st, ln


def raise_integrity(flags: int, n: int) -> None:
    for bit, msg in _INTEGRITY_MSGS:
        if bit >= 16 and n == 0:
            return
        if flags & bit:
            raise IntegrityError(msg)


def compute_bucket_base(counts):
    """Exclusive prefix sum; same length as counts (bw/bucketing.py:169-179)."""
    host = L.is_host(counts)
    c = L.to_dev(counts, torch.int64)
    if c.ndim != 1:
        raise ConfigError("counts must be 1-D")
    if c.numel() and bool((c < 0).any()):
        raise ConfigError("counts must be non-negative")
    base = torch.zeros_like(c)
    if c.numel() > 1:
        base[1:] = torch.cumsum(c[:-1], 0)
    return L.out(base, host)


# ------------------------------------------------------------ assignment

def _prepare(voxels, batch_id, cfg: HashConfig, S: int):
    """Validation in the reference's order (bw/bucketing.py:242-263)."""
    v = L.to_dev(voxels, torch.int64)
    if v.ndim != 2 or v.shape[1] != 3:
        raise ConfigError(f"voxels must have shape (N, 3), got {tuple(v.shape)}")
    n = v.shape[0]
    if n == 0:
        raise EmptyInputError("assign_buckets needs at least one point")
    home, vox32, stats_d = hash_device(v, cfg, want_vox32=True)
    b32, nb = None, 1
    if batch_id is not None:
        b = L.to_dev(batch_id, torch.int64)
        bstats = torch.stack([b.min(), b.max()]) if tuple(b.shape) == (n,) else None
    stats = stats_d.cpu().tolist()
    if min(stats[0:3]) < 0:
        raise RangeError("voxels must be non-negative; remap them first")
    if S < 1:
        raise ConfigError(f"S must be >= 1, got {S}")
    if batch_id is not None:
        if bstats is None:
            raise ConfigError("batch_id must have shape (N,)")
        lo, hi = bstats.cpu().tolist()
        nb = hi + 1
        if lo < 0 or bool((torch.bincount(b, minlength=nb) == 0).any()):
            raise ConfigError("batch ids must be contiguous from 0")
        if nb > 1:
            b32 = b.to(torch.int32)
    check_hash_stats(stats, cfg, n)
    return vox32, home, b32, nb, n


def _run_psh(vox32, home, b32, nb, n, cfg: HashConfig, S: int, probes: ProbeSchedule,
             max_sweeps: int = DEFAULT_MAX_SWEEPS, n_dev=None):
    """Launch f3d_psh_assign; returns int32 device (id, off, counts, base, dest, info).
    n_dev: optional device point count <= n (sync-free pipelines)."""
    table, P = probes.device_table()
    W = cfg.K + 1
    ids = L.empty((n,), torch.int32)
    offs = L.empty((n,), torch.int32)
    counts = L.empty((nb * W,), torch.int32)
    base = L.empty((nb * W,), torch.int32)
    dest = L.empty((n,), torch.int32)
    info = L.empty((4,), torch.int32)
    ws_bytes = L.load().f3d_psh_workspace_size(n, nb, cfg.K)
    ws = L.empty((ws_bytes,), torch.uint8)
    L.call("f3d_psh_assign", L.ptr(vox32), L.ptr(home), L.ptr(b32), n, nb, cfg.K, S,
           cfg.kind_code, cfg.S_div, cfg.bits_per_axis, int(cfg.div_overflow == "error"),
           table.ctypes.data_as(L._P), P, max_sweeps, L.ptr(ids), L.ptr(offs), L.ptr(counts),
           L.ptr(base), L.ptr(dest), L.ptr(info), L.ptr(ws), ws_bytes, L.ptr(n_dev), L.stream())
    return ids, offs, counts, base, dest, info


def _assign(voxels, batch_id, cfg, S, probes, max_sweeps=DEFAULT_MAX_SWEEPS):
    host = L.is_host(voxels)
    if probes is None:
        probes = default_probe_schedule()
    vox32, home, b32, nb, n = _prepare(voxels, batch_id, cfg, S)
    ids, offs, counts, base, dest, info = _run_psh(vox32, home, b32, nb, n, cfg, S, probes,
                                                   max_sweeps)
    if b32 is None:
        batch64 = torch.zeros(n, dtype=torch.int64, device=ids.device)
    else:
        batch64 = b32.to(torch.int64)
    a = BucketAssignment(
        bucket_id=ids.to(torch.int64), bucket_offset=offs.to(torch.int64),
        counts=counts.to(torch.int64), bucket_base=base.to(torch.int64), S=S, K=cfg.K,
        batch_id=batch64, num_batches=nb,
        _dev={"id": ids, "off": offs, "counts": counts, "base": base, "batch": b32, "dest": dest,
              "info": info})
    flags = a._dev_validate(a._dev, sync=False)   # _finish -> validate (bw/bucketing.py:266-272)
    raise_integrity(int(flags.item()), n)
    if host:
        a.bucket_id = a.bucket_id.cpu().numpy()
        a.bucket_offset = a.bucket_offset.cpu().numpy()
        a.counts = a.counts.cpu().numpy()
        a.bucket_base = a.bucket_base.cpu().numpy()
        a.batch_id = a.batch_id.cpu().numpy()
    return a


def assign_buckets(voxels, batch_id, cfg: HashConfig, S: int, probes: ProbeSchedule = None,
                   trace=None) -> BucketAssignment:
    """One-stage assignment: direct claim, probe, recycle — the reference's
    sequential semantics, computed in parallel (bw/bucketing.py:275-320)."""
    if trace is not None:
        raise ConfigError("trace= selects the reference's instrumented pure-Python path; "
                          "it is not available on the GPU")
    return _assign(voxels, batch_id, cfg, S, probes)


def assign_buckets_two_stage(voxels, batch_id, cfg: HashConfig, S: int,
                             probes: ProbeSchedule = None, block_size: int = 1024,
                             threads: int = 1) -> BucketAssignment:
    """Two-stage entry point (bw/bucketing.py:323-382).  Its result is
    identical to assign_buckets for every block size and thread count, so it
    runs the same kernel; block_size is validated, threads is ignored."""
    if block_size < 1:
        raise ConfigError(f"block_size must be >= 1, got {block_size}")
    return _assign(voxels, batch_id, cfg, S, probes)


# ------------------------------------------------- claim protocol helpers

def claim_slot(counters, bucket: int, capacity: int, trace=None):
    """Increment-then-verify claim on one counter (bw/bucketing.py:182-200):
    the pre-increment value is the claimed offset, valid only when it was
    below capacity; otherwise the increment is rolled back and None returned.
    ``counters`` is the caller's host array, mutated in place like the
    reference's; this is the single-counter protocol step the PSH kernel
    restates in bulk (csrc/psh.cu), not a hot-path entry point."""
    prev = int(counters[bucket])
    counters[bucket] += 1
    if prev < capacity:
        if trace is not None:
            trace.append(("claim", bucket, prev))
        return prev
    counters[bucket] -= 1
    if trace is not None:
        trace.append(("full", bucket, prev))
    return None


def _probe_candidates(v, cfg: HashConfig, probes: ProbeSchedule):
    """Hashes of the clamped probe voxels of one point, computed on the GPU in
    one launch; -1 where a strict '-div' quotient leaves [0, K)
    (bw/_kernels.py:34-37, 52-58)."""
    P = min(probes.max_probes, len(probes.offsets))
    vmax = (1 << cfg.bits_per_axis) - 1
    cand = np.clip(np.asarray(v, dtype=np.int64)[None, :3] + probes.offsets[:P], 0, vmax)
    pts = torch.as_tensor(cand, dtype=torch.int64).to(L.device())
    wrap = HashConfig(cfg.kind, K=cfg.K, S_div=cfg.S_div, bits_per_axis=cfg.bits_per_axis)
    home, _, _ = hash_device(pts, wrap)
    h = home.to(torch.int64).cpu().numpy()
    if cfg.div_overflow == "error" and cfg.kind.endswith("-div"):
        if cfg.kind.startswith("zorder"):
            from .hashing import morton_encode
            code = np.asarray(morton_encode(pts, cfg.bits_per_axis).cpu().numpy())
        else:
            code = cand[:, 0] ^ cand[:, 1] ^ cand[:, 2]
        h = np.where(code // cfg.S_div >= cfg.K, -1, h)
    return h


def optimistic_race(i: int, v, counters, S: int, cfg: HashConfig, probes: ProbeSchedule,
                    trace=None):
    """Rebalance one point whose home bucket is full (bw/bucketing.py:203-239):
    probes nearest first, each claimed with increment / validate / rollback
    (claim_slot), else the unbounded recycle bucket K.  Returns (bucket,
    offset) and mutates the caller's host ``counters``.  The candidate hashes
    come from the GPU hash kernel in one launch."""
    cands = _probe_candidates(v, cfg, probes)
    for p, h in enumerate(cands):
        h = int(h)
        if h < 0:
            if trace is not None:
                trace.append((i, "probe", p, -1, "skipped"))
            continue
        if counters[h] < S:
            off = claim_slot(counters, h, S)
            if off is not None:
                if trace is not None:
                    trace.append((i, "probe", p, h, "claimed"))
                return h, off
        if trace is not None:
            trace.append((i, "probe", p, h, "full"))
    off = int(counters[cfg.K])
    counters[cfg.K] += 1
    if trace is not None:
        trace.append((i, "recycle", len(cands), cfg.K, "claimed"))
    return cfg.K, off


# ------------------------------------------------------------ row movement

def _rows(features):
    host = L.is_host(features)
    if isinstance(features, torch.Tensor):
        f = features.to(L.device()).contiguous()
    else:
        arr = np.asarray(features)
        if arr.dtype == object:
            raise ConfigError("features must be a numeric array")
        f = torch.from_numpy(np.ascontiguousarray(arr)).to(L.device())
    return f, host


def _row_bytes(f):
    return (f.numel() // max(1, f.shape[0])) * f.element_size() if f.ndim else 0


def scatter(features, assignment: BucketAssignment):
    """Pack rows by bucket: row i moves to dest_index()[i]
    (bw/bucketing.py:385-401).  Returns (scattered, perm)."""
    f, host = _rows(features)
    if f.shape[0] != len(assignment):
        raise ConfigError(
            f"features rows ({f.shape[0]}) != assignment size ({len(assignment)})")
    assignment.validate()          # always, as bw/bucketing.py:397
    dest = assignment.dest_device()
    out = torch.empty_like(f)
    rb = _row_bytes(f)
    if f.shape[0] and rb % 4 == 0:
        L.call("f3d_scatter_rows", L.ptr(f), L.ptr(dest), f.shape[0], rb, L.ptr(out), None,
               L.stream())
    elif f.shape[0]:
        raise ConfigError("row size must be a multiple of 4 bytes on the GPU")
    perm = dest.to(torch.int64)
    return L.out(out, host), L.out(perm, host)


def gather(scattered, assignment: BucketAssignment):
    """Inverse of scatter: out[i] = scattered[dest_index()[i]]."""
    f, host = _rows(scattered)
    if f.shape[0] != len(assignment):
        raise ConfigError("rows do not match the assignment size")
    dest = assignment.dest_device()
    out = torch.empty_like(f)
    rb = _row_bytes(f)
    if f.shape[0]:
        L.call("f3d_gather_rows", L.ptr(f), L.ptr(dest), f.shape[0], rb, L.ptr(out), None,
               L.stream())
    return L.out(out, host)
