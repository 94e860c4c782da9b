"""Voxel-to-bucket hashes and Morton encoding on the GPU.

Drop-in for bw/hashing.py: same names, defaults, validation and exception
messages; the arithmetic runs in libf3d (csrc/hash.cu).  Host inputs
(numpy / lists) come back as numpy int64, CUDA tensors stay on the device.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .errors import ConfigError, RangeError

HASH_KINDS = ("xor-mod", "xor-div", "zorder-mod", "zorder-div")

_AXES = ("x", "y", "z")


@dataclass(frozen=True)
class HashConfig:
    """Parameters shared by every bucket hash (bw/hashing.py:28-57)."""

    kind: str
    K: int
    S_div: int = 8
    bits_per_axis: int = 10
    div_overflow: str = "wrap"

    def __post_init__(self):
        if self.kind not in HASH_KINDS:
            raise ConfigError(f"unknown hash kind {self.kind!r}; expected one of {HASH_KINDS}")
        if self.K < 1:
            raise ConfigError(f"K must be >= 1, got {self.K}")
        if self.S_div < 1:
            raise ConfigError(f"S_div must be >= 1, got {self.S_div}")
        if not 1 <= self.bits_per_axis <= 21:
            raise ConfigError(f"bits_per_axis must be in [1, 21], got {self.bits_per_axis}")
        if self.div_overflow not in ("wrap", "error"):
            raise ConfigError(f"div_overflow must be 'wrap' or 'error', got {self.div_overflow!r}")
        if self.K >= 2 ** 31 - 1:
            raise ConfigError("K must fit in int32 on the device")

    @property
    def kind_code(self) -> int:
        return HASH_KINDS.index(self.kind)


def raise_range(stats, bits: int) -> None:
    """Reproduce bw/hashing.py:60-75 from the device min/max statistics:
    the first axis in x, y, z order with a violation, negative first."""
    limit = 1 << bits
    for axis in range(3):
        lo, hi = int(stats[axis]), int(stats[3 + axis])
        if lo < 0:
            raise RangeError(
                f"{_AXES[axis]} component {lo} is negative; remap voxels to non-negative first")
        if hi >= limit:
            raise RangeError(f"{_AXES[axis]} component {hi} does not fit in {bits} bits")


def _as_points(v):
    """(..., 3) int64 device tensor flattened to (n, 3), plus the lead shape."""
    host = L.is_host(v)
    t = L.to_dev(v, torch.int64)
    if t.ndim == 0 or t.shape[-1] != 3:
        raise ConfigError(f"expected last dimension 3, got shape {tuple(t.shape)}")
    lead = tuple(t.shape[:-1])
    return t.reshape(-1, 3).contiguous(), lead, host


def morton_encode(v, bits_per_axis: int = 10):
    """Interleave (x, y, z) as ``z_k y_k x_k`` (bw/hashing.py:78-98)."""
    if not 1 <= bits_per_axis <= 21:
        raise ConfigError(f"bits_per_axis must be in [1, 21], got {bits_per_axis}")
    pts, lead, host = _as_points(v)
    n = pts.shape[0]
    codes = L.empty((n,), torch.int64)
    stats = L.empty((7,), torch.int64)
    L.call("f3d_morton_encode", L.ptr(pts), n, bits_per_axis, L.ptr(codes), L.ptr(stats), L.stream())
    if n:
        raise_range(stats.cpu().tolist(), bits_per_axis)
    codes = codes.reshape(lead)
    if len(lead) == 0:
        return int(codes.item())
    return L.out(codes, host)


def hash_device(pts: torch.Tensor, cfg: HashConfig, want_vox32: bool = False):
    """(n,3) int64 device voxels -> (home int32, vox32 int32 | None, stats).
    stats is a 7-vector on the host: axis min/max and the max div quotient."""
    n = pts.shape[0]
    home = L.empty((n,), torch.int32)
    vox32 = L.empty((n, 3), torch.int32) if want_vox32 else None
    stats = L.empty((7,), torch.int64)
    L.call("f3d_hash_bucket", L.ptr(pts), n, cfg.kind_code, cfg.K, cfg.S_div, cfg.bits_per_axis,
           L.ptr(home), L.ptr(vox32), L.ptr(stats), L.stream())
    return home, vox32, stats


def check_hash_stats(stats, cfg: HashConfig, n: int) -> None:
    """Range check then the strict quotient check (bw/hashing.py:111-122)."""
    if n == 0:
        return
    raise_range(stats, cfg.bits_per_axis)
    if cfg.kind.endswith("-div") and cfg.div_overflow == "error" and int(stats[6]) >= cfg.K:
        raise RangeError(
            f"hash quotient {int(stats[6])} exceeds K-1={cfg.K - 1}; "
            "increase S_div or use div_overflow='wrap'")


def hash_bucket(v, cfg: HashConfig):
    """Bucket ids in [0, K) under cfg (bw/hashing.py:101-125)."""
    pts, lead, host = _as_points(v)
    home, _, stats = hash_device(pts, cfg)
    check_hash_stats(stats.cpu().tolist(), cfg, pts.shape[0])
    out = home.to(torch.int64).reshape(lead)
    if len(lead) == 0:
        return int(out.item())
    return L.out(out, host)


def dense_batch(batch: torch.Tensor):
    """Arbitrary integer batch labels -> dense int32 ids in [0, B) (sorted
    label order, as np.unique in the reference) and B."""
    uniq, inv = torch.unique(batch, sorted=True, return_inverse=True)
    return inv.to(torch.int32).contiguous(), int(uniq.numel())


def remap_nonnegative(voxels, batch_id=None):
    """Shift voxels so each batch's per-axis minimum is zero
    (bw/hashing.py:128-149)."""
    host = L.is_host(voxels)
    v = L.to_dev(voxels, torch.int64)
    if v.ndim != 2 or v.shape[1] != 3:
        raise ConfigError(f"expected voxels of shape (N, 3), got {tuple(v.shape)}")
    n = v.shape[0]
    if n == 0:
        return L.out(v.clone(), host)
    b32, nb = None, 1
    if batch_id is not None:
        b = L.to_dev(batch_id, torch.int64)
        if tuple(b.shape) != (n,):
            raise ConfigError("batch_id must have shape (N,)")
        b32, nb = dense_batch(b)
    out = L.empty((n, 3), torch.int64)
    ws = L.empty((3 * nb,), torch.int64)
    L.call("f3d_remap_nonnegative", L.ptr(v), L.ptr(b32), n, nb, L.ptr(out), L.ptr(ws), L.stream())
    return L.out(out, host)
