"""Point clouds, voxel grids and GPU voxelization.

Drop-in for the hot-path part of bw/geometry.py: ``PointCloud``,
``VoxelGrid``, ``voxelize`` (csrc/hash.cu, IEEE f64 subtract + divide, then
floor) and the deterministic ``synth_cloud`` used to build benchmark inputs
(host-side input generation, bit-identical to the reference's PCG64 draws).
Text file I/O (load_xyz / load_ply / write_xyz) is out of scope.
"""

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .errors import ConfigError, EmptyInputError

SYNTH_DISTS = ("uniform-box", "gaussian-clusters", "surface-shell")


@dataclass
class PointCloud:
    """Float64 coordinates plus an int64 batch id per point
    (bw/geometry.py:13-52).  Host inputs become numpy float64; CUDA tensors
    stay on the device."""

    coords: object
    batch_id: object = field(default=None)

    def __post_init__(self):
        if isinstance(self.coords, torch.Tensor) and self.coords.is_cuda:
            self.coords = self.coords.to(torch.float64).contiguous()
            n = self.coords.shape[0] if self.coords.ndim == 2 else -1
            if self.coords.ndim != 2 or self.coords.shape[1] != 3:
                raise ConfigError(f"coords must have shape (N, 3), got {tuple(self.coords.shape)}")
            if self.batch_id is None:
                self.batch_id = torch.zeros(n, dtype=torch.int64, device=self.coords.device)
            else:
                self.batch_id = L.to_dev(self.batch_id, torch.int64)
            if tuple(self.batch_id.shape) != (n,):
                raise ConfigError("batch_id must have shape (N,)")
            if n:
                uniq = torch.unique(self.batch_id)
                if int(uniq[0]) != 0 or int(uniq[-1]) != len(uniq) - 1:
                    raise ConfigError(f"batch ids must be contiguous from 0, got {uniq.tolist()}")
            return
        self.coords = np.asarray(self.coords, dtype=np.float64)
        if self.coords.ndim != 2 or self.coords.shape[1] != 3:
            raise ConfigError(f"coords must have shape (N, 3), got {self.coords.shape}")
        if self.batch_id is None:
            self.batch_id = np.zeros(len(self.coords), dtype=np.int64)
        else:
            self.batch_id = np.asarray(self.batch_id, dtype=np.int64)
        if self.batch_id.shape != (len(self.coords),):
            raise ConfigError("batch_id must have shape (N,)")
        if len(self.coords):
            uniq = np.unique(self.batch_id)
            if uniq[0] != 0 or not np.array_equal(uniq, np.arange(len(uniq))):
                raise ConfigError(f"batch ids must be contiguous from 0, got {uniq.tolist()}")

    def __len__(self) -> int:
        return len(self.coords)

    @property
    def num_batches(self) -> int:
        if not len(self.coords):
            return 0
        return int(self.batch_id.max()) + 1


@dataclass(frozen=True)
class VoxelGrid:
    """Uniform grid: voxel v holds points with floor((p - origin)/size) == v."""

    voxel_size: float
    origin: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if not (self.voxel_size > 0 and math.isfinite(self.voxel_size)):
            raise ConfigError(f"voxel_size must be positive and finite, got {self.voxel_size}")
        if len(self.origin) != 3:
            raise ConfigError("origin must have 3 components")


def voxelize(cloud: PointCloud, grid: VoxelGrid):
    """Integer voxel coordinates (N, 3) int64, floor convention
    (bw/geometry.py:69-72), computed by f3d_voxelize."""
    host = L.is_host(cloud.coords)
    c = L.to_dev(cloud.coords, torch.float64)
    n = c.shape[0]
    out = L.empty((n, 3), torch.int64)
    org = (L._F64 * 3)(*[float(o) for o in grid.origin])
    L.call("f3d_voxelize", L.ptr(c), n, org, float(grid.voxel_size), L.ptr(out), L.stream())
    return L.out(out, host)


def synth_cloud(seed: int, n: int, dist: str = "uniform-box") -> PointCloud:
    """Deterministic synthetic cloud (bw/geometry.py:183-212); same PCG64
    draw order, so the reference sees bit-identical inputs."""
    if dist not in SYNTH_DISTS:
        raise ConfigError(f"unknown dist {dist!r}; expected one of {SYNTH_DISTS}")
    if n < 1:
        raise EmptyInputError(f"synth_cloud needs n >= 1, got {n}")
    rng = np.random.default_rng(seed)
    if dist == "uniform-box":
        pts = rng.random((n, 3))
    elif dist == "gaussian-clusters":
        centers = np.array([[0.2, 0.2, 0.2], [0.8, 0.8, 0.2], [0.2, 0.8, 0.8], [0.8, 0.2, 0.8]])
        which = rng.integers(0, 4, size=n)
        pts = centers[which] + rng.normal(0.0, 0.03, size=(n, 3))
    else:
        dirs = rng.normal(size=(n, 3))
        norms = np.linalg.norm(dirs, axis=1, keepdims=True)
        norms[norms == 0] = 1.0
        radius = 0.4 + rng.normal(0.0, 0.005, size=(n, 1))
        pts = 0.5 + dirs / norms * radius
    return PointCloud(pts)
