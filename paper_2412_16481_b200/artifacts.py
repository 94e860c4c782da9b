"""Text artifacts of the reference demo flow:
features / coordinates CSV with ``repr`` floats and the assignment CSV
``point,bucket_id,bucket_offset,dest_index`` (bw/cli.py:29-121), byte for
byte.  Device tensors are read back once; the writers format on the host
(text formatting is host work by nature), the readers rebuild a
``BucketAssignment`` and validate it on the GPU like the reference does.
"""

import numpy as np
import torch

from .bucketing import BucketAssignment, compute_bucket_base
from .errors import ConfigError, EmptyInputError, IntegrityError, ParseError


def _host(a):
    if isinstance(a, torch.Tensor):
        return a.detach().cpu().numpy()
    return np.asarray(a)


def _fmt(x) -> str:
    return repr(float(x))                        # bw/cli.py:29-30


def write_features_csv(path, feats) -> None:
    """Header f0..f{d-1}, one row per point, repr floats (bw/cli.py:39-44)."""
    f = _host(feats)
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(",".join(f"f{j}" for j in range(f.shape[1])) + "\n")
        for row in f:
            fh.write(",".join(_fmt(v) for v in row) + "\n")


def read_features_csv(path) -> np.ndarray:
    """bw/cli.py:47-54: ParseError on malformed text, EmptyInputError on no rows."""
    try:
        arr = np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)
    except ValueError as exc:
        raise ParseError(f"{path}: {exc}") from None
    if arr.size == 0:
        raise EmptyInputError(f"{path}: no feature rows")
    return arr


def write_coords_csv(path, coords) -> None:
    """Header x,y,z (bw/cli.py:57-61)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("x,y,z\n")
        for row in _host(coords):
            fh.write(",".join(_fmt(v) for v in row) + "\n")


def read_coords_csv(path) -> np.ndarray:
    """bw/cli.py:64-68."""
    arr = read_features_csv(path)
    if arr.shape[1] != 3:
        raise ParseError(f"{path}: expected 3 columns, got {arr.shape[1]}")
    return arr


def write_assignment_csv(path, a: BucketAssignment, hash_kind: str) -> None:
    """'# K= S= batches= hash=' comment, column header, one row per point
    (bw/cli.py:71-78)."""
    ids = _host(a.bucket_id).astype(np.int64)
    offs = _host(a.bucket_offset).astype(np.int64)
    dest = _host(a.dest_index()).astype(np.int64)
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"# K={a.K} S={a.S} batches={a.num_batches} hash={hash_kind}\n")
        fh.write("point,bucket_id,bucket_offset,dest_index\n")
        fh.writelines(f"{i},{ids[i]},{offs[i]},{dest[i]}\n" for i in range(len(ids)))


def read_assignment_csv(path) -> BucketAssignment:
    """Parse and validate a single-batch assignment file (bw/cli.py:81-121)."""
    with open(path, "r", encoding="utf-8") as fh:
        header = fh.readline().strip()
        if not header.startswith("#"):
            raise ParseError(f"{path}:1: missing '# K=.. S=..' header comment")
        meta = {}
        for tok in header.lstrip("#").split():
            if "=" in tok:
                key, val = tok.split("=", 1)
                meta[key] = val
        try:
            K, S = int(meta["K"]), int(meta["S"])
            batches = int(meta.get("batches", "1"))
        except (KeyError, ValueError):
            raise ParseError(f"{path}:1: header must carry K= and S=") from None
        if batches != 1:
            raise ConfigError("only single-batch assignment files are supported here")
        cols = fh.readline().strip()
        if cols != "point,bucket_id,bucket_offset,dest_index":
            raise ParseError(f"{path}:2: unexpected column header {cols!r}")
        rows = []
        for lineno, line in enumerate(fh, start=3):
            if not line.strip():
                continue
            try:
                rows.append([int(v) for v in line.split(",")])
            except ValueError:
                raise ParseError(f"{path}:{lineno}: malformed row") from None
    if not rows:
        raise EmptyInputError(f"{path}: no assignment rows")
    arr = np.array(rows, dtype=np.int64)
    if not np.array_equal(arr[:, 0], np.arange(len(arr))):
        raise ParseError(f"{path}: point column must be 0..N-1 in order")
    counts = np.bincount(arr[:, 1], minlength=K + 1)
    a = BucketAssignment(bucket_id=arr[:, 1], bucket_offset=arr[:, 2], counts=counts,
                         bucket_base=compute_bucket_base(counts), S=S, K=K)
    a.validate()
    if not np.array_equal(_host(a.dest_index()), arr[:, 3]):
        raise IntegrityError(f"{path}: dest_index column disagrees with the map")
    return a
