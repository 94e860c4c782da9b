"""Reference text artifacts (bw/cli.py:29-121), byte for byte against files
written by the reference's own writers (tests/golden/make_artifacts_golden.py)."""
import os

import numpy as np
import pytest

from paper_2412_16481_b200 import artifacts as AR
from paper_2412_16481_b200.errors import EmptyInputError, ParseError

GOLD = os.path.join(os.path.dirname(__file__), "golden", "artifacts")


def _read(p):
    with open(p, "rb") as fh:
        return fh.read()


def test_features_and_coords_roundtrip_bytes(tmp_path):
    feats = np.random.default_rng(3).normal(size=(512, 6))
    AR.write_features_csv(tmp_path / "f.csv", feats)
    assert _read(tmp_path / "f.csv") == _read(os.path.join(GOLD, "features.csv"))
    back = AR.read_features_csv(tmp_path / "f.csv")
    assert np.array_equal(back, feats)                     # repr floats round-trip exactly
    coords = AR.read_coords_csv(os.path.join(GOLD, "coords.csv"))
    AR.write_coords_csv(tmp_path / "c.csv", coords)
    assert _read(tmp_path / "c.csv") == _read(os.path.join(GOLD, "coords.csv"))


def test_reader_errors(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("f0,f1\n1.0,abc\n")
    with pytest.raises(ParseError):
        AR.read_features_csv(p)
    p.write_text("f0,f1\n")
    with pytest.raises((EmptyInputError, ParseError)):
        AR.read_features_csv(p)
    p.write_text("x,y\n1.0,2.0\n")
    with pytest.raises(ParseError):
        AR.read_coords_csv(p)
    p.write_text("point,bucket_id\n")
    with pytest.raises(ParseError):
        AR.read_assignment_csv(p)


@pytest.mark.gpu
def test_assignment_csv_bytes_match_reference(tmp_path):
    import paper_2412_16481_b200 as F
    coords = AR.read_coords_csv(os.path.join(GOLD, "coords.csv"))
    vox = F.remap_nonnegative(F.voxelize(F.PointCloud(coords), F.VoxelGrid(1 / 16)))
    a = F.assign_buckets(vox, None, F.HashConfig("zorder-div", K=8, S_div=512), 128)
    AR.write_assignment_csv(tmp_path / "a.csv", a, "zorder-div")
    assert _read(tmp_path / "a.csv") == _read(os.path.join(GOLD, "assignment.csv"))
    b = AR.read_assignment_csv(os.path.join(GOLD, "assignment.csv"))
    assert np.array_equal(np.asarray(b.bucket_id), np.asarray(a.bucket_id))
    assert np.array_equal(np.asarray(b.bucket_offset), np.asarray(a.bucket_offset))
