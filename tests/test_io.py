"""CPU: vector-file and PGIX index formats against files written by the
reference's own dataset_io (tests/golden/io): our loader
reads them identically, our writer reproduces them byte for byte, and
corrupt files raise CorruptIndexError / ValueError like the reference."""
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_2410_01231_b200 import ProximityGraph
from paper_2410_01231_b200 import io as pio

GOLD = Path(__file__).resolve().parent / "golden" / "io"
EXP = np.load(GOLD / "expect.npz")


@pytest.mark.parametrize("name,key", [("f.fvecs", "f"), ("i.ivecs", "i"), ("b.bvecs", "b")])
def test_vecs_match_reference_files(tmp_path, name, key):
    arr = pio.load_vecs(GOLD / name)
    np.testing.assert_array_equal(arr, EXP[key])
    assert arr.dtype == EXP[key].dtype
    pio.save_vecs(tmp_path / name, EXP[key])
    assert (tmp_path / name).read_bytes() == (GOLD / name).read_bytes()


@pytest.mark.parametrize("name", ["cfg1_2k", "blobs"])
def test_index_matches_reference_files(tmp_path, name):
    g = pio.load_index(GOLD / f"{name}.pgix")
    np.testing.assert_array_equal(g.adj, EXP[f"{name}_adj"])
    np.testing.assert_array_equal(g.counts, EXP[f"{name}_counts"])
    np.testing.assert_array_equal(g.over_cap, EXP[f"{name}_over"])
    assert g.ep == int(EXP[f"{name}_ep"]) and g.M == int(EXP[f"{name}_M"])
    pio.save_index(tmp_path / "x.pgix", g)
    assert (tmp_path / "x.pgix").read_bytes() == (GOLD / f"{name}.pgix").read_bytes()


def test_corrupt_and_bad_files(tmp_path):
    good = (GOLD / "cfg1_2k.pgix").read_bytes()
    cases = {
        "magic": b"XXXX" + good[4:],
        "truncated": good[:-3],
        "trailing": good + b"\0",
        "version": good[:4] + struct.pack("<I", 2) + good[8:],
    }
    for tag, blob in cases.items():
        p = tmp_path / f"{tag}.pgix"
        p.write_bytes(blob)
        with pytest.raises(pio.CorruptIndexError):
            pio.load_index(p)
    # a node above M without an over-cap tag
    g = ProximityGraph(adj=np.array([[1, 2], [0, -1], [0, -1]], np.int32),
                       counts=np.array([2, 1, 1], np.int32), M=1, ep=0)
    pio.save_index(tmp_path / "over.pgix", g)
    with pytest.raises(pio.CorruptIndexError, match="exceeds M"):
        pio.load_index(tmp_path / "over.pgix")
    (tmp_path / "e.fvecs").write_bytes(b"")
    with pytest.raises(ValueError, match="empty"):
        pio.load_vecs(tmp_path / "e.fvecs")
    (tmp_path / "x.txt").write_bytes(b"1234")
    with pytest.raises(ValueError, match="unknown vector extension"):
        pio.load_vecs(tmp_path / "x.txt")
    blob = (GOLD / "f.fvecs").read_bytes()
    (tmp_path / "t.fvecs").write_bytes(blob[:-1])
    with pytest.raises(ValueError, match="record size"):
        pio.load_vecs(tmp_path / "t.fvecs")
