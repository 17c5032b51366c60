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


LAY = np.load(GOLD / "expect_layered.npz")


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_layered_index_matches_reference_files(tmp_path, name):
    """Kind-1 (FastHNSW) files written by the reference (dataset_io.py:174-245):
    read identically, written back byte for byte."""
    lg = pio.load_index(GOLD / f"hnsw_{name}.pgix")
    assert len(lg.layers) == int(LAY[f"{name}_nlayers"]) and lg.ep == int(LAY[f"{name}_ep"])
    assert lg.m_factor == float(LAY[f"{name}_m_factor"])
    np.testing.assert_array_equal(lg.levels, LAY[f"{name}_levels"])
    for i, layer in enumerate(lg.layers):
        np.testing.assert_array_equal(layer.members, LAY[f"{name}_L{i}_members"])
        np.testing.assert_array_equal(layer.graph.adj, LAY[f"{name}_L{i}_adj"])
        np.testing.assert_array_equal(layer.graph.counts, LAY[f"{name}_L{i}_counts"])
        np.testing.assert_array_equal(layer.graph.over_cap, LAY[f"{name}_L{i}_over"])
        assert layer.graph.ep == int(LAY[f"{name}_L{i}_ep"])
        assert layer.graph.M == int(LAY[f"{name}_L{i}_M"])
    pio.save_index(tmp_path / "h.pgix", lg)
    assert (tmp_path / "h.pgix").read_bytes() == (GOLD / f"hnsw_{name}.pgix").read_bytes()


def test_layered_index_corruption(tmp_path):
    good = (GOLD / "hnsw_cfg1.pgix").read_bytes()
    lg = pio.load_index(GOLD / "hnsw_cfg1.pgix")
    # header: magic 4, u32 version, u8 kind, u32 M, u64 n, u64 ep, f64 m, u32 layers
    hdr = 4 + 4 + 1 + 4
    top = len(lg.layers) - 1
    not_top = int(np.flatnonzero(lg.levels < top)[0])
    cases = {
        "truncated": good[:-1],
        "trailing": good + b"\0",
        "kind": good[:8] + bytes([7]) + good[9:],
        "no_layers": good[:hdr + 24] + struct.pack("<I", 0) + good[hdr + 28:],
        "ep_not_top": good[:hdr + 8] + struct.pack("<Q", not_top) + good[hdr + 16:],
    }
    for tag, blob in cases.items():
        p = tmp_path / f"{tag}.pgix"
        p.write_bytes(blob)
        with pytest.raises(pio.CorruptIndexError):
            pio.load_index(p)
    # members of layer 1 not ascending
    off = hdr + 28 + 8 + 4 * lg.n + 4
    body0 = lg.layers[0].graph
    o, nb = body0.to_csr()
    off += 8 + 8 + 4 + 4 * len(body0.over_cap) + 8 * (lg.n + 1) + 4 * len(nb)
    m1 = lg.layers[1].members
    assert struct.unpack("<Q", good[off:off + 8])[0] == len(m1) and len(m1) >= 2
    swapped = np.array(m1, "<i4")
    swapped[[0, 1]] = swapped[[1, 0]]
    p = tmp_path / "order.pgix"
    p.write_bytes(good[:off + 8] + swapped.tobytes() + good[off + 8 + 4 * len(m1):])
    with pytest.raises(pio.CorruptIndexError, match="ascending"):
        pio.load_index(p)
