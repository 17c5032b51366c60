"""GPU parity for SURVEY 8(f) f3 -- NN-Descent, the classic and the
self-iterative (FastNSG) NSG builders and the layer-global FastHNSW -- against
the reference's own outputs (tests/golden/f3.npz, make_golden.py f3), on a
float (cfg1) and an exact-integer (cfg2) prefix.  Exact: rows, flags, the
per-round accepted-update counts (they drive the early stop), entry points,
adjacency, layer assignments and layered-search results."""
from pathlib import Path

import numpy as np
import pytest

from paper_2410_01231_b200 import Dataset
from paper_2410_01231_b200 import hnsw, knng, nsg

pytestmark = pytest.mark.gpu

G = np.load(Path(__file__).resolve().parent / "golden" / "f3.npz", allow_pickle=False)
NAMES = [str(x) for x in G["names"]]


def _live_equal(adj, counts, ref_adj, ref_counts, tag):
    np.testing.assert_array_equal(counts, ref_counts, err_msg=tag)
    live = np.arange(adj.shape[1])[None, :] < counts[:, None]
    assert adj.shape == ref_adj.shape, tag
    np.testing.assert_array_equal(np.where(live, adj, -1), np.where(live, ref_adj, -1),
                                  err_msg=tag)


@pytest.mark.parametrize("name", NAMES)
def test_nn_descent_rounds_match_reference(name):
    ds = Dataset.from_array(G[f"{name}_data"])
    st = knng.knng_init_random(ds, 16, seed=5)
    np.testing.assert_array_equal(st.ids, G[f"{name}_knng0_ids"])
    np.testing.assert_array_equal(st.dists, G[f"{name}_knng0_dists"])
    for r in range(1, 4):
        st = knng.knng_descent_iterate(ds, st, rho=1.0 if r != 2 else 0.5)
        np.testing.assert_array_equal(st.ids, G[f"{name}_knng{r}_ids"], err_msg=f"round {r}")
        np.testing.assert_array_equal(st.dists, G[f"{name}_knng{r}_dists"])
        np.testing.assert_array_equal(st.flags, G[f"{name}_knng{r}_flags"])
        assert st.last_updates == int(G[f"{name}_knng{r}_upd"]), r
    kb = knng.build_knng(ds, 12, iters=10, seed=7)
    assert kb.iterations == int(G[f"{name}_bknng_iters"])
    np.testing.assert_array_equal(kb.ids, G[f"{name}_bknng_ids"])


@pytest.mark.parametrize("name", NAMES)
def test_nsg_builders_match_reference(name):
    ds = Dataset.from_array(G[f"{name}_data"])
    g = nsg.build_nsg_original(ds, k0=12, k=24, L=32, M=12, seed=3)
    assert g.ep == int(G[f"{name}_nsg_ep"])
    _live_equal(g.adj, g.counts, G[f"{name}_nsg_adj"], G[f"{name}_nsg_counts"], "nsg")
    st = nsg.FastNsgStats()
    g = nsg.build_fastnsg(ds, k0=12, k=24, L=32, M=12, alpha=66.0, max_iters=2, seed=4,
                          stats=st)
    assert g.ep == int(G[f"{name}_fnsg_ep"])
    _live_equal(g.adj, g.counts, G[f"{name}_fnsg_adj"], G[f"{name}_fnsg_counts"], "fastnsg")
    np.testing.assert_array_equal(g.over_cap, G[f"{name}_fnsg_over"])
    fs = st.final_state
    np.testing.assert_array_equal(fs.counts, G[f"{name}_fnsg_state_counts"])
    np.testing.assert_array_equal(fs.ids, G[f"{name}_fnsg_state_ids"])
    np.testing.assert_array_equal(fs.fresh, G[f"{name}_fnsg_state_fresh"])


@pytest.mark.parametrize("name", NAMES)
def test_fasthnsw_and_layered_search_match_reference(name):
    ds = Dataset.from_array(G[f"{name}_data"])
    lg = hnsw.build_fasthnsw(ds, k0=12, ef=40, M=12, seed=6)
    np.testing.assert_array_equal(lg.levels, G[f"{name}_hnsw_levels"])
    assert lg.ep == int(G[f"{name}_hnsw_ep"])
    assert len(lg.layers) == int(G[f"{name}_hnsw_nlayers"])
    for i, layer in enumerate(lg.layers):
        np.testing.assert_array_equal(layer.members, G[f"{name}_hnsw_L{i}_members"])
        assert layer.graph.ep == int(G[f"{name}_hnsw_L{i}_ep"])
        _live_equal(layer.graph.adj, layer.graph.counts, G[f"{name}_hnsw_L{i}_adj"],
                    G[f"{name}_hnsw_L{i}_counts"], f"layer {i}")
    for j, q in enumerate(G[f"{name}_lq"]):
        ids, dists = hnsw.layered_search(ds, lg, q, 10, 40)
        m = len(ids)
        np.testing.assert_array_equal(ids, G[f"{name}_lq_ids"][j, :m])
        np.testing.assert_array_equal(dists, G[f"{name}_lq_dists"][j, :m])


@pytest.mark.parametrize("name", NAMES)
def test_gpu_fasthnsw_saves_the_reference_file(tmp_path, name):
    """The GPU-built hierarchy written as a layered PGIX index (kind 1) is the
    file the reference's dataset_io writes for its own build, byte for byte
    (tests/golden/io/hnsw_*.pgix), and loads back to the same layers."""
    from paper_2410_01231_b200 import io as pio
    ds = Dataset.from_array(G[f"{name}_data"])
    lg = hnsw.build_fasthnsw(ds, k0=12, ef=40, M=12, seed=6)
    ref = Path(__file__).resolve().parent / "golden" / "io" / f"hnsw_{name}.pgix"
    pio.save_index(tmp_path / "g.pgix", lg)
    assert (tmp_path / "g.pgix").read_bytes() == ref.read_bytes()
    back = pio.load_index(tmp_path / "g.pgix")
    assert back.ep == lg.ep and len(back.layers) == len(lg.layers)
    np.testing.assert_array_equal(back.levels, lg.levels)


C5 = Path(__file__).resolve().parent / "golden" / "cfg5.npz"


@pytest.mark.slow
def test_cfg5_full_size_fasthnsw_matches_reference():
    """BASELINE config 5 at its full size (200k x 128, config-2 recipe seed 4;
    k0=32, ef=200, M=32 on every layer -- SURVEY A.1 --, alpha 66): levels,
    entry point and every layer's adjacency equal the reference's own build
    (upper layers in full, layer 0 by CSR digest + 2,000 seeded rows), and the
    layered search over the 10,000 seeded queries returns the reference's ids
    at L=100 and its recall@10 at L = 50, 100, 200 (edge agreement 100 %,
    recall difference 0)."""
    import hashlib

    from paper_2410_01231_b200 import ground_truth_table, mean_recall, synth
    g = np.load(C5)
    base, q = synth.cfg5(200_000, 10_000)
    ds = Dataset.from_array(base)
    lg = hnsw.build_fasthnsw(ds, k0=32, ef=200, M=32, alpha=66.0, seed=4)
    np.testing.assert_array_equal(lg.levels, g["levels"].astype(np.int32))
    assert lg.ep == int(g["ep"]) and len(lg.layers) == int(g["nlayers"])
    dig = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    for i, layer in enumerate(lg.layers):
        off, nb = layer.graph.to_csr()
        assert dig(off.astype(np.int64)) + dig(nb.astype(np.int32)) == str(g[f"L{i}_csr_sha"]), i
        assert layer.graph.ep == int(g[f"L{i}_ep"])
        np.testing.assert_array_equal(layer.graph.over_cap, g[f"L{i}_over"])
        if i > 0:
            np.testing.assert_array_equal(layer.members, g[f"L{i}_members"])
            _live_equal(layer.graph.adj, layer.graph.counts, g[f"L{i}_adj"], g[f"L{i}_counts"],
                        f"layer {i}")
    rows = g["L0_rows"]
    a0 = lg.layers[0].graph
    np.testing.assert_array_equal(a0.counts, g["L0_counts"].astype(np.int32))
    ref_rows, mine = g["L0_rows_adj"], a0.adj[rows]
    W = max(ref_rows.shape[1], mine.shape[1])
    pad = lambda a, c: np.where(np.arange(W)[None, :] < c[:, None],  # noqa: E731
                                np.pad(a, ((0, 0), (0, W - a.shape[1])), constant_values=-1), -1)
    np.testing.assert_array_equal(pad(mine, a0.counts[rows]), pad(ref_rows, a0.counts[rows]))
    truth = ground_truth_table(ds, q, k=10)
    for L in (50, 100, 200):
        ids, _, _ = hnsw.layered_search_batch(ds, lg, q, 10, L)
        if L == 100:
            np.testing.assert_array_equal(ids, g["search_ids_L100"])
        assert mean_recall(ids, truth, 10) == pytest.approx(float(g[f"recall_L{L}"]), abs=1e-12)
