"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container only (the reference is not present on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src:. \
        python tests/golden/make_golden.py

It imports the read-only reference package ``pgann`` and records, for a set of
seeded inputs, the outputs of the hot-path composition the reference's own
tests use:

  * ``oracle.ground_truth_table(ds, None, k=K, exclude_self=True)`` (oracle.py:31-65)
  * fp32 list distances ``_kernels.squared_l2`` (_kernels.py:17-24) re-sorted by
    (fp32 dist, id) with ``_kernels.sort_pairs`` (_kernels.py:298-324)
  * ``prune.prune_all`` (prune.py:109-126) = phase A, and
    ``prune.add_reverse_and_prune`` (prune.py:129-151) = phase B,
    for strategy "rng" and "alpha" (66 degrees).

Large arrays are stored as sha256 digests plus a seeded row sample, small ones
in full.  The fixtures are what pins ``oracle/`` (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from numba import njit, prange  # noqa: E402

from pgann import _kernels  # noqa: E402  (reference)
from pgann.core import Dataset  # noqa: E402
from pgann.oracle import ground_truth_table  # noqa: E402
from pgann.prune import (PruneParams, add_reverse_and_prune, entry_point,  # noqa: E402
                         finish_refine, prune_all)
from pgann.graph import ProximityGraph, reachable_from  # noqa: E402
from pgann.search import kann_search, search_batch  # noqa: E402

from paper_2410_01231_b200 import synth  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@njit(parallel=True, cache=True)
def _list_dists(data, ids):
    n, k = ids.shape
    out = np.empty((n, k), np.float32)
    for u in prange(n):
        for j in range(k):
            out[u, j] = _kernels.squared_l2(data[ids[u, j]], data[u])
    return out


@njit(cache=True)
def _resort(ids, dists):
    for u in range(ids.shape[0]):
        _kernels.sort_pairs(ids[u], dists[u], ids.shape[1])


def reference_composition(data: np.ndarray, K: int, R: int):
    """Reference hot path: exact pool -> fp32 list dists -> phases A, B."""
    ds = Dataset.from_array(data)
    n = ds.n
    truth = ground_truth_table(ds, None, k=K, exclude_self=True)
    ids = truth.astype(np.int32).copy()
    dists = _list_dists(ds.data, ids)
    _resort(ids, dists)
    off = (np.arange(n + 1, dtype=np.int64) * K)
    cnt = np.full(n, K, np.int32)
    out = dict(truth=truth, pool_ids=ids, pool_dists=dists)
    for tag, params in (("rng", PruneParams(M=R, strategy="rng")),
                        ("a66", PruneParams(M=R, alpha=66.0, strategy="alpha"))):
        a_ids, a_d, a_c, a_de, a_ae = prune_all(ds, off, cnt, ids.ravel(),
                                                dists.ravel(), params)
        b_ids, b_d, b_c, b_de, b_ae = add_reverse_and_prune(ds, a_ids, a_d, a_c, params)
        out.update({f"{tag}_a_ids": a_ids, f"{tag}_a_dists": a_d, f"{tag}_a_counts": a_c,
                    f"{tag}_a_de": np.int64(a_de), f"{tag}_a_ae": np.int64(a_ae),
                    f"{tag}_b_ids": b_ids, f"{tag}_b_dists": b_d, f"{tag}_b_counts": b_c,
                    f"{tag}_b_de": np.int64(b_de), f"{tag}_b_ae": np.int64(b_ae)})
    return out


def save_config(name: str, data: np.ndarray, K: int, R: int, meta: dict,
                full: bool) -> None:
    res = reference_composition(data, K, R)
    rec = {"meta_" + k: np.asarray(v) for k, v in meta.items()}
    rec["data_digest"] = np.asarray(digest(data))
    rng = np.random.default_rng(1234)
    sample = np.sort(rng.choice(data.shape[0], size=min(256, data.shape[0]), replace=False))
    rec["sample_rows"] = sample.astype(np.int64)
    for k, v in res.items():
        v = np.asarray(v)
        if v.ndim == 0:
            rec[k] = v
            continue
        rec[k + "__sha256"] = np.asarray(digest(v))
        rec[k + "__sample"] = v[sample]
        if full:
            rec[k] = v
    np.savez_compressed(HERE / f"{name}.npz", **rec)
    print(name, {k: int(res[k]) for k in res if np.asarray(res[k]).ndim == 0})


# ---------------------------------------------------------------------------
# Edge cases taken from the reference's own prune tests (test_prune.py,
# test_acceptance.py c01): CSR candidate lists that are NOT exact-kNN pools,
# variable lengths, empty rows, self entries, duplicates and exact ties.
# ---------------------------------------------------------------------------

def _candidate_list(data, u, size, rng, allow_self=False):
    n = data.shape[0]
    others = np.array([v for v in range(n) if allow_self or v != u])
    size = min(size, len(others))
    pick = rng.choice(others, size=size, replace=False) if size else np.empty(0, int)
    dists = np.array([_kernels.squared_l2(data[v], data[u]) for v in pick], np.float32)
    order = np.lexsort((pick, dists))
    return pick[order].astype(np.int32), dists[order]


def csr_case(data, rng, max_len, allow_self, empty_frac=0.1):
    n = data.shape[0]
    lists = []
    for u in range(n):
        L = 0 if rng.random() < empty_frac else int(rng.integers(1, max_len + 1))
        lists.append(_candidate_list(data, u, L, rng, allow_self))
    counts = np.array([len(i) for i, _ in lists], np.int32)
    # leave slack between slices: offsets need not be dense (prune_batch reads
    # cand_counts[u] entries from cand_off[u])
    slack = rng.integers(0, 3, size=n)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(counts + slack, out=off[1:])
    ids = np.full(int(off[-1]), -7, np.int32)
    dists = np.full(int(off[-1]), np.nan, np.float32)
    for u, (i, d) in enumerate(lists):
        ids[off[u]:off[u] + len(i)] = i
        dists[off[u]:off[u] + len(i)] = d
    return off, counts, ids, dists


def save_cases() -> None:
    rec = {}
    rng = np.random.default_rng(2024)
    specs = [
        # (name, data, max_len, allow_self, M, alpha)
        ("unif", rng.random((200, 6)).astype(np.float32), 40, False, 12, 66.0),
        ("unif_self", rng.random((150, 4)).astype(np.float32), 30, True, 7, 90.0),
        ("lattice", np.stack(np.meshgrid(np.arange(12), np.arange(12)), -1)
         .reshape(-1, 2).astype(np.float32), 30, False, 6, 120.0),
        ("dups", np.repeat(rng.integers(0, 5, size=(40, 3)).astype(np.float32), 3, axis=0),
         25, False, 5, 150.0),
        ("gauss_d33", rng.standard_normal((120, 33)).astype(np.float32), 64, False, 24, 66.0),
        ("m1", rng.random((80, 5)).astype(np.float32), 20, False, 1, 70.0),
    ]
    names = []
    for name, data, max_len, allow_self, M, alpha in specs:
        ds = Dataset.from_array(data)
        off, counts, ids, dists = csr_case(data, rng, max_len, allow_self)
        rec[f"{name}_data"] = data
        rec[f"{name}_off"] = off
        rec[f"{name}_counts"] = counts
        rec[f"{name}_ids"] = ids
        rec[f"{name}_dists"] = dists
        rec[f"{name}_M"] = np.int64(M)
        rec[f"{name}_alpha"] = np.float64(alpha)
        for tag, params in (("rng", PruneParams(M=M, strategy="rng")),
                            ("alpha", PruneParams(M=M, alpha=alpha, strategy="alpha"))):
            a = prune_all(ds, off, counts, ids, dists, params)
            b = add_reverse_and_prune(ds, a[0], a[1], a[2], params)
            for ph, res in (("a", a), ("b", b)):
                rec[f"{name}_{tag}_{ph}_ids"] = res[0]
                rec[f"{name}_{tag}_{ph}_dists"] = res[1]
                rec[f"{name}_{tag}_{ph}_counts"] = res[2]
                rec[f"{name}_{tag}_{ph}_de"] = np.int64(res[3])
                rec[f"{name}_{tag}_{ph}_ae"] = np.int64(res[4])
        # exact pool on the same data (ties, duplicates)
        k = min(10, data.shape[0] - 1)
        rec[f"{name}_truth"] = ground_truth_table(ds, None, k=k, exclude_self=True)
        names.append(name)
    # hand triangle of test_prune.py:80-96 (angle at a ~ 147.27 degrees)
    pts = np.array([[0, 0], [1, 0], [2.4, 0.9]], np.float32)
    rec["tri_data"] = pts
    rec["tri_d01"] = np.float32(_kernels.squared_l2(pts[1], pts[0]))
    rec["tri_d02"] = np.float32(_kernels.squared_l2(pts[2], pts[0]))
    rec["names"] = np.array(names)
    np.savez_compressed(HERE / "cases.npz", **rec)
    print("cases", names)


# ---------------------------------------------------------------------------
# Phase C and beam search: search_batch (search.py:81-94
# -> _kernels.search_many / _search_core), entry_point (prune.py:154-162) and
# finish_refine(connect=True) (prune.py:202-229, _connect :165-199).
# ---------------------------------------------------------------------------

def _phase_ab(data, K, R, strategy="rng", alpha=60.0):
    ds = Dataset.from_array(data)
    n = ds.n
    truth = ground_truth_table(ds, None, k=K, exclude_self=True)
    ids = truth.astype(np.int32).copy()
    dists = _list_dists(ds.data, ids)
    _resort(ids, dists)
    off = (np.arange(n + 1, dtype=np.int64) * K)
    cnt = np.full(n, K, np.int32)
    params = PruneParams(M=R, alpha=alpha, strategy=strategy)
    a = prune_all(ds, off, cnt, ids.ravel(), dists.ravel(), params)
    return ds, params, a


def save_search() -> None:
    rec = {}
    names = []
    rng = np.random.default_rng(77)
    # two far-apart blobs with a small pool: phase B leaves the graph split
    blobs = np.vstack([rng.standard_normal((300, 8)), rng.standard_normal((300, 8)) + 40.0,
                       rng.standard_normal((5, 8)) + 80.0]).astype(np.float32)
    specs = [
        ("cfg1_2k", synth.cfg1(2_000), 64, 24, "rng", 60.0),
        ("cfg1_full", synth.cfg1(10_000), 64, 24, "rng", 60.0),
        ("cfg1_a66", synth.cfg1(2_000), 64, 24, "alpha", 66.0),
        ("blobs", blobs, 6, 4, "rng", 60.0),
        ("blobs_a", blobs, 8, 3, "alpha", 120.0),
    ]
    for name, data, K, R, strategy, alpha in specs:
        ds, params, a = _phase_ab(data, K, R, strategy, alpha)
        g = finish_refine(ds, a[0], a[1], a[2], params, connect=True, ep=None, seed=0)
        b_ids, b_d, b_c, _, _ = add_reverse_and_prune(ds, a[0], a[1], a[2], params)
        interim = ProximityGraph(adj=b_ids, counts=b_c, M=params.M, ep=0)
        L = max(params.M + 1, 32)
        ep = entry_point(ds, interim, k=1, L=L, seed=0)
        reach = reachable_from(interim, ep)
        q = rng.standard_normal((64, data.shape[1])).astype(np.float32) * data.std() + \
            data.mean(axis=0)
        q = np.vstack([q, data[rng.choice(ds.n, 16, replace=False)]]).astype(np.float32)
        for tag, kk, LL in (("k10L40", 10, 40), ("k1L16", 1, 16)):
            s_ids, s_d, s_cnt = search_batch(ds, g, q, kk, LL)
            rec[f"{name}_{tag}_ids"] = s_ids
            rec[f"{name}_{tag}_dists"] = s_d
            rec[f"{name}_{tag}_dcount"] = s_cnt
        k_ids, k_d = kann_search(ds, g, q[0], 5, 24, ep=int(ds.n // 2))
        rec.update({f"{name}_data": data, f"{name}_K": np.int64(K), f"{name}_R": np.int64(R),
                    f"{name}_strategy": np.asarray(strategy), f"{name}_alpha": np.float64(alpha),
                    f"{name}_b_ids": b_ids, f"{name}_b_counts": b_c, f"{name}_ep": np.int64(ep),
                    f"{name}_reach": reach, f"{name}_c_adj": g.adj, f"{name}_c_counts": g.counts,
                    f"{name}_c_ep": np.int64(g.ep), f"{name}_c_over": g.over_cap,
                    f"{name}_queries": q, f"{name}_kann_ids": k_ids, f"{name}_kann_dists": k_d})
        names.append(name)
        print(name, "ep", ep, "unreached", int((~reach).sum()), "width", g.adj.shape[1],
              "over", len(g.over_cap))
    rec["names"] = np.array(names)
    np.savez_compressed(HERE / "search.npz", **rec)


def save_io() -> None:
    """Files written by the reference's dataset_io (save_vecs / save_index,
    dataset_io.py:67-84, 164-190) for byte-level format checks."""
    from pgann import dataset_io
    out = HERE / "io"
    os.makedirs(out, exist_ok=True)
    rng = np.random.default_rng(8)
    f = rng.standard_normal((7, 5)).astype(np.float32)
    i = rng.integers(-50, 50, size=(4, 9)).astype(np.int32)
    b = rng.integers(0, 256, size=(6, 16)).astype(np.uint8)
    dataset_io.save_vecs(out / "f.fvecs", f)
    dataset_io.save_vecs(out / "i.ivecs", i)
    dataset_io.save_vecs(out / "b.bvecs", b)
    sg = np.load(HERE / "search.npz")
    rec = dict(f=f, i=i, b=b)
    for name in ("cfg1_2k", "blobs"):
        g = ProximityGraph(adj=sg[f"{name}_c_adj"], counts=sg[f"{name}_c_counts"],
                           M=int(sg[f"{name}_R"]), ep=int(sg[f"{name}_c_ep"]),
                           over_cap=sg[f"{name}_c_over"])
        dataset_io.save_index(out / f"{name}.pgix", g)
        h = dataset_io.load_index(out / f"{name}.pgix")
        rec[f"{name}_adj"], rec[f"{name}_counts"] = h.adj, h.counts
        rec[f"{name}_ep"], rec[f"{name}_M"] = np.int64(h.ep), np.int64(h.M)
        rec[f"{name}_over"] = h.over_cap
    np.savez_compressed(out / "expect.npz", **rec)
    print("io", sorted(p.name for p in out.iterdir()))


def save_io_layered() -> None:
    """Layered PGIX files (dataset_io.py:174-245) written by the reference
    for the FastHNSW hierarchies of f3.npz (same inputs and parameters)."""
    from pgann import dataset_io
    from pgann import hnsw as R_hnsw
    out = HERE / "io"
    rec = {}
    for name, data in (("cfg1", synth.cfg1(2_500)), ("cfg2", synth.cfg2(3_000))):
        lg = R_hnsw.build_fasthnsw(Dataset.from_array(data), k0=12, ef=40, M=12, seed=6)
        dataset_io.save_index(out / f"hnsw_{name}.pgix", lg)
        h = dataset_io.load_index(out / f"hnsw_{name}.pgix")
        rec[f"{name}_nlayers"], rec[f"{name}_ep"] = np.int64(len(h.layers)), np.int64(h.ep)
        rec[f"{name}_levels"], rec[f"{name}_m_factor"] = h.levels, np.float64(h.m_factor)
        for i, layer in enumerate(h.layers):
            rec[f"{name}_L{i}_members"] = layer.members
            rec[f"{name}_L{i}_adj"], rec[f"{name}_L{i}_counts"] = layer.graph.adj, layer.graph.counts
            rec[f"{name}_L{i}_ep"], rec[f"{name}_L{i}_M"] = np.int64(layer.graph.ep), np.int64(layer.graph.M)
            rec[f"{name}_L{i}_over"] = layer.graph.over_cap
    np.savez_compressed(out / "expect_layered.npz", **rec)
    print("io layered", sorted(p.name for p in out.iterdir()))


def save_cfg5() -> None:
    """Config 5 at full size: the reference's FastHNSW build
    of the 200k x 128 config-2-recipe data (seed 4; k0=32, ef=200, one M=32
    for all layers -- SURVEY A.1 --, alpha=66, max_iters=2) and its layered
    search over the 10,000 seeded queries.  Layer 0 is stored as digests plus
    2,000 seeded rows; upper layers in full; search ids at L=100 in full and
    recall@10 at L = 50, 100, 200 against the exact float64 top-10."""
    import time
    from pgann import hnsw as R_hnsw
    from pgann.oracle import mean_recall
    from pgann.search import layered_search
    base, q = synth.cfg5(200_000, 10_000)
    ds = Dataset.from_array(base)
    t0 = time.perf_counter()
    lg = R_hnsw.build_fasthnsw(ds, k0=32, ef=200, M=32, alpha=66.0, seed=4)
    build_s = time.perf_counter() - t0
    rec = dict(levels=lg.levels.astype(np.int8), ep=np.int64(lg.ep),
               nlayers=np.int64(len(lg.layers)), m_factor=np.float64(lg.m_factor),
               build_s=np.float64(build_s), threads=np.int64(int(os.environ.get("NUMBA_NUM_THREADS", os.cpu_count()))))
    for i, layer in enumerate(lg.layers):
        g = layer.graph
        off, nb = g.to_csr()
        rec[f"L{i}_csr_sha"] = np.array(digest(off.astype(np.int64)) + digest(nb.astype(np.int32)))
        rec[f"L{i}_ep"] = np.int64(g.ep)
        rec[f"L{i}_over"] = np.asarray(g.over_cap, np.int32)
        if i > 0:
            rec[f"L{i}_members"] = layer.members
            rec[f"L{i}_adj"], rec[f"L{i}_counts"] = g.adj, g.counts
        else:
            rec["L0_counts"] = g.counts.astype(np.int16)
            rows = np.sort(np.random.default_rng(55).choice(ds.n, 2000, replace=False))
            rec["L0_rows"] = rows
            rec["L0_rows_adj"] = g.adj[rows]
    x = base.astype(np.float64)
    xn = (x * x).sum(1)
    truth = np.empty((q.shape[0], 10), np.int32)
    for lo in range(0, q.shape[0], 500):
        qq = q[lo:lo + 500].astype(np.float64)
        d2 = np.maximum(xn[None, :] - 2.0 * (qq @ x.T) + (qq * qq).sum(1)[:, None], 0.0)
        truth[lo:lo + 500] = np.argsort(d2, axis=1, kind="stable")[:, :10]
    for L in (50, 100, 200):
        ids = np.full((q.shape[0], 10), -1, np.int32)
        for j in range(q.shape[0]):
            r = layered_search(ds, lg, q[j], 10, L)[0]
            ids[j, :len(r)] = r
        rec[f"recall_L{L}"] = np.float64(mean_recall(ids, truth, 10))
        if L == 100:
            rec["search_ids_L100"] = ids
        print("cfg5 L", L, "recall@10", float(rec[f"recall_L{L}"]), flush=True)
    print("cfg5 build_s", build_s, "layers", [len(l.members) for l in lg.layers])
    np.savez_compressed(HERE / "cfg5.npz", **rec)


def save_f3() -> None:
    """NN-Descent, FastNSG, NSG and FastHNSW outputs:
    knng.py:40-125, nsg.py:319-430, hnsw.py:141-192, search.py:97-130."""
    from pgann import hnsw as R_hnsw
    from pgann import knng as R_knng
    from pgann import nsg as R_nsg
    from pgann.search import layered_search
    rec = {}
    names = []
    for name, data in (("cfg1", synth.cfg1(2_500)), ("cfg2", synth.cfg2(3_000))):
        ds = Dataset.from_array(data)
        rec[f"{name}_data"] = data
        # NN-Descent: init + every round's rows / flags / update counts
        st = R_knng.knng_init_random(ds, 16, seed=5)
        rec[f"{name}_knng0_ids"], rec[f"{name}_knng0_dists"] = st.ids, st.dists
        for r in range(1, 4):
            st = R_knng.knng_descent_iterate(ds, st, rho=1.0 if r != 2 else 0.5)
            rec[f"{name}_knng{r}_ids"], rec[f"{name}_knng{r}_dists"] = st.ids, st.dists
            rec[f"{name}_knng{r}_flags"] = st.flags
            rec[f"{name}_knng{r}_upd"] = np.int64(st.last_updates)
        kb = R_knng.build_knng(ds, 12, iters=10, seed=7)
        rec[f"{name}_bknng_ids"], rec[f"{name}_bknng_iters"] = kb.ids, np.int64(kb.iterations)
        g = R_nsg.build_nsg_original(ds, k0=12, k=24, L=32, M=12, seed=3)
        rec[f"{name}_nsg_adj"], rec[f"{name}_nsg_counts"], rec[f"{name}_nsg_ep"] = \
            g.adj, g.counts, np.int64(g.ep)
        fst = R_nsg.FastNsgStats()
        g = R_nsg.build_fastnsg(ds, k0=12, k=24, L=32, M=12, alpha=66.0, max_iters=2, seed=4,
                                stats=fst)
        rec[f"{name}_fnsg_adj"], rec[f"{name}_fnsg_counts"], rec[f"{name}_fnsg_ep"] = \
            g.adj, g.counts, np.int64(g.ep)
        rec[f"{name}_fnsg_over"] = g.over_cap
        fs = fst.final_state
        rec[f"{name}_fnsg_state_ids"], rec[f"{name}_fnsg_state_counts"] = fs.ids, fs.counts
        rec[f"{name}_fnsg_state_fresh"] = fs.fresh
        rec[f"{name}_fnsg_search_dists"] = np.array([s.search_dists for s in fst.per_iteration])
        lg = R_hnsw.build_fasthnsw(ds, k0=12, ef=40, M=12, seed=6)
        rec[f"{name}_hnsw_levels"], rec[f"{name}_hnsw_ep"] = lg.levels, np.int64(lg.ep)
        rec[f"{name}_hnsw_nlayers"] = np.int64(len(lg.layers))
        for i, layer in enumerate(lg.layers):
            rec[f"{name}_hnsw_L{i}_members"] = layer.members
            rec[f"{name}_hnsw_L{i}_adj"] = layer.graph.adj
            rec[f"{name}_hnsw_L{i}_counts"] = layer.graph.counts
            rec[f"{name}_hnsw_L{i}_ep"] = np.int64(layer.graph.ep)
        rng = np.random.default_rng(31)
        q = data[rng.choice(ds.n, 40, replace=False)] + rng.normal(0, 0.5, (40, data.shape[1]))
        q = q.astype(np.float32)
        res = [layered_search(ds, lg, qq, 10, 40) for qq in q]
        rec[f"{name}_lq"] = q
        rec[f"{name}_lq_ids"] = np.array([np.pad(r[0], (0, 10 - len(r[0])), constant_values=-1)
                                          for r in res])
        rec[f"{name}_lq_dists"] = np.array([np.pad(r[1], (0, 10 - len(r[1])),
                                                   constant_values=np.inf) for r in res])
        names.append(name)
        print(name, "knng iters", kb.iterations, "hnsw layers", len(lg.layers),
              "upd", [int(rec[f"{name}_knng{r}_upd"]) for r in range(1, 4)])
    rec["names"] = np.array(names)
    np.savez_compressed(HERE / "f3.npz", **rec)


def main() -> None:
    os.makedirs(HERE, exist_ok=True)
    if len(sys.argv) > 1 and sys.argv[1] == "f3":
        save_f3()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "search":
        save_search()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "io":
        save_io()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "cfg5":
        save_cfg5()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "io_layered":
        save_io_layered()
        return
    save_cases()
    save_config("cfg1_full", synth.cfg1(10_000), 64, 24,
                dict(config=1, n=10_000, K=64, R=24), full=False)
    save_config("cfg1_2k", synth.cfg1(2_000), 64, 24,
                dict(config=1, n=2_000, K=64, R=24), full=True)
    save_config("cfg2_4k", synth.cfg2(4_000), 128, 32,
                dict(config=2, n=4_000, K=128, R=32), full=False)
    save_config("cfg3_2k", synth.cfg3(2_000), 128, 32,
                dict(config=3, n=2_000, K=128, R=32), full=False)
    save_config("cfg4_2k", synth.cfg4(2_000), 256, 64,
                dict(config=4, n=2_000, K=256, R=64), full=False)


if __name__ == "__main__":
    main()
