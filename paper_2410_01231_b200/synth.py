"""Seeded synthetic point sets for the BASELINE.json configurations.

These are host-side input generators, not part of the GPU path.  They restate
the reference's ``gen_synthetic`` (``pkg/src/pgann/dataset_io.py:92-107``) and
the explicit recipes of SURVEY.md Appendix A.2 (numpy ``default_rng(seed)``,
draw order fixed, float64 math, cast to float32 last).  Every recipe can emit
a *prefix* of the full-size array bit-for-bit: the cluster assignment is drawn
for the full N first (as the full-size recipe does) and the Gaussian noise is
drawn in row chunks, which numpy's PCG64 stream makes identical to one draw.
"""

from __future__ import annotations

import numpy as np

_CHUNK_ROWS = 65536


def _normal_rows(rng: np.random.Generator, n: int, d: int, out_fn) -> None:
    """Draw an (n, d) standard-normal block in row chunks, handing each chunk
    (lo, hi, block) to out_fn.  Chunked draws equal one (n, d) draw."""
    for lo in range(0, n, _CHUNK_ROWS):
        hi = min(n, lo + _CHUNK_ROWS)
        out_fn(lo, hi, rng.standard_normal((hi - lo, d)))


def gen_synthetic(n: int, d: int, dist: str = "uniform", seed: int = 0,
                  n_clusters: int = 16, cluster_std: float = 0.05) -> np.ndarray:
    """Same draws as the reference's ``gen_synthetic``
    (``dataset_io.py:92-107``); returns the float32 array."""
    rng = np.random.default_rng(seed)
    if dist == "uniform":
        return np.ascontiguousarray(rng.random((n, d), dtype=np.float32))
    if dist == "gaussian":
        return np.ascontiguousarray(rng.standard_normal((n, d), dtype=np.float32))
    if dist == "clustered":
        centers = rng.random((n_clusters, d))
        assign = rng.integers(0, n_clusters, size=n)
        out = np.empty((n, d), np.float32)

        def put(lo, hi, z):
            out[lo:hi] = (centers[assign[lo:hi]] + cluster_std * z).astype(np.float32)

        _normal_rows(rng, n, d, put)
        return out
    raise ValueError(f"unknown distribution {dist!r}")


def cfg1(n: int = 10_000) -> np.ndarray:
    """Config 1: N(0,1) fp32, d=32, seed 0 (== gen_synthetic(n, 32, "gaussian", 0))."""
    return gen_synthetic(n, 32, "gaussian", seed=0)


def cfg2(n: int = 1_000_000, n_full: int = 1_000_000, seed: int = 1) -> np.ndarray:
    """Config 2 (Sift1M stand-in): integer-valued features in [0, 255], d=128.
    c = 255*U[0,1)^(256x128); a ~ U{0..255}^N; x = clip(rint(c[a] + 20 z), 0, 255).
    Returns the first ``n`` rows of the ``n_full``-row array."""
    d, k = 128, 256
    rng = np.random.default_rng(seed)
    c = 255.0 * rng.random((k, d))
    a = rng.integers(0, k, size=n_full)[:n]
    out = np.empty((n, d), np.float32)

    def put(lo, hi, z):
        out[lo:hi] = np.clip(np.rint(c[a[lo:hi]] + 20.0 * z), 0.0, 255.0).astype(np.float32)

    _normal_rows(rng, n, d, put)
    return out


def cfg2_queries(n_queries: int = 10_000, seed: int = 1, query_seed: int = 1001) -> np.ndarray:
    """Recall queries for config 2 (BASELINE gives none; same
    recipe, distinct documented seed): the SAME 256 centres (the first draw
    of default_rng(seed)), then a ~ U{0..255} and the noise from
    default_rng(query_seed): x = clip(rint(c[a] + 20 z), 0, 255)."""
    d, k = 128, 256
    c = 255.0 * np.random.default_rng(seed).random((k, d))
    rng = np.random.default_rng(query_seed)
    qa = rng.integers(0, k, size=n_queries)
    q = np.clip(np.rint(c[qa] + 20.0 * rng.standard_normal((n_queries, d))), 0.0, 255.0)
    return q.astype(np.float32)


def cfg5(n: int = 200_000, n_queries: int = 10_000, seed: int = 4):
    """Config 5 (FastHNSW build): the config-2 recipe with seed 4 for the base
    rows; the queries continue the same generator after the base draws (same
    256 centres: a ~ U{0..255}, x = clip(rint(c[a] + 20 z), 0, 255)).
    Returns (base (n, 128), queries (n_queries, 128)) float32."""
    d, k = 128, 256
    rng = np.random.default_rng(seed)
    c = 255.0 * rng.random((k, d))
    a = rng.integers(0, k, size=n)
    base = np.empty((n, d), np.float32)

    def put(lo, hi, z):
        base[lo:hi] = np.clip(np.rint(c[a[lo:hi]] + 20.0 * z), 0.0, 255.0).astype(np.float32)

    _normal_rows(rng, n, d, put)
    qa = rng.integers(0, k, size=n_queries)
    q = np.clip(np.rint(c[qa] + 20.0 * rng.standard_normal((n_queries, d))), 0.0, 255.0)
    return base, q.astype(np.float32)


def cfg3(n: int = 1_000_000, n_full: int = 1_000_000, seed: int = 2) -> np.ndarray:
    """Config 3 (Gist1M stand-in): gen_synthetic(n_full, 960, "clustered", seed=2,
    n_clusters=100, cluster_std=0.1), first ``n`` rows."""
    d, k = 960, 100
    rng = np.random.default_rng(seed)
    centers = rng.random((k, d))
    a = rng.integers(0, k, size=n_full)[:n]
    out = np.empty((n, d), np.float32)

    def put(lo, hi, z):
        out[lo:hi] = (centers[a[lo:hi]] + 0.1 * z).astype(np.float32)

    _normal_rows(rng, n, d, put)
    return out


def cfg4(n: int = 2_000_000, n_full: int = 2_000_000, seed: int = 3) -> np.ndarray:
    """Config 4 (text-embedding stand-in): 1000-centre N(0,I) mixture, sigma 0.3,
    d=768, every row L2-normalised; first ``n`` rows of ``n_full``."""
    d, k = 768, 1000
    rng = np.random.default_rng(seed)
    c = rng.standard_normal((k, d))
    a = rng.integers(0, k, size=n_full)[:n]
    out = np.empty((n, d), np.float32)

    def put(lo, hi, z):
        x = c[a[lo:hi]] + 0.3 * z
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        out[lo:hi] = x.astype(np.float32)

    _normal_rows(rng, n, d, put)
    return out


# (N, d, K, R) of BASELINE.json configs 1-4.
CONFIGS = {
    1: dict(gen=cfg1, n=10_000, d=32, K=64, R=24),
    2: dict(gen=cfg2, n=1_000_000, d=128, K=128, R=32),
    3: dict(gen=cfg3, n=1_000_000, d=960, K=128, R=32),
    4: dict(gen=cfg4, n=2_000_000, d=768, K=256, R=64),
}
