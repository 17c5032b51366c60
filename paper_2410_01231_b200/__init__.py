"""B200-native (sm_100a) RNG proximity-graph construction hot path.

Drop-in for the reference pgann package's hot path (arXiv 2410.01231):
  * pool.ground_truth_table / knn_pools  -- exact k-NN candidate pools
  * prune.prune_all                       -- phase-A edge selection
  * prune.add_reverse_and_prune           -- phase-B reverse edges + re-prune
  * prune.refine / finish_refine, entry_point  -- phase C connectivity repair
  * search.kann_search / search_batch     -- beam search
  * io.load_vecs / save_vecs / load_index / save_index -- reference file formats
  * knng / nsg / hnsw -- NN-Descent, NSG, FastNSG and FastHNSW builders
  * index.build_rng_index / RngBuilder   -- the whole path in one call
All compute runs in libpgk.so (hand-written CUDA for sm_100a, C ABI in
include/pgk.h); there is no CPU fallback.
"""

from .core import Dataset, centroid
from .graph import EMPTY, ProximityGraph
from .pool import exact_knn, ground_truth_table, knn_pools, mean_recall, recall_at_k
from .prune import (PruneParams, RefineStats, add_reverse_and_prune, alpha_prune,
                    entry_point, finish_refine, prune_all, refine, rng_prune)
from .search import kann_search, search_batch
from . import hnsw, io, knng, nsg
from .index import RngBuilder, build_rng_index

__all__ = ["Dataset", "centroid", "EMPTY", "ProximityGraph", "exact_knn",
           "ground_truth_table", "knn_pools", "mean_recall", "recall_at_k", "PruneParams",
           "RefineStats", "add_reverse_and_prune", "alpha_prune", "entry_point",
           "finish_refine", "kann_search", "search_batch",
           "prune_all", "refine", "rng_prune", "RngBuilder", "build_rng_index"]
