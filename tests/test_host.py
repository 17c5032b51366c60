"""CPU-only host-logic tests (validation, containers) mirroring the
reference's test_prune.py:278-287, test_core.py:12-33, graph.py:41-61."""
import numpy as np
import pytest

from paper_2410_01231_b200 import Dataset, ProximityGraph, PruneParams, refine


def test_params_validation():
    with pytest.raises(ValueError):
        PruneParams(M=0)
    with pytest.raises(ValueError):
        PruneParams(M=4, strategy="tau")
    with pytest.raises(ValueError):
        PruneParams(M=4, alpha=59.0, strategy="alpha")
    with pytest.raises(ValueError):
        PruneParams(M=4, alpha=180.0, strategy="alpha")
    assert PruneParams(M=4, alpha=90.0).cos_alpha == pytest.approx(0.0)
    assert PruneParams(M=4, strategy="alpha").strategy_code == 1


def test_dataset_validation():
    ds = Dataset.from_array(np.arange(12, dtype=np.float64).reshape(4, 3))
    assert ds.data.dtype == np.float32 and (ds.n, ds.d) == (4, 3)
    with pytest.raises(ValueError):
        Dataset.from_array(np.zeros(5))
    with pytest.raises(ValueError):
        Dataset.from_array(np.zeros((0, 3)))
    bad = np.zeros((2, 2))
    bad[1, 1] = np.nan
    with pytest.raises(ValueError):
        Dataset.from_array(bad)
    with pytest.raises(ValueError):
        Dataset(np.zeros((3, 3), dtype=np.float64))


def test_graph_validate():
    g = ProximityGraph(adj=np.array([[1, -1], [0, -1]], np.int32),
                       counts=np.array([1, 1], np.int32), M=2, ep=0)
    g.validate()
    with pytest.raises(ValueError, match="self-loop"):
        ProximityGraph(adj=np.array([[0, -1], [0, -1]], np.int32),
                       counts=np.array([1, 1], np.int32), M=2, ep=0).validate()
    with pytest.raises(ValueError, match="duplicate"):
        ProximityGraph(adj=np.array([[1, 1], [0, -1]], np.int32),
                       counts=np.array([2, 1], np.int32), M=2, ep=0).validate()
    with pytest.raises(ValueError, match="degree"):
        ProximityGraph(adj=np.array([[1, 2], [0, -1], [0, -1]], np.int32),
                       counts=np.array([2, 1, 1], np.int32), M=1, ep=0).validate()
    off, nbrs = g.to_csr()
    assert off.tolist() == [0, 1, 2] and nbrs.tolist() == [1, 0]


def test_phase_c_has_no_cpu_fallback():
    """Phase C (refine(connect=True)) and the beam search run on the GPU only:
    without a CUDA device they raise instead of computing on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    from paper_2410_01231_b200 import ProximityGraph, kann_search
    ds = Dataset.from_array(np.zeros((3, 2), np.float32))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        refine(ds, np.zeros(4, np.int64), np.zeros(3, np.int32), np.zeros(0, np.int32),
               np.zeros(0, np.float32), PruneParams(M=2), connect=True)
    g = ProximityGraph(adj=np.array([[1], [0], [0]], np.int32),
                       counts=np.array([1, 1, 1], np.int32), M=2, ep=0)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        kann_search(ds, g, np.zeros(2, np.float32), 1, 4)
