"""Core types, mirroring the reference's ``core.py``.

``Dataset`` keeps the reference contract (float32, C-contiguous (n, d), finite,
n, d >= 1; core.py:18-47) and additionally caches the device copy the kernels
read and the exact-integer (U8) pool-mode flag.
"""

from __future__ import annotations

import numpy as np
import torch

from . import kernels


class Dataset:
    """A dense point set, float32, row-major, shape (n, d) (core.py:18-47).

    ``data`` is a numpy array (the reference's type) or a CUDA float32 tensor
    (device-resident datasets; ``data`` then stays on the device)."""

    def __init__(self, data):
        if isinstance(data, torch.Tensor):
            if data.dtype != torch.float32 or data.ndim != 2 or not data.is_contiguous():
                raise ValueError("dataset must be C-contiguous float32 (n, d); "
                                 "use Dataset.from_array to convert")
        elif (not isinstance(data, np.ndarray) or data.dtype != np.float32
              or data.ndim != 2 or not data.flags.c_contiguous):
            raise ValueError("dataset must be C-contiguous float32 (n, d); "
                             "use Dataset.from_array to convert")
        self.data = data
        self._dev = data if isinstance(data, torch.Tensor) and data.is_cuda else None
        self._u8 = None
        self._u8_rows = None

    @classmethod
    def from_array(cls, arr) -> "Dataset":
        if isinstance(arr, torch.Tensor):
            data = arr.to(torch.float32).contiguous()
            ok_shape = data.ndim == 2
            if ok_shape and (data.shape[0] < 1 or data.shape[1] < 1):
                raise ValueError("dataset must be non-empty")
            if not ok_shape:
                raise ValueError("dataset must be 2-dimensional")
            if not bool(torch.isfinite(data).all()):
                raise ValueError("dataset contains non-finite values")
            return cls(data)
        data = np.ascontiguousarray(arr, dtype=np.float32)
        if data.ndim != 2:
            raise ValueError("dataset must be 2-dimensional")
        if data.shape[0] < 1 or data.shape[1] < 1:
            raise ValueError("dataset must be non-empty")
        if not np.all(np.isfinite(data)):
            raise ValueError("dataset contains non-finite values")
        return cls(data)

    @property
    def n(self) -> int:
        return int(self.data.shape[0])

    @property
    def d(self) -> int:
        return int(self.data.shape[1])

    def device_data(self) -> torch.Tensor:
        """The (n, d) float32 CUDA copy the kernels read (uploaded once)."""
        if self._dev is None:
            self._dev = kernels._dev(self.data, torch.float32)
        return self._dev

    def is_u8(self) -> bool:
        """All values integers in [0, 255] (d <= 258): exact integer pools."""
        if self._u8 is None:
            self._u8 = kernels.detect_u8(self.device_data())
        return self._u8

    def device_u8(self):
        """(u8 rows (n, 128), int32 norms) for the exact-integer selection path,
        or None when the data are not [0,255] integers with d <= 128."""
        if self.d > 128 or not self.is_u8():
            return None
        if self._u8_rows is None:
            self._u8_rows = kernels.make_u8(self.device_data())
        return self._u8_rows


def centroid(ds: Dataset) -> np.ndarray:
    """Mean point, accumulated in float64, returned float32 (core.py:153-155)."""
    data = ds.data.cpu().numpy() if isinstance(ds.data, torch.Tensor) else ds.data
    return data.mean(axis=0, dtype=np.float64).astype(np.float32)
