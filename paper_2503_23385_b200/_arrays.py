"""Output allocation and key coercion shared by the API modules."""

from __future__ import annotations

import numpy as np

from ._native import is_torch_cuda


def like(shape, *inputs, dtype="f8"):
    """Empty output on the device of the first torch CUDA input, else numpy."""
    for x in inputs:
        if is_torch_cuda(x):
            import torch
            return torch.empty(shape, dtype=torch.float64 if dtype == "f8" else torch.int64,
                               device=x.device)
    return np.empty(shape, dtype=np.float64 if dtype == "f8" else np.int64)


def zeros_like_out(shape, *inputs):
    out = like(shape, *inputs)
    out[...] = 0
    return out


def as_keys(keys, n_rows: int):
    if keys is None:
        return None
    if is_torch_cuda(keys):
        import torch
        k = keys.to(torch.int64).contiguous().reshape(-1)
    else:
        k = np.ascontiguousarray(keys, dtype=np.int64).reshape(-1)
    if k.shape[0] != n_rows:
        raise ValueError("key column length does not match the row count")
    return k
