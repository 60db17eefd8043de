"""CSV ingest / output of the reference's data-io module.

Comma-separated, '.' decimal point, one row per line, optional single header row,
key column chosen by zero-based index; floats written with the shortest repr that
round-trips.  This is the data format either side of the path
and is excluded from every timing.  Ingest is native (jq_io.cu): a thread
pool parses the mmapped file, and with device="cuda" the rows stream into HBM through
pinned staging slots while the parse goes on.
"""

from __future__ import annotations

import os
from typing import Optional

import numpy as np

from . import _native as N
from .joins import Table
from .matrix import as_matrix


def read_table(path: str, has_header: bool = False, key_col: Optional[int] = None, device=None) -> Table:
    """Table from a CSV file; `key_col` (zero-based) is an int64 key
    column, sorted non-decreasing.  Parsed natively (jq_csv_scan / jq_csv_parse:
    mmapped file, thread pool, std::from_chars).  device=None returns numpy arrays;
    device="cuda" (or a torch.device) returns torch tensors in HBM, streamed through
    pinned staging with the H2D copies overlapping the parse.  Errors are ValueErrors
    naming the file line (ragged row, unparsable cell, non-finite value, unsorted keys)."""
    import ctypes as C
    rows, cols = np.zeros(1, dtype=np.int64), np.zeros(1, dtype=np.int64)
    bpath = os.fsencode(path)
    N.check(N.lib().jq_csv_scan(bpath, int(bool(has_header)), rows.ctypes.data, cols.ctypes.data))
    m, w = int(rows[0]), int(cols[0])
    if key_col is not None and not 0 <= key_col < max(w, 1):
        raise ValueError(f"{path}: key column {key_col} out of range (width {w})")
    ncols = w - (1 if key_col is not None else 0)
    if device is None:
        data = np.empty((m, ncols))
        keys = np.empty(m, dtype=np.int64) if key_col is not None else None
        N.check(N.lib().jq_csv_parse(None, bpath, int(bool(has_header)),
                                     -1 if key_col is None else int(key_col), m, w, N.ptr(data), N.ptr(keys)))
    else:
        import torch
        dev = torch.device(device)
        data = torch.empty((m, ncols), dtype=torch.float64, device=dev)
        keys = torch.empty(m, dtype=torch.int64, device=dev) if key_col is not None else None
        N.use_torch_stream(data)
        N.check(N.lib().jq_csv_parse(N.ctx(), bpath, int(bool(has_header)), -1 if key_col is None else int(key_col),
                                     m, w, N.ptr(data), N.ptr(keys)))
    return Table(data, keys)


def read_matrix(path: str, has_header: bool = False) -> np.ndarray:
    return np.asarray(read_table(path, has_header).data)


def _fmt(x: float) -> str:
    return repr(float(x))


def write_matrix(matrix, path: str) -> None:
    m = as_matrix(matrix)
    m = m.cpu().numpy() if hasattr(m, "cpu") else np.asarray(m)
    with open(path, "w", encoding="utf-8") as f:
        for row in m:
            f.write(",".join(_fmt(x) for x in row) + "\n")


def write_table(table: Table, path: str) -> None:
    """Key column (when present) first, then the data columns."""
    d = table.data.cpu().numpy() if hasattr(table.data, "cpu") else np.asarray(table.data)
    k = None if table.keys is None else (table.keys.cpu().numpy() if hasattr(table.keys, "cpu")
                                         else np.asarray(table.keys))
    with open(path, "w", encoding="utf-8") as f:
        for i, row in enumerate(d):
            cells = ([str(int(k[i]))] if k is not None else []) + [_fmt(x) for x in row]
            f.write(",".join(cells) + "\n")


def write_svd(result, path: str, v_path: Optional[str] = None) -> None:
    """Singular values one per line; V (row-major) to v_path when present."""
    vals = result.values.cpu().numpy() if hasattr(result.values, "cpu") else np.asarray(result.values)
    with open(path, "w", encoding="utf-8") as f:
        for x in vals:
            f.write(_fmt(x) + "\n")
    if v_path is not None and result.right_vectors is not None:
        write_matrix(result.right_vectors, v_path)
