"""CSV ingest / output of the reference's data-io module, host side.

Comma-separated, '.' decimal point, one row per line, optional single header row,
key column chosen by zero-based index; floats written with the shortest repr that
round-trips.  This is the data format either side of the path
and is excluded from every timing; the tables it returns go to the GPU
through the same API as any numpy input.
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from .joins import Table
from .matrix import as_matrix


def _rows(path: str, has_header: bool):
    with open(path, "r", encoding="utf-8") as f:
        lines = f.read().splitlines()
    start = 1 if has_header else 0
    out, width = [], None
    for ln, line in enumerate(lines[start:], start=start + 1):
        if not line.strip():
            continue
        cells = line.split(",")
        if width is None:
            width = len(cells)
        elif len(cells) != width:
            raise ValueError(f"{path}:{ln}: ragged row ({len(cells)} cells, expected {width})")
        out.append((ln, cells))
    return out, width or 0


def read_table(path: str, has_header: bool = False, key_col: Optional[int] = None) -> Table:
    """Table from a CSV file; `key_col` (zero-based) is an int64 key column, sorted."""
    rows, width = _rows(path, has_header)
    if key_col is not None and not 0 <= key_col < width:
        raise ValueError(f"{path}: key column {key_col} out of range (width {width})")
    ncols = width - (1 if key_col is not None else 0)
    data = np.empty((len(rows), ncols))
    keys = np.empty(len(rows), dtype=np.int64) if key_col is not None else None
    for r, (ln, cells) in enumerate(rows):
        c_out = 0
        for c, cell in enumerate(cells):
            try:
                if c == key_col:
                    keys[r] = int(cell)
                else:
                    data[r, c_out] = float(cell)
                    c_out += 1
            except ValueError:
                raise ValueError(f"{path}:{ln}: cannot parse column {c}: {cell!r}") from None
    if not np.all(np.isfinite(data)):
        raise ValueError(f"{path}: non-finite value")
    if keys is not None and len(keys) > 1 and np.any(keys[1:] < keys[:-1]):
        bad = int(np.argmax(keys[1:] < keys[:-1])) + 1
        raise ValueError(f"{path}:{rows[bad][0]}: keys are not sorted non-decreasing")
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
