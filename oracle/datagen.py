"""Synthetic inputs and the BASELINE configs.

PRNG (SPEC.md:468 asks for a named, documented generator): counter-based
SplitMix64.  Element k = row * cols + col of a table with seed s is
    x_k = mix64(s + (k + 1) * 0x9E3779B97F4A7C15)   (mod 2^64)
    u_k = ((x_k >> 11) + 0.5) * 2^-53                in the open interval (0, 1)
with mix64 the SplitMix64 finaliser (Steele, Lea, Flood 2014).  Any shard can
regenerate any element; the CUDA generator in the product computes the same
bits.  Test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .joins import Table

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * M1
    z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def splitmix64_uniform(seed: int, start: int, count: int) -> np.ndarray:
    """u_k for k in [start, start + count) as float64."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        x = _mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + k * GAMMA)
    return ((x >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def uniform_matrix(seed: int, rows: int, cols: int, row0: int = 0,
                   chunk: int = 1 << 24) -> np.ndarray:
    """rows x cols block starting at table row ``row0`` of the table with this seed."""
    out = np.empty(rows * cols)
    base = row0 * cols
    for s in range(0, rows * cols, chunk):
        n = min(chunk, rows * cols - s)
        out[s:s + n] = splitmix64_uniform(seed, base + s, n)
    return out.reshape(rows, cols)


def near_equal_keys(rows: int, key_groups: int) -> np.ndarray:
    """Sorted keys 0..key_groups-1, the first rows % key_groups groups one row larger
    (key_groups=2, rows=4 -> [0,0,1,1])."""
    if not 1 <= key_groups <= rows:
        raise ValueError("key_groups must lie in 1..rows")
    q, r = divmod(rows, key_groups)
    i = np.arange(rows, dtype=np.int64)
    big = r * (q + 1)
    return np.where(i < big, i // (q + 1), r + (i - big) // max(q, 1)).astype(np.int64)


def zipf_cdf(s: float, universe: int) -> np.ndarray:
    cdf = np.cumsum(np.arange(1, universe + 1, dtype=np.float64) ** (-s))
    return cdf / cdf[-1]


def zipf_keys(seed: int, rows: int, s: float = 1.1, universe: int = 1_000_000) -> np.ndarray:
    """Unsorted Zipf(s) keys in [0, universe): searchsorted(cdf, u_row, 'right')."""
    u = splitmix64_uniform(seed, 0, rows)
    return np.searchsorted(zipf_cdf(s, universe), u, side="right").astype(np.int64)


@dataclass
class GenSpec:
    """rows, cols, seed, optional key_groups."""

    rows: int
    cols: int
    seed: int
    key_groups: Optional[int] = None


def gen_uniform(spec: GenSpec) -> Table:
    """Uniform(0,1) table, bit-identical for the same spec."""
    if spec.rows < 1 or spec.cols < 1:
        raise ValueError("gen_uniform needs rows >= 1 and cols >= 1")
    data = uniform_matrix(spec.seed, spec.rows, spec.cols)
    keys = None if spec.key_groups is None else near_equal_keys(spec.rows, spec.key_groups)
    return Table(data, keys)


# BASELINE.json configs: seeds A = 1000c+1, B = 1000c+2.
CONFIGS = {
    1: dict(m=1000, n=4, keys=None),
    2: dict(m=1_000_000, n=16, keys="groups", key_groups=10_000),
    3: dict(m=10_000_000, n=32, keys="zipf", s=1.1, universe=1_000_000),
    4: dict(m=100_000_000, n=64, keys=None),
    5: dict(m=1_000_000, n=128, keys=None, want_vectors=True),
}


def config_keys(c: int, side: int, rows: Optional[int] = None) -> Optional[np.ndarray]:
    cfg = CONFIGS[c]
    rows = cfg["m"] if rows is None else rows
    if cfg["keys"] == "groups":
        return near_equal_keys(rows, cfg["key_groups"] * rows // cfg["m"])
    if cfg["keys"] == "zipf":
        k = zipf_keys(1000 * c + 2 + side, rows, cfg["s"], cfg["universe"])
        return np.sort(k, kind="stable")
    return None


def zipf_sorted_table(seed_keys: int, seed_data: int, rows: int, cols: int, s: float = 1.1,
                      universe: int = 1_000_000):
    """C3 recipe: keys and data rows in generation order, then a stable
    sort of (key, row) permutes the rows.  Returns (Table, perm), perm[r] = generation
    row of row r (np.argsort(kind="stable"), the GPU radix sort's parity target)."""
    k = zipf_keys(seed_keys, rows, s, universe)
    perm = np.argsort(k, kind="stable")
    return Table(uniform_matrix(seed_data, rows, cols)[perm], k[perm]), perm


def config_tables(c: int, rows: Optional[int] = None):
    """(A, B) Tables of config c; ``rows`` overrides m (a bounded sample, same recipe).
    C3: data rows permuted by the stable key sort (zipf_sorted_table)."""
    cfg = CONFIGS[c]
    m = cfg["m"] if rows is None else rows
    if cfg["keys"] == "zipf":
        a, _ = zipf_sorted_table(1000 * c + 3, 1000 * c + 1, m, cfg["n"], cfg["s"], cfg["universe"])
        b, _ = zipf_sorted_table(1000 * c + 4, 1000 * c + 2, m, cfg["n"], cfg["s"], cfg["universe"])
        return a, b
    a = Table(uniform_matrix(1000 * c + 1, m, cfg["n"]), config_keys(c, 1, m))
    b = Table(uniform_matrix(1000 * c + 2, m, cfg["n"]), config_keys(c, 2, m))
    return a, b
