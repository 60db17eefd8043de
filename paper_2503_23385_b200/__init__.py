"""paper_2503_23385_b200 — B200-native Figaro two-table QR / SVD (arXiv 2503.23385).

Drop-in mirror of the reference package `joinqr` for its hot path: the same
public names, argument layout, return types and error behaviour
(pkg/src/joinqr/__init__.py:20-77, SPEC.md), resolved lazily like the
reference (`__getattr__`, :65-73).  Every compute call goes through the C ABI
of libjoinqr.so (include/joinqr.h) to hand-written sm_100a kernels; there is
no CPU fallback.  Names of the reference that are not on the hot path
(bench-harness objects, determinant / Givens cross-checks) raise an
AttributeError that says so ("Out of scope").
"""

import importlib

__version__ = "0.1.0"

_EXPORTS = {
    "as_matrix": ".matrix",
    "matmul": ".matrix",
    "gram": ".matrix",
    "max_abs_diff": ".matrix",
    "transpose": ".matrix",
    "frobenius_norm": ".matrix",
    "hconcat": ".matrix",
    "vconcat": ".matrix",
    "scale": ".matrix",
    "row_slice": ".matrix",
    "is_upper_triangular": ".matrix",
    "head": ".headtail",
    "tail": ".headtail",
    "head_tail": ".headtail",
    "Table": ".joins",
    "ReducedMatrix": ".joins",
    "reduce_cartesian": ".joins",
    "reduce_natural_join": ".joins",
    "reduce_join": ".joins",
    "group_keys": ".joins",
    "argsort_keys": ".joins",
    "gather_rows": ".joins",
    "sort_by_key": ".joins",
    "householder_r": ".qr",
    "canonicalize": ".qr",
    "figaro_r": ".qr",
    "SvdResult": ".svd",
    "svd_of_r": ".svd",
    "figaro_svd": ".svd",
    "GenSpec": ".datagen",
    "gen_uniform": ".datagen",
    "set_device": "._native",
    "set_variant": "._native",
    "last_timing": "._native",
    "materialize_cartesian": ".bruteforce",
    "materialize_natural_join": ".bruteforce",
    "baseline_r": ".bruteforce",
    "baseline_svd": ".bruteforce",
    "join_r_bruteforce": ".bruteforce",
    "read_table": ".tableio",
    "read_matrix": ".tableio",
    "write_matrix": ".tableio",
    "write_table": ".tableio",
    "write_svd": ".tableio",
}

_OUT_OF_SCOPE = {
    "givens_r": "cross-validation reference only (SPEC.md:299)",
    "det_lu": "oracle plumbing (CPU checker lives in oracle/)",
    "BenchCell": "bench harness objects: use `joinqr bench` (cli.py) or bench.py",
    "BenchReport": "bench harness objects: use `joinqr bench` (cli.py) or bench.py",
    "run_bench": "bench harness objects: use `joinqr bench` (cli.py) or bench.py",
    "track_peak_memory": "host allocation tracking of the CPU harness (no GPU counterpart)",
}


def __getattr__(name):
    if name in _OUT_OF_SCOPE:
        raise AttributeError(f"{name} is not part of the B200 hot path: {_OUT_OF_SCOPE[name]}")
    try:
        module_name = _EXPORTS[name]
    except KeyError:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}") from None
    value = getattr(importlib.import_module(module_name, __name__), name)
    globals()[name] = value
    return value


def __dir__():
    return sorted(set(globals()) | set(_EXPORTS))
