"""CPU-side checks of the C-ABI boundary: libjoinqr.so loads, exports exactly the
entry points include/joinqr.h declares, and fails loudly without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "joinqr.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^JQ_API\s+[\w\s\*]+?\b(jq_\w+)\s*\(", src, re.M)))


def test_header_declares_the_api():
    names = declared_symbols()
    for n in ["jq_figaro_r", "jq_figaro_svd", "jq_svd_of_r", "jq_householder_r", "jq_reduce",
              "jq_head_tail", "jq_group_keys", "jq_canonicalize", "jq_tsqr_stack"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2503_23385_b200 import _native as N
    lib = N.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, f"{name} missing from the ctypes binding"
    assert lib.jq_version() == 100


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2503_23385_b200 import _native as N
    with pytest.raises(RuntimeError, match="no CUDA device"):
        N.ctx()
    import numpy as np
    import paper_2503_23385_b200 as P
    with pytest.raises(RuntimeError):
        P.figaro_r(P.Table(np.ones((2, 1))), P.Table(np.ones((2, 1))))


def test_drop_in_names_match_reference_exports():
    """Every hot-path name of the reference export table resolves in the mirror."""
    import paper_2503_23385_b200 as P
    import joinqr
    ref = ["matmul", "gram", "max_abs_diff", "transpose", "frobenius_norm", "hconcat", "vconcat",
           "scale", "row_slice", "is_upper_triangular", "head", "tail", "head_tail", "Table",
           "ReducedMatrix", "reduce_cartesian", "reduce_natural_join", "reduce_join",
           "householder_r", "canonicalize", "figaro_r", "SvdResult", "svd_of_r", "figaro_svd",
           "GenSpec", "gen_uniform", "materialize_cartesian", "materialize_natural_join", "baseline_r",
           "baseline_svd", "read_table", "read_matrix", "write_matrix", "write_table", "write_svd"]
    for n in ref:
        assert getattr(P, n) is getattr(joinqr, n)
    with pytest.raises(AttributeError, match="not part of the B200 hot path"):
        P.det_lu


def test_host_validation_errors_before_any_gpu_work():
    import numpy as np
    import paper_2503_23385_b200 as P
    with pytest.raises(ValueError):
        P.Table(np.ones((3, 2)), keys=[1, 2])             # key length mismatch
    with pytest.raises(ValueError):
        P.figaro_r(P.Table(np.ones((2, 1)), [1, 1]), P.Table(np.ones((2, 1))))
    with pytest.raises(ValueError):
        P.reduce_cartesian(np.zeros((0, 2)), np.ones((2, 2)))
    with pytest.raises(ValueError):
        P.head_tail(np.zeros((0, 3)))
    with pytest.raises(ValueError):
        P.householder_r(np.zeros((3, 0)))
    with pytest.raises(ValueError, match="square"):
        P.svd_of_r(np.ones((3, 4)))                        # R is n x n
    with pytest.raises(ValueError, match="square"):
        P.svd_of_r(np.ones((4, 3)), True)
    with pytest.raises(ValueError, match="512"):
        P.svd_of_r(np.eye(513))                            # wide cap (jq_svd.cu coop kernel)


def test_default_stream_maps_to_legacy_handle():
    """torch's default stream (handle 0) must reach the library as cudaStreamLegacy:
    NULL would select the library's own non-blocking stream (no ordering with torch)."""
    from paper_2503_23385_b200 import _native as N
    assert N.CUDA_STREAM_LEGACY == 1


def test_timing_struct_matches_header():
    """jq_timing (include/joinqr.h) and the ctypes mirror list the same fields in order."""
    import re
    from paper_2503_23385_b200._native import JqTiming
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "joinqr.h")).read()
    body = re.search(r"typedef struct jq_timing \{(.*?)\} jq_timing;", hdr, re.S).group(1)
    names = re.findall(r"^\s*(?:double|int64_t)\s+(\w+);", body, re.M)
    assert names == [f for f, _ in JqTiming._fields_]
