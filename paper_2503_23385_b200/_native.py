"""ctypes binding of libjoinqr.so (include/joinqr.h) — the only way the package
reaches the GPU.  There is no CPU fallback: if the library or a B200 is missing,
every call raises.

Arrays may be numpy arrays (host memory; the library copies them in and out) or
torch CUDA tensors (device memory, used in place).  Error codes map to the
reference's exception types (ValueError for bad input, RuntimeError for Jacobi
non-convergence / CUDA faults, MemoryError for allocation failures).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("JOINQR_LIB", os.path.join(_HERE, "lib", "libjoinqr.so"))

JQ_OK, JQ_E_INVALID, JQ_E_UNSORTED, JQ_E_KEYS, JQ_E_NOCONV, JQ_E_OOM, JQ_E_CUDA, JQ_E_NODEV = range(8)

_P = C.c_void_p
_I64 = C.c_int64

# name -> argtypes (restype int unless listed in _RESTYPE)
SIGNATURES = {
    "jq_version": [],
    "jq_last_error": [],
    "jq_ctx_create": [C.c_int, C.POINTER(_P)],
    "jq_ctx_destroy": [_P],
    "jq_ctx_set_stream": [_P, _P],
    "jq_ctx_sync": [_P],
    "jq_ctx_set_variant": [_P, C.c_int],
    "jq_last_timing": [_P, _P],
    "jq_kernel_launches": [_P],
    "jq_head_tail": [_P, _P, _I64, _I64, _P],
    "jq_group_keys": [_P, _P, _I64, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P],
    "jq_reduce": [_P, _P, _I64, _I64, _P, _P, _I64, _I64, _P, _P, _I64, _P, _P],
    "jq_householder_r": [_P, _P, _I64, _I64, _P],
    "jq_canonicalize": [_P, _P, _I64, _P],
    "jq_figaro_r": [_P, _P, _I64, _I64, _P, _P, _I64, _I64, _P, _P],
    "jq_svd_of_r": [_P, _P, _I64, C.c_int, _P, _P],
    "jq_figaro_svd": [_P, _P, _I64, _I64, _P, _P, _I64, _I64, _P, C.c_int, _P, _P, _P],
    "jq_gen_uniform": [_P, C.c_uint64, _I64, _I64, _I64, _P],
    "jq_gen_zipf_sorted_keys": [_P, C.c_uint64, _I64, _P, _I64, _P],
    "jq_gen_zipf_keys": [_P, C.c_uint64, _I64, _P, _I64, _P],
    "jq_sort_keys": [_P, _P, _I64, _P, _P],
    "jq_csv_scan": [C.c_char_p, C.c_int, _P, _P],
    "jq_csv_parse": [_P, C.c_char_p, C.c_int, C.c_int, _I64, _I64, _P, _P],
    "jq_gather_rows": [_P, _P, _I64, _I64, _P, _P],
    "jq_colsums": [_P, _P, _I64, _I64, _P],
    "jq_figaro_r_shard": [_P, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _P, C.c_int, _P],
    "jq_figaro_r_shard_local": [_P, _P, _I64, _I64, _I64, _P, _I64, _I64, _I64, _P, _P],
    "jq_tsqr_stack": [_P, _P, _I64, _I64, _P],
    "jq_split_group_rows": [_P, _P, _P, _P, _I64, _I64, _I64, _P, _I64, _P],
    "jq_materialize": [_P, _P, _I64, _I64, _P, _P, _I64, _I64, _P, _P, _I64, _P],
    "jq_join_r_bruteforce": [_P, _P, _I64, _I64, _P, _P, _I64, _I64, _P, _P],
}
_RESTYPE = {"jq_last_error": C.c_char_p, "jq_kernel_launches": C.c_int64}


class JqTiming(C.Structure):
    _fields_ = [("group_ms", C.c_double), ("scan_ms", C.c_double), ("tsqr_ms", C.c_double),
                ("tree_ms", C.c_double), ("svd_ms", C.c_double), ("total_ms", C.c_double),
                ("tsqr_ctas", C.c_int64), ("reduced_rows", C.c_int64),
                ("scan_tile_ms", C.c_double), ("scan_tile_bytes", C.c_double)]


_lib = None
_lib_lock = threading.Lock()
_tls = threading.local()


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libjoinqr.so and declare every entry point of include/joinqr.h."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ImportError(f"libjoinqr.so not found at {path}: build it with "
                                  "`python -c 'import __graft_entry__ as g; g.build()'` "
                                  "(there is no CPU fallback)")
            lib = C.CDLL(path)
            for name, args in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = _RESTYPE.get(name, C.c_int)
            _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == JQ_OK:
        return
    msg = load_library().jq_last_error().decode(errors="replace")
    if rc in (JQ_E_INVALID, JQ_E_UNSORTED, JQ_E_KEYS):
        raise ValueError(msg)
    if rc == JQ_E_OOM:
        raise MemoryError(msg)
    raise RuntimeError(f"libjoinqr error {rc}: {msg}")


_device = int(os.environ.get("JOINQR_DEVICE", "0"))


def set_device(device: int) -> None:
    """Select the GPU used by this thread's context (one process per GPU)."""
    global _device
    _device = int(device)
    if getattr(_tls, "ctx", None) is not None and _tls.device != _device:
        load_library().jq_ctx_destroy(_tls.ctx)
        _tls.ctx = None


VARIANTS = {"dense": 0, "footnote": 1, "auto": 2}
_variant = VARIANTS[os.environ.get("JOINQR_VARIANT", "auto")]


def get_variant() -> str:
    return {v: k for k, v in VARIANTS.items()}[_variant]


def set_variant(name: str) -> None:
    """figaro_r / figaro_svd internal reduction: "dense" = the Claim-1 reduced matrix
    (north star), "footnote" = head/tail of BOTH sides (PAPER.md:59
    footnote, 4x fewer TSQR flops at n1 = n2), "auto" (default) = footnote from
    (m1 + m2)(n1 + n2) > 1e8 reduced elements.  Same R (Gram-identical), parity-tested."""
    global _variant
    _variant = VARIANTS[name]
    c = getattr(_tls, "ctx", None)
    if c is not None:
        check(load_library().jq_ctx_set_variant(c, _variant))


def ctx():
    """This thread's library context (created on first use)."""
    c = getattr(_tls, "ctx", None)
    if c is None:
        lib = load_library()
        h = _P()
        check(lib.jq_ctx_create(_device, C.byref(h)))
        check(lib.jq_ctx_set_variant(h, _variant))
        _tls.ctx, _tls.device = h, _device
        c = h
    return c


def lib() -> C.CDLL:
    return load_library()


# ---------------------------------------------------------------- array hand-off
def is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def ptr(x):
    """Raw pointer of a numpy array / torch tensor (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data if x.size else None
    if is_torch_cuda(x) or type(x).__module__.startswith("torch"):
        return x.data_ptr() if x.numel() else None
    raise TypeError(f"unsupported array type {type(x)!r}")


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: the handle of the legacy default stream


def torch_stream_handle() -> int:
    """torch's current stream as a CUDA handle the library can order against.  torch
    reports its default stream as 0 (NULL), which the library would read as "use your
    own non-blocking stream" -- and a non-blocking stream does NOT wait for the legacy
    default stream, so the library could read a tensor before torch's producer kernel
    or non_blocking H2D copy has landed.  0 is therefore passed as cudaStreamLegacy."""
    import torch
    h = int(torch.cuda.current_stream().cuda_stream)
    return h if h != 0 else CUDA_STREAM_LEGACY


def use_torch_stream(*arrays) -> None:
    """Order library work after torch's producer kernels when device tensors flow in
    (the library then runs on torch's current stream, see torch_stream_handle)."""
    if any(is_torch_cuda(a) for a in arrays if a is not None):
        check(lib().jq_ctx_set_stream(ctx(), _P(torch_stream_handle())))
    else:
        check(lib().jq_ctx_set_stream(ctx(), None))


def last_timing() -> dict:
    t = JqTiming()
    check(lib().jq_last_timing(ctx(), C.byref(t)))
    return {f: getattr(t, f) for f, _ in JqTiming._fields_}


def kernel_launches() -> int:
    return int(lib().jq_kernel_launches(ctx()))
