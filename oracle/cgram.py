"""ctypes binding of oracle/c/gram_oracle.c (factorised join Gram of SplitMix64
tables, OpenMP).  Test infrastructure only (see oracle/__init__.py)."""
import ctypes as C
import os

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libjqoracle.so")


def available() -> bool:
    return os.path.exists(_LIB)


def join_gram(seed_a, m1, n1, seed_b, m2, n2, keys_a=None, keys_b=None, perm_a=None, perm_b=None) -> np.ndarray:
    """perm_x[r] = the generation row of row r (tables permuted by a stable key sort)."""
    lib = C.CDLL(_LIB)
    f = lib.jq_oracle_gram_perm
    f.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int64, C.c_int,
                  C.c_void_p, C.c_void_p, C.c_void_p]
    n = n1 + n2
    g = np.zeros((n, n))
    conv = lambda x: None if x is None else np.ascontiguousarray(x, dtype=np.int64)
    ka, kb, pa, pb = conv(keys_a), conv(keys_b), conv(perm_a), conv(perm_b)
    ptr = lambda x: None if x is None else x.ctypes.data
    f(seed_a, m1, n1, ptr(ka), ptr(pa), seed_b, m2, n2, ptr(kb), ptr(pb), g.ctypes.data)
    return g
