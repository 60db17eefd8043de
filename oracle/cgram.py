"""ctypes binding of oracle/c/gram_oracle.c (factorised join Gram of SplitMix64
tables, OpenMP).  Test infrastructure only (see oracle/__init__.py)."""
import ctypes as C
import os

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libjqoracle.so")


def available() -> bool:
    return os.path.exists(_LIB)


def join_gram(seed_a, m1, n1, seed_b, m2, n2, keys_a=None, keys_b=None) -> np.ndarray:
    lib = C.CDLL(_LIB)
    f = lib.jq_oracle_gram
    f.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_void_p, C.c_uint64, C.c_int64, C.c_int, C.c_void_p,
                  C.c_void_p]
    n = n1 + n2
    g = np.zeros((n, n))
    ka = None if keys_a is None else np.ascontiguousarray(keys_a, dtype=np.int64)
    kb = None if keys_b is None else np.ascontiguousarray(keys_b, dtype=np.int64)
    f(seed_a, m1, n1, None if ka is None else ka.ctypes.data, seed_b, m2, n2,
      None if kb is None else kb.ctypes.data, g.ctypes.data)
    return g
