"""Seeded synthetic inputs shared by the oracle tests, the CUDA-path tests and bench.py.

Holds none of the method's arithmetic (see gompgen.c). Generators return numpy uint8 arrays.
Recipes: DESIGN.md §4.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libgompgen.so")
        if not os.path.exists(path):
            raise RuntimeError("datagen/libgompgen.so missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        for name in ("gg_wiki", "gg_text", "gg_matrix", "gg_random"):
            fn = getattr(lib, name)
            fn.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64]
            fn.restype = ctypes.c_int
        lib.gg_nested.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32]
        lib.gg_nested.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def _run(name, seed, n, *extra):
    out = np.empty(int(n), dtype=np.uint8)
    if n:
        rc = getattr(_lib(), name)(int(seed), out.ctypes.data, int(n), *extra)
        if rc != 0:
            raise ValueError(f"{name}: bad parameters {extra}")
    return out


def wiki(n, seed=2):
    """Wikipedia-XML-shaped text (paper dataset 1)."""
    return _run("gg_wiki", seed, n)


def text(n, seed=1):
    """English-like article text (config C1)."""
    return _run("gg_text", seed, n)


def matrix(n, seed=5):
    """MatrixMarket coordinate text shaped like Hollywood-2009."""
    return _run("gg_matrix", seed, n)


def nested(n, depth, seed=3):
    """Nesting-depth dataset of PAPER.md:583-613 (depth D in {1,2,4,8,16,32})."""
    return _run("gg_nested", seed, n, ctypes.c_uint32(depth))


def random_bytes(n, seed=7):
    return _run("gg_random", seed, n)


def zeros(n):
    return np.zeros(int(n), dtype=np.uint8)


GENERATORS = {"wiki": wiki, "text": text, "matrix": matrix, "random": random_bytes}
