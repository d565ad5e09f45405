"""TEST INFRASTRUCTURE — ctypes wrapper of the compiled reference (oracle/_ref).

``libmdref.so`` is the unmodified reference library built with its own CMake
Release flags; ``libmdref_v3.so`` the same sources with ``-march=x86-64-v3``.
Both exist only where ``/root/reference`` was present at build time (this
container); the built files travel to the GPU box with the snapshot.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBS: dict = {}


def available(flavor: str = "v3") -> bool:
    return os.path.exists(_path(flavor))


def _path(flavor: str) -> str:
    return os.path.join(_HERE, "_ref", "libmdref.so" if flavor == "stock" else "libmdref_v3.so")


def lib(flavor: str = "v3"):
    if flavor not in _LIBS:
        L = C.CDLL(_path(flavor))
        L.mdref_trace.argtypes = [C.c_char_p, C.c_uint32, C.c_uint64, C.c_char_p, C.c_uint32,
                                  C.c_uint32, C.c_uint32, C.c_int, C.c_char_p, C.c_size_t]
        L.mdref_trace.restype = C.c_long
        L.mdref_round.argtypes = [np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS"),
                                  C.c_uint32, C.c_uint32, C.c_uint32, C.c_char_p, C.c_uint32,
                                  C.c_uint32, C.POINTER(C.c_uint64)]
        L.mdref_round.restype = C.c_long
        L.mdref_gen.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, C.c_char_p, C.c_size_t]
        L.mdref_gen.restype = C.c_long
        L.mdref_random_full_rank.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_char_p,
                                             C.c_size_t]
        L.mdref_random_full_rank.restype = C.c_long
        L.mdref_seeded_code.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_char_p,
                                        C.c_size_t]
        L.mdref_seeded_code.restype = C.c_long
        L.mdref_min_weight.argtypes = [C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint64, C.c_uint32]
        L.mdref_min_weight.restype = C.c_long
        _LIBS[flavor] = L
    return _LIBS[flavor]


def _text_call(fn, *args, cap=1 << 22) -> str:
    buf = C.create_string_buffer(cap)
    n = fn(*args, buf, cap)
    if n < 0:
        raise RuntimeError(buf.value.decode(errors="replace"))
    return buf.value.decode()


def trace(matrix_text: str, trials: int = 10, seed: int = 0, engine: str = "saved", s: int = 5,
          workers: int = 1, level_cap: int = 0, with_rows: bool = False, flavor: str = "v3") -> dict:
    L = lib(flavor)
    return json.loads(_text_call(L.mdref_trace, matrix_text.encode(), trials, seed, engine.encode(),
                                 s, workers, level_cap, 1 if with_rows else 0, cap=1 << 24))


def round_min(rows: np.ndarray, n: int, c: int, engine: str = "stack", s: int = 5, workers: int = 1,
              flavor: str = "v3") -> tuple[int, int]:
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    combos = C.c_uint64(0)
    w = lib(flavor).mdref_round(rows, rows.shape[0], n, c, engine.encode(), s, workers,
                                C.byref(combos))
    if w < 0:
        raise RuntimeError("mdref_round failed")
    return int(w), int(combos.value)


def gen(n: int, k: int, seed: int, identity: bool = True, flavor: str = "v3") -> str:
    return _text_call(lib(flavor).mdref_gen, n, k, seed, 1 if identity else 0)


def random_full_rank(n: int, k: int, seed: int, flavor: str = "v3") -> str:
    return _text_call(lib(flavor).mdref_random_full_rank, n, k, seed)


def seeded_code(seed: int, n_lo: int = 8, n_span: int = 21, k_cap: int = 14,
                flavor: str = "v3") -> str:
    return _text_call(lib(flavor).mdref_seeded_code, seed, n_lo, n_span, k_cap)


def min_weight_d(matrix_text: str, algorithm: str = "saved", trials: int = 10, seed: int = 0,
                 workers: int = 1, flavor: str = "v3") -> int:
    d = lib(flavor).mdref_min_weight(matrix_text.encode(), algorithm.encode(), trials, seed, workers)
    if d < 0:
        raise RuntimeError("mdref_min_weight failed")
    return int(d)
