"""TEST INFRASTRUCTURE — ctypes wrapper of the plain-C restatement (mdoracle.c).

Matrices are numpy ``uint64`` arrays of shape (k, W), W = ceil(n/64), bit i of
a row in word i//64 at position i%64 (LSB-first, the reference's bit order).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")


class _RoundRec(C.Structure):
    _fields_ = [("c", C.c_uint32), ("j", C.c_uint32), ("w", C.c_uint32), ("U_after", C.c_uint32)]


class _LevelRec(C.Structure):
    _fields_ = [("c", C.c_uint32), ("L_after", C.c_uint32), ("U_after", C.c_uint32)]


class _Result(C.Structure):
    _fields_ = [(f, C.c_uint32) for f in
                ("d", "capped", "m", "k", "n", "k_last", "g_final", "n_rounds", "n_levels")] + \
               [("combinations", C.c_uint64)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "build", "libmdoracle.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.run(["make", "-C", _HERE, "oracle"], check=True, capture_output=True)
        L = C.CDLL(path)
        L.mdo_gen_matrix.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, u64p]
        L.mdo_rank.argtypes = [u64p, C.c_uint32, C.c_uint32]
        L.mdo_rank.restype = C.c_uint32
        L.mdo_row_basis.argtypes = [u64p, C.c_uint32, C.c_uint32, u64p]
        L.mdo_row_basis.restype = C.c_uint32
        for f in (L.mdo_best_gamma,):
            f.argtypes = [u64p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, u64p, u32p, u32p,
                          C.POINTER(C.c_uint32)]
            f.restype = C.c_uint32
        L.mdo_compute_gamma.argtypes = [u64p, C.c_uint32, C.c_uint32, u64p, u32p, u32p,
                                        C.POINTER(C.c_uint32)]
        L.mdo_compute_gamma.restype = C.c_uint32
        L.mdo_lower_bound.argtypes = [C.c_uint32] * 4
        L.mdo_lower_bound.restype = C.c_uint32
        L.mdo_singleton_upper.argtypes = [C.c_uint32] * 2
        L.mdo_singleton_upper.restype = C.c_uint32
        L.mdo_round.argtypes = [u64p, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]
        L.mdo_round.restype = C.c_uint32
        L.mdo_round_hist.argtypes = [u64p, C.c_uint32, C.c_uint32, C.c_uint32, u64p]
        L.mdo_round_hist.restype = C.c_uint32
        L.mdo_brute.argtypes = [u64p, C.c_uint32, C.c_uint32]
        L.mdo_brute.restype = C.c_uint32
        L.mdo_hash_rows.argtypes = [u64p, C.c_uint32, C.c_uint32]
        L.mdo_hash_rows.restype = C.c_uint64
        L.mdo_min_weight.argtypes = [u64p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                     C.c_uint32, C.POINTER(_Result), C.POINTER(_RoundRec),
                                     C.c_uint32, C.POINTER(_LevelRec), C.c_uint32, u32p, u64p]
        L.mdo_min_weight.restype = C.c_int
        _LIB = L
    return _LIB


def words(n: int) -> int:
    return (n + 63) // 64


def gen_matrix(n: int, k: int, seed: int, identity: bool = True) -> np.ndarray:
    out = np.zeros((k, words(n)), dtype=np.uint64)
    lib().mdo_gen_matrix(n, k, seed, 1 if identity else 0, out)
    return out


def rank(rows: np.ndarray, n: int) -> int:
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    return int(lib().mdo_rank(rows, rows.shape[0], n))


def row_basis(rows: np.ndarray, n: int) -> np.ndarray:
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    out = np.zeros_like(rows)
    r = lib().mdo_row_basis(rows, rows.shape[0], n, out)
    return out[:r]


def round_min(rows: np.ndarray, n: int, c: int) -> tuple[int, int]:
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    combos = C.c_uint64(0)
    w = lib().mdo_round(rows, rows.shape[0], n, c, C.byref(combos))
    return int(w), int(combos.value)


def round_hist(rows: np.ndarray, n: int, c: int) -> tuple[int, np.ndarray]:
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    hist = np.zeros(n + 1, dtype=np.uint64)
    w = lib().mdo_round_hist(rows, rows.shape[0], n, c, hist)
    return int(w), hist


def brute(rows: np.ndarray, n: int) -> int:
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    return int(lib().mdo_brute(rows, rows.shape[0], n))


def hash_rows(rows: np.ndarray, n: int) -> str:
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    return "%016x" % lib().mdo_hash_rows(rows, rows.shape[0], n)


@dataclass
class GammaSet:
    gammas: np.ndarray          # (m, k, W)
    ranks: list
    column_perm: list
    k_last: int

    @property
    def m(self):
        return self.gammas.shape[0]


def best_gamma(G: np.ndarray, n: int, trials: int, seed: int) -> GammaSet:
    G = np.ascontiguousarray(G, dtype=np.uint64)
    k, W = G.shape
    mmax = (n + k - 1) // k
    gam = np.zeros(mmax * k * W, dtype=np.uint64)
    ranks = np.zeros(mmax, dtype=np.uint32)
    perm = np.zeros(n, dtype=np.uint32)
    kl = C.c_uint32(0)
    m = lib().mdo_best_gamma(G, k, n, trials, seed, gam, ranks, perm, C.byref(kl))
    if m == 0:
        raise ValueError("best_gamma: rank-deficient or invalid matrix")
    return GammaSet(gam[: m * k * W].reshape(m, k, W), [int(x) for x in ranks[:m]],
                    [int(x) for x in perm], int(kl.value))


@dataclass
class Trace:
    d: int
    capped: bool
    m: int
    k: int
    n: int
    k_last: int
    g_final: int
    combinations: int
    rounds: list = field(default_factory=list)   # [c, j, w, U_after]
    levels: list = field(default_factory=list)   # [c, L_after, U_after]
    column_perm: list = field(default_factory=list)
    gamma_hash: list = field(default_factory=list)


def min_weight(G: np.ndarray, n: int, trials: int = 10, seed: int = 0, level_cap: int = 0) -> Trace:
    G = np.ascontiguousarray(G, dtype=np.uint64)
    k = G.shape[0]
    res = _Result()
    cap_r, cap_l = 4096, 1024
    rr = (_RoundRec * cap_r)()
    ll = (_LevelRec * cap_l)()
    perm = np.zeros(n, dtype=np.uint32)
    hashes = np.zeros(n + 1, dtype=np.uint64)
    rc = lib().mdo_min_weight(G, k, n, trials, seed, level_cap, C.byref(res), rr, cap_r, ll, cap_l,
                              perm, hashes)
    if rc != 0:
        raise ValueError("min_weight: invalid matrix")
    return Trace(
        d=res.d, capped=bool(res.capped), m=res.m, k=res.k, n=res.n, k_last=res.k_last,
        g_final=res.g_final, combinations=res.combinations,
        rounds=[[r.c, r.j, r.w, r.U_after] for r in rr[: min(res.n_rounds, cap_r)]],
        levels=[[x.c, x.L_after, x.U_after] for x in ll[: min(res.n_levels, cap_l)]],
        column_perm=[int(x) for x in perm],
        gamma_hash=["%016x" % int(h) for h in hashes[: res.m]],
    )


def parse_matrix_text(text: str) -> tuple[np.ndarray, int]:
    """Reference text format (io.cpp:33-73), lenient: header 'n k', k rows of 0/1, '#' comments."""
    lines = [ln.strip() for ln in text.splitlines()]
    lines = [ln for ln in lines if ln and not ln.startswith("#")]
    n, k = (int(x) for x in lines[0].split())
    rows = np.zeros((k, words(n)), dtype=np.uint64)
    for r in range(k):
        s = lines[1 + r]
        assert len(s) == n
        for c, ch in enumerate(s):
            if ch == "1":
                rows[r, c // 64] |= np.uint64(1) << np.uint64(c % 64)
    return rows, n


def matrix_text(rows: np.ndarray, n: int) -> str:
    """Reference serialization (io.cpp:81-88)."""
    k = rows.shape[0]
    out = [f"{n} {k}"]
    for r in range(k):
        out.append("".join("1" if (int(rows[r, c // 64]) >> (c % 64)) & 1 else "0" for c in range(n)))
    return "\n".join(out) + "\n"
