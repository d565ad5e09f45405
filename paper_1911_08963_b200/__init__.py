"""B200-native Brouwer–Zimmermann minimum-distance engine (arXiv 1911.08963 hot path).

Python mirror of the reference's C++ interface for this path, over the C ABI
``include/mdg.h`` of ``lib/libmdg.so`` (ctypes). Names follow the reference
(``md::min_weight``, ``GammaSet``, ``run_bz_loop``, ``round_*``,
``lower_bound``, ``singleton_upper``, ``parse_matrix``); see the per-function
docstrings for the reference file:line each mirrors.

Matrices are numpy ``uint64`` arrays of shape (k, W), W = ceil(n/64), bit i of
a row in word i//64 at bit position i%64 (LSB-first, the reference's bit order).

There is no CPU fallback: every compute call goes to the CUDA engine, and
importing this package raises if ``libmdg.so`` is missing.
"""
from __future__ import annotations

import ctypes as C
import weakref
import os
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

__all__ = [
    "MdgError", "InvalidArgument", "OverflowError_", "CudaFailure", "lib", "Device", "GammaSet",
    "RoundOut", "RunResult", "min_weight", "min_weight_dist", "min_weight_multi", "run_bz_loop", "lower_bound",
    "singleton_upper", "brute_force", "bz_loop_batch", "nccl_unique_id", "parse_matrix", "serialize_matrix", "gen_matrix", "binomial",
    "rd_unrank", "rd_rank", "hash_rows", "rank_of", "words", "KERNEL_TAB", "KERNEL_RD",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MDG_LIB") or os.path.join(_HERE, "lib", "libmdg.so")  # MDG_LIB: A/B builds
KERNEL_TAB, KERNEL_RD = 0, 1


class MdgError(RuntimeError):
    """Internal / device failure (the reference's CLI exit code 1)."""


class InvalidArgument(ValueError):
    """std::invalid_argument family (ParseError, caps, bad config) — exit code 2."""


class OverflowError_(OverflowError):
    """std::overflow_error (binomial beyond 64 bits) — exit code 2."""


class CudaFailure(MdgError):
    """CUDA runtime failure."""


def words(n: int) -> int:
    return (n + 63) // 64


u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")


class _RoundOut(C.Structure):
    _fields_ = [("min_weight", C.c_uint32), ("stopped_early", C.c_uint32),
                ("bounded", C.c_uint32), ("plan_tag", C.c_uint32), ("argmin_key", C.c_uint64), ("combinations", C.c_uint64),
                ("evaluated", C.c_uint64), ("task_lo", C.c_uint64), ("task_hi", C.c_uint64),
                ("device_ms", C.c_double)]


class _Config(C.Structure):
    _fields_ = [("trials", C.c_uint32), ("seed", C.c_uint64), ("level_cap", C.c_uint32),
                ("kernel", C.c_int), ("want_witness", C.c_int), ("exact_rounds", C.c_int),
                ("gamma_search", C.c_int), ("split_min", C.c_uint64), ("workers", C.c_uint32)]


class _RunInfo(C.Structure):
    _fields_ = [(f, C.c_uint32) for f in ("d", "capped", "n", "k", "m", "k_last", "g_final",
                                          "n_rounds", "n_levels", "witness_ok")] + \
               [("combinations", C.c_uint64), ("evaluated", C.c_uint64),
                ("row_additions", C.c_uint64), ("wall_seconds", C.c_double),
                ("device_seconds", C.c_double), ("gamma_seconds", C.c_double),
                ("loop_seconds", C.c_double), ("launches", C.c_uint64), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64)]


class _RoundRec(C.Structure):
    _fields_ = [("c", C.c_uint32), ("j", C.c_uint32), ("w", C.c_uint32), ("U_after", C.c_uint32),
                ("bounded", C.c_uint32)]


class _LevelRec(C.Structure):
    _fields_ = [("c", C.c_uint32), ("L_after", C.c_uint32), ("U_after", C.c_uint32),
                ("pad", C.c_uint32)]


ROUND_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                       C.POINTER(C.c_uint32))
REDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_uint32)

_LIB = None

# exported symbols of include/mdg.h (tests check the .so exports exactly these)
SYMBOLS = {
    "mdg_last_error": (C.c_char_p, []),
    "mdg_version": (C.c_char_p, []),
    "mdg_open": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "mdg_close": (None, [C.c_void_p]),
    "mdg_load_gammas": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, u64p, C.c_void_p]),
    "mdg_round": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(_RoundOut)]),
    "mdg_round_tasks": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]),
    "mdg_round_split": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "mdg_plan_split": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "mdg_round_range": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                  C.c_uint64, C.POINTER(_RoundOut)]),
    "mdg_round_bounded": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.c_uint64, C.c_uint64, C.POINTER(_RoundOut)]),
    "mdg_round_hist": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, u64p, C.POINTER(_RoundOut)]),
    "mdg_shared_bound_create": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8)]),
    "mdg_shared_bound_open": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8)]),
    "mdg_shared_bound_close": (C.c_int, [C.c_void_p]),
    "mdg_round_hist_dist": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, u64p,
                                      C.POINTER(_RoundOut), C.POINTER(C.c_int)]),
    "mdg_round_witness": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(_RoundOut), u32p]),
    "mdg_set_kernel": (C.c_int, [C.c_void_p, C.c_int]),
    "mdg_set_pruning": (C.c_int, [C.c_void_p, C.c_int]),
    "mdg_gset_build": (C.c_int, [u64p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                 C.POINTER(C.c_void_p)]),
    "mdg_gset_build_gpu": (C.c_int, [C.c_void_p, u64p, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_uint64, C.POINTER(C.c_void_p)]),
    "mdg_gset_compute": (C.c_int, [u64p, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]),
    "mdg_gset_free": (None, [C.c_void_p]),
    "mdg_gset_info": (C.c_int, [C.c_void_p] + [C.POINTER(C.c_uint32)] * 4),
    "mdg_gset_gamma": (C.c_int, [C.c_void_p, C.c_uint32, u64p]),
    "mdg_gset_ranks": (C.c_int, [C.c_void_p, u32p]),
    "mdg_gset_perm": (C.c_int, [C.c_void_p, u32p]),
    "mdg_gset_hash": (C.c_uint64, [C.c_void_p, C.c_uint32]),
    "mdg_load_gset": (C.c_int, [C.c_void_p, C.c_void_p]),
    "mdg_lower_bound": (C.c_uint32, [C.c_uint32] * 4),
    "mdg_singleton_upper": (C.c_uint32, [C.c_uint32] * 2),
    "mdg_bz_loop_cb": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, ROUND_FN,
                                 C.c_void_p, C.POINTER(C.c_void_p)]),
    "mdg_config_default": (None, [C.POINTER(_Config)]),
    "mdg_min_weight": (C.c_int, [C.c_void_p, u64p, C.c_uint32, C.c_uint32, C.POINTER(_Config),
                                 C.POINTER(C.c_void_p)]),
    "mdg_min_weight_dist": (C.c_int, [C.c_void_p, u64p, C.c_uint32, C.c_uint32,
                                      C.POINTER(_Config), C.c_uint32, C.c_uint32, C.c_void_p,
                                      C.c_void_p, C.POINTER(C.c_void_p)]),
    "mdg_min_weight_batch": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.POINTER(C.c_uint64)), u32p, u32p,
                                       C.POINTER(_Config), C.c_uint32, C.POINTER(C.c_void_p)]),
    "mdg_bz_loop_device_batch": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_uint32,
                                           C.POINTER(_Config), C.c_uint32, C.POINTER(C.c_void_p)]),
    "mdg_bz_loop_device": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(_Config),
                                     C.POINTER(C.c_void_p)]),
    "mdg_bz_loop_device_dist": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(_Config), C.c_uint32,
                                          C.c_uint32, C.c_void_p, C.c_void_p,
                                          C.POINTER(C.c_void_p)]),
    "mdg_timer_start": (C.c_int, [C.c_void_p]),
    "mdg_timer_stop": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "mdg_ctx_counters": (C.c_int, [C.c_void_p] + [C.POINTER(C.c_uint64)] * 3),
    "mdg_device_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "mdg_brute_force": (C.c_int, [C.c_void_p, u64p, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.POINTER(C.c_void_p)]),
    "mdg_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "mdg_nccl_init": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint32, C.c_uint32]),
    "mdg_nccl_reduce_min": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_uint32]),
    "mdg_group_create": (C.c_int, [C.c_uint32, C.POINTER(C.c_void_p)]),
    "mdg_group_free": (None, [C.c_void_p]),
    "mdg_group_attach": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32]),
    "mdg_group_reduce_min": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_uint32]),
    "mdg_min_weight_multi": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, u64p, C.c_uint32, C.c_uint32,
                                       C.POINTER(_Config), C.POINTER(C.c_void_p)]),
    "mdg_run_info_get": (C.c_int, [C.c_void_p, C.POINTER(_RunInfo)]),
    "mdg_run_rounds": (C.c_int, [C.c_void_p, C.POINTER(_RoundRec)]),
    "mdg_run_levels": (C.c_int, [C.c_void_p, C.POINTER(_LevelRec)]),
    "mdg_run_witness": (C.c_int, [C.c_void_p, u64p]),
    "mdg_run_perm": (C.c_int, [C.c_void_p, u32p]),
    "mdg_run_round_perf": (C.c_int, [C.c_void_p, u64p, np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")]),
    "mdg_run_gamma_hash": (C.c_uint64, [C.c_void_p, C.c_uint32]),
    "mdg_run_json": (C.c_long, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "mdg_run_free": (None, [C.c_void_p]),
    "mdg_parse_matrix": (C.c_int, [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                   C.c_void_p]),
    "mdg_serialize_matrix": (C.c_long, [u64p, C.c_uint32, C.c_uint32, C.c_char_p, C.c_size_t]),
    "mdg_gen_matrix": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, u64p]),
    "mdg_rank": (C.c_uint32, [u64p, C.c_uint32, C.c_uint32]),
    "mdg_hash_rows": (C.c_uint64, [u64p, C.c_uint32, C.c_uint32]),
    "mdg_binomial": (C.c_int, [C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]),
    "mdg_rd_unrank": (C.c_int, [C.c_uint32, C.c_uint64, u32p]),
    "mdg_rd_rank": (C.c_uint64, [C.c_uint32, u32p]),
}


def lib():
    """Load lib/libmdg.so (built by ``__graft_entry__.build()``); raise if absent."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SYMBOLS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().mdg_last_error().decode(errors="replace")
    if rc == -2:
        raise InvalidArgument(msg)
    if rc == -3:
        raise OverflowError_(msg)
    if rc == -4:
        raise CudaFailure(msg)
    raise MdgError(msg)


def _rows(G: np.ndarray) -> np.ndarray:
    G = np.ascontiguousarray(G, dtype=np.uint64)
    if G.ndim != 2:
        raise InvalidArgument("matrix must be a 2-D uint64 array (k, W)")
    return G


# ----------------------------------------------------------------- helpers
def lower_bound(m: int, g: int, k: int, k_last: int) -> int:
    """gamma.cpp:96-100: (m-1)(g+1) + max(0, g+1-k+k_last)."""
    return int(lib().mdg_lower_bound(m, g, k, k_last))


def singleton_upper(n: int, k: int) -> int:
    """gamma.cpp:102-106: n - k + 1; raises on n < k or k < 1."""
    if k < 1 or n < k:
        raise InvalidArgument("singleton_upper: need n >= k >= 1")
    return int(lib().mdg_singleton_upper(n, k))


def binomial(p: int, q: int) -> int:
    """enumeration.cpp:9-20 (raises OverflowError_ past 64 bits)."""
    out = C.c_uint64(0)
    _check(lib().mdg_binomial(p, q, C.byref(out)))
    return int(out.value)


def rd_unrank(c: int, rank: int) -> list:
    idx = np.zeros(c, dtype=np.uint32)
    _check(lib().mdg_rd_unrank(c, rank, idx))
    return [int(x) for x in idx]


def rd_rank(idx) -> int:
    a = np.ascontiguousarray(idx, dtype=np.uint32)
    return int(lib().mdg_rd_rank(len(a), a))


def parse_matrix(text: str) -> tuple[np.ndarray, int]:
    """io.cpp:33-73 — returns (rows, n); raises InvalidArgument('line L, column C: ...')."""
    k, n = C.c_uint32(0), C.c_uint32(0)
    b = text.encode()
    _check(lib().mdg_parse_matrix(b, C.byref(k), C.byref(n), None))
    rows = np.zeros((k.value, words(n.value)), dtype=np.uint64)
    _check(lib().mdg_parse_matrix(b, None, None, rows.ctypes.data))
    return rows, int(n.value)


def serialize_matrix(rows: np.ndarray, n: int) -> str:
    """io.cpp:81-88."""
    rows = _rows(rows)
    cap = rows.shape[0] * (n + 1) + 64
    buf = C.create_string_buffer(cap)
    ln = lib().mdg_serialize_matrix(rows, rows.shape[0], n, buf, cap)
    if ln < 0:
        _check(int(ln))
    return buf.value.decode()


def gen_matrix(n: int, k: int, seed: int, identity: bool = True) -> np.ndarray:
    """SURVEY.md §8d input generator: std::mt19937_64(seed), bit = draw & 1, row-major."""
    out = np.zeros((k, words(n)), dtype=np.uint64)
    _check(lib().mdg_gen_matrix(n, k, seed, 1 if identity else 0, out))
    return out


def rank_of(rows: np.ndarray, n: int) -> int:
    rows = _rows(rows)
    return int(lib().mdg_rank(rows, rows.shape[0], n))


def hash_rows(rows: np.ndarray, n: int) -> str:
    rows = _rows(rows)
    return "%016x" % lib().mdg_hash_rows(rows, rows.shape[0], n)


# --------------------------------------------------------------- GammaSet
class GammaSet:
    """gamma.hpp:14-24. ``GammaSet.build`` = best_gamma_over_permutations(row_basis(G))."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        m, k, n, kl = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(lib().mdg_gset_info(self._h, C.byref(m), C.byref(k), C.byref(n), C.byref(kl)))
        self.m, self.k, self.n, self.k_last = int(m.value), int(k.value), int(n.value), int(kl.value)

    @classmethod
    def build(cls, G: np.ndarray, n: int, trials: int = 10, seed: int = 0,
              device: Optional["Device"] = None) -> "GammaSet":
        """gamma.cpp:77-94 over row_basis(G) (f2core.cpp:92-97). With a device the trials
        run on the GPU (mdg_gset_build_gpu): the same Gamma set, faster for many trials."""
        G = _rows(G)
        h = C.c_void_p()
        if device is None:
            _check(lib().mdg_gset_build(G, G.shape[0], n, trials, seed, C.byref(h)))
        else:
            _check(lib().mdg_gset_build_gpu(device.handle, G, G.shape[0], n, trials, seed,
                                            C.byref(h)))
        return cls(h.value)

    @classmethod
    def compute(cls, G: np.ndarray, n: int) -> "GammaSet":
        """gamma.cpp:32-75 (identity permutation only)."""
        G = _rows(G)
        h = C.c_void_p()
        _check(lib().mdg_gset_compute(G, G.shape[0], n, C.byref(h)))
        return cls(h.value)

    def gamma(self, j: int) -> np.ndarray:
        out = np.zeros((self.k, words(self.n)), dtype=np.uint64)
        _check(lib().mdg_gset_gamma(self._h, j, out))
        return out

    @property
    def gammas(self) -> np.ndarray:
        return np.stack([self.gamma(j) for j in range(self.m)])

    @property
    def ranks(self) -> list:
        out = np.zeros(self.m, dtype=np.uint32)
        _check(lib().mdg_gset_ranks(self._h, out))
        return [int(x) for x in out]

    @property
    def column_perm(self) -> list:
        out = np.zeros(self.n, dtype=np.uint32)
        _check(lib().mdg_gset_perm(self._h, out))
        return [int(x) for x in out]

    def hash(self, j: int) -> str:
        return "%016x" % lib().mdg_gset_hash(self._h, j)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _LIB is not None:
            _LIB.mdg_gset_free(self._h)
            self._h = C.c_void_p()


# ------------------------------------------------------------------ device
@dataclass
class RoundOut:
    min_weight: int
    stopped_early: bool
    bounded: bool
    argmin_key: int
    combinations: int
    evaluated: int
    task_lo: int
    task_hi: int
    device_ms: float
    _raw: object = field(default=None, repr=False)


def _round_out(o: _RoundOut) -> RoundOut:
    raw = _RoundOut()
    C.pointer(raw)[0] = o
    return RoundOut(int(o.min_weight), bool(o.stopped_early), bool(o.bounded), int(o.argmin_key),
                    int(o.combinations), int(o.evaluated), int(o.task_lo), int(o.task_hi),
                    float(o.device_ms), raw)


class Device:
    """A CUDA context of the engine (mdg_open). Rounds mirror round_* (engines.hpp:140-146)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        _check(lib().mdg_open(device, C.byref(self._h)))

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h and self._h.value:
            lib().mdg_close(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_gammas(self, gammas: np.ndarray, n: int, ranks: Optional[list] = None):
        """mdg_load_gammas: gammas (m, k, W); ranks None = raw matrices (no identity elision)."""
        g = np.ascontiguousarray(gammas, dtype=np.uint64)
        if g.ndim == 2:
            g = g[None]
        m, k = g.shape[0], g.shape[1]
        flat = g.reshape(-1)
        r = None if ranks is None else np.ascontiguousarray(ranks, dtype=np.uint32)
        _check(lib().mdg_load_gammas(self._h, m, k, n, flat, None if r is None else r.ctypes.data))
        self._keep = r

    def load_gset(self, gs: GammaSet):
        _check(lib().mdg_load_gset(self._h, gs._h))

    def set_kernel(self, kernel: int):
        _check(lib().mdg_set_kernel(self._h, kernel))

    def set_pruning(self, on: bool):
        """Stage-1 bound pruning of the tab kernel (default on); off = every weight exact."""
        _check(lib().mdg_set_pruning(self._h, 1 if on else 0))

    def round(self, j: int, c: int, stop_at: int = 0) -> RoundOut:
        o = _RoundOut()
        _check(lib().mdg_round(self._h, j, c, stop_at, C.byref(o)))
        return _round_out(o)

    def tasks(self, j: int, c: int) -> int:
        t = C.c_uint64(0)
        _check(lib().mdg_round_tasks(self._h, j, c, C.byref(t)))
        return int(t.value)

    def split_range(self, j: int, c: int, rank: int, world: int) -> tuple:
        """rank's codeword-balanced task range of round (j, c) (mdg_round_split)"""
        lo, hi = C.c_uint64(0), C.c_uint64(0)
        _check(lib().mdg_round_split(self._h, j, c, rank, world, C.byref(lo), C.byref(hi)))
        return int(lo.value), int(hi.value)

    def round_range(self, j: int, c: int, task_lo: int, task_hi: int, stop_at: int = 0) -> RoundOut:
        o = _RoundOut()
        _check(lib().mdg_round_range(self._h, j, c, stop_at, task_lo, task_hi, C.byref(o)))
        return _round_out(o)

    def round_bounded(self, j: int, c: int, cutoff: int, stop_at: int = 0, task_lo: int = 0,
                      task_hi: int = (1 << 64) - 1) -> RoundOut:
        """Round bounded by `cutoff` (only weights < cutoff matter): min(true min, cutoff)."""
        o = _RoundOut()
        _check(lib().mdg_round_bounded(self._h, j, c, stop_at, cutoff, task_lo, task_hi, C.byref(o)))
        return _round_out(o)

    def round_hist(self, j: int, c: int, n: int) -> tuple[RoundOut, np.ndarray]:
        hist = np.zeros(n + 1, dtype=np.uint64)
        o = _RoundOut()
        _check(lib().mdg_round_hist(self._h, j, c, hist, C.byref(o)))
        return _round_out(o), hist

    def round_hist_dist(self, j: int, c: int, n: int, rank: int, world: int):
        """mdg_round_hist_dist: this rank's share of round (j, c)'s histogram -- summed across
        the ranks over NCCL when a communicator is attached (reduced = True), else the rank's
        partial counts. Returns (RoundOut, hist, reduced)."""
        hist = np.zeros(n + 1, dtype=np.uint64)
        o = _RoundOut()
        red = C.c_int(0)
        _check(lib().mdg_round_hist_dist(self._h, j, c, rank, world, hist, C.byref(o), C.byref(red)))
        return _round_out(o), hist, bool(red.value)

    def shared_bound_create(self) -> bytes:
        """Rank 0 of a multi-process run: create the shared round-key ring; returns its 64-byte
        CUDA IPC handle for the other ranks' shared_bound_open (mdg_shared_bound_create)."""
        buf = (C.c_uint8 * 64)()
        _check(lib().mdg_shared_bound_create(self._h, buf))
        return bytes(buf)

    def shared_bound_open(self, handle: bytes):
        buf = (C.c_uint8 * 64).from_buffer_copy(handle)
        _check(lib().mdg_shared_bound_open(self._h, buf))

    def shared_bound_close(self):
        _check(lib().mdg_shared_bound_close(self._h))

    def round_witness(self, j: int, c: int, out: RoundOut) -> list:
        idx = np.zeros(c, dtype=np.uint32)
        _check(lib().mdg_round_witness(self._h, j, c, C.byref(out._raw), idx))
        return [int(x) for x in idx]

    def timer_start(self):
        _check(lib().mdg_timer_start(self._h))

    def timer_stop(self) -> float:
        """Milliseconds on the context's stream since timer_start (CUDA events)."""
        ms = C.c_double(0)
        _check(lib().mdg_timer_stop(self._h, C.byref(ms)))
        return float(ms.value)

    def counters(self) -> dict:
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().mdg_ctx_counters(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"launches": int(a.value), "h2d_bytes": int(b.value), "d2h_bytes": int(c.value)}

    def info(self) -> dict:
        sms, dev = C.c_int(), C.c_int()
        _check(lib().mdg_device_info(self._h, C.byref(sms), C.byref(dev)))
        return {"sm_count": int(sms.value), "device": int(dev.value)}

    def bz_loop(self, gs: "GammaSet", level_cap: int = 0, kernel: int = KERNEL_TAB,
                witness: bool = True, rank: int = 0, world: int = 1,
                reduce_min: Callable | str | None = None, exact_rounds: bool = False,
                split_min: int = 0) -> "RunResult":
        """run_bz_loop on the device over the Gamma set loaded with load_gset (no search,
        no upload): the device-resident level loop (+ witness). world > 1: see
        min_weight_dist (split_min)."""
        cfg = _config(0, 0, level_cap, kernel, witness, exact_rounds)
        cfg.split_min = split_min
        h = C.c_void_p()
        if world == 1:
            _check(lib().mdg_bz_loop_device(self._h, gs._h, C.byref(cfg), C.byref(h)))
        else:
            fn, user, keep = _reducer(reduce_min, self)
            _check(lib().mdg_bz_loop_device_dist(self._h, gs._h, C.byref(cfg), rank, world, fn,
                                                 user, C.byref(h)))
            del keep
        return _collect(h)

    def nccl_init(self, uid: bytes, rank: int, world: int):
        _check(lib().mdg_nccl_init(self._h, uid, rank, world))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().mdg_nccl_unique_id(buf))
    return buf.raw


# ------------------------------------------------------------------ runs
class RunResult:
    """One min_weight / bz_loop / brute-force run. Scalars come with the result; the per-round
    and per-level traces, column_perm, Gamma hashes, witness and JSON record are read from
    the C run object on first use (it is freed with this object)."""

    _SCALARS = ("d", "capped", "n", "k", "m", "k_last", "g_final", "witness_ok", "combinations",
                "evaluated", "row_additions", "wall_seconds", "device_seconds", "gamma_seconds",
                "loop_seconds", "launches", "h2d_bytes", "d2h_bytes")

    def __init__(self, h):
        info = _RunInfo()
        _check(lib().mdg_run_info_get(h, C.byref(info)))
        self._h = h
        self._info = info
        self._fin = weakref.finalize(self, lib().mdg_run_free, h)
        self._cache = {}
        for f in self._SCALARS:
            v = getattr(info, f)
            setattr(self, f, bool(v) if f in ("capped", "witness_ok") else v)

    def _rounds(self):
        if "rounds" not in self._cache:
            nr = self._info.n_rounds
            rr = (_RoundRec * max(1, nr))()
            _check(lib().mdg_run_rounds(self._h, rr))
            pe = np.zeros(max(1, nr), dtype=np.uint64)
            pm = np.zeros(max(1, nr), dtype=np.float64)
            _check(lib().mdg_run_round_perf(self._h, pe, pm))
            self._cache["rounds"] = ([[r.c, r.j, r.w, r.U_after] for r in rr[:nr]],
                                     [int(r.bounded) for r in rr[:nr]],
                                     [int(x) for x in pe[:nr]], [float(x) for x in pm[:nr]])
        return self._cache["rounds"]

    @property
    def rounds(self) -> list:            # [c, j, w, U_after]
        return self._rounds()[0]

    @property
    def round_bounded(self) -> list:     # per executed round: 1 when w is only the bound U
        return self._rounds()[1]

    @property
    def round_evaluated(self) -> list:   # per executed round: codewords evaluated (this rank)
        return self._rounds()[2]

    @property
    def round_ms(self) -> list:          # per executed round: kernel time
        return self._rounds()[3]

    @property
    def levels(self) -> list:            # [c, L_after, U_after]
        if "levels" not in self._cache:
            nl = self._info.n_levels
            ll = (_LevelRec * max(1, nl))()
            _check(lib().mdg_run_levels(self._h, ll))
            self._cache["levels"] = [[x.c, x.L_after, x.U_after] for x in ll[:nl]]
        return self._cache["levels"]

    @property
    def column_perm(self) -> list:
        if "perm" not in self._cache:
            perm = np.zeros(max(1, self.n), dtype=np.uint32)
            _check(lib().mdg_run_perm(self._h, perm))
            self._cache["perm"] = [int(x) for x in perm[: self.n]]
        return self._cache["perm"]

    @property
    def gamma_hash(self) -> list:
        if "hash" not in self._cache:
            self._cache["hash"] = ["%016x" % lib().mdg_run_gamma_hash(self._h, j) for j in range(self.m)]
        return self._cache["hash"]

    @property
    def witness(self) -> Optional[np.ndarray]:
        if "witness" not in self._cache:
            wit = np.zeros(words(self.n), dtype=np.uint64)
            self._cache["witness"] = wit if lib().mdg_run_witness(self._h, wit) == 0 else None
        return self._cache["witness"]

    @property
    def json(self) -> str:
        """The CLI's JSON record of this run (mdg_run_json)."""
        if "json" not in self._cache:
            cap = 1 << 12
            while True:
                buf = C.create_string_buffer(cap)
                ln = lib().mdg_run_json(self._h, buf, cap)
                if ln >= 0:
                    break
                cap = -ln + 16
            self._cache["json"] = buf.value.decode()
        return self._cache["json"]


def _collect(h) -> RunResult:
    return RunResult(h)


def _config(trials, seed, level_cap, kernel, witness, exact_rounds=False,
            gamma_search="host") -> _Config:
    cfg = _Config()
    lib().mdg_config_default(C.byref(cfg))
    cfg.trials, cfg.seed, cfg.level_cap = trials, seed, level_cap
    cfg.kernel, cfg.want_witness = kernel, 1 if witness else 0
    cfg.exact_rounds = 1 if exact_rounds else 0
    if gamma_search not in ("host", "gpu"):
        raise InvalidArgument("gamma_search must be 'host' or 'gpu'")
    cfg.gamma_search = 1 if gamma_search == "gpu" else 0
    return cfg


def min_weight(G: np.ndarray, n: int, trials: int = 10, seed: int = 0, level_cap: int = 0,
               kernel: int = KERNEL_TAB, witness: bool = True,
               device: Optional[Device] = None, exact_rounds: bool = False,
               gamma_search: str = "host") -> RunResult:
    """md::min_weight (engines.cpp:617-648) with the GPU engine, plus trace and witness.
    exact_rounds=True computes every round's exact minimum (per-round trace parity);
    the default bounds rounds by U (identical d and (L, U) trace)."""
    G = _rows(G)
    h = C.c_void_p()
    cfg = _config(trials, seed, level_cap, kernel, witness, exact_rounds, gamma_search)
    _check(lib().mdg_min_weight(device.handle if device else None, G, G.shape[0], n,
                                C.byref(cfg), C.byref(h)))
    return _collect(h)


def min_weight_batch(Gs, n, trials: int = 10, seed=0, level_cap: int = 0,
                     kernel: int = KERNEL_TAB, witness: bool = True, device: Optional[Device] = None,
                     exact_rounds: bool = False, streams: int = 4, gamma_search: str = "host") -> list:
    """min_weight for many codes on one device (mdg_min_weight_batch): up to `streams` codes
    in flight, each on its own engine/stream, so host Gamma searches overlap device loops.
    Gs: sequence of packed row arrays; n and seed: one value for all codes or one per code.
    Returns one RunResult per code, each equal to min_weight's."""
    if device is None:
        raise InvalidArgument("min_weight_batch needs a Device")
    mats = [_rows(G) for G in Gs]
    count = len(mats)
    ns = list(n) if hasattr(n, "__len__") else [n] * count
    if len(ns) != count:
        raise InvalidArgument("one n per code")
    P64 = C.POINTER(C.c_uint64)
    ptrs = (P64 * max(1, count))(*[m.ctypes.data_as(P64) for m in mats])
    ks = np.array([m.shape[0] for m in mats] or [0], dtype=np.uint32)
    nn = np.array(ns or [0], dtype=np.uint32)
    seeds = list(seed) if hasattr(seed, "__len__") else [seed] * count
    if len(seeds) != count:
        raise InvalidArgument("one seed per code")
    cfgs = (_Config * max(1, count))(*[_config(trials, sd, level_cap, kernel, witness, exact_rounds,
                                               gamma_search) for sd in seeds])
    hs = (C.c_void_p * max(1, count))()
    _check(lib().mdg_min_weight_batch(device.handle, count, ptrs, ks, nn, cfgs, streams, hs))
    return [_collect(C.c_void_p(hs[i])) for i in range(count)]


def min_weight_dist(G: np.ndarray, n: int, rank: int, world: int,
                    reduce_min: Callable[[np.ndarray], np.ndarray] | str = "nccl",
                    trials: int = 10, seed: int = 0, level_cap: int = 0,
                    kernel: int = KERNEL_TAB, witness: bool = True,
                    device: Optional[Device] = None, exact_rounds: bool = False,
                    split_min: int = 0) -> RunResult:
    """Multi-GPU min_weight: each rank evaluates a contiguous task range of every round of at
    least split_min codewords (0 = 2e8, 1 = every round; smaller rounds run whole on every
    rank); the per-round key is combined by NCCL allreduce(min) (reduce_min='nccl', device
    must have called nccl_init) or by a Python callable (numpy uint64 array -> elementwise
    global min)."""
    G = _rows(G)
    h = C.c_void_p()
    cfg = _config(trials, seed, level_cap, kernel, witness, exact_rounds)
    cfg.split_min = split_min
    fn, user, keep = _reducer(reduce_min, device)
    _check(lib().mdg_min_weight_dist(device.handle if device else None, G, G.shape[0], n,
                                     C.byref(cfg), rank, world, fn, user, C.byref(h)))
    del keep
    return _collect(h)


def bz_loop_batch(devices: list, gsets: list, level_cap: int = 0, kernel: int = KERNEL_TAB,
                  witness: bool = True, exact_rounds: bool = False, streams: int = 4) -> list:
    """Device-resident level loops of many codes at once (mdg_bz_loop_device_batch): gsets[i] is
    loaded in devices[i] (distinct Device objects), up to `streams` loops in flight from the
    library's worker threads. Returns one RunResult per code, each equal to Device.bz_loop's."""
    count = len(devices)
    if len(gsets) != count:
        raise InvalidArgument("bz_loop_batch: one Gamma set per device")
    cfg = _config(0, 0, level_cap, kernel, witness, exact_rounds)
    ctxs = (C.c_void_p * max(1, count))(*[d.handle.value for d in devices])
    gss = (C.c_void_p * max(1, count))(*[g._h.value for g in gsets])
    hs = (C.c_void_p * max(1, count))()
    _check(lib().mdg_bz_loop_device_batch(ctxs, gss, count, C.byref(cfg), streams, hs))
    return [_collect(C.c_void_p(hs[i])) for i in range(count)]


def min_weight_multi(G: np.ndarray, n: int, devices: list, trials: int = 10, seed: int = 0,
                     level_cap: int = 0, kernel: int = KERNEL_TAB, witness: bool = True,
                     exact_rounds: bool = False, split_min: int = 0) -> list:
    """Single-process multi-GPU min_weight (mdg_min_weight_multi): the contexts in `devices`
    (distinct Device objects; their GPUs may repeat) run one level loop together, every round
    of at least split_min codewords (0 = 2e8, 1 = every round) split across them and its key
    min-reduced through an in-process exchange group (stream-ordered events + a min kernel).
    Returns one RunResult per rank: the same d, trace and Gamma set on every rank."""
    G = _rows(G)
    world = len(devices)
    cfg = _config(trials, seed, level_cap, kernel, witness, exact_rounds)
    cfg.split_min = split_min
    ctxs = (C.c_void_p * max(1, world))(*[d.handle.value for d in devices])
    hs = (C.c_void_p * max(1, world))()
    _check(lib().mdg_min_weight_multi(ctxs, world, G, G.shape[0], n, C.byref(cfg), hs))
    return [_collect(C.c_void_p(hs[i])) for i in range(world)]


def plan_split(k: int, c: int, nw32: int, resident_blocks: int, rank: int, world: int) -> tuple:
    """Host-only tile plan split (mdg_plan_split): (task_lo, task_hi, codewords) of rank's range."""
    lo, hi, cw = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
    _check(lib().mdg_plan_split(k, c, nw32, resident_blocks, rank, world, C.byref(lo), C.byref(hi),
                                C.byref(cw)))
    return int(lo.value), int(hi.value), int(cw.value)


def brute_force(G: np.ndarray, n: int, brute_cap: int = 40,
                device: Optional[Device] = None) -> RunResult:
    """min_weight with Algorithm::brute_gray (engines.cpp:480-558, 623-628): all 2^k - 1
    nonzero codewords of row_basis(G) on the GPU; d + witness, no trace (m = k_last = 0)."""
    G = _rows(G)
    h = C.c_void_p()
    _check(lib().mdg_brute_force(device.handle if device else None, G, G.shape[0], n, brute_cap,
                                 C.byref(h)))
    return _collect(h)


def _reducer(reduce_min, device):
    if reduce_min == "nccl":
        return C.cast(lib().mdg_nccl_reduce_min, C.c_void_p), device.handle, None
    if reduce_min == "group":  # the context was attached to an exchange group
        return C.cast(lib().mdg_group_reduce_min, C.c_void_p), None, None

    def _cb(_user, keys, count):
        try:
            arr = np.ctypeslib.as_array(keys, shape=(count,))
            arr[:] = reduce_min(arr.copy())
            return 0
        except Exception:  # surfaced as a status
            return -1
    keep = REDUCE_FN(_cb)
    return C.cast(keep, C.c_void_p), None, keep


def run_bz_loop(gs: GammaSet, round_fn: Callable[[int, int, int], int], lower: int = 1,
                upper: Optional[int] = None, level_cap: int = 0) -> RunResult:
    """run_bz_loop (engines.cpp:447-476) in the native host library, driving a Python round
    ``round_fn(j, c, stop_at) -> w`` (the RoundRunner seam, engines.hpp:151)."""
    if upper is None:
        upper = singleton_upper(gs.n, gs.k)

    def _cb(_user, j, c, stop_at, w_out):
        try:
            w_out[0] = int(round_fn(int(j), int(c), int(stop_at)))
            return 0
        except Exception:
            return -1

    cb = ROUND_FN(_cb)
    h = C.c_void_p()
    _check(lib().mdg_bz_loop_cb(gs._h, lower, upper, level_cap, cb, None, C.byref(h)))
    return _collect(h)
