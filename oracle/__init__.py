"""ctypes wrapper around the plain-C MMAS oracle (oracle/mmas_oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2003_11902_b200) never imports this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mmas_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("m", ctypes.c_int32), ("cl", ctypes.c_int32),
        ("alpha", ctypes.c_double), ("beta", ctypes.c_double), ("rho", ctypes.c_double),
        ("p_best", ctypes.c_double), ("seed", ctypes.c_uint64),
        ("deposit_global", ctypes.c_int32), ("fallback_argmax", ctypes.c_int32),
        ("local_search", ctypes.c_int32), ("nthreads", ctypes.c_int32),
        ("tabu", ctypes.c_int32), ("selection", ctypes.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.POINTER
        L.orc_philox4x32_10.argtypes = [P(ctypes.c_uint32), P(ctypes.c_uint32), P(ctypes.c_uint32)]
        L.orc_uniform.argtypes = [ctypes.c_uint32]
        L.orc_uniform.restype = ctypes.c_float
        L.orc_det_log2.argtypes = [ctypes.c_float]
        L.orc_det_log2.restype = ctypes.c_float
        L.orc_update_trails.argtypes = [P(ctypes.c_float), ctypes.c_int32, ctypes.c_double, ctypes.c_float,
                                        ctypes.c_float, P(ctypes.c_int32), ctypes.c_int64]
        L.orc_inv_w.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_int32]
        L.orc_inv_w.restype = ctypes.c_float
        L.orc_heur.argtypes = [ctypes.c_int32, ctypes.c_double]
        L.orc_heur.restype = ctypes.c_float
        L.orc_det_log2_many.argtypes = [P(ctypes.c_float), P(ctypes.c_float), ctypes.c_int64]
        L.orc_dist.argtypes =[P(ctypes.c_double), ctypes.c_int32, ctypes.c_int32]
        L.orc_dist.restype = ctypes.c_int32
        L.orc_tour_length.argtypes = [P(ctypes.c_double), ctypes.c_int32, P(ctypes.c_int32)]
        L.orc_tour_length.restype = ctypes.c_int64
        L.orc_nn_tour.argtypes = [P(ctypes.c_double), ctypes.c_int32, P(ctypes.c_int32)]
        L.orc_nn_tour.restype = ctypes.c_int64
        L.orc_cand_lists.argtypes = [P(ctypes.c_double), ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int32)]
        L.orc_limits_factor.argtypes = [ctypes.c_int32, ctypes.c_double]
        L.orc_limits_factor.restype = ctypes.c_double
        L.orc_limits.argtypes = [ctypes.c_double, ctypes.c_int64, ctypes.c_double, P(ctypes.c_float), P(ctypes.c_float)]
        L.orc_create.argtypes = [P(_Params), P(ctypes.c_double)]
        L.orc_create.restype = ctypes.c_void_p
        L.orc_destroy.argtypes = [ctypes.c_void_p]
        L.orc_iterate.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.orc_iterate.restype = ctypes.c_int
        L.orc_select_next.argtypes = [P(ctypes.c_float), P(ctypes.c_int32), ctypes.c_int32, ctypes.c_char_p,
                                      ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint32,
                                      P(ctypes.c_uint32), ctypes.c_int32, P(ctypes.c_int32)]
        L.orc_select_next.restype = ctypes.c_int32
        L.orc_start_node.argtypes = [ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint32, P(ctypes.c_uint32)]
        L.orc_start_node.restype = ctypes.c_int32
        L.orc_prwm.argtypes = [P(ctypes.c_float), ctypes.c_int32, ctypes.c_float]
        L.orc_prwm.restype = ctypes.c_int32
        L.orc_ct_init.argtypes = [P(ctypes.c_int32), P(ctypes.c_int32), ctypes.c_int32]
        L.orc_ct_mark.argtypes = [P(ctypes.c_int32), P(ctypes.c_int32), ctypes.c_int32, ctypes.c_int32]
        L.orc_select_next_ct.argtypes = [P(ctypes.c_float), P(ctypes.c_int32), ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_uint32, ctypes.c_uint32, P(ctypes.c_uint32)]
        L.orc_select_next_ct.restype = ctypes.c_int32
        for name in ("orc_iteration", "orc_ib_ant"):
            getattr(L, name).argtypes = [ctypes.c_void_p]
            getattr(L, name).restype = ctypes.c_int32
        L.orc_nn_length.argtypes = [ctypes.c_void_p]
        L.orc_nn_length.restype = ctypes.c_int64
        L.orc_factor.argtypes = [ctypes.c_void_p]
        L.orc_factor.restype = ctypes.c_double
        L.orc_get_limits.argtypes = [ctypes.c_void_p, P(ctypes.c_float), P(ctypes.c_float)]
        for name, ct in (("orc_get_tours", ctypes.c_int32), ("orc_get_lengths", ctypes.c_int64),
                         ("orc_get_fallbacks", ctypes.c_int64), ("orc_get_tau", ctypes.c_float),
                         ("orc_get_inv_w", ctypes.c_float), ("orc_get_heur", ctypes.c_float),
                         ("orc_get_cand", ctypes.c_int32)):
            getattr(L, name).argtypes = [ctypes.c_void_p, P(ct)]
        L.orc_reverse.argtypes = [P(ctypes.c_int32), P(ctypes.c_int32), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
        L.orc_two_opt.argtypes = [P(ctypes.c_double), ctypes.c_int32, P(ctypes.c_int32), ctypes.c_int32,
                                  P(ctypes.c_int32), P(ctypes.c_int64)]
        L.orc_two_opt.restype = ctypes.c_int64
        L.orc_construct_ant.argtypes = [ctypes.c_void_p, ctypes.c_int32, P(ctypes.c_int32), P(ctypes.c_int64)]
        L.orc_construct_ant.restype = ctypes.c_int64
        L.orc_best_tour.argtypes = [ctypes.c_void_p, P(ctypes.c_int32)]
        L.orc_best_tour.restype = ctypes.c_int64
        _lib = L
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


# ---- primitives ---------------------------------------------------------------
def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c, ctypes.c_uint32), _ptr(k, ctypes.c_uint32), _ptr(out, ctypes.c_uint32))
    return out


def uniform(x: int) -> float:
    return lib().orc_uniform(int(x) & 0xFFFFFFFF)


def det_log2(u: float) -> float:
    return lib().orc_det_log2(float(u))


def det_log2_many(u: np.ndarray) -> np.ndarray:
    uu = np.ascontiguousarray(u, dtype=np.float32)
    out = np.empty_like(uu)
    lib().orc_det_log2_many(_ptr(uu, ctypes.c_float), _ptr(out, ctypes.c_float), uu.size)
    return out


def dist(coords: np.ndarray, i: int, j: int) -> int:
    c = np.ascontiguousarray(coords, dtype=np.float64).ravel()
    return lib().orc_dist(_ptr(c, ctypes.c_double), i, j)


def tour_length(coords: np.ndarray, route) -> int:
    c = np.ascontiguousarray(coords, dtype=np.float64).ravel()
    r = np.ascontiguousarray(route, dtype=np.int32)
    return lib().orc_tour_length(_ptr(c, ctypes.c_double), len(r), _ptr(r, ctypes.c_int32))


def nn_tour(coords: np.ndarray):
    c = np.ascontiguousarray(coords, dtype=np.float64).ravel()
    n = len(c) // 2
    r = np.zeros(n, dtype=np.int32)
    L = lib().orc_nn_tour(_ptr(c, ctypes.c_double), n, _ptr(r, ctypes.c_int32))
    return r, L


def cand_lists(coords: np.ndarray, cl: int) -> np.ndarray:
    c = np.ascontiguousarray(coords, dtype=np.float64).ravel()
    n = len(c) // 2
    out = np.zeros((n, cl), dtype=np.int32)
    lib().orc_cand_lists(_ptr(c, ctypes.c_double), n, cl, _ptr(out, ctypes.c_int32))
    return out


def limits_factor(n: int, p_best: float = 0.01) -> float:
    return lib().orc_limits_factor(n, p_best)


def limits(rho: float, cost: int, factor: float):
    tn, tx = ctypes.c_float(), ctypes.c_float()
    lib().orc_limits(rho, int(cost), factor, ctypes.byref(tn), ctypes.byref(tx))
    return tn.value, tx.value


def update_trails(tau: np.ndarray, rho: float, tmin: float, tmax: float, route, cost: int) -> np.ndarray:
    """Evaporate + deposit + clamp on a copy of the n x n matrix tau (Alg. 1)."""
    t = np.array(tau, dtype=np.float32, copy=True, order="C")
    r = np.ascontiguousarray(route, dtype=np.int32)
    lib().orc_update_trails(_ptr(t, ctypes.c_float), t.shape[0], rho, tmin, tmax, _ptr(r, ctypes.c_int32), int(cost))
    return t


def inv_w(tau: float, heur: float, alpha: int = 1) -> float:
    return lib().orc_inv_w(tau, heur, alpha)


def heur(d: int, beta: float = 2.0) -> float:
    return lib().orc_heur(d, beta)


def reverse(route, i, j):
    """The 2-opt segment reversal (R25) on a copy of `route`."""
    r = np.array(route, dtype=np.int32, copy=True)
    pos = np.zeros(len(r), dtype=np.int32)
    pos[r] = np.arange(len(r), dtype=np.int32)
    lib().orc_reverse(_ptr(r, ctypes.c_int32), _ptr(pos, ctypes.c_int32), len(r), i, j)
    return r, pos


def two_opt(coords, route, K=32):
    """2-opt with neighbour lists and a FIFO of active nodes (row a8, R25).
    Returns (new_route, length_delta, moves)."""
    c = np.ascontiguousarray(coords, dtype=np.float64).ravel()
    n = len(c) // 2
    K = min(K, n - 1)
    nn = cand_lists(coords, K)
    r = np.array(route, dtype=np.int32, copy=True)
    moves = ctypes.c_int64()
    d = lib().orc_two_opt(_ptr(c, ctypes.c_double), n, _ptr(nn, ctypes.c_int32), K, _ptr(r, ctypes.c_int32),
                          ctypes.byref(moves))
    return r, int(d), moves.value


def select_next(inv_w_row, cand_row, visited, s, a, it, seed, fallback_argmax=0):
    """One node-selection step (exposed for the sampler pins)."""
    w = np.ascontiguousarray(inv_w_row, dtype=np.float32)
    cr = np.ascontiguousarray(cand_row if cand_row is not None else [], dtype=np.int32)
    vis = bytes(np.asarray(visited, dtype=np.uint8))
    key = np.array([seed & 0xFFFFFFFF, seed >> 32], dtype=np.uint32)
    fb = ctypes.c_int32()
    c = lib().orc_select_next(_ptr(w, ctypes.c_float), _ptr(cr, ctypes.c_int32) if len(cr) else None,
                              len(cr), vis, len(w), s, a, it, _ptr(key, ctypes.c_uint32),
                              fallback_argmax, ctypes.byref(fb))
    return c, fb.value


def ct_init(n):
    """Compact tabu: returns (entries, L)."""
    e = np.zeros(n, dtype=np.int32)
    L = ctypes.c_int32()
    lib().orc_ct_init(_ptr(e, ctypes.c_int32), ctypes.byref(L), n)
    return e, L.value


def ct_mark(entries, L, u):
    """CT mark(u) on a copy; returns (entries, L)."""
    e = np.array(entries, dtype=np.int32, copy=True)
    Lc = ctypes.c_int32(L)
    lib().orc_ct_mark(_ptr(e, ctypes.c_int32), ctypes.byref(Lc), len(e), int(u))
    return e, Lc.value


def select_next_ct(inv_w_row, entries, L, s, a, it, seed):
    """One full-row step over the CT's list (Alg. 3, R27)."""
    w = np.ascontiguousarray(inv_w_row, dtype=np.float32)
    e = np.ascontiguousarray(entries, dtype=np.int32)
    key = np.array([seed & 0xFFFFFFFF, seed >> 32], dtype=np.uint32)
    return lib().orc_select_next_ct(_ptr(w, ctypes.c_float), _ptr(e, ctypes.c_int32), int(L), s, a, it,
                                    _ptr(key, ctypes.c_uint32))


def prwm(weights, u):
    """Parallel roulette wheel over `weights` with uniform u (R28); -1 if all are 0."""
    w = np.ascontiguousarray(weights, dtype=np.float32)
    return lib().orc_prwm(_ptr(w, ctypes.c_float), len(w), float(np.float32(u)))


def start_node(n, a, it, seed):
    key = np.array([seed & 0xFFFFFFFF, seed >> 32], dtype=np.uint32)
    return lib().orc_start_node(n, a, it, _ptr(key, ctypes.c_uint32))


# ---- colony -------------------------------------------------------------------
class Colony:
    """The oracle's MMAS colony: Alg. 1 step by step on the CPU."""

    def __init__(self, coords, n_ants, cand_len, alpha=1.0, beta=2.0, rho=0.5, seed=42,
                 p_best=0.01, deposit_global=False, fallback_argmax=False, local_search=False,
                 nthreads=None, tabu=0, selection=0):
        c = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 2)
        self.coords = c
        self.n = c.shape[0]
        self.m = int(n_ants)
        self.cl = int(cand_len)
        if nthreads is None:
            nthreads = os.cpu_count() or 1
        p = _Params(self.n, self.m, self.cl, float(alpha), float(beta), float(rho), float(p_best),
                    int(seed) & 0xFFFFFFFFFFFFFFFF, int(deposit_global), int(fallback_argmax),
                    int(local_search), int(nthreads), int(tabu), int(selection))
        flat = c.ravel()
        h = lib().orc_create(ctypes.byref(p), _ptr(flat, ctypes.c_double))
        if not h:
            raise ValueError("oracle rejected the parameters")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().orc_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def iterate(self, iters=1):
        if lib().orc_iterate(self._h, int(iters)) != 0:
            raise ValueError("iters must be >= 1")

    @property
    def iteration(self):
        return lib().orc_iteration(self._h)

    @property
    def nn_length(self):
        return lib().orc_nn_length(self._h)

    @property
    def factor(self):
        return lib().orc_factor(self._h)

    @property
    def ib_ant(self):
        return lib().orc_ib_ant(self._h)

    def limits(self):
        tn, tx = ctypes.c_float(), ctypes.c_float()
        lib().orc_get_limits(self._h, ctypes.byref(tn), ctypes.byref(tx))
        return tn.value, tx.value

    def _get(self, name, shape, dt, ct):
        out = np.zeros(shape, dtype=dt)
        getattr(lib(), name)(self._h, _ptr(out, ct))
        return out

    def tours(self):
        return self._get("orc_get_tours", (self.m, self.n), np.int32, ctypes.c_int32)

    def lengths(self):
        return self._get("orc_get_lengths", (self.m,), np.int64, ctypes.c_int64)

    def fallbacks(self):
        return self._get("orc_get_fallbacks", (self.m,), np.int64, ctypes.c_int64)

    def tau(self):
        return self._get("orc_get_tau", (self.n, self.n), np.float32, ctypes.c_float)

    def inv_w(self):
        return self._get("orc_get_inv_w", (self.n, self.n), np.float32, ctypes.c_float)

    def heur(self):
        return self._get("orc_get_heur", (self.n, self.n), np.float32, ctypes.c_float)

    def cand(self):
        return self._get("orc_get_cand", (self.n, max(self.cl, 0)), np.int32, ctypes.c_int32)

    def construct_ant(self, a):
        """Route of global ant `a` at the current iteration (colony not advanced)."""
        out = np.zeros(self.n, dtype=np.int32)
        fb = ctypes.c_int64()
        L = lib().orc_construct_ant(self._h, int(a), _ptr(out, ctypes.c_int32), ctypes.byref(fb))
        return out, int(L), fb.value

    def best_tour(self):
        out = np.zeros(self.n, dtype=np.int32)
        L = lib().orc_best_tour(self._h, _ptr(out, ctypes.c_int32))
        return (None, None) if L < 0 else (out, L)
