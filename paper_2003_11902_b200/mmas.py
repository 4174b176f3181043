"""Thin ctypes binding of the C ABI in include/mmas.h (argument marshalling only).

Every step of the hot path runs in libmmas.so's CUDA kernels; this module only
converts numpy / torch arguments to pointers.  It fails loudly when the library
is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MMAS_LIB: an alternative in-tree build of the same library (e.g. the -DMMAS_TRACE build
# tools/trace_phases.py makes); the CUDA path is the only path either way
LIB_PATH = os.environ.get("MMAS_LIB") or os.path.join(_HERE, "libmmas.so")

MMAS_OK, MMAS_EINVAL, MMAS_ENOMEM, MMAS_ECUDA, MMAS_ENCCL, MMAS_ESTATE, MMAS_ETIMEDOUT = 0, -1, -2, -3, -4, -5, -6
DEPOSIT_ITERATION_BEST, DEPOSIT_GLOBAL_BEST = 0, 1
FALLBACK_WRS, FALLBACK_ARGMAX = 0, 1
TABU_BITMASK, TABU_COMPACT = 0, 1
SELECT_WRS, SELECT_RWM = 0, 1
PHEROMONE_DENSE, PHEROMONE_LEAN = 0, 1

# every symbol include/mmas.h declares (checked by tests/test_capi.py)
EXPORTED = (
    "mmas_last_error", "mmas_config_init", "mmas_create", "mmas_create_ex", "mmas_iterate",
    "mmas_record_bytes", "mmas_construct", "mmas_update", "mmas_best_tour", "mmas_best_length",
    "mmas_best_length_async", "mmas_destroy",
    "mmas_exchange_bytes", "mmas_exchange_buffer", "mmas_exchange_ipc_handle", "mmas_exchange_open_ipc",
    "mmas_exchange_attach", "mmas_construct_publish", "mmas_update_exchange", "mmas_iterate_exchange",
    "mmas_exchange_status", "mmas_device_status",
    "mmas_select_colony", "mmas_colonies", "mmas_pheromone_bytes", "mmas_state_bytes", "mmas_save_state",
    "mmas_load_state", "mmas_n", "mmas_iteration", "mmas_get_tours", "mmas_get_lengths", "mmas_get_pheromone",
    "mmas_get_inv_w", "mmas_get_heuristic", "mmas_get_candidates", "mmas_get_limits",
    "mmas_get_stats", "mmas_profile", "mmas_get_phase_times", "mmas_kernel_launches",
    "mmas_stream", "mmas_sync", "mmas_debug_philox", "mmas_debug_log2",
    "mmas_debug_trace", "mmas_debug_trace_warps", "mmas_debug_fb_cycles",
)


class MMASError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"mmas error {status}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [
        ("coords", ctypes.POINTER(ctypes.c_double)), ("n", ctypes.c_int32),
        ("alpha", ctypes.c_double), ("beta", ctypes.c_double), ("rho", ctypes.c_double),
        ("n_ants", ctypes.c_int32), ("cand_len", ctypes.c_int32), ("seed", ctypes.c_uint64),
        ("p_best", ctypes.c_double), ("deposit", ctypes.c_int32), ("fallback", ctypes.c_int32),
        ("local_search", ctypes.c_int32), ("device", ctypes.c_int32), ("stream", ctypes.c_void_p),
        ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("use_caller_stream", ctypes.c_int32),
        ("tabu", ctypes.c_int32), ("selection", ctypes.c_int32), ("separate_update", ctypes.c_int32),
        ("colonies", ctypes.c_int32), ("pheromone", ctypes.c_int32),
    ]


class Stats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("fallback_steps", ctypes.c_int64),
                ("ant_steps", ctypes.c_int64), ("ants_local", ctypes.c_int32), ("first_ant", ctypes.c_int32),
                ("local_search_moves", ctypes.c_int64), ("update_fused", ctypes.c_int32),
                ("fallback_lane_cap", ctypes.c_int32)]


class PhaseTimes(ctypes.Structure):
    _fields_ = [("construct_ms", ctypes.c_double), ("select_ms", ctypes.c_double),
                ("update_ms", ctypes.c_double), ("local_search_ms", ctypes.c_double), ("iterations", ctypes.c_int64)]


_lib = None


def lib():
    """Load libmmas.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2003_11902_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, V = ctypes.POINTER, ctypes.c_void_p
    L.mmas_last_error.restype = ctypes.c_char_p
    L.mmas_config_init.argtypes = [P(Config)]
    L.mmas_create.argtypes = [P(ctypes.c_double), ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                              ctypes.c_double, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64]
    L.mmas_create.restype = V
    L.mmas_create_ex.argtypes = [P(Config), P(V)]
    L.mmas_iterate.argtypes = [V, ctypes.c_int32]
    L.mmas_record_bytes.argtypes = [V]
    L.mmas_record_bytes.restype = ctypes.c_int64
    L.mmas_construct.argtypes = [V, V]
    L.mmas_update.argtypes = [V, V, ctypes.c_int32]
    L.mmas_exchange_bytes.argtypes = [V]
    L.mmas_exchange_bytes.restype = ctypes.c_int64
    L.mmas_exchange_buffer.argtypes = [V, ctypes.POINTER(ctypes.c_void_p)]
    L.mmas_exchange_ipc_handle.argtypes = [V, ctypes.c_char_p]
    L.mmas_exchange_open_ipc.argtypes = [V, ctypes.c_char_p]
    L.mmas_exchange_attach.argtypes = [V, ctypes.POINTER(ctypes.c_void_p)]
    for name in ("mmas_construct_publish", "mmas_update_exchange", "mmas_exchange_status"):
        getattr(L, name).argtypes = [V]
    # symbols newer than round 1: an older in-tree build (A/B runs) may lack them;
    # tests/test_capi.py fails loudly on a library that does not export every one
    for name, args, res in (("mmas_device_status", [V], None), ("mmas_select_colony", [V, ctypes.c_int32], None),
                            ("mmas_colonies", [V], None), ("mmas_pheromone_bytes", [V], ctypes.c_int64),
                            ("mmas_state_bytes", [V], ctypes.c_int64),
                            ("mmas_save_state", [V, ctypes.c_void_p, ctypes.c_int64], None),
                            ("mmas_load_state", [V, ctypes.c_void_p, ctypes.c_int64], None)):
        if hasattr(L, name):
            getattr(L, name).argtypes = args
            if res is not None:
                getattr(L, name).restype = res
    L.mmas_iterate_exchange.argtypes = [V, ctypes.c_int32]
    L.mmas_best_tour.argtypes = [V, P(ctypes.c_int32)]
    L.mmas_best_tour.restype = ctypes.c_int64
    L.mmas_best_length.argtypes = [V]
    L.mmas_best_length.restype = ctypes.c_int64
    L.mmas_best_length_async.argtypes = [V, ctypes.c_void_p]
    L.mmas_destroy.argtypes = [V]
    L.mmas_destroy.restype = None
    L.mmas_n.argtypes = [V]
    L.mmas_iteration.argtypes = [V]
    L.mmas_get_tours.argtypes = [V, P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int32)]
    L.mmas_get_lengths.argtypes = [V, P(ctypes.c_int64)]
    for f in ("mmas_get_pheromone", "mmas_get_inv_w", "mmas_get_heuristic"):
        getattr(L, f).argtypes = [V, P(ctypes.c_float)]
    L.mmas_get_candidates.argtypes = [V, P(ctypes.c_int32)]
    L.mmas_get_limits.argtypes = [V, P(ctypes.c_float), P(ctypes.c_float)]
    L.mmas_get_stats.argtypes = [V, P(Stats)]
    L.mmas_profile.argtypes = [V, ctypes.c_int32]
    L.mmas_get_phase_times.argtypes = [V, P(PhaseTimes)]
    L.mmas_kernel_launches.argtypes = [V]
    L.mmas_kernel_launches.restype = ctypes.c_int64
    L.mmas_stream.argtypes = [V]
    L.mmas_stream.restype = V
    L.mmas_sync.argtypes = [V]
    L.mmas_debug_philox.argtypes = [P(ctypes.c_uint32), ctypes.c_int64, P(ctypes.c_uint32), P(ctypes.c_float)]
    L.mmas_debug_log2.argtypes = [P(ctypes.c_float), ctypes.c_int64, P(ctypes.c_float)]
    _lib = L
    return L


def _err(status):
    if status < 0:
        raise MMASError(status, lib().mmas_last_error().decode())
    return status


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class Colony:
    """One MMAS colony (shard) on one GPU; wraps an mmas_ctx*."""

    def __init__(self, coords, n_ants, cand_len, alpha=1.0, beta=2.0, rho=0.5, seed=42, p_best=0.01,
                 deposit_global=False, fallback_argmax=False, local_search=False, device=-1, stream=None,
                 rank=0, world=1, tabu=TABU_BITMASK, selection=SELECT_WRS,
                 separate_update=False, colonies=1, pheromone=PHEROMONE_DENSE):
        L = lib()
        c = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 2)
        self.n = c.shape[0]
        self.m = int(n_ants)
        self.cl = int(cand_len)
        cfg = Config()
        L.mmas_config_init(ctypes.byref(cfg))
        flat = c.ravel()
        cfg.coords = _ptr(flat, ctypes.c_double)
        cfg.n = self.n
        cfg.alpha, cfg.beta, cfg.rho = float(alpha), float(beta), float(rho)
        cfg.n_ants, cfg.cand_len = self.m, self.cl
        cfg.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        cfg.p_best = float(p_best)
        cfg.deposit = DEPOSIT_GLOBAL_BEST if deposit_global else DEPOSIT_ITERATION_BEST
        cfg.fallback = FALLBACK_ARGMAX if fallback_argmax else FALLBACK_WRS
        cfg.local_search = int(bool(local_search))
        cfg.device = int(device)
        # stream=None: a stream owned by the context; otherwise the given cudaStream_t
        # (0 = the legacy default stream, which is torch's default current stream)
        cfg.stream = stream if stream else None
        cfg.use_caller_stream = 0 if stream is None else 1
        cfg.rank, cfg.world = int(rank), int(world)
        cfg.tabu = int(tabu)
        cfg.selection = int(selection)
        cfg.separate_update = int(bool(separate_update))
        cfg.colonies = int(colonies)
        cfg.pheromone = int(pheromone)
        h = ctypes.c_void_p()
        _err(L.mmas_create_ex(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self.rank, self.world = int(rank), int(world)

    # -- lifecycle --
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().mmas_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- the path --
    def iterate(self, iters=1):
        _err(lib().mmas_iterate(self._h, int(iters)))

    @property
    def record_bytes(self):
        return int(lib().mmas_record_bytes(self._h))

    def construct(self, record_dev_ptr: int):
        _err(lib().mmas_construct(self._h, ctypes.c_void_p(record_dev_ptr)))

    # -- peer-memory exchange (include/mmas.h; R21 without a collective library) --
    def exchange_ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _err(lib().mmas_exchange_ipc_handle(self._h, buf))
        return buf.raw

    def exchange_open_ipc(self, handles):
        """handles: every rank's 64-byte handle in rank order."""
        blob = b"".join(handles)
        _err(lib().mmas_exchange_open_ipc(self._h, blob))

    def exchange_buffer(self) -> int:
        p = ctypes.c_void_p()
        _err(lib().mmas_exchange_buffer(self._h, ctypes.byref(p)))
        return p.value

    def exchange_attach(self, buffers):
        arr = (ctypes.c_void_p * len(buffers))(*buffers)
        _err(lib().mmas_exchange_attach(self._h, arr))

    def construct_publish(self):
        _err(lib().mmas_construct_publish(self._h))

    def update_exchange(self):
        _err(lib().mmas_update_exchange(self._h))

    def iterate_exchange(self, iters=1):
        _err(lib().mmas_iterate_exchange(self._h, int(iters)))

    def exchange_status(self):
        _err(lib().mmas_exchange_status(self._h))

    def status(self):
        """Raises MMASError (MMAS_ETIMEDOUT) if a bounded device-side wait gave up."""
        _err(lib().mmas_device_status(self._h))

    def update(self, records_dev_ptr: int, count: int):
        _err(lib().mmas_update(self._h, ctypes.c_void_p(records_dev_ptr), int(count)))

    def best_tour(self):
        out = np.zeros(self.n, dtype=np.int32)
        L = lib().mmas_best_tour(self._h, _ptr(out, ctypes.c_int32))
        if L == MMAS_ESTATE:
            return None, None
        _err(L)
        return out, int(L)

    def best_length(self):
        """Global best length only (synchronises; 8-byte read-back), None before iteration 1."""
        L = lib().mmas_best_length(self._h)
        if L == MMAS_ESTATE:
            return None
        return int(_err(L))

    def best_length_async(self, host_ptr: int):
        """Enqueue the 8-byte copy of the global best length (int64, -1 if none) to host_ptr
        (pinned host memory) on the context's stream; no synchronisation."""
        _err(lib().mmas_best_length_async(self._h, ctypes.c_void_p(host_ptr)))

    # -- introspection --
    @property
    def colonies(self):
        return int(lib().mmas_colonies(self._h))

    @property
    def pheromone_bytes(self):
        L = lib()
        if not hasattr(L, "mmas_pheromone_bytes"):   # an older in-tree build (A/B runs)
            return None
        return int(L.mmas_pheromone_bytes(self._h))

    def save_state(self) -> bytes:
        """Checkpoint: the colony's whole state (include/mmas.h mmas_save_state)."""
        L = lib()
        nb = int(_err(L.mmas_state_bytes(self._h)))
        buf = ctypes.create_string_buffer(nb)
        _err(L.mmas_save_state(self._h, buf, nb))
        return buf.raw

    def load_state(self, state: bytes):
        """Resume from save_state() of a context with the same coordinates and configuration."""
        buf = ctypes.create_string_buffer(bytes(state), len(state))
        _err(lib().mmas_load_state(self._h, buf, len(state)))

    def select_colony(self, colony: int):
        """Introspection and best_tour/best_length report colony `colony` from now on."""
        _err(lib().mmas_select_colony(self._h, int(colony)))

    @property
    def iteration(self):
        return int(lib().mmas_iteration(self._h))

    def tours(self):
        first, count = ctypes.c_int32(), ctypes.c_int32()
        _err(lib().mmas_get_tours(self._h, None, ctypes.byref(first), ctypes.byref(count)))
        out = np.zeros((count.value, self.n), dtype=np.int32)
        _err(lib().mmas_get_tours(self._h, _ptr(out, ctypes.c_int32), ctypes.byref(first), ctypes.byref(count)))
        return out

    def shard(self):
        first, count = ctypes.c_int32(), ctypes.c_int32()
        _err(lib().mmas_get_tours(self._h, None, ctypes.byref(first), ctypes.byref(count)))
        return first.value, count.value

    def lengths(self):
        _, count = self.shard()
        out = np.zeros(count, dtype=np.int64)
        _err(lib().mmas_get_lengths(self._h, _ptr(out, ctypes.c_int64)))
        return out

    def _matrix(self, fn):
        out = np.zeros((self.n, self.n), dtype=np.float32)
        _err(getattr(lib(), fn)(self._h, _ptr(out, ctypes.c_float)))
        return out

    def tau(self):
        return self._matrix("mmas_get_pheromone")

    def inv_w(self):
        return self._matrix("mmas_get_inv_w")

    def heur(self):
        return self._matrix("mmas_get_heuristic")

    def cand(self):
        out = np.zeros((self.n, self.cl), dtype=np.int32)
        _err(lib().mmas_get_candidates(self._h, _ptr(out, ctypes.c_int32)))
        return out

    def limits(self):
        tn, tx = ctypes.c_float(), ctypes.c_float()
        _err(lib().mmas_get_limits(self._h, ctypes.byref(tn), ctypes.byref(tx)))
        return tn.value, tx.value

    def stats(self):
        s = Stats()
        _err(lib().mmas_get_stats(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    def profile(self, enable=True):
        _err(lib().mmas_profile(self._h, int(bool(enable))))

    def phase_times(self):
        t = PhaseTimes()
        _err(lib().mmas_get_phase_times(self._h, ctypes.byref(t)))
        return {f: getattr(t, f) for f, _ in PhaseTimes._fields_}

    @property
    def kernel_launches(self):
        return int(lib().mmas_kernel_launches(self._h))

    @property
    def stream(self):
        return lib().mmas_stream(self._h)

    def sync(self):
        _err(lib().mmas_sync(self._h))


def debug_philox(ctr_key: np.ndarray):
    """Device Philox4x32-10 + det_log2 on rows (c0, c1, c2, c3, k0, k1) -> (words[.,4], log2u[.,4])."""
    ck = np.ascontiguousarray(ctr_key, dtype=np.uint32).reshape(-1, 6)
    words = np.zeros((ck.shape[0], 4), dtype=np.uint32)
    logs = np.zeros((ck.shape[0], 4), dtype=np.float32)
    _err(lib().mmas_debug_philox(_ptr(ck, ctypes.c_uint32), ck.shape[0], _ptr(words, ctypes.c_uint32),
                                 _ptr(logs, ctypes.c_float)))
    return words, logs


def debug_log2(u: np.ndarray) -> np.ndarray:
    uu = np.ascontiguousarray(u, dtype=np.float32)
    out = np.zeros_like(uu)
    _err(lib().mmas_debug_log2(_ptr(uu, ctypes.c_float), uu.size, _ptr(out, ctypes.c_float)))
    return out
