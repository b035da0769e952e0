"""ctypes binding of libgscan.so (include/gscan.h).

This is the only way the host package reaches the device: there is no CPU
fallback.  If the shared library is missing the import fails loudly with the
command that builds it.
"""

from __future__ import annotations

import ctypes
import os
import threading
from fractions import Fraction

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgscan.so")

GS_OK = 0
GS_EINVAL = 1
GS_EBUDGET = 2
GS_ECUDA = 3
GS_ENOMEM = 4
GS_EINTERNAL = 5
GS_EPARSE = 6

GS_PH_H2D, GS_PH_BUILD, GS_PH_IDENTIFY, GS_PH_CLEANUP = 0, 1, 2, 3
GS_PH_CLUSTER, GS_PH_CLASSIFY, GS_PH_D2H, GS_PH_TOTAL = 4, 5, 6, 7
GS_PH_SIM_KERNELS = 8
ABI_VERSION = 3  # GS_ABI_VERSION of include/gscan.h
# identify pass by kernel class (gs_stats.phase_ms / kernel_bytes order)
(GS_PH_K_PREP, GS_PH_K_HUGE, GS_PH_K_LARGE, GS_PH_K_MEDIUM, GS_PH_K_SMALL, GS_PH_K_TINY,
 GS_PH_K_SKETCH) = range(9, 16)
KERNEL_CLASSES = ("prep: thresholds + degree tables + hub split + sketch build + Lemma-1 pre-pass",
                  "k_sim_hash<1024,L2 table> (deg b >= 28672)",
                  "k_sim_hash<1024> (4096 <= deg b < 28672)",
                  "k_sim_hash<512> (512 <= deg b < 4096)",
                  "k_sim_warp (64 <= deg b < 512)",
                  "k_sim_tiny (deg b < 64)",
                  "k_sk_filter (sketch bound, thread per surviving edge, deg b >= 64)")
GS_PH_COUNT = 16


class GsEps2(ctypes.Structure):
    _fields_ = [
        ("p_lo", ctypes.c_uint64),
        ("p_hi", ctypes.c_uint64),
        ("q_lo", ctypes.c_uint64),
        ("q_hi", ctypes.c_uint64),
    ]


class GsStats(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("m", ctypes.c_int64),
        ("sim_evals", ctypes.c_int64),
        ("adj_probes", ctypes.c_int64),
        ("union_retries", ctypes.c_int64),
        ("probe_bound_violations", ctypes.c_int64),
        ("sim_decided_by_bound", ctypes.c_int64),
        ("sim_intersections", ctypes.c_int64),
        ("alg_bytes_sim", ctypes.c_int64),
        ("n_core", ctypes.c_int64),
        ("n_member", ctypes.c_int64),
        ("n_hub", ctypes.c_int64),
        ("n_outlier", ctypes.c_int64),
        ("n_clusters", ctypes.c_int64),
        ("partitions", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
        ("peak_device_bytes", ctypes.c_int64),
        ("sim_decided_by_sketch", ctypes.c_int64),
        ("phase_ms", ctypes.c_double * GS_PH_COUNT),
        ("kernel_bytes", ctypes.c_int64 * 7),
        ("wsim_bytes", ctypes.c_int64),
        ("pcie_bytes", ctypes.c_int64),
    ]


class InfeasibleBudget(ValueError):
    """GS_EBUDGET from the library (mapped to InfeasibleBudgetError above)."""


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32

# (name, restype, argtypes) for every symbol declared in include/gscan.h
SIGNATURES = [
    ("gs_engine_create", ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(_P)]),
    ("gs_engine_destroy", None, [_P]),
    ("gs_engine_stream", _P, [_P]),
    ("gs_engine_load_csr", ctypes.c_int, [_P, _I64, _I64, _P, _P, ctypes.c_int]),
    ("gs_engine_load_edges", ctypes.c_int, [_P, _I64, _I64, _P, ctypes.c_int]),
    ("gs_engine_load_csr_part", ctypes.c_int,
     [_P, _I64, _I64, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P]),
    ("gs_engine_load_finish", ctypes.c_int, [_P]),
    ("gs_engine_scan", ctypes.c_int,
     [_P, _I32, ctypes.POINTER(GsEps2), _P, _P, ctypes.c_int, ctypes.POINTER(GsStats)]),
    ("gs_engine_set_shard", ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int]),
    ("gs_engine_phase_begin", ctypes.c_int, [_P, _I32, ctypes.POINTER(GsEps2)]),
    ("gs_engine_phase_identify", ctypes.c_int, [_P, _P]),
    ("gs_engine_phase_resolve", ctypes.c_int, [_P, _P, ctypes.POINTER(_I64)]),
    ("gs_engine_phase_union", ctypes.c_int, [_P, _P, ctypes.POINTER(_I64)]),
    ("gs_engine_phase_merge", ctypes.c_int, [_P, _P, _I64]),
    ("gs_engine_phase_attach", ctypes.c_int, [_P, _P]),
    ("gs_engine_phase_finish", ctypes.c_int,
     [_P, _P, _P, _P, ctypes.c_int, ctypes.POINTER(GsStats)]),
    ("gs_scan_csr", ctypes.c_int,
     [_I64, _I64, _P, _P, _I32, ctypes.POINTER(GsEps2), _P, _P, ctypes.POINTER(GsStats)]),
    ("gs_scan_edges", ctypes.c_int,
     [_I64, _I64, _P, _I32, ctypes.POINTER(GsEps2), _P, _P, ctypes.POINTER(GsStats)]),
    ("gs_build_graph", ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _P]),
    ("gs_build_csr_device", ctypes.c_int, [_I64, _I64, _P, _P, _P, _P]),
    ("gs_engine_phase_stats", ctypes.c_int, [_P, ctypes.POINTER(GsStats)]),
    ("gs_engine_export_state", ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, _P, _P, _P]),
    ("gs_engine_check_sim", ctypes.c_int, [_P, _I64, _P, _P, ctypes.POINTER(GsEps2), _P]),
    ("gs_scan_partitioned", ctypes.c_int,
     [_I64, _I64, _P, _P, _I32, ctypes.POINTER(GsEps2), ctypes.c_uint64, _P, _P,
      ctypes.POINTER(GsStats)]),
    ("gs_plan_partitions", ctypes.c_int,
     [_I64, _P, ctypes.c_uint64, _P, _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    ("gs_scan_partitioned_plan", ctypes.c_int,
     [_I64, _I64, _P, _P, _I32, ctypes.POINTER(GsEps2), ctypes.c_uint64, _I64, _P, _P, _P,
      ctypes.POINTER(GsStats)]),
    ("gs_plan_closure", ctypes.c_int,
     [_I64, _I64, _P, _P, _P, _P, ctypes.c_uint64, _I64, _P, _P, _P, _I64,
      ctypes.POINTER(_I64), _P]),
    ("gs_rmat_generate", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _P, _P, _P]),
    ("gs_chunglu_generate", ctypes.c_int,
     [ctypes.c_int, ctypes.c_double, ctypes.c_double, _I64, ctypes.c_uint64, _P, _P, _P]),
    ("gs_normalize_edges", ctypes.c_int, [_I64, _P, _P, _P, ctypes.POINTER(_I64), _P]),
    ("gs_parse_edge_text", ctypes.c_int,
     [ctypes.c_char_p, _I64, ctypes.c_int, _P, _P, _I64, ctypes.POINTER(_I64),
      ctypes.POINTER(_I64)]),
    ("gs_normalize_sparse", ctypes.c_int,
     [_I64, _P, _P, _P, ctypes.POINTER(_I64), _P, ctypes.POINTER(_I64)]),
    ("gs_format_result", ctypes.c_int,
     [_I64, _P, _P, _P, ctypes.c_int, _P, _I64, ctypes.POINTER(_I64)]),
    ("gs_device_count", ctypes.c_int, []),
    ("gs_last_error", ctypes.c_char_p, []),
    ("gs_version", ctypes.c_int, []),
    ("gs_warmup", ctypes.c_int, [ctypes.c_int]),
]

_lib = None
_lock = threading.Lock()


_warm_thread: Optional[threading.Thread] = None


def load() -> ctypes.CDLL:
    """Load libgscan.so (once).  Raises ImportError if it was never built.

    A caller other than the warm-up thread first waits for it: two threads
    loading kernels lazily at once serialise on the driver and took 3-5 s
    together where either alone takes ~1 s."""
    global _lib
    w = _warm_thread
    if w is not None and w is not threading.current_thread() and w.is_alive():
        w.join(timeout=30)
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA engine first "
                "(python -c 'import __graft_entry__ as g; g.build()' or "
                "make -C paper_2311_12281_b200/csrc)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.gs_version() != ABI_VERSION:  # a stale build would misread gs_stats
            raise ImportError(f"{LIB_PATH} has ABI {lib.gs_version()}, this package needs "
                              f"{ABI_VERSION}: rebuild (make -C paper_2311_12281_b200/csrc)")
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a GS_* return code onto the reference's exception taxonomy."""
    if rc == GS_OK:
        return
    msg = load().gs_last_error().decode("utf-8", "replace")
    if rc == GS_EINVAL:
        raise ValueError(msg)
    if rc == GS_EBUDGET:
        raise InfeasibleBudget(msg)
    if rc == GS_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libgscan error {rc}: {msg}")


_MASK64 = (1 << 64) - 1


def eps2_struct(eps: Fraction, dmax=None) -> GsEps2:
    """epsilon (exact Fraction in (0,1]) -> exact epsilon^2 = p/q halves.

    p and q must fit in 128 bits for the device predicate.  When they do not
    (only for absurdly fine rationals) and the threshold is below what any
    edge of the graph can reach, the equivalent "everything similar" ratio is
    used; otherwise ValueError.  ``dmax`` may be a callable (it is needed
    only on that path).
    """
    f2 = eps * eps
    p, q = f2.numerator, f2.denominator
    if p >= 1 << 128 or q >= 1 << 128:
        if callable(dmax):  # computed only on this (rare) path
            dmax = dmax()
        if dmax is not None and p * (dmax + 1) ** 2 <= 4 * q:
            p, q = 1, 1 << 127  # every (c+2)^2/D >= 4/(dmax+1)^2 >= eps^2
        else:
            raise ValueError(
                "epsilon^2 needs more than 128-bit numerator/denominator; "
                "pass a shorter decimal or Fraction"
            )
    return GsEps2(p & _MASK64, p >> 64, q & _MASK64, q >> 64)


class Engine:
    """A device context (stream + memory pool + resident graph)."""

    def __init__(self, device: int = -1, hbm_cap_bytes: int = 0):
        lib = load()
        h = ctypes.c_void_p()
        check(lib.gs_engine_create(device, hbm_cap_bytes, ctypes.byref(h)))
        self._h = h
        self._lib = lib

    @property
    def handle(self):
        return self._h

    def stream(self) -> int:
        return self._lib.gs_engine_stream(self._h) or 0

    def close(self) -> None:
        if self._h:
            self._lib.gs_engine_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def thread_engine() -> Engine:
    """One reusable engine per host thread (engines are not thread-safe)."""
    eng = getattr(_tls, "engine", None)
    if eng is None:
        eng = Engine()
        _tls.engine = eng
    return eng


def warm_up_async() -> Optional[threading.Thread]:
    """Create the CUDA context (and load the scan kernels) in a daemon thread,
    overlapped with whatever the process does before its first scan
    (gs_warmup).  Without a device or library it does nothing."""
    if os.environ.get("GS_NO_WARMUP"):
        return None

    def run():
        try:
            lib = load()
            count = lib.gs_device_count()
            if count > 0:  # torchrun ranks warm their own device
                local = os.environ.get("LOCAL_RANK")
                lib.gs_warmup(int(local) % count if local and local.isdigit() else -1)
        except Exception:  # no library / no device: the first real call reports it
            pass

    global _warm_thread
    t = threading.Thread(target=run, name="gscan-warmup", daemon=True)
    _warm_thread = t
    t.start()
    return t
