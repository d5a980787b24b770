"""ctypes binding of libfastbdt_b200.so (include/fastbdt_b200.h).

There is no CPU fallback: if the shared library is missing or a CUDA device
is absent, fitting and prediction raise.  ``lib()`` loads the in-tree build
(``paper_1609_06119_b200/libfastbdt_b200.so``, produced by
``__graft_entry__.build()`` / ``make -C paper_1609_06119_b200/csrc``).
ctypes releases the GIL for the duration of each call.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BB_LIB_VARIANT=check loads the device-bounds-check build (make -C csrc check);
# any other value loads libfastbdt_b200_<value>.so (tuning builds)
_VARIANT = os.environ.get("BB_LIB_VARIANT")
LIB_PATH = os.path.join(_HERE, f"libfastbdt_b200_{_VARIANT}.so" if _VARIANT else "libfastbdt_b200.so")

BB_OK, BB_EINVAL, BB_ECUDA, BB_ESTATE = 0, 1, 2, 3
BB_F32, BB_F64 = 0, 1


class FitConfigC(C.Structure):
    _fields_ = [
        ("n_trees", C.c_int32),
        ("depth", C.c_int32),
        ("binning_levels", C.c_int32),
        ("flags", C.c_int32),
        ("shrinkage", C.c_double),
        ("subsample", C.c_double),
        ("pcg_state_hi", C.c_uint64),
        ("pcg_state_lo", C.c_uint64),
        ("pcg_inc_hi", C.c_uint64),
        ("pcg_inc_lo", C.c_uint64),
        ("pcg_has_uint32", C.c_int32),
        ("pcg_uinteger", C.c_uint32),
        ("f0_override", C.c_double),
    ]

    def __init__(self, **kw):
        kw.setdefault("f0_override", float("nan"))
        super().__init__(**kw)


class ForcedCutC(C.Structure):
    _fields_ = [("tree", C.c_int32), ("node", C.c_int32), ("valid", C.c_int32), ("feature", C.c_int32),
                ("cut_bin", C.c_int32)]


class FitOutC(C.Structure):
    _fields_ = [
        ("boundaries", C.c_void_p),
        ("feature", C.c_void_p),
        ("cut_bin", C.c_void_p),
        ("valid", C.c_void_p),
        ("threshold", C.c_void_p),
        ("gain", C.c_void_p),
        ("node_weight", C.c_void_p),
        ("node_purity", C.c_void_p),
        ("f0", C.c_void_p),
        ("fixed_shift", C.c_void_p),
        ("n_sig", C.c_void_p),
        ("leaves", C.c_void_p),
        ("scores", C.c_void_p),
        ("timing_ms", C.c_void_p),
    ]


class ForestC(C.Structure):
    _fields_ = [
        ("n_trees", C.c_int32),
        ("depth", C.c_int32),
        ("n_features", C.c_int32),
        ("reserved0", C.c_int32),
        ("f0", C.c_double),
        ("feature", C.c_void_p),
        ("valid", C.c_void_p),
        ("threshold", C.c_void_p),
        ("node_weight", C.c_void_p),
    ]


# every symbol include/fastbdt_b200.h declares, with its ctypes signature
_SIGS = {
    "bb_last_error": (C.c_char_p, []),
    "bb_abi_version": (C.c_int, []),
    "bb_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "bb_ctx_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "bb_ctx_destroy": (C.c_int, [C.c_void_p]),
    "bb_ctx_init_comm": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "bb_fit": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_void_p, C.c_int32,
                         C.c_void_p, C.c_int32, C.POINTER(FitConfigC), C.c_void_p, C.c_int32, C.POINTER(FitOutC)]),
    "bb_predict": (C.c_int, [C.c_void_p, C.POINTER(ForestC), C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                             C.c_void_p, C.c_void_p, C.c_int32]),
    "bb_bin": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "bb_layer_hist": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int32,
                                C.c_int32, C.c_int32, C.c_void_p]),
    "bb_split": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "bb_subsample_masks": (C.c_int, [C.c_int64, C.c_int64, C.c_double, C.c_int32, C.POINTER(FitConfigC), C.c_void_p]),
    "bb_subsample_masks_gpu": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_int32,
                                         C.POINTER(FitConfigC), C.c_void_p]),
    "bb_pairwise_sum": (C.c_double, [C.c_void_p, C.c_int64]),
    "bb_csv_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "bb_csv_n_header": (C.c_int32, [C.c_void_p]),
    "bb_csv_n_records": (C.c_int64, [C.c_void_p]),
    "bb_csv_header": (C.c_void_p, [C.c_void_p, C.c_int32, C.POINTER(C.c_int64)]),
    "bb_csv_parse": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    "bb_csv_error": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                               C.POINTER(C.c_int32), C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                               C.POINTER(C.c_double)]),
    "bb_csv_close": (C.c_int, [C.c_void_p]),
    "bb_vgroup_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "bb_vgroup_destroy": (C.c_int, [C.c_void_p]),
    "bb_ctx_init_virtual": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "bb_roc_auc": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "bb_elim_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                 C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "bb_elim_fit": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(FitConfigC), C.c_void_p,
                              C.c_void_p]),
    "bb_elim_destroy": (C.c_int, [C.c_void_p]),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load the in-tree shared library (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build the CUDA library first "
                    "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_1609_06119_b200/csrc)"
                )
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


class NativeError(RuntimeError):
    pass


def check(rc: int) -> None:
    if rc == BB_OK:
        return
    msg = lib().bb_last_error().decode("utf-8", "replace")
    if rc == BB_EINVAL:
        raise ValueError(msg)
    raise NativeError(msg)


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


_ctx = {}
_ctx_lock = threading.Lock()


def context(device: int = 0):
    """Process-wide context per device (one CUDA stream; calls serialise)."""
    with _ctx_lock:
        h = _ctx.get(device)
        if h is None:
            out = C.c_void_p()
            check(lib().bb_ctx_create(device, C.byref(out)))
            h = out
            _ctx[device] = h
        return h


_pool = {}


def worker_contexts(device: int, k: int) -> list:
    """k contexts on `device` (the first is the process-wide one): each owns a
    CUDA stream, so calls from different threads run concurrently."""
    with _ctx_lock:
        pool = _pool.setdefault(device, [])
    first = context(device)
    with _ctx_lock:
        while len(pool) < k - 1:
            out = C.c_void_p()
            check(lib().bb_ctx_create(device, C.byref(out)))
            pool.append(out)
        return [first] + pool[: k - 1]


def pcg_config(seed) -> dict:
    """numpy PCG64(seed) state split into 64-bit words (boosting.py:162)."""
    st = np.random.PCG64(seed).state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return dict(pcg_state_hi=s >> 64, pcg_state_lo=s & m, pcg_inc_hi=inc >> 64, pcg_inc_lo=inc & m,
                pcg_has_uint32=int(st["has_uint32"]), pcg_uinteger=int(st["uinteger"]))
