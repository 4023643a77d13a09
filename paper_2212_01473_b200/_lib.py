"""ctypes binding of libmce_b200.so (include/mce_b200.h).

There is no fallback: if the shared library is missing or fails to load,
every entry point raises.  Build it with ``python -m
paper_2212_01473_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os

HIST_MAX = 4096
_PKG = os.path.dirname(os.path.abspath(__file__))
# MCE_LIB_PATH: load an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("MCE_LIB_PATH") or os.path.join(_PKG, "libmce_b200.so")


class MceError(RuntimeError):
    """A failed libmce_b200 call (CUDA error or device limit)."""


class CapacityError(ValueError):
    """|P| does not fit the bitset capacity (reference induced.py:21-22)."""


class RunConfigC(ctypes.Structure):
    _fields_ = [
        ("roots", ctypes.c_int),
        ("induced_full", ctypes.c_int),
        ("workers", ctypes.c_int),
        ("worker_list", ctypes.c_int),
        ("donation_min_p", ctypes.c_int),
        ("hash_labels", ctypes.c_int),
        ("root_begin", ctypes.c_int64),
        ("root_end", ctypes.c_int64),
        ("root_stride", ctypes.c_int64),
        ("include_isolated", ctypes.c_int),
        ("collect_cap", ctypes.c_int64),
        ("capacity_bits", ctypes.c_int64),
        ("mem_fraction", ctypes.c_double),
        ("measure_bytes", ctypes.c_int),
        ("partial_xrows_min_w", ctypes.c_int),
        ("donation_min_x", ctypes.c_int),
        ("no_pivot", ctypes.c_int),
        ("timing", ctypes.c_int),
    ]


class RunResultC(ctypes.Structure):
    _fields_ = [
        ("cliques", ctypes.c_int64),
        ("nodes", ctypes.c_int64),
        ("hash", ctypes.c_uint64),
        ("max_size", ctypes.c_int64),
        ("donations", ctypes.c_int64),
        ("workers", ctypes.c_int64),
        ("launches", ctypes.c_int64),
        ("collect_len", ctypes.c_int64),
        ("kernel_ms", ctypes.c_double),
        ("build_bytes", ctypes.c_int64),
        ("hist", ctypes.c_int64 * HIST_MAX),
        ("induced_full", ctypes.c_int64),
        ("phase1_ms", ctypes.c_double),
        ("phase2_ms", ctypes.c_double),
        ("clock_khz", ctypes.c_double),
    ]


WM_COLS = 9  # MCE_WM_COLS


EXPORTS = {
    "mce_last_error": (ctypes.c_char_p, []),
    "mce_graph_from_edges": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int, ctypes.c_void_p,
                                            ctypes.POINTER(ctypes.c_void_p)]),
    "mce_graph_from_edges32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int, ctypes.c_void_p,
                                            ctypes.POINTER(ctypes.c_void_p)]),
    "mce_graph_from_text": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_void_p,
                                           ctypes.POINTER(ctypes.c_void_p),
                                           ctypes.POINTER(ctypes.c_int64),
                                           ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int64)]),
    "mce_graph_from_csr": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.POINTER(ctypes.c_void_p)]),
    "mce_graph_info": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int64)] * 5),
    "mce_graph_copy_csr": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "mce_graph_free": (None, [ctypes.c_void_p]),
    "mce_degeneracy_order": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                            ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                            ctypes.c_void_p]),
    "mce_reorder": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                   ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "mce_preprocess": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                      ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "mce_enumerate": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(RunConfigC),
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.POINTER(RunResultC), ctypes.c_void_p]),
    "mce_launch_count": (ctypes.c_int64, []),
    "mce_gen_rmat": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]),
}

_lib = None


def lib():
    """Load libmce_b200.so (raises if absent -- there is no CPU path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise MceError(f"{LIB_PATH} is missing: build it with "
                           "`python -m paper_2212_01473_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = (lib().mce_last_error() or b"").decode(errors="replace")
    if rc == -4:
        raise CapacityError(msg)
    if rc == -2:
        raise ValueError(f"{what}: {msg}")
    raise MceError(f"{what} failed (rc={rc}): {msg}")


def require_device() -> None:
    """Fail loudly when no CUDA device is visible (no CPU fallback exists)."""
    count = ctypes.c_int(0)
    try:
        cudart = _cudart()
        rc = cudart.cudaGetDeviceCount(ctypes.byref(count))
    except OSError as exc:  # pragma: no cover
        raise MceError(f"CUDA runtime unavailable: {exc}") from exc
    if rc != 0 or count.value == 0:
        raise MceError("no CUDA device visible: the MCE engine runs only on the GPU")


_cudart_handle = None


def _cudart():
    global _cudart_handle
    if _cudart_handle is None:
        for name in ("libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so.12", "libcudart.so"):
            try:
                _cudart_handle = ctypes.CDLL(name)
                break
            except OSError:
                continue
        if _cudart_handle is None:
            raise OSError("libcudart not found")
        _cudart_handle.cudaGetDeviceCount.argtypes = [ctypes.POINTER(ctypes.c_int)]
    return _cudart_handle


def ptr(a) -> ctypes.c_void_p:
    """Raw data pointer of a contiguous numpy array or torch tensor."""
    if a is None:
        return ctypes.c_void_p(0)
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    assert a.flags.c_contiguous
    return ctypes.c_void_p(a.ctypes.data)
