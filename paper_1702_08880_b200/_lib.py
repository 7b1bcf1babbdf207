"""ctypes binding of liblandau_b200.so (include/landau_b200.h).

Error mapping follows the reference: argument errors raise ValueError (as
`fused_sweep` does for a species mismatch, kernel.py:517-518), CUDA failures
and a missing device raise RuntimeError.  There is no CPU fallback: if the
library or the GPU is missing, every compute call fails loudly.
"""

from __future__ import annotations

import atexit
import ctypes as C
import os
import sys
import threading
import weakref
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "liblandau_b200.so"

LB_OK, LB_EINVAL, LB_ECUDA, LB_ENODEV, LB_ENOMEM, LB_ESINGULAR = 0, 1, 2, 3, 4, 5
MAX_SPECIES = 8

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p
_i = C.c_int
_d = C.c_double

# symbol -> (restype, argtypes); mirrors include/landau_b200.h one to one
SIGNATURES = {
    "lb_version": (_i, []),
    "lb_last_error": (C.c_char_p, []),
    "lb_device_count": (_i, []),
    "lb_ctx_create": (_i, [_i, C.POINTER(_vp)]),
    "lb_ctx_destroy": (_i, [_vp]),
    "lb_record_stride": (_i, [_i, _dp, _dp]),
    "lb_accumulator_sets": (_i, [_i, _dp, _dp]),
    "lb_chunk_len": (_i, [_i]),
    "lb_fused_sweep": (_i, [_vp, _i, _dp, _dp, _i, _i, _dp, _dp, _dp, _dp, _dp, _dp,
                            _dp, _dp, _d, _dp, _dp]),
    "lb_assemble_elements": (_i, [_vp, _i, _dp, _i, _dp, _dp, _dp, _dp, _dp, _dp,
                                  _dp, _dp, _d, _dp, _dp, _dp, _dp, _dp, _dp]),
    "lb_fused_sweep_all": (_i, [_vp, _i, _i, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _d,
                                _dp, _dp]),
    "lb_tensor_pairs": (_i, [_vp, _i, _dp, _dp, _dp, _dp, _dp, _dp]),
    "lb_mesh_create": (_i, [_vp, _i, _dp, _dp, _dp, _i, _ip, _i, _ip, _dp, C.POINTER(_vp)]),
    "lb_mesh_destroy": (_i, [_vp]),
    "lb_elements_csr": (_i, [_vp, _vp, _i, _dp, _dp, _dp, _dp]),
    "lb_operator_partial_dev": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "lb_mesh_set_geometry": (_i, [_vp, _dp, _dp, _dp, _ip, _i, _i, _ip, _ip, _dp]),
    "lb_sample_state": (_i, [_vp, _vp, _i, _dp, _dp]),
    "lb_sample_state_dev": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "lb_assemble_state": (_i, [_vp, _vp, _i, _dp, _dp, _dp, _d, _dp, _dp, _dp]),
    "lb_assemble_csr": (_i, [_vp, _vp, _i, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _d, _dp,
                             _dp, _dp, _dp]),
    "lb_sym_supported": (_i, [_i, _dp, _dp]),
    "lb_sym_npad": (_i, [_i]),
    "lb_sym_prepare_dev": (_i, [_vp, _i, _i, _dp, _dp, _vp, _vp]),
    "lb_sym_partial_dev": (_i, [_vp, _i, _d, _i, _i, _vp, _vp]),
    "lb_sym_combine_dev": (_i, [_vp, _i, _vp, _dp, _dp, _i, _i, _vp, _vp, _vp]),
    "lb_pack_records_dev": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _dp, _dp, _vp, _vp]),
    "lb_sweep_dev": (_i, [_vp, _i, _vp, _vp, _i, _i, _vp, _dp, _dp, _d, _vp, _vp, _vp]),
    "lb_elements_dev": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "lb_last_launch_count": (_i, [_vp]),
    "lb_fp64_peak": (_i, [_vp, _dp, _dp]),
    "lb_elliptic_ke": (_i, [_vp, _i, _dp, _dp, _dp]),
    "lb_sym_combine_groups_dev": (_i, [_vp, _i, C.POINTER(_vp), _dp, _dp, _i, _i, _vp, _vp, _vp]),
    "lb_sym_groups": (_i, [_i, _i, _ip, _ip]),
    "lb_sym_counters": (_i, [_vp, _i, C.POINTER(C.c_ulonglong)]),
    "lb_ipc_alloc": (_i, [_vp, C.c_size_t, C.POINTER(_vp), C.c_char_p]),
    "lb_ipc_open": (_i, [_vp, C.c_char_p, C.POINTER(_vp)]),
    "lb_ipc_close": (_i, [_vp, _vp]),
    "lb_ipc_free": (_i, [_vp, _vp]),
    "lb_cn_create": (_i, [_vp, _vp, _i, _i, _ip, _ip, _ip, _i, C.POINTER(_vp)]),
    "lb_cn_destroy": (_i, [_vp]),
    "lb_cn_set_mass": (_i, [_vp, _dp]),
    "lb_cn_get_mass": (_i, [_vp, _dp]),
    "lb_cn_newton": (_i, [_vp, _dp, _dp, _d, _d, _dp, _dp, _dp, _i, _dp, _dp, _dp, _dp]),
    "lb_cn_linear_step": (_i, [_vp, _d, _dp, _dp, _dp]),
    "lb_cn_theta_step": (_i, [_vp, _d, _d, _dp, _dp, _dp]),
    "lb_cn_stats": (_i, [_vp, _dp, _ip, _ip]),
}

_lib = None
_lib_lock = threading.Lock()


def load(path: Path | None = None):
    """Load (once) and type the shared library; raise if it is missing."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        # LB_LIB overrides the in-tree library (used to A/B kernel variants)
        p = Path(path) if path else Path(os.environ.get("LB_LIB", LIB_PATH))
        if not p.exists():
            raise RuntimeError(
                f"{p} not built: run `python -m paper_1702_08880_b200.build` "
                "(there is no CPU fallback for the B200 path)")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class SingularSystem(RuntimeError):
    """Zero pivot or non-finite update in a device linear solve (the
    solver layer re-raises it as solver.StepFailure, solver.py:124-132)."""


def check(rc: int) -> None:
    if rc == LB_OK:
        return
    msg = load().lb_last_error().decode(errors="replace")
    if rc == LB_EINVAL:
        raise ValueError(msg)
    if rc == LB_ESINGULAR:
        raise SingularSystem(msg)
    raise RuntimeError(f"liblandau_b200 error {rc}: {msg}")


def iptr(a: np.ndarray):
    """ctypes int* to a C-contiguous int32 array (caller keeps it alive)."""
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


def dptr(a: np.ndarray):
    """ctypes double* to a C-contiguous float64 array (caller keeps it alive)."""
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class Context:
    """One lb_ctx (stream + device scratch) bound to a device."""

    def __init__(self, device: int = 0):
        lib = load()
        h = _vp()
        check(lib.lb_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = int(device)
        self._lib = lib
        register_native(self, 2)

    def close(self):
        if getattr(self, "handle", None):
            self._lib.lb_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self, _finalizing=sys.is_finalizing):  # pragma: no cover - teardown order varies
        if _finalizing():  # bound at definition: module globals may be gone at shutdown
            return
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()

# Native objects are released in dependency order (CN solvers, then meshes,
# then contexts) by an atexit hook, before interpreter finalization: a
# __del__ during finalization can run after the context an object uses was
# destroyed (garbage-collection order at shutdown is arbitrary), so __del__
# does nothing once the interpreter is finalizing.
_NATIVE: "list[weakref.WeakSet]" = []


def register_native(obj, level: int) -> None:
    """Track `obj` (with a close() method) for release at exit; lower levels
    are released first (0 solvers, 1 meshes, 2 contexts)."""
    while len(_NATIVE) <= level:
        _NATIVE.append(weakref.WeakSet())
    _NATIVE[level].add(obj)


@atexit.register
def _release_native() -> None:
    for objs in _NATIVE:
        for o in list(objs):
            try:
                o.close()
            except Exception:
                pass


def finalizing() -> bool:
    return sys.is_finalizing()


def context(device: int | None = None) -> Context:
    """Per-(thread, device) cached context (the reference is single-threaded
    per call; contexts are not shared across host threads)."""
    if device is None:
        device = current_device()
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    if device not in cache:
        cache[device] = Context(device)
    return cache[device]


def current_device() -> int:
    """Device for the calling thread: torch's current device if torch is
    already imported and initialised, else 0."""
    import sys
    torch = sys.modules.get("torch")
    if torch is not None:
        try:
            if torch.cuda.is_available() and torch.cuda.is_initialized():
                return int(torch.cuda.current_device())
        except Exception:
            pass
    return 0


def device_count() -> int:
    return int(load().lb_device_count())
