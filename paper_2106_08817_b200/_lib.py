"""ctypes binding of libmorphreg_sm100.so (include/morphreg_sm100.h).

The library is the only compute path: there is no CPU fallback.  If the shared
object is missing or no CUDA device is visible, every compute entry point raises
RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .errors import FieldError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmorphreg_sm100.so")

MR_F32 = 0
MR_F64 = 1
MR_MAX_RADIUS = 32
MR_OPT_DETERMINISTIC = 1

# Scheme codes (MR_SCHEME_*, include/morphreg_sm100.h) by Scheme value.
SCHEME_CODES = {"semi-lagrangian": 0, "eulerian": 1, "hybrid": 2}

GUARD_BITS = (
    (1 << 0, "non-finite image"),
    (1 << 1, "image magnitude above guard"),
    (1 << 2, "non-finite momentum"),
    (1 << 3, "momentum magnitude above guard"),
    (1 << 4, "non-finite velocity"),
    (1 << 5, "velocity magnitude above guard"),
)

# Every symbol include/morphreg_sm100.h declares.
EXPORTS = (
    "mr_velocity",
    "mr_sl_step",
    "mr_sl_step_adjoint",
    "mr_velocity_adjoint",
    "mr_shoot_forward",
    "mr_shoot_forward_scheme",
    "mr_forward_workspace_bytes",
    "mr_adjoint_workspace_bytes",
    "mr_shoot_adjoint",
    "mr_shoot_adjoint_scheme",
    "mr_shoot_adjoint_ex",
    "mr_cost_workspace_bytes",
    "mr_cost_terms",
    "mr_smooth",
    "mr_scheme_step",
    "mr_axis_diff",
    "mr_gradient",
    "mr_divergence",
    "mr_conv1d",
    "mr_interpolate",
    "mr_interpolate_adjoint",
    "mr_interpolate_coord_grad",
    "mr_reduce",
    "mr_last_error",
    "mr_strerror",
    "mr_version",
)


class MrGrid(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("batch", ctypes.c_int32), ("n", ctypes.c_int32 * 3)]


class MrKernel(ctypes.Structure):
    _fields_ = [("radius", ctypes.c_int32), ("weights", ctypes.POINTER(ctypes.c_double))]


_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_d = ctypes.c_double

_SIGNATURES = {
    "mr_velocity": (_i32, [_i32, MrGrid, MrKernel, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mr_sl_step": (_i32, [_i32, MrGrid, _d, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mr_sl_step_adjoint": (_i32, [_i32, MrGrid, _d, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mr_velocity_adjoint": (_i32, [_i32, MrGrid, MrKernel, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mr_shoot_forward": (_i32, [_i32, MrGrid, MrKernel, _d, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mr_shoot_forward_scheme": (
        _i32, [_i32, MrGrid, MrKernel, _i32, _d, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mr_forward_workspace_bytes": (ctypes.c_size_t, [_i32, MrGrid]),
    "mr_adjoint_workspace_bytes": (ctypes.c_size_t, [_i32, MrGrid]),
    "mr_shoot_adjoint": (
        _i32,
        [_i32, MrGrid, MrKernel, _d, _i32, _d, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    ),
    "mr_shoot_adjoint_scheme": (
        _i32,
        [_i32, MrGrid, MrKernel, _i32, _d, _i32, _d, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
         _vp],
    ),
    "mr_shoot_adjoint_ex": (
        _i32,
        [_i32, MrGrid, MrKernel, _i32, _d, _i32, _d, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
         _i32, _vp],
    ),
    "mr_cost_workspace_bytes": (ctypes.c_size_t, [_i32, MrGrid]),
    "mr_cost_terms": (_i32, [_i32, MrGrid, _d, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mr_smooth": (_i32, [_i32, MrGrid, MrKernel, _vp, _vp, _i32, _vp]),
    "mr_scheme_step": (_i32, [_i32, MrGrid, _i32, _d, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mr_axis_diff": (_i32, [_i32, MrGrid, _i32, _vp, _vp, _i32, _vp]),
    "mr_gradient": (_i32, [_i32, MrGrid, _vp, _vp, _i32, _vp]),
    "mr_divergence": (_i32, [_i32, MrGrid, _vp, _vp, _vp]),
    "mr_conv1d": (_i32, [_i32, MrGrid, MrKernel, _i32, _vp, _vp, _i32, _vp]),
    "mr_interpolate": (_i32, [_i32, MrGrid, _vp, _vp, _vp, _i32, _vp, _vp]),
    "mr_interpolate_adjoint": (_i32, [_i32, MrGrid, _vp, _vp, _vp, _vp, _vp]),
    "mr_interpolate_coord_grad": (_i32, [_i32, MrGrid, _vp, _vp, _vp, _vp, _vp]),
    "mr_reduce": (_i32, [_i32, MrGrid, _i32, _vp, _vp, _vp, _vp]),
    "mr_last_error": (ctypes.c_char_p, []),
    "mr_strerror": (ctypes.c_char_p, [_i32]),
    "mr_version": (_i32, []),
}

_lock = threading.Lock()
_lib = None


def load_library(require_cuda: bool = True):
    """Load (once) and return the ctypes handle; raise loudly if unavailable."""
    global _lib
    if require_cuda and not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2106_08817_b200 needs a CUDA device (sm_100a); there is no CPU fallback"
        )
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "or `make -C paper_2106_08817_b200/csrc`"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = _lib.mr_last_error().decode(errors="replace")
    if rc > 0:
        raise FieldError(msg)
    raise RuntimeError(f"libmorphreg_sm100: {msg}")


def dtype_code(dtype: torch.dtype) -> int:
    if dtype == torch.float32:
        return MR_F32
    if dtype == torch.float64:
        return MR_F64
    raise FieldError(f"unsupported dtype {dtype}; use float32 or float64")


def make_grid(batch: int, shape) -> MrGrid:
    g = MrGrid()
    g.ndim = len(shape)
    g.batch = int(batch)
    n = list(shape) + [1] * (3 - len(shape))
    for i in range(3):
        g.n[i] = int(n[i])
    return g


class KernelHandle:
    """Keeps the float64 tap array alive for the duration of the ctypes call."""

    def __init__(self, weights):
        import numpy as np

        self._w = np.ascontiguousarray(weights, dtype=np.float64)
        r = (len(self._w) - 1) // 2
        if r > MR_MAX_RADIUS:
            raise FieldError(
                f"kernel radius {r} exceeds the device limit {MR_MAX_RADIUS}"
            )
        self.struct = MrKernel()
        self.struct.radius = r
        self.struct.weights = self._w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def ptr(t) -> ctypes.c_void_p | None:
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
