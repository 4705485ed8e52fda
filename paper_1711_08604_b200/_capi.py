"""ctypes binding of include/afd_capi.h (the C ABI of libafd_b200.so).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_1711_08604_b200.build``) into
``paper_1711_08604_b200/lib/libafd_b200.so``.  There is no fallback: if the
library is missing or no CUDA device is present, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libafd_b200.so")

AFD_OK = 0
AFD_E_INVALID = -1
AFD_E_CUDA = -2
AFD_E_UNSUPPORTED = -3
AFD_E_NOMEM = -4

STEP_DTYPE = np.dtype([("s", np.int64), ("j", np.int64), ("radius", np.float64),
                       ("a_re", np.float64), ("a_im", np.float64),
                       ("c_re", np.float64), ("c_im", np.float64),
                       ("residual", np.float64), ("flags", np.int32), ("margin", np.float32)])
CAND_DTYPE = np.dtype([("mag2", np.float64), ("flat", np.int64),
                       ("re", np.float64), ("im", np.float64)])

STEP_FLAG_POW_AMBIGUOUS = 1
PLAN_FAST = 1  # AFD_PLAN_FAST
PLAN_MARGINS = 2  # AFD_PLAN_MARGINS

# (name, restype, argtypes) for every symbol include/afd_capi.h declares
_VP = C.c_void_p
_I64 = C.c_int64
_D = C.c_double
_I = C.c_int
SIGNATURES = [
    ("afd_last_error", C.c_char_p, []),
    ("afd_version", _I, []),
    ("afd_plan_create", _I, [C.POINTER(_VP), _I, _I64, _I64, _I64, _I64, _I64, _VP, _VP, _VP,
                             _VP, _I]),
    ("afd_plan_destroy", _I, [_VP]),
    ("afd_dft_forward", _I, [_VP, _VP, _VP, _I64, _VP]),
    ("afd_dft_inverse", _I, [_VP, _VP, _VP, _I64, _VP]),
    ("afd_analytic_projection", _I, [_VP, _VP, _VP, _I64, _VP]),
    ("afd_field", _I, [_VP, _VP, _VP, _I64, _I64, _VP]),
    ("afd_field_argmax", _I, [_VP, _VP, _VP, _I64, _VP]),
    ("afd_plan_set_engine", _I, [_VP, _I]),
    ("afd_field_direct", _I, [_VP, _VP, _VP, _I64, _I64, _VP]),
    ("afd_argmax", _I, [_VP, _VP, _I64, _VP, _VP]),
    ("afd_atom", _I, [_VP, _I, _VP, _D, _D, _D, _D, _D, _VP, _VP]),
    ("afd_energy", _I, [_VP, _VP, _VP, _I64, _VP]),
    ("afd_energy_diff", _I, [_VP, _VP, _VP, _VP, _I64, _VP]),
    ("afd_decompose", _I, [_VP, _VP, _I64, _I, _D, _I, _VP, _VP, _VP, _VP, _VP]),
    ("afd_decompose_host", _I, [_VP, _VP, _I64, _I, _D, _I, _VP, _VP, _VP, _VP, _VP, _VP,
                                _VP]),
    ("afd_sharded_begin", _I, [_VP, _VP, _I64, _VP]),
    ("afd_select_local", _I, [_VP, _I, _I, _VP, _I64, _VP]),
    ("afd_apply_step", _I, [_VP, _I, _I, _D, _I, _VP, _I, _I64, _VP, _VP]),
    ("afd_sharded_finish", _I, [_VP, _I64, _VP, _VP, _VP, _VP, _VP]),
    ("afd_comm_unique_id", _I, [_VP]),
    ("afd_comm_init", _I, [C.POINTER(_VP), _VP, _I, _I, _I]),
    ("afd_comm_destroy", _I, [_VP]),
    ("afd_decompose_sharded", _I, [_VP, _VP, _VP, _I64, _I, _D, _I, _VP, _VP, _VP, _VP, _VP]),
    ("afd_error_trace", _I, [_VP, _VP, _VP, _I, _VP, _I64, _VP, _VP, _VP, _VP]),
    ("afd_launch_count", _I64, [_VP]),
    ("afd_time_field", _I, [_VP, _VP, _I64, _I, _VP, _VP]),
    ("afd_fp64_peak", _I, [_I, _VP, _VP]),
    ("afd_field_split", _I, [_VP, _VP, _VP, _VP]),
    ("afd_field_tiers", _I, [_VP, _VP, _VP]),
    ("afd_field_tier_rows", _I, [_VP, _VP, _VP, _I, _VP, _VP]),
]

_LIB = None


class AfdCudaUnavailable(RuntimeError):
    """The CUDA extension is missing or unusable; there is no CPU fallback."""


def load(path=None):
    """Load libafd_b200.so and declare every exported signature.

    AFD_LIB_PATH overrides the in-tree library (used to A/B kernel variants)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = path or os.environ.get("AFD_LIB_PATH") or LIB_PATH
    if not os.path.exists(path):
        raise AfdCudaUnavailable(
            "libafd_b200.so not built (%s); run __graft_entry__.build()" % path)
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(rc):
    """Map an AFD status code to the reference's exception types."""
    if rc == AFD_OK:
        return
    msg = load().afd_last_error().decode(errors="replace")
    if rc == AFD_E_INVALID:
        raise ValueError(msg)
    if rc == AFD_E_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == AFD_E_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError("AFD CUDA error: " + msg)
