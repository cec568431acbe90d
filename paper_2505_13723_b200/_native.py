"""ctypes binding of libsapgp_b200.so (the C ABI in include/sapgp_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2505_13723_b200/csrc``). There is no fallback: if the
library is missing, or no CUDA device is visible when a device entry point
is called, this module raises ``WorkerError`` -- the package never computes
the hot path on the CPU.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .errors import ContractError, NumericalError, WorkerError

# SAP_LIB_PATH selects an alternative build of the same library (kernel tuning sweeps)
LIB_PATH = os.environ.get("SAP_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libsapgp_b200.so")

SAP_OK, SAP_ERR_CONTRACT, SAP_ERR_NUMERICAL, SAP_ERR_DEVICE = 0, 1, 2, 3
SAP_TC_KA_F16 = 48  # include/sapgp_b200.h: 32 fp16 features per point
SAP_TC_KA_F16X64 = 96  # 64 fp16 features per point
FAMILY_CODES = {"rbf": 0, "matern32": 1, "matern52": 2}
ABI_VERSION = 1

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/sapgp_b200.h exactly
SIGNATURES = {
    "sap_abi_version": (_I, []),
    "sap_last_error": (ctypes.c_char_p, []),
    "sap_launch_count": (ctypes.c_longlong, []),
    "sap_ffma_peak": (_I, [_P, _I, _P]),
    "sap_prepare_points": (_I, [_P, _I64, _I, _P, _P, _I, _P, _P]),
    "sap_gather_points": (_I, [_P, _P, _I, _P, _I64, _I64, _P, _P, _P]),
    "sap_krows_workspace": (_SZ, [_I64, _I, _I64]),
    "sap_krows_times": (_I, [_P, _P, _I, _I64, _P, _I64, _P, _P, _P, _I64, _I, _P, _P, _I64, _I,
                             _D, _D, _I, _D, _P, _I64, _I, _P, _SZ, _P]),
    "sap_ktile": (_I, [_P, _P, _P, _I64, _P, _P, _P, _I64, _I, _I, _I, _D, _P, _I64, _P]),
    "sap_ktile64": (_I, [_P, _P, _I, _P, _I64, _P, _I64, _I, _D, _P, _I64, _P]),
    "sap_ktile_f32": (_I, [_P, _P, _P, _I64, _P, _P, _P, _I64, _I, _I, _I, _D, _P, _I64, _P]),
    "sap_ktile_f32_batch": (_I, [_P, _I64, _P, _I64, _I, _I, _I, _I, _I, _D, _P, _I64, _I64, _P]),
    "sap_ktile_f32_batch_split": (_I, [_P, _I64, _P, _I64, _I, _I, _I, _I, _I, _D, _P, _I64, _I64,
                                       _P, _P, _I64, _I64, _P]),
    "sap_power_stepsize": (_I, [_P, _I64, _I64, _P, _I64, _I, _P, _P, _P, _I, _I, _D, _I, _P,
                                _P, _P]),
    "sap_grad_gather": (_I, [_P, _I64, _P, _P, _P, _I64, _D, _D, _P, _I64, _I, _D, _P, _I64, _P]),
    "sap_pq_update": (_I, [_P, _P, _I64, _P, _I64, _I, _P, _I64, _P, _D, _D, _D, _D, _P, _I64,
                           _P, _P, _P]),
    "sap_combine": (_I, [_P, _I64, _P, _P, _I64, _I64, _I, _D, _D, _P]),
    "sap_tc_points": (_I, [_P, _I64, _I, _P, _I, _I, _P, _P, _P]),
    "sap_tc_gather_rows": (_I, [_P, _I, _P, _I64, _I64, _P, _P]),
    "sap_tc_gather_cols": (_I, [_P, _I, _I, _I, _P, _I64, _I64, _P, _P]),
    "sap_z_operand": (_I, [_P, _P, _I64, _I64, _I, _D, _D, _P, _P, _I, _I64, _P, _P, _P, _P]),
    "sap_colabsmax": (_I, [_P, _I64, _I64, _I, _P, _P]),
    "sap_krows_tc_workspace": (_SZ, [_I64, _I, _I64]),
    "sap_tc_supported": (_I, [_I, _I]),
    "sap_cos_features": (_I, [_P, _I64, _I, _P, _P, _I64, _P, _P, _P]),
    "sap_sdd_update": (_I, [_P, _P, _P, _I64, _I64, _I, _P, _I64, _P, _I64, _D, _D, _D, _P, _P,
                            _P]),
    "sap_normal_workspace": (_SZ, [_I64, _I]),
    "sap_normal_fill": (_I, [_P, _I, _I64, _P, _I64, _P, _SZ, _P]),
    "sap_normal_status": (_P, [_P]),
    "sap_normal_words": (_P, [_P]),
    "sap_host_draws": (_I, [ctypes.c_uint64, _I64, _I, _I64, _I64, _P, _P, _P, _P, _I]),
    "sap_krows_tc": (_I, [_P, _I64, _I, _P, _I64, _P, _I64, _I64, _P, _P, _I, _I64, _P, _I, _I, _D,
                          _P, _I64, _I, _P, _SZ, _P]),
    "sap_krows_tc_next": (_I, [_P, _I64, _I, _P, _I64, _P, _I64, _I64, _P, _P, _I, _I64, _P, _I,
                               _I, _D, _P, _I64, _I, _P, _SZ, _I, _P, _P, _P, _I64, _D, _D, _P,
                               _P, _P, _P, _P, _P]),
    "sap_block_step_workspace": (_SZ, [_I64, _I, _I]),
    "sap_block_step_supported": (_I, [_I64, _I, _I]),
    "sap_block_step": (_I, [_P, _I, _P, _SZ, _P]),
    "sap_woodbury_apply": (_I, [_P, _P, _I64, _I64, _I, _P, _I64, _I, _P, _P, _I64, _P, _SZ, _P]),
    "sap_sym_eig_workspace": (_SZ, [_I, _I]),
    "sap_sym_eig_batch": (_I, [_P, _I64, _I, _I, _I, _P, _P, _I64, _I, _I, _P, _P, _SZ, _P]),
}


class StepArgs(ctypes.Structure):
    """``sap_step_args`` (include/sapgp_b200.h): arguments of sap_block_step."""
    _fields_ = [
        ("part", _P), ("splits", _I), ("variance", ctypes.c_float), ("zscale", _P),
        ("G", _P), ("ldg", _I64),
        ("P", _P), ("Q", _P), ("Y", _P), ("ldp", _I64), ("zp", _D), ("zq", _D), ("lam", _D),
        ("loc", _P), ("b", _I64), ("m", _I), ("g", _P), ("ldgo", _I64),
        ("U", _P), ("UMc", _P), ("ldu", _I64), ("r", _I),
        ("Pw", _P), ("Qw", _P), ("eta_dev", _P), ("e0", _D), ("e1", _D), ("WB", _P),
        ("ldwb", _I64), ("Pb", _P), ("Qb", _P),
        ("D", _P), ("ldd", _I64), ("dscale_dev", _P),
        ("Zhi_next", _P), ("Zlo_next", _P), ("ldz", _I64), ("zscale_next", _P), ("zp1", _D),
        ("zq1", _D), ("zflag", _P), ("flag_idx", _I), ("n_local", _I64),
    ]


STEP_GRAD, STEP_APPLY = 1, 2

_lib = None


def load():
    """Load (once) and return the shared library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise WorkerError(
            f"CUDA library {LIB_PATH} is not built; run __graft_entry__.build() "
            "(there is no CPU fallback)")
    # SAP_PYDLL=1: the launch wrappers are called with the GIL held (they return
    # in microseconds; releasing the GIL around each lets a producer thread in
    # for up to a switch interval); sap_host_draws always releases it
    pydll = os.environ.get("SAP_PYDLL", "0") == "1"
    lib = (ctypes.PyDLL if pydll else ctypes.CDLL)(LIB_PATH)
    free = ctypes.CDLL(LIB_PATH) if pydll else lib
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(free if name == "sap_host_draws" else lib, name)
        fn.restype = res
        fn.argtypes = args
        if pydll and name == "sap_host_draws":
            setattr(lib, name, fn)
    if lib.sap_abi_version() != ABI_VERSION:
        raise WorkerError("libsapgp_b200.so ABI version mismatch; rebuild")
    _lib = lib
    return lib


def require_cuda():
    if not torch.cuda.is_available():
        raise WorkerError("no CUDA device visible: the B200 path has no CPU fallback")


def check(rc):
    if rc == SAP_OK:
        return
    msg = load().sap_last_error().decode("utf-8", "replace")
    if rc == SAP_ERR_CONTRACT:
        raise ContractError(msg)
    if rc == SAP_ERR_NUMERICAL:
        raise NumericalError(msg)
    raise WorkerError(msg)


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def call(name, *args):
    check(getattr(load(), name)(*args))
