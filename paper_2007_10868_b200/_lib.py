"""ctypes binding of the C-ABI in include/polycert_b200.h.

The shared library is built in-tree by ``build.build()``
(paper_2007_10868_b200/libpolycert_b200.so). There is no fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpolycert_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "polycert_b200.h")

PC_OK, PC_ERR_INVALID_ARGUMENT, PC_ERR_MODEL, PC_ERR_LOGIC, PC_ERR_CUDA, PC_ERR_OOM = range(6)
KIND = {"input": 0, "dense": 1, "conv": 2, "relu": 3, "residual_join": 4}


class PcLayerDesc(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int), ("n_preds", ctypes.c_int), ("preds", ctypes.c_int * 2),
        ("n_out", ctypes.c_int),
        ("fw", ctypes.c_int), ("fh", ctypes.c_int), ("sw", ctypes.c_int), ("sh", ctypes.c_int),
        ("pw", ctypes.c_int), ("ph", ctypes.c_int), ("cin", ctypes.c_int), ("cout", ctypes.c_int),
        ("weights", ctypes.c_void_p), ("bias", ctypes.c_void_p),
    ]


class PcOptions(ctypes.Structure):
    _fields_ = [("early_term", ctypes.c_int), ("chunk_rows", ctypes.c_longlong),
                ("memory_budget", ctypes.c_longlong), ("device", ctypes.c_int),
                ("exec_mode", ctypes.c_int), ("numeric_mode", ctypes.c_int)]


class PcStats(ctypes.Structure):
    _fields_ = [("rows_total", ctypes.c_longlong), ("rows_terminated_early", ctypes.c_longlong),
                ("gbc_madds", ctypes.c_longlong), ("gbc_dense_equiv", ctypes.c_longlong),
                ("dense_madds", ctypes.c_longlong), ("checkpoints", ctypes.c_longlong)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


# int (*pc_allgather_fn)(void* user, const void* d_send, void* d_recv, size_t bytes, void* stream)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_size_t, ctypes.c_void_p)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i, ll, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_double
    sig = {
        "pc_default_options": (None, [vp]),
        "pc_validate": (i, [vp, i, i, i, i, vp]),
        "pc_net_create": (i, [vp, i, i, i, i, vp, vp]),
        "pc_net_destroy": (None, [vp]),
        "pc_net_num_layers": (i, [vp]),
        "pc_net_layer_numel": (ll, [vp, i]),
        "pc_net_total_neurons": (ll, [vp]),
        "pc_net_output_size": (i, [vp]),
        "pc_input_box": (i, [vp, i, d, i, vp, vp]),
        "pc_net_test": (i, [vp, vp, vp, i, vp, vp, vp, vp, vp, vp, vp]),
        "pc_net_test_ex": (i, [vp, vp, vp, vp, i, vp, vp, vp, vp, vp, vp, vp]),
        "pc_net_test_device": (i, [vp, vp, vp, i, vp, vp, vp]),
        "pc_net_test_batch": (i, [vp, i, vp, vp, i, vp, i, vp, vp, vp, vp]),
        "pc_net_stream": (vp, [vp]),
        "pc_net_candidate": (i, [vp, vp, vp, vp]),
        "pc_last_launch_count": (ll, []),
        "pc_last_timing": (None, [vp, vp, vp, vp]),
        "pc_last_dense_madds": (d, []),
        "pc_last_kernel_timing": (None, [i, vp, vp, vp]),
        "pc_last_conv_executed_madds": (ctypes.c_double, []),
        "pc_net_set_serial": (i, [vp, i]),
        "pc_fp64_peak": (i, [i, vp]),
        "pc_scalar_ops": (i, [i, vp, vp, vp, ll]),
        "pc_chain_fold": (i, [i, i, vp, vp, vp, vp]),
        "pc_scan_stats": (i, [i, vp]),
        "pc_last_profile": (i, [ctypes.c_char_p, i]),
        "pc_last_error": (ctypes.c_char_p, []),
        "pc_net_set_sharding": (i, [vp, i, i, ALLGATHER_FN, vp]),
        "pc_nccl_unique_id": (i, [vp, ctypes.c_char_p, i]),
        "pc_nccl_comm_create": (vp, [i, i, i, vp, ctypes.c_char_p, i]),
        "pc_nccl_comm_destroy": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def header_symbols() -> list[str]:
    """Function names declared in include/polycert_b200.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:pc_status|void|int|long long|double|const char)\s*\**\s*(pc_\w+)\(",
                                 txt, flags=re.M)))


lib = _load()


class PcError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class ModelError(PcError):
    """std::runtime_error from validate_model."""


class InvalidArgument(PcError, ValueError):
    """std::invalid_argument."""


class LogicError(PcError):
    """std::logic_error."""


class CudaError(PcError):
    """No device or CUDA failure (there is no CPU fallback)."""


def check(status: int):
    if status == PC_OK:
        return
    msg = (lib.pc_last_error() or b"").decode()
    cls = {PC_ERR_MODEL: ModelError, PC_ERR_INVALID_ARGUMENT: InvalidArgument,
           PC_ERR_LOGIC: LogicError, PC_ERR_CUDA: CudaError}.get(status, PcError)
    raise cls(status, msg)
