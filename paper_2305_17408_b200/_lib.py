"""ctypes binding of libadaptgear_b200.so (declared in include/adaptgear_b200.h).

This is the only place Python touches the native library.  Every entry point
returns an AG_* status; non-zero statuses are raised as the reference's
exception types (ValueError / KernelError / RuntimeError) with the library's
thread-local message.  There is no CPU fallback: if the library or a CUDA
device is missing, the product path raises.
"""
from __future__ import annotations

import ctypes
import pathlib
import threading

import torch

from .errors import KernelError

PKG = pathlib.Path(__file__).resolve().parent
LIB_PATH = PKG / "libadaptgear_b200.so"

AG_OK, AG_ERR_VALUE, AG_ERR_KERNEL, AG_ERR_CUDA = 0, 1, 2, 3
AG_OP = {"sum": 0, "mean": 1, "max": 2}
AG_EPI_COMBINE, AG_EPI_GIN, AG_EPI_EMPTY_OTHER, AG_EPI_RELU_MASK, AG_EPI_RELU = 1, 2, 4, 8, 16
AG_EPI_INTER_COO = 32
AG_GEMM_RELU = 1

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
F32 = ctypes.c_float
F64 = ctypes.c_double
U64 = ctypes.c_uint64

# name -> argtypes (restype is int unless listed in _RESTYPES)
SIGNATURES: dict[str, list] = {
    "ag_abi_version": [],
    "ag_last_error": [],
    "ag_device_sm_count": [],
    "ag_launch_count": [],
    "ag_canonicalize": [I64, I64, P, P, P, P, P, P, P, P],
    "ag_relabel": [I64, P, P, P, P, P, P],
    "ag_gcn_normalize": [I64, I64, P, P, P, P, P, P, P],
    "ag_in_degrees": [I64, I64, P, P, P],
    "ag_decompose_count": [I64, P, P, I64, P, P],
    "ag_decompose_split": [I64, P, P, P, I64, P, P, P, P, P, P, P],
    "ag_build_row_ptr": [I64, I64, P, P, P],
    "ag_row_touched": [I64, P, P, P],
    "ag_first_off_block": [I64, P, P, I64, P, P],
    "ag_blocks_count": [I64, I64, P, I64, P, P],
    "ag_blocks_fill": [I64, I64, P, P, P, I64, I64, P, P, P, P, P],
    "ag_csr_spmm": [I64, I64, P, P, P, P, P, I32, I32, P, P, F32, P],
    "ag_csr_intra_spmm": [I64, I64, I64, I64, P, P, P, P, P, I32, I32, P, P, F32, P],
    "ag_coo_spmm": [I64, I64, I64, P, P, P, P, P, I32, P],
    "ag_coo_gather_spmm": [I64, I64, P, P, P, P, P, P],
    "ag_gather_pair_spmm": [I64, I64, P, P, P, P, P, I32, F32, P, P, P],
    "ag_dense_block_spmm": [I64, I64, I64, P, P, P, P, P, I32, I32, P, P, F32, P],
    "ag_role_csr_build": [I64, P, P, P, I64, P, P, P, P],
    "ag_fused_spmm": [I64, I64, I32, P, P, P, P, P, P, I32, P, I64, P, P, I32, I32, P, P, F32,
                      P, P, I64, I32, P],
    "ag_relu_bits": [I64, I64, P, I64, P, I64, P],
    "ag_dense_block_pack": [I64, I64, I64, P, P, P, I64, P],
    "ag_block_diag_gemm_tf32x3": [I64, I64, I64, P, I64, P, I64, I64, P, I64, F32, P],
    "ag_slab_window": [I64, P, P, F64, P, P],
    "ag_slab_codes": [I64, P, P, P, P, I32, P, P, P, P, P],
    "ag_slab_far_capacity": [],
    "ag_band_max_window": [],
    "ag_band_capacity": [],
    "ag_band_sizes": [I64, P, P, P, P, P],
    "ag_band_records": [I64, P, P, P, P, I32, P, P, P, P, P],
    "ag_band_spmm": [I64, I64, P, P, P, P, P, P, I64, P, P, I32, F32, P, P, I64, I32, P],
    "ag_slab_dense_blocks": [I64, P, P, P, P, P, P],
    "ag_combine": [I64, I64, P, P, P, P, P, I32, P, P],
    "ag_gemm_f32": [I64, I64, I64, P, I64, I32, P, I64, I32, P, I64, F32, F32, I32, P, I64, P,
                    I64, P],
    "ag_gemm_tf32x3": [I64, I64, I64, P, I64, I32, P, I64, I32, P, P, I64, F32, F32, I32, P,
                       I64, P, I64, P],
    "ag_tf32_split_lo": [I64, P, P, P],
    "ag_softmax_xent": [I64, I64, I64, P, P, P, I64, P, P, I64, P],
    "ag_relu_backward": [I64, P, P, P],
    "ag_sgd_step": [I64, P, P, F32, P],
    "ag_cluster_bfs": [I64, I64, P, P, I64, P, P],
    "ag_partition_from_ids": [I64, P, I64, P, P],
    "ag_synth_candidates": [I64, I64, F64, F64, I64, I64, U64, I64, I64, P, P, P],
    "ag_synth_vertex_keys": [I64, U64, P, P],
}
_RESTYPES = {"ag_last_error": ctypes.c_char_p, "ag_launch_count": ctypes.c_uint64}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load (never build) the native library; raise loudly if it is absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (there is no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, args in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = _RESTYPES.get(name, ctypes.c_int)
            _lib = lib
    return _lib


def launch_count() -> int:
    """Kernels launched by libadaptgear_b200 so far (process-wide)."""
    return int(load().ag_launch_count())


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def call(name: str, *args) -> None:
    fn = getattr(load(), name)
    rc = fn(*args)
    if rc != AG_OK:
        msg = load().ag_last_error().decode("utf-8", "replace")
        if rc == AG_ERR_VALUE:
            raise ValueError(msg)
        if rc == AG_ERR_KERNEL:
            raise KernelError(msg)
        raise RuntimeError(f"{name}: {msg}")


def ptr(t: torch.Tensor | None):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr()) if t.numel() else None


def host_ptr(a):
    """Pointer to a contiguous numpy array."""
    return a.ctypes.data_as(ctypes.c_void_p)


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def out_i64():
    return ctypes.c_int64(0)


def out_i32():
    return ctypes.c_int32(0)


def byref(x):
    return ctypes.byref(x)


_device_checked = False


def device() -> torch.device:
    """The CUDA device the path runs on; raises if there is none."""
    global _device_checked
    if not torch.cuda.is_available():
        raise RuntimeError("adaptgear_b200 needs a CUDA device (sm_100a); none is visible and "
                           "there is no CPU fallback")
    if not _device_checked:
        load()
        _device_checked = True
    return torch.device("cuda", torch.cuda.current_device())
