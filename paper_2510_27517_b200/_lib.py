"""ctypes binding of libspaigraph_b200.so (the C-ABI declared in include/spaigraph_b200.h).

There is no CPU fallback: every compute call goes through this library on a CUDA device, and a
missing library or a missing GPU raises immediately.  Device buffers are torch tensors
(plumbing only: allocation, streams); the library receives raw pointers and the current stream.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SG_LIB_PATH: an alternative build of the same library (kernel-variant A/B runs in profiles/)
LIB_PATH = os.environ.get("SG_LIB_PATH") or os.path.join(HERE, "libspaigraph_b200.so")

SG_OK, SG_EINVAL, SG_ENOTSPD, SG_ECUDA, SG_EUNSUPPORTED, SG_EDUPLICATE = range(6)
PRECOND_IDENTITY, PRECOND_JACOBI, PRECOND_LEARNED = 0, 1, 2

vp, i64, i32, f64, szp = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.POINTER(C.c_size_t)


class SolveConfigC(C.Structure):
    _fields_ = [("rtol", C.c_double), ("max_iters", C.c_int64), ("refresh_period", C.c_int64),
                ("termination", C.c_int32), ("track_history", C.c_int32)]


class SolveResultC(C.Structure):
    _fields_ = [("k", C.c_int64), ("converged", C.c_int32), ("status", C.c_int32),
                ("fail_iter", C.c_int64), ("fail_value", C.c_double), ("fail_kind", C.c_int32),
                ("hist_len", C.c_int64)]


# name -> (restype, argtypes); mirrors include/spaigraph_b200.h one-for-one
SIGNATURES = {
    "sg_abi_version": (C.c_int, []),
    "sg_last_error": (C.c_char_p, []),
    "sg_csr_from_coo": (C.c_int, [i64, i64, i64, vp, vp, vp, vp, vp, vp, C.POINTER(C.c_int64), vp, szp, vp]),
    "sg_narrow_index": (C.c_int, [vp, vp, i64, i64, i64, i64, vp, szp, vp]),
    "sg_narrow_index_segments": (C.c_int, [vp, vp, i64, vp, vp, vp, i32, vp, szp, vp]),
    "sg_csr_validate": (C.c_int, [i64, i64, i64, vp, vp, vp, szp, vp]),
    "sg_csr_transpose": (C.c_int, [i64, i64, i64, vp, vp, vp, vp, vp, vp, szp, vp]),
    "sg_pattern_is_symmetric": (C.c_int, [i64, i64, vp, vp, C.POINTER(C.c_int32), vp, szp, vp]),
    "sg_pattern_square": (C.c_int, [i64, vp, vp, vp, vp, C.POINTER(C.c_int64), vp, szp, vp]),
    "sg_gram_pattern": (C.c_int, [i64, vp, vp, vp, vp, vp, vp, C.POINTER(C.c_int64), vp, szp, vp]),
    "sg_gram_values": (C.c_int, [i64, vp, vp, vp, vp, vp, C.c_double, vp, vp]),
    "sg_csr_pad_to_pattern": (C.c_int, [i64, vp, vp, vp, vp, vp, vp, vp, szp, vp]),
    "sg_row_expand": (C.c_int, [i64, vp, vp, vp]),
    "sg_gather_f64": (C.c_int, [vp, vp, vp, i64, vp]),
    "sg_csr_diagonal": (C.c_int, [i64, vp, vp, vp, vp, vp, vp]),
    "sg_gen_poisson2d": (C.c_int, [i64, i64, vp, i64, i64, vp, vp, vp, vp]),
    "sg_gen_poisson3d": (C.c_int, [i64, i64, i64, vp, vp, vp, vp]),
    "sg_matrix_norm": (C.c_int, [vp, i64, C.c_int, vp, vp, szp, vp]),
    "sg_matrix_norm_batched": (C.c_int, [vp, vp, i32, i64, C.c_int, vp, vp, szp, vp]),
    "sg_graph_features_batched": (C.c_int, [vp, i32, i64, vp, vp, vp, vp, C.c_int, vp, vp, vp, vp, vp,
                                            vp, vp]),
    "sg_graph_features": (C.c_int, [i64, i64, vp, vp, vp, vp, C.c_int, i64, i64, vp, f64, vp, vp, vp]),
    "sg_gnn_forward": (C.c_int, [vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, i64, i64,
                                 vp, vp, vp, vp, vp, vp, vp, szp, vp]),
    "sg_gnn_forward_ex": (C.c_int, [vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, i64, i64,
                                    vp, vp, vp, vp, vp, vp, i32, vp, szp, vp]),
    "sg_spmv": (C.c_int, [i64, vp, vp, vp, vp, vp, vp]),
    "sg_spmv_seq": (C.c_int, [i64, vp, vp, vp, vp, vp, vp]),
    "sg_spmv_warp": (C.c_int, [i64, vp, vp, vp, vp, vp, vp]),
    "sg_learned_apply": (C.c_int, [i64, vp, vp, vp, vp, vp, vp, f64, vp, vp, vp, vp]),
    "sg_axpby": (C.c_int, [vp, vp, vp, f64, i64, C.c_int, vp]),
    "sg_dot": (C.c_int, [vp, vp, i64, vp, vp, szp, vp]),
    "sg_pcg_create": (C.c_int, [C.POINTER(vp), i32, C.POINTER(C.c_int64), vp, vp, vp, C.c_int,
                                vp, vp, vp, vp, vp, vp, vp, f64, vp]),
    "sg_pcg_solve": (C.c_int, [vp, vp, vp, C.POINTER(SolveConfigC), C.POINTER(SolveResultC),
                               C.POINTER(C.c_int64), vp]),
    "sg_pcg_history": (C.c_int, [vp, i32, vp, i64]),
    "sg_pcg_destroy": (None, [vp]),
    "sg_pcg_rebind_values": (C.c_int, [vp, vp, vp, vp, vp]),
    "sg_pcg_rebind": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "sg_pcg_set_profile": (C.c_int, [vp, i32]),
    "sg_pcg_set_trace": (C.c_int, [vp, vp]),
    "sg_pcg_rebuilds": (C.c_int, [vp, C.POINTER(C.c_int64)]),
    "sg_pcg_apply_ns": (C.c_int, [vp, C.POINTER(C.c_int64)]),
    "sg_pcg_set_stencil": (C.c_int, [vp, vp, i64, i64, C.POINTER(C.c_int32)]),
    "sg_pcg_stats": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), vp, i32]),
    "sg_sai_loss": (C.c_int, [i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, f64, vp,
                              C.c_int, C.POINTER(C.c_double), vp, vp, szp, vp]),
    "sg_dense_affine": (C.c_int, [i64, i32, i32, vp, i32, vp, i32, i32, vp, vp, vp, i32, i32, vp]),
    "sg_edge_pre": (C.c_int, [i64, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "sg_relu_grad": (C.c_int, [i64, vp, vp, vp, vp]),
    "sg_segment_sum": (C.c_int, [i64, i32, vp, vp, vp, vp, i32, vp]),
    "sg_outer_sum": (C.c_int, [i64, i32, i32, vp, i32, vp, i32, vp, i32, vp, szp, vp]),
    "sg_adamw": (C.c_int, [i64, vp, vp, vp, vp, f64, f64, f64, f64, f64, i64, f64, vp]),
    "sg_fsai_build": (C.c_int, [i64, vp, vp, vp, vp, vp, vp, C.POINTER(C.c_int64), vp]),
    "sg_loss_norm_partial": (C.c_int, [vp, i64, C.c_int, vp, vp, szp, vp]),
    "sg_loss_norm_combine": (C.c_int, [vp, i32, i64, C.c_int, vp, vp]),
    "sg_sai_loss_part_fwd": (C.c_int, [i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, f64, vp, vp, i64, i64, vp, vp, vp, vp,
                                       szp, vp]),
    "sg_loss_sum_parts": (C.c_int, [vp, i32, C.POINTER(C.c_double), vp]),
    "sg_sai_loss_part_bwd": (C.c_int, [i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, vp, vp, szp,
                                       vp]),
    "sg_tc_gemm_selftest": (C.c_int, [vp, vp, i32, i32, i32, vp, vp]),
    "sg_pcg_set_partition": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "sg_pcg_peer_info_size": (C.c_int, []),
    "sg_pcg_peer_export": (C.c_int, [vp, i64, i64, i32, vp]),
    "sg_pcg_set_peers": (C.c_int, [vp, i32, i32, vp]),
    "sg_csr_row_block": (C.c_int, [vp, vp, i64, i64, i64, i64, i64, i64, vp, vp, vp, C.POINTER(C.c_int64), vp, szp,
                                   vp]),
    "sg_graph_features_block": (C.c_int, [i64, i64, i64, vp, vp, vp, vp, C.c_int, i64, i64, vp, f64, vp, vp, vp]),
    "sg_norm_acc_size": (C.c_int, []),
    "sg_norm_accum": (C.c_int, [vp, i64, C.c_int, vp, vp, szp, vp]),
    "sg_norm_from_acc": (C.c_int, [vp, i64, C.c_int, vp, vp]),
}

_lib = None


class NativeLibraryError(RuntimeError):
    pass


def load_library(require_gpu: bool = True):
    """Load the shared library (and, by default, insist on a CUDA device)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2510_27517_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_gpu:
        import torch
        if not torch.cuda.is_available():
            raise NativeLibraryError("paper_2510_27517_b200 requires a CUDA device (B200); none is visible")
    return _lib


def lib():
    return load_library(True)


def last_error() -> str:
    return load_library(False).sg_last_error().decode()


def check(status: int, what: str = ""):
    if status == SG_OK:
        return
    msg = last_error()
    if status in (SG_EINVAL, SG_EDUPLICATE):
        raise ValueError(msg)
    if status == SG_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"{what}: {msg}" if what else msg)


def stream_ptr():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def device():
    import torch
    load_library(True)  # no device => NativeLibraryError before any allocation
    return torch.device("cuda", torch.cuda.current_device())


def empty(n: int, dtype):
    """Device buffer with 16 bytes of slack past the end (vector-load staging may over-read)."""
    import torch
    pad = 16 // torch.tensor([], dtype=dtype).element_size()
    return torch.empty(int(n) + pad, dtype=dtype, device=device())[: int(n)]


def zeros(n: int, dtype):
    import torch
    pad = 16 // torch.tensor([], dtype=dtype).element_size()
    return torch.zeros(int(n) + pad, dtype=dtype, device=device())[: int(n)]


def to_device(a, dtype):
    """Host array -> padded device tensor (torch only does the copy)."""
    import numpy as np
    import torch
    a = np.ascontiguousarray(a)
    t = empty(len(a), dtype)
    if len(a):
        t.copy_(torch.from_numpy(a), non_blocking=False)
    return t


def workspace(fn, *args):
    """Query + allocate a workspace for an entry point that takes (..., ws, ws_bytes, stream)."""
    import torch
    nbytes = C.c_size_t(0)
    check(fn(*args, None, C.byref(nbytes), stream_ptr()))
    buf = torch.empty(max(int(nbytes.value), 16), dtype=torch.uint8, device=device())
    return buf, nbytes


def call_ws(fn, *args, what=""):
    buf, nbytes = workspace(fn, *args)
    check(fn(*args, ptr(buf), C.byref(nbytes), stream_ptr()), what)
    return buf
