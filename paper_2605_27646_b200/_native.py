"""ctypes binding of the C-ABI library (include/hqmq_b200.h).

The library is built in-tree (python -m paper_2605_27646_b200.build) and
loaded from paper_2605_27646_b200/_lib/libhqmq_b200.so.  There is no CPU
fallback: if the library is missing, or no CUDA device is available, every
codec entry point raises NativeLibraryMissing.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import NativeLibraryMissing

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libhqmq_b200.so")

F16, BF16, F32, F64 = 0, 1, 2, 3
SEARCH_AUTO, SEARCH_CUDA_CORE, SEARCH_TENSOR_CORE = 0, 1, 2
DEVERR_SIGMA = 0x1
DEVERR_INDEX = 0x2

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_vp = ctypes.c_void_p


class EncodeArgs(ctypes.Structure):
    _fields_ = [
        ("batch", c_i64), ("heads", c_i64), ("tokens", c_i64), ("head_dim", c_i64),
        ("codebook_size", c_i32), ("radius_bits", c_i32), ("index_bits", c_i32),
        ("input_dtype", c_i32),
        ("outlier_multiplier", ctypes.c_double),
        ("per_head_pooling", c_i32), ("_pad0", c_i32),
        ("data", c_vp), ("rot_f32", c_vp), ("joint_f64", c_vp),
        ("scales", c_vp), ("index_words", c_vp), ("radius_words", c_vp),
        ("flag_words", c_vp), ("payloads", c_vp), ("token_offsets", c_vp),
        ("payload_capacity", c_i64),
        ("counters", c_vp), ("error_word", c_vp),
        ("workspace", c_vp), ("workspace_bytes", ctypes.c_size_t),
        ("index_capacity_words", ctypes.c_size_t),
        ("radius_capacity_words", ctypes.c_size_t),
        ("flag_capacity_words", ctypes.c_size_t),
        ("search_path", c_i32), ("_pad1", c_i32),
        ("fixed_thresholds", c_vp), ("thresholds_out", c_vp),
    ]


class DecodeArgs(ctypes.Structure):
    _fields_ = [
        ("batch", c_i64), ("heads", c_i64), ("tokens", c_i64), ("head_dim", c_i64),
        ("codebook_size", c_i32), ("radius_bits", c_i32), ("index_bits", c_i32),
        ("out_dtype", c_i32),
        ("token_start", c_i64), ("token_stop", c_i64),
        ("scales", c_vp), ("index_words", c_vp), ("radius_words", c_vp),
        ("flag_words", c_vp), ("payloads", c_vp), ("token_offsets", c_vp),
        ("joint_f32", c_vp), ("joint_f64", c_vp),
        ("out", c_vp), ("error_word", c_vp),
        ("joint_f16", c_vp),
    ]


class PackedView(ctypes.Structure):
    _fields_ = [
        ("scales", c_vp), ("index_words", c_vp), ("radius_words", c_vp),
        ("flag_words", c_vp), ("payloads", c_vp), ("token_offsets", c_vp),
        ("joint_f32", c_vp),
        ("joint_f16", c_vp),
        ("joint_f64", c_vp),
    ]


class AttentionArgs(ctypes.Structure):
    _fields_ = [
        ("batch", c_i64), ("q_heads", c_i64), ("kv_heads", c_i64), ("q_tokens", c_i64),
        ("kv_tokens", c_i64), ("head_dim", c_i64),
        ("codebook_size", c_i32), ("radius_bits", c_i32), ("index_bits", c_i32),
        ("causal", c_i32),
        ("scale", ctypes.c_double),
        ("q", c_vp), ("k", PackedView), ("v", PackedView), ("out", c_vp),
        ("num_splits", c_i32), ("precise", c_i32),
        ("workspace", c_vp), ("workspace_bytes", ctypes.c_size_t),
    ]


class PagedView(ctypes.Structure):
    _fields_ = [
        ("index_pages", c_vp), ("radius_pages", c_vp), ("scale_pages", c_vp),
        ("joint_f32", c_vp), ("joint_f16", c_vp),
        ("flag_pages", c_vp), ("payoff_pages", c_vp), ("payloads", c_vp),
    ]


class PagedAttentionArgs(ctypes.Structure):
    _fields_ = [
        ("batch", c_i64), ("q_heads", c_i64), ("kv_heads", c_i64), ("head_dim", c_i64),
        ("codebook_size", c_i32), ("radius_bits", c_i32), ("index_bits", c_i32),
        ("page_tokens", c_i32),
        ("max_pages", c_i32), ("max_kv_tokens", c_i32),
        ("scale", ctypes.c_double),
        ("kv_lens", c_vp), ("block_table", c_vp), ("q", c_vp),
        ("k", PagedView), ("v", PagedView), ("out", c_vp),
        ("num_splits", c_i32), ("_pad", c_i32),
        ("workspace", c_vp), ("workspace_bytes", ctypes.c_size_t),
    ]


class PagedAppendArgs(ctypes.Structure):
    _fields_ = [
        ("n_seq", c_i32), ("kv_heads", c_i32), ("n_new", c_i32), ("max_pages", c_i32),
        ("page_tokens", c_i32), ("index_bits", c_i32), ("radius_bits", c_i32), ("_pad", c_i32),
        ("num_pages", c_i64),
        ("seq_ids", c_vp), ("seq_start", c_vp), ("block_table", c_vp),
        ("src_index", c_vp), ("src_radius", c_vp), ("src_scales", c_vp),
        ("src_flags", c_vp), ("src_payoff", c_vp),
        ("index_pages", c_vp), ("radius_pages", c_vp), ("scale_pages", c_vp),
        ("flag_pages", c_vp), ("payoff_pages", c_vp), ("error_word", c_vp),
    ]


# Every symbol include/hqmq_b200.h declares, with its ctypes signature.
SIGNATURES = {
    "hqmq_version": ([], ctypes.c_char_p),
    "hqmq_status_string": ([c_i32], ctypes.c_char_p),
    "hqmq_last_error": ([], ctypes.c_char_p),
    "hqmq_fp32_probe": ([c_vp, c_i32, c_i32, c_i32, c_vp], c_i32),
    "hqmq_nearest_scan": ([c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp], c_i32),
    "hqmq_encode_workspace_bytes": ([ctypes.POINTER(EncodeArgs)], ctypes.c_size_t),
    "hqmq_encode": ([ctypes.POINTER(EncodeArgs), c_vp], c_i32),
    "hqmq_decode": ([ctypes.POINTER(DecodeArgs), c_vp], c_i32),
    "hqmq_unpack": ([ctypes.POINTER(DecodeArgs), c_vp, c_vp, c_vp, c_vp], c_i32),
    "hqmq_expand_tokens": ([ctypes.POINTER(DecodeArgs), c_vp, c_vp, c_vp, ctypes.c_uint32, c_vp],
                           c_i32),
    "hqmq_paged_append": ([ctypes.POINTER(PagedAppendArgs), c_vp], c_i32),
    "hqmq_pack": ([c_i64, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                   ctypes.c_size_t, c_vp], c_i32),
    "hqmq_pack_workspace_bytes": ([c_i64], ctypes.c_size_t),
    "hqmq_token_offsets": ([c_i64, c_i32, c_vp, c_vp, c_vp, ctypes.c_size_t, c_vp], c_i32),
    "hqmq_token_offsets_workspace_bytes": ([c_i64], ctypes.c_size_t),
    "hqmq_validate_indices": ([c_vp, c_i64, c_i32, c_i64, c_vp, c_vp], c_i32),
    "hqmq_attention_workspace_bytes": ([ctypes.POINTER(AttentionArgs)], ctypes.c_size_t),
    "hqmq_attention_decode": ([ctypes.POINTER(AttentionArgs), c_vp], c_i32),
    "hqmq_attention_kernel_name": ([ctypes.POINTER(AttentionArgs)], ctypes.c_char_p),
    "hqmq_paged_attention_workspace_bytes": ([ctypes.POINTER(PagedAttentionArgs)], ctypes.c_size_t),
    "hqmq_attention_decode_paged": ([ctypes.POINTER(PagedAttentionArgs), c_vp], c_i32),
    "hqmq_crc32_workspace_bytes": ([ctypes.c_uint64], ctypes.c_size_t),
    "hqmq_crc32": ([c_vp, ctypes.c_uint64, c_vp, c_vp, ctypes.c_size_t, c_vp], c_i32),
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the library (no device needed) and bind every declared symbol."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryMissing(
                f"{path} is missing; build it with `python -m paper_2605_27646_b200.build`"
            )
        lib = ctypes.CDLL(path)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load()


class NativeError(RuntimeError):
    pass


def check(status: int, what: str) -> None:
    if status != 0:
        L = lib()
        msg = L.hqmq_status_string(status).decode()
        last = L.hqmq_last_error().decode()
        from .errors import InvalidArgument

        if status == 1:
            raise InvalidArgument(f"{what}: {msg}")
        raise NativeError(f"{what}: {msg} {last}".strip())


_cuda_ok = False


def require_cuda(device) -> None:
    global _cuda_ok
    if _cuda_ok:
        return
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryMissing(
            "no CUDA device: the HQMQ codec runs only on the sm_100a kernels (no CPU fallback)"
        )
    lib()
    _cuda_ok = True


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def launch(device, what: str, fn, *args) -> None:
    """Call a C-ABI entry point on `device`'s current stream with `device`
    made the thread's current CUDA device for the call (the library launches
    on the current device, so a tensor on cuda:1 must not be driven from a
    thread whose current device is cuda:0)."""
    import torch

    dev = device if isinstance(device, torch.device) else torch.device(device)
    cur = torch.cuda.current_device()
    if dev.index is None or dev.index == cur:  # the common case: no device switch
        status = fn(*args, torch.cuda.current_stream().cuda_stream)
    else:
        with torch.cuda.device(dev):
            status = fn(*args, torch.cuda.current_stream(dev).cuda_stream)
    if status:
        check(status, what)
