"""ctypes bindings to the in-tree native libraries (include/mfhost.h,
include/mfgpu.h, include/mfgpu_test.h).

There is no Python fallback: if a library is missing or fails to load, the
import of the corresponding accessor raises, loudly. `build()` in
`__graft_entry__` (or `python -m paper_2408_11853_b200._build`) produces them.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
_lock = threading.Lock()
_host = None
_gpu = None

i32, i64, f32p = C.c_int32, C.c_int64, C.POINTER(C.c_float)
i32p, i64p = C.POINTER(C.c_int32), C.POINTER(C.c_int64)


class NativeLibraryError(RuntimeError):
    pass


def _load(name):
    path = os.path.join(_LIB_DIR, name)
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} is missing; build it with `python -m paper_2408_11853_b200._build` "
            "(there is no CPU fallback for the scoring path)")
    try:
        return C.CDLL(path, mode=C.RTLD_GLOBAL)
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {path}: {exc}") from None


def host():
    """libmfhost.so: tokenizer / planner / packer."""
    global _host
    with _lock:
        if _host is None:
            lib = _load("libmfhost.so")
            lib.mfh_vocab_create.argtypes = [C.c_char_p, i64, i32, C.POINTER(C.c_void_p)]
            lib.mfh_vocab_create.restype = C.c_int
            lib.mfh_vocab_destroy.argtypes = [C.c_void_p]
            lib.mfh_vocab_destroy.restype = None
            lib.mfh_vocab_size.argtypes = [C.c_void_p]
            lib.mfh_vocab_size.restype = i32
            lib.mfh_vocab_max_piece.argtypes = [C.c_void_p]
            lib.mfh_vocab_max_piece.restype = i32
            lib.mfh_encode.argtypes = [C.c_void_p, C.c_char_p, i64, i32p, i64]
            lib.mfh_encode.restype = i64
            lib.mfh_encode_records.argtypes = [C.c_void_p, i32, i32, C.c_char_p, i64p, i32, i32,
                                               i32p, i64, i64p]
            lib.mfh_encode_records.restype = i64
            lib.mfh_encode_tsv.argtypes = [C.c_void_p, i32, C.c_char_p, i64p, i64, i32, i32, i32p,
                                           i64, i64p, i64p, i32p]
            lib.mfh_encode_tsv.restype = i64
            lib.mfh_plan.argtypes = [i64p, i64, i32, i32, i32, i64p]
            lib.mfh_plan.restype = C.c_int
            lib.mfh_pack_roles.argtypes = [i32p, i64p, i32, i64p, i64, i32p, i64p]
            lib.mfh_pack_roles.restype = C.c_int
            _host = lib
    return _host


class MfgConfig(C.Structure):
    _fields_ = [("container_path", C.c_char_p), ("device", i32), ("precision", i32),
                ("max_tokens", i64), ("max_records", i32), ("profile", i32)]


class MfgModelInfo(C.Structure):
    _fields_ = [(n, i32) for n in ("kind", "vocab_size", "d_model", "n_heads", "n_layers", "d_ffn",
                                   "max_position", "pre_norm", "n_roles", "n_head_stages",
                                   "precision", "num_sms")] + [("device_bytes", i64),
                                                               ("load_ms", C.c_double * 6)]
LOAD_PHASES = ("context", "open", "embeddings", "layers", "head", "workspaces")


NCLASS = 8
CLASS_NAMES = ("qkv", "o_proj", "ffn1", "ffn2", "attention", "layernorm", "embed", "head")


class MfgStats(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("calls", i64), ("records", i64), ("tokens", i64),
                ("chunks", i64), ("kernel_launches", i64),
                ("class_ms", C.c_double * NCLASS), ("class_launches", i64 * NCLASS),
                ("class_flops", C.c_double * NCLASS), ("class_bytes", C.c_double * NCLASS),
                ("fallback_chunks", i64), ("fallback_records", i64)]


def gpu():
    """libmfgpu.so: the sm_100a scoring engine."""
    global _gpu
    with _lock:
        if _gpu is None:
            # MFG_GPU_LIB selects another build in lib/ (same-box A/B timing runs)
            lib = _load(os.environ.get("MFG_GPU_LIB", "libmfgpu.so"))
            lib.mfg_create.argtypes = [C.POINTER(MfgConfig), C.POINTER(C.c_void_p)]
            lib.mfg_create.restype = C.c_int
            lib.mfg_score_batch.argtypes = [C.c_void_p, i32, i32, i32p, i64p, f32p]
            lib.mfg_score_batch.restype = C.c_int
            lib.mfg_score_device.argtypes = [C.c_void_p, i32, i32, C.c_void_p, i64p, C.c_void_p]
            lib.mfg_score_device.restype = C.c_int
            lib.mfg_set_stream.argtypes = [C.c_void_p, C.c_void_p]
            lib.mfg_set_stream.restype = C.c_int
            lib.mfg_last_error.argtypes = [C.c_void_p, i32p, C.c_char_p, C.c_size_t]
            lib.mfg_last_error.restype = C.c_int
            lib.mfg_destroy.argtypes = [C.c_void_p]
            lib.mfg_destroy.restype = None
            lib.mfg_check_container.argtypes = [C.c_char_p]
            lib.mfg_check_container.restype = C.c_int
            lib.mfg_get_model_info.argtypes = [C.c_void_p, C.POINTER(MfgModelInfo)]
            lib.mfg_get_model_info.restype = C.c_int
            lib.mfg_get_stats.argtypes = [C.c_void_p, C.POINTER(MfgStats)]
            lib.mfg_get_stats.restype = C.c_int
            lib.mfg_set_profile.argtypes = [C.c_void_p, i32]
            lib.mfg_set_profile.restype = C.c_int
            lib.mfg_reset_stats.argtypes = [C.c_void_p]
            lib.mfg_reset_stats.restype = C.c_int
            lib.mfgt_gemm.argtypes = [i32, i32, i32, i32, i32, f32p, f32p, f32p, f32p, f32p]
            lib.mfgt_gemm.restype = C.c_int
            lib.mfgt_attention.argtypes = [i32, i32, i32p, i32, i32, f32p, f32p, i32]
            lib.mfgt_attention.restype = C.c_int
            lib.mfgt_layernorm.argtypes = [i32, i32, f32p, f32p, f32p, f32p]
            lib.mfgt_layernorm.restype = C.c_int
            lib.mfgt_att_trace.argtypes = [i32, C.POINTER(C.c_longlong)]
            lib.mfgt_att_trace.restype = C.c_int
            lib.mfgt_plan_tiles.argtypes = [i32p, i32, i32, i32p, i32p, i32p, i32p, i32]
            lib.mfgt_plan_tiles.restype = C.c_int
            _gpu = lib
    return _gpu


def last_error(ctx=None):
    code = i32(0)
    buf = C.create_string_buffer(4096)
    gpu().mfg_last_error(ctx, C.byref(code), buf, len(buf))
    return int(code.value), buf.value.decode("utf-8", "replace")


def ptr(arr, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))
