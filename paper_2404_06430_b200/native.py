"""ctypes binding of libfedsim_b200.so (the C ABI in include/fedsim_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a) into ``paper_2404_06430_b200/lib/``.  There is no fallback: if the
library or a CUDA device is missing, :func:`lib` raises
``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import NativeError, NativeUnavailable

LIB_DIR = Path(__file__).resolve().parent / "lib"
LIB_PATH = LIB_DIR / "libfedsim_b200.so"
ABI_VERSION = 1

_p = C.c_void_p
_i32 = C.c_int
_i64 = C.c_int64
_u64 = C.c_uint64
_f32 = C.c_float
_f64 = C.c_double

# name -> (restype, argtypes); must match include/fedsim_b200.h
SIGNATURES: dict[str, tuple] = {
    "fb_abi_version": (_i32, []),
    "fb_last_error": (C.c_char_p, []),
    "fb_device_info": (_i32, [_i32, C.POINTER(_i32), C.POINTER(_i64)]),
    "fb_launch_count": (_i64, []),
    "fb_timing_enable": (None, [_i32]),
    "fb_timing_report": (_i32, [C.c_char_p, _i32, C.POINTER(_f64), C.POINTER(_i64), _i32]),
    "fb_user_permutations": (_i32, [_u64, _p, _p, _i32, _p, _i32, _p, _p]),
    "fb_derive_seed": (_i32, [_p, _i64, C.POINTER(_u64)]),
    "fb_eval_linear_f32": (_i32, [_p, _i32, _i32, _p, _p, _p, _p, _i32, _p, _p, _p]),
    "fb_eval_mlp_f32": (_i32, [_p, _i32, _i32, _i32, _p, _p, _p, _p, _i32, _p, _p, _p]),
    "fb_local_sgd_linear_f32": (
        _i32,
        [_p, _i32, _i32, _p, _p, _p, _p, _p, _p, _i32, _i32, _i32, _f32, _f32, _p, _i64, _p, _i64, _p, _p],
    ),
    "fb_local_sgd_mlp_f32": (
        _i32,
        [_p, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _i32, _i32, _i32, _f32, _f32, _p, _i64, _p, _i64, _p, _p],
    ),
    "fb_gather_rows": (_i32, [_p, _i64, _p, _p, _i32, _p, _p, _i64, _p]),
    "fb_gather_rows_lite": (_i32, [_p, _i64, _p, _p, _i32, _p, _p, _i32, _p]),
    "fb_upload_pinned": (_i32, [_p, _p, _i64, _p]),
    "fb_cnn_workspace_bytes": (_i64, [_i32, _i32, _i32]),
    "fb_cnn_set_conv_impl": (_i32, [_i32]),
    "fb_eval_cnn_f32": (_i32, [_p, _p, _p, _p, _p, _i32, _i64, _p, _p, _i32, _p, _i64, _p, _p, _i32, _p]),
    "fb_local_sgd_cnn_f32": (
        _i32,
        [_p, _p, _p, _p, _p, _p, _p, _i32, _i32, _i32, _i32, _f32, _f32, _p, _i64, _p, _i32, _i32, _p, _i64, _p, _p,
         _i64, _p, _i32, _p, _p, _p],
    ),
    "fb_cnn_fc1_aggregate_f32": (_i32, [_p, _i32, _i32, _i32, _f32, _f32, _i32, _i32, _p, _i64, _p, _p]),
    "fb_lm_set_gemm_impl": (_i32, [_i32]),
    "fb_lm_num_params": (_i64, [_p]),
    "fb_lm_workspace_bytes": (_i64, [_p, _i32, _i32, _i32]),
    "fb_eval_lm_f32": (_i32, [_p, _p, _p, _p, _p, _p, _i32, _p, _p, _i32, _i32, _p, _i64, _p, _p, _i32, _p]),
    "fb_local_sgd_lm_f32": (
        _i32,
        [_p, _p, _p, _p, _p, _p, _p, _p, _i32, _i32, _i32, _f32, _f32, _p, _i64, _p, _i64, _p, _i32, _p, _i64, _p, _p,
         _p],
    ),
    "fb_resnet_num_params": (_i64, [_p]),
    "fb_resnet_workspace_bytes": (_i64, [_p, _i32, _i32]),
    "fb_eval_resnet_f32": (_i32, [_p, _p, _p, _i64, _p, _p, _p, _i32, _p, _p, _i32, _i32, _p, _i64, _p, _p, _i32, _p]),
    "fb_local_sgd_resnet_f32": (
        _i32,
        [_p, _p, _p, _i64, _p, _p, _p, _p, _p, _i32, _i32, _i32, _f32, _f32, _p, _i64, _p, _i64, _p, _i32, _p, _i64,
         _p, _p, _p],
    ),
    "fb_clip_workspace_bytes": (_i64, [_i32, _i64]),
    "fb_delta_norm_clip_f32": (_i32, [_p, _i64, _i32, _i64, _p, _f64, _p, _p, _p, _p, _p, _i64, _p]),
    "fb_delta_norm_clip_ex_f32": (_i32, [_p, _i64, _i32, _i64, _i64, _i64, _p, _p, _f64, _p, _p, _p, _p, _p, _i64, _p]),
    "fb_weighted_sum_workspace_bytes": (_i64, [_i32, _i64]),
    "fb_weighted_sum_f32": (_i32, [_p, _i64, _i32, _i64, _p, _p, _i32, _p, _i64, _p]),
    "fb_clip_aggregate_max_columns": (_i64, []),
    "fb_clip_aggregate_workspace_bytes": (_i64, [_i32, _i64]),
    "fb_clip_aggregate_f32": (_i32, [_p, _i64, _i32, _i64, _p, _f64, _p, _p, _p, _p, _p, _i32, _p, _i64, _p]),
    "fb_clip_aggregate_rows_f32": (_i32, [_p, _p, _i64, _i32, _i64, _p, _f64, _p, _p, _p, _p, _p, _i32, _p, _i64, _p]),
    "fb_sumsq_f32": (_i32, [_p, _i64, _p, _p, _i64, _p]),
    "fb_context_sums": (_i32, [_p, _p, _p, _p, _p, _p, _p, _i32, _i32, _p, _p]),
    "fb_gaussian_f32": (_i32, [_p, _i64, _f64, _u64, _u64, _i32, _p]),
    "fb_noise_avg_sgd_f32": (_i32, [_p, _p, _i64, _f64, _u64, _p, _f64, _f64, _p, _p]),
    "fb_scaffold_correction_f32": (_i32, [_p, _p, _i64, _p, _i32, _i64, _p, _i64, _p]),
    "fb_scaffold_payload_f32": (_i32, [_p, _i64, _p, _p, _i64, _p, _p, _i32, _i64, _p, _i64, _p, _i64, _p]),
    "fb_scatter_rows_f32": (_i32, [_p, _i64, _p, _p, _i64, _i32, _i64, _p]),
    "fb_noise_avg_adam_f32": (_i32, [_p, _p, _p, _p, _i64, _f64, _u64, _p, _f64, _f64, _f64, _f64, _f64, _i64, _p,
                                     _p]),
}

_LIB: C.CDLL | None = None


def load_library(path: str | os.PathLike | None = None) -> C.CDLL:
    """dlopen the library and declare every signature (no CUDA needed)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise NativeUnavailable(
            f"{p} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError = header/library mismatch
        fn.restype = res
        fn.argtypes = args
    if lib.fb_abi_version() != ABI_VERSION:
        raise NativeUnavailable(f"ABI mismatch: library {lib.fb_abi_version()} != {ABI_VERSION}")
    if path is None:
        _LIB = lib
    return lib


def lib() -> C.CDLL:
    """The loaded library, requiring a visible CUDA device."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible; the GPU engine has no CPU fallback")
    return load_library()


def check(status: int, what: str) -> None:
    if status != 0:
        msg = (_LIB.fb_last_error() or b"").decode(errors="replace") if _LIB else ""
        kind = {-1: ValueError, -3: NativeError}.get(status, NativeError)
        raise kind(f"{what} failed ({status}): {msg}")


def call(name: str, *args) -> int:
    """Invoke an fb_* entry point; raise on a non-zero status."""
    fn = getattr(lib(), name)
    rc = fn(*args)
    if SIGNATURES[name][0] is _i32 and name not in ("fb_abi_version", "fb_timing_report"):
        check(rc, name)
    return rc


def timing_report(max_entries: int = 256) -> dict[str, tuple[float, int]]:
    """{kernel name: (summed device ms, launches)} since fb_timing_enable(1)."""
    L = lib()
    names = C.create_string_buffer(64 * max_entries)
    ms = (_f64 * max_entries)()
    cnt = (_i64 * max_entries)()
    k = L.fb_timing_report(names, len(names), ms, cnt, max_entries)
    check(0 if k >= 0 else k, "fb_timing_report")
    keys = names.value.decode().split("\n")[:k]
    return {n: (ms[i], cnt[i]) for i, n in enumerate(keys)}


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
