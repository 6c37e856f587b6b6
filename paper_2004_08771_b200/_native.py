"""ctypes binding of the in-tree C ABI (include/hogbatch_b200.h).

The product path has exactly one implementation: `libhogbatch_b200.so`.
If the library is missing or a call fails there is no fallback -- the error
surfaces as ValueError (argument/shape errors, as the reference raises at
linalg.py:40-44 / nn.py:110-113) or RuntimeError (CUDA/NCCL/state errors).
ctypes releases the GIL for the duration of each call, so device waits never
block the coordinator or Hogwild threads (SURVEY.md §8b "Threading").
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("HOGBATCH_B200_LIB", _PKG / "libhogbatch_b200.so"))

HB_OK, HB_EINVAL, HB_ECUDA, HB_ENCCL, HB_ESTATE, HB_EPARSE = 0, 1, 2, 3, 4, 5
HB_SPARSE_INPUT = 1
HB_PRECISION_TF32 = 2
HB_SPARSE_KERNELS = 4
HB_DENSIFY_MAX_DIN = 512
HB_STEP_EMIT_GRAD = 1
HB_STEP_TIMED = 2
HB_STEP_ASYNC = 4
HB_STEP_MERGE = 8
HB_STEP_SOLE_WRITER = 16
HB_STEP_LAND_ASYNC = 32
HB_PEER_HANDLE_BYTES = 128

_p = C.c_void_p
_i32, _i64, _u32, _f64 = C.c_int, C.c_int64, C.c_uint32, C.c_double
_dp, _fp = C.POINTER(C.c_double), C.POINTER(C.c_float)
_i64p, _i32p = C.POINTER(C.c_int64), C.POINTER(C.c_int32)

# name -> (restype, argtypes); every symbol include/hogbatch_b200.h declares
SIGNATURES = {
    "hb_last_error": (C.c_char_p, []),
    "hb_version": (C.c_char_p, []),
    "hb_device_count": (_i32, [C.POINTER(_i32)]),
    "hb_ctx_create": (_i32, [C.POINTER(_p), _i32, _i32, C.POINTER(_i32), _i32, _u32]),
    "hb_ctx_destroy": (_i32, [_p]),
    "hb_set_weights_f64": (_i32, [_p, _i32, _dp]),
    "hb_set_bias_f64": (_i32, [_p, _i32, _dp]),
    "hb_get_weights_f64": (_i32, [_p, _i32, _dp]),
    "hb_get_weights_f32": (_i32, [_p, _i32, _fp]),
    "hb_merge_grad_into_f64": (_i32, [_p, _i32, _dp, _f64]),
    "hb_get_grad_f32": (_i32, [_p, _i32, _fp]),
    "hb_set_weights_all_f64": (_i32, [_p, C.POINTER(_dp)]),
    "hb_merge_grads_all_into_f64": (_i32, [_p, C.POINTER(_dp), _f64]),
    "hb_host_register": (_i32, [_p, C.c_size_t]),
    "hb_host_unregister": (_i32, [_p]),
    "hb_stage_dense_f64": (_i32, [_p, _dp, _i64, _i64, _i64p]),
    "hb_stage_dense_f32": (_i32, [_p, _fp, _i64, _i64, _i64p]),
    "hb_stage_csr": (_i32, [_p, _i64p, _i32p, _fp, _i64, _i64p]),
    "hb_stage_dense_as_csr_f64": (_i32, [_p, _dp, _i64, _i64, _i64p]),
    "hb_staged_rows": (_i64, [_p]),
    "hb_stage_blobs": (_i32, [_p, _i64, _i64, _i32, _dp, C.c_uint64]),
    "hb_read_staged": (_i32, [_p, _i64, _i64, _fp, _i64p]),
    "hb_permute_epoch": (_i32, [_p, _i64p, _i64]),
    "hb_libsvm_scan": (_i32, [C.c_char_p, C.c_size_t, _i64, _i32, _i64p, _i64p]),
    "hb_libsvm_fill": (_i32, [C.c_char_p, C.c_size_t, _i64, _i32, _i64p, _i32p, _dp, _i64p]),
    "hb_train_step": (_i32, [_p, _i64, _i32, _f64, _u32, _dp]),
    "hb_train_step_host_dense": (_i32, [_p, _fp, _i64, _i64p, _i32, _f64, _u32, _dp]),
    "hb_train_step_host_csr": (_i32, [_p, _i64p, _i32p, _fp, _i64p, _i32, _f64, _u32, _dp]),
    "hb_replica_begin": (_i32, [_p, C.POINTER(_dp), _i64, _i32, _f64, _u32]),
    "hb_replica_end": (_i32, [_p, _dp]),
    "hb_replica_landed": (_i32, [_p]),
    "hb_replica_step": (_i32, [_p, C.POINTER(_dp), _i64, _i32, _f64, _u32, _dp]),
    # host batch arrays pass as integer addresses (ndarray.ctypes.data): half the cost of data_as per call
    "hb_replica_step_host_dense": (_i32, [_p, C.POINTER(_dp), _p, _i64, _p, _i32, _f64, _u32, _dp]),
    "hb_replica_step_host_csr": (_i32, [_p, C.POINTER(_dp), _p, _p, _p, _p, _i32, _f64, _u32, _dp]),
    "hb_eval_loss_sum": (_i32, [_p, _i64, _i64, _dp]),
    "hb_forward": (_i32, [_p, _i64, _i32]),
    "hb_get_activation_f32": (_i32, [_p, _i32, _i32, _fp]),
    "hb_last_step_ms": (_i32, [_p, _fp]),
    "hb_last_step_launches": (_i32, [_p, C.POINTER(_i32)]),
    "hb_last_xfer_bytes": (_i32, [_p, _i64p, _i64p]),
    "hb_synchronize": (_i32, [_p]),
    "hb_profile_enable": (_i32, [_p, _i32]),
    "hb_profile_filter": (_i32, [_p, C.c_char_p]),
    "hb_profile_read": (_i32, [_p, _i32, C.c_char_p, _dp, C.POINTER(_i32), C.POINTER(_i32)]),
    "hb_nccl_unique_id": (_i32, [_p]),
    "hb_comm_init": (_i32, [_p, _p, _i32, _i32]),
    "hb_merge_allreduce": (_i32, [_p]),
    "hb_comm_destroy": (_i32, [_p]),
    "hb_host_merge_threads": (_i32, [_i32, _i32]),
    "hb_host_pool_selftest": (_i32, [_i32, _i64p]),
    "hb_probe_l2_gather": (_i32, [_i32, _i64, _i32, _i32, _i32, _dp]),
    "hb_peer_handle": (_i32, [_p, _p]),
    "hb_peer_attach": (_i32, [_p, _i32, _i32, _p]),
}

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def load(build_if_missing: bool = False):
    """Load (once) and type the shared library.  Raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        if build_if_missing:
            from . import build

            build.build()
        else:
            raise NativeLibraryMissing(
                f"{LIB_PATH} not found: build it with `python -m paper_2004_08771_b200.build` "
                "(the GPU path has no CPU fallback)"
            )
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return (load().hb_last_error() or b"").decode(errors="replace")


def check(rc: int) -> None:
    if rc == HB_OK:
        return
    msg = (_lib.hb_last_error() or b"").decode(errors="replace")
    if rc in (HB_EINVAL, HB_EPARSE):
        raise ValueError(msg)
    raise RuntimeError(f"hogbatch_b200 error {rc}: {msg}")


def device_count() -> int:
    lib = load()
    n = _i32(0)
    check(lib.hb_device_count(C.byref(n)))
    return n.value


def ptr(a, ctype):
    """Raw pointer of a C-contiguous numpy array (no copy)."""
    return a.ctypes.data_as(C.POINTER(ctype))
