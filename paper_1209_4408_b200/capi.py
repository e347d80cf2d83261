"""ctypes binding of the C-ABI in include/life_gpu.h (liblife_gpu.so).

Loading fails loudly when the CUDA library is missing: there is no CPU
fallback in this package.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LIFE_GPU_LIB") or os.path.join(PKG, "liblife_gpu.so")

# Status codes (include/life_gpu.h).
OK = 0
ERR_CONFIG = 1
ERR_DIMENSION_TOO_SMALL = 2
ERR_TOO_MANY_PARTS = 3
ERR_OUT_OF_BOUNDS = 4
ERR_STATE = 5
ERR_CUDA = 10
ERR_NO_DEVICE = 11
ERR_OUT_OF_MEMORY = 12

ENGINE_PACKED = 0
ENGINE_BYTE = 1
ENGINE_RESIDENT = 2
MAX_TEMPORAL_DEPTH = 16
PAIR_MAX_DEPTH = 12  # packed_il_kernel<K, 2> (W % 64 == 0)
QUAD_MAX_DEPTH = 7   # packed_il_kernel<K, 4> (W % 128 == 0)
MAX_BYTE_DEPTH = 8

OPT_PROFILE = 1
OPT_BATCH_TRAPEZOID = 2
OPT_HALO = 3
OPT_PAIR_DEPTH = 4
OPT_QUAD_DEPTH = 5
HALO_PEER = 0
HALO_COPY = 1

LAUNCH_STEP1 = 0
LAUNCH_FAST = 1
LAUNCH_ALL_PATHS = 2
LAUNCH_SPLIT = 3


class BandStats(C.Structure):
    """life_band_stats (include/life_gpu.h)."""
    _fields_ = [("band", C.c_int32), ("device", C.c_int32), ("y0", C.c_int64),
                ("rows", C.c_int64), ("passes", C.c_int64), ("run_ms", C.c_double),
                ("interior_ms", C.c_double), ("edge_ms", C.c_double), ("wait_ms", C.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}

# Every function the header declares: (name, restype, argtypes).
_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_u64 = C.c_uint64
SIGNATURES = [
    ("life_last_error", C.c_char_p, []),
    ("life_version", C.c_char_p, []),
    ("life_ctx_create", C.c_int, [C.c_int, C.POINTER(_vp)]),
    ("life_ctx_create_multi", C.c_int, [_i32, C.POINTER(C.c_int), C.POINTER(_vp)]),
    ("life_ctx_destroy", C.c_int, [_vp]),
    ("life_ctx_set_stream", C.c_int, [_vp, _vp]),
    ("life_ctx_sync", C.c_int, [_vp]),
    ("life_ctx_bands", C.c_int, [_vp, C.POINTER(_i32), _vp, _vp, C.POINTER(_i32)]),
    ("life_ctx_set_option", C.c_int, [_vp, _i32, _i64]),
    ("life_ctx_get_option", C.c_int, [_vp, _i32, C.POINTER(_i64)]),
    ("life_ctx_band_stats", C.c_int, [_vp, _i32, C.POINTER(BandStats)]),
    ("life_grid_upload_u8", C.c_int, [_vp, _vp, _i64, _i64, _i64]),
    ("life_grid_upload_packed", C.c_int, [_vp, _vp, _i64, _i64, _i64]),
    ("life_grid_init_random", C.c_int, [_vp, _i64, _i64, C.c_double, _u64, C.c_int]),
    ("life_grid_init_soup", C.c_int, [_vp, _i64, _i64, C.c_double, _i32, C.c_double, _u64,
                                      C.c_int]),
    ("life_grid_place_u8", C.c_int, [_vp, _vp, _i64, _i64, _i64, _i64]),
    ("life_grid_download_u8", C.c_int, [_vp, _vp, _i64]),
    ("life_grid_download_packed", C.c_int, [_vp, _vp, _i64]),
    ("life_grid_window_u8", C.c_int, [_vp, _i64, _i64, _i64, _i64, _vp]),
    ("life_grid_dims", C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64)]),
    ("life_population", C.c_int, [_vp, C.POINTER(_u64)]),
    ("life_grid_hash", C.c_int, [_vp, C.POINTER(_u64)]),
    ("life_run", C.c_int, [_vp, _i64, C.c_int, C.c_int, _vp, _i32, _vp]),
    ("life_step", C.c_int, [_vp, C.c_int]),
    ("life_run_batch", C.c_int, [_vp, _vp, _vp, _i32, _i64, _i64, _i64, _i64, C.c_int,
                                 C.POINTER(C.c_float)]),
    ("life_packed_auto_depth", C.c_int, [_i64, _i64]),
    ("life_packed_launch_kind", C.c_int, [_i64, _i64, _i32]),
    ("life_dev_packed_run", C.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i32,
                                      C.POINTER(_i32), _vp]),
    ("life_band_bounds", C.c_int, [_i64, _i32, _vp]),
    ("life_packed_pitch_words", _i64, [_i64]),
    ("life_byte_pitch", _i64, [_i64]),
    ("life_dev_packed_step", C.c_int, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i32,
                                       _vp]),
    ("life_dev_packed_step_peer", C.c_int, [_vp, _vp, _i64, _vp, _i64, _i64, _i64, _vp, _i64,
                                            _i64, _i64, _i32, _vp]),
    ("life_interleave_auto", C.c_int, [_i64, _i64, _i32, _i32, _i32, C.POINTER(_i32)]),
    ("life_dev_packed_zip", C.c_int, [_vp, _i64, _i64, _i64, _i64, _i32, _i32, _vp]),
    ("life_dev_packed_step_il", C.c_int, [_i32, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64,
                                          _i64, _i32, _vp]),
    ("life_dev_packed_run_il", C.c_int, [_i32, _vp, _vp, _i64, _i64, _i64, _i64, _i32,
                                         C.POINTER(_i32), _vp]),
    ("life_dev_packed_step_il_peer", C.c_int, [_i32, _vp, _vp, _i64, _vp, _i64, _i64, _i64, _vp,
                                               _i64, _i64, _i64, _i32, _vp]),
    ("life_dev_packed_run_resident", C.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, _vp]),
    ("life_resident_cluster_size", C.c_int, [_i64, _i64]),
    ("life_dev_alloc", C.c_int, [_i64, C.POINTER(_vp)]),
    ("life_dev_free", C.c_int, [_vp]),
    ("life_ipc_get_handle", C.c_int, [_vp, _vp]),
    ("life_ipc_open", C.c_int, [_vp, C.POINTER(_vp)]),
    ("life_ipc_close", C.c_int, [_vp]),
    ("life_dev_flag_write", C.c_int, [_vp, C.c_uint32, _vp]),
    ("life_dev_flag_wait_geq", C.c_int, [_vp, C.c_uint32, _vp]),
    ("life_dev_byte_step", C.c_int, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _vp]),
    ("life_dev_byte_pass", C.c_int, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i32,
                                     _vp]),
    ("life_dev_packed_random", C.c_int, [_vp, _i64, _i64, _i64, _i64, C.c_double, _u64, _vp]),
    ("life_dev_byte_random", C.c_int, [_vp, _i64, _i64, _i64, _i64, C.c_double, _u64, _vp]),
    ("life_dev_packed_population", C.c_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    ("life_dev_packed_row_hashes", C.c_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    ("life_fnv1a64", _u64, [_vp, _i64, _u64]),
    ("life_dev_pack", C.c_int, [_vp, _i64, _vp, _i64, _i64, _i64, _vp]),
    ("life_dev_unpack", C.c_int, [_vp, _i64, _vp, _i64, _i64, _i64, _vp]),
    ("life_measure_int_peak", C.c_int, [C.c_int, _i64, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]),
    ("life_kernel_launches", _u64, []),
]

_lib = None


class LibraryMissing(ImportError):
    pass


def lib() -> C.CDLL:
    """Loads liblife_gpu.so (built by paper_1209_4408_b200.build); raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is not built; run `python -m paper_1209_4408_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().life_last_error().decode(errors="replace")
