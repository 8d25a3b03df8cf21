"""ctypes binding of libsrm_b200.so (the C ABI declared in include/srm_b200.h).

The library is built in-tree (``make lib`` / ``__graft_entry__.build()``).  There is no
CPU fallback: if the shared object is missing, importing the bindings raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SRM_B200_LIB: an alternative build of the same library (tools/ tuning variants only)
LIB_PATH = os.environ.get("SRM_B200_LIB") or os.path.join(_HERE, "libsrm_b200.so")

c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)
c_int64_p = C.POINTER(C.c_int64)
c_int_p = C.POINTER(C.c_int)
c_uint32_p = C.POINTER(C.c_uint32)
c_uint8_p = C.POINTER(C.c_uint8)

NPHASE = 4


class Params(C.Structure):
    """engine.hpp:22-32 SrmParams (srm_b200_params)."""

    _fields_ = [
        ("c_w", C.c_double),
        ("c_m", C.c_double),
        ("c_r", C.c_double),
        ("n_k", C.c_int32),
        ("n_l", C.c_int32),
        ("f_target", C.c_double),
        ("max_iterations", C.c_int64),
        ("seed", C.c_uint64),
        ("reorder_period", C.c_int32),
    ]


class SnapshotMeta(C.Structure):
    """srm_b200_snapshot_meta: the Snapshot fields a file carries (snapshot_io.cpp:128-148)."""

    _fields_ = [
        ("volume_fraction", C.c_double),
        ("iteration_count", C.c_int64),
        ("seed", C.c_uint64),
        ("params", Params),
    ]


class ProgressRecord(C.Structure):
    _fields_ = [
        ("iteration", C.c_int64),
        ("volume_fraction", C.c_double),
        ("accepted", C.c_int32),
        ("elapsed_seconds", C.c_double),
        ("rounds", C.c_int32),
    ]


class GenerateOut(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("volume_fraction", C.c_double),
        ("iteration_count", C.c_int64),
        ("accepted_iterations", C.c_int64),
        ("rounds", C.c_int64),
        ("shake_rounds", C.c_int64),
    ]


class RoundStats(C.Structure):
    _fields_ = [
        ("overlap_pairs", C.c_int64),
        ("max_penetration", C.c_double),
        ("candidate_pairs", C.c_int64),
        ("movers", C.c_int64),
    ]


PROGRESS_FN = C.CFUNCTYPE(None, C.POINTER(ProgressRecord), C.c_void_p)

# name -> (restype, argtypes)
_SIGS = {
    "srm_b200_create": (C.c_int, [C.c_int, C.c_int, c_double_p, C.c_int64, C.c_int, C.POINTER(C.c_void_p)]),
    "srm_b200_destroy": (None, [C.c_void_p]),
    "srm_b200_last_error": (C.c_char_p, [C.c_void_p]),
    "srm_b200_create_error": (C.c_char_p, []),
    "srm_b200_upload": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "srm_b200_download": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "srm_b200_upload_records": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64]),
    "srm_b200_download_records": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64]),
    "srm_b200_count": (C.c_int64, [C.c_void_p]),
    "srm_b200_generate": (C.c_int, [C.c_void_p, C.POINTER(Params), C.c_int64, PROGRESS_FN, C.c_void_p, C.POINTER(GenerateOut)]),
    "srm_b200_relax_sweeps": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int, C.c_uint64]),
    "srm_b200_swell_all": (C.c_int, [C.c_void_p, C.c_double]),
    "srm_b200_reorder_by_locality": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p]),
    "srm_b200_max_bounding_radius": (C.c_int, [C.c_void_p, c_double_p]),
    "srm_b200_volume_fraction": (C.c_int, [C.c_void_p, c_double_p]),
    "srm_b200_grid_dims": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_double, c_int32_p, c_double_p, c_int64_p]),
    "srm_b200_grid_build": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
    "srm_b200_overlap_stats": (C.c_int, [C.c_void_p, C.c_double, C.POINTER(RoundStats)]),
    "srm_b200_round": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.c_void_p, C.POINTER(RoundStats)]),
    "srm_b200_rounds": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.POINTER(RoundStats)]),
    "srm_b200_rsa_place": (C.c_int, [C.c_int, c_double_p, C.c_int64, C.c_void_p, C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p, c_int64_p]),
    "srm_b200_describe": (C.c_int, [C.c_void_p, c_int_p, c_int_p, c_double_p]),
    "srm_b200_snapshot_encode": (C.c_int, [C.c_int, C.c_int, c_double_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                           c_int64_p]),
    "srm_b200_save_snapshot": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int]),
    "srm_b200_snapshot_info": (C.c_int, [C.c_char_p, c_int_p, c_int_p, c_int64_p, c_double_p, C.c_void_p]),
    "srm_b200_load_snapshot": (C.c_int, [C.c_void_p, C.c_char_p]),
    "srm_b200_io_error": (C.c_char_p, []),
    "srm_b200_rsa_platelets_device": (C.c_int, [C.c_void_p, C.c_int64, C.c_double, C.c_double, C.c_uint64, C.c_int64,
                                                c_int64_p, c_int64_p]),
    "srm_b200_rsa_device": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64, C.c_int64, c_int64_p, c_int64_p]),
    "srm_b200_nnd_histogram": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_void_p, c_int64_p, c_int64_p,
                                         C.c_void_p]),
    "srm_b200_pair_counts": (C.c_int, [C.c_void_p, c_double_p, C.c_int, C.c_void_p]),
    "srm_b200_platelet_order": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p]),
    "srm_b200_rsa_clustered": (C.c_int, [C.c_int, c_double_p, C.c_int64, C.c_void_p, C.c_int64, C.c_double, C.c_int64,
                                         C.c_uint64, C.c_void_p, C.c_void_p, c_int64_p]),
    "srm_b200_rsa_platelets": (C.c_int, [C.c_int64, C.c_double, C.c_double, c_double_p, C.c_int64, C.c_uint64, C.c_void_p,
                                         C.c_void_p, C.c_void_p, c_int64_p]),
    "srm_b200_upload_platelets": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p]),
    "srm_b200_download_platelets": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "srm_b200_set_rotation": (C.c_int, [C.c_void_p, C.c_double]),
    "srm_b200_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "srm_b200_launch_count": (C.c_int64, [C.c_void_p]),
    "srm_b200_reset_launch_count": (None, [C.c_void_p]),
    "srm_b200_graph_builds": (C.c_int64, [C.c_void_p]),
    "srm_b200_timing_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "srm_b200_timing_get": (C.c_int, [C.c_void_p, c_double_p, c_int64_p]),
    "srm_b200_sync": (C.c_int, [C.c_void_p]),
    "srm_b200_stopwatch": (C.c_int, [C.c_void_p, C.c_int, c_double_p]),
    "srm_b200_last_round_info": (C.c_int, [C.c_void_p, c_int64_p]),
    "srm_b200_set_generate_mode": (C.c_int, [C.c_void_p, C.c_int]),
    "srm_b200_selftest_philox": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "srm_b200_selftest_unit_vectors": (C.c_int, [C.c_int, C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p,
                                                 C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Load libsrm_b200.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
                "the B200 SRM path has no CPU fallback")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib
