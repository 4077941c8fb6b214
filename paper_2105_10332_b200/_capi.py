"""ctypes binding of the C-ABI in include/sweptgpu.h (libsweptgpu.so, in-tree).

The library is the product: there is no Python or CPU fallback.  Loading fails
loudly if the shared object is missing; calls that need a GPU fail with
``CudaError`` when no device is visible.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libsweptgpu.so"

SG_OK, SG_EINVAL, SG_ENONPHYS, SG_ETRANSPORT, SG_EIO, SG_ELOGIC, SG_ECUDA = range(7)
SG_HEAT, SG_EULER = 0, 1
SG_SWEPT, SG_STANDARD = 0, 1
SG_WALL, SG_VIRTUAL = 0, 1


class sg_config(C.Structure):
    _fields_ = [
        ("problem", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("block", C.c_int),
        ("share", C.c_double), ("steps", C.c_long), ("ranks", C.c_int), ("engine", C.c_int),
        ("mode", C.c_int), ("link_latency", C.c_double), ("link_bandwidth", C.c_double),
        ("pool_a_workers", C.c_int), ("pool_a_cost", C.c_double),
        ("pool_b_workers", C.c_int), ("pool_b_cost", C.c_double),
        ("cell_cost", C.c_double), ("heat_alpha", C.c_double), ("heat_fourier", C.c_double),
        ("gamma", C.c_double), ("cfl", C.c_double), ("snapshot_path", C.c_char_p),
        ("snapshot_every", C.c_long), ("px", C.c_int), ("py", C.c_int), ("devices", C.c_int),
    ]


class sg_result(C.Structure):
    _fields_ = [
        ("engine", C.c_int), ("problem", C.c_int), ("mode", C.c_int),
        ("nx", C.c_int), ("ny", C.c_int), ("block", C.c_int), ("ranks", C.c_int),
        ("px", C.c_int), ("py", C.c_int), ("nvars", C.c_int),
        ("steps_requested", C.c_long), ("actual_steps", C.c_long), ("total_levels", C.c_long),
        ("octahedra", C.c_long), ("communicates", C.c_long), ("final_level", C.c_long),
        ("dt", C.c_double), ("dx", C.c_double), ("dy", C.c_double),
        ("setup_seconds", C.c_double), ("wall_seconds", C.c_double), ("solve_seconds", C.c_double),
        ("modeled_seconds", C.c_double), ("messages", C.c_long), ("bytes", C.c_longlong),
        ("cell_updates", C.c_longlong), ("snapshot_frames", C.c_long), ("kernel_launches", C.c_long),
        ("final_field", C.POINTER(C.c_double)),
        ("nparts", C.c_int), ("part_messages", C.POINTER(C.c_long)), ("part_bytes", C.POINTER(C.c_longlong)),
    ]


# every symbol include/sweptgpu.h declares (tests check the export table)
EXPORTS = (
    "sg_config_default", "sg_validate", "sg_run", "sg_free_result", "sg_solver_create",
    "sg_solver_reset", "sg_solver_solve", "sg_solver_fetch", "sg_solver_kernel_stats",
    "sg_solver_upload", "sg_solver_download", "sg_solver_initial", "sg_solver_set_profile", "sg_solver_destroy", "sg_plan_info", "sg_max_levels", "sg_schedule",
    "sg_measure_fp64_peak",
    "sg_div_selftest",
    "sg_substep", "sg_fnv1a64", "sg_version", "sg_device_count", "sg_dist_create", "sg_dist_blob", "sg_dist_connect",
)

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2105_10332_b200/csrc` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(str(LIB_PATH))
    cp, rp = C.POINTER(sg_config), C.POINTER(sg_result)
    sp = C.c_void_p
    L.sg_config_default.argtypes = [cp]
    L.sg_config_default.restype = None
    L.sg_validate.argtypes = [cp, C.c_char_p, C.c_size_t]
    L.sg_run.argtypes = [cp, rp, C.c_char_p, C.c_size_t]
    L.sg_free_result.argtypes = [rp]
    L.sg_free_result.restype = None
    L.sg_solver_create.argtypes = [cp, C.POINTER(sp), C.c_char_p, C.c_size_t]
    L.sg_solver_reset.argtypes = [sp, C.c_char_p, C.c_size_t]
    L.sg_solver_solve.argtypes = [sp, C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
    L.sg_solver_fetch.argtypes = [sp, rp, C.c_char_p, C.c_size_t]
    L.sg_solver_kernel_stats.argtypes = [sp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_long),
                                         C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.sg_solver_set_profile.argtypes = [sp, C.c_int]
    L.sg_solver_upload.argtypes = [sp, C.c_void_p, C.c_char_p, C.c_size_t]
    L.sg_solver_download.argtypes = [sp, C.c_void_p, C.c_char_p, C.c_size_t]
    L.sg_solver_initial.argtypes = [sp, C.c_void_p, C.c_char_p, C.c_size_t]
    L.sg_solver_destroy.argtypes = [sp]
    L.sg_solver_destroy.restype = None
    L.sg_plan_info.argtypes = [C.c_int, C.c_int, C.c_long, C.POINTER(C.c_long), C.c_char_p, C.c_size_t,
                               C.c_char_p, C.c_size_t]
    L.sg_max_levels.argtypes = [C.c_int, C.c_int]
    L.sg_measure_fp64_peak.argtypes = []
    L.sg_measure_fp64_peak.restype = C.c_double
    L.sg_div_selftest.argtypes = [C.c_long, C.c_uint64, C.POINTER(C.c_double)]
    L.sg_div_selftest.restype = C.c_long
    L.sg_schedule.argtypes = [C.c_long, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_long)]
    L.sg_schedule.restype = C.c_long
    L.sg_substep.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                             C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_double), C.c_void_p,
                             C.c_char_p, C.c_size_t]
    L.sg_dist_create.argtypes = [cp, C.c_int, C.c_int, C.POINTER(sp), C.c_char_p, C.c_size_t]
    L.sg_dist_blob.argtypes = [sp, C.c_void_p, C.c_long, C.c_char_p, C.c_size_t]
    L.sg_dist_blob.restype = C.c_long
    L.sg_dist_connect.argtypes = [sp, C.c_void_p, C.c_long, C.c_char_p, C.c_size_t]
    L.sg_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
    L.sg_fnv1a64.restype = C.c_uint64
    L.sg_version.argtypes = []
    L.sg_version.restype = C.c_char_p
    L.sg_device_count.argtypes = []
    _lib = L
    return L


def errbuf():
    return C.create_string_buffer(2048)


os.environ.setdefault("CUDA_MODULE_LOADING", "LAZY")
