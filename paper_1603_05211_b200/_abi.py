"""ctypes binding of include/af_gpu.h (libafgpu.so).

There is no fallback: if the library is missing or fails to load, importing
the solver API raises. The product path is the CUDA library and nothing else.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

LIB_PATH = _build.LIB

AF_OK = 0
AF_E_NONPHYSICAL = 1
AF_E_REGISTER_MISMATCH = 2
AF_E_CONFIG = 3
AF_E_LEVEL_MISMATCH = 4
AF_E_CUDA = 5
AF_E_NCCL = 6
AF_E_ARGUMENT = 7
AF_E_UNSUPPORTED = 8
AF_E_INTERNAL = 9
AF_E_IO = 10


class Config(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("level", C.c_int), ("origin", C.c_double), ("extent", C.c_double),
        ("gamma", C.c_double), ("bc", C.c_int * 6), ("flux", C.c_int), ("limiter", C.c_int),
        ("integrator", C.c_int), ("device", C.c_int),
    ]


class RunSummary(C.Structure):
    _fields_ = [("wall_seconds", C.c_double), ("sum_cells", C.c_double),
                ("sum_leaves", C.c_double), ("n_steps", C.c_long), ("l1_rho", C.c_double)]


class Rates(C.Structure):
    _fields_ = [("cpu_compression", C.c_double), ("memory_compression", C.c_double),
                ("mesh_compression", C.c_double), ("perturbation", C.c_double),
                ("overhead", C.c_double)]


class StepDiag(C.Structure):
    _fields_ = [("max_wave_speed", C.c_double), ("fallbacks", C.c_long)]


class RunDiag(C.Structure):
    _fields_ = [("max_wave_speed", C.c_double), ("max_cfl", C.c_double),
                ("fallbacks", C.c_long), ("steps_done", C.c_long), ("t", C.c_double)]


class ErrorRec(C.Structure):
    _fields_ = [("status", C.c_int), ("step", C.c_long), ("stage", C.c_int), ("i", C.c_int),
                ("j", C.c_int), ("k", C.c_int), ("level", C.c_int), ("is_ghost", C.c_int),
                ("rho", C.c_double), ("p", C.c_double), ("message", C.c_char * 512)]


class MROptions(C.Structure):
    _fields_ = [("eps", C.c_double), ("eps_level", C.POINTER(C.c_double)),
                ("min_leaf_level", C.c_int), ("local_time", C.c_int), ("lt_gap", C.c_int),
                ("storage", C.c_int), ("brick_shift", C.c_int)]


class MRCycle(C.Structure):
    _fields_ = [("leaves", C.c_long), ("nodes", C.c_long), ("sub", C.c_long), ("top", C.c_int),
                ("dt", C.c_double), ("updates", C.c_long)]


class AmrOptions(C.Structure):
    _fields_ = [("eps_rho", C.c_double), ("eps_p", C.c_double),
                ("cluster_efficiency", C.c_double), ("time_refine", C.c_int),
                ("flux_correction", C.c_int), ("max_levels", C.c_int)]


AMR_IC = C.CFUNCTYPE(None, C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double), C.c_void_p)


class SnapshotHeader(C.Structure):
    _fields_ = [("dim", C.c_int), ("level", C.c_int), ("gamma", C.c_double),
                ("time", C.c_double), ("origin", C.c_double), ("extent", C.c_double)]


# name -> (restype, argtypes); the complete exported surface of af_gpu.h
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p
SIGNATURES = {
    "af_version": (C.c_char_p, []),
    "af_abi_version": (C.c_int, []),
    "af_case_fill": (C.c_int, [C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_int, C.c_int, _dp]),
    "af_comm_unique_id": (C.c_int, [C.c_char_p]),
    "af_comm_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
    "af_comm_destroy": (C.c_int, [_vp]),
    "af_comm_create_local": (C.c_int, [C.c_int, C.c_int, C.POINTER(_vp)]),
    "af_uniform_create": (C.c_int, [C.POINTER(Config), _vp, C.POINTER(_vp)]),
    "af_uniform_destroy": (C.c_int, [_vp]),
    "af_uniform_set_stream": (C.c_int, [_vp, _vp]),
    "af_uniform_set_numerics": (C.c_int, [_vp, C.c_int]),
    "af_uniform_local_extent": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "af_slab_extent": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                 C.POINTER(C.c_int)]),
    "af_uniform_upload": (C.c_int, [_vp, _vp]),
    "af_uniform_download": (C.c_int, [_vp, _vp]),
    "af_uniform_step": (C.c_int, [_vp, C.c_double, C.POINTER(StepDiag)]),
    "af_rates_compute": (C.c_int, [C.POINTER(RunSummary), C.POINTER(RunSummary), C.c_double,
                                   C.POINTER(Rates)]),
    "af_uniform_rk2_stage": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, _vp, C.POINTER(StepDiag)]),
    "af_uniform_run": (C.c_int, [_vp, C.c_long, C.c_double, C.c_double, _dp,
                                 C.POINTER(RunDiag)]),
    "af_uniform_speed_sum": (C.c_int, [_vp, _dp]),
    "af_uniform_sync": (C.c_int, [_vp]),
    "af_uniform_last_error": (C.c_int, [_vp, C.POINTER(ErrorRec)]),
    "af_uniform_kernel_launches": (C.c_int, [_vp, C.POINTER(C.c_long)]),
    "af_uniform_create_group": (C.c_int, [C.POINTER(Config), C.c_int, C.POINTER(_vp)]),
    "af_uniform_run_group": (C.c_int, [C.POINTER(_vp), C.c_int, C.c_long, C.c_double, C.c_double,
                                       _dp, C.POINTER(RunDiag)]),
    "af_mr_create": (C.c_int, [C.POINTER(Config), C.POINTER(MROptions), C.POINTER(_vp)]),
    "af_mr_create_dist": (C.c_int, [C.POINTER(Config), C.POINTER(MROptions), _vp,
                                    C.POINTER(_vp)]),
    "af_mr_set_numerics": (C.c_int, [_vp, C.c_int]),
    "af_mr_local_rows": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "af_mr_memory": (C.c_int, [_vp, C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong),
                               C.POINTER(C.c_ulonglong)]),
    "af_mr_destroy": (C.c_int, [_vp]),
    "af_mr_set_stream": (C.c_int, [_vp, _vp]),
    "af_mr_build": (C.c_int, [_vp, _vp]),
    "af_mr_refine": (C.c_int, [_vp, C.c_int]),
    "af_mr_refine_buffer": (C.c_int, [_vp, C.c_double, C.POINTER(C.c_int), C.c_int]),
    "af_mr_solver_stats": (C.c_int, [_vp, _dp, C.POINTER(C.c_long)]),
    "af_mr_add_virtual_leaves": (C.c_int, [_vp]),
    "af_mr_remove_virtual_leaves": (C.c_int, [_vp]),
    "af_mr_coarsen": (C.c_int, [_vp]),
    "af_mr_evolve_global": (C.c_int, [_vp, C.c_double, C.POINTER(StepDiag)]),
    "af_mr_advance_local": (C.c_int, [_vp, C.c_int, C.c_double, C.c_double,
                                      C.POINTER(StepDiag)]),
    "af_mr_run": (C.c_int, [_vp, C.c_long, C.c_double, C.c_double, C.POINTER(MRCycle), C.c_long,
                            C.POINTER(RunDiag)]),
    "af_mr_counts": (C.c_int, [_vp, C.POINTER(C.c_long), C.POINTER(C.c_long),
                               C.POINTER(C.c_long)]),
    "af_mr_coarsest_leaf_level": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "af_mr_leaf_keys": (C.c_int, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_size_t)]),
    "af_mr_to_uniform": (C.c_int, [_vp, C.c_int, _vp]),
    "af_mr_details": (C.c_int, [_vp, C.c_int, _vp]),
    "af_mr_profile": (C.c_int, [_vp, C.c_int]),
    "af_mr_stage_stats": (C.c_int, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_long),
                                    C.POINTER(C.c_long)]),
    "af_mr_last_error": (C.c_int, [_vp, C.POINTER(ErrorRec)]),
    "af_mr_kernel_launches": (C.c_int, [_vp, C.POINTER(C.c_long)]),
    "af_snapshot_write": (C.c_int, [C.c_char_p, C.POINTER(SnapshotHeader), _vp]),
    "af_snapshot_read": (C.c_int, [C.c_char_p, C.POINTER(SnapshotHeader), _vp]),
    "af_restrict_to_level": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, _vp]),
    "af_l1_error": (C.c_int, [C.c_int, C.c_int, C.c_double, _vp, C.c_int, _vp, _dp]),
    "af_check_division": (C.c_int, [C.c_long, C.c_uint64, C.c_int, C.c_int,
                                    C.POINTER(C.c_ulonglong)]),
    "af_mr_dump": (C.c_int, [_vp, C.c_char_p, C.POINTER(C.c_size_t)]),
    "af_amr_create": (C.c_int, [C.POINTER(Config), C.POINTER(AmrOptions), C.POINTER(_vp)]),
    "af_amr_destroy": (C.c_int, [_vp]),
    "af_amr_initialize": (C.c_int, [_vp, AMR_IC, _vp]),
    "af_amr_initialize_case": (C.c_int, [_vp, C.c_int, C.c_uint64, C.c_double]),
    "af_amr_sync_ghosts": (C.c_int, [_vp, C.c_int, C.c_double]),
    "af_amr_remesh": (C.c_int, [_vp, C.c_int]),
    "af_amr_update_level": (C.c_int, [_vp, C.c_int, C.c_double, C.POINTER(StepDiag)]),
    "af_amr_average_down": (C.c_int, [_vp, C.c_int]),
    "af_amr_flux_correct": (C.c_int, [_vp, C.c_int]),
    "af_amr_run": (C.c_int, [_vp, C.c_long, C.c_double, C.POINTER(C.c_long), C.POINTER(C.c_long),
                             C.POINTER(RunDiag)]),
    "af_amr_n_levels": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "af_amr_level_info": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_long), _dp, _dp]),
    "af_amr_boxes": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_int), C.c_int]),
    "af_amr_patch_data_cells": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(C.c_long)]),
    "af_amr_patch_data": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp]),
    "af_amr_assemble_level": (C.c_int, [_vp, C.c_int, _vp]),
    "af_amr_total_conserved": (C.c_int, [_vp, _dp]),
    "af_amr_l1_error": (C.c_int, [_vp, C.c_int, _vp, _dp]),
    "af_amr_counts": (C.c_int, [_vp, C.POINTER(C.c_long), C.POINTER(C.c_long)]),
    "af_amr_properly_nested": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "af_amr_dump_boxes": (C.c_int, [_vp, C.POINTER(C.c_char_p)]),
    "af_amr_last_error": (C.c_int, [_vp, C.POINTER(ErrorRec)]),
    "af_amr_kernel_launches": (C.c_int, [_vp, C.POINTER(C.c_long)]),
    "af_amr_cell_updates": (C.c_int, [_vp, C.POINTER(C.c_long)]),
    "af_amr_profile": (C.c_int, [_vp, C.c_int]),
    "af_amr_stage_stats": (C.c_int, [_vp, _dp, C.POINTER(C.c_long), C.POINTER(C.c_long)]),
    "af_amr_remesh_stats": (C.c_int, [_vp, _dp, C.POINTER(C.c_long)]),
    "af_amr_cluster_device": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_double,
                                        C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int)]),
    "af_amr_cluster": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                 C.c_double, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int)]),
}

_lib = None


def load(build_if_missing: bool = True):
    """Loads libafgpu.so (building it in-tree first if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing:
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libafgpu.so not found at {LIB_PATH}; run "
                          "`python -m paper_1603_05211_b200.build`")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
