"""ctypes binding of libswe_b200.so (include/swe_dev.h, include/swe_host.h).

The library is required: importing the package without it raises -- there is
no CPU fallback for the step.  Build it with paper_1807_00672_b200.build or
__graft_entry__.build().
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("SWE_B200_LIB", Path(__file__).resolve().parent / "libswe_b200.so"))

c_int, c_ll, c_long, c_double, c_void_p, c_char_p, c_uint = (
    C.c_int, C.c_longlong, C.c_long, C.c_double, C.c_void_p, C.c_char_p, C.c_uint)
P_double = C.POINTER(C.c_double)
P_int = C.POINTER(C.c_int)
P_ll = C.POINTER(C.c_longlong)
P_long = C.POINTER(C.c_long)


class swe_params(C.Structure):
    _fields_ = [("g", c_double), ("h_dry", c_double), ("cfl", c_double),
                ("dt_max", c_double), ("h_ref", c_double)]


class swe_mesh_view(C.Structure):
    _fields_ = [("n_cells", c_int), ("n_edges", c_int),
                ("area", P_double), ("inradius", P_double), ("bed", P_double),
                ("manning", P_double), ("cx", P_double), ("cy", P_double),
                ("cell_edge", P_int), ("cell_sign", P_int),
                ("edge_left", P_int), ("edge_right", P_int),
                ("nx", P_double), ("ny", P_double), ("len", P_double),
                ("n_owned", c_int)]


class swe_status(C.Structure):
    _fields_ = [("code", c_int), ("index", c_ll), ("step", c_ll), ("dt", c_double),
                ("h", c_double)]


class swe_step_record(C.Structure):
    _fields_ = [("step", c_ll), ("t", c_double), ("dt", c_double),
                ("max_speed", c_double), ("mass", c_double)]


SWE_OK, SWE_NONFINITE_SPEED, SWE_NEGATIVE_DEPTH, SWE_BLOWUP, SWE_CUDA, SWE_NCCL, SWE_INVALID = range(7)
SWE_FLAG_IDENTITY_ORDER = 1
SWE_FLAG_NO_GRAPH = 2
SWE_FLAG_TWO_PHASE = 4

_SIGS = {
    # device solver (swe_dev.h)
    "swe_dev_create": (c_int, [C.POINTER(swe_mesh_view), C.POINTER(swe_params), c_int, c_uint,
                               C.POINTER(c_void_p)]),
    "swe_dev_destroy": (c_int, [c_void_p]),
    "swe_dev_set_state": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_ll]),
    "swe_dev_get_state": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, P_double, P_ll]),
    "swe_dev_set_state_device": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_ll]),
    "swe_dev_get_state_device": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "swe_dev_get_ledger": (c_int, [c_void_p, P_double, P_ll]),
    "swe_dev_set_ledger": (c_int, [c_void_p, c_double, c_ll]),
    "swe_dev_step": (c_int, [c_void_p, c_double, C.POINTER(swe_step_record), C.POINTER(swe_status)]),
    "swe_dev_advance": (c_int, [c_void_p, c_double, c_ll, c_double, c_void_p, c_ll, P_ll,
                                C.POINTER(swe_status)]),
    "swe_dev_advance_n_async": (c_int, [c_void_p, c_ll, c_double]),
    "swe_dev_advance_async": (c_int, [c_void_p, c_double, c_ll, c_double, c_ll]),
    "swe_dev_records": (c_int, [c_void_p, c_void_p, c_ll, P_ll, C.POINTER(swe_status)]),
    "swe_dev_synchronize": (c_int, [c_void_p, C.POINTER(swe_status)]),
    "swe_dev_snapshot_async": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "swe_dev_snapshot_wait": (c_int, [c_void_p, c_int]),
    "swe_dev_host_alloc": (c_void_p, [c_ll]),
    "swe_dev_host_free": (None, [c_void_p]),
    "swe_dev_host_register": (c_int, [c_void_p, c_ll]),
    "swe_dev_host_unregister": (c_int, [c_void_p]),
    "swe_dev_compute_fluxes": (c_int, [c_void_p, c_void_p, c_void_p, C.POINTER(swe_status)]),
    "swe_dev_total_mass": (c_int, [c_void_p, P_double]),
    "swe_dev_set_profiling": (c_int, [c_void_p, c_int]),
    "swe_dev_kernel_times": (c_int, [c_void_p, P_double, P_ll, c_int]),
    "swe_dev_info": (c_int, [c_void_p, P_ll, c_int]),
    "swe_dev_set_halo_plan": (c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p]),
    "swe_dev_pack_halo": (c_int, [c_void_p, c_void_p]),
    "swe_dev_unpack_halo": (c_int, [c_void_p, c_void_p]),
    "swe_dev_local_cfl": (c_int, [c_void_p, P_double, P_double, P_double,
                                  C.POINTER(swe_status)]),
    "swe_dev_step_global": (c_int, [c_void_p, c_double, c_double, c_double,
                                    C.POINTER(swe_step_record), C.POINTER(swe_status)]),
    "swe_dev_link_export": (c_int, [c_void_p, C.POINTER(c_void_p), c_void_p]),
    "swe_dev_link": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_int,
                             c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double]),
    "swe_dev_link_phase": (c_int, [c_void_p, c_int, c_double]),
    "swe_dev_last_record": (c_int, [c_void_p, C.POINTER(swe_step_record), C.POINTER(swe_status)]),
    "swe_dev_run_ranks": (c_int, [c_void_p, c_int, c_ll, c_double, c_int]),
    "swe_dev_cell_skip": (c_int, [c_void_p, c_void_p]),
    "swe_dev_cell_order": (c_int, [c_void_p, c_void_p]),
    "swe_dev_stream": (c_void_p, [c_void_p]),
    "swe_dev_memory_bytes": (c_ll, [c_void_p]),
    "swe_dev_launch_count": (c_ll, []),
    "swe_dev_point_eval": (c_int, [c_int, c_ll, C.POINTER(swe_params), c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p]),
    "swe_dev_stable_dt": (c_int, [c_int, c_ll, C.POINTER(swe_params), c_void_p, c_void_p, c_void_p,
                                  c_void_p, P_double, P_ll]),
    "swe_dev_mass": (c_int, [c_int, c_ll, c_void_p, c_void_p, P_double]),
    "swe_dev_step_timed": (c_int, [c_void_p, c_double, C.POINTER(swe_step_record),
                                   C.POINTER(swe_status), P_double, P_double]),
    "swe_dev_strerror": (c_char_p, [c_int]),
    "swe_dev_last_error": (c_char_p, []),
    # host input producers (swe_host.h)
    "swe_host_raw_square": (c_void_p, [c_int, c_int, c_double, c_double, c_char_p, c_int]),
    "swe_host_raw_unstructured": (c_void_p, [c_int, c_int, c_double, c_double, c_double,
                                             C.c_ulonglong, c_char_p, c_int]),
    "swe_host_raw_arrays": (c_void_p, [c_int, c_void_p, c_int, c_void_p]),
    "swe_host_raw_sizes": (None, [c_void_p, P_int, P_int]),
    "swe_host_raw_export": (None, [c_void_p, c_void_p, c_void_p]),
    "swe_host_raw_free": (None, [c_void_p]),
    "swe_host_case_defaults": (c_int, [c_char_p, c_void_p]),
    "swe_host_init_case": (c_int, [c_void_p, c_char_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_char_p, c_int]),
    "swe_host_scenario": (c_void_p, [c_char_p, c_double, c_int, C.c_ulonglong, c_int, P_double,
                                     c_char_p, c_int]),
    "swe_host_scenario_raw": (c_void_p, [c_void_p]),
    "swe_host_scenario_fields": (None, [c_void_p] + [c_void_p] * 5),
    "swe_host_scenario_free": (None, [c_void_p]),
    "swe_host_build_mesh": (c_void_p, [c_void_p, c_void_p, c_void_p, c_char_p, c_int]),
    "swe_host_build_mesh_device": (c_void_p, [c_void_p, c_void_p, c_void_p, c_int, c_char_p,
                                              c_int]),
    "swe_dev_build_mesh": (c_int, [c_int, c_int, c_void_p, c_int, c_void_p, C.POINTER(c_void_p),
                                   c_char_p, c_int]),
    "swe_dev_built_sizes": (c_int, [c_void_p, P_int, P_int, P_int]),
    "swe_dev_built_export": (c_int, [c_void_p] + [c_void_p] * 13),
    "swe_dev_built_free": (None, [c_void_p]),
    "swe_host_mesh_sizes": (None, [c_void_p, P_int, P_int, P_int]),
    "swe_host_mesh_export": (None, [c_void_p] + [c_void_p] * 13),
    "swe_host_mesh_free": (None, [c_void_p]),
    "swe_host_partition": (c_int, [c_void_p, c_int, c_void_p]),
    "swe_host_partition_weighted": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "swe_host_local_mesh": (c_void_p, [c_void_p, c_void_p, c_int, c_char_p, c_int]),
    "swe_host_partition_raw": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "swe_host_rank_mesh": (c_void_p, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_char_p,
                                      c_int]),
    "swe_host_local_sizes": (None, [c_void_p] + [P_int] * 6),
    "swe_host_local_export": (None, [c_void_p] + [c_void_p] * 15),
    "swe_host_local_plan": (None, [c_void_p] + [c_void_p] * 5),
    "swe_host_local_free": (None, [c_void_p]),
    "swe_host_swemesh_read": (c_void_p, [c_char_p, c_int, c_char_p, c_int]),
    "swe_host_swemesh_parse": (c_void_p, [c_char_p, c_ll, c_int, c_char_p, c_int]),
    "swe_host_swemesh_raw": (c_void_p, [c_void_p]),
    "swe_host_swemesh_fields": (None, [c_void_p, c_void_p, c_void_p]),
    "swe_host_swemesh_free": (None, [c_void_p]),
    "swe_host_swemesh_write": (c_int, [c_char_p, c_void_p, c_void_p, c_void_p, c_int, c_char_p,
                                       c_int]),
    # the C++ drop-in engine behind reference-shaped entry points
    "swe_api_compute_fluxes": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_int, c_char_p, c_int]),
    "swe_api_total_mass": (c_int, [c_void_p, c_void_p, c_void_p, c_int, P_double, c_char_p, c_int]),
    "swe_api_advance": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, P_double, P_long,
                                c_double, c_long, c_int, c_int, c_void_p, c_void_p, P_double,
                                P_long, P_long, c_char_p, c_int]),
    "swe_api_run": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, P_double, P_long,
                            c_double, c_double, c_long, c_int, c_void_p, c_long, P_long, c_void_p,
                            c_void_p, c_long, P_long, c_void_p, c_char_p, c_int]),
}

# every symbol include/swe_dev.h and include/swe_host.h declare
DECLARED = [n for n in _SIGS if n.startswith(("swe_dev_", "swe_host_"))]

_lib = None


def load() -> C.CDLL:
    """Load libswe_b200.so; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -m paper_1807_00672_b200.build); there is no CPU fallback")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def ptr(a):
    """ctypes void* of a numpy array (or None)."""
    return None if a is None else a.ctypes.data_as(c_void_p)


def dptr(a):
    return a.ctypes.data_as(P_double)


def iptr(a):
    return a.ctypes.data_as(P_int)
