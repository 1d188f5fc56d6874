"""ctypes binding of ``libhbem_b200.so`` (C ABI declared in include/hbem_b200.h).

There is no fallback: if the shared library is missing the import of any
product module fails with a message telling how to build it.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HBEM_LIB") or os.path.join(_HERE, "libhbem_b200.so")

HBEM_OK = 0
_CODE_TO_EXC = {
    1: errors.ContractViolationError,
    2: errors.CapacityError,
    3: errors.ConfigError,
    4: errors.DeviceError,
    5: errors.HbemError,
    6: errors.KernelError,
    7: errors.MeshError,
    8: errors.MeshParseError,
}

EQUATIONS = {"laplace": 0, "helmholtz": 1}
OPERATORS = {"slp": 0, "dlp": 1, "adlp": 2, "hyps": 3}
PRECISIONS = {"double": 0, "single": 1}
FAMILIES = {"p0": 0, "p1c": 1, "p1d": 2}

c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)
c_int32_p = C.POINTER(C.c_int32)


class CtxDesc(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("equation", C.c_int32),
        ("op", C.c_int32),
        ("precision", C.c_int32),
        ("wavenumber", C.c_double),
        ("test_family", C.c_int32),
        ("trial_family", C.c_int32),
        ("n_vertices", C.c_int64),
        ("vertices", c_double_p),
        ("n_elements", C.c_int64),
        ("elements", c_int64_p),
        ("n_q", C.c_int32),
        ("rule_points", c_double_p),
        ("rule_weights", c_double_p),
        ("qpoints", c_double_p),
        ("normals", c_double_p),
        ("jacobians", c_double_p),
        ("curls", c_double_p),
        ("test_values", c_double_p),
        ("trial_values", c_double_p),
        ("sing_n", C.c_int64 * 3),
        ("sing_points", c_double_p * 3),
        ("sing_weights", c_double_p * 3),
    ]


class HmatDesc(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int64),
        ("n_cols", C.c_int64),
        ("row_perm", c_int64_p),
        ("col_perm", c_int64_p),
        ("n_row_nodes", C.c_int64),
        ("n_col_nodes", C.c_int64),
        ("row_nodes", c_int64_p),
        ("col_nodes", c_int64_p),
        ("n_leaves", C.c_int64),
        ("leaves", c_int64_p),
        ("test_dofmap", c_int64_p),
        ("trial_dofmap", c_int64_p),
        ("epsilon", C.c_double),
        ("k_max", C.c_int64),
        ("rank_capacity", C.c_int32),
        ("pointers_on_device", C.c_int32),
        ("out_u", C.c_void_p),
        ("out_v", C.c_void_p),
        ("out_dense", C.c_void_p),
        ("out_u_cap", C.c_int64),
        ("out_v_cap", C.c_int64),
        ("out_dense_cap", C.c_int64),
    ]


class HmatStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "regular_pairs", "singular_pairs", "aca_converged", "aca_exhausted",
        "aca_fallback_dense", "dense_leaves", "lowrank_leaves", "waves", "row_jobs",
        "col_jobs", "capacity_retries", "u_entries", "v_entries", "dense_entries",
        "launches", "aca_entries")] + [
        (n, C.c_double) for n in ("aca_kernel_ms", "nearfield_kernel_ms", "seconds",
                                  "seconds_setup", "seconds_aca", "seconds_finalize")] + [
        ("int_kernel_ms", C.c_double), ("int_launches", C.c_int64),
        ("sing_table_pairs", C.c_int64)]


# (name, restype, argtypes) of every exported symbol in include/hbem_b200.h
SIGNATURES = [
    ("hbem_abi_version", C.c_int, []),
    ("hbem_last_error", C.c_char_p, []),
    ("hbem_device_count", C.c_int, [c_int32_p]),
    ("hbem_ctx_create", C.c_int, [C.POINTER(CtxDesc), C.POINTER(C.c_void_p)]),
    ("hbem_ctx_destroy", C.c_int, [C.c_void_p]),
    ("hbem_ctx_info", C.c_int, [C.c_void_p, c_int32_p, c_int32_p, c_int32_p, c_int32_p]),
    ("hbem_ctx_geometry", C.c_int, [C.c_void_p, c_double_p, c_double_p, c_double_p]),
    ("hbem_integrate_regular", C.c_int,
     [C.c_void_p, c_int64_p, C.c_int64, C.c_void_p, C.c_void_p]),
    ("hbem_integrate_any", C.c_int,
     [C.c_void_p, c_int64_p, C.c_int64, C.c_void_p, C.c_void_p, c_int64_p]),
    ("hbem_integrate_regular_device", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("hbem_integrate_any_device", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("hbem_cluster_tree", C.c_int, [c_double_p, C.c_int64, C.c_int32, C.POINTER(C.c_void_p)]),
    ("hbem_tree_size", C.c_int, [C.c_void_p, c_int64_p, c_int64_p]),
    ("hbem_tree_copy", C.c_int, [C.c_void_p, c_int64_p, c_int64_p, c_double_p]),
    ("hbem_tree_destroy", C.c_int, [C.c_void_p]),
    ("hbem_block_tree", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_double, C.c_int32, C.POINTER(C.c_void_p)]),
    ("hbem_blocks_size", C.c_int, [C.c_void_p, c_int64_p]),
    ("hbem_blocks_copy", C.c_int, [C.c_void_p, c_int64_p]),
    ("hbem_blocks_destroy", C.c_int, [C.c_void_p]),
    ("hbem_gmsh_read", C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    ("hbem_gmsh_size", C.c_int, [C.c_void_p, c_int64_p, c_int64_p, c_int64_p]),
    ("hbem_gmsh_copy", C.c_int, [C.c_void_p, c_double_p, c_int64_p]),
    ("hbem_gmsh_error_location", C.c_int, [c_int64_p, C.c_char_p, C.c_int32]),
    ("hbem_gmsh_destroy", C.c_int, [C.c_void_p]),
    ("hbem_hmat_assemble", C.c_int,
     [C.c_void_p, C.POINTER(HmatDesc), C.c_void_p, C.POINTER(C.c_void_p)]),
    ("hbem_hmat_execute", C.c_int, [C.c_void_p, C.c_void_p]),
    ("hbem_hmat_stats_get", C.c_int, [C.c_void_p, C.POINTER(HmatStats)]),
    ("hbem_hmat_leaf_residual", C.c_int, [C.c_void_p, c_double_p]),
    ("hbem_hmat_leaf_meta", C.c_int,
     [C.c_void_p, c_int32_p, c_int32_p, c_int32_p, c_int64_p, c_int64_p, c_int64_p]),
    ("hbem_hmat_copy_arenas", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("hbem_hmat_matvec", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("hbem_hmat_matvec_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("hbem_hmat_destroy", C.c_int, [C.c_void_p]),
    ("hbem_host_alloc", C.c_int, [C.c_int64, C.POINTER(C.c_void_p)]),
    ("hbem_host_free", C.c_int, [C.c_void_p]),
    ("hbem_far_field", C.c_int, [C.c_int32, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("hbem_probe_fma", C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_double)]),
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(`make` at the repo root or `python -c 'import __graft_entry__ as g; g.build()'`). "
            "There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    """Raise the reference exception class matching a non-zero status."""
    if status == HBEM_OK:
        return
    msg = lib.hbem_last_error().decode("utf-8", "replace")
    if status == 8:
        # MeshParseError: the message already carries the location suffix;
        # expose line / section as attributes like the reference
        line, sec = C.c_int64(-1), C.create_string_buffer(64)
        lib.hbem_gmsh_error_location(C.byref(line), sec, 64)
        exc = errors.MeshParseError(msg)
        exc.line = int(line.value) if line.value >= 0 else None
        exc.section = sec.value.decode() or None
        raise exc
    raise _CODE_TO_EXC.get(status, errors.HbemError)(msg)


def ptr(a, ctype):
    """ctypes pointer to a contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def vptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def device_count() -> int:
    n = C.c_int32(0)
    check(lib.hbem_device_count(C.byref(n)))
    return int(n.value)
