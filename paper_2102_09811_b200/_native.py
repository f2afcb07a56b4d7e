"""ctypes binding of the sm_100a library ``lib/libheatbem_b200.so``.

The structures mirror include/heatbem_b200.h field for field.  There is no
CPU fallback: if the library or a CUDA device is missing, every compute
entry point raises :class:`NativeUnavailable`.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HB_LIB_PATH") or os.path.join(_HERE, "lib", "libheatbem_b200.so")

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_INT = ctypes.c_int


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a CUDA device) is not available."""


class HBError(RuntimeError):
    """A C-ABI call returned an error code."""

    def __init__(self, fn: str, code: int, message: str):
        super().__init__(f"{fn} failed ({code}): {message}")
        self.code = code


class MeshDesc(ctypes.Structure):
    _fields_ = [
        ("E_x", _I64), ("N_x", _I64),
        ("tri_nodes_dev", _P), ("verts_tri_dev", _P), ("normals_dev", _P),
        ("centroids_dev", _P), ("diameters_dev", _P), ("areas_dev", _P),
        ("reg_hats_dev", _P), ("reg_w_dev", _P), ("reg_pts_dev", _P), ("n_reg", _I64),
        ("near_hats_dev", _P), ("near_w_dev", _P), ("near_pts_dev", _P), ("n_near", _I64),
        ("tn_indptr_dev", _P), ("tn_idx_dev", _P), ("tn_case_dev", _P),
        ("tn_permt_dev", _P), ("tn_perms_dev", _P),
        ("duf_off_dev", _P), ("duf_t_dev", _P), ("duf_s_dev", _P), ("duf_w_dev", _P),
        ("sing_pos_dev", _P), ("sing_rowptr_dev", _P), ("sing_max_per_row", _I64),
        ("sing_row_dev", _P),
        ("star_indptr_dev", _P), ("star_elem_dev", _P), ("star_local_dev", _P),
        ("star_max", _I64),
        ("curl_tile_eptr_dev", _P), ("curl_tile_elem_dev", _P), ("curl_star_pos_dev", _P),
        ("curl_tile_emax", _I64), ("curl_tile_smax", _I64),
    ]


class AssemblyStats(ctypes.Structure):
    _fields_ = [("pair_ms", _D), ("finalize_ms", _D), ("pair_launches", _I64), ("launches", _I64)]


class AssemblyDesc(ctypes.Structure):
    _fields_ = [
        ("op", _INT), ("test_p1", _INT), ("trial_p1", _INT), ("symmetric", _INT),
        ("E_t", _I64), ("step", _D), ("alpha", _D), ("d_eps", _D), ("r_eps", _D),
        ("d_begin", _I64), ("d_end", _I64),
        ("blocks_dev", _P), ("workspace_dev", _P), ("workspace_bytes", ctypes.c_size_t),
        ("stats", ctypes.POINTER(AssemblyStats)),
        ("row_begin", _I64), ("row_end", _I64), ("block_ptrs_dev", _P),
        ("n_row_shards", _I64), ("row_shard_bounds_dev", _P), ("row_shard_ptrs_dev", _P),
    ]


class HeatDatum(ctypes.Structure):
    _fields_ = [("kind", _INT), ("src", _D * 3), ("alpha", _D), ("time_shift", _D)]


class DataDesc(ctypes.Structure):
    _fields_ = [
        ("E_x", _I64), ("N_x", _I64), ("nq", _I64),
        ("qpts_dev", _P), ("qw_dev", _P), ("hats_dev", _P), ("areas_dev", _P), ("normals_dev", _P),
        ("tri_nodes_dev", _P), ("star_indptr_dev", _P), ("star_elem_dev", _P), ("star_local_dev", _P),
        ("n_tq", _I64), ("tq", _D * 8), ("tw", _D * 8),
    ]


# every symbol include/heatbem_b200.h declares (checked by tests/test_capi.py)
EXPORTED = (
    "hb_version", "hb_last_error", "hb_assemble", "hb_assemble_min_workspace",
    "hb_assemble_full_workspace", "hb_curl_combine", "hb_potential",
    "hb_toeplitz_apply", "hb_forward_subst_step", "hb_fp64_probe", "hb_pair_classes",
    "hb_toeplitz_apply_range", "hb_curl_workspace", "hb_ipc_export", "hb_ipc_import", "hb_ipc_close",
    "hb_forward_solve", "hb_forward_solve_workspace", "hb_forward_solve_ws", "hb_forward_history_far", "hb_forward_history_near", "hb_forward_history", "hb_inv_apply", "hb_represent_grid",
    "hb_project_workspace", "hb_project_data", "hb_p1_mass_solve", "hb_error_sigma", "hb_copy_row_slab_d2h",
    "hb_represent_grid_elem", "hb_toeplitz_apply_workspace", "hb_toeplitz_apply_ws",
    "hb_assemble_vd", "hb_assemble_vd_min_workspace", "hb_assemble_vd_full_workspace", "hb_curl_combine_parts",
)

_lib = None


def load():
    """Load the library (no GPU needed).  Raises NativeUnavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or ./build_native.sh (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.hb_version.restype = _INT
    L.hb_last_error.restype = ctypes.c_char_p
    L.hb_assemble.argtypes = [ctypes.POINTER(MeshDesc), ctypes.POINTER(AssemblyDesc), _P]
    L.hb_assemble.restype = _INT
    L.hb_assemble_vd.argtypes = [ctypes.POINTER(MeshDesc), ctypes.POINTER(AssemblyDesc), _P, _P, _P]
    L.hb_assemble_vd.restype = _INT
    for fn in ("hb_assemble_min_workspace", "hb_assemble_full_workspace", "hb_assemble_vd_min_workspace",
               "hb_assemble_vd_full_workspace"):
        getattr(L, fn).argtypes = [ctypes.POINTER(MeshDesc), ctypes.POINTER(AssemblyDesc)]
        getattr(L, fn).restype = ctypes.c_size_t
    L.hb_curl_combine.argtypes = [ctypes.POINTER(MeshDesc), _I64, _D, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]
    L.hb_curl_workspace.argtypes = [ctypes.POINTER(MeshDesc), _I64]
    L.hb_curl_workspace.restype = ctypes.c_size_t
    L.hb_curl_combine.restype = _INT
    L.hb_curl_combine_parts.argtypes = [ctypes.POINTER(MeshDesc), _I64, _D, _P, _P, _I64, _P, _I64, _P, _P]
    L.hb_curl_combine_parts.restype = _INT
    L.hb_potential.argtypes = [_INT, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _I64,
                               _P, _P, _P, _P, _P, _D, _D, _D, _D, _P, _P]
    L.hb_potential.restype = _INT
    L.hb_toeplitz_apply.argtypes = [_I64, _I64, _I64, _P, _INT, _INT, _I64, _P, _P, _P]
    L.hb_toeplitz_apply.restype = _INT
    L.hb_toeplitz_apply_workspace.argtypes = [_I64, _I64, _I64, _INT, _INT, _I64]
    L.hb_toeplitz_apply_workspace.restype = ctypes.c_size_t
    L.hb_toeplitz_apply_ws.argtypes = [_I64, _I64, _I64, _P, _INT, _INT, _I64, _P, _P, _P, ctypes.c_size_t, _P]
    L.hb_toeplitz_apply_ws.restype = _INT
    L.hb_toeplitz_apply_range.argtypes = [_I64, _I64, _I64, _I64, _P, _INT, _I64, _P, _P, _P]
    L.hb_toeplitz_apply_range.restype = _INT
    L.hb_forward_subst_step.argtypes = [_I64, _I64, _I64, _P, _INT, _I64, _P, _P, _P]
    L.hb_forward_subst_step.restype = _INT
    L.hb_pair_classes.argtypes = [ctypes.POINTER(MeshDesc), _I64, _I64, _P, _P]
    L.hb_pair_classes.restype = _INT
    L.hb_fp64_probe.argtypes = [_I64, _I64, _P, _P]
    L.hb_ipc_export.argtypes = [_P, _P, ctypes.POINTER(_I64)]
    L.hb_ipc_import.argtypes = [_P, _I64, ctypes.POINTER(_P)]
    L.hb_ipc_close.argtypes = [_P, _I64]
    L.hb_forward_solve.argtypes = [_I64, _I64, _P, _INT, _INT, _I64, _P, _P, _P, _P, _P]
    L.hb_forward_solve.restype = _INT
    L.hb_forward_solve_workspace.argtypes = [_I64]
    L.hb_forward_solve_workspace.restype = ctypes.c_size_t
    L.hb_forward_solve_ws.argtypes = [_I64, _I64, _P, _INT, _INT, _I64, _P, _P, _P, _P, ctypes.c_size_t, _P]
    L.hb_forward_solve_ws.restype = _INT
    L.hb_forward_history_far.argtypes = [_I64, _I64, _I64, _P, _I64, _I64, _P, _P, _P]
    L.hb_forward_history_far.restype = _INT
    L.hb_forward_history_near.argtypes = [_I64, _I64, _I64, _P, _I64, _I64, _P, _P, _P, _P]
    L.hb_forward_history_near.restype = _INT
    L.hb_fp64_probe.restype = _INT
    L.hb_forward_history.argtypes = [_I64, _I64, _I64, _P, _I64, _P, _P, _P]
    L.hb_forward_history.restype = _INT
    L.hb_inv_apply.argtypes = [_I64, _P, _P, _P, _P, _P]
    L.hb_inv_apply.restype = _INT
    L.hb_represent_grid.argtypes = [_I64, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _P, _P, _P, _P, _P,
                                    _D, _D, _D, _D, _P, _P]
    L.hb_represent_grid.restype = _INT
    L.hb_project_workspace.argtypes = [ctypes.POINTER(DataDesc), _INT, _I64]
    L.hb_project_workspace.restype = ctypes.c_size_t
    L.hb_project_data.argtypes = [ctypes.POINTER(DataDesc), ctypes.POINTER(HeatDatum), _INT, _I64, _D, _P, _P,
                                  ctypes.c_size_t, _D, _I64, ctypes.POINTER(_I64), _P]
    L.hb_project_data.restype = _INT
    L.hb_p1_mass_solve.argtypes = [ctypes.POINTER(DataDesc), _I64, _P, _P, _P, ctypes.c_size_t, _D, _I64, _P]
    L.hb_p1_mass_solve.restype = _INT
    L.hb_error_sigma.argtypes = [ctypes.POINTER(DataDesc), ctypes.POINTER(HeatDatum), _I64, _D, _P, _INT, _P, _P,
                                 ctypes.c_size_t, _P]
    L.hb_error_sigma.restype = _INT
    L.hb_copy_row_slab_d2h.argtypes = [_P, _P, _I64, _I64, _I64, _I64, _I64, _P]
    L.hb_copy_row_slab_d2h.restype = _INT
    L.hb_represent_grid_elem.argtypes = [_I64, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P,
                                         _D, _D, _D, _D, _D, _P, _P]
    L.hb_represent_grid_elem.restype = _INT
    _lib = L
    return L


def call(fn: str, *args) -> int:
    L = load()
    rc = getattr(L, fn)(*args)
    if rc != 0:
        msg = L.hb_last_error()
        raise HBError(fn, rc, msg.decode() if msg else "")
    return rc


def require_cuda():
    """Device + library check for compute entry points (no fallback)."""
    import torch

    load()
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the heat-BEM operators run only on the GPU")


def stream_handle(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)
