"""ctypes bindings of the C ABI declared in include/pmg_types.h, pmg_host.h and
pmg_cuda.h.  The CUDA library is loaded on first use and its absence is an
error, never a fallback."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"


class PmgCycleParams(C.Structure):
    _fields_ = [("nu", C.c_int), ("mu", C.c_int), ("tau", C.c_double), ("sigma_scale", C.c_double),
                ("damp_coarse", C.c_int)]


class PmgPieceDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("patch", C.c_int), ("ndofs", C.c_int64), ("dofs", C.POINTER(C.c_int32)),
        ("naxes", C.c_int), ("dims", C.c_int * 3), ("V", C.POINTER(C.c_double) * 3),
        ("diag", C.POINTER(C.c_double)),
        ("chol_dim", C.c_int), ("chol_bw", C.c_int), ("chol_l", C.POINTER(C.c_double)),
        ("scalar", C.c_double),
    ]


class PmgLevelDesc(C.Structure):
    _fields_ = [
        ("elements", C.c_int), ("num_dofs", C.c_int64), ("l2g", C.POINTER(C.c_int32)),
        ("band_format", C.c_int), ("band", C.POINTER(C.c_double)),
        ("csr_row_ptr", C.POINTER(C.POINTER(C.c_int64))), ("csr_cols", C.POINTER(C.POINTER(C.c_int32))),
        ("csr_vals", C.POINTER(C.POINTER(C.c_double))),
        ("ts_fine_dim", C.c_int), ("ts_coarse_dim", C.c_int),
        ("ts_row_start", C.POINTER(C.c_int32)), ("ts_row_len", C.POINTER(C.c_int32)),
        ("ts_row_off", C.POINTER(C.c_int32)), ("ts_vals", C.POINTER(C.c_double)),
        ("num_pieces", C.c_int), ("pieces", C.POINTER(PmgPieceDesc)),
    ]


class PmgPatchGeometry(C.Structure):
    _fields_ = [("degree", C.c_int * 3), ("elements", C.c_int * 3), ("ctrl", C.POINTER(C.c_double))]


PMG_BAND_TENSOR, PMG_BAND_CSR, PMG_BAND_ASSEMBLE, PMG_BAND_KRONECKER = 0, 1, 2, 3
PMGH_DEVICE_ASSEMBLY, PMGH_KRONECKER = 1, 2


class PmgHierarchyDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("degree", C.c_int), ("num_patches", C.c_int), ("num_levels", C.c_int),
        ("params", PmgCycleParams), ("levels", C.POINTER(PmgLevelDesc)),
        ("coarse_n", C.c_int), ("coarse_A", C.POINTER(C.c_double)), ("coarse_L", C.POINTER(C.c_double)),
        ("geometry", C.POINTER(PmgPatchGeometry)),
    ]


class PmgCommDesc(C.Structure):
    _fields_ = [("rank", C.c_int), ("size", C.c_int), ("patch_begin", C.c_int), ("patch_end", C.c_int),
                ("transport", C.c_int), ("nccl_id", C.c_ubyte * 128), ("hub", C.c_void_p)]


PMG_TRANSPORT_NONE, PMG_TRANSPORT_NCCL, PMG_TRANSPORT_HUB = 0, 1, 2


class PmghRankPlanView(C.Structure):
    _fields_ = [("n_iface", C.c_int), ("iface_g", C.POINTER(C.c_int32)), ("rep_off", C.POINTER(C.c_int32)),
                ("rep_slot", C.POINTER(C.c_int32)), ("comb_off", C.POINTER(C.c_int32)),
                ("comb_src", C.POINTER(C.c_int32)), ("n_neighbors", C.c_int), ("nb_rank", C.POINTER(C.c_int32)),
                ("nb_off", C.POINTER(C.c_int32)), ("nb_iface", C.POINTER(C.c_int32))]

PMG_OK = 0
PMG_ERR_CONFIG = 2
PMG_ERR_DIVERGENCE = 3
PMG_ERR_TRANSPORT = 4
PMG_ERR_DOMAIN = 5
PMG_ERR_DEFINITENESS = 6
PMG_ERR_DECOMPOSITION = 7
PMG_ERR_GEOMETRY = 8
PMG_ERR_NONMATCHING = 9
PMG_ERR_CUDA = 10

PIECE_INTERIOR, PIECE_FACE, PIECE_EDGE, PIECE_VERTEX = 0, 1, 2, 3

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_vp = C.c_void_p


def _sig(lib, name, restype, argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = argtypes
    return fn


_host = None
_cuda = None


def host_lib():
    global _host
    if _host is None:
        path = LIB_DIR / "libpmg_host.so"
        if not path.exists():
            raise RuntimeError(f"{path} missing: run `python -m paper_1804_02539_b200.build`")
        lib = C.CDLL(str(path))
        _sig(lib, "pmgh_build", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(PmgCycleParams),
                                          C.c_int, C.c_uint64, C.c_int, C.POINTER(_vp)])
        _sig(lib, "pmgh_build_ex", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.POINTER(PmgCycleParams), C.c_int, C.c_uint64, C.c_int, C.c_int,
                                             C.POINTER(_vp)])
        _sig(lib, "pmgh_free", None, [_vp])
        _sig(lib, "pmgh_last_error", C.c_char_p, [])
        _sig(lib, "pmgh_describe", C.c_int, [_vp, C.POINTER(PmgHierarchyDesc)])
        _sig(lib, "pmgh_rhs", C.c_int, [_vp, C.POINTER(_dp), C.POINTER(C.c_int64)])
        _sig(lib, "pmgh_set_rhs", C.c_int, [_vp, C.c_int, C.c_uint64, C.c_int])
        _sig(lib, "pmgh_seconds", C.c_double, [_vp, C.c_int])
        _sig(lib, "pmgh_stored_entries", C.c_int64, [C.c_int, C.c_int, C.c_int, C.c_int])
        _sig(lib, "pmgh_resolve_rhs_kind", C.c_int, [C.c_char_p, C.c_int, C.c_int])
        _sig(lib, "pmgh_reps", C.c_int, [_vp, C.c_int, C.POINTER(_ip), C.POINTER(_ip), C.POINTER(_ip)])
        _sig(lib, "pmgh_interfaces", C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(_ip)])
        _sig(lib, "pmgh_rank_plan", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(PmghRankPlanView)])
        _sig(lib, "pmgh_gauss_legendre", C.c_int, [C.c_int, _dp, _dp])
        _sig(lib, "pmgh_eval_basis", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                               C.POINTER(C.c_int), _dp])
        _sig(lib, "pmgh_gram", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), _dp])
        _sig(lib, "pmgh_two_scale", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                              C.POINTER(C.c_int), _dp])
        _sig(lib, "pmgh_gen_eig", C.c_int, [C.c_int, _dp, _dp, _dp, _dp])
        _sig(lib, "pmgh_banded_cholesky_solve", C.c_int, [C.c_int, C.c_int, _dp, _dp, _dp])
        _host = lib
    return _host


CUDA_SYMBOLS = [
    "pmg_ctx_create", "pmg_ctx_destroy", "pmg_last_error", "pmg_ctx_info", "pmg_set_stream",
    "pmg_vec_create", "pmg_vec_free", "pmg_vec_upload", "pmg_vec_download", "pmg_vec_zero", "pmg_vec_copy",
    "pmg_vec_lattice_upload", "pmg_vec_lattice_download",
    "pmg_apply_op", "pmg_residual", "pmg_accumulate", "pmg_smooth", "pmg_restrict", "pmg_add_prolonged",
    "pmg_coarse_solve", "pmg_dot", "pmg_axpy", "pmg_xpay",
    "pmg_mg_cycle", "pmg_precondition", "pmg_pcg_solve_device", "pmg_pcg_solve",
    "pmg_kernel_stats", "pmg_synchronize", "pmg_profile", "pmg_profile_read",
    "pmg_band_download", "pmg_assemble_load",
    "pmg_nccl_unique_id", "pmg_hub_create", "pmg_hub_destroy", "pmg_hub_poison", "pmg_comm_bytes",
]


def cuda_lib():
    """The sm_100a library.  Raises if it was not built: there is no CPU path."""
    global _cuda
    if _cuda is None:
        path = LIB_DIR / "libpmg_cuda.so"
        if not path.exists():
            raise RuntimeError(f"{path} missing: the CUDA path is required (no CPU fallback); "
                               "run `python -m paper_1804_02539_b200.build`")
        lib = C.CDLL(str(path))
        for name in CUDA_SYMBOLS:
            getattr(lib, name)  # every declared entry point must exist
        _sig(lib, "pmg_ctx_create", C.c_int, [C.POINTER(PmgHierarchyDesc), C.c_int, C.POINTER(PmgCommDesc),
                                              C.POINTER(_vp)])
        _sig(lib, "pmg_nccl_unique_id", C.c_int, [C.POINTER(C.c_ubyte * 128)])
        _sig(lib, "pmg_hub_create", C.c_int, [C.c_int, C.POINTER(_vp)])
        _sig(lib, "pmg_hub_destroy", None, [_vp])
        _sig(lib, "pmg_hub_poison", C.c_int, [_vp, C.c_char_p])
        _sig(lib, "pmg_comm_bytes", C.c_int, [_vp, C.POINTER(C.c_uint64)])
        _sig(lib, "pmg_ctx_destroy", None, [_vp])
        _sig(lib, "pmg_last_error", C.c_char_p, [_vp])
        _sig(lib, "pmg_ctx_info", C.c_int, [_vp, C.c_int, C.POINTER(C.c_int64)])
        _sig(lib, "pmg_set_stream", C.c_int, [_vp, _vp])
        _sig(lib, "pmg_band_download", C.c_int, [_vp, C.c_int, _dp, C.c_int64])
        _sig(lib, "pmg_assemble_load", C.c_int, [_vp, C.c_int, C.c_uint64, _vp])
        _sig(lib, "pmg_vec_create", C.c_int, [_vp, C.c_int, C.POINTER(_vp)])
        _sig(lib, "pmg_vec_free", None, [_vp])
        _sig(lib, "pmg_vec_upload", C.c_int, [_vp, _vp, C.c_int, _dp, C.c_int64])
        _sig(lib, "pmg_vec_download", C.c_int, [_vp, _vp, C.c_int, _dp, C.c_int64])
        _sig(lib, "pmg_vec_lattice_upload", C.c_int, [_vp, _vp, _dp, C.c_int64])
        _sig(lib, "pmg_vec_lattice_download", C.c_int, [_vp, _vp, _dp, C.c_int64])
        _sig(lib, "pmg_vec_zero", C.c_int, [_vp, _vp])
        _sig(lib, "pmg_vec_copy", C.c_int, [_vp, _vp, _vp])
        _sig(lib, "pmg_apply_op", C.c_int, [_vp, C.c_int, _vp, _vp])
        _sig(lib, "pmg_residual", C.c_int, [_vp, C.c_int, _vp, _vp, _vp])
        _sig(lib, "pmg_accumulate", C.c_int, [_vp, C.c_int, _vp, _vp])
        _sig(lib, "pmg_smooth", C.c_int, [_vp, C.c_int, _vp, _vp])
        _sig(lib, "pmg_restrict", C.c_int, [_vp, C.c_int, _vp, _vp])
        _sig(lib, "pmg_add_prolonged", C.c_int, [_vp, C.c_int, _vp, C.c_double, _vp])
        _sig(lib, "pmg_coarse_solve", C.c_int, [_vp, _vp, _vp])
        _sig(lib, "pmg_dot", C.c_int, [_vp, C.c_int, _vp, _vp, _dp])
        _sig(lib, "pmg_axpy", C.c_int, [_vp, C.c_double, _vp, _vp])
        _sig(lib, "pmg_xpay", C.c_int, [_vp, _vp, C.c_double, _vp])
        _sig(lib, "pmg_mg_cycle", C.c_int, [_vp, C.c_int, _vp, _vp])
        _sig(lib, "pmg_precondition", C.c_int, [_vp, _vp, _vp])
        _sig(lib, "pmg_pcg_solve_device", C.c_int, [_vp, _vp, C.c_double, C.c_int, _vp, _dp, C.POINTER(C.c_int)])
        _sig(lib, "pmg_pcg_solve", C.c_int, [_vp, _dp, C.c_int64, C.c_double, C.c_int, _dp, _dp,
                                             C.POINTER(C.c_int)])
        _sig(lib, "pmg_kernel_stats", C.c_int, [_vp, C.c_int, C.POINTER(C.c_int64), _dp])
        _sig(lib, "pmg_synchronize", C.c_int, [_vp])
        _sig(lib, "pmg_profile", C.c_int, [_vp, C.c_int])
        _sig(lib, "pmg_profile_read", C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(C.c_int64), _dp, _dp])
        _cuda = lib
    return _cuda
