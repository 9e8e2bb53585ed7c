"""ctypes binding of libhhg_b200.so (the C ABI declared in include/hhg_b200.h).

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a).
There is no fallback: if the shared object is missing, or no CUDA device is
present when a device operation is requested, the call raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

__all__ = ["lib", "LIB_PATH", "HhgGrid", "HhgSurface", "HhgSurfaceGS", "HhgFace", "HhgTransfer",
           "check",
           "HhgError",
           "VAR", "FLAG_RESIDUAL", "FLAG_FAST", "FLAG_MIRROR", "EXPORTS"]

# HHG_LIB selects another build of the library (e.g. the bounds-checked
# debug build of tools/bounds_check.sh); default: the in-tree product build
LIB_PATH = Path(os.environ.get("HHG_LIB") or
                Path(__file__).resolve().parent / "libhhg_b200.so").resolve()

HHG_OK, HHG_ERR_ARG, HHG_ERR_CUDA, HHG_ERR_ZERO_DIAG, HHG_ERR_TABLE = 0, -1, -2, -3, -4
VAR = {"scaling": 0, "nodal": 1, "const": 2, "stored": 3}
FLAG_RESIDUAL, FLAG_FAST, FLAG_MIRROR = 1, 2, 4

c_i64p = ctypes.POINTER(ctypes.c_int64)
vp = ctypes.c_void_p


class HhgError(RuntimeError):
    pass


class HhgGrid(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("ntets", ctypes.c_int32),
                ("lat_size", ctypes.c_int64), ("nvol", ctypes.c_int64),
                ("shell_size", ctypes.c_int64), ("n_nodes", ctypes.c_int64),
                ("vol_start", vp), ("srow", vp), ("shell_gid", vp),
                ("ghost", vp), ("kc", vp), ("tiles", vp),
                ("ntiles", ctypes.c_int32), ("nmtiles", ctypes.c_int32), ("mtiles", vp)]


class HhgSurface(ctypes.Structure):
    _fields_ = [("nrows", ctypes.c_int64), ("rows", vp), ("row_nodal", vp),
                ("inc_ptr", vp), ("inc_tet", vp), ("inc_code", vp),
                ("inc_cls", vp), ("psh", vp), ("pfac", vp),
                ("ndir", ctypes.c_int64), ("dir_ids", vp),
                ("ninc", ctypes.c_int64), ("p_tet", vp), ("p_code", vp),
                ("p_cls", vp), ("p_nodal", vp), ("row_inc", vp), ("partial", vp),
                ("nfaces", ctypes.c_int64), ("faces", vp), ("nface_tiles", ctypes.c_int64),
                ("face_tiles", vp), ("nsub", ctypes.c_int64), ("sub_rows", vp),
                ("face_k", vp), ("face_g", vp), ("face_sq", ctypes.c_int32),
                ("pad_", ctypes.c_int32)]


class HhgTransfer(ctypes.Structure):
    _fields_ = [("nf", ctypes.c_int32), ("nc", ctypes.c_int32),
                ("ntets", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("f_vol_start", vp), ("c_vol_start", vp), ("c_shell_gid", vp),
                ("c_shell_size", ctypes.c_int64),
                ("p_nrows", ctypes.c_int64), ("p_rows", vp), ("p_ptr", vp), ("p_col", vp),
                ("p_val", vp),
                ("r_nrows", ctypes.c_int64), ("r_rows", vp), ("r_ptr", vp), ("r_col", vp),
                ("r_val", vp),
                ("ndir", ctypes.c_int64), ("c_dir_ids", vp)]


class HhgFace(ctypes.Structure):
    _fields_ = [("tet", ctypes.c_int32 * 2), ("cls", ctypes.c_int32 * 2),
                ("A", (ctypes.c_int32 * 6) * 2), ("c", (ctypes.c_int32 * 3) * 2),
                ("nb", (ctypes.c_int32 * 3) * 2),
                ("dl", (ctypes.c_int8 * 14) * 2), ("da", (ctypes.c_int8 * 14) * 2),
                ("db", (ctypes.c_int8 * 14) * 2),
                ("nodal", ctypes.c_int32),
                ("fs", ctypes.c_int64), ("rbase", ctypes.c_int64)]


class HhgSurfaceGS(ctypes.Structure):
    _fields_ = [("level_rows", vp), ("level_ptr", vp), ("nlev", ctypes.c_int64),
                ("ent_ptr", vp), ("ent_col", vp), ("ent_val", vp), ("row_diag", vp),
                ("nslots", ctypes.c_int64), ("slot_gid", vp), ("slot_cnt", vp),
                ("slot_diag", vp), ("slot_col", vp), ("slot_val", vp), ("slot_dyn", vp),
                ("sweep_bar", vp)]


SURF_SLOT_PF = 24   # HHG_SURF_SLOT_PF


# name -> (restype, argtypes); every symbol of include/hhg_b200.h
EXPORTS = {
    "hhg_apply_scaling_3d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp, vp]),
    "hhg_apply_nodal_3d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, c_i64p,
                                          ctypes.c_int64, c_i64p, vp, c_i64p,
                                          c_i64p, vp, vp]),
    "hhg_apply_const_3d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp,
                                          ctypes.c_double, vp, vp]),
    "hhg_apply_stored_3d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp]),
    "hhg_apply_scaling_2d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "hhg_gs_scaling_2d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp,
                                         ctypes.c_double, vp]),
    "hhg_csr_gs": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp,
                                  ctypes.c_double, vp]),
    "hhg_gs_scaling_3d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp,
                                         ctypes.c_double, vp]),
    "hhg_gs_nodal_3d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, c_i64p,
                                       ctypes.c_int64, c_i64p, vp, c_i64p, c_i64p,
                                       ctypes.c_double, vp]),
    "hhg_dump_stencils": (ctypes.c_int, [ctypes.POINTER(HhgGrid), ctypes.c_int, vp, vp, vp]),
    "hhg_ghost_update": (ctypes.c_int, [ctypes.POINTER(HhgGrid), vp, vp]),
    "hhg_volume_apply": (ctypes.c_int, [ctypes.POINTER(HhgGrid), ctypes.c_int,
                                        ctypes.c_int, vp, vp, vp, vp, vp, vp]),
    "hhg_surface_apply": (ctypes.c_int, [ctypes.POINTER(HhgGrid),
                                         ctypes.POINTER(HhgSurface), ctypes.c_int,
                                         ctypes.c_int, vp, vp, vp, vp]),
    "hhg_smooth_surface_level": (ctypes.c_int, [ctypes.POINTER(HhgGrid),
                                                ctypes.POINTER(HhgSurface), vp,
                                                ctypes.c_int64, ctypes.c_double,
                                                vp, vp, vp]),
    "hhg_smooth_surface_prepare": (ctypes.c_int, [ctypes.POINTER(HhgGrid),
                                                  ctypes.POINTER(HhgSurface),
                                                  ctypes.POINTER(HhgSurfaceGS), vp]),
    "hhg_surface_apply_csr": (ctypes.c_int, [ctypes.POINTER(HhgGrid),
                                             ctypes.POINTER(HhgSurface),
                                             ctypes.POINTER(HhgSurfaceGS), ctypes.c_int,
                                             vp, vp, vp, vp]),
    "hhg_smooth_surface_slots": (ctypes.c_int, [ctypes.POINTER(HhgGrid),
                                                ctypes.POINTER(HhgSurface),
                                                ctypes.POINTER(HhgSurfaceGS), vp,
                                                ctypes.c_int64, vp]),
    "hhg_smooth_surface_all": (ctypes.c_int, [ctypes.POINTER(HhgGrid),
                                              ctypes.POINTER(HhgSurface),
                                              ctypes.POINTER(HhgSurfaceGS), ctypes.c_double,
                                              vp, vp, vp]),
    "hhg_smooth_volume": (ctypes.c_int, [ctypes.POINTER(HhgGrid), ctypes.c_int, vp,
                                         ctypes.c_double, vp, vp, vp]),
    "hhg_skew_coefficient": (ctypes.c_int, [ctypes.POINTER(HhgGrid), vp, vp]),
    "hhg_smooth_volume_skew": (ctypes.c_int, [ctypes.POINTER(HhgGrid), ctypes.c_int, vp,
                                              ctypes.c_double, vp, vp, vp, vp, vp,
                                              ctypes.c_int, vp]),
    "hhg_apply_scaling_tensor_3d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp,
                                                   ctypes.c_int64, vp, vp, vp]),
    "hhg_apply_nodal_tensor_3d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, ctypes.c_int64,
                                                 c_i64p, ctypes.c_int64, c_i64p, vp, c_i64p,
                                                 c_i64p, vp, vp]),
    "hhg_gs_scaling_tensor_3d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp,
                                                ctypes.c_int64, vp, ctypes.c_double, vp]),
    "hhg_gs_nodal_tensor_3d": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, ctypes.c_int64,
                                              c_i64p, ctypes.c_int64, c_i64p, vp, c_i64p,
                                              c_i64p, ctypes.c_double, vp]),
    "hhg_tensor_volume_apply": (ctypes.c_int, [ctypes.POINTER(HhgGrid), ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int, vp, vp, vp, vp,
                                               vp, vp, vp]),
    "hhg_tensor_smooth_volume": (ctypes.c_int, [ctypes.POINTER(HhgGrid), ctypes.c_int,
                                                ctypes.c_int, vp, vp, ctypes.c_double, vp,
                                                vp, vp, vp]),
    "hhg_tensor_surface_prepare": (ctypes.c_int, [ctypes.POINTER(HhgGrid),
                                                  ctypes.POINTER(HhgSurface),
                                                  ctypes.POINTER(HhgSurfaceGS), ctypes.c_int,
                                                  vp, vp]),
    "hhg_surface_apply_csr_push": (ctypes.c_int, [ctypes.POINTER(HhgGrid),
                                                  ctypes.POINTER(HhgSurface),
                                                  ctypes.POINTER(HhgSurfaceGS), vp, vp, vp,
                                                  vp, vp, ctypes.c_int64, vp]),
    "hhg_p2p_signal": (ctypes.c_int, [vp, vp]),
    "hhg_p2p_pull": (ctypes.c_int, [vp, vp, ctypes.c_int64, vp, vp, ctypes.c_uint64,
                                    ctypes.c_int, vp, vp]),
    "hhg_device_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    "hhg_device_free": (ctypes.c_int, [vp]),
    "hhg_launch_count": (ctypes.c_longlong, []),
    "hhg_ipc_get_handle": (ctypes.c_int, [vp, vp]),
    "hhg_ipc_open_handle": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_void_p)]),
    "hhg_ipc_close_handle": (ctypes.c_int, [vp]),
    "hhg_dot": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp]),
    "hhg_axpy_ratio": (ctypes.c_int, [ctypes.c_int64, vp, vp, ctypes.c_double, vp,
                                      vp, vp]),
    "hhg_xpay_ratio": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp]),
    "hhg_cg_update": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                     vp]),
    "hhg_pcg_update": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                      vp]),
    "hhg_dot2": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp, vp]),
    "hhg_dot_masked": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp, vp]),
    "hhg_csr_spmv": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp, vp,
                                    ctypes.c_int, vp]),
    "hhg_prolongate": (ctypes.c_int, [ctypes.POINTER(HhgTransfer), vp, vp, ctypes.c_int, vp]),
    "hhg_restrict": (ctypes.c_int, [ctypes.POINTER(HhgTransfer), vp, vp, vp]),
    "hhg_scatter_zero": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp]),
    "hhg_gather": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp]),
    "hhg_interface_add": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, ctypes.c_int, vp, vp]),
    "hhg_status": (ctypes.c_int, []),
    "hhg_status_reset": (ctypes.c_int, []),
    "hhg_build_info": (ctypes.c_char_p, []),
    "hhg_volume_tile_rows": (ctypes.c_int, []),
    "hhg_volume_tile_cols_mirror": (ctypes.c_int, []),
    "hhg_face_tile": (ctypes.c_int, []),
    "hhg_host_gs_levels": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp]),
    "hhg_host_gs_levels_seeded": (ctypes.c_int, [ctypes.c_int64, vp, vp, vp, vp]),
    "hhg_smooth_surface_rows": (ctypes.c_int, [ctypes.POINTER(HhgGrid),
                                               ctypes.POINTER(HhgSurface),
                                               ctypes.POINTER(HhgSurfaceGS), vp,
                                               ctypes.c_int64, ctypes.c_double, vp, vp, vp]),
    "hhg_smooth_surface_partial": (ctypes.c_int, [ctypes.POINTER(HhgGrid),
                                                  ctypes.POINTER(HhgSurface),
                                                  ctypes.POINTER(HhgSurfaceGS), vp,
                                                  ctypes.c_int64, vp, vp, vp, vp]),
    "hhg_smooth_surface_finish": (ctypes.c_int, [ctypes.POINTER(HhgGrid),
                                                 ctypes.POINTER(HhgSurface),
                                                 ctypes.POINTER(HhgSurfaceGS), vp,
                                                 ctypes.c_int64, vp, vp, ctypes.c_double, vp,
                                                 vp, vp]),
}


def _load():
    if not LIB_PATH.exists():
        raise HhgError(
            f"{LIB_PATH.name} is not built; run `python -c 'import __graft_entry__ as g; "
            "g.build()'` (nvcc sm_100a). There is no CPU fallback.")
    handle = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL | ctypes.RTLD_GLOBAL * 0)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    return handle


class _Lazy:
    _h = None

    def __getattr__(self, name):
        if _Lazy._h is None:
            _Lazy._h = _load()
        return getattr(_Lazy._h, name)


lib = _Lazy()


def check(rc, what=""):
    if rc == HHG_OK:
        return
    if rc == HHG_ERR_ZERO_DIAG:
        raise ValueError("zero central stencil entry")
    if rc == HHG_ERR_TABLE:
        raise ValueError(f"{what}: patch tables differ from the compiled ones")
    raise HhgError(f"{what} failed with code {rc}")
