"""TEST INFRASTRUCTURE: ctypes binding of liboracle.so (C restatement of the
reference numba kernels, kernels.py).  See oracle/__init__.py."""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SO = HERE / "liboracle.so"

_P = ctypes.c_void_p
_I = ctypes.c_int64
_D = ctypes.c_double


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def _load():
    if not SO.exists():
        build()
    h = ctypes.CDLL(str(SO))
    sig = {
        "oracle_apply_scaling_3d": (None, [_I, _P, _P, _P, _P, _P]),
        "oracle_apply_nodal_3d": (None, [_I, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P]),
        "oracle_apply_const_3d": (None, [_I, _P, _P, _P, _D, _P]),
        "oracle_apply_stored_3d": (None, [_I, _P, _P, _P, _P]),
        "oracle_gs_scaling_3d": (ctypes.c_int, [_I, _P, _P, _P, _P, _P, _D]),
        "oracle_gs_nodal_3d": (ctypes.c_int, [_I, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _D]),
        "oracle_csr_gs": (ctypes.c_int, [_I, _P, _P, _P, _P, _P, _P, _P, _D]),
        "oracle_apply_scaling_3d_batch": (None, [_I, _P, _I, _P, _P, _P, _P, _I]),
        "oracle_num_threads": (ctypes.c_int, []),
        "oracle_apply_scaling_2d": (None, [_I, _P, _P, _P, _P, _P, _P, _P]),
        "oracle_gs_scaling_2d": (ctypes.c_int, [_I, _P, _P, _P, _P, _P, _P, _P, _D]),
        "oracle_apply_scaling_tensor_3d": (None, [_I, _P, _P, _P, _I, _P, _P]),
        "oracle_apply_nodal_tensor_3d": (ctypes.c_int, [_I, _P, _P, _P, _I, _P, _I, _P, _P,
                                                        _P, _P, _P]),
        "oracle_gs_scaling_tensor_3d": (ctypes.c_int, [_I, _P, _P, _P, _P, _I, _P, _D]),
        "oracle_gs_nodal_tensor_3d": (ctypes.c_int, [_I, _P, _P, _P, _P, _I, _P, _I, _P, _P,
                                                     _P, _P, _D]),
    }
    for name, (res, args) in sig.items():
        f = getattr(h, name)
        f.restype = res
        f.argtypes = args
    return h


_h = None


def lib():
    global _h
    if _h is None:
        _h = _load()
    return _h


def _p(a):
    return a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def nvol_of(n):
    return (n - 1) * (n - 2) * (n - 3) // 6 if n >= 4 else 0


def apply_scaling_3d(n, base, v, kc, sh):
    out = np.empty(nvol_of(n))
    base, v, kc, sh = _c(base, np.int64), _c(v, float), _c(kc, float), _c(sh, float)
    lib().oracle_apply_scaling_3d(n, _p(base), _p(v), _p(kc), _p(sh), _p(out))
    return out


def apply_nodal_3d(n, base, v, kc, sched, sums, fac, tptr, telem):
    out = np.empty(nvol_of(n))
    a = [_c(base, np.int64), _c(v, float), _c(kc, float), _c(sched, np.int64),
         _c(sums, np.int64), _c(fac, float), _c(tptr, np.int64), _c(telem, np.int64)]
    lib().oracle_apply_nodal_3d(n, _p(a[0]), _p(a[1]), _p(a[2]), _p(a[3]), len(a[3]),
                                _p(a[4]), _p(a[5]), _p(a[6]), _p(a[7]), _p(out))
    return out


def apply_const_3d(n, base, v, s, c0):
    out = np.empty(nvol_of(n))
    base, v, s = _c(base, np.int64), _c(v, float), _c(s, float)
    lib().oracle_apply_const_3d(n, _p(base), _p(v), _p(s), float(c0), _p(out))
    return out


def apply_stored_3d(n, base, v, w):
    out = np.empty(nvol_of(n))
    base, v, w = _c(base, np.int64), _c(v, float), _c(w, float)
    lib().oracle_apply_stored_3d(n, _p(base), _p(v), _p(w), _p(out))
    return out


def gs_scaling_3d(n, base, u, fv, kc, sh, omega):
    """In place on u (must be a C-contiguous float64 array)."""
    base, fv, kc, sh = _c(base, np.int64), _c(fv, float), _c(kc, float), _c(sh, float)
    rc = lib().oracle_gs_scaling_3d(n, _p(base), _p(u), _p(fv), _p(kc), _p(sh), float(omega))
    if rc:
        raise ValueError("zero central stencil entry")
    return u


def gs_nodal_3d(n, base, u, fv, kc, sched, sums, fac, tptr, telem, omega):
    a = [_c(base, np.int64), _c(fv, float), _c(kc, float), _c(sched, np.int64),
         _c(sums, np.int64), _c(fac, float), _c(tptr, np.int64), _c(telem, np.int64)]
    rc = lib().oracle_gs_nodal_3d(n, _p(a[0]), _p(u), _p(a[1]), _p(a[2]), _p(a[3]),
                                  len(a[3]), _p(a[4]), _p(a[5]), _p(a[6]), _p(a[7]),
                                  float(omega))
    if rc:
        raise ValueError("zero central stencil entry")
    return u


def apply_scaling_tensor_3d(n, base, v, km, shm):
    """km: (M, L), shm: (M, 14) (kernels.py:192-232)."""
    out = np.empty(nvol_of(n))
    base, v, km, shm = _c(base, np.int64), _c(v, float), _c(km, float), _c(shm, float)
    lib().oracle_apply_scaling_tensor_3d(n, _p(base), _p(v), _p(km), km.shape[0], _p(shm),
                                         _p(out))
    return out


def apply_nodal_tensor_3d(n, base, v, km, sched, sums, fac, tptr, telem):
    """km: (M, L), fac: (M, 72) (kernels.py:235-286)."""
    out = np.empty(nvol_of(n))
    a = [_c(base, np.int64), _c(v, float), _c(km, float), _c(sched, np.int64),
         _c(sums, np.int64), _c(fac, float), _c(tptr, np.int64), _c(telem, np.int64)]
    rc = lib().oracle_apply_nodal_tensor_3d(n, _p(a[0]), _p(a[1]), _p(a[2]), a[2].shape[0],
                                            _p(a[3]), len(a[3]), _p(a[4]), _p(a[5]),
                                            _p(a[6]), _p(a[7]), _p(out))
    if rc:
        raise ValueError("too many tensor components for the oracle")
    return out


def gs_scaling_tensor_3d(n, base, u, fv, km, shm, omega):
    base, fv, km, shm = _c(base, np.int64), _c(fv, float), _c(km, float), _c(shm, float)
    rc = lib().oracle_gs_scaling_tensor_3d(n, _p(base), _p(u), _p(fv), _p(km), km.shape[0],
                                           _p(shm), float(omega))
    if rc:
        raise ValueError("zero central stencil entry")
    return u


def gs_nodal_tensor_3d(n, base, u, fv, km, sched, sums, fac, tptr, telem, omega):
    a = [_c(base, np.int64), _c(fv, float), _c(km, float), _c(sched, np.int64),
         _c(sums, np.int64), _c(fac, float), _c(tptr, np.int64), _c(telem, np.int64)]
    rc = lib().oracle_gs_nodal_tensor_3d(n, _p(a[0]), _p(u), _p(a[1]), _p(a[2]),
                                         a[2].shape[0], _p(a[3]), len(a[3]), _p(a[4]),
                                         _p(a[5]), _p(a[6]), _p(a[7]), float(omega))
    if rc:
        raise ValueError("zero central stencil entry")
    return u


def csr_gs(rows, indptr, indices, data, diag, u, f, omega):
    a = [_c(rows, np.int64), _c(indptr, np.int32), _c(indices, np.int32),
         _c(data, float), _c(diag, float), _c(f, float)]
    rc = lib().oracle_csr_gs(len(a[0]), _p(a[0]), _p(a[1]), _p(a[2]), _p(a[3]),
                             _p(a[4]), _p(u), _p(a[5]), float(omega))
    if rc:
        raise ValueError("zero central stencil entry")
    return u


def apply_scaling_2d(n, base, v, kc, kg, g, sh):
    """kernels.apply_scaling_2d with the MA2 gray-edge selector g (6 flags)."""
    a = [_c(base, np.int64), _c(v, np.float64), _c(kc, np.float64), _c(kg, np.float64),
         _c(np.asarray(g) != 0, np.uint8), _c(sh, np.float64)]
    out = np.empty((n - 1) * (n - 2) // 2 if n >= 3 else 0)
    lib().oracle_apply_scaling_2d(n, *(_p(x) for x in a), _p(out))
    return out


def gs_scaling_2d(n, base, u, fv, kc, kg, g, sh, omega):
    """kernels.gs_scaling_2d, in place on u (float64, contiguous)."""
    a = [_c(fv, np.float64), _c(kc, np.float64), _c(kg, np.float64),
         _c(np.asarray(g) != 0, np.uint8), _c(sh, np.float64)]
    rc = lib().oracle_gs_scaling_2d(n, _p(_c(base, np.int64)), _p(u), *(_p(x) for x in a),
                                    omega)
    if rc:
        raise ValueError("zero central stencil entry")
    return u


def apply_scaling_3d_batch(n, base, v, kc, sh, nthreads=0):
    """v, kc: (ntets, L); sh: (ntets, 14) -> (ntets, nvol), one POSIX thread
    per core pulling macro elements (nthreads=0: all online cores)."""
    ntets = v.shape[0]
    out = np.empty((ntets, nvol_of(n)))
    base, v, kc, sh = _c(base, np.int64), _c(v, float), _c(kc, float), _c(sh, float)
    lib().oracle_apply_scaling_3d_batch(n, _p(base), ntets, _p(v), _p(kc), _p(sh), _p(out),
                                        int(nthreads))
    return out


def num_threads():
    return int(lib().oracle_num_threads())
