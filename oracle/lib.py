"""ctypes loader for oracle/liborc.so (built from oracle/zpic_oracle.c with plain gcc).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "zpic_oracle.c")
SO = os.path.join(HERE, "liborc.so")

_lib = None
_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int32)


def build(force=False):
    """Compile the oracle (no -ffast-math: expressions are evaluated as written)."""
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        tmp = SO + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fno-fast-math", "-ffp-contract=off",
                               "-o", tmp, SRC, "-lm"])
        os.replace(tmp, SO)
    return SO


def load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(SO)
        lib.orc_interpolate.argtypes = [_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_long, _I, _I, _D, _D, _D, _D]
        lib.orc_interpolate.restype = None
        lib.orc_boris.argtypes = [ctypes.c_long, _D, _D, _D, _D, _D, ctypes.c_double, ctypes.c_double, _D]
        lib.orc_boris.restype = None
        lib.orc_advance_deposit.argtypes = [ctypes.c_long, _I, _I, _D, _D, _D, _D, _D, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_double, ctypes.c_double, _D,
                                            ctypes.c_int, ctypes.c_int]
        lib.orc_advance_deposit.restype = ctypes.c_long
        lib.orc_refresh_guards.argtypes = [_D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.orc_refresh_guards.restype = None
        lib.orc_fold_current.argtypes = [_D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.orc_fold_current.restype = None
        lib.orc_filter_x.argtypes = [_D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, _D]
        lib.orc_filter_x.restype = None
        lib.orc_yee_advance.argtypes = [_D, _D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int, ctypes.c_int, _D]
        lib.orc_yee_advance.restype = None
        lib.orc_field_energy.argtypes = [_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double]
        lib.orc_field_energy.restype = ctypes.c_double
        _lib = lib
    return _lib


def dp(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def ip(a):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_I)


# ---- thin per-stage wrappers (used by sim.py and by the pin tests) ----------------------

def grid(nx, ny):
    """A zeroed guard-extended 3-component grid, shape (3, ny+3, nx+3); interior (i,j) at [.., j+1, i+1]."""
    return np.zeros((3, ny + 3, nx + 3), dtype=np.float64)


def interpolate(E, B, ix, iy, x, y):
    lib = load()
    ny, nx = E.shape[1] - 3, E.shape[2] - 3
    n = len(ix)
    Ep = np.zeros((n, 3)); Bp = np.zeros((n, 3))
    lib.orc_interpolate(dp(E), dp(B), nx, ny, n, ip(ix), ip(iy), dp(x), dp(y), dp(Ep), dp(Bp))
    return Ep, Bp


def boris(ux, uy, uz, Ep, Bp, m_q, dt):
    """In place on ux, uy, uz; returns sum |u-|^2/(1+g-)."""
    lib = load()
    ke = np.zeros(1)
    lib.orc_boris(len(ux), dp(ux), dp(uy), dp(uz), dp(np.ascontiguousarray(Ep)), dp(np.ascontiguousarray(Bp)),
                  m_q, dt, dp(ke))
    return float(ke[0])


def advance_deposit(ix, iy, x, y, ux, uy, uz, q, dt, dx, dy, J):
    """In place on ix, iy, x, y and J; returns the count of >= 1 cell moves."""
    lib = load()
    ny, nx = J.shape[1] - 3, J.shape[2] - 3
    return lib.orc_advance_deposit(len(ix), ip(ix), ip(iy), dp(x), dp(y), dp(ux), dp(uy), dp(uz), q, dt, dx, dy,
                                   dp(J), nx, ny)


def fold_current(J, bcx, bcy):
    ny, nx = J.shape[1] - 3, J.shape[2] - 3
    load().orc_fold_current(dp(J), nx, ny, bcx, bcy)


def refresh_guards(F, bcx, bcy, is_E):
    ny, nx = F.shape[1] - 3, F.shape[2] - 3
    load().orc_refresh_guards(dp(F), nx, ny, bcx, bcy, int(is_E))


def filter_x(J, bcx, bcy, n_pass, compensated):
    ny, nx = J.shape[1] - 3, J.shape[2] - 3
    row = np.zeros(nx + 2)
    load().orc_filter_x(dp(J), nx, ny, bcx, bcy, n_pass, int(compensated), dp(row))


def yee_advance(E, B, J, dt, dx, dy, bcx, bcy):
    ny, nx = E.shape[1] - 3, E.shape[2] - 3
    save = np.zeros(16 * (max(nx, ny) + 3))
    load().orc_yee_advance(dp(E), dp(B), dp(J), nx, ny, dt, dx, dy, bcx, bcy, dp(save))


def field_energy(E, B, dx, dy):
    ny, nx = E.shape[1] - 3, E.shape[2] - 3
    return load().orc_field_energy(dp(E), dp(B), nx, ny, dx, dy)
