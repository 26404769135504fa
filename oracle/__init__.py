"""fp64 CPU oracle for the separable dexel dilation / erosion / shell.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package.  The product
path (paper_1804_08968_b200/) never imports it; the two share no code.

Implementations (see dexel_oracle.c for the passage each one follows):
  method="brute"  O1 -- the definition, Eq. 1 PAPER.md:235-238 on the lattice,
                   the paper's own brute-force baseline PAPER.md:592-594.
  method="sep"    O2 -- the paper's two passes in
                   plain gather form: closest-parent extrusion, then power
                   dilation of the weighted pieces.
  erode  = U \\ D_r(U \\ S)
  shell  = D_rout(S) n D_rin(U \\ S)    PAPER.md:58-61 (dilation minus erosion)
  pass1  = the intermediate S_Mid as (lo, hi, kappa) pieces

Pins (tests/test_oracle_pins.py) tie both implementations to closed forms,
a brute-force distance test, the SPEC's hand-derived examples and
invariants; see DESIGN.md "Oracle and pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

OP_DILATE, OP_ERODE, OP_SHELL, OP_PASS1 = 0, 1, 2, 3


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "dexel_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm", "-lpthread"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        u64pp = ctypes.POINTER(ctypes.POINTER(ctypes.c_uint64))
        f64pp = ctypes.POINTER(ctypes.POINTER(ctypes.c_double))
        u8pp = ctypes.POINTER(ctypes.POINTER(ctypes.c_uint8))
        lib.oracle_run.restype = ctypes.c_int
        lib.oracle_run.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
            u64pp, f64pp, u8pp, ctypes.POINTER(ctypes.c_uint64)]
        lib.oracle_free.restype = None
        lib.oracle_free.argtypes = [ctypes.c_void_p]
        _lib = lib
    return _lib


class Result:
    """Per-column fp64 intervals in CSR: off uint64[ncols+1], z float64[2n] (local frame)."""

    def __init__(self, off, z, k=None, cols=None):
        self.off, self.z, self.k, self.cols = off, z, k, cols

    def column(self, t: int) -> np.ndarray:
        a, b = int(self.off[t]), int(self.off[t + 1])
        return self.z[2 * a:2 * b].reshape(-1, 2)

    def kappa(self, t: int) -> np.ndarray:
        a, b = int(self.off[t]), int(self.off[t + 1])
        return self.k[a:b]

    def columns(self):
        return [self.column(t) for t in range(len(self.off) - 1)]


def _run(op, method, grid, r, r2, complement, cols, nthreads):
    lib = _load()
    off = np.ascontiguousarray(grid.off, dtype=np.uint64)
    ep = np.ascontiguousarray(grid.ep, dtype=np.float32)
    if ep.size == 0:
        ep = np.zeros(2, np.float32)
    c = None if cols is None else np.ascontiguousarray(cols, dtype=np.int64)
    ncols = 0 if c is None else len(c)
    if c is not None and ncols == 0:
        return Result(np.zeros(1, np.uint64), np.zeros(0), np.zeros(0, np.uint8), c)
    po = ctypes.POINTER(ctypes.c_uint64)()
    pz = ctypes.POINTER(ctypes.c_double)()
    pk = ctypes.POINTER(ctypes.c_uint8)()
    n = ctypes.c_uint64(0)
    rc = lib.oracle_run(op, method, grid.nx, grid.ny, off.ctypes.data, ep.ctypes.data,
                        float(grid.z_lo), float(grid.z_hi), float(r), float(r2), float(grid.spacing),
                        int(complement), None if c is None else c.ctypes.data, ncols,
                        int(nthreads or os.cpu_count() or 1),
                        ctypes.byref(po), ctypes.byref(pz), ctypes.byref(pk), ctypes.byref(n))
    if rc != 0:
        raise ValueError("oracle: invalid arguments (r < 0, spacing <= 0 or R > 255)")
    m = grid.ncol if c is None else ncols
    o = np.ctypeslib.as_array(po, shape=(m + 1,)).copy()
    z = np.ctypeslib.as_array(pz, shape=(2 * n.value + 2,))[:2 * n.value].copy()
    k = None
    if op == OP_PASS1:
        k = np.ctypeslib.as_array(pk, shape=(n.value + 1,))[:n.value].copy()
        lib.oracle_free(ctypes.cast(pk, ctypes.c_void_p))
    lib.oracle_free(ctypes.cast(po, ctypes.c_void_p))
    lib.oracle_free(ctypes.cast(pz, ctypes.c_void_p))
    return Result(o, z, k, c)


_METHOD = {"brute": 0, "sep": 1}


def dilate(grid, r, method="sep", complement=False, cols=None, nthreads=None) -> Result:
    """D_r(S) (or D_r(U\\S) with complement=True), clipped to U, per output column."""
    return _run(OP_DILATE, _METHOD[method], grid, r, r, complement, cols, nthreads)


def erode(grid, r, method="sep", cols=None, nthreads=None) -> Result:
    """E_r(S) = U \\ D_r(U \\ S)."""
    return _run(OP_ERODE, _METHOD[method], grid, r, r, 0, cols, nthreads)


def shell(grid, r_out, r_in, method="sep", cols=None, nthreads=None) -> Result:
    """D_rout(S) \\ E_rin(S) = D_rout(S) n D_rin(U \\ S)."""
    return _run(OP_SHELL, _METHOD[method], grid, r_out, r_in, 0, cols, nthreads)


def pass1(grid, r, complement=False, cols=None, nthreads=None) -> Result:
    """S_Mid pieces (lo, hi, kappa) of the closest-parent extrusion along x."""
    return _run(OP_PASS1, 1, grid, r, r, complement, cols, nthreads)
