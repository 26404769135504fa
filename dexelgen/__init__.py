"""Seeded synthetic dexel inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no dilation, erosion, pass 1
or pass 2).  It rasterises analytic solids onto the dexel lattice (sphere
chords, boxes, a noisy gyroid) and does the per-column CSG that defines the
input solid.  The recipe for each of BASELINE.json's five configs is written
out in DESIGN.md ("Input recipe") and SURVEY.md 8(d):

  C1  64^2,   z in [0,64]:   sphere R=20 @ (32,32,32)  U  box [10,25]x[40,55]x[5,50]
  C2  512^2,  z in [0,512]:  U 200 spheres (centres U[0,512)^3, radii U[5,40])
                             U 50 boxes (min corner U[0,512)^3, edges U[8,64])
  C3  1024^2, z in [0,1024]: gyroid, period 64, t = 0.2, noise U[-0.05,0.05]
  C4  2048^2, z in [0,2048]: U 2000 spheres (radii U[10,120]) \\ U 1000 voids (U[10,120])
  C5  4096^2, z in [0,4096]: U 20000 spheres (radii U[8,200]) \\ U 10000 voids (U[8,200])

Random numbers come from a counter-based splitmix64 keyed by
(seed, stream, index) so results never depend on thread order.  Seeds are
1804089680 + k for config Ck; streams: 0 solid centres, 1 solid radii,
2 void centres, 3 void radii, 4 box corners, 5 box edges, 6 C3 noise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libdexelgen.so")
_lib = None

SEED_BASE = 1804089680


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "dexelgen.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm", "-lpthread"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        f32p = ctypes.POINTER(ctypes.c_float)
        lib.dexelgen_u64.restype = ctypes.c_uint64
        lib.dexelgen_u64.argtypes = [ctypes.c_uint64] * 3
        lib.dexelgen_uniform.restype = ctypes.c_double
        lib.dexelgen_uniform.argtypes = [ctypes.c_uint64] * 3
        lib.dexelgen_shapes.restype = ctypes.c_int
        lib.dexelgen_shapes.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int, ctypes.POINTER(u64p), ctypes.POINTER(f32p), u64p]
        lib.dexelgen_gyroid.restype = ctypes.c_int
        lib.dexelgen_gyroid.argtypes = [
            ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
            ctypes.c_int, ctypes.POINTER(u64p), ctypes.POINTER(f32p), u64p]
        lib.dexelgen_free.restype = None
        lib.dexelgen_free.argtypes = [ctypes.c_void_p]
        _lib = lib
    return _lib


@dataclass
class Grid:
    """Canonical dexel buffer in CSR form (host, numpy).

    off: uint64[nx*ny+1], column c = j*nx+i owns ep[2*off[c] : 2*off[c+1]]
    ep:  float32[2n], (z_in, z_out) pairs in the LOCAL frame z - z_ref
    z_lo, z_hi: the domain [zmin, zmax] in the local frame (fp32-exact)
    """
    nx: int
    ny: int
    off: np.ndarray
    ep: np.ndarray
    z_lo: float
    z_hi: float
    z_ref: float = 0.0
    spacing: float = 1.0

    @property
    def ncol(self) -> int:
        return self.nx * self.ny

    @property
    def n(self) -> int:
        return int(self.off[-1])

    def column(self, i: int, j: int) -> np.ndarray:
        c = j * self.nx + i
        a, b = int(self.off[c]), int(self.off[c + 1])
        return self.ep[2 * a:2 * b].reshape(-1, 2)

    def columns(self):
        """list of (k,2) float32 arrays, column order."""
        e = self.ep.reshape(-1, 2)
        o = self.off
        return [e[int(o[c]):int(o[c + 1])] for c in range(self.ncol)]


def from_columns(nx: int, ny: int, cols, z_lo: float, z_hi: float, z_ref: float = 0.0) -> Grid:
    cnt = np.array([len(c) for c in cols], dtype=np.uint64)
    off = np.zeros(nx * ny + 1, dtype=np.uint64)
    np.cumsum(cnt, out=off[1:])
    ep = np.concatenate([np.asarray(c, dtype=np.float32).reshape(-1) for c in cols]) if off[-1] else np.zeros(0, np.float32)
    return Grid(nx, ny, off, ep.astype(np.float32), float(np.float32(z_lo)), float(np.float32(z_hi)), z_ref)


# ---- counter RNG, vectorised (bitwise identical to dexelgen_u64 in C) ----
_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def rng_u64(seed: int, stream: int, index) -> np.ndarray:
    idx = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        k = _mix64(np.uint64(seed)) ^ (np.uint64(stream) * np.uint64(0xD1B54A32D192ED03))
        return _mix64(_mix64(k) ^ idx)


def rng_uniform(seed: int, stream: int, index) -> np.ndarray:
    return (rng_u64(seed, stream, index) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _call_shapes(nx, ny, zmin, zmax, sph, sph_sign, box, box_sign, nthreads):
    lib = _load()
    sph = np.ascontiguousarray(sph, dtype=np.float64).reshape(-1, 4)
    box = np.ascontiguousarray(box, dtype=np.float64).reshape(-1, 6)
    ss = np.ascontiguousarray(sph_sign, dtype=np.int32)
    bs = np.ascontiguousarray(box_sign, dtype=np.int32)
    offp = ctypes.POINTER(ctypes.c_uint64)()
    epp = ctypes.POINTER(ctypes.c_float)()
    n = ctypes.c_uint64(0)
    rc = lib.dexelgen_shapes(nx, ny, zmin, zmax, len(sph), sph.ctypes.data, ss.ctypes.data,
                             len(box), box.ctypes.data, bs.ctypes.data, int(nthreads),
                             ctypes.byref(offp), ctypes.byref(epp), ctypes.byref(n))
    if rc != 0:
        raise RuntimeError(f"dexelgen_shapes failed rc={rc}")
    return _wrap(nx, ny, offp, epp, n.value, zmin, zmax)


def _wrap(nx, ny, offp, epp, n, zmin, zmax) -> Grid:
    lib = _load()
    off = np.ctypeslib.as_array(offp, shape=(nx * ny + 1,)).copy()
    ep = np.ctypeslib.as_array(epp, shape=(2 * n + 2,))[:2 * n].copy()
    lib.dexelgen_free(ctypes.cast(offp, ctypes.c_void_p))
    lib.dexelgen_free(ctypes.cast(epp, ctypes.c_void_p))
    zref = 0.5 * (zmin + zmax)
    return Grid(nx, ny, off, ep, float(np.float32(zmin - zref)), float(np.float32(zmax - zref)), zref)


def shapes(nx: int, ny: int, zmin: float, zmax: float, spheres=(), voids=(), boxes=(), box_voids=(),
           nthreads: int | None = None) -> Grid:
    """Rasterise (U spheres U boxes) \\ (U voids U box_voids).  spheres: (cx,cy,cz,R) rows;
    boxes: (x0,x1,y0,y1,z0,z1) rows (a column is inside when its centre is in [x0,x1]x[y0,y1])."""
    sp = np.array(list(spheres) + list(voids), dtype=np.float64).reshape(-1, 4)
    ssg = np.array([1] * len(spheres) + [-1] * len(voids), dtype=np.int32)
    bx = np.array(list(boxes) + list(box_voids), dtype=np.float64).reshape(-1, 6)
    bsg = np.array([1] * len(boxes) + [-1] * len(box_voids), dtype=np.int32)
    return _call_shapes(nx, ny, float(zmin), float(zmax), sp, ssg, bx, bsg, nthreads or os.cpu_count() or 1)


def gyroid(n: int, period: float = 64.0, t: float = 0.2, amp: float = 0.05, seed: int = SEED_BASE + 3,
           nthreads: int | None = None) -> Grid:
    lib = _load()
    offp = ctypes.POINTER(ctypes.c_uint64)()
    epp = ctypes.POINTER(ctypes.c_float)()
    nn = ctypes.c_uint64(0)
    rc = lib.dexelgen_gyroid(n, period, t, amp, seed, int(nthreads or os.cpu_count() or 1),
                             ctypes.byref(offp), ctypes.byref(epp), ctypes.byref(nn))
    if rc != 0:
        raise RuntimeError("dexelgen_gyroid failed")
    return _wrap(n, n, offp, epp, nn.value, 0.0, float(n))


def _random_spheres(seed, n_pos, n_neg, N, rpos, rneg):
    k = np.arange(n_pos, dtype=np.uint64)
    c = rng_uniform(seed, 0, (3 * k[:, None] + np.arange(3, dtype=np.uint64)[None, :])) * N
    r = rpos[0] + (rpos[1] - rpos[0]) * rng_uniform(seed, 1, k)
    pos = np.concatenate([c, r[:, None]], axis=1)
    kv = np.arange(n_neg, dtype=np.uint64)
    cv = rng_uniform(seed, 2, (3 * kv[:, None] + np.arange(3, dtype=np.uint64)[None, :])) * N
    rv = rneg[0] + (rneg[1] - rneg[0]) * rng_uniform(seed, 3, kv)
    neg = np.concatenate([cv, rv[:, None]], axis=1)
    return pos, neg


CONFIGS = {
    "C1": dict(n=64, op=("dilate", "erode"), r=[3.0]),
    "C2": dict(n=512, op=("dilate", "erode", "shell"), r=[4.0]),
    "C3": dict(n=1024, op=("dilate", "erode"), r=[8.0]),
    "C4": dict(n=2048, op=("dilate",), r=[1.0, 2.0, 4.0, 8.0, 16.0, 32.0, 64.0]),
    "C5": dict(n=4096, op=("shell",), r=[16.0]),
}


def shape_config(name: str):
    """The analytic solid of a shape config (C1, C2, C4, C5) as arrays, without rasterising:
    (n, zmin, zmax, sph float64[k,4], sph_sign int32[k], box float64[m,6], box_sign int32[m])."""
    k = int(name[1])
    seed = SEED_BASE + k
    N = CONFIGS[name]["n"]
    box = np.zeros((0, 6))
    if name == "C1":
        sph, ssg = np.array([(32.0, 32.0, 32.0, 20.0)]), np.array([1])
        box = np.array([(10.0, 25.0, 40.0, 55.0, 5.0, 50.0)])
    elif name == "C2":
        pos, _ = _random_spheres(seed, 200, 0, N, (5.0, 40.0), (0.0, 0.0))
        kb = np.arange(50, dtype=np.uint64)
        corner = rng_uniform(seed, 4, 3 * kb[:, None] + np.arange(3, dtype=np.uint64)[None, :]) * N
        edge = 8.0 + 56.0 * rng_uniform(seed, 5, 3 * kb[:, None] + np.arange(3, dtype=np.uint64)[None, :])
        hi = np.minimum(corner + edge, N)
        box = np.stack([corner[:, 0], hi[:, 0], corner[:, 1], hi[:, 1], corner[:, 2], hi[:, 2]], axis=1)
        sph, ssg = pos, np.ones(len(pos))
    elif name in ("C4", "C5"):
        npos, nneg, rr = (2000, 1000, (10.0, 120.0)) if name == "C4" else (20000, 10000, (8.0, 200.0))
        pos, neg = _random_spheres(seed, npos, nneg, N, rr, rr)
        sph, ssg = np.concatenate([pos, neg]), np.array([1] * len(pos) + [-1] * len(neg))
    else:
        raise KeyError(f"{name} is not a shape config")
    return (N, 0.0, float(N), np.asarray(sph, np.float64).reshape(-1, 4), np.asarray(ssg, np.int32),
            np.asarray(box, np.float64).reshape(-1, 6), np.ones(len(box), np.int32))


def config(name: str, nthreads: int | None = None) -> Grid:
    """Build one of BASELINE.json's configs (C1..C5) deterministically."""
    k = int(name[1])
    seed = SEED_BASE + k
    N = CONFIGS[name]["n"]
    if name == "C1":
        return shapes(64, 64, 0.0, 64.0, spheres=[(32.0, 32.0, 32.0, 20.0)],
                      boxes=[(10.0, 25.0, 40.0, 55.0, 5.0, 50.0)], nthreads=nthreads)
    if name == "C2":
        pos, _ = _random_spheres(seed, 200, 0, N, (5.0, 40.0), (0.0, 0.0))
        kb = np.arange(50, dtype=np.uint64)
        corner = rng_uniform(seed, 4, 3 * kb[:, None] + np.arange(3, dtype=np.uint64)[None, :]) * N
        edge = 8.0 + 56.0 * rng_uniform(seed, 5, 3 * kb[:, None] + np.arange(3, dtype=np.uint64)[None, :])
        hi = np.minimum(corner + edge, N)
        boxes = np.stack([corner[:, 0], hi[:, 0], corner[:, 1], hi[:, 1], corner[:, 2], hi[:, 2]], axis=1)
        return shapes(N, N, 0.0, float(N), spheres=pos, boxes=boxes, nthreads=nthreads)
    if name == "C3":
        return gyroid(N, 64.0, 0.2, 0.05, seed, nthreads)
    if name == "C4":
        pos, neg = _random_spheres(seed, 2000, 1000, N, (10.0, 120.0), (10.0, 120.0))
        return shapes(N, N, 0.0, float(N), spheres=pos, voids=neg, nthreads=nthreads)
    if name == "C5":
        pos, neg = _random_spheres(seed, 20000, 10000, N, (8.0, 200.0), (8.0, 200.0))
        return shapes(N, N, 0.0, float(N), spheres=pos, voids=neg, nthreads=nthreads)
    raise KeyError(name)


def random_grid(nx: int, ny: int, max_per_col: int, z_lo: float, z_hi: float, seed: int,
                p_empty: float = 0.3, quantum: float | None = None) -> Grid:
    """Random canonical columns (test inputs).  With `quantum`, endpoints are
    multiples of it (creates exact ties / touching neighbours on purpose)."""
    rs = np.random.default_rng(seed)
    cols = []
    for _ in range(nx * ny):
        if rs.random() < p_empty:
            cols.append(np.zeros((0, 2), np.float32))
            continue
        k = int(rs.integers(1, max_per_col + 1))
        if quantum:
            pts = np.unique(np.round(rs.uniform(z_lo, z_hi, 2 * k) / quantum) * quantum)
        else:
            pts = np.unique(rs.uniform(z_lo, z_hi, 2 * k).astype(np.float32))
        pts = np.clip(pts, z_lo, z_hi).astype(np.float32)
        pts = np.unique(pts)
        if len(pts) % 2:
            pts = pts[:-1]
        cols.append(pts.reshape(-1, 2))
    return from_columns(nx, ny, cols, z_lo, z_hi)


def stats(g: Grid) -> dict:
    cnt = np.diff(g.off.astype(np.int64))
    nz = cnt[cnt > 0]
    return dict(ncol=g.ncol, n=g.n, mean_per_col=float(cnt.mean()), mean_nonempty=float(nz.mean()) if len(nz) else 0.0,
                max_per_col=int(cnt.max()) if len(cnt) else 0, frac_nonempty=float((cnt > 0).mean()))
