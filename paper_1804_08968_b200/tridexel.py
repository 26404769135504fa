"""Tri-dexel offsets: a solid held as three dexel
buffers, the rays of each parallel to one axis, offset buffer by buffer.

Each buffer is an ordinary library grid over a permutation of the axes:
    z-buffer: grid (x, y), rays along z      shapes as given
    x-buffer: grid (y, z), rays along x      (cx, cy, cz) -> (cy, cz, cx)
    y-buffer: grid (z, x), rays along y      (cx, cy, cz) -> (cz, cx, cy)
Eq. 1 is invariant under a permutation of the axes, so the offset of a
tri-dexel solid is the library op on each buffer (the paper's estimate: about 3x the run
time of one buffer).  This module only composes C-ABI calls (marshalling and
axis bookkeeping); every step runs in the library's kernels.  The domain is a cube
[0, n]^3 sampled by n x n rays per buffer (the shape configs C1, C2, C4, C5)."""
from __future__ import annotations

import numpy as np

from . import (Grid, dexel_dilate, dexel_erode, dexel_rasterize_shapes, dexel_shell)

AXES = ("z", "x", "y")
# coordinate order (world axis index per buffer axis: grid i, grid j, ray) of each buffer
_PERM = {"z": (0, 1, 2), "x": (1, 2, 0), "y": (2, 0, 1)}


def permute_shapes(axis: str, sph, box):
    """shapes in the frame of one buffer: spheres (cx, cy, cz, R), boxes (x0, x1, y0, y1, z0, z1)."""
    p = _PERM[axis]
    sph = np.asarray(sph, dtype=np.float64).reshape(-1, 4)
    box = np.asarray(box, dtype=np.float64).reshape(-1, 6)
    s2 = np.concatenate([sph[:, list(p)], sph[:, 3:4]], axis=1)
    b2 = np.concatenate([box[:, [2 * p[0], 2 * p[0] + 1]], box[:, [2 * p[1], 2 * p[1] + 1]],
                         box[:, [2 * p[2], 2 * p[2] + 1]]], axis=1)
    return np.ascontiguousarray(s2), np.ascontiguousarray(b2)


class TriDexel:
    """Three buffers of one solid on one device (dict axis -> Grid)."""

    def __init__(self, n: int, zmin: float, zmax: float, device: int = 0, stream=None):
        self.n, self.zmin, self.zmax = int(n), float(zmin), float(zmax)
        zref = 0.5 * (self.zmin + self.zmax)
        z_lo = float(np.float32(self.zmin - zref))
        z_hi = float(np.float32(self.zmax - zref))
        self.buf = {a: Grid(self.n, self.n, z_lo, z_hi, zref, 1.0, device, stream) for a in AXES}

    @classmethod
    def from_shapes(cls, n, zmin, zmax, sph, sph_sign, box, box_sign, device: int = 0, stream=None):
        """rasterise (U solids) minus (U voids) into the three buffers (dexel_rasterize_shapes)."""
        t = cls(n, zmin, zmax, device, stream)
        for a in AXES:
            s2, b2 = permute_shapes(a, sph, box)
            dexel_rasterize_shapes(t.buf[a], zmin, zmax, s2, sph_sign, b2, box_sign)
        return t

    def like(self) -> "TriDexel":
        t = TriDexel.__new__(TriDexel)
        t.n, t.zmin, t.zmax = self.n, self.zmin, self.zmax
        t.buf = {a: Grid.like(self.buf[a]) for a in AXES}
        return t

    def _apply(self, fn, out: "TriDexel | None", *args) -> "TriDexel":
        out = out or self.like()
        for a in AXES:
            fn(self.buf[a], *args, out.buf[a])
        return out

    def dilate(self, r: float, out: "TriDexel | None" = None) -> "TriDexel":
        return self._apply(dexel_dilate, out, r)

    def erode(self, r: float, out: "TriDexel | None" = None) -> "TriDexel":
        return self._apply(dexel_erode, out, r)

    def shell(self, r_out: float, r_in: float, out: "TriDexel | None" = None) -> "TriDexel":
        return self._apply(dexel_shell, out, r_out, r_in)

    def size(self) -> int:
        return sum(self.buf[a].size() for a in AXES)

    def close(self) -> None:
        for a in AXES:
            self.buf[a].close()
