"""Test helpers (no method arithmetic): CSR column extraction and sampling."""
import numpy as np


def take_columns(off, ep, cols):
    """Sub-CSR of the given column ids -> (off uint64[len+1], z float64[2n])."""
    off = np.asarray(off, dtype=np.int64)
    e = np.asarray(ep, dtype=np.float64).reshape(-1, 2)
    cols = np.asarray(cols, dtype=np.int64)
    a, b = off[cols], off[cols + 1]
    cnt = b - a
    o = np.zeros(len(cols) + 1, np.int64)
    np.cumsum(cnt, out=o[1:])
    if o[-1] == 0:
        return o.astype(np.uint64), np.zeros(0)
    idx = np.repeat(a - o[:-1], cnt) + np.arange(o[-1])
    return o.astype(np.uint64), e[idx].reshape(-1)


def sample_columns(nx, ny, n_random, n_rows, n_lines, seed, extra_rows=()):
    """Seeded random columns + full rows + full column-lines (+ given rows)."""
    rs = np.random.default_rng(seed)
    cols = [rs.integers(0, nx * ny, n_random)]
    for j in list(rs.integers(0, ny, n_rows)) + list(extra_rows):
        cols.append(np.arange(nx) + int(j) * nx)
    for i in rs.integers(0, nx, n_lines):
        cols.append(np.arange(ny) * nx + int(i))
    return np.unique(np.concatenate(cols)).astype(np.int64)
