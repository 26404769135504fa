"""Comparator for dexel results (test infrastructure; applied identically to
both sides).  BASELINE.json north_star: "Per-column interval counts must be
identical after merging gaps smaller than 1e-4 dexel spacing. Endpoints must
agree within 1e-4 x dexel spacing."  DESIGN.md reading R8 adds the dual rule:
intervals shorter than tau are dropped after merging.

Vectorised over all columns with numpy.
"""
from __future__ import annotations

import numpy as np


def canonical(off, z, tau):
    """Merge gaps < tau, then drop intervals shorter than tau.  Returns (off, z) float64."""
    off = np.asarray(off, dtype=np.int64)
    z = np.asarray(z, dtype=np.float64).reshape(-1, 2)
    ncol = len(off) - 1
    n = len(z)
    if n == 0:
        return np.zeros(ncol + 1, np.int64), np.zeros((0, 2))
    col = np.repeat(np.arange(ncol), np.diff(off))
    newgrp = np.ones(n, dtype=bool)
    if n > 1:
        same = col[1:] == col[:-1]
        gap = z[1:, 0] - z[:-1, 1]
        newgrp[1:] = ~(same & (gap < tau))
    gid = np.cumsum(newgrp) - 1
    first = np.flatnonzero(newgrp)
    last = np.r_[first[1:] - 1, n - 1]
    lo = z[first, 0]
    hi = np.maximum.reduceat(z[:, 1], first)
    gcol = col[first]
    keep = (hi - lo) >= tau
    lo, hi, gcol = lo[keep], hi[keep], gcol[keep]
    cnt = np.bincount(gcol, minlength=ncol)
    o = np.zeros(ncol + 1, np.int64)
    np.cumsum(cnt, out=o[1:])
    del gid, last
    return o, np.stack([lo, hi], axis=1)


def compare(off_a, z_a, off_b, z_b, tau=1e-4):
    """Returns dict(ok, count_mismatch, max_err, first_bad, n_a, n_b)."""
    oa, za = canonical(off_a, z_a, tau)
    ob, zb = canonical(off_b, z_b, tau)
    ca, cb = np.diff(oa), np.diff(ob)
    mism = np.flatnonzero(ca != cb)
    good = ca == cb
    # endpoints of columns with equal counts
    ia = np.repeat(good, ca)
    ib = np.repeat(good, cb)
    ea, eb = za[ia], zb[ib]
    err = np.abs(ea - eb)
    max_err = float(err.max()) if err.size else 0.0
    bad_ep = np.flatnonzero((err > tau).any(axis=1)) if err.size else np.zeros(0, np.int64)
    first_bad = None
    if len(mism):
        first_bad = int(mism[0])
    elif len(bad_ep):
        colsa = np.repeat(np.arange(len(ca)), ca)[ia]
        first_bad = int(colsa[bad_ep[0]])
    return dict(ok=bool(len(mism) == 0 and len(bad_ep) == 0), count_mismatch=int(len(mism)),
                endpoint_fail=int(len(bad_ep)), max_err=max_err, first_bad=first_bad,
                n_a=int(oa[-1]), n_b=int(ob[-1]))


def describe(off_a, z_a, off_b, z_b, c):
    a = np.asarray(z_a).reshape(-1, 2)[int(off_a[c]):int(off_a[c + 1])]
    b = np.asarray(z_b).reshape(-1, 2)[int(off_b[c]):int(off_b[c + 1])]
    return f"column {c}:\n  A={a.tolist()}\n  B={b.tolist()}"
