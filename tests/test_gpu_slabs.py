"""y-slabs through the CUDA library on one GPU (loopback): every rank's slab is
run in turn with the halos the exchange would deliver, and the concatenated
owned rows are bitwise equal to the single-handle result.  (The exchange itself
is tested with gloo in test_slabs_gloo.py; no two "ranks" ever wait on each
other on this one GPU.)"""
import numpy as np
import pytest

import dexelgen as G
from paper_1804_08968_b200.slabs import csr_rows, slab_bounds

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_08968_b200 as dx
    from paper_1804_08968_b200 import build as B
    B.build()
    return dx


def run_full(dx, host, op, r):
    src = dx.Grid.from_host(host)
    dst = dx.Grid.like(src)
    getattr(dx, "dexel_" + op)(src, r, *( (r,) if op.startswith("shell") else ()), dst)
    return dst.download()


def run_slabs(dx, host, op, r, world):
    R = int(np.floor(r))
    offs, eps = [], []
    for g in range(world):
        y0, y1 = slab_bounds(host.ny, world, g)
        src = dx.Grid(host.nx, host.ny, host.z_lo, host.z_hi, host.z_ref, 1.0, 0, None, y0, y1, g, world)
        src.upload(*csr_rows(host.off, host.ep, host.nx, y0, y1 - y0))
        nlo, nhi = min(R, y0), min(R, host.ny - y1)
        if nlo:
            src.upload_halo(0, *csr_rows(host.off, host.ep, host.nx, y0 - nlo, nlo), nlo)
        if nhi:
            src.upload_halo(1, *csr_rows(host.off, host.ep, host.nx, y1, nhi), nhi)
        dst = dx.Grid.like(src)
        getattr(dx, "dexel_" + op)(src, r, *((r,) if op == "shell" else ()), dst)
        o, e = dst.download()
        offs.append(o)
        eps.append(e)
    # concatenate slab CSRs
    base, o_all = 0, [np.zeros(1, np.uint64)]
    for o in offs:
        o_all.append(o[1:] + np.uint64(base))
        base += int(o[-1])
    return np.concatenate(o_all), np.concatenate(eps)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("op,r", [("dilate", 4.0), ("erode", 3.0), ("shell", 4.0)])
def test_slabs_bitwise_equal_single(dx, world, op, r):
    host = G.config("C2")
    a = run_full(dx, host, op, r)
    b = run_slabs(dx, host, op, r, world)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_slab_download_rows_roundtrip(dx):
    host = G.config("C1")
    src = dx.Grid.from_host(host)
    for b, n in ((0, 3), (10, 7), (61, 3)):
        o, e = src.download_rows(b, n)
        o2, e2 = csr_rows(host.off, host.ep, host.nx, b, n)
        assert np.array_equal(o, o2) and np.array_equal(e, e2)


def test_slab_missing_halo_rejected(dx):
    host = G.config("C1")
    y0, y1 = slab_bounds(host.ny, 2, 1)
    src = dx.Grid(host.nx, host.ny, host.z_lo, host.z_hi, host.z_ref, 1.0, 0, None, y0, y1, 1, 2)
    src.upload(*csr_rows(host.off, host.ep, host.nx, y0, y1 - y0))
    dst = dx.Grid.like(src)
    with pytest.raises(dx.DexelError) as e:
        dx.dexel_dilate(src, 3.0, dst)
    assert e.value.status == dx.DEXEL_EINVAL and "halo" in str(e.value)
    src.upload_halo(0, *csr_rows(host.off, host.ep, host.nx, y0 - 2, 2), 2)   # too short for R = 3
    with pytest.raises(dx.DexelError):
        dx.dexel_dilate(src, 3.0, dst)
    src.upload_halo(0, *csr_rows(host.off, host.ep, host.nx, y0 - 3, 3), 3)
    dx.dexel_dilate(src, 3.0, dst)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("op", ["dilate_slices", "erode_slices", "shell_slices"])
def test_slice_ops_on_slabs_need_no_halo(dx, world, op):
    """2D slice offsets read no other row: y-slab handles without any halo give, concatenated,
    bitwise the single-handle result."""
    host = G.config("C2")
    r = 4.0
    full = run_full(dx, host, op, r)
    offs, eps = [], []
    for g in range(world):
        y0, y1 = slab_bounds(host.ny, world, g)
        src = dx.Grid(host.nx, host.ny, host.z_lo, host.z_hi, host.z_ref, 1.0, 0, None, y0, y1, g, world)
        src.upload(*csr_rows(host.off, host.ep, host.nx, y0, y1 - y0))
        dst = dx.Grid.like(src)
        getattr(dx, "dexel_" + op)(src, r, *((r,) if op == "shell_slices" else ()), dst)
        o, e = dst.download()
        offs.append(o)
        eps.append(e)
    base, o_all = 0, [np.zeros(1, np.uint64)]
    for o in offs:
        o_all.append(o[1:] + np.uint64(base))
        base += int(o[-1])
    assert np.array_equal(np.concatenate(o_all), full[0])
    assert np.array_equal(np.concatenate(eps), full[1])
