"""y-slabs through the CUDA library on one GPU.

* loopback transport (dexel_link_slabs): the library itself fetches every op's halo rows from
  the neighbouring slab handles -- the halo layout and the split pass-1 launches the NCCL
  transport uses -- and the concatenated owned rows are bitwise equal to the single-handle
  result;
* caller-managed halos (dexel_upload_halo) with the rows the exchange would deliver, likewise.
No two "ranks" ever wait on each other's kernels on this one GPU (loopback copies read the
neighbours' already-uploaded inputs)."""
import numpy as np
import pytest

import dexelgen as G
from paper_1804_08968_b200.slabs import concat_slabs, csr_rows, loopback_slabs, slab_bounds

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


def run_loopback(dx, host, op, r, world, r2=None):
    slabs = loopback_slabs(host, world)
    parts = []
    for sl in slabs:
        sl.op(op, r, r2)
        parts.append(sl.dst.download())
    for sl in slabs:
        sl.close()
    return concat_slabs(parts)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("op,r", [("dilate", 4.0), ("erode", 3.0), ("shell", 4.0), ("dilate", 9.5)])
def test_loopback_slabs_bitwise_equal_single(dx, world, op, r):
    """In-library halo exchange (loopback transport): slabs == one handle, bitwise."""
    host = G.config("C2")
    a = run_full(dx, host, op, r)
    b = run_loopback(dx, host, op, r, world)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_loopback_shell_radii_and_slices(dx):
    """Shell with r_out != r_in (halo = max R), and slice ops (no halo at all)."""
    host = G.config("C1")
    src = dx.Grid.from_host(host)
    dst = dx.Grid.like(src)
    dx.dexel_shell(src, 5.0, 2.5, dst)
    a = dst.download()
    b = run_loopback(dx, host, "shell", 5.0, 3, 2.5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    dx.dexel_erode_slices(src, 3.0, dst)
    a = dst.download()
    b = run_loopback(dx, host, "erode_slices", 3.0, 4)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_loopback_band_split(dx):
    """Row bands smaller than the slab (DEXEL_BAND_ROWS), tiny level capacities and a halo spanning
    several bands: the split pass-1 launches (own rows first, halo rows after the exchange event)
    still give the single-handle result bitwise.  Subprocess: the overrides are read once."""
    import os
    import subprocess
    import sys
    code = r"""
import sys, hashlib; sys.path.insert(0, %r)
import numpy as np, dexelgen as G, paper_1804_08968_b200 as dx
from paper_1804_08968_b200.slabs import loopback_slabs, concat_slabs
host = G.random_grid(45, 61, 5, -20.0, 20.0, 5)
for op, r in (("dilate", 6.0), ("shell", 4.5), ("erode", 2.0)):
    src = dx.Grid.from_host(host); dst = dx.Grid.like(src)
    (dx.dexel_shell(src, r, r, dst) if op == "shell" else getattr(dx, "dexel_" + op)(src, r, dst))
    a = dst.download()
    slabs = loopback_slabs(host, 3)
    b = concat_slabs([sl.op(op, r).download() for sl in slabs])
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), op
print("OK")
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DEXEL_BAND_ROWS="4", DEXEL_LEV_CAP="1", DEXEL_P1_CAP="2")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "OK" in out.stdout, out.stdout + out.stderr


def test_loopback_errors(dx):
    """A slab shorter than R fails with EINVAL; badly ordered link lists are rejected."""
    host = G.config("C1")
    slabs = loopback_slabs(host, 8)            # 8 rows per slab
    with pytest.raises(dx.DexelError) as e:
        slabs[3].op("dilate", 9.0)             # R = 9 > 8 rows of the neighbours
    assert e.value.status == dx.DEXEL_EINVAL
    slabs[3].op("dilate", 8.0)                 # R = 8 fits
    with pytest.raises(dx.DexelError):
        dx.link_slabs([slabs[1].src, slabs[0].src])
    for sl in slabs:
        sl.close()


def test_nccl_single_rank_comm(dx):
    """A one-rank NCCL communicator through the C ABI (dexel_nccl_comm_init / destroy): a handle
    carrying it runs ops like any single-GPU handle."""
    uid = dx.nccl_unique_id()
    comm = dx.nccl_comm_init(uid, 1, 0, 0)
    try:
        host = G.config("C1")
        g = dx.Grid(host.nx, host.ny, host.z_lo, host.z_hi, host.z_ref, 1.0, 0, None, 0, host.ny, 0, 1, comm)
        g.upload(host.off, host.ep)
        d = dx.Grid.like(g)
        dx.dexel_dilate(g, 3.0, d)
        a = run_full(dx, host, "dilate", 3.0)
        b = d.download()
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        g.close()
        d.close()
    finally:
        dx.nccl_comm_destroy(comm)
