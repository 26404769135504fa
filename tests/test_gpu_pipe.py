"""dexel_pipe_*: host-to-host ops streamed in y-slabs (upload / op / download overlapped on three
host threads, include/dexel.h).  The streamed result must be bitwise the result of
dexel_upload + op + dexel_download on one handle of the whole grid (per-column results do not
depend on the partition), and is compared with the oracle as every op is."""
import numpy as np
import pytest

import dexelgen as G
import oracle as O
from oracle.compare import compare

pytestmark = pytest.mark.gpu
TAU = 1e-4


@pytest.fixture(scope="module")
def dx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_08968_b200 as dx
    from paper_1804_08968_b200 import build as B
    B.build()
    return dx


def run_full(dx, host, op, r, r2):
    src = dx.Grid.from_host(host)
    dst = dx.Grid.like(src)
    if op == "shell":
        dx.dexel_shell(src, r, r2, dst)
    else:
        getattr(dx, "dexel_" + op)(src, r, dst)
    out = dst.download()
    src.close()
    dst.close()
    return out


def run_pipe(dx, host, op, r, r2, nslabs, pinned=False, runs=1):
    pipe = dx.Pipe(host.nx, host.ny, host.z_lo, host.z_hi, nslabs)
    ncol = host.nx * host.ny
    cap = 64 * ncol + 1024
    off = np.ascontiguousarray(host.off, dtype=np.uint64)
    ep = np.ascontiguousarray(host.ep, dtype=np.float32)
    if pinned:
        import torch
        t_off = torch.from_numpy(off.view(np.int64)).pin_memory()
        t_ep = torch.from_numpy(ep).pin_memory() if ep.size else torch.zeros(2, dtype=torch.float32).pin_memory()
        o_off = torch.empty(ncol + 1, dtype=torch.int64).pin_memory()
        o_ep = torch.empty(2 * cap, dtype=torch.float32).pin_memory()
        for _ in range(runs):
            o_off.fill_(-1)
            n = pipe.run(op, r, r2, t_off, t_ep, o_off, o_ep)
        out = o_off.numpy().view(np.uint64).copy(), o_ep.numpy()[:2 * n].copy()
    else:
        o_off = np.full(ncol + 1, 2**63, np.uint64)
        o_ep = np.empty(2 * cap, np.float32)
        for _ in range(runs):
            n = pipe.run(op, r, r2, off, ep if ep.size else np.zeros(2, np.float32), o_off, o_ep)
        out = o_off, o_ep[:2 * n].copy()
    pipe.close()
    assert int(out[0][-1]) == n
    return out


@pytest.mark.parametrize("nslabs", [1, 2, 3, 7])
@pytest.mark.parametrize("op,r,r2", [("dilate", 3.5, 0.0), ("erode", 2.0, 0.0), ("shell", 4.0, 4.0),
                                     ("shell", 3.0, 1.5), ("dilate", 0.5, 0.0), ("dilate", 12.0, 0.0)])
def test_pipe_bitwise_equal_single_handle(dx, nslabs, op, r, r2):
    host = G.random_grid(70, 45, 5, -20.0, 30.0, seed=1000 + nslabs)
    a = run_full(dx, host, op, r, r2)
    b = run_pipe(dx, host, op, r, r2, nslabs)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_pipe_slabs_shorter_than_the_halo(dx):
    # slabs of 2 rows with R = 5: every slab's halo spans several other slabs (it comes from the host CSR)
    host = G.random_grid(40, 12, 4, -10.0, 10.0, seed=77)
    a = run_full(dx, host, "dilate", 5.0, 0.0)
    b = run_pipe(dx, host, "dilate", 5.0, 0.0, 6)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    b = run_pipe(dx, host, "dilate", 5.0, 0.0, 12)       # one row per slab
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("op,r,r2", [("dilate", 3.0, 0.0), ("shell", 2.5, 2.5)])
def test_pipe_matches_oracle(dx, op, r, r2):
    host = G.random_grid(48, 37, 4, -16.0, 16.0, seed=5)
    b = run_pipe(dx, host, op, r, r2, 4)
    ref = O.shell(host, r, r2) if op == "shell" else getattr(O, op)(host, r)
    res = compare(b[0], b[1], ref.off, ref.z, TAU)
    assert res["ok"], res


def test_pipe_c2_pinned_repeated(dx):
    # a BASELINE config, pinned buffers (the copies overlap the kernels), the pipeline reused
    host = G.config("C2")
    a = run_full(dx, host, "shell", 4.0, 4.0)
    b = run_pipe(dx, host, "shell", 4.0, 4.0, 4, pinned=True, runs=3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_pipe_partition_and_bytes(dx):
    host = G.random_grid(16, 40, 3, -4.0, 4.0, seed=9)
    for ns in (1, 2, 3, 5, 8, 40):
        pipe = dx.Pipe(16, 40, -4.0, 4.0, ns)
        rows = [pipe.slab_rows(q) for q in range(ns)]
        assert rows[0][0] == 0 and rows[-1][1] == 40
        assert all(a < b for a, b in rows) and all(rows[q][1] == rows[q + 1][0] for q in range(ns - 1))
        if 3 <= ns <= 8:                                    # the end slabs are about half the others
            mid = rows[1][1] - rows[1][0]
            assert rows[0][1] - rows[0][0] <= mid and rows[-1][1] - rows[-1][0] <= mid
        off = np.ascontiguousarray(host.off, dtype=np.uint64)
        ep = np.ascontiguousarray(host.ep, dtype=np.float32)
        o_off, o_ep = np.zeros(16 * 40 + 1, np.uint64), np.zeros(2 * 20000, np.float32)
        n = pipe.run("dilate", 2.0, 0.0, off, ep, o_off, o_ep)
        h2d, d2h = pipe.last_bytes()
        R, want = 2, 0
        for a, b in rows:
            for lo, hi in ((a, b), (max(0, a - R), a), (b, min(40, b + R))):
                if hi > lo:
                    want += 8 * ((hi - lo) * 16 + 1) + 8 * int(off[hi * 16] - off[lo * 16])
        assert h2d == want and d2h == 8 * (16 * 40 + ns) + 8 * n
        pipe.close()


def test_pipe_empty_and_full(dx):
    nx, ny = 33, 9
    off = np.zeros(nx * ny + 1, np.uint64)
    host = G.Grid(nx, ny, off, np.zeros(0, np.float32), -4.0, 4.0)
    o, e = run_pipe(dx, host, "dilate", 2.0, 0.0, 3)
    assert int(o[-1]) == 0 and not o.any()
    o, e = run_pipe(dx, host, "erode", 2.0, 0.0, 3)
    assert int(o[-1]) == 0


def test_pipe_errors(dx):
    host = G.random_grid(16, 8, 3, -4.0, 4.0, seed=3)
    with pytest.raises(dx.DexelError) as e:
        dx.Pipe(16, 8, -4.0, 4.0, 0)
    assert e.value.status == dx.DEXEL_EINVAL
    with pytest.raises(dx.DexelError) as e:
        dx.Pipe(16, 8, -4.0, 4.0, 9)                      # more slabs than rows
    assert e.value.status == dx.DEXEL_EINVAL
    pipe = dx.Pipe(16, 8, -4.0, 4.0, 2)
    off = np.ascontiguousarray(host.off, dtype=np.uint64)
    ep = np.ascontiguousarray(host.ep, dtype=np.float32)
    o_off = np.zeros(16 * 8 + 1, np.uint64)
    with pytest.raises(dx.DexelError) as e:              # capacity too small
        pipe.run("dilate", 2.0, 0.0, off, ep, o_off, np.zeros(2, np.float32))
    assert e.value.status == dx.DEXEL_EOVERFLOW
    with pytest.raises(dx.DexelError) as e:              # bad radius
        pipe.run("dilate", -1.0, 0.0, off, ep, o_off, np.zeros(4096, np.float32))
    assert e.value.status == dx.DEXEL_EINVAL
    bad = ep.copy()
    k = int(off[16 * 5 + 3])                             # an interval in the second slab (row 5)
    assert int(off[16 * 8]) > k
    bad[2 * k + 1] = np.nan
    with pytest.raises(dx.DexelError) as e:
        pipe.run("dilate", 2.0, 0.0, off, bad, o_off, np.zeros(4096, np.float32))
    assert e.value.status == dx.DEXEL_EINVAL
    # the pipeline still works after the errors
    o_ep = np.zeros(2 * 4096, np.float32)
    n = pipe.run("dilate", 2.0, 0.0, off, ep, o_off, o_ep)
    a = run_full(dx, host, "dilate", 2.0, 0.0)
    assert np.array_equal(a[0], o_off) and np.array_equal(a[1], o_ep[:2 * n])
    pipe.close()
