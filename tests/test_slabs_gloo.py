"""Multi-rank y-slab path on CPU (gloo, world_size 2 and 3): the halo exchange of
paper_1804_08968_b200.slabs moves exactly the R boundary rows each neighbour
needs, and the slab decomposition is exact -- the oracle run on every rank's
extended slab (lower halo + owned rows + upper halo) reproduces, on the owned
rows, the oracle run on the whole grid, bitwise (per-column results depend
only on rows within R).  The CUDA library's halo handling is tested on one GPU
in test_gpu_slabs.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import dexelgen as G
import oracle as O
from paper_1804_08968_b200.slabs import check_slabs, csr_rows, halo_exchange, slab_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _host(seed):
    return G.random_grid(13, 17, 3, -9.0, 9.0, seed, quantum=0.5 if seed % 2 else None)


def _worker(rank, world, port, seed, r, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        host = _host(seed)
        R = int(np.floor(r))
        nx, ny = host.nx, host.ny
        y0, y1 = slab_bounds(ny, world, rank)
        nrows = y1 - y0
        send = min(R, nrows)
        def rows(b, n):
            o, e = csr_rows(host.off, host.ep, nx, b, n)
            return torch.from_numpy(o.astype(np.int64)), torch.from_numpy(e)
        lo = rows(y0, send) if rank > 0 else None
        hi = rows(y1 - send, send) if rank + 1 < world else None
        nlo, nhi = min(R, y0), min(R, ny - y1)
        halo_lo, halo_hi = halo_exchange(lo, hi, rank, world, nlo, nhi, nx)
        # the received halos are exactly the neighbours' boundary rows
        if halo_lo is not None:
            o, e = csr_rows(host.off, host.ep, nx, y0 - nlo, nlo)
            assert np.array_equal(halo_lo[0].numpy().astype(np.uint64), o) and np.array_equal(halo_lo[1].numpy(), e)
        if halo_hi is not None:
            o, e = csr_rows(host.off, host.ep, nx, y1, nhi)
            assert np.array_equal(halo_hi[0].numpy().astype(np.uint64), o) and np.array_equal(halo_hi[1].numpy(), e)
        # extended slab = halo_lo + owned + halo_hi, built only from what this rank holds
        parts = []
        if halo_lo is not None:
            parts.append((halo_lo[0].numpy().astype(np.uint64), halo_lo[1].numpy()))
        parts.append(csr_rows(host.off, host.ep, nx, y0, nrows))
        if halo_hi is not None:
            parts.append((halo_hi[0].numpy().astype(np.uint64), halo_hi[1].numpy()))
        cols = []
        for o, e in parts:
            ee = e.reshape(-1, 2)
            cols += [ee[int(o[c]):int(o[c + 1])] for c in range(len(o) - 1)]
        hl = nlo if halo_lo is not None else 0
        ext = G.from_columns(nx, len(cols) // nx, cols, host.z_lo, host.z_hi)
        owned = np.arange(hl * nx, (hl + nrows) * nx, dtype=np.int64)
        full_cols = np.arange(y0 * nx, y1 * nx, dtype=np.int64)
        for op in ("dilate", "erode", "shell"):
            if op == "shell":
                a, b = O.shell(ext, r, r * 0.5, cols=owned), O.shell(host, r, r * 0.5, cols=full_cols)
            else:
                a, b = getattr(O, op)(ext, r, cols=owned), getattr(O, op)(host, r, cols=full_cols)
            assert np.array_equal(a.off, b.off) and np.array_equal(a.z, b.z), (op, rank)
        q.put((rank, "ok"))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,seed,r", [(2, 1, 2.0), (2, 2, 3.5), (3, 3, 2.0), (3, 4, 4.0)])
def test_slab_halo_exchange_gloo(world, seed, r):
    check_slabs(17, world, int(r))
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, seed, r, q), nprocs=world, join=True, start_method="spawn")
    res = sorted(q.get() for _ in range(world))
    assert all(v == "ok" for _, v in res), res


def test_slab_bounds_partition():
    for ny in (1, 5, 64, 4096):
        for world in (1, 2, 3, 8):
            if world > ny:
                continue
            rows = [slab_bounds(ny, world, g) for g in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == ny
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            assert max(b - a for a, b in rows) - min(b - a for a, b in rows) <= 1
    with pytest.raises(ValueError):
        check_slabs(20, 8, 3)


def _uid_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1804_08968_b200.slabs import broadcast_unique_id
        uid = broadcast_unique_id(rank)
        q.put((rank, uid.hex()))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, "ERR " + repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_nccl_unique_id_broadcast_gloo(world):
    """The communicator bootstrap of the in-library NCCL transport: rank 0 draws the 128-byte
    NCCL unique id through the C ABI (dexel_nccl_unique_id; no GPU needed), torch.distributed
    broadcasts it, and every rank holds the same non-trivial bytes for dexel_nccl_comm_init."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    mp.start_processes(_uid_worker, args=(world, port, q), nprocs=world, join=True, start_method="spawn")
    res = sorted(q.get() for _ in range(world))
    ids = {v for _, v in res}
    assert len(ids) == 1 and not next(iter(ids)).startswith("ERR"), res
    assert len(bytes.fromhex(next(iter(ids)))) == 128 and int(next(iter(ids)), 16) != 0
