"""Multi-GPU y-slabs: one process per GPU, halo rows exchanged inside the library.

The path shards along y ("the 2D dilations can be
performed completely independently in every slice").  Rank g owns rows
[y0, y1).  Pass 1 runs along x and is row-local; pass 2 runs along y and reads
R = floor(r/s) rows of input beyond each slab boundary -- the only data-path
exchange.  Transports (include/dexel.h "Multi-GPU"):

  "nccl"      the library's own NCCL send/recv inside every (collective) op,
              overlapped with pass 1 of the slab's interior rows.  The
              communicator is bootstrapped here: rank 0 draws the NCCL unique
              id, torch.distributed broadcasts its 128 bytes, every rank calls
              dexel_nccl_comm_init.
  "loopback"  several slab handles in one process (one GPU in tests): the
              library copies the halo rows from the linked neighbour handles
              (dexel_link_slabs) -- the same halo layout and pass-1 split.
  "caller"    the caller moves the rows: dexel_download_rows packs them, a
              torch.distributed point-to-point exchange (gloo in the CPU tests)
              moves them, dexel_upload_halo attaches them.

Host-side helpers here hold no method arithmetic; they are plumbing.
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np


def slab_bounds(ny: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, as-even-as-possible row ranges [y0, y1) per rank."""
    base, extra = divmod(ny, world)
    y0 = rank * base + min(rank, extra)
    return y0, y0 + base + (1 if rank < extra else 0)


def check_slabs(ny: int, world: int, R: int):
    """Halos come from the adjacent rank only, so every slab needs >= R rows."""
    for g in range(world):
        y0, y1 = slab_bounds(ny, world, g)
        if world > 1 and y1 - y0 < R:
            raise ValueError(f"slab {g} has {y1 - y0} rows < R = {R}; use fewer ranks or a smaller radius")


def csr_rows(off: np.ndarray, ep: np.ndarray, nx: int, row_begin: int, nrows: int):
    """CSR slice of rows [row_begin, row_begin+nrows) with offsets rebased to 0 (host numpy)."""
    c0, c1 = row_begin * nx, (row_begin + nrows) * nx
    o = np.asarray(off[c0:c1 + 1], dtype=np.uint64)
    a, b = int(o[0]), int(o[-1])
    return (o - np.uint64(a)).astype(np.uint64), np.asarray(ep[2 * a:2 * b], dtype=np.float32)


def halo_exchange(send_lo, send_hi, rank: int, world: int, nrows_lo: int, nrows_hi: int, nx: int,
                  group=None):
    """Exchange boundary rows with the neighbouring ranks.

    send_lo: (off int64[.], ep float32[.]) of my first rows -> rank-1 (its upper halo)
    send_hi: my last rows -> rank+1 (its lower halo)
    nrows_lo / nrows_hi: rows expected FROM rank-1 / rank+1 (0 at the grid edge).
    Returns (halo_lo, halo_hi), each (off, ep) tensors on the send tensors' device, or None.
    Phase 1 exchanges interval counts, phase 2 the offsets and endpoints."""
    import torch
    import torch.distributed as dist

    ref = send_lo[0] if send_lo is not None else send_hi[0]
    dev = ref.device
    lo_peer = rank - 1 if rank > 0 else None
    hi_peer = rank + 1 if rank + 1 < world else None
    # phase 1: sizes
    ops, n_lo, n_hi = [], None, None
    if lo_peer is not None:
        ops.append(dist.P2POp(dist.isend, torch.tensor([send_lo[1].numel() // 2], dtype=torch.int64, device=dev),
                              lo_peer, group))
        n_lo = torch.zeros(1, dtype=torch.int64, device=dev)
        ops.append(dist.P2POp(dist.irecv, n_lo, lo_peer, group))
    if hi_peer is not None:
        ops.append(dist.P2POp(dist.isend, torch.tensor([send_hi[1].numel() // 2], dtype=torch.int64, device=dev),
                              hi_peer, group))
        n_hi = torch.zeros(1, dtype=torch.int64, device=dev)
        ops.append(dist.P2POp(dist.irecv, n_hi, hi_peer, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    # phase 2: payloads
    ops, halo_lo, halo_hi = [], None, None
    if lo_peer is not None:
        ops.append(dist.P2POp(dist.isend, send_lo[0].contiguous(), lo_peer, group))
        ops.append(dist.P2POp(dist.isend, send_lo[1].contiguous(), lo_peer, group))
        halo_lo = (torch.empty(nrows_lo * nx + 1, dtype=torch.int64, device=dev),
                   torch.empty(2 * int(n_lo.item()), dtype=torch.float32, device=dev))
        ops.append(dist.P2POp(dist.irecv, halo_lo[0], lo_peer, group))
        ops.append(dist.P2POp(dist.irecv, halo_lo[1], lo_peer, group))
    if hi_peer is not None:
        ops.append(dist.P2POp(dist.isend, send_hi[0].contiguous(), hi_peer, group))
        ops.append(dist.P2POp(dist.isend, send_hi[1].contiguous(), hi_peer, group))
        halo_hi = (torch.empty(nrows_hi * nx + 1, dtype=torch.int64, device=dev),
                   torch.empty(2 * int(n_hi.item()), dtype=torch.float32, device=dev))
        ops.append(dist.P2POp(dist.irecv, halo_hi[0], hi_peer, group))
        ops.append(dist.P2POp(dist.irecv, halo_hi[1], hi_peer, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return halo_lo, halo_hi


def broadcast_unique_id(rank: int, device: Optional[int] = None, group=None) -> bytes:
    """Rank 0 draws the 128-byte NCCL unique id (dexel_nccl_unique_id); torch.distributed
    broadcasts it (a CUDA tensor under the nccl backend, a CPU tensor under gloo)."""
    import torch
    import torch.distributed as dist

    import paper_1804_08968_b200 as dx
    on_gpu = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", device or 0) if on_gpu else torch.device("cpu")
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(dx.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=0, group=group)
    return bytes(buf.cpu().tolist())


def nccl_bootstrap(rank: int, world: int, device: int, group=None) -> int:
    """ncclComm_t for the library: the broadcast unique id, then dexel_nccl_comm_init on every
    rank (collective)."""
    import paper_1804_08968_b200 as dx
    return dx.nccl_comm_init(broadcast_unique_id(rank, device, group), world, rank, device)


class Slab:
    """One rank's slab of a dexel grid on its GPU (src handle + dst handle)."""

    def __init__(self, host, rank: int, world: int, device: int, stream: Optional[int] = None,
                 transport: str = "caller", comm: Optional[int] = None):
        import paper_1804_08968_b200 as dx
        if transport not in ("nccl", "loopback", "caller"):
            raise ValueError(f"unknown transport {transport!r}")
        if transport == "nccl" and world > 1 and not comm:
            raise ValueError("transport 'nccl' needs a communicator (nccl_bootstrap)")
        self.dx = dx
        self.transport = transport
        self.rank, self.world, self.nx, self.ny = rank, world, host.nx, host.ny
        self.y0, self.y1 = slab_bounds(host.ny, world, rank)
        self.src = dx.Grid(host.nx, host.ny, host.z_lo, host.z_hi, getattr(host, "z_ref", 0.0),
                           getattr(host, "spacing", 1.0), device, stream, self.y0, self.y1, rank, world,
                           comm if transport == "nccl" else None)
        off, ep = csr_rows(host.off, host.ep, host.nx, self.y0, self.y1 - self.y0)
        self.src.upload(off, ep)
        self.dst = dx.Grid.like(self.src)
        self.halo_rows = -1

    def refresh_halos(self, R: int, group=None):
        """Caller-managed transport only: exchange R boundary rows with the neighbours over
        torch.distributed (device buffers) and attach them.  (NCCL / loopback slabs exchange
        inside every op.)"""
        if self.transport != "caller":
            return
        check_slabs(self.ny, self.world, R)   # (a neighbour sends min(R, its rows): every slab needs R rows)
        nrows = self.y1 - self.y0
        send = min(R, nrows)
        lo = self.src.download_rows(0, send, device=True) if self.rank > 0 else None
        hi = self.src.download_rows(nrows - send, send, device=True) if self.rank + 1 < self.world else None
        nlo = min(R, self.y0)
        nhi = min(R, self.ny - self.y1)
        if self.world > 1:
            halo_lo, halo_hi = halo_exchange(lo, hi, self.rank, self.world, nlo, nhi, self.nx, group)
            # the receives complete on torch's current stream; the library reads the buffers on the
            # handle's own stream: order them (Work.wait() orders only torch's stream)
            recv = halo_lo if halo_lo is not None else halo_hi
            if recv is not None and recv[0].is_cuda:
                import torch
                torch.cuda.current_stream(recv[0].device).synchronize()
        else:
            halo_lo = halo_hi = None
        self.src.upload_halo(0, *(halo_lo if halo_lo is not None else (None, None)), nlo if halo_lo is not None else 0)
        self.src.upload_halo(1, *(halo_hi if halo_hi is not None else (None, None)), nhi if halo_hi is not None else 0)
        self.halo_rows = R

    def op(self, op: str, r: float, r2: Optional[float] = None):
        dx = self.dx
        if op in ("dilate", "erode", "dilate_slices", "erode_slices", "open", "close"):
            getattr(dx, "dexel_" + op)(self.src, r, self.dst)
        elif op in ("shell", "shell_slices"):
            getattr(dx, "dexel_" + op)(self.src, r, r if r2 is None else r2, self.dst)
        else:
            raise ValueError(f"unknown op {op!r}")
        return self.dst

    def close(self):
        self.src.close()
        self.dst.close()


def loopback_slabs(host, world: int, device: int = 0, stream: Optional[int] = None):
    """`world` slab handles of one grid in this process, linked for in-library halo copies
    (dexel_link_slabs); their ops need no exchange by the caller."""
    import paper_1804_08968_b200 as dx
    slabs = [Slab(host, g, world, device, stream, transport="loopback") for g in range(world)]
    if world > 1:
        dx.link_slabs([s.src for s in slabs])
    return slabs


def concat_slabs(parts):
    """Concatenate per-slab CSRs (off, ep) in rank order into one global CSR (host numpy)."""
    base, offs, eps = 0, [np.zeros(1, np.uint64)], []
    for o, e in parts:
        o = np.asarray(o, dtype=np.uint64)
        offs.append(o[1:] + np.uint64(base))
        base += int(o[-1])
        eps.append(np.asarray(e, dtype=np.float32))
    return np.concatenate(offs), (np.concatenate(eps) if eps else np.zeros(0, np.float32))
