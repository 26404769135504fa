"""B200-native separable dexel offsets (arXiv 1804.08968) -- Python binding.

Thin ctypes marshalling over libdexel.so (the C ABI declared in
include/dexel.h).  Every step of the path runs in the library's CUDA
kernels; this module only moves pointers, sizes and status codes.  There is
no CPU fallback: if the shared library is missing, every call raises.

PyTorch is used only for device memory (optional caching-allocator hook),
streams and -- in multi-process code -- process groups.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdexel.so")

DEXEL_OK, DEXEL_EINVAL, DEXEL_ENOMEM, DEXEL_EMISMATCH, DEXEL_EOVERFLOW, DEXEL_ECUDA, DEXEL_ENCCL = range(7)
_STATUS = {1: "EINVAL", 2: "ENOMEM", 3: "EMISMATCH", 4: "EOVERFLOW", 5: "ECUDA", 6: "ENCCL"}

# every symbol include/dexel.h declares (checked by tests/test_abi.py)
EXPORTS = ["dexel_create", "dexel_upload", "dexel_dilate", "dexel_erode", "dexel_shell", "dexel_open", "dexel_close",
           "dexel_dilate_slices", "dexel_erode_slices", "dexel_shell_slices", "dexel_rasterize_shapes", "dexel_rasterize_gyroid", "dexel_trim_workspace", "dexel_size",
           "dexel_download", "dexel_pass1", "dexel_sync", "dexel_destroy", "dexel_last_error",
           "dexel_set_allocator", "dexel_last_stats", "dexel_set_timing", "dexel_upload_halo",
           "dexel_download_rows", "dexel_nccl_unique_id", "dexel_nccl_comm_init", "dexel_nccl_comm_destroy",
           "dexel_link_slabs", "dexel_pipe_create", "dexel_pipe_run", "dexel_pipe_destroy",
           "dexel_pipe_suggest_slabs", "dexel_pipe_slab_rows", "dexel_pipe_last_bytes"]


class DexelError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"dexel {_STATUS.get(status, status)}: {msg}")
        self.status = status


class dexel_desc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("spacing", ctypes.c_double),
                ("z_ref", ctypes.c_double), ("z_lo", ctypes.c_float), ("z_hi", ctypes.c_float),
                ("device", ctypes.c_int32), ("stream", ctypes.c_void_p), ("nccl_comm", ctypes.c_void_p),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("y0", ctypes.c_int32),
                ("y1", ctypes.c_int32)]


NKERNELS = 8
KERNEL_NAMES = ["pass1", "pass1_list", "levels", "pass2", "compact", "scan", "other", "raster"]


class dexel_stats(ctypes.Structure):
    _fields_ = [("n_in", ctypes.c_uint64), ("n_mid", ctypes.c_uint64), ("n_lev", ctypes.c_uint64),
                ("n_out", ctypes.c_uint64), ("launches", ctypes.c_uint32),
                ("kernel_calls", ctypes.c_uint32 * NKERNELS), ("kernel_ms", ctypes.c_float * NKERNELS),
                ("lev_cap", ctypes.c_uint32), ("p2_acc", ctypes.c_uint32), ("bands", ctypes.c_uint32)]


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p)

_lib = None
_alloc_keep = []   # every allocator callback pair ever installed (kept alive)


def lib():
    """Load libdexel.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, u64, u64p = ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)
        sig = {
            "dexel_create": ([ctypes.POINTER(dexel_desc), ctypes.POINTER(vp)], ctypes.c_int),
            "dexel_upload": ([vp, vp, vp, u64, ctypes.c_int], ctypes.c_int),
            "dexel_dilate": ([vp, ctypes.c_float, vp], ctypes.c_int),
            "dexel_erode": ([vp, ctypes.c_float, vp], ctypes.c_int),
            "dexel_shell": ([vp, ctypes.c_float, ctypes.c_float, vp], ctypes.c_int),
            "dexel_open": ([vp, ctypes.c_float, vp], ctypes.c_int),
            "dexel_close": ([vp, ctypes.c_float, vp], ctypes.c_int),
            "dexel_dilate_slices": ([vp, ctypes.c_float, vp], ctypes.c_int),
            "dexel_erode_slices": ([vp, ctypes.c_float, vp], ctypes.c_int),
            "dexel_shell_slices": ([vp, ctypes.c_float, ctypes.c_float, vp], ctypes.c_int),
            "dexel_rasterize_shapes": ([vp, ctypes.c_double, ctypes.c_double, ctypes.c_int, vp, vp, ctypes.c_int, vp,
                                        vp, ctypes.c_int], ctypes.c_int),
            "dexel_rasterize_gyroid": ([vp, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, u64], ctypes.c_int),
            "dexel_trim_workspace": ([ctypes.c_int], ctypes.c_int),
            "dexel_size": ([vp, u64p], ctypes.c_int),
            "dexel_download": ([vp, vp, vp, u64, ctypes.c_int], ctypes.c_int),
            "dexel_pass1": ([vp, ctypes.c_float, ctypes.c_int, vp, vp, vp, u64, u64p, ctypes.c_int], ctypes.c_int),
            "dexel_sync": ([vp], ctypes.c_int),
            "dexel_destroy": ([vp], None),
            "dexel_last_error": ([], ctypes.c_char_p),
            "dexel_set_allocator": ([ALLOC_FN, FREE_FN, vp], ctypes.c_int),
            "dexel_last_stats": ([vp, ctypes.POINTER(dexel_stats)], ctypes.c_int),
            "dexel_set_timing": ([ctypes.c_int], ctypes.c_int),
            "dexel_upload_halo": ([vp, ctypes.c_int, vp, vp, ctypes.c_int, u64, ctypes.c_int], ctypes.c_int),
            "dexel_download_rows": ([vp, ctypes.c_int, ctypes.c_int, vp, vp, u64, u64p, ctypes.c_int], ctypes.c_int),
            "dexel_nccl_unique_id": ([vp], ctypes.c_int),
            "dexel_nccl_comm_init": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)], ctypes.c_int),
            "dexel_nccl_comm_destroy": ([vp], ctypes.c_int),
            "dexel_link_slabs": ([ctypes.POINTER(vp), ctypes.c_int], ctypes.c_int),
            "dexel_pipe_create": ([ctypes.POINTER(dexel_desc), ctypes.c_int, ctypes.POINTER(vp)], ctypes.c_int),
            "dexel_pipe_run": ([vp, ctypes.c_int, ctypes.c_float, ctypes.c_float, vp, vp, vp, vp, u64, u64p],
                               ctypes.c_int),
            "dexel_pipe_destroy": ([vp], None),
            "dexel_pipe_suggest_slabs": ([ctypes.POINTER(dexel_desc), ctypes.c_float], ctypes.c_int),
            "dexel_pipe_slab_rows": ([vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)],
                                     ctypes.c_int),
            "dexel_pipe_last_bytes": ([vp, u64p, u64p], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(status: int):
    if status != DEXEL_OK:
        raise DexelError(status, lib().dexel_last_error().decode())


def _ptr(a) -> int:
    """data pointer of a numpy array or torch tensor"""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _is_dev(a) -> bool:
    return not isinstance(a, np.ndarray) and getattr(a, "is_cuda", False)


# ---------------------------------------------------------------- allocator hook
_alloc_refs = None


def use_torch_allocator(enable: bool = True):
    """Route library device allocations through the PyTorch caching allocator."""
    global _alloc_refs
    L = lib()
    if not enable:
        # the callbacks stay referenced (module-level list): buffers allocated through them
        # are still released through them by the library
        _check(L.dexel_set_allocator(ALLOC_FN(), FREE_FN(), None))
        return
    import torch

    def _alloc(nbytes, device, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), int(device), stream)
        except Exception:  # noqa: BLE001 -- reported to C as NULL -> DEXEL_ENOMEM
            return None

    def _free(ptr, nbytes, device, stream, ctx):
        torch.cuda.caching_allocator_delete(ptr)

    _alloc_refs = (ALLOC_FN(_alloc), FREE_FN(_free))
    _alloc_keep.append(_alloc_refs)
    _check(L.dexel_set_allocator(_alloc_refs[0], _alloc_refs[1], None))


# ---------------------------------------------------------------- grid handle
class Grid:
    """A dexel buffer on one device (one handle of the C ABI)."""

    def __init__(self, nx: int, ny: int, z_lo: float, z_hi: float, z_ref: float = 0.0, spacing: float = 1.0,
                 device: int = 0, stream: Optional[int] = None, y0: int = 0, y1: Optional[int] = None,
                 rank: int = 0, nranks: int = 1, nccl_comm: Optional[int] = None):
        self.desc = dexel_desc(nx, ny, spacing, z_ref, z_lo, z_hi, device, stream, nccl_comm, rank, nranks,
                               y0, ny if y1 is None else y1)
        h = ctypes.c_void_p()
        _check(lib().dexel_create(ctypes.byref(self.desc), ctypes.byref(h)))
        self.h = h

    @classmethod
    def like(cls, g: "Grid") -> "Grid":
        d = g.desc
        return cls(d.nx, d.ny, d.z_lo, d.z_hi, d.z_ref, d.spacing, d.device, d.stream, d.y0, d.y1, d.rank,
                   d.nranks, d.nccl_comm)

    @classmethod
    def from_host(cls, hg, device: int = 0, stream: Optional[int] = None) -> "Grid":
        """from a dexelgen.Grid-like object (nx, ny, off, ep, z_lo, z_hi, z_ref, spacing)"""
        g = cls(hg.nx, hg.ny, hg.z_lo, hg.z_hi, getattr(hg, "z_ref", 0.0), getattr(hg, "spacing", 1.0), device,
                stream)
        g.upload(hg.off, hg.ep)
        return g

    @property
    def ncol(self) -> int:
        return self.desc.nx * (self.desc.y1 - self.desc.y0)

    def upload(self, off, ep):
        if isinstance(off, np.ndarray):
            off = np.ascontiguousarray(off, dtype=np.uint64)
            ep = np.ascontiguousarray(ep, dtype=np.float32)
        n = (int(off[-1]) if isinstance(off, np.ndarray) else int(ep.numel()) // 2)
        _check(lib().dexel_upload(self.h, _ptr(off), _ptr(ep) if n else None, n, 1 if _is_dev(off) else 0))

    def size(self) -> int:
        n = ctypes.c_uint64()
        _check(lib().dexel_size(self.h, ctypes.byref(n)))
        return n.value

    def download(self, device: bool = False):
        n = self.size()
        if device:
            import torch
            dev = torch.device("cuda", self.desc.device)
            off = torch.empty(self.ncol + 1, dtype=torch.int64, device=dev)
            ep = torch.empty(max(2 * n, 2), dtype=torch.float32, device=dev)
            _check(lib().dexel_download(self.h, off.data_ptr(), ep.data_ptr(), n, 1))
            return off, ep[:2 * n]
        off = np.empty(self.ncol + 1, dtype=np.uint64)
        ep = np.empty(max(2 * n, 2), dtype=np.float32)
        _check(lib().dexel_download(self.h, off.ctypes.data, ep.ctypes.data, n, 0))
        return off, ep[:2 * n]

    def upload_halo(self, side: int, off, ep, nrows: int):
        """attach nrows halo rows below (side 0) or above (side 1) the slab (numpy or CUDA tensors)."""
        if nrows == 0:
            _check(lib().dexel_upload_halo(self.h, side, None, None, 0, 0, 0))
            return
        if isinstance(off, np.ndarray):
            off = np.ascontiguousarray(off, dtype=np.uint64)
            ep = np.ascontiguousarray(ep, dtype=np.float32)
        n = int(off[-1]) if isinstance(off, np.ndarray) else int(ep.numel()) // 2
        _check(lib().dexel_upload_halo(self.h, side, _ptr(off), _ptr(ep) if n else None, nrows, n,
                                       1 if _is_dev(off) else 0))

    def download_rows(self, row_begin: int, nrows: int, device: bool = False):
        """local rows [row_begin, row_begin+nrows) as a CSR slice (offsets rebased to 0)."""
        L = lib()
        n = ctypes.c_uint64()
        _check(L.dexel_download_rows(self.h, row_begin, nrows, None, None, 0, ctypes.byref(n), 0))
        nc = nrows * self.desc.nx
        if device:
            import torch
            dev = torch.device("cuda", self.desc.device)
            off = torch.empty(nc + 1, dtype=torch.int64, device=dev)
            ep = torch.empty(max(2 * n.value, 2), dtype=torch.float32, device=dev)
            _check(L.dexel_download_rows(self.h, row_begin, nrows, off.data_ptr(), ep.data_ptr(), n.value,
                                         ctypes.byref(n), 1))
            return off, ep[:2 * n.value]
        off = np.empty(nc + 1, dtype=np.uint64)
        ep = np.empty(max(2 * n.value, 2), dtype=np.float32)
        _check(L.dexel_download_rows(self.h, row_begin, nrows, off.ctypes.data, ep.ctypes.data, n.value,
                                     ctypes.byref(n), 0))
        return off, ep[:2 * n.value]

    def stats(self) -> dict:
        s = dexel_stats()
        _check(lib().dexel_last_stats(self.h, ctypes.byref(s)))
        return dict(n_in=s.n_in, n_mid=s.n_mid, n_lev=s.n_lev, n_out=s.n_out, launches=s.launches,
                    kernel_calls=dict(zip(KERNEL_NAMES, list(s.kernel_calls))),
                    kernel_ms=dict(zip(KERNEL_NAMES, list(s.kernel_ms))),
                    capacities=dict(lev_cap=s.lev_cap, p2_acc=s.p2_acc, bands=s.bands))

    def sync(self):
        _check(lib().dexel_sync(self.h))

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().dexel_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class Pipe:
    """Host-to-host ops streamed in y-slabs (dexel_pipe_*): upload, op and download overlap."""

    OPS = {"dilate": 0, "erode": 1, "shell": 2}

    def __init__(self, nx: int, ny: int, z_lo: float, z_hi: float, nslabs: int = 4, z_ref: float = 0.0,
                 spacing: float = 1.0, device: int = 0):
        self.desc = dexel_desc(nx, ny, spacing, z_ref, z_lo, z_hi, device, None, None, 0, 1, 0, ny)
        h = ctypes.c_void_p()
        _check(lib().dexel_pipe_create(ctypes.byref(self.desc), nslabs, ctypes.byref(h)))
        self.h = h

    @staticmethod
    def suggest_slabs(nx: int, ny: int, r: float, spacing: float = 1.0) -> int:
        d = dexel_desc(nx, ny, spacing, 0.0, 0.0, 1.0, 0, None, None, 0, 1, 0, ny)
        return int(lib().dexel_pipe_suggest_slabs(ctypes.byref(d), r))

    def run(self, op: str, r_a: float, r_b: float, off, ep, out_off, out_ep) -> int:
        """host CSR (off, ep) -> host CSR written into (out_off, out_ep); returns the interval count.
        Arrays are numpy or CPU torch tensors (uint64/int64 offsets, float32 endpoints)."""
        cap = (out_ep.size if isinstance(out_ep, np.ndarray) else out_ep.numel()) // 2
        n = ctypes.c_uint64()
        _check(lib().dexel_pipe_run(self.h, self.OPS[op], r_a, r_b, _ptr(off), _ptr(ep), _ptr(out_off),
                                    _ptr(out_ep), cap, ctypes.byref(n)))
        return n.value

    def slab_rows(self, q: int):
        a, b = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().dexel_pipe_slab_rows(self.h, q, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def last_bytes(self):
        """(host -> device, device -> host) bytes the last run copied"""
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().dexel_pipe_last_bytes(self.h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().dexel_pipe_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (ncclGetUniqueId) for dexel_nccl_comm_init; broadcast it to every rank."""
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().dexel_nccl_unique_id(buf))
    return bytes(buf)


def nccl_comm_init(uid: bytes, nranks: int, rank: int, device: int) -> int:
    """ncclCommInitRank through the library (collective): the ncclComm_t for Grid(..., nccl_comm=)."""
    if len(uid) != 128:
        raise ValueError("NCCL unique id must be 128 bytes")
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    c = ctypes.c_void_p()
    _check(lib().dexel_nccl_comm_init(buf, int(nranks), int(rank), int(device), ctypes.byref(c)))
    return c.value


def nccl_comm_destroy(comm: Optional[int]) -> None:
    _check(lib().dexel_nccl_comm_destroy(comm))


def link_slabs(slabs) -> None:
    """Loopback halo transport (dexel_link_slabs): slab handles of rank 0..n-1 of one process fetch
    their halo rows from each other inside every op."""
    arr = (ctypes.c_void_p * len(slabs))(*[g.h.value for g in slabs])
    _check(lib().dexel_link_slabs(arr, len(slabs)))


def set_timing(on: bool):
    """per-kernel CUDA-event timing inside the library (dexel_set_timing)."""
    _check(lib().dexel_set_timing(1 if on else 0))


# ---------------------------------------------------------------- operations (same names as the C ABI)
def dexel_dilate(src: Grid, r: float, dst: Grid) -> Grid:
    _check(lib().dexel_dilate(src.h, float(r), dst.h))
    return dst


def dexel_erode(src: Grid, r: float, dst: Grid) -> Grid:
    _check(lib().dexel_erode(src.h, float(r), dst.h))
    return dst


def dexel_shell(src: Grid, r_out: float, r_in: float, dst: Grid) -> Grid:
    _check(lib().dexel_shell(src.h, float(r_out), float(r_in), dst.h))
    return dst


def dexel_dilate_slices(src: Grid, r: float, dst: Grid) -> Grid:
    """Every row on its own as a 2D slice (x, z): dst row j := D_r(src row j)."""
    _check(lib().dexel_dilate_slices(src.h, float(r), dst.h))
    return dst


def dexel_erode_slices(src: Grid, r: float, dst: Grid) -> Grid:
    """Every row on its own as a 2D slice: dst row j := E_r(src row j)."""
    _check(lib().dexel_erode_slices(src.h, float(r), dst.h))
    return dst


def dexel_shell_slices(src: Grid, r_out: float, r_in: float, dst: Grid) -> Grid:
    """Every row on its own as a 2D slice: dst row j := D_rout(row j) minus E_rin(row j)."""
    _check(lib().dexel_shell_slices(src.h, float(r_out), float(r_in), dst.h))
    return dst


def dexel_rasterize_shapes(g: Grid, zmin: float, zmax: float, sph=None, sph_sign=None, box=None, box_sign=None) -> Grid:
    """GPU dexelisation: g := (U solid spheres/boxes) minus (U void ones) on
    g's rows.  sph: float64[n,4] (cx,cy,cz,R); box: float64[m,6] (x0,x1,y0,y1,z0,z1); signs +1/-1."""
    sph = np.ascontiguousarray(np.zeros((0, 4)) if sph is None else sph, dtype=np.float64).reshape(-1, 4)
    box = np.ascontiguousarray(np.zeros((0, 6)) if box is None else box, dtype=np.float64).reshape(-1, 6)
    ss = np.ascontiguousarray(np.ones(len(sph)) if sph_sign is None else sph_sign, dtype=np.int32)
    bs = np.ascontiguousarray(np.ones(len(box)) if box_sign is None else box_sign, dtype=np.int32)
    _check(lib().dexel_rasterize_shapes(g.h, float(zmin), float(zmax), len(sph), sph.ctypes.data if len(sph) else None,
                                        ss.ctypes.data if len(ss) else None, len(box),
                                        box.ctypes.data if len(box) else None, bs.ctypes.data if len(bs) else None, 0))
    return g


def dexel_rasterize_gyroid(g: Grid, zmin: float, zmax: float, period: float = 64.0, t: float = 0.2,
                           amp: float = 0.05, seed: int = 0) -> Grid:
    """GPU dexelisation of the noisy gyroid (config C3): g := {F + eps > t} on g's
    rows, bitwise the host generator dexelgen.gyroid with the same (period, t, amp, seed)."""
    _check(lib().dexel_rasterize_gyroid(g.h, float(zmin), float(zmax), float(period), float(t), float(amp),
                                        int(seed) & 0xFFFFFFFFFFFFFFFF))
    return g


def trim_workspace(device: int = 0) -> None:
    """Free the device's idle op workspace (kept for reuse by later ops otherwise)."""
    _check(lib().dexel_trim_workspace(int(device)))


def dexel_pass1(src: Grid, r: float, complement: bool = False):
    """S_Mid pieces of pass 1 -> (offsets uint64[ncol+1], z float32[2m], kappa uint8[m]) on the host."""
    L = lib()
    m = ctypes.c_uint64()
    st = L.dexel_pass1(src.h, float(r), int(complement), None, None, None, 0, ctypes.byref(m), 0)
    if st not in (DEXEL_OK, DEXEL_EOVERFLOW):
        _check(st)
    off = np.empty(src.ncol + 1, dtype=np.uint64)
    z = np.empty(max(2 * m.value, 2), dtype=np.float32)
    k = np.empty(max(m.value, 1), dtype=np.uint8)
    _check(L.dexel_pass1(src.h, float(r), int(complement), off.ctypes.data, z.ctypes.data, k.ctypes.data,
                         m.value, ctypes.byref(m), 0))
    return off, z[:2 * m.value], k[:m.value]


def dexel_open(src: Grid, r: float, dst: Grid) -> Grid:
    """dst := D_r(E_r(src)) (opening)."""
    _check(lib().dexel_open(src.h, float(r), dst.h))
    return dst


def dexel_close(src: Grid, r: float, dst: Grid) -> Grid:
    """dst := E_r(D_r(src)) (closing)."""
    _check(lib().dexel_close(src.h, float(r), dst.h))
    return dst


def clean(src: Grid, r: float, dst: Grid, order: str = "open-close") -> Grid:
    """Topological cleaning (fig. cleaning): an opening followed by a
    closing ("open-close", removes thin features then fills thin gaps) or the reverse."""
    tmp = Grid.like(src)
    try:
        if order == "open-close":
            dexel_open(src, r, tmp)
            dexel_close(tmp, r, dst)
        else:
            dexel_close(src, r, tmp)
            dexel_open(tmp, r, dst)
    finally:
        tmp.close()
    return dst


dilate, erode, shell, pass1 = dexel_dilate, dexel_erode, dexel_shell, dexel_pass1
opening, closing = dexel_open, dexel_close
