#!/usr/bin/env python
"""bench.py -- dexel columns/s of the separable dexel offset on B200.

Contract:
  python bench.py --gpus N --steps K --warmup W [--impl b200|reference]
prints ONE JSON line on rank 0.  A step = one pass of the whole hot path
(pass 1 with complement-on-load, level sets, pass 2 with the shell epilogue)
over the workload, default BASELINE.json configs[4] (C5: 4096^2, shell =
dilate r=16 minus erode r=16) -- the config the 1/2/4/8-GPU metric is quoted
on.  `--config C4 --op dilate --r 16` selects the 2048^2 dilation workload.

value        output columns / s, whole job, inputs resident in HBM
e2e          same metric through the C ABI with pinned HOST buffers: H2D of
             the input CSR + op + D2H of the result inside the timed region
roofline     dominant kernel: algorithmic bytes / its CUDA-event time, vs
             MEASURED_PEAKS.json hbm_gbs
cpu_baseline the fp64 oracle (O2, as it stands) on a bounded band of rows of
             the same workload, on this host's cores
--impl reference   times that oracle arm alone (the base contract's reference arm)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

DEFAULT_R = {"C1": 3.0, "C2": 4.0, "C3": 8.0, "C4": 16.0, "C5": 16.0}
DEFAULT_OP = {"C1": "dilate", "C2": "shell", "C3": "dilate", "C4": "dilate", "C5": "shell"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--op", default=None, choices=[None, "dilate", "erode", "shell", "dilate_slices", "erode_slices",
                                                   "shell_slices", "rasterize", "tridexel_dilate", "tridexel_erode",
                                                   "tridexel_shell"])
    ap.add_argument("--r", type=float, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-slabs", type=int, default=-1,
                    help="y-slabs of the streamed host-to-host op (dexel_pipe_run) the e2e number is measured "
                         "with at N=1; -1: the library's suggestion (dexel_pipe_suggest_slabs; 1 = serial); "
                         "0: only the serial upload + op + download")
    ap.add_argument("--cpu-rows", type=int, default=None, help="rows in the oracle band sample")
    a = ap.parse_args()
    a.op = a.op or DEFAULT_OP[a.config]
    a.r = a.r if a.r is not None else DEFAULT_R[a.config]
    return a


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ oracle arm
def oracle_band(host, op, r, rows, nthreads):
    """time the fp64 oracle O2 on a band of full rows in the middle of the grid."""
    import oracle as O
    j0 = host.ny // 2 - rows // 2
    cols = np.arange(j0 * host.nx, (j0 + rows) * host.nx, dtype=np.int64)
    if op.endswith("_slices"):   # 2D slice offsets: the oracle op on each row's one-row grid
        import dexelgen as G
        base = op[:-len("_slices")]
        t = time.perf_counter()
        for j in range(j0, j0 + rows):
            o = np.asarray(host.off[j * host.nx:(j + 1) * host.nx + 1], dtype=np.uint64)
            a0, b0 = int(o[0]), int(o[-1])
            rg = G.Grid(host.nx, 1, o - np.uint64(a0), np.asarray(host.ep[2 * a0:2 * b0], dtype=np.float32),
                        host.z_lo, host.z_hi, host.z_ref, host.spacing)
            if base == "shell":
                O.shell(rg, r, r, nthreads=nthreads)
            else:
                getattr(O, base)(rg, r, nthreads=nthreads)
        return len(cols), time.perf_counter() - t
    t = time.perf_counter()
    if op == "shell":
        O.shell(host, r, r, cols=cols, nthreads=nthreads)
    elif op == "erode":
        O.erode(host, r, cols=cols, nthreads=nthreads)
    else:
        O.dilate(host, r, cols=cols, nthreads=nthreads)
    dt = time.perf_counter() - t
    return len(cols), dt


def oracle_sample(host, op, r, nthreads, budget_s=15.0, seed=1804, reps=3):
    """BASELINE.md section 3's sample: seeded random output columns (2^17 when the oracle is fast
    enough) + 16 full rows + 16 full column-lines of the workload, the fp64 oracle O2 (as it
    stands) on all host cores, median of `reps` runs.  A pilot run of 2048 random columns sizes the
    sample to about `budget_s` per run (large radii: fewer columns, rows and lines dropped first),
    so the default bench stays within minutes.  Returns (columns, median seconds, description)."""
    import oracle as O

    def run(cols):
        t = time.perf_counter()
        if op == "shell":
            O.shell(host, r, r, cols=cols, nthreads=nthreads)
        elif op == "erode":
            O.erode(host, r, cols=cols, nthreads=nthreads)
        else:
            O.dilate(host, r, cols=cols, nthreads=nthreads)
        return time.perf_counter() - t

    rs = np.random.default_rng(seed)
    pilot = rs.integers(0, host.ncol, 2048).astype(np.int64)
    rate = len(pilot) / max(run(pilot), 1e-6)
    n_cols = int(rate * budget_s)
    lines = 16 * (host.nx + host.ny)
    n_random = int(min(1 << 17, max(1 << 12, n_cols - lines if n_cols > lines + (1 << 17) // 2 else n_cols)))
    cols = [rs.integers(0, host.ncol, n_random)]
    n_rows = n_lines = 16 if n_cols >= n_random + lines else 0
    for j in rs.integers(0, host.ny, n_rows):
        cols.append(np.arange(host.nx) + int(j) * host.nx)
    for i in rs.integers(0, host.nx, n_lines):
        cols.append(np.arange(host.ny) * host.nx + int(i))
    cols = np.unique(np.concatenate(cols)).astype(np.int64)
    dt = float(np.median([run(cols) for _ in range(reps)]))
    desc = (f"O2 fp64 oracle on {len(cols)} output columns of {host.nx}x{host.ny} ({n_random} seeded random "
            f"+ {n_rows} full rows + {n_lines} full column-lines), median of {reps} runs {dt:.1f} s")
    return len(cols), dt, desc


def default_band_rows(cfg, op, r):
    # about 10-30 s of CPU work on a 16-core host (oracle O2, measured in the dev container)
    n = {"C1": 64, "C2": 64, "C3": 16, "C4": 8, "C5": 16}[cfg]
    if cfg == "C4" and r >= 32:
        n = 2
    if op and op.endswith("_slices"):   # 2D: about 2R+1 times less work per output column
        n = min(n * 16, {"C1": 64, "C2": 512, "C3": 1024, "C4": 2048, "C5": 4096}[cfg])
    return n


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def metric_name(op):
    return f"dexel columns/sec ({op}), whole job"


def run_reference(a, rank, world):
    if rank != 0:
        return
    import dexelgen as G
    host = G.config(a.config)
    cores = host_cores()
    if a.op == "rasterize":   # the host generator dexelgen.c on the whole grid
        _, host_gen, _ = raster_job(a.config, G)
        ts = []
        for it in range(a.warmup + a.steps):
            t0 = time.perf_counter()
            host_gen(cores)
            if it >= a.warmup:
                ts.append(time.perf_counter() - t0)
        tot = sum(ts)
        v = host.ncol * len(ts) / tot
        print(json.dumps({"impl": "reference", "metric": metric_name(a.op), "value": v, "unit": "columns/s",
                          "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000 * tot / len(ts),
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic (seeded generator, DESIGN.md input recipe)",
                          "config": {"workload": f"{a.config} rasterize", "grid": f"{host.nx}x{host.ny}"},
                          "cpu_baseline": {"kind": "oracle", "cores": cores, "value": v,
                                           "sample": "host generator dexelgen.c on the whole grid per step"},
                          "e2e": {"value": v, "unit": "columns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
              flush=True)
        return
    rows = a.cpu_rows or max(1, default_band_rows(a.config, a.op, a.r) // 4)
    for _ in range(a.warmup):
        oracle_band(host, a.op, a.r, rows, cores)
    ts, ncols = [], 0
    for _ in range(a.steps):
        ncols, dt = oracle_band(host, a.op, a.r, rows, cores)
        ts.append(dt)
    tot = sum(ts)
    v = ncols * len(ts) / tot
    sample = f"{rows} full rows ({ncols} output columns) from the middle of {a.config} per step"
    line = {"impl": "reference", "metric": metric_name(a.op), "value": v, "unit": "columns/s",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000 * tot / len(ts),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, DESIGN.md input recipe)",
            "config": {"workload": f"{a.config} {a.op} r={a.r}", "grid": f"{host.nx}x{host.ny}", "r": a.r,
                       "op": a.op, "sample": sample},
            "cpu_baseline": {"value": v, "unit": "columns/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "columns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def raster_job(config, G, dx=None):
    """rasterize of a config's solid: (GPU step on a grid, the host generator
    dexelgen.c on the whole grid with `cores` threads, host->device bytes per GPU step).  C3 is
    the noisy gyroid (dexel_rasterize_gyroid, its parameters only cross), the others the analytic
    spheres and boxes (dexel_rasterize_shapes, the shape arrays cross)."""
    if config == "C3":
        n = G.CONFIGS["C3"]["n"]
        gp = (64.0, 0.2, 0.05, G.SEED_BASE + 3)
        return (lambda g: dx.dexel_rasterize_gyroid(g, 0.0, float(n), *gp),
                lambda cores: G.gyroid(n, *gp, nthreads=cores), 6 * 8)
    n, zmin_w, zmax_w, sph, ssg, box, bsg = G.shape_config(config)
    return (lambda g: dx.dexel_rasterize_shapes(g, zmin_w, zmax_w, sph, ssg, box, bsg),
            lambda cores: G.shapes(n, n, zmin_w, zmax_w, spheres=sph[ssg > 0], voids=sph[ssg < 0], boxes=box[bsg > 0],
                                   box_voids=box[bsg < 0], nthreads=cores),
            int(sph.nbytes + ssg.nbytes + box.nbytes + bsg.nbytes))


# ------------------------------------------------------------------ algorithmic bytes
def algorithmic_bytes(kind, st, ncol, R_list, nfam, fused=False):
    """Unique HBM bytes the method must move, per kernel kind, summed over the op's
    launches of that kind: every array the kernel must read
    or write, counted once -- re-reads (the COUNT/WRITE recomputation, halo rows,
    the two output rows that read each level list, L1/L2 re-use) are not algorithmic.
      input CSR     8 B/column offset + 8 B/interval               (n_in)
      S_Mid pieces  8 B z-pair + 1 B kappa per piece, 4 B count per column   (n_mid)
      level sets    8 B/interval (n_lev) + 2 B count per (column, level)
      output        8 B/interval (n_out) + 4 B count per column (staging), then CSR
    fused: the shell's two pass-1 families ran as one sweep (p1_dual_kernel), which reads
    the input once."""
    n_in, m, nl, n_out = st["n_in"], st["n_mid"], st["n_lev"], st["n_out"]
    off = 8 * (ncol + 1)
    lev_cnt = sum(2 * (R + 1) * ncol for R in R_list)
    if kind == "pass1":          # read the input CSR, write pieces + counts
        reads = 1 if fused else nfam
        return reads * (off + 8 * n_in) + nfam * 4 * ncol + 9 * m
    if kind == "levels":         # read pieces + counts, write level slots + counts
        return nfam * 4 * ncol + 9 * m + 8 * nl + lev_cnt
    if kind == "pass2":          # read level slots + counts, write staged output + counts
        return 8 * nl + lev_cnt + 8 * n_out + 4 * ncol
    if kind == "raster":         # (dexelisation) write the staged output + counts; shapes are KB
        return 8 * n_out + 4 * ncol
    if kind == "compact":        # read staged output + counts + offsets, write the output CSR
        return 8 * n_out + 4 * ncol + off + 8 * n_out
    return 0


# ------------------------------------------------------------------ b200 arm
def run_b200(a, rank, world, local_rank):
    import torch

    import dexelgen as G
    import paper_1804_08968_b200 as dx
    from paper_1804_08968_b200 import build as B

    if not os.path.exists(dx.LIB_PATH):
        B.build()
    torch.cuda.set_device(local_rank)
    dev = local_rank
    host = G.config(a.config)
    ncol = host.ncol
    stream = torch.cuda.Stream(device=dev)
    dist = None
    comm = None
    from paper_1804_08968_b200.slabs import Slab, check_slabs, csr_rows, nccl_bootstrap
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        # the library's own NCCL communicator: every op exchanges its halo rows inside the C ABI
        comm = nccl_bootstrap(rank, world, dev)
    R = int(np.floor(a.r))
    check_slabs(host.ny, world, R)
    slab = Slab(host, rank, world, dev, stream.cuda_stream, transport="nccl" if world > 1 else "caller", comm=comm)
    src, dst = slab.src, slab.dst
    ncol_local = src.ncol   # columns this rank writes
    # rasterize: a step dexelises the config's analytic solid into the grid
    raster = a.op == "rasterize"
    if raster:
        gpu_gen, host_gen, raster_h2d = raster_job(a.config, G, dx)
    out_grid = src if raster else dst

    def step():
        if raster:
            gpu_gen(src)
            return
        # (y-slabs: the op exchanges its R halo rows with ranks g-1 / g+1 over NCCL internally)
        slab.op(a.op, a.r)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier(device_ids=[dev])
        torch.cuda.synchronize()

    for _ in range(max(a.warmup, 3)):
        step()
    barrier()

    # ---- timed region: K steps, per-kernel CUDA events inside the library on the same stream
    # (1) the timed region proper: K steps, no per-kernel instrumentation
    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    barrier()
    e0.record(stream)
    for _ in range(a.steps):
        step()
        launches += out_grid.stats()["launches"]
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    total_ms = e0.elapsed_time(e1)
    # (2) the same K steps again with per-kernel CUDA events inside the library (launch stream),
    # for the kernel breakdown and the roofline of the dominant kernel
    dx.set_timing(True)
    kern_ms = {k: 0.0 for k in dx.KERNEL_NAMES}
    kern_calls = {k: 0 for k in dx.KERNEL_NAMES}
    barrier()
    for _ in range(a.steps):
        step()
        st = out_grid.stats()
        for k in dx.KERNEL_NAMES:
            kern_ms[k] += st["kernel_ms"][k]
            kern_calls[k] += st["kernel_calls"][k]
    barrier()
    dx.set_timing(False)
    if dist is not None:                      # max over ranks, on the device clocks of each rank
        t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / a.steps
    st = out_grid.stats()
    value = ncol / (ms / 1e3)                 # whole-grid output columns / s (all ranks)

    # ---- roofline for the dominant kernel
    peak, peak_src = peaks()
    R = int(np.floor(a.r))
    nfam = 2 if a.op.startswith("shell") else (0 if a.op == "rasterize" else 1)
    R_list = [0 if a.op.endswith("_slices") else R] * nfam   # (slices: only L_0 is built and read)
    dom = max((k for k in dx.KERNEL_NAMES if k not in ("scan", "other")), key=lambda k: kern_ms[k])
    # the library fuses the shell's pass-1 families when r_out and r_in share R <= 16
    # (DESIGN.md p1_dual_kernel; DEXEL_NO_FUSE=1 turns it off)
    fused = (a.op.startswith("shell") and R <= 16 and os.environ.get("DEXEL_NO_FUSE", "0") in ("", "0")
             and os.environ.get("DEXEL_NO_PRUNE", "0") in ("", "0"))
    byts = algorithmic_bytes(dom, st, ncol_local, R_list, nfam, fused)
    t_dom = kern_ms[dom] / a.steps / 1e3            # s per step for that kernel kind
    achieved = byts / t_dom / 1e9 if t_dom > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        key = f"{a.config}:{a.op}:{a.r}:{dom}"
        traffic = tj.get(key)
    # traffic: dram__bytes_read.sum + dram__bytes_write.sum of the same kernel kind, summed over one
    # step's launches of an ncu --set full capture (profiles/traffic.json, tools/ncu_traffic.py),
    # i.e. per step like `achieved`
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_step": byts, "kernel_ms_per_step": 1e3 * t_dom,
                "kernel_launches_per_step": kern_calls[dom] / a.steps,
                "share_of_step": (kern_ms[dom] / a.steps) / ms}

    # ---- e2e through the C ABI with pinned host buffers
    e2e = None
    if not a.no_e2e and world == 1 and raster:
        # the shapes from host arrays (copied inside the call) and the result CSR to pinned host memory
        nout_cap = int(st["n_out"] * 1.1) + 1024
        o_off = torch.empty(ncol + 1, dtype=torch.int64).pin_memory()
        o_ep = torch.empty(2 * nout_cap, dtype=torch.float32).pin_memory()
        L = dx.lib()
        ke = max(1, min(a.steps, 5))
        step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(ke):
            step()
            nout = src.size()
            dx._check(L.dexel_download(src.h, o_off.data_ptr(), o_ep.data_ptr(), nout_cap, 0))
        torch.cuda.synchronize()
        e_ms = 1e3 * (time.perf_counter() - t0) / ke
        e2e = {"value": ncol / (e_ms / 1e3), "unit": "columns/s",
               "h2d_bytes_per_step": raster_h2d,
               "d2h_bytes_per_step": 8 * (ncol + 1) + 8 * nout, "ms_per_step": e_ms}
    elif not a.no_e2e:
        # every rank: its slab's input CSR from pinned host memory, the (collective) op, its output
        # slab back to pinned host memory -- through the C ABI, timed as the max over ranks
        s_off, s_ep = csr_rows(host.off, host.ep, host.nx, slab.y0, slab.y1 - slab.y0)
        n_in_local = int(s_off[-1])
        h_off = torch.from_numpy(s_off.view(np.int64)).pin_memory()
        h_ep = torch.from_numpy(s_ep).pin_memory()
        nout_cap = int(st["n_out"] * 1.1) + 1024
        o_off = torch.empty(ncol_local + 1, dtype=torch.int64).pin_memory()
        o_ep = torch.empty(2 * nout_cap, dtype=torch.float32).pin_memory()
        L = dx.lib()
        ke = max(1, min(a.steps, 5))

        def e2e_step():
            dx._check(L.dexel_upload(src.h, h_off.data_ptr(), h_ep.data_ptr(), n_in_local, 0))
            step()
            n = dst.size()
            dx._check(L.dexel_download(dst.h, o_off.data_ptr(), o_ep.data_ptr(), nout_cap, 0))
            return n

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(ke):
            nout = e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ev_ms = e0.elapsed_time(e1) / ke
        # the library synchronises the stream around host copies, so wall-clock and events agree;
        # report the larger (host copies are stream-ordered on the same stream)
        e_ms = max(ev_ms, 1e3 * wall / ke)
        byts = [8 * (ncol_local + 1) + 8 * n_in_local, 8 * (ncol_local + 1) + 8 * nout]
        if dist is not None:
            t = torch.tensor([e_ms] + byts, dtype=torch.float64, device=f"cuda:{dev}")
            tm = t[:1].clone()
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            e_ms, byts = float(tm.item()), [int(v) for v in t[1:].tolist()]
        e2e = {"value": ncol / (e_ms / 1e3), "unit": "columns/s",
               "h2d_bytes_per_step": byts[0], "d2h_bytes_per_step": byts[1], "ms_per_step": e_ms,
               "api": "dexel_upload + op + dexel_download (serial)"}
        if a.e2e_slabs < 0:
            a.e2e_slabs = dx.Pipe.suggest_slabs(host.nx, host.ny, a.r, getattr(host, "spacing", 1.0))
            if a.e2e_slabs == 1:
                a.e2e_slabs = 0        # the library suggests no split: the serial calls are the e2e path
        if world == 1 and a.e2e_slabs > 0 and a.op in ("dilate", "erode", "shell"):
            # the streamed host-to-host call (dexel_pipe_run): the same pinned host CSRs, cut into
            # y-slabs so the upload of slab q+1, the op on slab q and the download of slab q-1 overlap;
            # each slab also uploads its R halo rows per side (counted in h2d_bytes_per_step)
            ns = min(a.e2e_slabs, host.ny)
            pipe = dx.Pipe(host.nx, host.ny, host.z_lo, host.z_hi, ns, getattr(host, "z_ref", 0.0),
                           getattr(host, "spacing", 1.0), dev)
            r_b = a.r if a.op == "shell" else 0.0
            for _ in range(max(a.warmup, 3)):     # (every slab handle settles its capacities in its first ops)
                pipe.run(a.op, a.r, r_b, h_off, h_ep, o_off, o_ep)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(ke):
                nout_p = pipe.run(a.op, a.r, r_b, h_off, h_ep, o_off, o_ep)
            p_ms = 1e3 * (time.perf_counter() - t0) / ke     # (the call returns when the host CSR is complete)
            p_h2d, p_d2h = pipe.last_bytes()       # counted by the library from the copies it made
            slab_rows = [pipe.slab_rows(q) for q in range(ns)]
            pipe.close()
            assert nout_p == nout, (nout_p, nout)
            serial = e2e
            e2e = {"value": ncol / (p_ms / 1e3), "unit": "columns/s",
                   "h2d_bytes_per_step": p_h2d, "d2h_bytes_per_step": p_d2h,
                   "ms_per_step": p_ms, "api": f"dexel_pipe_run, {ns} y-slabs (upload / op / download overlapped)",
                   "slab_rows": slab_rows, "serial": serial}

    # ---- cpu baseline (rank 0, N=1 only)
    cpu = None
    if not a.no_cpu and rank == 0 and world == 1 and raster:
        cores = host_cores()
        t0 = time.perf_counter()
        host_gen(cores)
        dt = time.perf_counter() - t0
        cpu = {"value": ncol / dt, "unit": "columns/s", "cores": cores, "kind": "oracle",
               "sample": f"the host generator dexelgen.c (fp64 per-column CSG, the definition the GPU path is "
                         f"tested bitwise against) on the whole {a.config} grid, {dt:.1f} s"}
    elif not a.no_cpu and rank == 0 and world == 1:
        cores = host_cores()
        if a.op.endswith("_slices") or a.cpu_rows:
            rows = a.cpu_rows or default_band_rows(a.config, a.op, a.r)
            ncols_s, dt = oracle_band(host, a.op, a.r, rows, cores)
            desc = (f"O2 fp64 oracle on {rows} full rows ({ncols_s} output columns) from the middle of "
                    f"{a.config}, {dt:.1f} s")
        else:   # >= 2^17 random columns + 16 rows + 16 column-lines, median of 3
            ncols_s, dt, desc = oracle_sample(host, a.op, a.r, cores)
        cpu = {"value": ncols_s / dt, "unit": "columns/s", "cores": cores, "kind": "oracle", "sample": desc}

    line = {
        "metric": metric_name(a.op), "value": value, "unit": "columns/s", "n_gpus": world, "steps": a.steps,
        "warmup": max(a.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded generator, DESIGN.md input recipe)",
        "config": {"workload": f"{a.config} {a.op} r={a.r}", "grid": f"{host.nx}x{host.ny}", "r": a.r,
                   "op": a.op, "n_in": int(st["n_in"]), "n_mid": int(st["n_mid"]), "n_lev": int(st["n_lev"]),
                   "n_out": int(st["n_out"]), "capacities": st.get("capacities"),
                   "parallelism": f"y-slabs x{world}",
                   "l2": f"inputs larger than L2 ({8 * host.n / 2**20:.0f} MiB endpoints + intermediates)"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "gpu_launches_per_step": launches / a.steps, "clocks": clk,
        "kernel_ms_per_step": {k: v / a.steps for k, v in kern_ms.items()},
        "gpu": torch.cuda.get_device_name(dev),
    }
    if world > 1:
        line["config"]["slab_rows"] = [slab.y0, slab.y1]
        line["config"]["halo_rows"] = R
    if world > 1:
        line["config"]["halo"] = "in-library NCCL send/recv (dexel_nccl_comm_init), overlapped with interior pass 1"
    if rank == 0:
        print(json.dumps(line), flush=True)
    slab.close()
    if comm:
        torch.cuda.synchronize()
        dx.nccl_comm_destroy(comm)
    if dist is not None:
        dist.destroy_process_group()


def run_tridexel(a, rank, world):
    """Tri-dexel offsets: the config's solid rasterised into three axis buffers
    (setup, untimed); a step = the op on all three buffers (one stream, CUDA events).  Replicas
    only: under torchrun every rank runs its own copy and rank 0 reports its own time."""
    import torch

    import dexelgen as G
    import paper_1804_08968_b200 as dx
    from paper_1804_08968_b200.tridexel import AXES, TriDexel
    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    n, zmin, zmax, sph, ssg, box, bsg = G.shape_config(a.config)
    td = TriDexel.from_shapes(n, zmin, zmax, sph, ssg, box, bsg, device=dev, stream=stream.cuda_stream)
    out = td.like()
    op = a.op[len("tridexel_"):]

    def step():
        if op == "shell":
            td.shell(a.r, a.r, out)
        else:
            getattr(td, op)(a.r, out)

    for _ in range(max(a.warmup, 3)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    launches = 0
    for _ in range(a.steps):
        step()
        launches += sum(out.buf[x].stats()["launches"] for x in AXES)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / a.steps
    ncol = 3 * n * n
    line = {"metric": metric_name(a.op), "value": ncol / (ms / 1e3), "unit": "columns/s", "n_gpus": 1,
            "steps": a.steps, "warmup": max(a.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "replicas", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generator, rasterised on the GPU into three axis buffers)",
            "config": {"workload": f"{a.config} {a.op} r={a.r}", "grid": f"3 x {n}x{n}", "r": a.r,
                       "n_in": int(td.size()), "n_out": int(out.size())},
            "roofline": None, "cpu_baseline": None, "e2e": None, "gpu_launches": launches,
            "clocks": clk, "gpu": torch.cuda.get_device_name(dev)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    td.close()
    out.close()


def spawn_ranks(a):
    """--gpus N > 1 without a launcher: re-exec this command under torchrun with N ranks (one per
    GPU), or fail loudly when the box has fewer GPUs -- never bench one GPU as N."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < a.gpus:
        print(json.dumps({"error": f"--gpus {a.gpus} requested but this box has {have} CUDA device(s)"}), flush=True)
        sys.stderr.write(f"bench.py: --gpus {a.gpus} needs {a.gpus} GPUs, found {have}\n")
        sys.exit(2)
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    os.environ.setdefault("NCCL_DEBUG", "INFO")          # the NCCL init log shows all N ranks
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "b200" and "WORLD_SIZE" not in os.environ and a.gpus > 1:
        spawn_ranks(a)
    if a.impl == "b200" and world > 1 and a.gpus != world:
        sys.exit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")
    if a.impl == "reference":
        run_reference(a, rank, world)
    elif a.op.startswith("tridexel_"):
        run_tridexel(a, rank, world)
    else:
        run_b200(a, rank, world, local_rank)


if __name__ == "__main__":
    main()
