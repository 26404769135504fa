"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bars:
  * pass-1 pieces (selection only): bitwise equal to the oracle's P1;
  * dilate / erode / shell: identical per-column interval counts after merging
    gaps < tau and dropping slivers < tau, endpoints within tau, with
    tau = 1e-4 x spacing (BASELINE.json north_star).
Small cases compare every column; the big configs C3-C5 compare seeded
samples of columns (random columns + full rows + full column-lines + the
first and last rows), in the same launch configuration bench.py times.
"""
import numpy as np
import pytest

import dexelgen as G
import oracle as O
from oracle.compare import compare, describe

from tests._util import sample_columns, take_columns

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


def run_gpu(dx, host, op, r, r2=None):
    src = dx.Grid.from_host(host)
    dst = dx.Grid.like(src)
    if op == "dilate":
        dx.dexel_dilate(src, r, dst)
    elif op == "erode":
        dx.dexel_erode(src, r, dst)
    else:
        dx.dexel_shell(src, r, r if r2 is None else r2, dst)
    off, ep = dst.download()
    st = dst.stats()
    src.close()
    dst.close()
    return off, ep, st


def run_oracle(host, op, r, r2=None, cols=None):
    if op == "shell":
        return O.shell(host, r, r if r2 is None else r2, cols=cols)
    return getattr(O, op)(host, r, cols=cols)


# parity summary per (config, op, r) for BASELINE.md section 3 (written when DEXEL_PARITY_REPORT names
# a file: max endpoint error, count mismatches, columns compared)
REPORT = {}


@pytest.fixture(scope="module", autouse=True)
def _parity_report():
    yield
    import json
    import os
    path = os.environ.get("DEXEL_PARITY_REPORT")
    if path and REPORT:
        old = {}
        if os.path.exists(path):
            with open(path) as f:
                old = json.load(f)
        old.update(REPORT)
        with open(path, "w") as f:
            json.dump(old, f, indent=1, sort_keys=True)


def check(off, ep, ref, cols=None, what=""):
    if cols is not None:
        off, ep = take_columns(off, ep, cols)
    res = compare(off, ep, ref.off, ref.z, TAU)
    REPORT[what] = dict(max_err=res["max_err"], count_mismatch=res["count_mismatch"],
                        endpoint_fail=res["endpoint_fail"], columns=int(len(ref.off) - 1), n=res["n_b"])
    if not res["ok"]:
        c = res["first_bad"]
        raise AssertionError(f"{what}: {res}\n" + describe(off, ep, ref.off, ref.z, c))
    return res


# ------------------------------------------------------------------ pass 1 (bitwise)
@pytest.mark.parametrize("seed", range(40))
def test_pass1_bitwise_random(dx, seed):
    rs = np.random.default_rng(seed)
    nx, ny = int(rs.integers(1, 80)), int(rs.integers(1, 6))
    host = G.random_grid(nx, ny, 4, -16.0, 16.0, seed, quantum=0.5 if seed % 2 else None)
    r = float(rs.choice([0.0, 0.7, 1.0, 2.5, 4.0, 9.0, 16.0, 17.0, 33.0, 40.5, 64.0, 100.0, 200.0]))
    src = dx.Grid.from_host(host)
    for comp in (False, True):
        off, z, k = dx.dexel_pass1(src, r, comp)
        ref = O.pass1(host, r, complement=comp)
        assert np.array_equal(off, ref.off), (r, comp)
        assert np.array_equal(z.astype(np.float64), ref.z), (r, comp)
        assert np.array_equal(k, ref.k), (r, comp)


@pytest.mark.parametrize("name,r", [("C1", 3.0), ("C2", 4.0)])
def test_pass1_bitwise_configs(dx, name, r):
    host = G.config(name)
    src = dx.Grid.from_host(host)
    for comp in (False, True):
        off, z, k = dx.dexel_pass1(src, r, comp)
        ref = O.pass1(host, r, complement=comp)
        assert np.array_equal(off, ref.off) and np.array_equal(z.astype(np.float64), ref.z) \
            and np.array_equal(k, ref.k)


def test_pass1_bitwise_c3_rows(dx):
    host = G.config("C3")
    src = dx.Grid.from_host(host)
    off, z, k = dx.dexel_pass1(src, 8.0)
    cols = sample_columns(host.nx, host.ny, 4096, 3, 0, 33, extra_rows=(0, host.ny - 1))
    ref = O.pass1(host, 8.0, cols=cols)
    o2, z2 = take_columns(off, z, cols)
    assert np.array_equal(o2, ref.off) and np.array_equal(z2, ref.z)
    kk = np.concatenate([k[int(off[c]):int(off[c + 1])] for c in cols])
    assert np.array_equal(kk, ref.k)


# ------------------------------------------------------------------ ops, small grids, all columns
@pytest.mark.parametrize("seed", range(60))
def test_ops_random_small(dx, seed):
    rs = np.random.default_rng(1000 + seed)
    nx, ny = int(rs.integers(1, 40)), int(rs.integers(1, 40))
    host = G.random_grid(nx, ny, 4, -12.0, 12.0, seed, quantum=0.25 if seed % 3 == 0 else None)
    r = float(rs.choice([0.0, 0.3, 1.0, 1.5, 2.0, 3.0, 4.0, 5.5, 8.0, 12.0, 20.0]))
    for op in ("dilate", "erode", "shell"):
        off, ep, _ = run_gpu(dx, host, op, r, r * 0.75 if op == "shell" else None)
        ref = run_oracle(host, op, r, r * 0.75 if op == "shell" else None)
        check(off, ep, ref, what=f"{op} r={r} seed={seed}")


@pytest.mark.parametrize("name,r", [("C1", 3.0), ("C2", 4.0)])
def test_configs_all_columns(dx, name, r):
    host = G.config(name)
    for op in G.CONFIGS[name]["op"]:
        off, ep, _ = run_gpu(dx, host, op, r)
        check(off, ep, run_oracle(host, op, r), what=f"{name} {op} r={r}")


# ------------------------------------------------------------------ big configs, sampled columns
def sampled(dx, name, op, r, n_random=4096, n_rows=2, n_lines=2, seed=7):
    host = G.config(name)
    off, ep, st = run_gpu(dx, host, op, r)
    cols = sample_columns(host.nx, host.ny, n_random, n_rows, n_lines, seed, extra_rows=(0, host.ny - 1))
    ref = run_oracle(host, op, r, cols=cols)
    return check(off, ep, ref, cols, what=f"{name} {op} r={r}")


@pytest.mark.parametrize("op", ["dilate", "erode"])
def test_c3_sampled(dx, op):
    sampled(dx, "C3", op, 8.0)


@pytest.mark.parametrize("r", [1.0, 2.0, 4.0, 8.0, 16.0, 32.0, 64.0])
def test_c4_sampled(dx, r):
    sampled(dx, "C4", "dilate", r, n_random=2048 if r >= 32 else 4096, n_lines=1)


@pytest.mark.slow
def test_c5_shell_sampled(dx):
    sampled(dx, "C5", "shell", 16.0, n_random=2048, n_rows=1, n_lines=1)


# ------------------------------------------------------------------ edge cases
def _grid(nx, ny, cols, lo=-8.0, hi=8.0):
    return G.from_columns(nx, ny, [np.array(c, np.float32).reshape(-1, 2) for c in cols], lo, hi)


@pytest.mark.parametrize("op", ["dilate", "erode", "shell"])
def test_edge_cases(dx, op):
    cases = [
        _grid(6, 5, [[]] * 30),                                   # empty
        _grid(6, 5, [[(-8.0, 8.0)]] * 30),                        # full domain
        _grid(1, 1, [[(-1.0, 2.0), (3.0, 4.0)]]),                 # single column
        _grid(7, 3, [[(-8.0, -7.0), (7.5, 8.0)]] * 21),           # touching z_lo / z_hi
        _grid(5, 5, [[(0.0, 1.0)] if (i + j) % 2 else [(1.0, 2.0)] for j in range(5) for i in range(5)]),  # touching neighbours
        _grid(40, 2, [[(float(i % 7) - 4, float(i % 7) - 3.5)] for i in range(80)]),
    ]
    for host in cases:
        for r in (0.0, 0.5, 1.0, 2.0, 7.0, 45.0):                 # r = 0, 0<r<1, r > grid size
            off, ep, _ = run_gpu(dx, host, op, r)
            check(off, ep, run_oracle(host, op, r), what=f"edge {op} r={r} {host.nx}x{host.ny}")


def test_errors(dx):
    host = _grid(4, 4, [[(0.0, 1.0)]] * 16)
    src = dx.Grid.from_host(host)
    dst = dx.Grid.like(src)
    with pytest.raises(dx.DexelError) as e:
        dx.dexel_dilate(src, -1.0, dst)
    assert e.value.status == dx.DEXEL_EINVAL
    with pytest.raises(dx.DexelError) as e:
        dx.dexel_dilate(src, 300.0, dst)                          # R > 255
    assert e.value.status == dx.DEXEL_EINVAL
    with pytest.raises(dx.DexelError) as e:
        dx.dexel_dilate(src, float("nan"), dst)
    assert e.value.status == dx.DEXEL_EINVAL
    with pytest.raises(dx.DexelError) as e:
        dx.dexel_dilate(src, 1.0, src)
    assert e.value.status == dx.DEXEL_EINVAL
    other = dx.Grid(5, 4, -8.0, 8.0)
    with pytest.raises(dx.DexelError) as e:
        dx.dexel_dilate(src, 1.0, other)
    assert e.value.status == dx.DEXEL_EMISMATCH
    # corrupt inputs: unsorted, NaN, out of domain, zero length -> EINVAL, grid unchanged
    before = src.download()
    for bad in ([(1.0, 0.5)], [(0.0, float("nan"))], [(0.0, 9.0)], [(0.0, 1.0), (0.5, 2.0)], [(1.0, 1.0)]):
        cols = [[(0.0, 1.0)]] * 15 + [bad]
        g = _grid(4, 4, [[]] * 16)
        off = np.zeros(17, np.uint64)
        np.cumsum([len(c) for c in cols], out=off[1:])
        ep = np.array([v for c in cols for iv in c for v in iv], np.float32)
        with pytest.raises(dx.DexelError) as e:
            src.upload(off, ep)
        assert e.value.status == dx.DEXEL_EINVAL and "column 15" in str(e.value)
    after = src.download()
    assert np.array_equal(before[0], after[0]) and np.array_equal(before[1], after[1])
    # capacity too small
    dx.dexel_dilate(src, 1.0, dst)
    n = dst.size()
    from paper_1804_08968_b200 import lib
    offb = np.empty(17, np.uint64)
    epb = np.empty(2 * n, np.float32)
    assert lib().dexel_download(dst.h, offb.ctypes.data, epb.ctypes.data, n - 1, 0) == dx.DEXEL_EOVERFLOW


def test_deterministic(dx):
    host = G.config("C2")
    a = run_gpu(dx, host, "shell", 4.0)
    b = run_gpu(dx, host, "shell", 4.0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_device_buffers_roundtrip(dx):
    import torch
    host = G.config("C1")
    off = torch.from_numpy(host.off.astype(np.int64)).cuda()
    ep = torch.from_numpy(host.ep).cuda()
    src = dx.Grid(host.nx, host.ny, host.z_lo, host.z_hi)
    src.upload(off, ep)
    o2, e2 = src.download(device=True)
    assert torch.equal(o2.cpu(), off.cpu()) and torch.equal(e2.cpu(), ep.cpu())


def test_torch_allocator_hook(dx):
    dx.use_torch_allocator(True)
    try:
        host = G.config("C1")
        off, ep, _ = run_gpu(dx, host, "dilate", 3.0)
        check(off, ep, run_oracle(host, "dilate", 3.0), what="torch allocator")
    finally:
        dx.use_torch_allocator(False)



def test_pass2_accumulator_fitted_to_the_handle(dx):
    """The pass-2 accumulator follows the longest union any op on the handle held (a multiple of 4,
    at least 8; default 32 for the first op): the fitted ops give bitwise the first op's result,
    the capacity never falls when ops alternate, and an op that needs more than the fitted
    capacity (a larger radius after a small one: more merged lists, then a many-layer input
    uploaded into the same handle) reruns and still matches the oracle."""
    host = G.random_grid(64, 40, 4, -16.0, 16.0, seed=31)
    src = dx.Grid.from_host(host)
    dst = dx.Grid.like(src)
    dx.dexel_dilate(src, 2.0, dst)
    first, cap0 = dst.download(), dst.stats()["capacities"]["p2_acc"]
    dx.dexel_dilate(src, 2.0, dst)
    again, cap1 = dst.download(), dst.stats()["capacities"]["p2_acc"]
    assert cap0 == 32 and 8 <= cap1 <= 32 and cap1 % 4 == 0
    assert np.array_equal(first[0], again[0]) and np.array_equal(first[1], again[1])
    caps = []
    for r in (0.5, 6.0, 0.5, 6.0, 0.5):                       # alternating ops on one handle
        dx.dexel_shell(src, r, r, dst)
        off, ep = dst.download()
        check(off, ep, run_oracle(host, "shell", r), what=f"fitted accumulator shell r={r}")
        caps.append(dst.stats()["capacities"]["p2_acc"])
    assert caps[2:] == sorted(caps[2:]) and caps[4] == caps[3]  # settled at the handle's maximum
    # a column-rich input into the same handle: unions far longer than the fitted capacity
    rs = np.random.default_rng(5)
    cols = []
    for c in range(64 * 40):
        k = 60 if c % 7 == 0 else 2
        z = np.sort(rs.uniform(-15.5, 15.5, 2 * k)).astype(np.float32)
        z = z[: 2 * (len(np.unique(z)) // 2)]
        cols.append(np.unique(z).reshape(-1, 2) if len(np.unique(z)) == len(z) else np.zeros((0, 2), np.float32))
    off = np.zeros(64 * 40 + 1, np.uint64)
    np.cumsum([len(c) for c in cols], out=off[1:])
    ep = np.concatenate([c.reshape(-1) for c in cols]).astype(np.float32)
    rich = G.Grid(64, 40, off, ep, host.z_lo, host.z_hi)
    src.upload(off, ep)
    dx.dexel_dilate(src, 0.05, dst)
    o2, e2 = dst.download()
    check(o2, e2, run_oracle(rich, "dilate", 0.05), what="fitted accumulator, many-layer input")
    assert dst.stats()["capacities"]["p2_acc"] > caps[-1]
    src.close()
    dst.close()


@pytest.mark.parametrize("lev_cap,acc,band,p1cap", [("1", "1", "3", "1"), ("2", "4", "7", "6")])
def test_capacity_regrowth(dx, lev_cap, acc, band, p1cap):
    """Start every capacity at its minimum (level slots per list, pass-2 accumulator:
    DEXEL_LEV_CAP / DEXEL_P2_ACC) so every op overflows and reruns with grown
    capacities, and cut the grid into 3-row bands (DEXEL_BAND_ROWS); results still
    match the oracle.  Subprocess: the hints are read when a handle is created."""
    import os
    import subprocess
    import sys
    code = r'''
import sys; sys.path.insert(0, %r)
import numpy as np, dexelgen as G, oracle as O, paper_1804_08968_b200 as dx
from oracle.compare import compare
for seed in range(12):
    rs = np.random.default_rng(77 + seed)
    host = G.random_grid(int(rs.integers(2, 40)), int(rs.integers(2, 30)), 6, -12.0, 12.0, seed)
    r = float(rs.choice([1.0, 2.5, 4.0, 7.0, 16.0, 20.0, 40.0]))
    src = dx.Grid.from_host(host); dst = dx.Grid.like(src)
    for op in ("dilate", "erode", "shell"):
        if op == "shell":
            dx.dexel_shell(src, r, r, dst); ref = O.shell(host, r, r)
        else:
            getattr(dx, "dexel_" + op)(src, r, dst); ref = getattr(O, op)(host, r)
        off, ep = dst.download()
        res = compare(off, ep, ref.off, ref.z, 1e-4); assert res["ok"], (op, r, res)
print("OK")
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DEXEL_LEV_CAP=lev_cap, DEXEL_P2_ACC=acc, DEXEL_BAND_ROWS=band, DEXEL_P1_CAP=p1cap)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "OK" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("op", ["dilate", "erode", "shell"])
def test_many_intervals_fallback(dx, op):
    """Columns whose level sets and unions hold more intervals than the default
    capacities (8 per level list, 24 per pass-2 union) make the op rerun with grown
    capacities; results still match the oracle."""
    col = [(float(t) * 0.5 - 40.0, float(t) * 0.5 - 39.8) for t in range(120)]   # 120 thin layers
    cols = [col if (i + j) % 3 == 0 else [] for j in range(4) for i in range(5)]
    host = _grid(5, 4, cols, -41.0, 41.0)
    for r in (0.05, 1.2):
        off, ep, _ = run_gpu(dx, host, op, r)
        check(off, ep, run_oracle(host, op, r), what=f"many-intervals {op} r={r}")


def test_pass1_bitwise_unstaged_windows(dx):
    """Windows with more endpoints than the shared-memory staging area (2048 keys per warp)
    take the global-memory path of the pass-1 sweep; pieces stay bitwise equal."""
    col = [(float(t) * 0.5 - 40.0, float(t) * 0.5 - 39.8) for t in range(120)]
    cols = [col if (i * 7 + j) % 3 else col[::2] for j in range(3) for i in range(40)]
    host = _grid(40, 3, cols, -41.0, 41.0)
    src = dx.Grid.from_host(host)
    for r in (1.0, 6.0):
        for comp in (False, True):
            off, z, k = dx.dexel_pass1(src, r, comp)
            ref = O.pass1(host, r, complement=comp)
            assert np.array_equal(off, ref.off) and np.array_equal(z.astype(np.float64), ref.z) \
                and np.array_equal(k, ref.k)


def test_pass1_bitwise_overflow_arena(dx):
    """Pass-1 pieces of columns that outgrow their slots (DEXEL_P1_CAP=2) come from the
    overflow arena (second, tile-list launch); still bitwise equal to the oracle's P1."""
    import os
    import subprocess
    import sys
    code = r'''
import sys; sys.path.insert(0, %r)
import numpy as np, dexelgen as G, oracle as O, paper_1804_08968_b200 as dx
for seed in range(10):
    rs = np.random.default_rng(900 + seed)
    host = G.random_grid(int(rs.integers(20, 70)), int(rs.integers(2, 9)), 5, -10.0, 10.0, seed,
                         quantum=0.25 if seed %% 2 else None)
    r = float(rs.choice([1.0, 3.0, 6.5, 20.0]))
    src = dx.Grid.from_host(host)
    for comp in (False, True):
        off, z, k = dx.dexel_pass1(src, r, comp)
        ref = O.pass1(host, r, complement=comp)
        assert np.array_equal(off, ref.off) and np.array_equal(z.astype(np.float64), ref.z) \
            and np.array_equal(k, ref.k), (seed, r, comp)
print("OK")
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DEXEL_P1_CAP="2")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "OK" in out.stdout, out.stdout + out.stderr


def test_capsule_pruning_is_exact(dx):
    """The pass-1 capsule-domination filter (on by default in the ops) drops pieces whose
    capsule lies inside a neighbour's at every level: results with DEXEL_NO_PRUNE=1 (every
    piece kept) and without both match the oracle, and the filtered run holds fewer pieces."""
    import os
    import subprocess
    import sys
    code = r'''
import sys; sys.path.insert(0, %r)
import numpy as np, dexelgen as G, oracle as O, paper_1804_08968_b200 as dx
from oracle.compare import compare
host = G.config("C2")
src = dx.Grid.from_host(host); dst = dx.Grid.like(src)
for op in ("dilate", "erode", "shell"):
    for r in (4.0, 9.5):
        if op == "shell":
            dx.dexel_shell(src, r, r, dst); ref = O.shell(host, r, r)
        else:
            getattr(dx, "dexel_" + op)(src, r, dst); ref = getattr(O, op)(host, r)
        off, ep = dst.download()
        res = compare(off, ep, ref.off, ref.z, 1e-4); assert res["ok"], (op, r, res)
        print(op, r, dst.stats()["n_mid"])
print("OK")
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    mids = {}
    for flag in ("0", "1"):
        env = dict(os.environ, DEXEL_NO_PRUNE=flag)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0 and "OK" in out.stdout, out.stdout + out.stderr
        mids[flag] = [int(line.split()[-1]) for line in out.stdout.splitlines() if line[:1].isalpha() and line != "OK"]
    assert all(a < b for a, b in zip(mids["0"], mids["1"])), mids


@pytest.mark.parametrize("p1cap", [None, "3"])
def test_fused_shell_pass1_is_bitwise_separate(dx, p1cap):
    """The shell's two pass-1 families in one sweep (p1_dual_kernel, used when r_out and r_in
    share R <= 16) give bitwise the output of two separate sweeps (DEXEL_NO_FUSE=1), and match
    the oracle -- also with tiny pass-1 slots (overflow columns redone per family in list mode),
    with S touching z_lo / z_hi (zero-length complement pieces) and with r_out != r_in."""
    import hashlib
    import os
    import subprocess
    import sys
    code = r"""
import sys, hashlib; sys.path.insert(0, %r)
import numpy as np, dexelgen as G, oracle as O, paper_1804_08968_b200 as dx
from oracle.compare import compare
cases = [("C2", G.config("C2"), 4.0, 4.0), ("C2", G.config("C2"), 6.5, 6.2), ("C1", G.config("C1"), 3.0, 3.0)]
rng = np.random.default_rng(7)
cols = []
for c in range(40 * 24):          # columns touching the domain ends
    k = int(rng.integers(0, 4)); pts = np.sort(rng.uniform(-8, 8, 2 * k)).astype(np.float32)
    iv = [(float(pts[2*t]), float(pts[2*t+1])) for t in range(k) if pts[2*t] < pts[2*t+1]]
    if c %% 3 == 0: iv = [(-8.0, -7.0)] + [x for x in iv if x[0] > -7.0]
    if c %% 5 == 0: iv = [x for x in iv if x[1] < 7.5] + [(7.5, 8.0)]
    cols.append(iv)
cases.append(("edge", G.from_columns(40, 24, cols, -8.0, 8.0), 5.0, 5.0))
h = hashlib.sha256()
for name, host, ro, ri in cases:
    src = dx.Grid.from_host(host); dst = dx.Grid.like(src)
    dx.dexel_shell(src, ro, ri, dst)
    off, ep = dst.download()
    h.update(np.asarray(off).tobytes()); h.update(np.asarray(ep).tobytes())
    ref = O.shell(host, ro, ri)
    res = compare(off, ep, ref.off, ref.z, 1e-4); assert res["ok"], (name, ro, ri, res)
print("HASH", h.hexdigest())
print("OK")
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hashes = {}
    for fuse in ("0", "1"):
        env = dict(os.environ, DEXEL_NO_FUSE=fuse)
        if p1cap:
            env["DEXEL_P1_CAP"] = p1cap
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0 and "OK" in out.stdout, out.stdout + out.stderr
        hashes[fuse] = [l for l in out.stdout.splitlines() if l.startswith("HASH")][0]
    assert hashes["0"] == hashes["1"], hashes


# ---------------------------------------------------------------- openings / closings (NEXT #1)
def _to_host_grid(host, res):
    """an oracle Result as an fp32 canonical input grid (touching after rounding: merged)."""
    off = np.asarray(res.off, dtype=np.int64)
    z = np.asarray(res.z, dtype=np.float64).reshape(-1, 2)
    cols = []
    for c in range(host.ncol):
        iv = z[off[c]:off[c + 1]].astype(np.float32)
        out = []
        for a, b in iv:
            if not a < b:
                continue
            if out and a <= out[-1][1]:
                out[-1][1] = max(out[-1][1], b)
            else:
                out.append([a, b])
        cols.append(np.array(out, dtype=np.float32).reshape(-1, 2))
    return G.from_columns(host.nx, host.ny, cols, host.z_lo, host.z_hi, getattr(host, "z_ref", 0.0))


def _contained(off_a, ep_a, off_b, ep_b, tau=TAU):
    """every interval of A lies inside some interval of B (up to tau), column by column."""
    za, zb = np.asarray(ep_a, np.float64).reshape(-1, 2), np.asarray(ep_b, np.float64).reshape(-1, 2)
    for c in range(len(off_a) - 1):
        A = za[int(off_a[c]):int(off_a[c + 1])]
        B = zb[int(off_b[c]):int(off_b[c + 1])]
        for a, b in A:
            if b - a < tau:
                continue
            if not any(lo - tau <= a and b <= hi + tau for lo, hi in B):
                return False
    return True


@pytest.mark.parametrize("name_or_seed,r", [("C1", 3.0), (11, 2.0), (12, 3.5), (13, 1.0)])
def test_open_close_match_oracle_composition(dx, name_or_seed, r):
    """dexel_open = D_r(E_r(S)) and dexel_close = E_r(D_r(S)) match
    the oracle's composition; open(S) <= S <= close(S); both idempotent (within tau)."""
    if isinstance(name_or_seed, str):
        host = G.config(name_or_seed)
    else:
        host = G.random_grid(23, 19, 4, -9.0, 9.0, name_or_seed)
    src = dx.Grid.from_host(host)
    dst = dx.Grid.like(src)
    dst2 = dx.Grid.like(src)
    for op, first, second in (("open", O.erode, O.dilate), ("close", O.dilate, O.erode)):
        getattr(dx, "dexel_" + op)(src, r, dst)
        off, ep = dst.download()
        ref = second(_to_host_grid(host, first(host, r)), r)
        check(off, ep, ref, what=f"{op} r={r}")
        # idempotence
        getattr(dx, "dexel_" + op)(dst, r, dst2)
        off2, ep2 = dst2.download()
        res = compare(off2, ep2, off, ep, TAU)
        assert res["ok"], (op, "not idempotent", res)
        if op == "open":
            assert _contained(off, ep, host.off, host.ep), "opening not inside S"
        else:
            assert _contained(host.off, host.ep, off, ep), "S not inside its closing"
    # topological cleaning composes the two
    dx.clean(src, r, dst2)
    off, ep = dst2.download()
    ref = O.erode(_to_host_grid(host, O.dilate(_to_host_grid(host, O.dilate(_to_host_grid(host, O.erode(host, r)), r)), r)), r)
    check(off, ep, ref, what=f"clean r={r}")
    for g in (src, dst, dst2):
        g.close()


# ---------------------------------------------------------------- 2D slice offsets (NEXT #2)
def _row_grid(host, j):
    """row j of a host grid as a grid of its own (ny = 1): the 2D slice (x, z)."""
    nx = host.nx
    o = np.asarray(host.off[j * nx:(j + 1) * nx + 1], dtype=np.uint64)
    a, b = int(o[0]), int(o[-1])
    return G.Grid(nx, 1, (o - np.uint64(a)).astype(np.uint64), np.asarray(host.ep[2 * a:2 * b], dtype=np.float32),
                  host.z_lo, host.z_hi, host.z_ref, host.spacing)


def _check_slices(dx, host, op, r, rows):
    src = dx.Grid.from_host(host)
    dst = dx.Grid.like(src)
    if op == "shell":
        dx.dexel_shell_slices(src, r, r, dst)
    else:
        getattr(dx, "dexel_" + op + "_slices")(src, r, dst)
    off, ep = dst.download()
    for j in rows:
        rg = _row_grid(host, int(j))
        ref = O.shell(rg, r, r) if op == "shell" else getattr(O, op)(rg, r)
        o, z = take_columns(off, ep, np.arange(host.nx) + int(j) * host.nx)
        res = compare(o, z, ref.off, ref.z, 1e-4)
        assert res["ok"], (op, r, int(j), res)
    src.close()
    dst.close()


@pytest.mark.parametrize("cfg,op,r", [("C1", "dilate", 3.0), ("C1", "erode", 3.0), ("C1", "shell", 3.0),
                                      ("C2", "dilate", 4.0), ("C2", "erode", 4.0), ("C2", "shell", 4.0),
                                      ("C2", "dilate", 16.0), ("C3", "erode", 8.0)])
def test_slices_match_oracle_per_row(dx, cfg, op, r):
    """2D slice offsets: every row of the grid offset on its own equals
    the oracle's op on the one-row grid of that row (Eq. 1 in the (x, z) plane)."""
    host = G.config(cfg)
    rows = np.arange(host.ny) if host.ny <= 64 else np.random.default_rng(5).choice(host.ny, 24, replace=False)
    _check_slices(dx, host, op, r, rows)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_slices_random_small(dx, seed):
    """Random grids, radii incl. 0 and non-integer, all three ops, every row."""
    rs = np.random.default_rng(100 + seed)
    nx, ny = int(rs.integers(1, 70)), int(rs.integers(1, 9))
    cols = []
    for _ in range(nx * ny):
        k = int(rs.integers(0, 4))
        pts = np.sort(rs.uniform(-20, 20, 2 * k)).astype(np.float32)
        cols.append([(float(pts[2 * t]), float(pts[2 * t + 1])) for t in range(k) if pts[2 * t] < pts[2 * t + 1]
                     and (t == 0 or pts[2 * t] > pts[2 * t - 1])])
    host = G.from_columns(nx, ny, cols, -20.0, 20.0)
    for op in ("dilate", "erode", "shell"):
        for r in (0.0, 1.0, 2.5, 7.0):
            _check_slices(dx, host, op, r, np.arange(ny))


def test_slices_differ_from_3d_and_match_ny1(dx):
    """On a one-row grid the slice op is the 3D op (bitwise); on a taller grid it is not
    (rows do not reach each other), and the slab halo is not needed."""
    host = G.config("C1")
    r = 3.0
    rg = _row_grid(host, 32)
    a = dx.Grid.from_host(rg)
    d3, d2 = dx.Grid.like(a), dx.Grid.like(a)
    dx.dexel_dilate(a, r, d3)
    dx.dexel_dilate_slices(a, r, d2)
    o3, e3 = d3.download()
    o2, e2 = d2.download()
    assert np.array_equal(o3, o2) and np.array_equal(e3, e2)
    full = dx.Grid.from_host(host)
    f3, f2 = dx.Grid.like(full), dx.Grid.like(full)
    dx.dexel_dilate(full, r, f3)
    dx.dexel_dilate_slices(full, r, f2)
    assert f2.size() < f3.size() or not np.array_equal(f2.download()[1], f3.download()[1])
    for g in (a, d3, d2, full, f3, f2):
        g.close()


# ---------------------------------------------------------------- GPU dexelisation (NEXT #3)
@pytest.mark.parametrize("cfg", ["C1", "C2", "C4"])
def test_rasterize_shapes_bitwise_host_generator(dx, cfg):
    """dexel_rasterize_shapes on the GPU gives bitwise the CSR the host generator
    (dexelgen.c, fp64 per-column CSG) builds for the config."""
    n, zmin, zmax, sph, ss, box, bs = G.shape_config(cfg)
    host = G.config(cfg)
    g = dx.Grid.from_host(host)          # (frame and a previous content to replace)
    g2 = dx.Grid.like(g)
    dx.dexel_rasterize_shapes(g2, zmin, zmax, sph, ss, box, bs)
    off, ep = g2.download()
    assert np.array_equal(off.astype(np.uint64), host.off.astype(np.uint64))
    assert np.array_equal(ep, host.ep)
    g.close()
    g2.close()


def test_rasterize_shapes_c5_slab(dx):
    """C5 (20000 spheres minus 10000 voids) on a y-slab handle: its rows equal the host's."""
    n, zmin, zmax, sph, ss, box, bs = G.shape_config("C5")
    host = G.config("C5")
    y0, y1 = 1500, 1628
    g = dx.Grid(n, n, host.z_lo, host.z_hi, host.z_ref, 1.0, 0, None, y0, y1, 1, 3)
    dx.dexel_rasterize_shapes(g, zmin, zmax, sph, ss, box, bs)
    off, ep = g.download()
    a, b = int(host.off[y0 * n]), int(host.off[y1 * n])
    assert np.array_equal(off.astype(np.int64), host.off[y0 * n:y1 * n + 1].astype(np.int64) - a)
    assert np.array_equal(ep, host.ep[2 * a:2 * b])
    g.close()


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_rasterize_shapes_random(dx, seed):
    """Random spheres and boxes of both signs, partly outside the grid and the z domain, with
    integer / half-integer placements (ties on column centres and touching chords)."""
    rs = np.random.default_rng(200 + seed)
    nx, ny = int(rs.integers(1, 90)), int(rs.integers(1, 40))
    zmin, zmax = -5.0, float(rs.integers(10, 60))
    k, m = int(rs.integers(0, 40)), int(rs.integers(0, 12))
    sph = np.stack([rs.uniform(-10, nx + 10, k), rs.uniform(-10, ny + 10, k), rs.uniform(zmin - 5, zmax + 5, k),
                    rs.uniform(0.3, 15, k)], axis=1)
    if seed % 2:
        sph[:, :3] = np.round(sph[:, :3] * 2) / 2
        sph[:, 3] = np.round(sph[:, 3] * 2) / 2 + 0.5
    x0, y0 = rs.uniform(-5, nx, m), rs.uniform(-5, ny, m)
    z0 = rs.uniform(zmin - 3, zmax, m)
    box = np.stack([x0, x0 + rs.uniform(0, 20, m), y0, y0 + rs.uniform(0, 20, m), z0, z0 + rs.uniform(0, 20, m)], axis=1)
    if seed % 2:
        box = np.round(box * 2) / 2
    ss = np.where(rs.random(k) < 0.3, -1, 1).astype(np.int32)
    bs = np.where(rs.random(m) < 0.3, -1, 1).astype(np.int32)
    host = G.shapes(nx, ny, zmin, zmax, spheres=sph[ss > 0], voids=sph[ss < 0], boxes=box[bs > 0],
                    box_voids=box[bs < 0])
    g = dx.Grid(nx, ny, host.z_lo, host.z_hi, host.z_ref)
    dx.dexel_rasterize_shapes(g, zmin, zmax, sph, ss, box, bs)
    off, ep = g.download()
    assert np.array_equal(off.astype(np.uint64), host.off.astype(np.uint64))
    assert np.array_equal(ep, host.ep)
    g.close()


def test_rasterize_shapes_many_chords(dx):
    """Columns beyond the first attempt's capacities (64 chord intervals per sign, 32 output
    intervals): 150 small spheres stacked along z, every third one carved by a void, plus 90 thin
    box layers -- the library reruns with its large capacities; bitwise the host generator."""
    nx, ny, zmin, zmax = 20, 12, 0.0, 640.0
    k = np.arange(150)
    sph = np.stack([np.full(150, 9.7), np.full(150, 6.2), 3.0 + 4.0 * k, np.full(150, 1.6)], axis=1)
    voids = np.stack([np.full(50, 9.9), np.full(50, 6.1), 3.0 + 12.0 * np.arange(50), np.full(50, 0.6)], axis=1)
    j = np.arange(90)
    box = np.stack([np.full(90, 2.0), np.full(90, 6.0), np.full(90, 1.0), np.full(90, 5.0), 10.0 + 6.0 * j,
                    11.5 + 6.0 * j], axis=1)
    host = G.shapes(nx, ny, zmin, zmax, spheres=sph, voids=voids, boxes=box)
    per_col = np.diff(host.off.astype(np.int64))
    assert per_col.max() > 64                                   # (beyond both first-attempt capacities)
    allsph = np.concatenate([sph, voids])
    ss = np.concatenate([np.ones(150), -np.ones(50)]).astype(np.int32)
    g = dx.Grid(nx, ny, host.z_lo, host.z_hi, host.z_ref)
    dx.dexel_rasterize_shapes(g, zmin, zmax, allsph, ss, box, np.ones(90, np.int32))
    off, ep = g.download()
    assert np.array_equal(off.astype(np.uint64), host.off.astype(np.uint64))
    assert np.array_equal(ep, host.ep)
    # beyond the large capacities too: DEXEL_EOVERFLOW
    k = np.arange(600)
    sph = np.stack([np.full(600, 9.7), np.full(600, 6.2), 0.5 + 1.0 * k, np.full(600, 0.4)], axis=1)
    with pytest.raises(dx.DexelError) as e:
        dx.dexel_rasterize_shapes(g, zmin, zmax, sph, np.ones(600, np.int32))
    assert e.value.status == dx.DEXEL_EOVERFLOW
    g.close()


def test_rasterize_shapes_errors(dx):
    host = G.config("C1")
    g = dx.Grid.from_host(host)
    before = g.download()
    with pytest.raises(Exception):   # frame mismatch
        dx.dexel_rasterize_shapes(g, 0.0, 32.0, np.array([(32.0, 32.0, 16.0, 4.0)]), np.array([1]))
    after = g.download()
    assert np.array_equal(before[1], after[1])
    dx.dexel_rasterize_shapes(g, 0.0, 64.0)   # no shapes: the empty solid
    assert g.size() == 0
    g.close()


@pytest.mark.parametrize("n,period,t,amp,seed", [(1024, 64.0, 0.2, 0.05, G.SEED_BASE + 3),   # C3 itself
                                                  (37, 16.0, 0.2, 0.05, 7), (64, 12.5, -0.3, 0.4, 11),
                                                  (50, 24.0, 0.0, 0.0, 3), (33, 64.0, 2.0, 0.05, 5)])
def test_rasterize_gyroid_bitwise_host_generator(dx, n, period, t, amp, seed):
    """dexel_rasterize_gyroid gives bitwise the CSR of the host generator's noisy gyroid
    (dexelgen.c, fp64 samples + linear roots): C3 at full size, small grids with other periods,
    thresholds (t = 2: the empty solid), noise off and strong noise (many short intervals)."""
    host = G.gyroid(n, period, t, amp, seed)
    g = dx.Grid(n, n, host.z_lo, host.z_hi, host.z_ref)
    dx.dexel_rasterize_gyroid(g, 0.0, float(n), period, t, amp, seed)
    off, ep = g.download()
    assert np.array_equal(off.astype(np.uint64), host.off.astype(np.uint64))
    assert np.array_equal(ep, host.ep)
    g.close()


def test_rasterize_gyroid_slab_and_errors(dx):
    """A y-slab handle gets the host's rows [y0, y1); invalid arguments leave the grid unchanged."""
    n = 96
    host = G.gyroid(n, 20.0, 0.1, 0.1, 99)
    y0, y1 = 40, 71
    g = dx.Grid(n, n, host.z_lo, host.z_hi, host.z_ref, 1.0, 0, None, y0, y1, 1, 3)
    dx.dexel_rasterize_gyroid(g, 0.0, float(n), 20.0, 0.1, 0.1, 99)
    off, ep = g.download()
    a, b = int(host.off[y0 * n]), int(host.off[y1 * n])
    assert np.array_equal(off.astype(np.int64), host.off[y0 * n:y1 * n + 1].astype(np.int64) - a)
    assert np.array_equal(ep, host.ep[2 * a:2 * b])
    before = g.download()
    for args in [(0.0, 48.0, 20.0, 0.1, 0.1, 1), (0.0, float(n), 0.0, 0.1, 0.1, 1),
                 (0.0, float(n), 20.0, 0.1, -1.0, 1)]:
        with pytest.raises(Exception):
            dx.dexel_rasterize_gyroid(g, *args)
        after = g.download()
        assert np.array_equal(before[0], after[0]) and np.array_equal(before[1], after[1])
    g.close()


# ---------------------------------------------------------------- tri-dexel offsets (NEXT #4)
@pytest.mark.parametrize("cfg,op,r", [("C1", "dilate", 3.0), ("C2", "shell", 4.0), ("C2", "erode", 4.0)])
def test_tridexel_buffers_match_oracle(dx, cfg, op, r):
    """Tri-dexel: each of the three buffers is rasterised bitwise like the host generator on the
    permuted shapes, and its offset matches the oracle's op on that buffer's input."""
    from paper_1804_08968_b200.tridexel import AXES, TriDexel, permute_shapes
    n, zmin, zmax, sph, ss, box, bs = G.shape_config(cfg)
    td = TriDexel.from_shapes(n, zmin, zmax, sph, ss, box, bs)
    out = td.shell(r, r) if op == "shell" else getattr(td, op)(r)
    for a in AXES:
        s2, b2 = permute_shapes(a, sph, box)
        host = G.shapes(n, n, zmin, zmax, spheres=s2[ss > 0], voids=s2[ss < 0], boxes=b2[bs > 0], box_voids=b2[bs < 0])
        o_in, e_in = td.buf[a].download()
        assert np.array_equal(o_in.astype(np.uint64), host.off.astype(np.uint64)) and np.array_equal(e_in, host.ep)
        cols = sample_columns(n, n, 400, 2, 2, seed=11)
        ref = O.shell(host, r, r, cols=cols) if op == "shell" else getattr(O, op)(host, r, cols=cols)
        o, e = out.buf[a].download()
        oo, zz = take_columns(o, e, cols)
        res = compare(oo, zz, ref.off, ref.z, 1e-4)
        assert res["ok"], (a, op, r, res)
    td.close()
    out.close()


def test_fused_shell_c5_bitwise_separate(dx):
    """At full C5 size in the bench's configuration (3 bands), the fused shell pass 1 gives the
    bitwise output of two separate sweeps."""
    import gc
    import os
    import subprocess
    import sys

    import torch
    gc.collect()                      # (earlier tests' handles and cached blocks: the children
    dx.trim_workspace(0)              # need the device's memory)
    torch.cuda.empty_cache()
    code = r"""
import sys, hashlib; sys.path.insert(0, %r)
import numpy as np, dexelgen as G, paper_1804_08968_b200 as dx
host = G.config("C5")
src = dx.Grid.from_host(host); dst = dx.Grid.like(src)
dx.dexel_shell(src, 16.0, 16.0, dst)
off, ep = dst.download()
h = hashlib.sha256(); h.update(np.asarray(off).tobytes()); h.update(np.asarray(ep).tobytes())
print("HASH", h.hexdigest(), dst.stats()["capacities"]["bands"])
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hashes = {}
    for fuse in ("0", "1"):
        env = dict(os.environ, DEXEL_NO_FUSE=fuse)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        assert out.returncode == 0, out.stdout + out.stderr
        hashes[fuse] = [l.split()[1] for l in out.stdout.splitlines() if l.startswith("HASH")][0]
    assert hashes["0"] == hashes["1"], hashes


def test_trim_workspace_keeps_results(dx):
    """dexel_trim_workspace frees the idle device workspace and trims the pool; later ops
    allocate again and give bitwise the same output."""
    host = G.config("C2")
    src = dx.Grid.from_host(host)
    dst = dx.Grid.like(src)
    dx.dexel_shell(src, 4.0, 4.0, dst)
    a = dst.download()
    dx.trim_workspace(0)
    dx.dexel_shell(src, 4.0, 4.0, dst)
    b = dst.download()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    with pytest.raises(Exception):
        dx.trim_workspace(-1)
    src.close()
    dst.close()


# ---------------------------------------------------------------- parameter space (round 2)
@pytest.mark.parametrize("r", [65.0, 80.5, 128.0, 255.0])
def test_ops_large_radius(dx, r):
    """Ops at R = floor(r/s) in (64, 255]: every pass-1 mask width (NW = 5, 9, 17) and level
    chunking, against the oracle on every column."""
    host = G.random_grid(37, 29, 4, -300.0, 300.0, int(r) + 5)
    for op in ("dilate", "erode", "shell"):
        off, ep, _ = run_gpu(dx, host, op, r, r if op == "shell" else None)
        check(off, ep, run_oracle(host, op, r), what=f"{op} r={r}")


@pytest.mark.parametrize("s", [0.5, 1.7, 0.3])
def test_ops_spacing(dx, s):
    """Lateral spacing s != 1 (R = floor(r/s), weights r^2 - (kappa^2 + dy^2) s^2)."""
    for seed in range(3):
        host = G.random_grid(31, 23, 4, -12.0, 12.0, 300 + seed, quantum=0.25 if seed == 1 else None)
        host.spacing = s
        for r in (0.2, 1.0, 2.6, 5.0):
            for op in ("dilate", "erode", "shell"):
                off, ep, _ = run_gpu(dx, host, op, r, r * 0.8 if op == "shell" else None)
                check(off, ep, run_oracle(host, op, r, r * 0.8 if op == "shell" else None),
                      what=f"spacing {s} {op} r={r}")


@pytest.mark.parametrize("op", ["dilate", "erode", "shell"])
def test_many_layer_column(dx, op):
    """300 thin layers in a column (level lists and unions far beyond every default capacity,
    level lists beyond the old 255-interval arena): the op succeeds and matches the oracle."""
    col = [(float(t) * 0.5 - 80.0, float(t) * 0.5 - 79.8) for t in range(300)]
    cols = [col if (i + 2 * j) % 3 == 0 else (col[::3] if i % 2 else []) for j in range(5) for i in range(6)]
    host = _grid(6, 5, cols, -81.0, 81.0)
    for r in (0.05, 0.4, 1.3):
        off, ep, _ = run_gpu(dx, host, op, r)
        check(off, ep, run_oracle(host, op, r), what=f"300 layers {op} r={r}")


@pytest.mark.parametrize("op", ["dilate", "shell"])
def test_level_list_beyond_arena(dx, op):
    """1500 thin layers: level lists longer than the largest slot capacity (255) and its default
    arena (4 x 255 entries) saturate their offsets, the op reruns with a doubled arena until they
    fit (levels.cuh spill cell), and the result matches the oracle."""
    col = [(float(t) * 0.25 - 200.0, float(t) * 0.25 - 199.9) for t in range(1500)]
    cols = [col if (i + j) % 2 == 0 else col[::5] for j in range(3) for i in range(4)]
    host = _grid(4, 3, cols, -201.0, 201.0)
    for r in (0.05, 1.3):
        off, ep, _ = run_gpu(dx, host, op, r)
        check(off, ep, run_oracle(host, op, r), what=f"1500 layers {op} r={r}")


def test_caller_stream(dx):
    """A handle on a caller-supplied stream (torch side stream): ops run on it, results match the
    oracle, and work queued on the stream before the op is ordered before it."""
    import torch
    host = G.config("C2")
    st = torch.cuda.Stream()
    src = dx.Grid(host.nx, host.ny, host.z_lo, host.z_hi, host.z_ref, 1.0, 0, st.cuda_stream)
    with torch.cuda.stream(st):
        off_d = torch.from_numpy(host.off.astype(np.int64)).cuda()
        ep_d = torch.from_numpy(host.ep).cuda()
    src.upload(off_d, ep_d)
    dst = dx.Grid.like(src)
    assert dst.desc.stream == st.cuda_stream
    dx.dexel_shell(src, 4.0, 4.0, dst)
    off, ep = dst.download(device=True)
    st.synchronize()
    check(off.cpu().numpy().astype(np.uint64), ep.cpu().numpy(), run_oracle(host, "shell", 4.0), what="caller stream")
    src.close()
    dst.close()


def test_error_leaves_dst_empty(dx):
    """An op that fails after dst was already written leaves dst empty (dexel.h), and dst is
    usable afterwards."""
    host = G.config("C1")
    src = dx.Grid.from_host(host)
    dst = dx.Grid.like(src)
    dx.dexel_dilate(src, 3.0, dst)
    assert dst.size() > 0
    with pytest.raises(dx.DexelError):
        dx.dexel_dilate(src, float("inf"), dst)
    assert dst.size() == 0
    off, _ = dst.download()
    assert not off.any()
    dx.dexel_dilate(src, 3.0, dst)
    check(*dst.download(), run_oracle(host, "dilate", 3.0), what="after error")
