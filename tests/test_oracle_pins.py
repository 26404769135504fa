"""Pins for the fp64 oracle (-m "not gpu").

The oracle is pinned to things other than itself (PAPER.md has no numeric
worked example of a dilation):
  P2  O1 (brute force) == O2 (separable) on random grids      App. A1 / SURVEY 8(c)
  P3  brute-force point-to-solid distance at every endpoint     Eq. 1
  P4  single interval / Pythagorean closed forms (golden)       SPEC.md:402, Eq. 1
  P5  box dilation closed form                                   derived from Eq. 1
  P6  box erosion closed form; SPEC 4^3 cube example
  P7  sphere sandwich ball(rho+r-sqrt2) c D c ball(rho+r)        App. A3 of SURVEY
  P8  D(A u B) = D(A) u D(B)
  P9  special cases (r = 0, 0<r<1, empty, full, 2D capsule)
  P10 invariants (extensive, monotone, E c S, open c S c close, semigroup inclusion)
  P11 symmetries (mirror x / y / z, transpose)                   separability PAPER.md:219
  Pass-1 pieces: union == row extrusion, kappa == brute closest parent
Each pin runs against both O1 and O2 where it applies.
"""
import math
import os

import numpy as np
import pytest

import dexelgen as G
import oracle as O
from oracle.compare import compare

GOLD = os.path.join(os.path.dirname(__file__), "golden")
METHODS = ["brute", "sep"]


# ---------------------------------------------------------------- helpers
def cols_of(res):
    return [np.asarray(c, dtype=np.float64) for c in res.columns()]


def grid_cols(g):
    return [np.asarray(c, dtype=np.float64) for c in g.columns()]


def union_list(ivs):
    ivs = sorted((float(a), float(b)) for a, b in ivs)
    out = []
    for a, b in ivs:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def contained(a, b, tol=0.0):
    """every interval of a lies inside some interval of b (within tol)."""
    b = union_list(b)
    for lo, hi in a:
        if hi - lo <= tol:
            continue
        if not any(blo - tol <= lo and hi <= bhi + tol for blo, bhi in b):
            return False
    return True


def dist_to_solid(cols, nx, ny, i, j, z, s=1.0):
    """min Euclidean distance from the point (i, j, z) to the lattice solid (fp64 brute force)."""
    best = math.inf
    for jj in range(ny):
        for ii in range(nx):
            c = cols[jj * nx + ii]
            if len(c) == 0:
                continue
            lat2 = ((ii - i) ** 2 + (jj - j) ** 2) * s * s
            if lat2 >= best * best:
                continue
            for a, b in c:
                dz = max(0.0, a - z, z - b)
                best = min(best, math.sqrt(lat2 + dz * dz))
    return best


def complement_cols(g):
    out = []
    for c in grid_cols(g):
        cur, lst = g.z_lo, []
        for a, b in c:
            if a > cur:
                lst.append((cur, a))
            cur = b
        if g.z_hi > cur:
            lst.append((cur, g.z_hi))
        out.append(np.array(lst, dtype=np.float64).reshape(-1, 2))
    return out


def load_golden(name):
    lines = [l.split() for l in open(os.path.join(GOLD, name)) if l.strip() and not l.startswith("#")]
    hdr = lines[0]
    nx, ny = int(hdr[1]), int(hdr[2])
    z_lo, z_hi, r = float(hdr[3]), float(hdr[4]), float(hdr[5])
    cols = [[] for _ in range(nx * ny)]
    outs, empties = {}, []
    for l in lines[1:]:
        if l[0] == "in":
            cols[int(l[2]) * nx + int(l[1])].append((float(l[3]), float(l[4])))
        elif l[0] == "out":
            outs.setdefault(int(l[2]) * nx + int(l[1]), []).append((float(l[3]), float(l[4])))
        elif l[0] == "empty":
            empties.append(int(l[2]) * nx + int(l[1]))
    g = G.from_columns(nx, ny, [np.array(c, np.float32).reshape(-1, 2) for c in cols], z_lo, z_hi)
    return g, r, outs, empties


def random_case(seed, maxn=8, maxk=3, rvals=(0.0, 0.4, 1.0, 1.5, 2.0, 2.5, 3.0, 4.2, 5.0)):
    rs = np.random.default_rng(seed)
    nx, ny = (int(v) for v in rs.integers(1, maxn + 1, 2))
    q = 0.25 if seed % 3 == 0 else None
    g = G.random_grid(nx, ny, maxk, -6.0, 6.0, seed, quantum=q)
    r = float(rs.choice(rvals))
    return g, r


# ---------------------------------------------------------------- P4 golden
@pytest.mark.parametrize("name", ["spec_s402_single_interval_r1.txt", "spec_s207_capsule_2d.txt",
                                  "pythagorean_r5.txt"])
@pytest.mark.parametrize("method", METHODS)
def test_golden_closed_forms(name, method):
    g, r, outs, empties = load_golden(name)
    d = O.dilate(g, r, method)
    for c, want in outs.items():
        got = d.column(c).tolist()
        assert got == [list(w) for w in want], (c, got, want)
    for c in empties:
        assert len(d.column(c)) == 0
    if name.startswith("spec_s402"):
        # everything not listed is empty (diagonals in particular)
        for c in range(g.ncol):
            if c not in outs:
                assert len(d.column(c)) == 0


# ---------------------------------------------------------------- P2
@pytest.mark.parametrize("seed", range(120))
def test_brute_equals_separable(seed):
    g, r = random_case(seed)
    for op in ("dilate", "erode"):
        a = getattr(O, op)(g, r, "brute")
        b = getattr(O, op)(g, r, "sep")
        res = compare(a.off, a.z, b.off, b.z, 1e-9)
        assert res["ok"], (op, res)
        # bitwise in practice (App. A1): identical candidate expressions
        assert np.array_equal(a.off, b.off) and np.array_equal(a.z, b.z)
    a = O.shell(g, r, r * 0.5, "brute")
    b = O.shell(g, r, r * 0.5, "sep")
    assert compare(a.off, a.z, b.off, b.z, 1e-9)["ok"]


# ---------------------------------------------------------------- P3
@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("method", METHODS)
def test_endpoint_distance_bruteforce(seed, method):
    g, r = random_case(seed + 1000, maxn=5, maxk=2, rvals=(1.0, 1.5, 2.0, 2.7))
    S = grid_cols(g)
    d = O.dilate(g, r, method)
    for c in range(g.ncol):
        i, j = c % g.nx, c // g.nx
        iv = d.column(c)
        for lo, hi in iv:
            for e in (lo, hi):
                if e in (g.z_lo, g.z_hi):
                    continue
                assert abs(dist_to_solid(S, g.nx, g.ny, i, j, e) - r) <= 1e-9 * max(1.0, r)
            assert dist_to_solid(S, g.nx, g.ny, i, j, 0.5 * (lo + hi)) <= r + 1e-12
        # gaps (including the domain ends) are uncovered
        pts = [g.z_lo] + [x for ab in iv for x in ab] + [g.z_hi]
        for a, b in zip(pts[0::2], pts[1::2]):
            if b - a > 1e-9:
                assert dist_to_solid(S, g.nx, g.ny, i, j, 0.5 * (a + b)) > r
    # erosion: distance to the complement C (neutral boundary: out-of-grid columns absent)
    C = complement_cols(g)
    e = O.erode(g, r, method)
    for c in range(g.ncol):
        i, j = c % g.nx, c // g.nx
        for lo, hi in e.column(c):
            assert dist_to_solid(C, g.nx, g.ny, i, j, 0.5 * (lo + hi)) > r
            for z in (lo, hi):
                if z in (g.z_lo, g.z_hi):
                    continue
                assert abs(dist_to_solid(C, g.nx, g.ny, i, j, z) - r) <= 1e-9 * max(1.0, r)


# ---------------------------------------------------------------- P5 / P6
def _box_grid(nx, ny, box, z_lo=-20.0, z_hi=20.0):
    i0, i1, j0, j1, z0, z1 = box
    cols = []
    for j in range(ny):
        for i in range(nx):
            inside = i0 <= i <= i1 and j0 <= j <= j1
            cols.append(np.array([[z0, z1]] if inside else [], np.float32).reshape(-1, 2))
    return G.from_columns(nx, ny, cols, z_lo, z_hi)


@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("r", [1.0, 2.0, 2.5, 3.7, 5.0])
def test_box_dilation_closed_form(method, r):
    box = (6, 9, 5, 11, -3.0, 4.5)
    g = _box_grid(18, 17, box)
    d = O.dilate(g, r, method)
    i0, i1, j0, j1, z0, z1 = box
    for c in range(g.ncol):
        i, j = c % g.nx, c // g.nx
        di = max(i0 - i, 0, i - i1)
        dj = max(j0 - j, 0, j - j1)
        d2 = float(di * di + dj * dj)
        got = d.column(c).tolist()
        if d2 > r * r:
            assert got == []
        else:
            h = math.sqrt(r * r - d2)   # nearest footprint column gives the largest growth
            assert len(got) == 1
            assert abs(got[0][0] - max(z0 - h, g.z_lo)) < 1e-12 and abs(got[0][1] - min(z1 + h, g.z_hi)) < 1e-12


@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("r", [1.0, 1.5, 2.0, 3.0])
def test_box_erosion_closed_form(method, r):
    box = (4, 11, 3, 12, -6.0, 5.0)
    g = _box_grid(16, 16, box)
    e = O.erode(g, r, method)
    i0, i1, j0, j1, z0, z1 = box
    for c in range(g.ncol):
        i, j = c % g.nx, c // g.nx
        inside = i0 <= i <= i1 and j0 <= j <= j1
        m = min(i - i0 + 1, i1 - i + 1, j - j0 + 1, j1 - j + 1) if inside else 0
        got = e.column(c).tolist()
        if not inside or m <= r or z1 - z0 <= 2 * r:
            assert got == [], (i, j, got)
        else:
            assert got == [[z0 + r, z1 - r]]


@pytest.mark.parametrize("method", METHODS)
def test_spec_cube_erosion_and_shell(method):
    # 4x4x4 cube, r = 1 -> 2x2x2.  SPEC.md:461: 6^3 cube, r_out = 0, r_in = 1 -> 1-thick crust.
    g = _box_grid(10, 10, (3, 6, 3, 6, -2.0, 2.0), -5.0, 5.0)
    e = O.erode(g, 1.0, method)
    solid = {c: e.column(c).tolist() for c in range(g.ncol) if len(e.column(c))}
    assert solid == {j * 10 + i: [[-1.0, 1.0]] for i in (4, 5) for j in (4, 5)}
    g6 = _box_grid(12, 12, (3, 8, 3, 8, -3.0, 3.0), -6.0, 6.0)
    sh = O.shell(g6, 0.0, 1.0, method)
    for c in range(g6.ncol):
        i, j = c % 12, c // 12
        got = sh.column(c).tolist()
        if not (3 <= i <= 8 and 3 <= j <= 8):
            assert got == []
        elif i in (3, 8) or j in (3, 8):
            assert got == [[-3.0, 3.0]]
        else:
            assert got == [[-3.0, -2.0], [2.0, 3.0]]


# ---------------------------------------------------------------- P7
@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("r", [2.0, 3.5, 6.0])
def test_sphere_sandwich(method, r):
    rho, o = 9.3, (20.2, 19.7, 0.4)
    g = G.shapes(40, 40, 0.0, 60.0, spheres=[(o[0], o[1], o[2] + 30.0, rho)])  # z_ref = 30
    d = O.dilate(g, r, method)
    s2 = math.sqrt(2.0)
    for c in range(g.ncol):
        i, j = c % 40, c // 40
        lat2 = (i + 0.5 - o[0]) ** 2 + (j + 0.5 - o[1]) ** 2
        got = d.column(c).tolist()
        outer = (rho + r) ** 2 - lat2
        if outer <= 0:
            assert got == []
            continue
        hz = math.sqrt(outer)
        for lo, hi in got:
            assert lo >= o[2] - hz - 1e-9 and hi <= o[2] + hz + 1e-9
        inner = (rho + r - s2) ** 2 - lat2
        if inner > 0:
            hin = math.sqrt(inner)
            assert any(lo <= o[2] - hin + 1e-9 and o[2] + hin - 1e-9 <= hi for lo, hi in got)


# ---------------------------------------------------------------- P8
@pytest.mark.parametrize("seed", range(10))
def test_union_identity(seed):
    ga, r = random_case(seed + 2000, maxn=7)
    gb = G.random_grid(ga.nx, ga.ny, 2, -6.0, 6.0, seed + 3000)
    cols = [union_list(list(map(tuple, a)) + list(map(tuple, b))) for a, b in zip(grid_cols(ga), grid_cols(gb))]
    gu = G.from_columns(ga.nx, ga.ny, [np.array(c, np.float32).reshape(-1, 2) for c in cols], -6.0, 6.0)
    for m in METHODS:
        du, da, db = (cols_of(O.dilate(x, r, m)) for x in (gu, ga, gb))
        for c in range(ga.ncol):
            want = union_list(list(map(tuple, da[c])) + list(map(tuple, db[c])))
            assert np.allclose(np.array(want).reshape(-1, 2), du[c], atol=1e-12) and len(want) == len(du[c])


# ---------------------------------------------------------------- P9
@pytest.mark.parametrize("method", METHODS)
def test_special_cases(method):
    g, _ = random_case(7, maxn=6)
    d = O.dilate(g, 0.0, method)
    assert [c.tolist() for c in cols_of(d)] == [c.tolist() for c in grid_cols(g)]       # r = 0: identity
    e = O.erode(g, 0.0, method)
    assert [c.tolist() for c in cols_of(e)] == [c.tolist() for c in grid_cols(g)]
    r = 0.6                                                                              # 0 < r < s: z only
    d = O.dilate(g, r, method)
    for c, col in enumerate(grid_cols(g)):
        want = union_list([(max(a - r, g.z_lo), min(b + r, g.z_hi)) for a, b in col])
        assert np.allclose(np.array(want).reshape(-1, 2), d.column(c)) and len(want) == len(d.column(c))
    empty = G.from_columns(5, 4, [np.zeros((0, 2), np.float32)] * 20, -3, 3)
    assert O.dilate(empty, 2.0, method).off[-1] == 0
    assert O.erode(empty, 2.0, method).off[-1] == 0
    full = G.from_columns(5, 4, [np.array([[-3, 3]], np.float32)] * 20, -3, 3)
    for res in (O.dilate(full, 2.0, method), O.erode(full, 2.0, method)):                  # neutral boundary
        assert all(c.tolist() == [[-3.0, 3.0]] for c in cols_of(res))


# ---------------------------------------------------------------- P10
@pytest.mark.parametrize("seed", range(15))
def test_invariants(seed):
    g, r = random_case(seed + 4000, maxn=7, rvals=(1.0, 1.5, 2.0, 3.0))
    S = grid_cols(g)
    D = cols_of(O.dilate(g, r))
    D2 = cols_of(O.dilate(g, r + 1.25))
    E = cols_of(O.erode(g, r))
    for c in range(g.ncol):
        assert contained(S[c], D[c])                # extensive
        assert contained(D[c], D2[c])               # monotone in r
        assert contained(E[c], S[c])                # anti-extensive
    # opening c S c closing, semigroup inclusion D_a(D_b S) c D_(a+b) S (fp32 re-quantisation tolerance)
    def as_grid(cols):
        return G.from_columns(g.nx, g.ny, [np.array(c, np.float32).reshape(-1, 2) for c in cols], g.z_lo, g.z_hi)
    opening = cols_of(O.dilate(as_grid(E), r))
    closing = cols_of(O.erode(as_grid(D), r))
    DD = cols_of(O.dilate(as_grid(D), 1.0))
    Dab = cols_of(O.dilate(g, r + 1.0))
    for c in range(g.ncol):
        assert contained(opening[c], S[c], 1e-5)
        assert contained(S[c], closing[c], 1e-5)
        assert contained(DD[c], Dab[c], 1e-5)


# ---------------------------------------------------------------- P11
@pytest.mark.parametrize("seed", range(8))
def test_symmetries(seed):
    g, r = random_case(seed + 5000, maxn=7)
    nx, ny = g.nx, g.ny
    S = grid_cols(g)

    def remap(cols, f, nx2, ny2):
        out = [None] * (nx2 * ny2)
        for c, col in enumerate(cols):
            i, j = c % nx, c // nx
            i2, j2 = f(i, j)
            out[j2 * nx2 + i2] = col
        return out

    def mk(cols, nx2, ny2):
        return G.from_columns(nx2, ny2, [np.array(c, np.float32).reshape(-1, 2) for c in cols], g.z_lo, g.z_hi)

    D = cols_of(O.dilate(g, r))
    for f, nx2, ny2 in [(lambda i, j: (nx - 1 - i, j), nx, ny), (lambda i, j: (i, ny - 1 - j), nx, ny),
                        (lambda i, j: (j, i), ny, nx)]:
        Dm = cols_of(O.dilate(mk(remap(S, f, nx2, ny2), nx2, ny2), r))
        want = remap(D, f, nx2, ny2)
        for c in range(nx * ny):
            assert np.array_equal(Dm[c], want[c])
    # z -> -z (exact in fp; domain symmetric)
    Sz = [(-np.asarray(c)[::-1, ::-1]) for c in S]
    Dz = cols_of(O.dilate(mk(Sz, nx, ny), r))
    for c in range(nx * ny):
        assert np.array_equal(Dz[c], -D[c][::-1, ::-1])


# ---------------------------------------------------------------- pass-1 pieces
@pytest.mark.parametrize("seed", range(25))
def test_pass1_pieces(seed):
    g, r = random_case(seed + 6000, maxn=8, maxk=3, rvals=(1.0, 2.0, 3.0, 4.5))
    R = int(math.floor(r))
    for comp in (False, True):
        S = complement_cols(g) if comp else grid_cols(g)
        p = O.pass1(g, r, complement=comp)
        for c in range(g.ncol):
            i, j = c % g.nx, c // g.nx
            z, k = p.column(c), p.kappa(c)
            # canonical: sorted, positive length, touching neighbours differ in kappa
            for t in range(len(z)):
                assert z[t, 0] < z[t, 1]
                if t:
                    assert z[t, 0] >= z[t - 1, 1]
                    if z[t, 0] == z[t - 1, 1]:
                        assert k[t] != k[t - 1]
            # union == flat extrusion of the row within |dx| <= R
            ext = union_list([tuple(iv) for dx in range(-R, R + 1) if 0 <= i + dx < g.nx
                              for iv in S[j * g.nx + i + dx]])
            assert union_list([tuple(iv) for iv in z]) == ext
            # kappa == brute-force closest parent at piece midpoints
            for (lo, hi), kk in zip(z, k):
                zm = 0.5 * (lo + hi)
                best = min(abs(dx) for dx in range(-R, R + 1) if 0 <= i + dx < g.nx
                           and any(a <= zm <= b for a, b in S[j * g.nx + i + dx]))
                assert best == kk


def test_generator_rng_matches_c():
    lib = G._load()
    for s, st, i in [(1, 0, 0), (1804089681, 3, 12345), (7, 6, 2 ** 40)]:
        assert int(G.rng_u64(s, st, i)) == lib.dexelgen_u64(s, st, i)


def test_generator_c1_deterministic():
    a, b = G.config("C1"), G.config("C1", nthreads=1)
    assert np.array_equal(a.off, b.off) and np.array_equal(a.ep, b.ep)
    # every non-empty column of C1 is one interval (sphere chords overlap the box z-range)
    assert G.stats(a)["max_per_col"] == 1


# ---------------------------------------------------------------- lateral spacing s != 1
def _with_spacing(g, s):
    g.spacing = float(s)
    return g


@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("s,r", [(0.5, 1.3), (0.5, 2.6), (1.7, 3.5), (2.0, 4.0), (0.25, 1.1)])
def test_box_dilation_closed_form_spacing(method, s, r):
    """P5 with lateral spacing s: the nearest footprint column lies at lateral distance
    d = s * sqrt(di^2 + dj^2); the column dilates to [z0 - h, z1 + h], h = sqrt(r^2 - d^2)."""
    box = (6, 9, 5, 11, -3.0, 4.5)
    g = _with_spacing(_box_grid(18, 17, box), s)
    d = O.dilate(g, r, method)
    i0, i1, j0, j1, z0, z1 = box
    for c in range(g.ncol):
        i, j = c % g.nx, c // g.nx
        di = max(i0 - i, 0, i - i1)
        dj = max(j0 - j, 0, j - j1)
        d2 = float(di * di + dj * dj) * s * s
        got = d.column(c).tolist()
        if d2 > r * r:
            assert got == [], (i, j, got)
        else:
            h = math.sqrt(r * r - d2)
            assert len(got) == 1
            assert abs(got[0][0] - max(z0 - h, g.z_lo)) < 1e-12 and abs(got[0][1] - min(z1 + h, g.z_hi)) < 1e-12


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("method", METHODS)
def test_endpoint_distance_bruteforce_spacing(seed, method):
    """P3 with lateral spacing s != 1: every non-clip output endpoint lies at distance exactly r
    from the lattice solid, interval midpoints within r, gap midpoints beyond r."""
    g, r = random_case(seed + 2000, maxn=5, maxk=2, rvals=(1.0, 1.5, 2.7))
    s = (0.6, 1.4, 0.35)[seed % 3]
    _with_spacing(g, s)
    S = grid_cols(g)
    d = O.dilate(g, r, method)
    for c in range(g.ncol):
        i, j = c % g.nx, c // g.nx
        iv = d.column(c)
        for lo, hi in iv:
            for e in (lo, hi):
                if e in (g.z_lo, g.z_hi):
                    continue
                assert abs(dist_to_solid(S, g.nx, g.ny, i, j, e, s) - r) <= 1e-9 * max(1.0, r)
            assert dist_to_solid(S, g.nx, g.ny, i, j, 0.5 * (lo + hi), s) <= r + 1e-12
        pts = [g.z_lo] + [x for ab in iv for x in ab] + [g.z_hi]
        for a, b in zip(pts[0::2], pts[1::2]):
            if b - a > 1e-9:
                assert dist_to_solid(S, g.nx, g.ny, i, j, 0.5 * (a + b), s) > r


@pytest.mark.parametrize("seed", range(10))
def test_brute_equals_separable_spacing(seed):
    """P2 (App. A1) with s != 1: O1 and O2 agree bitwise."""
    g, r = random_case(seed + 3000)
    _with_spacing(g, (0.5, 1.5, 0.8, 2.25)[seed % 4])
    for op in ("dilate", "erode"):
        a = getattr(O, op)(g, r, "brute")
        b = getattr(O, op)(g, r, "sep")
        assert np.array_equal(a.off, b.off) and np.array_equal(a.z, b.z), op


# ---------------------------------------------------------------- large radii R in (64, 255]
@pytest.mark.parametrize("r", [70.0, 100.5, 255.0])
def test_brute_equals_separable_large_radius(r):
    """P2 at radii whose level count R + 1 exceeds 65 (u8 kappa up to 255)."""
    g = G.random_grid(9, 7, 3, -300.0, 300.0, int(r))
    for op in ("dilate", "erode"):
        a = getattr(O, op)(g, r, "brute")
        b = getattr(O, op)(g, r, "sep")
        assert np.array_equal(a.off, b.off) and np.array_equal(a.z, b.z), op


# ---------------------------------------------------------------- the sampled-column path
@pytest.mark.parametrize("seed", range(30))
def test_sampled_columns_equal_full_run(seed):
    """oracle_run on a list of columns (the path every C3-C5 parity test and the cpu baseline
    use) gives bitwise the full run's result for those columns, for every op."""
    rs = np.random.default_rng(4000 + seed)
    g = G.random_grid(int(rs.integers(1, 30)), int(rs.integers(1, 30)), 4, -10.0, 10.0, seed,
                      quantum=0.5 if seed % 2 else None)
    r = float(rs.choice([0.0, 0.7, 1.0, 2.5, 4.0, 7.0]))
    cols = np.unique(rs.integers(0, g.ncol, max(1, g.ncol // 3))).astype(np.int64)
    for op in ("dilate", "erode", "shell", "pass1"):
        if op == "shell":
            full, part = O.shell(g, r, r * 0.5), O.shell(g, r, r * 0.5, cols=cols)
        else:
            full, part = getattr(O, op)(g, r), getattr(O, op)(g, r, cols=cols)
        want = [full.column(int(c)) for c in cols]
        got = [part.column(t) for t in range(len(cols))]
        assert all(np.array_equal(a, b) for a, b in zip(want, got)), (op, r)
        if op == "pass1":
            assert all(np.array_equal(full.kappa(int(c)), part.kappa(t)) for t, c in enumerate(cols))
