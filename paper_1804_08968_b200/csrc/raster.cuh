// raster.cuh -- GPU dexelisation of analytic solids: spheres and
// axis-aligned boxes, each solid (+1) or void (-1), rasterised onto the ray lattice as the
// canonical fp32 dexel CSR of (U solids) \ (U voids) (PAPER.md:114-118 dexel buffers,
// :170 / :42 "CSG operations can be carried out easily in dexel space").
//
// Column (i, j) is the ray at ((i + 1/2) s, (j + 1/2) s), s = 1.  Per column, in fp64 with no
// contraction (every product and sum rounded on its own, as the host generator computes it):
//   sphere (cx, cy, cz, R): rr = R*R - dy*dy, dy = y - cy; if rr > 0 and the column lies in
//     [ceil(cx - sqrt(rr) - 1/2), floor(cx + sqrt(rr) - 1/2)] and q = rr - dx*dx > 0,
//     dx = x - cx, the chord is [cz - sqrt(q), cz + sqrt(q)];
//   box (x0, x1, y0, y1, z0, z1): y in [y0, y1] and the column in [ceil(x0 - 1/2), floor(x1 - 1/2)]
//     give the chord [z0, z1].
// The column's solid is union(solid chords) \ union(void chords) (closed intervals, touching
// merges), clipped to [zmin, zmax], shifted to the local frame z - zref, rounded to fp32 and
// canonicalised (touching after rounding merges, zero length after rounding drops).  The
// result equals dexelgen.c (the input generator) bit for bit: the unions of closed intervals
// are unique, so building them by insertion instead of sort + sweep changes nothing, and every
// endpoint is the same fp64 expression rounded once to fp32.
//
// One thread per column; a block is a tile of RT_X x RT_Y columns (a warp = 32 consecutive
// columns of a row) and walks the tile's shape list (binned on the device, conservative); every lane
// reads the same shape (broadcast load).  The unions live in per-thread local memory.
// Results go to a [t][column] staging array, then the scan and compact_kernel (pass2.cuh).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dexel {

constexpr int RT_X = 32, RT_Y = 8;
constexpr int RS_CAP = 64;     // intervals per union (solid chords, void chords) of one column: first attempt
constexpr int RS_OUT = 32;     // output intervals per column (staging): first attempt
constexpr int RS_CAP_BIG = 512;   // second attempt after an overflow (16 KB of local memory per thread)

struct RasterArgs {
  int nx, nrows, y0;           // local rows [0, nrows) are global rows y0 + jl
  double zmin, zmax, zref;
  int nsph;
  const double* sph;           // [nsph][4] cx, cy, cz, R (world)
  const int32_t* sph_sign;
  int nbox;
  const double* box;           // [nbox][6] x0, x1, y0, y1, z0, z1
  const int32_t* box_sign;
  const uint64_t* tile_off;    // [ntiles + 1]
  const int32_t* tile_ids;     // shape ids: sphere k -> k, box k -> nsph + k
  int ntx;                     // tiles per tile row
  float2* stage;               // [out_cap][ncol]
  uint32_t* cnt;               // [ncol]
  unsigned* flags;             // [0] a union or the output outgrew its capacity
  int out_cap;                 // output intervals per column the staging array holds
};

// insert the closed interval [lo, hi] into the sorted disjoint union V[0..n) (touching merges)
template <int CAP>
__device__ __forceinline__ void rs_union_insert(double2* V, int& n, double lo, double hi, bool& ovf) {
  int p = 0;
  while (p < n && V[p].y < lo) ++p;
  if (p < n && V[p].x <= hi) {   // overlaps or touches V[p]: merge the run p..q
    double nlo = fmin(lo, V[p].x), nhi = fmax(hi, V[p].y);
    int q = p;
    while (q + 1 < n && V[q + 1].x <= nhi) {
      ++q;
      nhi = fmax(nhi, V[q].y);
    }
    V[p] = make_double2(nlo, nhi);
    const int drop = q - p;
    if (drop) {
      for (int t = q + 1; t < n; ++t) V[t - drop] = V[t];
      n -= drop;
    }
    return;
  }
  if (n >= CAP) {
    ovf = true;
    return;
  }
  for (int t = n; t > p; --t) V[t] = V[t - 1];
  V[p] = make_double2(lo, hi);
  ++n;
}

template <int CAP>
__global__ void __launch_bounds__(RT_X* RT_Y) raster_kernel(RasterArgs A) {
  const int tile = blockIdx.x;
  const int tx = tile % A.ntx, ty = tile / A.ntx;
  const int i = tx * RT_X + threadIdx.x, jl = ty * RT_Y + threadIdx.y;
  const bool live = i < A.nx && jl < A.nrows;
  const double x = (double)i + 0.5, y = (double)(A.y0 + jl) + 0.5;
  double2 P[CAP], N[CAP];
  int np = 0, nn = 0;
  bool ovf = false;
  for (uint64_t t = A.tile_off[tile]; t < A.tile_off[tile + 1]; ++t) {
    const int id = A.tile_ids[t];
    double lo, hi;
    int sg;
    if (id < A.nsph) {
      const double* s = A.sph + 4 * (size_t)id;
      const double dy = __dsub_rn(y, s[1]), R = s[3];
      const double rr = __dsub_rn(__dmul_rn(R, R), __dmul_rn(dy, dy));
      if (!(rr > 0.0)) continue;
      const double hx = sqrt(rr);
      const int i0 = (int)ceil(__dsub_rn(__dsub_rn(s[0], hx), 0.5));
      const int i1 = (int)floor(__dsub_rn(__dadd_rn(s[0], hx), 0.5));
      if (i < i0 || i > i1) continue;
      const double dx = __dsub_rn(x, s[0]);
      const double q = __dsub_rn(rr, __dmul_rn(dx, dx));
      if (!(q > 0.0)) continue;
      const double h = sqrt(q);
      lo = __dsub_rn(s[2], h);
      hi = __dadd_rn(s[2], h);
      sg = A.sph_sign[id];
    } else {
      const int b = id - A.nsph;
      const double* s = A.box + 6 * (size_t)b;
      if (y < s[2] || y > s[3]) continue;
      const int i0 = (int)ceil(__dsub_rn(s[0], 0.5)), i1 = (int)floor(__dsub_rn(s[1], 0.5));
      if (i < i0 || i > i1) continue;
      lo = s[4];
      hi = s[5];
      sg = A.box_sign[b];
    }
    if (!live) continue;
    // (the host generator keeps chords with lo > hi out of nothing: none exist, h >= 0 and
    // boxes have z0 <= z1 by construction; a degenerate box still enters its union as given)
    if (sg > 0) rs_union_insert<CAP>(P, np, lo, hi, ovf);
    else rs_union_insert<CAP>(N, nn, lo, hi, ovf);
  }
  if (!live) return;
  const int64_t c = (int64_t)jl * A.nx + i;
  const int64_t ncol = (int64_t)A.nrows * A.nx;
  // difference P \ N (sorted, disjoint), then clip, shift, round, canonicalise
  uint32_t k = 0;
  float la = 0.f, lb = 0.f;    // last written output interval (merge target)
  auto emit = [&](double dlo, double dhi) {
    const double clo = dlo < A.zmin ? A.zmin : dlo;
    const double chi = dhi > A.zmax ? A.zmax : dhi;
    if (!(clo < chi)) return;
    const float a = (float)__dsub_rn(clo, A.zref), b = (float)__dsub_rn(chi, A.zref);
    if (k > 0 && a <= lb) {                 // touches / overlaps after rounding
      if (b > lb) {
        lb = b;
        A.stage[(int64_t)(k - 1) * ncol + c] = make_float2(la, lb);
      }
      return;
    }
    if (!(a < b)) return;                   // zero length after rounding
    if (k >= (uint32_t)A.out_cap) {
      ovf = true;
      return;
    }
    la = a;
    lb = b;
    A.stage[(int64_t)k * ncol + c] = make_float2(a, b);
    ++k;
  };
  int jb = 0;
  for (int ia = 0; ia < np; ++ia) {
    double lo = P[ia].x;
    const double hi = P[ia].y;
    while (jb < nn && N[jb].y <= lo) ++jb;
    int t = jb;
    while (t < nn && N[t].x < hi) {
      if (N[t].x > lo) emit(lo, N[t].x);
      if (N[t].y > lo) lo = N[t].y;
      if (lo >= hi) break;
      ++t;
    }
    if (lo < hi) emit(lo, hi);
  }
  A.cnt[c] = k;
  if (ovf) atomicOr(A.flags, 1u);
}

// ---- tile binning on the device: every shape's conservative tile range, a count per tile, the
// scan (host helper), then the fill; the order of ids inside a tile is arbitrary (the per-column
// unions do not depend on it)
struct RasterBin {
  int nx, nrows, y0, ntx, nsph, nshape;
  const double* sph;
  const double* box;
};

__device__ __forceinline__ bool rs_tile_range(const RasterBin& B, int id, int& t0, int& t1, int& u0, int& u1) {
  double xa, xb, ya, yb;
  if (id < B.nsph) {
    const double* q = B.sph + 4 * (size_t)id;
    xa = q[0] - q[3]; xb = q[0] + q[3]; ya = q[1] - q[3]; yb = q[1] + q[3];
  } else {
    const double* q = B.box + 6 * (size_t)(id - B.nsph);
    xa = q[0]; xb = q[1]; ya = q[2]; yb = q[3];
  }
  const double ia = floor(xa - 0.5) - 1, ib = ceil(xb - 0.5) + 1;
  const double ja = floor(ya - 0.5) - 1 - B.y0, jb = ceil(yb - 0.5) + 1 - B.y0;
  if (!(ib >= 0 && ia <= B.nx - 1 && jb >= 0 && ja <= B.nrows - 1)) return false;
  t0 = (int)fmax(0.0, ia) / RT_X;
  t1 = (int)fmin((double)B.nx - 1, ib) / RT_X;
  u0 = (int)fmax(0.0, ja) / RT_Y;
  u1 = (int)fmin((double)B.nrows - 1, jb) / RT_Y;
  return true;
}

__global__ void raster_bin_count(RasterBin B, uint32_t* __restrict__ cnt) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= B.nshape) return;
  int t0, t1, u0, u1;
  if (!rs_tile_range(B, id, t0, t1, u0, u1)) return;
  for (int u = u0; u <= u1; ++u)
    for (int t = t0; t <= t1; ++t) atomicAdd(cnt + (int64_t)u * B.ntx + t, 1u);
}

__global__ void raster_bin_fill(RasterBin B, const uint64_t* __restrict__ off, uint32_t* __restrict__ cur,
                                int32_t* __restrict__ ids) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= B.nshape) return;
  int t0, t1, u0, u1;
  if (!rs_tile_range(B, id, t0, t1, u0, u1)) return;
  for (int u = u0; u <= u1; ++u)
    for (int t = t0; t <= t1; ++t) {
      const int64_t tile = (int64_t)u * B.ntx + t;
      ids[off[tile] + atomicAdd(cur + tile, 1u)] = id;
    }
}

// ---- the noisy gyroid of config C3 (BASELINE.json configs[2]; SURVEY 8(f) NEXT #3's implicit
// solid): F = sin X cos Y + sin Y cos Z + sin Z cos X, X = 2 pi x / period (same for Y, Z), solid
// where F + eps - t > 0.  F + eps is sampled at z = zmin + m + 1/2 (m = 0 .. nz - 1) with eps =
// amp (2u - 1), u uniform from the counter generator (splitmix64 of key ^ (column * nz + m)),
// linearly interpolated in z; endpoints are the linear roots between samples; beyond the first /
// last sample the field is held (the column's first interval may start at zmin, its last end at
// zmax).  Exactly the host generator's arithmetic (dexelgen.c, dexelgen_gyroid), in fp64 without
// contraction: the sin / cos values come from the host's libm as tables (sn / cs[k] =
// sin / cos(w (k + 1/2))), so the CSR is bitwise the host's.
// One thread per column, two launches: count (FILL = false) and, after the scan, fill.
struct GyroidArgs {
  int nx, nrows, y0, nz, z0;    // columns, local rows (global y0 + jl), samples, integral zmin
  double t, amp, zref;
  uint64_t key;                 // mix64(mix64(seed) ^ stream 6 * K): the generator's per-stream key
  const double* sn;             // [max(nx, y0 + nrows, z0 + nz)]
  const double* cs;
  uint32_t* cnt;                // [ncol] (count launch)
  const uint64_t* off;          // [ncol + 1] (fill launch)
  float2* ep;
};

__device__ __forceinline__ uint64_t gy_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

template <bool FILL>
__global__ void __launch_bounds__(256) gyroid_kernel(GyroidArgs A) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)A.nrows * A.nx) return;
  const int i = (int)(c % A.nx), j = A.y0 + (int)(c / A.nx);
  const double sx = A.sn[i], cx = A.cs[i], sy = A.sn[j], cy = A.cs[j];
  const uint64_t col = (uint64_t)j * (uint64_t)A.nx + (uint64_t)i;
  const double zmin = (double)A.z0, zmax = (double)(A.z0 + A.nz);
  auto field = [&](int m) {
    const double u = (double)(gy_mix64(A.key ^ (col * (uint64_t)A.nz + (uint64_t)m)) >> 11) * (1.0 / 9007199254740992.0);
    const double eps = __dmul_rn(A.amp, __dsub_rn(__dmul_rn(2.0, u), 1.0));
    const double sz = A.sn[A.z0 + m], cz = A.cs[A.z0 + m];
    const double f = __dadd_rn(__dadd_rn(__dmul_rn(sx, cy), __dmul_rn(sy, cz)), __dmul_rn(sz, cx));
    return __dsub_rn(__dadd_rn(f, eps), A.t);
  };
  uint32_t k = 0;
  float la = 0.f, lb = 0.f;   // last output interval (merge target)
  float2* out = FILL ? A.ep + A.off[c] : nullptr;
  // clip, shift to the local frame, round to fp32, canonicalise (dexelgen.c finish_column)
  auto emit = [&](double dlo, double dhi) {
    const double clo = dlo < zmin ? zmin : dlo;
    const double chi = dhi > zmax ? zmax : dhi;
    if (!(clo < chi)) return;
    const float a = (float)__dsub_rn(clo, A.zref), b = (float)__dsub_rn(chi, A.zref);
    if (k > 0 && a <= lb) {
      if (b > lb) {
        lb = b;
        if (FILL) out[k - 1] = make_float2(la, lb);
      }
      return;
    }
    if (!(a < b)) return;
    la = a;
    lb = b;
    if (FILL) out[k] = make_float2(a, b);
    ++k;
  };
  double f0 = field(0);
  bool inside = f0 > 0.0;
  double start = zmin;
  for (int m = 0; m + 1 < A.nz; ++m) {
    const double f1 = field(m + 1);
    const bool nin = f1 > 0.0;
    if (nin != inside) {
      const double zc = __dadd_rn(__dadd_rn((double)(A.z0 + m), 0.5), __ddiv_rn(f0, __dsub_rn(f0, f1)));
      if (nin) start = zc;
      else emit(start, zc);
      inside = nin;
    }
    f0 = f1;
  }
  if (inside) emit(start, zmax);
  if (!FILL) A.cnt[c] = k;
}

}  // namespace dexel
