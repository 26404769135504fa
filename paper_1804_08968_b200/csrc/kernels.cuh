// kernels.cuh -- sm_100a kernels of the separable dexel offset (arXiv 1804.08968).
//
//   validate_kernel   upload check (strictly increasing, finite, in domain)
//   pass1_kernel      pass 1 along x: closest-parent extrusion S_In -> S_Mid
//                     (PAPER.md:494-501).  One warp per 32 output columns of a
//                     row; the warp sweeps z over the window's endpoints (merged
//                     across lanes with a REDUX min on order-preserving keys), keeps
//                     the active neighbour columns as a ballot bitmask and each lane
//                     reads its closest parent kappa = nearest set bit within R.
//   levels4_kernel    the 1D half-space power diagram along z of a column's
//                     pieces (start anchors grow down, end anchors grow up, power
//                     weight W = r^2 - kappa^2 s^2; App. B),
//                     cut at the levels k^2 s^2, k = 0..R:  L_k = U_f(k) u U_r(k)
//                     (2D dilation of the row by sqrt(r^2 - k^2 s^2)).
//   pass2_kernel      pass 2 along y: out(i,j) = U_{|dy|<=R} L_|dy|(i, j+dy)
//                     (a row at lateral distance dy contributes where F >= dy^2,
//                     i.e. power weight r^2 - kappa^2 - dy^2 >= 0), clipped to U,
//                     with the dilate / erode / shell epilogue.
// pass1 and pass2 run twice (two-phase allocation): COUNT writes per-column
// counts, WRITE recomputes and writes at the scanned offsets; levels4 stages its
// output in shared memory and reserves arena blocks with one atomic per column.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dexel {

constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t KEY_NONE = 0xffffffffu;
constexpr int KNONE = 255;  // "no parent within R"

// order-preserving u32 key of a float (-0 folded onto +0)
__device__ __forceinline__ uint32_t fkey(float f) {
  if (f == 0.0f) f = 0.0f;
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float keyf(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// ------------------------------------------------------------------ validate
__global__ void validate_kernel(const uint64_t* __restrict__ off, const float* __restrict__ ep, int64_t ncol,
                                float zlo, float zhi, unsigned long long* __restrict__ first_bad) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  uint64_t a = off[c], b = off[c + 1];
  bool ok = a <= b;
  float prev = -INFINITY;
  for (uint64_t t = a; ok && t < b; ++t) {
    float lo = ep[2 * t], hi = ep[2 * t + 1];
    ok = isfinite(lo) && isfinite(hi) && lo < hi && lo > prev && lo >= zlo && hi <= zhi;
    prev = hi;
  }
  if (!ok) atomicMin(first_bad, (unsigned long long)c);
}

// ------------------------------------------------------------------ pass 1
struct SrcRows {
  const uint64_t* off;  // CSR offsets of the source rows (nrows*nx + 1)
  const float* ep;      // flat endpoints
  int nx, nrows;
  float zlo, zhi;
};

// Virtual endpoint list of one column: S itself, or its complement within
// [zlo,zhi] (complement-on-load): [zlo,a0],[b0,a1],...,[b_{n-1},zhi]
// with zero-length end pieces dropped.  Even virtual index = start, odd = end.
struct ColCursor {
  uint64_t base;
  uint32_t n, v, vend;
};

__device__ __forceinline__ float col_value(const SrcRows& s, const ColCursor& c, uint32_t v, int complement) {
  if (!complement) return __ldg(s.ep + 2 * c.base + v);
  if (v == 0) return s.zlo;
  if (v == 2 * c.n + 1) return s.zhi;
  return __ldg(s.ep + 2 * c.base + v - 1);
}

__device__ __forceinline__ void col_open(const SrcRows& s, int i, int j, int complement, ColCursor& c) {
  if (i < 0 || i >= s.nx || j < 0 || j >= s.nrows) { c.base = 0; c.n = 0; c.v = 0; c.vend = 0; return; }
  size_t col = (size_t)j * s.nx + i;
  uint64_t a = __ldg(s.off + col), b = __ldg(s.off + col + 1);
  c.base = a;
  c.n = (uint32_t)(b - a);
  if (!complement) { c.v = 0; c.vend = 2 * c.n; return; }
  c.v = 0;
  c.vend = 2 * c.n + 2;
  if (c.n > 0 && __ldg(s.ep + 2 * a) <= s.zlo) c.v = 2;                 // S touches z_lo
  if (c.n > 0 && __ldg(s.ep + 2 * (b - 1) + 1) >= s.zhi) c.vend = 2 * c.n;  // S touches z_hi
  if (s.zlo >= s.zhi) c.vend = c.v;
}

// nearest set bit of the window mask to position p, within R (KNONE if none)
template <int NW>
__device__ __forceinline__ int nearest_parent(const uint32_t (&M)[NW], int p, int R) {
  int best = KNONE;
#pragma unroll
  for (int t = 0; t < NW; ++t) {
    uint32_t w = M[t];
    if (!w) continue;
    const int b0 = 32 * t;
    const int sh = p - b0;
    if (sh >= 0) {  // bits at positions <= p
      uint32_t m = sh >= 31 ? w : (w & ((2u << sh) - 1u));
      if (m) best = min(best, p - (b0 + 31 - __clz(m)));
    }
    if (sh <= 31) {  // bits at positions >= p
      uint32_t m = sh <= 0 ? w : (w & ~((1u << sh) - 1u));
      if (m) best = min(best, b0 + __ffs(m) - 1 - p);
    }
  }
  return best <= R ? best : KNONE;
}

template <>
__device__ __forceinline__ int nearest_parent<2>(const uint32_t (&M)[2], int p, int R) {
  const unsigned long long m = ((unsigned long long)M[1] << 32) | M[0];
  const unsigned long long left = m & ((2ull << p) - 1ull);          // positions <= p (p <= 62)
  const unsigned long long right = m >> p;                            // positions >= p
  const int dl = left ? p - (63 - __clzll(left)) : KNONE;
  const int dr = right ? __ffsll(right) - 1 : KNONE;
  const int d = min(dl, dr);
  return d <= R ? d : KNONE;
}

// One warp = output columns [32*tile, 32*tile+32) of output row jr (source row j = row0 + jr).
// NW = number of 32-bit words of the window mask (window = 32 + 2R columns).
// The window's endpoints (S, or its complement within [z_lo, z_hi], as
// order-preserving u32 keys) are first staged in shared memory -- one
// contiguous copy per window column -- so the sweep loop touches no global
// memory; windows larger than the staging area fall back to __ldg reads.
constexpr int P1_WARPS = 4;
constexpr int P1_STAGE = 2048;   // keys per warp (8 KB)

template <int NW, bool WRITE>
__global__ void __launch_bounds__(P1_WARPS * 32) pass1_kernel(SrcRows src, int R, int complement, int row0,
                                                               int nrows_out, uint32_t* __restrict__ cnt,
                                                               const uint64_t* __restrict__ moff,
                                                               float2* __restrict__ mz, uint8_t* __restrict__ mk) {
  __shared__ uint32_t stage_all[P1_WARPS][P1_STAGE];
  const int lane = threadIdx.x & 31;
  uint32_t* stage = stage_all[threadIdx.x >> 5];
  const int ntiles = (src.nx + 31) >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= (int64_t)nrows_out * ntiles) return;  // warp-uniform
  const int jr = (int)(gw / ntiles), tile = (int)(gw % ntiles);
  const int j = row0 + jr;
  const int i0 = tile * 32;
  const int W = 32 + 2 * R;

  ColCursor cur[NW];
  uint32_t sb[NW], pos[NW], end[NW], nkey[NW];
  uint32_t total = 0;
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    const int w = lane + 32 * q;
    if (w < W) col_open(src, i0 - R + w, j, complement, cur[q]);
    else { cur[q].base = 0; cur[q].n = 0; cur[q].v = 0; cur[q].vend = 0; }
    const uint32_t nv = cur[q].vend - cur[q].v;
    uint32_t incl = nv;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, d);
      if (lane >= d) incl += y;
    }
    sb[q] = total + incl - nv;
    total += __shfl_sync(FULL, incl, 31);
  }
  const bool staged = total <= (uint32_t)P1_STAGE;
  if (staged) {
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      const uint32_t nv = cur[q].vend - cur[q].v;
      for (uint32_t t = 0; t < nv; ++t) stage[sb[q] + t] = fkey(col_value(src, cur[q], cur[q].v + t, complement));
      pos[q] = sb[q];
      end[q] = sb[q] + nv;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < NW; ++q) nkey[q] = pos[q] < end[q] ? stage[pos[q]] : KEY_NONE;
  } else {
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      pos[q] = cur[q].v;
      end[q] = cur[q].vend;
      nkey[q] = pos[q] < end[q] ? fkey(col_value(src, cur[q], pos[q], complement)) : KEY_NONE;
    }
  }

  const int i = i0 + lane;
  const bool out_ok = i < src.nx;
  const int64_t c = (int64_t)jr * src.nx + i;
  uint64_t wbase = 0;
  if (WRITE && out_ok) wbase = moff[c];
  uint32_t npieces = 0;
  uint32_t act = 0;
  int kap = KNONE;
  float zstart = 0.f;

  for (;;) {
    uint32_t my = KEY_NONE;
#pragma unroll
    for (int q = 0; q < NW; ++q) my = min(my, nkey[q]);
    const uint32_t zk = __reduce_min_sync(FULL, my);
    if (zk == KEY_NONE) break;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      if (nkey[q] == zk) {
        // virtual index parity: even = interval start (cur.v is even)
        const uint32_t rel = pos[q] - (staged ? sb[q] : 0u) + (staged ? cur[q].v : 0u);
        act = (rel & 1u) == 0u ? (act | (1u << q)) : (act & ~(1u << q));
        ++pos[q];
        nkey[q] = pos[q] < end[q] ? (staged ? stage[pos[q]] : fkey(col_value(src, cur[q], pos[q], complement)))
                                  : KEY_NONE;
      }
    }
    uint32_t M[NW];
#pragma unroll
    for (int t = 0; t < NW; ++t) M[t] = __ballot_sync(FULL, (act >> t) & 1u);
    const int knew = nearest_parent<NW>(M, lane + R, R);
    if (knew != kap) {
      const float z = keyf(zk);
      if (kap != KNONE && out_ok) {
        if (WRITE) {
          mz[wbase + npieces] = make_float2(zstart, z);
          mk[wbase + npieces] = (uint8_t)kap;
        }
        ++npieces;
      }
      kap = knew;
      zstart = z;
    }
  }
  if (!WRITE && out_ok) cnt[c] = npieces;
}

// ------------------------------------------------------------------ levels
// Superlevel sets of the 1D half-space power diagram of a column's pieces.
// A piece p = (lo, hi, kappa) of S_Mid is a segment with power weight
// W_p = r^2 - kappa^2 s^2 (weight r^2 per P:1084-1088).  Seen
// from a row at lateral distance k (pass 2 offset dy = +-k) its capsule
// cuts the ray in [lo - h, hi + h], h = h(kappa,k) =
// sqrt(W_p - k^2 s^2), valid iff W_p >= k^2 s^2.  Level k of column c:
//   L_k(c) = U_{p valid at k} [lo_p - h, hi_p + h]
// = the 2D dilation of the row at radius sqrt(r^2 - k^2 s^2), evaluated at c.
// Split by the half-space decomposition (start anchors grow DOWN, end anchors UP):
//   U_f(k) = U_p [lo_p, hi_p + h]   (box + end anchor)    -- ascending running union
//   U_r(k) = U_p [lo_p - h, hi_p]   (box + start anchor)  -- descending running union
// so L_k = U_f(k) u U_r(k) and each half needs O(1) state per level: the pieces
// are sorted by z, U_f intervals start at lo_p (ascending) and U_r intervals end
// at hi_p (descending).  Pass 2 consumes the halves directly.
//
// Layout: one warp handles G = 32/(R+1) columns (R < 32) or one column with
// NS = ceil((R+1)/32) level slots per lane; lane (g, k) runs level k of column
// g.  Pieces are loaded coalesced and broadcast with shuffles.  Results are
// staged per lane in shared memory, then the column reserves a contiguous block
// of the output arena with one atomicAdd and copies out; per column a
// directory (block base, prefix of the 2(R+1) list starts) locates the lists.
// A lane whose list outgrows its staging slot makes its column recompute the
// lists writing straight to the reserved block.
struct LevelTables {
  const float* h;      // [(R+1)^2] fl32(sqrt(r^2 - (kappa^2+k^2) s^2)), -1 where negative
  int R;
};

struct LevelOut {
  uint64_t* dbase;              // [ncol] arena offset of the column's block
  uint32_t* rel;                // [ncol * (2(R+1)+1)] list starts relative to dbase, last = total
  float2* arena;
  uint64_t cap;                 // arena capacity (intervals)
  unsigned long long* counter;  // arena fill (may exceed cap: host reallocates and reruns)
};

// One thread per column ("lanes = columns"): the 2(R+1) running unions live in
// registers (LMAX = compile-time bound on R+1, unrolled), pieces are read with
// a one-piece prefetch.  The kernel makes two passes over the column's pieces:
// COUNT (per-list counts, packed u16 pairs), then reserves the column's block
// in the arena with one atomicAdd, writes the directory, and WRITE re-runs the
// unions storing each list at its place (U_r, produced descending, is stored
// from the end of its list).  No separate count kernel, scan or host sync.
// ---- lanes = levels variant (used for R >= 33, where the register-resident
// per-column state of levels5 no longer fits): one warp per column, lane k
// (plus 32*s for slot s) runs level k; pieces are loaded coalesced and broadcast
// with shuffles; lists are staged per lane in shared memory and copied to the
// column's arena block after one atomicAdd; a staging overflow makes the warp
// recompute writing straight to the block.
constexpr int STG_C = 16;   // staged intervals per lane, per (direction, level slot)

template <int NS>
struct Lv4Cfg {
  static constexpr int WARPS = NS == 1 ? 8 : (NS == 2 ? 4 : (NS <= 4 ? 2 : 1));
};

template <int NS>
__global__ void __launch_bounds__(Lv4Cfg<NS>::WARPS * 32) levels4_kernel(
    int64_t ncol, const uint64_t* __restrict__ moff, const float2* __restrict__ mz, const uint8_t* __restrict__ mk,
    LevelTables T, int h_in_smem, float zlo, float zhi, LevelOut O) {
  constexpr int WARPS = Lv4Cfg<NS>::WARPS;
  extern __shared__ float4 lv4_smem4[];
  float2* stg_all = reinterpret_cast<float2*>(lv4_smem4);                       // [WARPS][2][NS][STG_C][32]
  float* Hsm = reinterpret_cast<float*>(stg_all + WARPS * 2 * NS * STG_C * 32);  // [(R+1)^2] if h_in_smem
  const int R = T.R, L = R + 1;
  if (h_in_smem) {
    for (int t = threadIdx.x; t < L * L; t += blockDim.x) Hsm[t] = T.h[t];
    __syncthreads();
  }
  const float* Hs = h_in_smem ? Hsm : T.h;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int G = NS == 1 ? 32 / L : 1;
  const int LC = NS == 1 ? L : 32;
  const int g = lane / LC, u0 = lane % LC;
  const int64_t c = ((int64_t)blockIdx.x * WARPS + wib) * G + g;
  const bool col_ok = g < G && c < ncol;
  float2* stg = stg_all + (size_t)wib * 2 * NS * STG_C * 32 + lane;             // stg[((dir*NS+s)*STG_C + i)*32]
  uint64_t base = 0;
  int m = 0;
  if (col_ok) { base = moff[c]; m = (int)(moff[c + 1] - base); }
  const int mmax = __reduce_max_sync(FULL, (unsigned)m);
  int kk[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) kk[s] = u0 + 32 * s;
  uint32_t cnt[2][NS];
  uint32_t ncur[2][NS] = {};
  uint64_t dst[2][NS] = {};
  bool ovf = false;
  bool direct = false, wr = false;

  // dir 0 -> U_f ascending, dir 1 -> U_r descending
  auto run_dir = [&](int dir) {
    float a[NS], b[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) { a[s] = dir ? INFINITY : 0.f; b[s] = dir ? 0.f : -INFINITY; cnt[dir][s] = 0; }
    auto emit = [&](int s, float lo, float hi) {
      lo = fmaxf(lo, zlo);
      hi = fminf(hi, zhi);
      if (!(lo < hi)) return;
      const uint32_t i = cnt[dir][s]++;
      if (direct) {
        if (wr) O.arena[dir ? dst[dir][s] + ncur[dir][s] - 1 - i : dst[dir][s] + i] = make_float2(lo, hi);
      } else if (i < STG_C) {
        stg[((dir * NS + s) * STG_C + i) * 32] = make_float2(lo, hi);
      } else {
        ovf = true;
      }
    };
    for (int t0 = 0; t0 < mmax; t0 += LC) {
      float2 pz = make_float2(0.f, 0.f);
      int pk = 0;
      const int ti = t0 + u0;
      if (ti < m) {
        const uint64_t idx = base + (dir ? (uint64_t)(m - 1 - ti) : (uint64_t)ti);
        pz = mz[idx];
        pk = mk[idx];
      }
      const int nu = min(LC, mmax - t0);
      for (int u = 0; u < nu; ++u) {
        const int srcl = g * LC + u;
        const float lo = __shfl_sync(FULL, pz.x, srcl);
        const float hi = __shfl_sync(FULL, pz.y, srcl);
        const int kap = __shfl_sync(FULL, pk, srcl);
        if (!col_ok || t0 + u >= m) continue;
        const float* hrow = Hs + kap * L;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          if (kk[s] > R) continue;
          const float h = hrow[kk[s]];
          if (h < 0.f) continue;
          if (dir == 0) {
            const float e = hi + h;
            if (lo <= b[s]) b[s] = fmaxf(b[s], e);
            else { if (b[s] > -INFINITY) emit(s, a[s], b[s]); a[s] = lo; b[s] = e; }
          } else {
            const float st = lo - h;
            if (hi >= a[s]) a[s] = fminf(a[s], st);
            else { if (a[s] < INFINITY) emit(s, a[s], b[s]); a[s] = st; b[s] = hi; }
          }
        }
      }
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (!col_ok || kk[s] > R) continue;
      if (dir == 0 ? b[s] > -INFINITY : a[s] < INFINITY) emit(s, a[s], b[s]);
    }
  };
  run_dir(0);
  run_dir(1);

  // list starts in task order (dir, k), prefix inside the column group
  uint32_t pre[2][NS], tot = 0;
  {
    uint32_t run = 0;
#pragma unroll
    for (int dir = 0; dir < 2; ++dir)
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const uint32_t v = (col_ok && kk[s] <= R) ? cnt[dir][s] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(FULL, incl, d);
          if (u0 >= d) incl += y;
        }
        const uint32_t gsum = __shfl_sync(FULL, incl, g * LC + LC - 1);
        pre[dir][s] = run + incl - v;
        run += gsum;
      }
    tot = run;
  }
  unsigned long long blk = 0;
  if (col_ok && u0 == 0) blk = atomicAdd(O.counter, (unsigned long long)tot);
  blk = __shfl_sync(FULL, blk, g * LC);
  const int ntask = 2 * L;
  if (col_ok) {
    if (u0 == 0) {
      O.dbase[c] = blk;
      O.rel[c * (ntask + 1) + ntask] = tot;
    }
#pragma unroll
    for (int dir = 0; dir < 2; ++dir)
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if (kk[s] <= R) O.rel[c * (ntask + 1) + dir * L + kk[s]] = pre[dir][s];
  }
  wr = col_ok && blk + tot <= O.cap;   // else: the host grows the arena and reruns
  const bool any_ovf = __any_sync(FULL, ovf && col_ok);
  if (!any_ovf) {
    if (wr) {
#pragma unroll
      for (int dir = 0; dir < 2; ++dir)
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          if (kk[s] > R) continue;
          const uint64_t o = blk + pre[dir][s];
          const uint32_t n = cnt[dir][s];
          for (uint32_t i = 0; i < n; ++i) {
            const float2 v = stg[((dir * NS + s) * STG_C + i) * 32];
            O.arena[dir ? o + n - 1 - i : o + i] = v;     // U_r was produced descending
          }
        }
    }
    return;
  }
  // a staging slot overflowed somewhere in this warp: recompute writing straight to the blocks
  direct = true;
#pragma unroll
  for (int dir = 0; dir < 2; ++dir)
#pragma unroll
    for (int s = 0; s < NS; ++s) { dst[dir][s] = blk + pre[dir][s]; ncur[dir][s] = cnt[dir][s]; }
  run_dir(0);
  run_dir(1);
}

// Branch-free inner loop: per (piece, level) a table load, an add, two compares
// and selects; an interval is emitted (counted, or stored with a predicated
// store) only when a new component starts.  The h table is padded to LMAX
// columns (-1 = invalid) so no level bound is tested in the loop.
template <int LMAX, bool WRITE>
__device__ __forceinline__ void lv5_unions(const float* __restrict__ Hs, const float2* __restrict__ mz,
                                           const uint8_t* __restrict__ mk, uint64_t base, int m, float zlo, float zhi,
                                           float2* __restrict__ arena, uint64_t blk, uint32_t (&cf)[LMAX],
                                           uint32_t (&cr)[LMAX]) {
  float a[LMAX], b[LMAX];
  // ---- U_f: ascending running union of [lo, hi + h]
#pragma unroll
  for (int k = 0; k < LMAX; ++k) { a[k] = 0.f; b[k] = -INFINITY; }
  float2 nz = m > 0 ? mz[base] : make_float2(0.f, 0.f);
  int nk = m > 0 ? mk[base] : 0;
  for (int t = 0; t < m; ++t) {
    const float2 p = nz;
    const float* hrow = Hs + nk * LMAX;
    if (t + 1 < m) { nz = mz[base + t + 1]; nk = mk[base + t + 1]; }   // prefetch
#pragma unroll
    for (int k = 0; k < LMAX; ++k) {
      const float h = hrow[k];
      const bool valid = h >= 0.f;
      const float e = p.y + h;
      const bool brk = valid && p.x > b[k];
      const float lo = fmaxf(a[k], zlo), hi = fminf(b[k], zhi);
      const bool ok = brk && lo < hi;                 // b = -inf never passes lo < hi
      if (WRITE) { if (ok) arena[blk + cf[k]] = make_float2(lo, hi); }
      cf[k] += ok ? 1u : 0u;
      a[k] = brk ? p.x : a[k];
      b[k] = valid ? (brk ? e : fmaxf(b[k], e)) : b[k];
    }
  }
#pragma unroll
  for (int k = 0; k < LMAX; ++k) {
    const float lo = fmaxf(a[k], zlo), hi = fminf(b[k], zhi);
    const bool ok = lo < hi;
    if (WRITE) { if (ok) arena[blk + cf[k]] = make_float2(lo, hi); }
    cf[k] += ok ? 1u : 0u;
  }
  // ---- U_r: descending running union of [lo - h, hi]; stored from the end of its list
#pragma unroll
  for (int k = 0; k < LMAX; ++k) { a[k] = INFINITY; b[k] = 0.f; }
  nz = m > 0 ? mz[base + m - 1] : make_float2(0.f, 0.f);
  nk = m > 0 ? mk[base + m - 1] : 0;
  for (int t = m - 1; t >= 0; --t) {
    const float2 p = nz;
    const float* hrow = Hs + nk * LMAX;
    if (t > 0) { nz = mz[base + t - 1]; nk = mk[base + t - 1]; }
#pragma unroll
    for (int k = 0; k < LMAX; ++k) {
      const float h = hrow[k];
      const bool valid = h >= 0.f;
      const float st = p.x - h;
      const bool brk = valid && p.y < a[k];
      const float lo = fmaxf(a[k], zlo), hi = fminf(b[k], zhi);
      const bool ok = brk && lo < hi;                 // a = +inf never passes lo < hi
      if (WRITE) { if (ok) arena[blk + cr[k] - 1] = make_float2(lo, hi); }
      cr[k] += WRITE ? (ok ? ~0u : 0u) : (ok ? 1u : 0u);
      b[k] = brk ? p.y : b[k];
      a[k] = valid ? (brk ? st : fminf(a[k], st)) : a[k];
    }
  }
#pragma unroll
  for (int k = 0; k < LMAX; ++k) {
    const float lo = fmaxf(a[k], zlo), hi = fminf(b[k], zhi);
    const bool ok = lo < hi;
    if (WRITE) { if (ok) arena[blk + cr[k] - 1] = make_float2(lo, hi); }
    cr[k] += WRITE ? (ok ? ~0u : 0u) : (ok ? 1u : 0u);
  }
}

// LMAX <= 17: registers (fully unrolled).  Larger R use levels4_kernel.
template <int LMAX>
__global__ void __launch_bounds__(128) levels5_kernel(int64_t ncol, const uint64_t* __restrict__ moff,
                                                      const float2* __restrict__ mz, const uint8_t* __restrict__ mk,
                                                      LevelTables T, float zlo, float zhi, LevelOut O) {
  __shared__ float lv5_h[LMAX * LMAX];
  const int R = T.R, L = R + 1;
  for (int t = threadIdx.x; t < LMAX * LMAX; t += blockDim.x) {
    const int kap = t / LMAX, k = t % LMAX;
    lv5_h[t] = (kap < L && k < L) ? T.h[kap * L + k] : -1.0f;
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const uint64_t base = moff[c];
  const int m = (int)(moff[c + 1] - base);
  uint32_t cf[LMAX], cr[LMAX];
#pragma unroll
  for (int k = 0; k < LMAX; ++k) { cf[k] = 0; cr[k] = 0; }
  lv5_unions<LMAX, false>(lv5_h, mz, mk, base, m, zlo, zhi, O.arena, 0, cf, cr);   // COUNT
  uint32_t tot = 0;
  const int ntask = 2 * L;
  uint32_t* rl = O.rel + c * (ntask + 1);
#pragma unroll
  for (int k = 0; k < LMAX; ++k)
    if (k < L) { rl[k] = tot; const uint32_t n = cf[k]; cf[k] = tot; tot += n; }
#pragma unroll
  for (int k = 0; k < LMAX; ++k)
    if (k < L) { rl[L + k] = tot; tot += cr[k]; cr[k] = tot; }
  rl[ntask] = tot;
  const unsigned long long blk = atomicAdd(O.counter, (unsigned long long)tot);
  O.dbase[c] = blk;
  if (blk + tot > O.cap) return;                    // host grows the arena and reruns
  lv5_unions<LMAX, true>(lv5_h, mz, mk, base, m, zlo, zhi, O.arena, blk, cf, cr);  // WRITE
}

// ---- envelope variant (production for every R): O(m + sum_k |L_k|) per column.
// F(z) = max_p g_p(z), g_p(z) = W_p - dist(z, [lo_p, hi_p])^2 (plateau W_p on the
// piece, the start anchor's half-parabola below it, the end anchor's above it:
// PAPER.md:538-541 with power weights, App. B).  For pieces p below q, g_p - g_q
// is continuous and strictly decreasing, so every pair crosses once and the upper
// envelope is built by the classic stack sweep (Felzenszwalb-Huttenlocher): a new
// piece pops the top while it wins from the top's segment start.  Segments whose
// end lies below lo_q - r can no longer change (a piece grows at most r), so they
// are walked immediately and leave the deque: its depth stays ~ the staircase
// height, not m.  Walking a segment emits the crossings of F with the levels
// k^2 s^2 at the owner's candidates lo - h(kappa,k) / hi + h(kappa,k); L_k is the
// set where F >= k^2 s^2 (= the union of the grown pieces valid at level k).
// Envelope arithmetic is fp64; endpoints are the fp32 table candidates, clamped
// into their segment and rounded once.  Two in-kernel passes (COUNT, WRITE)
// around a per-column arena reservation, as levels5.
constexpr int ENV_D = 256;          // deque capacity (local memory), power of two

struct EnvTables {
  const float* h;     // [(R+1)^2] fl32(sqrt(r^2 - (kappa^2+k^2)s^2)), -1 where negative
  const double* W;    // [R+1] r^2 - kappa^2 s^2
  const double* Tk;   // [R+1] k^2 s^2
  int R;
  double r;           // radius (finalisation window)
  double inv_s2;
};

__device__ __forceinline__ double env_g(double z, double lo, double hi, double W) {
  const double d = lo - z > 0.0 ? lo - z : (z - hi > 0.0 ? z - hi : 0.0);
  return W - d * d;
}

// crossing of g_p and g_q, p below q (lp < hp <= lq < hq): g_p - g_q is strictly decreasing
__device__ __forceinline__ double env_cross(double lp, double hp, double Wp, double lq, double hq, double Wq) {
  const double dW = Wp - Wq;
  // D(z) at the region boundaries
  const double Dlp = dW + (lq - lp) * (lq - lp);
  if (Dlp <= 0.0) return fmin(0.5 * (lq + lp) + dW / (2.0 * (lq - lp)), lp);
  const double Dhp = dW + (lq - hp) * (lq - hp);
  if (Dhp <= 0.0) return fmax(lp, fmin(lq - sqrt(fmax(-dW, 0.0)), hp));
  const double Dlq = dW - (lq - hp) * (lq - hp);
  if (Dlq <= 0.0) return fmax(hp, fmin(0.5 * (lq + hp) + dW / (2.0 * (lq - hp)), lq));
  const double Dhq = dW - (hq - hp) * (hq - hp);
  if (Dhq <= 0.0) return fmax(lq, fmin(hp + sqrt(fmax(dW, 0.0)), hq));
  return fmax(0.5 * (hp + hq) + dW / (2.0 * (hq - hp)), hq);
}

struct EnvEmit {
  float* open_lo;       // smem [L][blockDim] (stride = blockDim)
  uint32_t* cur;        // smem [L][blockDim]: COUNT -> count, WRITE -> next slot
  int stride;
  float2* arena;
  uint64_t blk;
  float zlo, zhi;
  bool write;
  int lam;              // level of the open segment to the left (-1 = outside)
  float zlast;
  __device__ __forceinline__ void rise(int k, float z) { open_lo[k * stride] = z; }
  __device__ __forceinline__ void fall(int k, float z) {
    const float lo = fmaxf(open_lo[k * stride], zlo), hi = fminf(z, zhi);
    if (lo < hi) {
      const uint32_t i = cur[k * stride]++;
      if (write) arena[blk + i] = make_float2(lo, hi);
    }
  }
  __device__ __forceinline__ void set_at(float z, int target) {
    z = fmaxf(z, zlast);
    zlast = z;
    while (lam < target) rise(++lam, z);
    while (lam > target) fall(lam--, z);
  }
};

__device__ __forceinline__ int env_level(const EnvTables& T, double v) {
  if (!(v >= 0.0)) return -1;
  int k = (int)sqrtf((float)(v * T.inv_s2));
  if (k > T.R) k = T.R;
  while (k < T.R && T.Tk[k + 1] <= v) ++k;
  while (k >= 0 && T.Tk[k] > v) --k;
  return k;
}

// walk one envelope segment [zs, ze] owned by piece (lo, hi, kappa)
__device__ __forceinline__ void env_walk(const EnvTables& T, EnvEmit& E, float lo32, float hi32, int kp, double zs,
                                         double ze) {
  const double lo = lo32, hi = hi32, W = T.W[kp];
  const int L = T.R + 1;
  const float* hrow = T.h + kp * L;
  const int kmax = env_level(T, W);
  if (zs < lo) {                                       // down-arc (increasing)
    const double z1 = fmin(ze, lo);
    const int t1 = z1 >= lo ? kmax : env_level(T, env_g(z1, lo, hi, W));
    if (t1 < E.lam) {
      E.set_at((float)zs, t1);
    } else {
      while (E.lam < t1) {
        const int k = E.lam + 1;
        const double zc = fmax(zs, fmin((double)(lo32 - hrow[k]), z1));
        E.set_at((float)zc, k);
      }
    }
  }
  if (zs < hi && ze > lo) {                            // plateau
    if (kmax != E.lam) E.set_at((float)fmax(zs, lo), kmax);
  }
  if (ze > hi) {                                       // up-arc (decreasing)
    const double z0 = fmax(zs, hi);
    const int t1 = ze == INFINITY ? -1 : env_level(T, env_g(ze, lo, hi, W));
    if (t1 > E.lam) {
      E.set_at((float)z0, t1);
    } else {
      while (E.lam > t1) {
        const int k = E.lam;
        const double zc = k <= kmax ? fmax(z0, fmin((double)(hi32 + hrow[k]), ze)) : z0;
        E.set_at((float)zc, k - 1);
      }
    }
  }
}

// full envelope + walk of one column; returns false on deque overflow
__device__ bool env_column(const EnvTables& T, EnvEmit& E, const float2* __restrict__ mz,
                           const uint8_t* __restrict__ mk, uint64_t base, int m) {
  uint32_t dq_i[ENV_D];
  double dq_s[ENV_D];
  int b = 0, n = 0;
  double walked = -INFINITY;
  E.lam = -1;
  E.zlast = -INFINITY;
  const double win = T.r + 1.0;
  for (int q = 0; q < m; ++q) {
    const float2 pq = mz[base + q];
    const int kq = mk[base + q];
    const double Wq = T.W[kq];
    double s = walked;
    while (n > 0) {
      const int t = (b + n - 1) & (ENV_D - 1);
      const uint32_t p = dq_i[t];
      const float2 pp = mz[base + p];
      const double z = env_cross(pp.x, pp.y, T.W[mk[base + p]], pq.x, pq.y, Wq);
      if (z <= dq_s[t]) {
        --n;
      } else {
        s = z;
        break;
      }
    }
    if (n == 0) s = walked;
    if (n == ENV_D) return false;
    const int t = (b + n) & (ENV_D - 1);
    dq_i[t] = (uint32_t)q;
    dq_s[t] = s;
    ++n;
    // finalise: segments ending below lo_q - r cannot change any more
    const double lim = (double)pq.x - win;
    while (n >= 2 && dq_s[(b + 1) & (ENV_D - 1)] <= lim) {
      const uint32_t p = dq_i[b];
      const float2 pp = mz[base + p];
      const double ze = dq_s[(b + 1) & (ENV_D - 1)];
      env_walk(T, E, pp.x, pp.y, mk[base + p], dq_s[b], ze);
      walked = ze;
      b = (b + 1) & (ENV_D - 1);
      --n;
    }
  }
  for (int u = 0; u < n; ++u) {
    const int t = (b + u) & (ENV_D - 1);
    const uint32_t p = dq_i[t];
    const float2 pp = mz[base + p];
    const double ze = u + 1 < n ? dq_s[(t + 1) & (ENV_D - 1)] : INFINITY;
    env_walk(T, E, pp.x, pp.y, mk[base + p], dq_s[t], ze);
  }
  return true;
}

__global__ void __launch_bounds__(128) levels6_kernel(int64_t ncol, const uint64_t* __restrict__ moff,
                                                      const float2* __restrict__ mz, const uint8_t* __restrict__ mk,
                                                      EnvTables T, float zlo, float zhi, LevelOut O) {
  extern __shared__ float4 lv6_smem4[];
  const int L = T.R + 1;
  float* open_lo = reinterpret_cast<float*>(lv6_smem4);            // [L][128]
  uint32_t* cur = reinterpret_cast<uint32_t*>(open_lo + L * 128);  // [L][128]
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const uint64_t base = moff[c];
  const int m = (int)(moff[c + 1] - base);
  for (int k = 0; k < L; ++k) cur[k * 128 + threadIdx.x] = 0;
  EnvEmit E{open_lo + threadIdx.x, cur + threadIdx.x, 128, O.arena, 0, zlo, zhi, false, -1, -INFINITY};
  bool ok = env_column(T, E, mz, mk, base, m);                     // COUNT
  uint32_t tot = 0;
  uint32_t* rl = O.rel + c * (L + 1);
  for (int k = 0; k < L; ++k) {
    const uint32_t v = cur[k * 128 + threadIdx.x];
    rl[k] = tot;
    cur[k * 128 + threadIdx.x] = tot;
    tot += v;
  }
  rl[L] = tot;
  const unsigned long long blk = atomicAdd(O.counter, (unsigned long long)tot);
  O.dbase[c] = blk;
  if (!ok) { atomicExch(O.counter + 1, 1ull); return; }
  if (blk + tot > O.cap) return;                                   // host grows the arena and reruns
  E.blk = blk;
  E.write = true;
  env_column(T, E, mz, mk, base, m);                               // WRITE
}

// ------------------------------------------------------------------ pass 2
struct LevelFamily {
  const uint64_t* dbase;  // [ncol] column block base in the arena
  const uint32_t* rel;    // [ncol * (ndir(R+1)+1)] list starts (dir, k), relative to dbase
  const float2* arena;
  int R;
  int ndir;               // 1: L_k lists (envelope), 2: U_f / U_r halves (running unions)
  int64_t ncol;           // columns (rows_L * nx)
  int row0;               // global row of level row 0
  int nrows;              // rows available
};

constexpr int ACC_CAP = 256;

// union of sorted disjoint A (local) and sorted disjoint B (global) -> out; returns count (may exceed cap)
__device__ __forceinline__ int merge_union(const float2* A, int na, const float2* __restrict__ B, int nb,
                                           float2* out, int cap) {
  int ia = 0, ib = 0, no = 0;
  float cs = 0.f, ce = 0.f;
  bool have = false;
  while (ia < na || ib < nb) {
    float2 x;
    if (ib >= nb || (ia < na && A[ia].x <= B[ib].x)) x = A[ia++];
    else x = B[ib++];
    if (!have) { cs = x.x; ce = x.y; have = true; }
    else if (x.x <= ce) ce = fmaxf(ce, x.y);
    else { if (no < cap) out[no] = make_float2(cs, ce); ++no; cs = x.x; ce = x.y; }
  }
  if (have) { if (no < cap) out[no] = make_float2(cs, ce); ++no; }
  return no;
}

// y-union for output column (i, j): returns count in buf (ACC_CAP-limited, *ovf set on overflow)
__device__ int y_union(const LevelFamily& F, int i, int jg, int nx, float2* a, float2* b, bool* ovf) {
  int na = 0;
  float2* cur = a;
  float2* nxt = b;
  for (int t = 0; t <= 2 * F.R; ++t) {
    const int dy = (t & 1) ? ((t + 1) >> 1) : -(t >> 1);  // 0, 1, -1, 2, -2, ...
    const int jl = jg + dy - F.row0;
    if (jl < 0 || jl >= F.nrows) continue;
    const int k = dy < 0 ? -dy : dy;
    const int64_t cc = (int64_t)jl * nx + i;
    const int ntask = F.ndir * (F.R + 1);
    const uint64_t b0 = F.dbase[cc];
    const uint32_t* rl = F.rel + cc * (ntask + 1);
    for (int dir = 0; dir < F.ndir; ++dir) {
      const int tsk = dir * (F.R + 1) + k;
      const uint32_t s0 = rl[tsk], s1 = rl[tsk + 1];
      if (s1 == s0) continue;
      int n = merge_union(cur, na, F.arena + b0 + s0, (int)(s1 - s0), nxt, ACC_CAP);
      if (n > ACC_CAP) { *ovf = true; n = ACC_CAP; }
      float2* tmp = cur; cur = nxt; nxt = tmp;
      na = n;
    }
  }
  if (cur != a)
    for (int t = 0; t < na; ++t) a[t] = cur[t];
  return na;
}

enum { OP_DILATE = 0, OP_ERODE = 1, OP_SHELL = 2 };

template <int OP, bool WRITE>
__global__ void __launch_bounds__(128) pass2_kernel(LevelFamily FA, LevelFamily FB, int nx, int row0, int nrows_out,
                                                    float zlo, float zhi, uint32_t* __restrict__ ocnt,
                                                    const uint64_t* __restrict__ ooff, float2* __restrict__ oz,
                                                    int* __restrict__ overflow) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)nrows_out * nx) return;
  const int i = (int)(c % nx), jg = row0 + (int)(c / nx);
  float2 a[ACC_CAP], b[ACC_CAP];
  bool ovf = false;
  int na = y_union(FA, i, jg, nx, a, b, &ovf);
  uint64_t w = WRITE ? ooff[c] : 0;
  uint32_t n = 0;
  if (OP == OP_DILATE) {
    if (WRITE) for (int t = 0; t < na; ++t) oz[w + t] = a[t];
    n = na;
  } else if (OP == OP_ERODE) {
    float cur = zlo;
    for (int t = 0; t < na; ++t) {
      if (a[t].x > cur) { if (WRITE) oz[w + n] = make_float2(cur, a[t].x); ++n; }
      cur = a[t].y;
    }
    if (zhi > cur) { if (WRITE) oz[w + n] = make_float2(cur, zhi); ++n; }
  } else {  // shell: D_rout(S) n D_rin(C)
    float2 c2[ACC_CAP];
    int nc = y_union(FB, i, jg, nx, b, c2, &ovf);
    int p = 0, q = 0;
    while (p < na && q < nc) {
      const float lo = fmaxf(a[p].x, b[q].x), hi = fminf(a[p].y, b[q].y);
      if (lo < hi) { if (WRITE) oz[w + n] = make_float2(lo, hi); ++n; }
      if (a[p].y < b[q].y) ++p; else ++q;
    }
  }
  if (!WRITE) ocnt[c] = n;
  if (ovf) atomicExch(overflow, 1);
}

}  // namespace dexel
