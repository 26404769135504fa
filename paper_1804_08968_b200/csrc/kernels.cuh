// kernels.cuh -- sm_100a kernels of the separable dexel offset (arXiv 1804.08968).
//
//   validate_kernel   upload check (strictly increasing, finite, in domain)
//   p1_kernel         pass 1 along x: closest-parent extrusion S_In -> S_Mid
//                     (PAPER.md:494-501).  One warp per 32 output columns of a
//                     row; the warp sweeps z over the window's endpoints (merged
//                     across lanes with a REDUX min on order-preserving keys), keeps
//                     the active neighbour columns as a ballot bitmask and each lane
//                     reads its closest parent kappa = nearest set bit within R.
// The z-resolution (levels.cuh) and pass 2 (pass2.cuh) live in their own headers.
// Pass 1 runs once per band: pieces go to per-column slots, the rare columns that
// outgrow them are recomputed into an arena by a second, list-driven launch.
#pragma once
#include <cstdint>
#include <type_traits>
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
// The rows an op reads, in "extended" numbering 0 .. nrows-1: up to three CSR segments stacked
// along y -- the halo rows below the slab (segment 0: received from rank g-1, DESIGN.md
// "Multi-GPU"), the slab's own rows (1), the halo rows above it (2).  Each segment is a plain
// CSR with offsets starting at 0; no copy joins them.
struct SrcRows {
  const uint64_t* off[3];   // CSR offsets of each segment's rows (rows[s]*nx + 1)
  const float* ep[3];       // flat endpoints of each segment
  int rows[3];
  int nx, nrows;            // nrows = rows[0] + rows[1] + rows[2]
  float zlo, zhi;
};

// Virtual endpoint list of one column: S itself, or its complement within
// [zlo,zhi] (complement-on-load): [zlo,a0],[b0,a1],...,[b_{n-1},zhi]
// with zero-length end pieces dropped.  Even virtual index = start, odd = end.
struct ColCursor {
  const float* p;   // the column's first endpoint
  uint32_t n, v, vend;
};

__device__ __forceinline__ float col_value(const SrcRows& s, const ColCursor& c, uint32_t v, int complement) {
  if (!complement) return __ldg(c.p + v);
  if (v == 0) return s.zlo;
  if (v == 2 * c.n + 1) return s.zhi;
  return __ldg(c.p + v - 1);
}

__device__ __forceinline__ void col_close(ColCursor& c) { c.p = nullptr; c.n = 0; c.v = 0; c.vend = 0; }

__device__ __forceinline__ void col_open(const SrcRows& s, int i, int j, int complement, ColCursor& c) {
  if (i < 0 || i >= s.nx || j < 0 || j >= s.nrows) { col_close(c); return; }
  int seg = 0;
  if (j >= s.rows[0]) { j -= s.rows[0]; seg = 1; }
  if (seg == 1 && j >= s.rows[1]) { j -= s.rows[1]; seg = 2; }
  const uint64_t* off = s.off[seg];
  size_t col = (size_t)j * s.nx + i;
  uint64_t a = __ldg(off + col), b = __ldg(off + col + 1);
  c.p = s.ep[seg] + 2 * a;
  c.n = (uint32_t)(b - a);
  if (!complement) { c.v = 0; c.vend = 2 * c.n; return; }
  c.v = 0;
  c.vend = 2 * c.n + 2;
  if (c.n > 0 && __ldg(c.p) <= s.zlo) c.v = 2;                              // S touches z_lo
  if (c.n > 0 && __ldg(c.p + 2 * (c.n - 1) + 1) >= s.zhi) c.vend = 2 * c.n;  // S touches z_hi
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

// Pass-1 output: the pieces of every column of a band of rows in per-column slots.
// Slot-major: piece t of column (row, i) at z[(row*(cap+1) + t)*nx + i] -- a warp of 32
// consecutive columns reads (levels kernel) 256 contiguous bytes per slot.  Slot `cap` is a
// spill cell: writes beyond cap are clamped there, the column is listed, and a second
// launch ("list mode") rewrites the listed columns' pieces into an arena of ovf_cap pieces
// per column.
struct PieceSlots {
  float2* z;           // [nrows][cap+1][nx]  (lo, hi)
  uint8_t* k;          // [nrows][cap+1][nx]  kappa
  uint32_t* cnt;       // [nrows*nx]          true piece count
  int cap, nx, nrows;
  int32_t* ovf_idx;    // [nrows*nx] arena slot of an overflow column, -1 elsewhere
  float2* ovf_z;       // [n_ovf][ovf_cap]
  uint8_t* ovf_k;
  int ovf_cap;
  uint32_t* ovf_list;  // overflow columns (main pass appends)
  unsigned ovf_list_cap;
  uint32_t* tile_flag; // [nrows * ntiles] a tile holds an overflow column
  uint32_t* tile_list; // tiles to rerun in list mode
  unsigned* flags;     // [0] overflow columns, [1] longest column (when > cap), [2] tiles listed
  unsigned long long* total;   // pieces (statistics)
};

__host__ __device__ __forceinline__ size_t piece_index(const PieceSlots& P, int row, int t, int i) {
  return ((size_t)row * (P.cap + 1) + t) * P.nx + i;
}

// One warp = output columns [32*tile, 32*tile+32) of output row jr (source row j = row0 + jr).
// NW = number of 32-bit words of the window mask (window = 32 + 2R columns).
// The window's endpoints (S, or its complement within [z_lo, z_hi], as order-preserving
// u32 keys) are first staged in shared memory -- one contiguous copy per window column --
// so the sweep touches no global memory (windows larger than the staging area read
// through __ldg).  Each step of the sweep takes the next z over the whole window with one
// REDUX min, toggles the window's activity mask with one ballot per word (a column's
// events alternate start / end), and every lane reads its closest parent
// kappa = min |dx| as the nearest set bit within R of its own position.
// Pure selection: lo / hi are copies of input values, kappa an integer.
constexpr int P1_WARPS = 4;
constexpr int P1_STAGE = 2048;   // keys per warp (8 KB)
constexpr int P1_RING = 8;       // pending closed pieces per lane

// Capsule domination (prune != nullptr): piece q dominates piece p when kappa_q <= kappa_p and
//   max(lo_q - lo_p, hi_p - hi_q) <= h(kappa_q, 0) - h(kappa_p, 0),   h(kappa, k) = sqrt(r^2 - (kappa^2+k^2)s^2):
// h(kappa_q,k) - h(kappa_p,k) grows with k, so then p's capsule cross-section lies inside q's at
// every level where p reaches, and dropping p leaves every level set L_k -- hence the result --
// unchanged (the union of the capsules is all pass 2 needs).  Each lane keeps
// its last piece pending and tests it against the next one (a dominated staircase step of a
// sphere is typically shorter than the h difference of its neighbour): about 45% of the pieces
// of the synthetic configs go.  The next piece n lies above the pending one p, so the two tests
// reduce to  n dominates p: kn <= kp and lo_n - lo_p <= H[kn] - H[kp];  p dominates n:
// kp <= kn and hi_n - hi_p <= H[kp] - H[kn]  (H = h(., 0), fp32).  Both sides are differences
// of nearby values.  A piece is only dropped with a margin of 1e-6 (1 + |D|) + 16 r 2^-24
// (prune[R+1]): the H table rounds each h(., 0) <= r by <= ulp(r)/2 and the two differences
// round by <= ulp(r)/2 each, so a dropped piece's capsule lies inside the dominating one's in
// exact arithmetic with a slack of >= ulp(r) at level 0 (the margin 16 r 2^-24 is >= 8 ulp(r);
// the threshold's own fp32 roundings and that of z - phi cost at most 3.5 ulp(r)) -- and the slack only grows with the
// level k -- which also covers the fp32 rounding of the level-k grown endpoints
// fl32(lo - fl32(h)): pruning leaves the output bitwise unchanged (GPU test against
// DEXEL_NO_PRUNE=1).  Rounding can keep a dominated piece, never drop a needed one.
// predicated store of one piece (8-byte z pair + kappa byte) without a branch
__device__ __forceinline__ void st_pred_piece(float2* zp, uint8_t* kp, float lo, float hi, int k, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.global.v2.f32 [%0], {%2, %3};\n\t"
               "@q st.global.u8 [%1], %4;\n\t}"
               :: "l"(zp), "l"(kp), "f"(lo), "f"(hi), "r"(k), "r"((int)pred));
}

__device__ __forceinline__ bool dom_margin(float lhs, float rhs, float mabs) {
  return lhs <= rhs - 1e-6f * (1.0f + fabsf(rhs)) - mabs;
}

// capsule-domination thresholds of every (pending kappa, new kappa) pair (see p1_kernel)
__device__ __forceinline__ void p1_thr_init(float2* thr, const float* __restrict__ prune, int R) {
  const float mabs = prune[R + 1];   // absolute part of the margin (16 r 2^-24, see above)
  for (int t = threadIdx.x; t < 18 * 32; t += blockDim.x) {
    const int kp = t >> 5, kn = t & 31;
    float2 v = make_float2(-INFINITY, -INFINITY);
    if (kp <= R && kn <= R) {
      const float D = prune[kp] - prune[kn];                // H[kp] - H[kn]
      if (kp <= kn) v.x = D - 1e-6f * (1.0f + fabsf(D)) - mabs;    // drop new:     hi_n - hi_p <= x
      if (kn <= kp) v.y = -D - 1e-6f * (1.0f + fabsf(D)) - mabs;   // drop pending: lo_n - lo_p <= y
    }
    thr[t] = v;
  }
}

// SKIP (host: R >= 8): steps where no lane's kappa changes skip the filter / emission half
template <int NW, bool RING, bool SKIP = true>
__global__ void __launch_bounds__(P1_WARPS * 32) p1_kernel(SrcRows src, int R, int complement, int row0,
                                                            int jr0, int nrows_out, PieceSlots P, int64_t nlist,
                                                            const float* __restrict__ prune) {
  __shared__ uint32_t stage_all[P1_WARPS][P1_STAGE];
  __shared__ float h0[256];
  // NW == 2 (R <= 16), inline filter: both domination thresholds of every (pending kappa,
  // new kappa) pair, margin included: x for "new dominates pending", y for "pending
  // dominates new"; -inf where the kappa order rules the test out, in the row of "no pending
  // piece" (17) and the column of KNONE (31)
  __shared__ float2 thr[(NW == 2 && !RING) ? 18 * 32 : 1];
  __shared__ float2 ring_z[P1_WARPS][RING ? P1_RING : 1][32];   // closed pieces awaiting the filter / store
  __shared__ uint8_t ring_k[P1_WARPS][RING ? P1_RING : 1][32];
  const float mabs = prune ? prune[R + 1] : 0.f;   // absolute part of the domination margin
  if (prune) {
    for (int t = threadIdx.x; t <= R; t += blockDim.x) h0[t] = prune[t];
    if constexpr (NW == 2 && !RING) p1_thr_init(thr, prune, R);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t* stage = stage_all[threadIdx.x >> 5];
  const int ntiles = (src.nx + 31) >> 5;
  const bool list_mode = nlist >= 0;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= (list_mode ? nlist : (int64_t)nrows_out * ntiles)) return;  // warp-uniform
  // main mode: slot rows jr0 .. jr0 + nrows_out - 1 of the band; list mode: the listed tiles
  const int64_t tl = list_mode ? (int64_t)P.tile_list[gw] : gw + (int64_t)jr0 * ntiles;
  const int jr = (int)(tl / ntiles), tile = (int)(tl % ntiles);
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
    else col_close(cur[q]);
    const uint32_t nv = cur[q].vend - cur[q].v + 1;    // + a KEY_NONE sentinel
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
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    const uint32_t nv = cur[q].vend - cur[q].v;
    if (staged) {
      for (uint32_t t = 0; t < nv; ++t) stage[sb[q] + t] = fkey(col_value(src, cur[q], cur[q].v + t, complement));
      stage[sb[q] + nv] = KEY_NONE;             // sentinel: the advance needs no bound check
      pos[q] = sb[q];
      end[q] = sb[q] + nv;
    } else {
      pos[q] = cur[q].v;
      end[q] = cur[q].vend;
    }
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < NW; ++q)
    nkey[q] = pos[q] < end[q] ? (staged ? stage[pos[q]] : fkey(col_value(src, cur[q], pos[q], complement)))
                              : KEY_NONE;

  const int i = i0 + lane;
  const bool out_ok = i < src.nx;
  const int64_t c = (int64_t)jr * src.nx + i;
  // where this lane's pieces go: slots (main pass), the arena (list mode, overflow columns), or
  // nowhere -- then the stores go to a spill cell (slot cap of a column of this row, never read),
  // so the store predicate needs no extra term
  float2* zb = P.z + piece_index(P, jr, P.cap, out_ok ? i : 0);
  uint8_t* kb = P.k + piece_index(P, jr, P.cap, out_ok ? i : 0);
  uint32_t zstep = 0, tmax = 0;
  bool has_out = false;
  if (out_ok) {
    if (!list_mode) {
      zb = P.z + piece_index(P, jr, 0, i);
      kb = P.k + piece_index(P, jr, 0, i);
      zstep = (uint32_t)P.nx;
      tmax = (uint32_t)P.cap;                      // spill cell
      has_out = true;
    } else if (P.ovf_idx[c] >= 0) {
      const size_t q = (size_t)P.ovf_idx[c] * P.ovf_cap;
      zb = P.ovf_z + q;
      kb = P.ovf_k + q;
      zstep = 1;
      tmax = (uint32_t)P.ovf_cap - 1;
      has_out = true;
    }
  }
  // opaque per-lane base pointers (as in p1_fam_init: no per-store 64-bit index arithmetic)
  asm("mov.b64 %0, %0;" : "+l"(zb));
  asm("mov.b64 %0, %0;" : "+l"(kb));
  uint32_t M[NW];
#pragma unroll
  for (int q = 0; q < NW; ++q) M[q] = 0u;          // window activity mask (warp-uniform)
  uint32_t np = 0;
  int kap = KNONE;
  float zstart = 0.f;
  // pending piece of the capsule-domination filter (hpk caches H[pk])
  float plo = 0.f, phi = 0.f, hpk = 0.f;
  int pk = KNONE;
  uint32_t woff = 0;                       // next slot (float2 / byte offset from zb / kb)
  const uint32_t wlim = tmax * zstep;      // the spill cell
  auto put = [&](float lo, float hi, int k) {
    if (has_out) {
      const uint32_t t = min(np, tmax);
      zb[(size_t)t * zstep] = make_float2(lo, hi);
      kb[(size_t)t * zstep] = (uint8_t)k;
    }
    ++np;
  };
  // Small R: closed pieces enter a per-lane ring in shared memory (a few predicated
  // instructions per sweep step); the filter and the global stores run when some lane's ring
  // is full, once per piece instead of once per step (some lane closes a piece at almost every
  // step).  Larger R (more work per step elsewhere, fewer closes per step): inline.
  constexpr bool use_ring = RING;   // host: R < 8
  const int wid = threadIdx.x >> 5;
  uint32_t rc = 0, rd = 0;                 // ring: written / drained
  auto drain = [&]() {
    const uint32_t nd = __reduce_max_sync(FULL, rc - rd);
    for (uint32_t u = 0; u < nd; ++u) {
      if (rd == rc) continue;
      const float2 v = ring_z[wid][rd % P1_RING][lane];
      const int kv = ring_k[wid][rd % P1_RING][lane];
      ++rd;
      if (!prune) {
        put(v.x, v.y, kv);
      } else if (pk == KNONE) {
        plo = v.x; phi = v.y; pk = kv;
      } else {
        const float D = h0[pk] - h0[kv];                    // H[kp] - H[kn]
        if (pk <= kv && dom_margin(v.y - phi, D, mabs)) continue; // the pending piece covers the new one
        if (!(kv <= pk && dom_margin(v.x - plo, -D, mabs))) put(plo, phi, pk);
        plo = v.x; phi = v.y; pk = kv;
      }
    }
    __syncwarp();
  };
  // NW == 2 (R <= 16): the closest parent from two 32-bit windows of the 64-bit mask around this
  // lane's position p = lane + R: the bits at or below p (top-aligned) and at or above p
  const int pp = lane + R;
  const int shr = pp < 32 ? pp : pp - 32;          // right window: bits p .. p+31
  const int shl = pp >= 31 ? pp - 31 : 31 - pp;    // left window: bits p-31 .. p, bit p on top
  const bool rlow = pp < 32, lhigh = pp >= 31;      // per-lane constants: selects, not branches
  // (a sentinel bit at distance 31 > R keeps both windows non-zero: no zero tests)
  auto nearest2 = [&](uint32_t m0, uint32_t m1) -> int {
    const uint32_t rw = __funnelshift_r(rlow ? m0 : m1, rlow ? m1 : 0u, shr) | 0x80000000u;
    const uint32_t la = __funnelshift_r(m0, m1, shl), lb = __funnelshift_l(0u, m0, shl);
    const uint32_t lw = (lhigh ? la : lb) | 1u;
    const int d = min(__clz(lw), __ffs(rw) - 1);
    return d <= R ? d : KNONE;
  };
  // the sweep, versioned on the (warp-uniform) staging decision so the hot loop carries no
  // global-memory fallback
  auto sweep = [&](auto stg, auto prn) {
  for (;;) {
    uint32_t my = KEY_NONE;
#pragma unroll
    for (int q = 0; q < NW; ++q) my = min(my, nkey[q]);
    const uint32_t zk = __reduce_min_sync(FULL, my);
    if (zk == KEY_NONE) break;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      const bool hit = nkey[q] == zk;
      M[q] ^= __ballot_sync(FULL, hit);
      if constexpr (decltype(stg)::value) {         // sentinel-terminated lists in shared memory
        pos[q] += hit ? 1u : 0u;
        if (hit) nkey[q] = stage[pos[q]];
      } else if (hit) {
        ++pos[q];
        nkey[q] = pos[q] < end[q] ? fkey(col_value(src, cur[q], pos[q], complement)) : KEY_NONE;
      }
    }
    int knew;
    if constexpr (NW == 2) knew = nearest2(M[0], M[1]);
    else knew = nearest_parent<NW>(M, lane + R, R);
    if constexpr (use_ring) {
      const bool chg = knew != kap;
      const bool closed = chg && kap != KNONE;
      const float z = keyf(zk);
      if (closed) {
        ring_z[wid][rc % P1_RING][lane] = make_float2(zstart, z);
        ring_k[wid][rc % P1_RING][lane] = (uint8_t)kap;
      }
      rc += closed ? 1u : 0u;
      kap = chg ? knew : kap;
      zstart = chg ? z : zstart;
      if (__any_sync(FULL, rc - rd == (uint32_t)P1_RING)) drain();
    } else {                                 // inline filter, branch-free (measured faster for larger R)
      const bool chg = knew != kap;
      // an event changes kappa only for lanes within R of its column: steps where no lane of
      // the warp changes (often: halo events) skip the filter / emission half (warp-uniform)
      if (SKIP && !__any_sync(FULL, chg)) continue;
      const bool closed = chg && kap != KNONE;
      const float z = keyf(zk);
      if constexpr (decltype(prn)::value) {   // (the sweep is versioned on prune != nullptr)
        const bool hp = pk != KNONE;
        bool drop_new, drop_pend;
        if constexpr (NW == 2) {             // thresholds from the (kp, kn) table
          const float2 th = thr[min(pk, 17) * 32 + (kap & 31)];
          drop_new = z - phi <= th.x;
          drop_pend = zstart - plo <= th.y;
        } else {
          const float D = hpk - h0[kap & 255];                  // H[kp] - H[kn] (garbage when unused)
          drop_new = hp && pk <= kap && dom_margin(z - phi, D, mabs);
          drop_pend = kap <= pk && dom_margin(zstart - plo, -D, mabs);
          hpk = (closed && !drop_new) ? h0[kap & 255] : hpk;
        }
        // the pending piece is stored (unless the new one dominates it) before it is replaced
        const bool wr = closed && hp && !drop_new && !drop_pend;
        st_pred_piece(zb + woff, kb + woff, plo, phi, pk, wr);
        np += wr ? 1u : 0u;
        woff += (wr && woff < wlim) ? zstep : 0u;
        const bool take = closed && !drop_new;
        plo = take ? zstart : plo;
        phi = take ? z : phi;
        pk = take ? kap : pk;
      } else {
        st_pred_piece(zb + woff, kb + woff, zstart, z, kap, closed);
        np += closed ? 1u : 0u;
        woff += (closed && woff < wlim) ? zstep : 0u;
      }
      kap = chg ? knew : kap;
      zstart = chg ? z : zstart;
    }
  }
  };
  if (staged) {
    if (prune) sweep(std::true_type{}, std::true_type{});
    else sweep(std::true_type{}, std::false_type{});
  } else {
    if (prune) sweep(std::false_type{}, std::true_type{});
    else sweep(std::false_type{}, std::false_type{});
  }
  if (use_ring) drain();
  if (prune && pk != KNONE) put(plo, phi, pk);
  if (!list_mode) {
    if (out_ok) {
      P.cnt[c] = np;
      if (np > (uint32_t)P.cap) {                    // hand the column to list mode
        atomicMax(P.flags + 1, np);
        const unsigned slot = atomicAdd(P.flags, 1u);
        if (slot < P.ovf_list_cap) {
          P.ovf_idx[c] = (int32_t)slot;
          const size_t tf = (size_t)jr * ntiles + tile;
          if (atomicExch(P.tile_flag + tf, 1u) == 0u) {
            const unsigned ts = atomicAdd(P.flags + 2, 1u);
            P.tile_list[ts] = (uint32_t)tf;
          }
        }
      }
    }
    const unsigned wsum = __reduce_add_sync(FULL, (out_ok && np <= (uint32_t)P.cap) ? np : 0u);   // arena: list launch
    if (lane == 0 && wsum) atomicAdd(P.total, (unsigned long long)wsum);
  } else if (has_out) {
    P.cnt[c] = np;                                   // the filtered count of an arena column
    atomicAdd(P.total, (unsigned long long)np);
  }
}

// ------------------------------------------------------------------ pass 1, both shell families
// The shell needs pass 1 of S (r_out) and of C = U \ S (r_in).  When both radii give the same
// R <= 16 one sweep serves both: C's endpoints are S's (plus z_lo / z_hi), so the window events
// are the same, and between two events a window column is in C exactly when it is in the grid
// and not in S -- C's activity mask is G & ~M (G = the window's in-grid columns).  C's pieces
// start at z_lo (before the first event every in-grid column is in C) and its last piece
// closes at z_hi; zero-length C pieces (an S interval starting at z_lo or ending at z_hi) are
// dropped, exactly as complement-on-load drops them (col_open).  The unfiltered piece sequence
// of each family is therefore the one its own sweep produces, and so are the filtered pieces.
// The event half of a sweep step (REDUX, ballots, key advance) and the key staging run once
// for both families.  Main pass only (overflow columns are redone per family in list mode).

// one family's output state in the dual sweep
struct P1Fam {
  float2* zb;
  uint8_t* kb;
  uint32_t zstep, woff, wlim, np;
  bool has_out;
  float plo, phi;   // pending piece of the domination filter
  int pk;
  const float2* trow;   // the threshold-table row of pk (row 17: no pending piece)
};

__device__ __forceinline__ void p1_fam_init(P1Fam& F, const PieceSlots& P, int jr, int i, bool out_ok,
                                            const float2* thr) {
  // lanes without output store into a spill cell (slot cap, never read)
  F.zb = P.z + piece_index(P, jr, out_ok ? 0 : P.cap, out_ok ? i : 0);
  F.kb = P.k + piece_index(P, jr, out_ok ? 0 : P.cap, out_ok ? i : 0);
  // opaque per-lane base pointers: otherwise the compiler rebuilds them from the kernel
  // parameter with 64-bit index arithmetic at every store (6 instructions instead of 3)
  asm("mov.b64 %0, %0;" : "+l"(F.zb));
  asm("mov.b64 %0, %0;" : "+l"(F.kb));
  F.zstep = out_ok ? (uint32_t)P.nx : 0u;
  F.wlim = (uint32_t)P.cap * F.zstep;   // the spill cell
  F.woff = 0;
  F.np = 0;
  F.has_out = out_ok;
  F.plo = F.phi = 0.f;
  F.pk = KNONE;
  F.trow = thr + 17 * 32;
}

// a piece [zstart, z] at level kap closed (closed == true): the domination filter against the
// pending piece, branch-free (the p1_kernel inline path with the threshold table)
__device__ __forceinline__ void p1_fam_step(P1Fam& F, bool closed, float zstart, float z, int kap,
                                            const float2* thr) {
  const bool hp = F.pk != KNONE;
  const float2 th = F.trow[kap & 31];
  const bool drop_new = z - F.phi <= th.x;
  const bool drop_pend = zstart - F.plo <= th.y;
  const bool wr = closed && hp && !drop_new && !drop_pend;
  st_pred_piece(F.zb + F.woff, F.kb + F.woff, F.plo, F.phi, F.pk, wr);
  F.np += wr ? 1u : 0u;
  F.woff += (wr && F.woff < F.wlim) ? F.zstep : 0u;
  const bool take = closed && !drop_new;
  F.plo = take ? zstart : F.plo;
  F.phi = take ? z : F.phi;
  F.pk = take ? kap : F.pk;
  F.trow = take ? thr + (kap & 31) * 32 : F.trow;   // (kap <= 16 whenever a piece is taken)
}

// flush the pending piece, store the count, list an overflowing column for list mode
__device__ __forceinline__ void p1_fam_finish(P1Fam& F, PieceSlots& P, int64_t c, int jr, int tile, int ntiles) {
  if (F.has_out && F.pk != KNONE) {
    const uint32_t t = min(F.np, (uint32_t)P.cap);
    F.zb[(size_t)t * F.zstep] = make_float2(F.plo, F.phi);
    F.kb[(size_t)t * F.zstep] = (uint8_t)F.pk;
    ++F.np;
  }
  if (F.has_out) {
    P.cnt[c] = F.np;
    if (F.np > (uint32_t)P.cap) {
      atomicMax(P.flags + 1, F.np);
      const unsigned slot = atomicAdd(P.flags, 1u);
      if (slot < P.ovf_list_cap) {
        P.ovf_idx[c] = (int32_t)slot;
        const size_t tf = (size_t)jr * ntiles + tile;
        if (atomicExch(P.tile_flag + tf, 1u) == 0u) {
          const unsigned ts = atomicAdd(P.flags + 2, 1u);
          P.tile_list[ts] = (uint32_t)tf;
        }
      }
    }
  }
  const unsigned wsum = __reduce_add_sync(FULL, (F.has_out && F.np <= (uint32_t)P.cap) ? F.np : 0u);
  if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(P.total, (unsigned long long)wsum);
}

template <bool SKIP>
__global__ void __launch_bounds__(P1_WARPS * 32) p1_dual_kernel(SrcRows src, int R, int row0, int jr0, int nrows_out,
                                                                 PieceSlots PS, PieceSlots PC,
                                                                 const float* __restrict__ prune_s,
                                                                 const float* __restrict__ prune_c) {
  __shared__ uint32_t stage_all[P1_WARPS][P1_STAGE];
  __shared__ float2 thr_s[18 * 32], thr_c[18 * 32];
  p1_thr_init(thr_s, prune_s, R);
  p1_thr_init(thr_c, prune_c, R);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t* stage = stage_all[threadIdx.x >> 5];
  const int ntiles = (src.nx + 31) >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= (int64_t)nrows_out * ntiles) return;  // warp-uniform
  const int jr = jr0 + (int)(gw / ntiles), tile = (int)(gw % ntiles);
  const int j = row0 + jr;
  const int i0 = tile * 32;
  const int W = 32 + 2 * R;
  constexpr int NW = 2;

  // the window's S endpoints as keys (as p1_kernel with complement = 0)
  ColCursor cur[NW];
  uint32_t sb[NW], pos[NW], end[NW], nkey[NW], G[NW];
  uint32_t total = 0;
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    const int w = lane + 32 * q;
    const int gi = i0 - R + w;
    G[q] = __ballot_sync(FULL, w < W && gi >= 0 && gi < src.nx);   // in-grid window columns
    if (w < W) col_open(src, gi, j, 0, cur[q]);
    else col_close(cur[q]);
    const uint32_t nv = cur[q].vend - cur[q].v + 1;
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
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    const uint32_t nv = cur[q].vend - cur[q].v;
    if (staged) {
      for (uint32_t t = 0; t < nv; ++t) stage[sb[q] + t] = fkey(col_value(src, cur[q], cur[q].v + t, 0));
      stage[sb[q] + nv] = KEY_NONE;
      pos[q] = sb[q];
      end[q] = sb[q] + nv;
    } else {
      pos[q] = cur[q].v;
      end[q] = cur[q].vend;
    }
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < NW; ++q)
    nkey[q] = pos[q] < end[q] ? (staged ? stage[pos[q]] : fkey(col_value(src, cur[q], pos[q], 0))) : KEY_NONE;

  const int i = i0 + lane;
  const bool out_ok = i < src.nx;
  const int64_t c = (int64_t)jr * src.nx + i;
  P1Fam FS, FC;
  p1_fam_init(FS, PS, jr, i, out_ok, thr_s);
  p1_fam_init(FC, PC, jr, i, out_ok, thr_c);
  const int pp = lane + R;
  const int shr = pp < 32 ? pp : pp - 32;
  const int shl = pp >= 31 ? pp - 31 : 31 - pp;
  const bool rlow = pp < 32, lhigh = pp >= 31;
  // this lane's two 32-bit windows of a 64-bit window mask: bits p .. p+31 (right) and
  // p-31 .. p with bit p on top (left)
  auto win_r = [&](uint32_t m0, uint32_t m1) { return __funnelshift_r(rlow ? m0 : m1, rlow ? m1 : 0u, shr); };
  auto win_l = [&](uint32_t m0, uint32_t m1) {
    const uint32_t la = __funnelshift_r(m0, m1, shl), lb = __funnelshift_l(0u, m0, shl);
    return lhigh ? la : lb;
  };
  // nearest set bit from the windows (a sentinel at distance 31 > R keeps both non-zero)
  auto nearest_w = [&](uint32_t rw, uint32_t lw) -> int {
    const int d = min(__clz(lw | 1u), __ffs(rw | 0x80000000u) - 1);
    return d <= R ? d : KNONE;
  };
  // C's mask is G & ~M: its windows are ~window(M) & window(G), window(G) fixed for the sweep
  const uint32_t gr = win_r(G[0], G[1]), gl = win_l(G[0], G[1]);
  uint32_t M0 = 0u, M1 = 0u;                   // S activity of the window (warp-uniform)
  int kap = KNONE, kapc = nearest_w(gr, gl);
  float zstart = 0.f, zstartc = src.zlo;
  auto sweep = [&](auto stg) {
    for (;;) {
      const uint32_t zk = __reduce_min_sync(FULL, min(nkey[0], nkey[1]));
      if (zk == KEY_NONE) break;
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        const bool hit = nkey[q] == zk;
        const uint32_t b = __ballot_sync(FULL, hit);
        if (q == 0) M0 ^= b; else M1 ^= b;
        if constexpr (decltype(stg)::value) {
          pos[q] += hit ? 1u : 0u;
          if (hit) nkey[q] = stage[pos[q]];
        } else if (hit) {
          ++pos[q];
          nkey[q] = pos[q] < end[q] ? fkey(col_value(src, cur[q], pos[q], 0)) : KEY_NONE;
        }
      }
      const float z = keyf(zk);
      const uint32_t mr = win_r(M0, M1), ml = win_l(M0, M1);
      const int knew = nearest_w(mr, ml);
      const int knewc = nearest_w(gr & ~mr, gl & ~ml);
      const bool chg = knew != kap, chgc = knewc != kapc;
      // an event changes kappa only for lanes within R of its column: steps where no lane of
      // the warp changes (often: halo events) skip the filter / emission half (warp-uniform)
      if (!SKIP || __any_sync(FULL, chg)) {
        p1_fam_step(FS, chg && kap != KNONE, zstart, z, kap, thr_s);
        kap = chg ? knew : kap;
        zstart = chg ? z : zstart;
      }
      if (!SKIP || __any_sync(FULL, chgc)) {
        p1_fam_step(FC, chgc && kapc != KNONE && zstartc < z, zstartc, z, kapc, thr_c);
        kapc = chgc ? knewc : kapc;
        zstartc = chgc ? z : zstartc;
      }
    }
  };
  if (staged) sweep(std::true_type{});
  else sweep(std::false_type{});
  // C's last piece closes at z_hi
  p1_fam_step(FC, kapc != KNONE && zstartc < src.zhi, zstartc, src.zhi, kapc, thr_c);
  p1_fam_finish(FS, PS, c, jr, tile, ntiles);
  p1_fam_finish(FC, PC, c, jr, tile, ntiles);
}

// pieces of a band (slots + arena) -> CSR (dexel_pass1, parity testing only)
__global__ void pieces_to_csr(PieceSlots P, int64_t ncol, const uint64_t* __restrict__ off, float2* __restrict__ oz,
                              uint8_t* __restrict__ ok) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const int row = (int)(c / P.nx), i = (int)(c % P.nx);
  const uint32_t m = P.cnt[c];
  const uint64_t o = off[c];
  const bool arena = P.ovf_idx[c] >= 0;
  for (uint32_t t = 0; t < m; ++t) {
    if (!arena) {
      oz[o + t] = P.z[piece_index(P, row, (int)t, i)];
      ok[o + t] = P.k[piece_index(P, row, (int)t, i)];
    } else {
      const size_t q = (size_t)P.ovf_idx[c] * P.ovf_cap + t;
      oz[o + t] = P.ovf_z[q];
      ok[o + t] = P.ovf_k[q];
    }
  }
}

}  // namespace dexel
