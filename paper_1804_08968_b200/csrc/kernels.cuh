// kernels.cuh -- sm_100a kernels of the separable dexel offset (arXiv 1804.08968).
//
//   validate_kernel   upload check (strictly increasing, finite, in domain)
//   pass1_kernel      pass 1 along x: closest-parent extrusion S_In -> S_Mid
//                     (PAPER.md:494-501).  One warp per 32 output columns of a
//                     row; the warp sweeps z over the window's endpoints (merged
//                     across lanes with a REDUX min on order-preserving keys), keeps
//                     the active neighbour columns as a ballot bitmask and each lane
//                     reads its closest parent kappa = nearest set bit within R.
// The z-resolution (levels.cuh) and pass 2 (pass2.cuh) live in their own headers.
// pass1 runs twice (two-phase allocation): COUNT writes per-column counts, WRITE
// recomputes and writes at the scanned offsets.
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

}  // namespace dexel
