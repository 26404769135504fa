// levels.cuh -- the z-resolution between pass 1 and pass 2: per column of
// S_Mid, the level sets of its 1D half-space power diagram.
//
// Input: the pass-1 pieces p = (lo, hi, kappa) of one column, sorted and disjoint
// (PAPER.md:494-501).  Each piece is a segment seed with power weight
// W_p = r^2 - kappa^2 s^2 (weight r^2 per App. B,
// PAPER.md:1084-1088, readings R1/R2).  Seen from a row at lateral
// offset k = |dy| it covers the capsule cross-section
//     [lo_p - h, hi_p + h],   h = h(kappa_p, k) = sqrt(r^2 - (kappa_p^2 + k^2) s^2),
// valid iff kappa_p^2 + k^2 <= (r/s)^2.  By the capsule decomposition
// (D^p = D^box u D^o, start endpoints grow down, end endpoints
// grow up) this splits into two half-space parts:
//     [lo_p, hi_p + h]   box + end anchor (grows UP)
//     [lo_p - h, hi_p]   box + start anchor (grows DOWN)
// so the level set pass 2 needs, L_k = U_p [lo_p - h, hi_p + h], is
//     L_k = U_f(k) u U_r(k),   U_f(k) = U_p [lo_p, hi_p + h],  U_r(k) = U_p [lo_p - h, hi_p].
// U_f's intervals start at lo_p, ascending with p, so one forward running union
// builds it (the forward half-space sweep); U_r's end at hi_p, so one backward
// running union builds it (the backward sweep).  Each (piece, level) step is a
// table load, one fp32 add and a few compares/selects -- no branches, no
// square roots (the h table is fp64 on the host, rounded once to fp32,
// DESIGN.md reading R20).  A thread owns one column and a chunk of LMAX levels
// held in registers (blockIdx.y = chunk), so the kernel is SIMT-uniform: every
// lane walks its own column's pieces with the same instruction stream.
// (An O(m + output) explicit upper-envelope variant was measured first and ran
// 4-6x slower: 4 of 32 lanes active per instruction.)
//
// Layout (HBM): level slots, direction d = 0 (U_f, ascending) / 1 (U_r, stored
// descending):  z[(((row*2 + d)*(R+1) + k)*cap + t)*nx + i]  (float2), counts
// cnt[((row*2 + d)*(R+1) + k)*nx + i] (u8).  For a fixed (row, d, k, t) the nx
// columns of a row are contiguous, so a warp of 32 consecutive columns writes
// and (in pass 2) reads 256 contiguous bytes.  A list longer than cap raises a
// flag: the column is listed and an overflow pass rewrites all its lists into an
// arena of 255-entry lists (pass 2 reads a list there when its count > cap); if too
// many columns overflow the host reruns the band with a larger cap (DESIGN.md
// "Capacities").
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dexel {

constexpr int LV_OVF_CAP = 255;   // list capacity in the overflow arena (counts are u8)

struct LevelSlots {
  uint8_t* cnt;      // [nrows][2][R+1][nx]  true list lengths (<= 255)
  float2* z;         // [nrows][2][R+1][cap][nx]
  int R, cap, nx, nrows;
  int row0;          // row (in the op's extended-row numbering) of slot row 0
  // columns with a list longer than cap keep all their lists in the overflow arena:
  // list (d, k) of overflow slot q at ovf_z[((q*2 + d)*(R+1) + k)*LV_OVF_CAP + t]
  int32_t* ovf_idx;  // [nrows*nx] overflow slot of a column (valid only where some count > cap)
  float2* ovf_z;
};

__host__ __device__ __forceinline__ size_t slot_cnt_index(const LevelSlots& L, int row, int d, int k, int i) {
  return (((size_t)row * 2 + d) * (L.R + 1) + k) * L.nx + i;
}
__host__ __device__ __forceinline__ size_t slot_z_index(const LevelSlots& L, int row, int d, int k, int t, int i) {
  return ((((size_t)row * 2 + d) * (L.R + 1) + k) * L.cap + t) * L.nx + i;
}

__host__ __device__ __forceinline__ size_t ovf_z_index(const LevelSlots& L, int q, int d, int k, int t) {
  return (((size_t)q * 2 + d) * (L.R + 1) + k) * LV_OVF_CAP + t;
}

struct LvArgs {
  const uint64_t* moff;    // pieces CSR offsets [ncol+1] (columns of the level rows)
  const float2* mz;        // (lo, hi)
  const uint8_t* mk;       // kappa
  int64_t ncol;
  const float* h;          // [(R+1)^2] fl32(sqrt(r^2 - (kappa^2 + k^2) s^2)), -1 where negative
  float zlo, zhi;
  LevelSlots L;
  unsigned* flags;         // [0] longest list seen, [1] overflow columns
  unsigned long long* nlev;  // total level intervals (statistics)
  uint32_t* ovf_list;      // main pass: columns with a list longer than cap
  unsigned ovf_list_cap;
  const uint32_t* list;    // overflow pass: the listed columns, written to the overflow arena
  int64_t nlist;
};

constexpr int LV_T = 128;

// q < 0: main pass (slots); q >= 0: overflow pass (arena slot q)
__device__ __forceinline__ void lv_emit(const LvArgs& A, int q, int row, int d, int k, int i, uint32_t& n, float lo,
                                        float hi) {
  lo = fmaxf(lo, A.zlo);
  hi = fminf(hi, A.zhi);
  if (lo < hi) {
    if (q < 0) {
      if (n < (uint32_t)A.L.cap) A.L.z[slot_z_index(A.L, row, d, k, (int)n, i)] = make_float2(lo, hi);
    } else if (n < (uint32_t)LV_OVF_CAP) {
      A.L.ovf_z[ovf_z_index(A.L, q, d, k, (int)n)] = make_float2(lo, hi);
    }
    ++n;
  }
}

// blockIdx.y = level chunk: this thread runs levels k0 .. k0+LMAX-1 of column c.
// The h table rows are HS = LMAX | 1 floats apart: an odd stride puts the rows of
// different kappa (the lanes' pieces differ) in different banks.
template <int LMAX>
__global__ void __launch_bounds__(LV_T) levels_kernel(LvArgs A) {
  constexpr int HS = LMAX | 1;
  __shared__ float Hs[256 * HS];          // h(kappa, k0 + k), -1 beyond R or invalid
  __shared__ unsigned long long blk_total;
  __shared__ unsigned blk_max;
  const int R = A.L.R, L1 = R + 1;
  const int k0 = blockIdx.y * LMAX;
  for (int t = threadIdx.x; t < L1 * HS; t += LV_T) {
    const int kap = t / HS, k = k0 + t % HS;
    Hs[t] = (k <= R && t % HS < LMAX) ? A.h[kap * L1 + k] : -1.0f;
  }
  if (threadIdx.x == 0) { blk_total = 0; blk_max = 0; }
  __syncthreads();
  const int64_t g = (int64_t)blockIdx.x * LV_T + threadIdx.x;
  if (g < (A.list ? A.nlist : A.ncol)) {
    const int64_t c = A.list ? (int64_t)A.list[g] : g;
    const int q = A.list ? (int)g : -1;
    const int row = (int)(c / A.L.nx), i = (int)(c % A.L.nx);
    const uint64_t base = A.moff[c];
    const int m = (int)(A.moff[c + 1] - base);
    float a[LMAX], b[LMAX];
    uint32_t n[LMAX];
    uint32_t tot = 0, mx = 0;
    // ---- U_f: forward running union of [lo, hi + h]
#pragma unroll
    for (int k = 0; k < LMAX; ++k) { a[k] = 0.f; b[k] = -INFINITY; n[k] = 0; }
    {
      float2 nz = m > 0 ? A.mz[base] : make_float2(0.f, 0.f);
      int nk = m > 0 ? A.mk[base] : 0;
      for (int t = 0; t < m; ++t) {
        const float2 p = nz;
        const float* hrow = Hs + nk * HS;
        if (t + 1 < m) { nz = A.mz[base + t + 1]; nk = A.mk[base + t + 1]; }   // prefetch
        if (hrow[0] < 0.f) continue;        // validity is monotone in k: the whole chunk is out of reach
#pragma unroll
        for (int k = 0; k < LMAX; ++k) {
          const float h = hrow[k];
          const bool valid = h >= 0.f;
          const bool brk = valid && p.x > b[k];
          if (brk) lv_emit(A, q, row, 0, k0 + k, i, n[k], a[k], b[k]);   // b = -inf emits nothing
          a[k] = brk ? p.x : a[k];
          const float e = p.y + h;
          b[k] = valid ? (brk ? e : fmaxf(b[k], e)) : b[k];
        }
      }
#pragma unroll
      for (int k = 0; k < LMAX; ++k) {
        lv_emit(A, q, row, 0, k0 + k, i, n[k], a[k], b[k]);
        if (k0 + k <= R) {
          A.L.cnt[slot_cnt_index(A.L, row, 0, k0 + k, i)] = (uint8_t)min(n[k], 255u);
          tot += n[k];
          mx = max(mx, n[k]);
        }
      }
    }
    // ---- U_r: backward running union of [lo - h, hi]; stored in descending order
#pragma unroll
    for (int k = 0; k < LMAX; ++k) { a[k] = INFINITY; b[k] = 0.f; n[k] = 0; }
    {
      float2 nz = m > 0 ? A.mz[base + m - 1] : make_float2(0.f, 0.f);
      int nk = m > 0 ? A.mk[base + m - 1] : 0;
      for (int t = m - 1; t >= 0; --t) {
        const float2 p = nz;
        const float* hrow = Hs + nk * HS;
        if (t > 0) { nz = A.mz[base + t - 1]; nk = A.mk[base + t - 1]; }
        if (hrow[0] < 0.f) continue;
#pragma unroll
        for (int k = 0; k < LMAX; ++k) {
          const float h = hrow[k];
          const bool valid = h >= 0.f;
          const bool brk = valid && p.y < a[k];
          if (brk) lv_emit(A, q, row, 1, k0 + k, i, n[k], a[k], b[k]);   // a = +inf emits nothing
          b[k] = brk ? p.y : b[k];
          const float st = p.x - h;
          a[k] = valid ? (brk ? st : fminf(a[k], st)) : a[k];
        }
      }
#pragma unroll
      for (int k = 0; k < LMAX; ++k) {
        lv_emit(A, q, row, 1, k0 + k, i, n[k], a[k], b[k]);
        if (k0 + k <= R) {
          A.L.cnt[slot_cnt_index(A.L, row, 1, k0 + k, i)] = (uint8_t)min(n[k], 255u);
          tot += n[k];
          mx = max(mx, n[k]);
        }
      }
    }
    if (q < 0) atomicAdd(&blk_total, (unsigned long long)tot);   // the overflow pass recounts nothing
    if (mx > (unsigned)A.L.cap) {
      atomicMax(&blk_max, mx);
      if (q < 0) {                                                  // hand the column to the overflow pass
        const unsigned slot = atomicAdd(A.flags + 1, 1u);
        if (slot < A.ovf_list_cap) {
          A.ovf_list[slot] = (uint32_t)c;
          A.L.ovf_idx[c] = (int32_t)slot;
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (A.nlev) atomicAdd(A.nlev, blk_total);
    if (blk_max) atomicMax(A.flags, blk_max);
  }
}

}  // namespace dexel
