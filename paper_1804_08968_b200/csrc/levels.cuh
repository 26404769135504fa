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
// descending):  z[(((row*2 + d)*cap + t)*(R+2) + k)*nx + i]  (float2), counts
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

#include "kernels.cuh"

namespace dexel {

constexpr int LV_OVF_CAP = 255;   // list capacity in the overflow arena (counts are u8)

struct LevelSlots {
  uint8_t* cnt;      // [nrows][2][R+1][nx]  true list lengths (<= 255)
  float2* z;         // [nrows][2][cap][R+2][nx]  (unclipped; level R+1 of the last slot = spill cell)
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
// z slots, slot-major inside a (row, d) block: z[(((row*2 + d)*cap + t)*(R+2) + k)*nx + i].
// Level R+1 of the last slot is a spill cell: an emission is written at
// min(offset, spill), so an overflowing list (t >= cap) only ever hits the spill cell
// (its column is then redone in the overflow arena) and never another list.
__host__ __device__ __forceinline__ size_t slot_z_index(const LevelSlots& L, int row, int d, int k, int t, int i) {
  return ((((size_t)row * 2 + d) * L.cap + t) * (L.R + 2) + k) * L.nx + i;
}

__host__ __device__ __forceinline__ size_t ovf_z_index(const LevelSlots& L, int q, int d, int k, int t) {
  return (((size_t)q * 2 + d) * (L.R + 1) + k) * LV_OVF_CAP + t;
}

struct LvArgs {
  PieceSlots P;            // pass-1 pieces of the level rows (kernels.cuh)
  int64_t ncol;
  const float* h;          // [(R+1)^2] fl32(sqrt(r^2 - (kappa^2 + k^2) s^2)), -1 where negative
  float zlo, zhi;
  LevelSlots L;
  unsigned* flags;         // [0] longest list seen, [1] overflow columns
  unsigned long long* nlev;  // total level intervals (statistics)
  unsigned long long* dbg; // diagnostics or nullptr: [0] sum of per-warp max piece counts, [1] warps
  uint32_t* ovf_list;      // main pass: columns with a list longer than cap
  unsigned ovf_list_cap;
  const uint32_t* list;    // overflow pass: the listed columns, written to the overflow arena
  int64_t nlist;
};

constexpr int LV_T = 128;

// predicated 8-byte store without a branch (the compiler otherwise wraps each level's rare
// emission in a BSSY/BRA/BSYNC region that some lane of the warp takes almost every step)
__device__ __forceinline__ void st_pred_f2(float2* p, float x, float y, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.global.v2.f32 [%0], {%1, %2};\n\t}"
               :: "l"(p), "f"(x), "f"(y), "r"((int)pred));
}

// blockIdx.y = level chunk: this thread runs levels k0 .. k0+LMAX-1 of column c.
// The h table holds -inf where a piece is out of reach (kappa^2 + k^2 > (r/s)^2): then
// hi + h = -inf and lo - h = +inf leave the running union unchanged without a validity
// test, and a "break" by such a piece only closes a component that no later piece (all
// start higher) could extend anyway.  Rows are HS floats (HS/4 odd): a row is read with
// 128-bit loads, and 8 lanes with different kappa hit 8 different bank groups.
template <int LMAX>
struct LvTab {
  static constexpr int NV = (LMAX + 3) / 4;                 // float4 per row actually used
  static constexpr int HS = 4 * (NV | 1);                   // row stride (floats), HS/4 odd
};

template <int LMAX>
__global__ void __launch_bounds__(LV_T, LMAX >= 12 ? 3 : 4) levels_kernel(LvArgs A) {
  constexpr int NV = LvTab<LMAX>::NV, HS = LvTab<LMAX>::HS;
  __shared__ __align__(16) float Hs[257 * HS];   // h(kappa, k0 + k), -inf beyond R or out of reach;
                                                  // row R+1: all -inf (the "null piece")
  const int R = A.L.R, L1 = R + 1;
  const int k0 = blockIdx.y * LMAX;
  for (int t = threadIdx.x; t < (L1 + 1) * HS; t += LV_T) {
    const int kap = t / HS, kk = t % HS, k = k0 + kk;
    const float h = (kap <= R && kk < LMAX && k <= R) ? A.h[kap * L1 + k] : -1.0f;
    Hs[t] = h >= 0.f ? h : -INFINITY;
  }
  __shared__ uint16_t cntS[2][LMAX][64];          // both directions' list lengths of the block's columns
  __shared__ uint8_t ovfS[2][64];                  // a direction outgrew its slots (no merge)
  __syncthreads();
  uint32_t tot = 0, mx = 0;
  int tot_adj = 0;
  // block = 64 columns x 2 directions: warps 0-1 run U_f (d = 0), warps 2-3 U_r (d = 1) of the
  // same 64 columns (halves the live state per thread); afterwards they merge U_f(k) and U_r(k)
  // into L_k in place
  const int d = threadIdx.x >> 6;
  const int lc = threadIdx.x & 63;
  const int64_t g = (int64_t)blockIdx.x * 64 + lc;
  const bool live = g < (A.list ? A.nlist : A.ncol);
  // every lane of the warp walks the same piece index t (0..mmax-1 forward, mmax-1..0 backward):
  // the slot reads stay coalesced and the loop never diverges; a lane past its own count
  // processes the "null piece", which leaves both running unions unchanged
  const int m_live = live ? (int)A.P.cnt[A.list ? (int64_t)A.list[g] : g] : 0;
  const int mmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)m_live);
  if (A.dbg && (threadIdx.x & 31) == 0) {                 // diagnostics (DEXEL_DEBUG): sum of warp maxima
    atomicAdd(A.dbg, (unsigned long long)mmax);
    atomicAdd(A.dbg + 1, 1ull);
  }
  {   // all 32 lanes run the loop (warp-uniform trip count and __all_sync); dead lanes see m = 0
    const int64_t c = live ? (A.list ? (int64_t)A.list[g] : g) : 0;
    const int q = A.list ? (int)g : -1;
    const int row = (int)(c / A.L.nx), i = (int)(c % A.L.nx);
    // this column's pieces: slots (stride nx, coalesced across the warp) or the overflow arena
    const int m = m_live;
    const float2* zc;
    const uint8_t* kc;
    int64_t ps;
    if (m <= A.P.cap) {   // (a column's pieces live in the arena exactly when it has more than cap)
      zc = A.P.z + piece_index(A.P, row, 0, i);
      kc = A.P.k + piece_index(A.P, row, 0, i);
      ps = A.P.nx;
    } else {
      const size_t qo = (size_t)A.P.ovf_idx[c] * A.P.ovf_cap;
      zc = A.P.ovf_z + qo;
      kc = A.P.ovf_k + qo;
      ps = 1;
    }
    float a[LMAX], b[LMAX];
    uint32_t o[LMAX];   // next slot of level k0+k, as a float2 offset from slot 0 / level k0 of the block
    const uint32_t nx = (uint32_t)A.L.nx, S = (uint32_t)(R + 2) * nx;      // S = one slot (all levels)
    const uint32_t omax = (uint32_t)(A.L.cap - 1) * S + (uint32_t)(R + 1 - k0) * nx;   // the spill cell
    {
      // main pass: slots of (row, d, level k0); overflow pass: the arena lists of slot q
      float2* Zd = q < 0 ? A.L.z + slot_z_index(A.L, row, d, k0, 0, i)
                         : A.L.ovf_z + ovf_z_index(A.L, q, d, k0, 0);
      const uint32_t ostep = q < 0 ? S : 1u, olev = q < 0 ? nx : (uint32_t)LV_OVF_CAP;
      const uint32_t olim = q < 0 ? omax : (uint32_t)(R + 1 - k0) * LV_OVF_CAP - 1u;
#pragma unroll
      for (int k = 0; k < LMAX; ++k) {
        a[k] = d ? INFINITY : 0.f;
        b[k] = d ? 0.f : -INFINITY;
        o[k] = (uint32_t)k * olev;
      }
      // emission: closed component [a, b] of level k (empty placeholders have a >= b);
      // branch-free -- a predicated store, the slot clamped into the spill zone
#define LV_EMIT(k, pred)                                                      \
  {                                                                           \
    const bool ok_ = (pred) && a[k] < b[k];                                   \
    st_pred_f2(Zd + min(o[k], olim), a[k], b[k], ok_);                        \
    o[k] += ok_ ? ostep : 0u;                                                 \
  }
      // null piece: U_f (-inf, -inf), U_r (+inf, +inf), kappa row R+1 (all -inf)
      const float2 nullp = d ? make_float2(INFINITY, INFINITY) : make_float2(-INFINITY, -INFINITY);
      auto fetch = [&](int s, float2& z, int& kk) {
        const int t = d ? mmax - 1 - s : s;
        if (s < mmax && t < m) { z = zc[(int64_t)t * ps]; kk = kc[(int64_t)t * ps]; }
        else { z = nullp; kk = L1; }
      };
      float2 nz, nz2;
      int nk, nk2;
      fetch(0, nz, nk);
      fetch(1, nz2, nk2);
      for (int s = 0; s < mmax; ++s) {
        const float2 p = nz;
        const float4* hrow = reinterpret_cast<const float4*>(Hs + nk * HS);
        nz = nz2; nk = nk2;
        fetch(s + 2, nz2, nk2);
        float hv[4 * NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const float4 v = hrow[j];
          hv[4 * j] = v.x; hv[4 * j + 1] = v.y; hv[4 * j + 2] = v.z; hv[4 * j + 3] = v.w;
        }
        // reach is monotone in k: skip when no lane's piece reaches this chunk (warp-uniform)
        if (__all_sync(0xffffffffu, hv[0] == -INFINITY)) continue;
        if (d == 0) {                        // U_f: forward running union of [lo, hi + h]
#pragma unroll
          for (int k = 0; k < LMAX; ++k) {
            const bool brk = p.x > b[k];
            LV_EMIT(k, brk);
            a[k] = brk ? p.x : a[k];
            const float e = p.y + hv[k];
            b[k] = brk ? e : fmaxf(b[k], e);
          }
        } else {                             // U_r: backward running union of [lo - h, hi]
#pragma unroll
          for (int k = 0; k < LMAX; ++k) {
            const bool brk = p.y < a[k];
            LV_EMIT(k, brk);
            b[k] = brk ? p.y : b[k];
            const float st = p.x - hv[k];
            a[k] = brk ? st : fminf(a[k], st);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < LMAX; ++k) {
        LV_EMIT(k, true);
#undef LV_EMIT
        const uint32_t nk_ = (o[k] - (uint32_t)k * olev) / ostep;
        cntS[d][k][lc] = (uint16_t)min(nk_, 65535u);
        if (live && k0 + k <= R) {
          if (q < 0) A.L.cnt[slot_cnt_index(A.L, row, d, k0 + k, i)] = (uint8_t)min(nk_, 255u);
          tot += nk_;
          mx = max(mx, nk_);
        }
      }
    }
    ovfS[d][lc] = (uint8_t)(mx > (unsigned)A.L.cap);
    __syncthreads();
    // L_k = U_f(k) u U_r(k), merged in place into U_f's slots: every component
    // of L_k contains a U_f component, so |L_k| <= |U_f(k)| and the write index never passes the
    // read index.  U_r's count becomes 0 -- pass 2 then reads one list per (row, level) instead of
    // two.  Each direction's threads merge half of the levels; columns whose lists went to the
    // overflow arena keep both lists (pass 2 reads both).
    if (live && q < 0 && !ovfS[0][lc] && !ovfS[1][lc]) {
      const int64_t ts = (int64_t)(R + 2) * A.L.nx;     // one slot
      for (int k = d; k < LMAX; k += 2) {
        if (k0 + k > R) break;
        const int nf = cntS[0][k][lc], nr = cntS[1][k][lc];
        if (nr == 0) continue;
        float2* F = A.L.z + slot_z_index(A.L, row, 0, k0 + k, 0, i);
        const float2* Rl = A.L.z + slot_z_index(A.L, row, 1, k0 + k, 0, i);   // stored descending
        int fi = 0, ri = nr - 1, w = 0;
        float2 xf = nf > 0 ? F[0] : make_float2(INFINITY, INFINITY);
        float2 xr = Rl[(int64_t)ri * ts];
        float cs = 0.f, ce = 0.f;
        bool have = false;
        while (fi < nf || ri >= 0) {
          float2 x;
          if (ri < 0 || (fi < nf && xf.x <= xr.x)) {
            x = xf;
            if (++fi < nf) xf = F[(int64_t)fi * ts];
          } else {
            x = xr;
            if (--ri >= 0) xr = Rl[(int64_t)ri * ts];
          }
          if (!have) {
            cs = x.x; ce = x.y; have = true;
          } else if (x.x <= ce) {
            ce = fmaxf(ce, x.y);
          } else {
            F[(int64_t)(w++) * ts] = make_float2(cs, ce);
            cs = x.x; ce = x.y;
          }
        }
        if (have) F[(int64_t)(w++) * ts] = make_float2(cs, ce);
        A.L.cnt[slot_cnt_index(A.L, row, 0, k0 + k, i)] = (uint8_t)w;
        A.L.cnt[slot_cnt_index(A.L, row, 1, k0 + k, i)] = 0;
        tot_adj += w - nf - nr;
      }
    }
    tot += (uint32_t)tot_adj;              // (level intervals as stored, after the merge)
    if (q >= 0) tot = 0;                    // the overflow pass recounts nothing
    if (live && mx > (unsigned)A.L.cap) {
      atomicMax(A.flags, mx);
      // hand the column to the overflow pass -- once, whichever direction's thread gets here first
      if (q < 0 && atomicCAS(A.L.ovf_idx + c, -1, -2) == -1) {
        const unsigned slot = atomicAdd(A.flags + 1, 1u);
        if (slot < A.ovf_list_cap) {
          A.ovf_list[slot] = (uint32_t)c;
          A.L.ovf_idx[c] = (int32_t)slot;
        }
      }
    }
  }
  // statistics: one atomic per warp, no block barrier (warps retire independently)
  const unsigned wsum = __reduce_add_sync(0xffffffffu, tot);
  if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(A.nlev, (unsigned long long)wsum);
}

}  // namespace dexel
