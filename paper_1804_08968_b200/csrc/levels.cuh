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
// so the level set pass 2 needs is
//     L_k = U_p [lo_p - h, hi_p + h]    (= U_f(k) u U_r(k) with U_f = U_p [lo_p, hi_p + h] and
//                                         U_r = U_p [lo_p - h, hi_p], the two half-space parts)
// The pieces are sorted and disjoint, so their grown intervals come in ascending lo_p but
// not ascending lo_p - h.  One forward sweep builds L_k as a list of components (the
// half-space envelope's sweep, restated for level sets): the top
// component [cs, ce] lives in registers; a grown interval starting above ce closes it
// (push: written to the level's slots), otherwise it extends it.  A grown interval that
// reaches below the end of components pushed earlier (a small-kappa piece swallowing a gap
// left by out-of-reach pieces; ~1-3 times per column per ~3000 (piece, level) steps on C5)
// is not merged with them: the list stays sorted by component end and pass 2, a union,
// takes it as it is (its cursor restarts where a list's starts decrease).  So the main step
// is two fp32 adds (one packed FADD2 per two levels), two compares / min-max and a
// predicated store -- no branches, no square roots (the h table is fp64 on the host,
// rounded once to fp32, reading R20).  A thread owns one column and a chunk of
// LMAX levels held in registers (blockIdx.y = chunk), so the kernel is SIMT-uniform.  (An
// explicit upper-envelope variant ran 4-10x slower; two half-space sweeps U_f / U_r in
// separate threads plus a merge ran ~1.5x slower: DESIGN.md "What was tried".)
//
// Input: pass-1 piece chunks (kernels.cuh PieceSlots) through a cp.async ring.
// Layout (HBM): level slots  z[((row*(cap+1) + t)*(R+2) + k)*nx + i]  (float2), t = 1..cap
// hold L_k ascending (slot 0 is a dummy that absorbs the sweep's first, empty, push), and
// counts cnt[(row*(R+1) + k)*nx + i] (u16).  For a fixed (row, k, t) the nx columns of a
// row are contiguous, so a warp of 32 consecutive columns writes and (in pass 2) reads
// 256 contiguous bytes.  A list longer than cap raises a flag: the column is listed and
// an overflow pass rewrites all its lists into an arena of lists and flags their counts
// (LV_IN_ARENA: the flag, not the count, tells pass 2 where a list is); if too many
// columns overflow the host reruns the band with a larger cap.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace dexel {

constexpr int LV_SLOT_MAX = 255;    // largest slot capacity the host grows to (then: the arena)
constexpr int LV_CNT_MAX = 0x7fff;  // longest list a u16 count (bit 15 = arena flag) can describe
constexpr uint16_t LV_IN_ARENA = 0x8000;   // count flag: the column's lists live in the overflow arena
// the level sweep clamps its slot offsets once per LV_CLAMP pieces (not per piece): a list may run
// LV_CLAMP - 1 slots past the clamp point before the next clamp, so the last LV_CLAMP - 1 slots of a
// row (spill level R+1) and LV_CLAMP spill entries per arena slot absorb those writes, and a list is
// complete only if it ends LV_CLAMP - 1 slots short of the capacity (slot capacity >= LV_CLAMP)
constexpr int LV_CLAMP = 4;

struct LevelSlots {
  uint16_t* cnt;     // [nrows][R+1][nx]  list lengths (<= LV_CNT_MAX); LV_IN_ARENA set: the list is in the arena
  float2* z;         // [nrows][cap+1][R+2][nx]  (unclipped; slot 0 dummy; level R+1 of the last slot = spill cell)
  int R, cap, nx, nrows;
  int ry;            // row offsets pass 2 reads: |dy| <= ry (R; 0 for slices, 2D offsets of each row)
  int row0;          // row (in the op's extended-row numbering) of slot row 0
  // columns with a list longer than cap keep all their lists in the overflow arena:
  // list k of overflow slot q at ovf_z[q*((R+1)*(ovf_cap+1) + LV_CLAMP) + k*(ovf_cap+1) + t], t = 1..ovf_cap
  // (0 dummy; the LV_CLAMP extra entries per slot are its spill cells);
  // ovf_cap = the most pieces of any listed column (a level list never holds more components
  // than the column has pieces: each push starts with one)
  int32_t* ovf_idx;  // [nrows*nx] overflow slot of a column (valid only where some count > cap)
  float2* ovf_z;
  int ovf_cap;
};

__host__ __device__ __forceinline__ size_t slot_cnt_index(const LevelSlots& L, int row, int k, int i) {
  return ((size_t)row * (L.R + 1) + k) * L.nx + i;
}
// z slots, slot-major inside a row: z[((row*(cap+1) + t)*(R+2) + k)*nx + i], list element e
// (0-based) in slot t = e + 1.  Level R+1 of the last slot is a spill cell: a push is written
// at min(offset, spill), so an overflowing list (t > cap) only ever hits the spill cell (its
// column is then redone in the overflow arena) and never another list.
__host__ __device__ __forceinline__ size_t slot_z_index(const LevelSlots& L, int row, int k, int t, int i) {
  return (((size_t)row * (L.cap + 1) + t) * (L.R + 2) + k) * L.nx + i;
}

__host__ __device__ __forceinline__ size_t ovf_z_index(const LevelSlots& L, int q, int k, int t) {
  return (size_t)q * ((size_t)(L.R + 1) * (L.ovf_cap + 1) + LV_CLAMP) + (size_t)k * (L.ovf_cap + 1) + t;
}

struct LvArgs {
  PieceSlots P;            // pass-1 pieces of the level rows (kernels.cuh)
  int64_t ncol;
  const float* h;          // [(R+1)^2] fl32(sqrt(r^2 - (kappa^2 + k^2) s^2)), -1 where negative
  float zlo, zhi;
  LevelSlots L;
  unsigned* flags;         // [1] overflow columns (device counter of this band/family)
  unsigned long long* nlev;  // total level intervals (statistics, the op's counter)
  unsigned long long* dbg; // diagnostics or nullptr: [0] sum of per-warp max piece counts, [1] warps, [2] pieces
  uint32_t* ovf_list;      // main pass: columns with a list longer than cap
  unsigned ovf_list_cap;
  const uint32_t* list;    // overflow pass: the listed columns (count flags[1], read on the device)
  unsigned* opf;           // the op's flag words (kernels.cuh OpFlag)
  uint32_t one = 1;        // 1, opaque to the compiler (a predicated multiply-add by it is a move that
                           // issues on the FMA pipe; ptxas turns plain predicated moves into ALU selects)
};

#ifndef LV_T_N
#define LV_T_N 64
#endif
constexpr int LV_T = LV_T_N;
#ifndef LV_DC_N
#define LV_DC_N 3
#endif
constexpr int LV_DC = LV_DC_N;     // piece chunks (4 pieces each) per thread in the cp.async ring

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {   // dst: shared address
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// predicated 8-byte store without a branch (the compiler otherwise wraps each level's rare
// emission in a BSSY/BRA/BSYNC region that some lane of the warp takes almost every step)
__device__ __forceinline__ void st_pred_f2(float2* p, float x, float y, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.global.v2.f32 [%0], {%1, %2};\n\t}"
               :: "l"(p), "f"(x), "f"(y), "r"((int)pred));
}

// blockIdx.y = level chunk: this thread runs levels k0 .. k0+LMAX-1 of column c.
// The h table holds NaN where a piece is out of reach (kappa^2 + k^2 > (r/s)^2): then
// s = lo - h and e = hi + h are NaN, "s > ce" is false (no push) and fminf/fmaxf ignore
// NaN -- an out-of-reach piece leaves the sweep unchanged without a validity test.
// Rows are HS floats (HS/4 odd): a row is read with 128-bit loads, and 8 lanes with
// different kappa hit 8 different bank groups.
template <int LMAX>
struct LvTab {
  static constexpr int NV = (LMAX + 3) / 4;                 // float4 per row actually used
  static constexpr int HS = 4 * (NV | 1);                   // row stride (floats), HS/4 odd
};

template <int LMAX>
__global__ void __launch_bounds__(LV_T, 512 / LV_T) levels_kernel(LvArgs A) {
  constexpr int NV = LvTab<LMAX>::NV, HS = LvTab<LMAX>::HS;
  __shared__ __align__(16) float Hs[257 * HS];   // h(kappa, k0 + k), NaN beyond R or out of reach;
                                                  // row R+1: all NaN (the "null piece")
  const int R = A.L.R, L1 = R + 1;
  const int k0 = blockIdx.y * LMAX;
  for (int t = threadIdx.x; t < (L1 + 1) * HS; t += LV_T) {
    const int kap = t / HS, kk = t % HS, k = k0 + kk;
    const float h = (kap <= R && kk < LMAX && k <= R) ? A.h[kap * L1 + k] : -1.0f;
    Hs[t] = h >= 0.f ? h : __int_as_float(0x7fc00000);   // quiet NaN
  }
  // pieces stream through a per-thread ring of LV_DC chunks (4 pieces = 32 bytes of z pairs as two
  // float4 halves + the 32-bit word of their kappa bytes) filled by cp.async: LV_DC - 1 chunks in
  // flight per thread, no registers held
  __shared__ float4 ringz[LV_DC][2][LV_T];
  __shared__ uint32_t ringk[LV_DC][LV_T];
  __syncthreads();
  // the main pass covers every column once; the overflow pass walks the listed columns (their
  // count read on the device, no host round trip), grid-stride, whole warps together
  const int64_t nwork = A.list ? (int64_t)min(A.ovf_list_cap, A.flags[1]) : A.ncol;
  const int64_t gstep = A.list ? (int64_t)gridDim.x * LV_T : (int64_t)1 << 62;
  for (int64_t gb = (int64_t)blockIdx.x * LV_T; gb < nwork; gb += gstep) {
  uint32_t tot = 0, mx = 0;
  const int64_t g = gb + threadIdx.x;
  const bool live = g < nwork;
  // every lane of the warp walks the same piece index t = 0..mmax-1: the chunk reads stay
  // coalesced and the loop never diverges; a lane past its own count processes the "null
  // piece" (kappa row R+1, all NaN), which leaves the sweep unchanged
  // (a column that outgrew its slots but found no arena slot has no pieces to read: the op is
  // rerun with larger capacities anyway -- OPF_P1_RERUN -- so it contributes nothing now)
  int m = live ? (int)A.P.cnt[A.list ? (int64_t)A.list[g] : g] : 0;
  if (m > A.P.cap && A.P.ovf_idx[A.list ? (int64_t)A.list[g] : g] < 0) m = 0;
  const int mmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)m);
  if (A.dbg) {                 // diagnostics (DEXEL_DEBUG): sums of warp maxima and of counts, warps
    const unsigned msum = __reduce_add_sync(0xffffffffu, (unsigned)m);
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(A.dbg, (unsigned long long)mmax);
      atomicAdd(A.dbg + 1, 1ull);
      atomicAdd(A.dbg + 2, (unsigned long long)msum);
    }
  }
  const int64_t c = live ? (A.list ? (int64_t)A.list[g] : g) : 0;
  const int q = A.list ? (int)g : -1;
  const int row = (int)(c / A.L.nx), i = (int)(c % A.L.nx);
  // this column's piece chunks: slots (chunk stride nx, coalesced across the warp) or the
  // pass-1 overflow arena (stride 1)
  const float4* zc;
  const uint32_t* kc;
  int64_t cstr;
  if (A.P.ovf_idx[c] < 0) {   // (a listed column's pieces live in the arena)
    zc = A.P.z + 2 * chunk_index(A.P, row, 0, i);
    kc = A.P.k + chunk_index(A.P, row, 0, i);
    cstr = A.P.nx;
  } else {
    const size_t qo = (size_t)A.P.ovf_idx[c] * (A.P.ovf_cap / 4);
    zc = A.P.ovf_z + 2 * qo;
    kc = A.P.ovf_k + qo;
    cstr = 1;
  }
  // main pass: slots of (row, level k0); overflow pass: the arena lists of slot q.
  // o[k] = offset (float2) of the next free slot of level k0+k from Zd; slot 0 is the dummy.
  float2* Zd = q < 0 ? A.L.z + slot_z_index(A.L, row, k0, 0, i) : A.L.ovf_z + ovf_z_index(A.L, q, k0, 0);
  const uint32_t nx = (uint32_t)A.L.nx;
  const uint32_t ostep = q < 0 ? (uint32_t)(R + 2) * nx : 1u;           // one slot
  const uint32_t olev = q < 0 ? nx : (uint32_t)(A.L.ovf_cap + 1);      // one level
  const uint32_t ncap = q < 0 ? (uint32_t)A.L.cap : (uint32_t)A.L.ovf_cap;
  // the spill cells: level R+1 of the last LV_CLAMP slots (main pass), the arena slot's extra entries
  // (overflow pass) -- never list entries.  Offsets are clamped to osat once per LV_CLAMP pieces, so
  // a list at or beyond osat after a clamp has overflowed (its pushes in between land in the spill
  // cells osat .. osat + (LV_CLAMP-1) ostep, or in its own slots up to the capacity).
  const uint32_t osat = q < 0 ? (ncap - (uint32_t)(LV_CLAMP - 1)) * ostep + (uint32_t)(R + 1 - k0) * nx
                              : (uint32_t)(R + 1 - k0) * olev;
  float cs[LMAX], ce[LMAX];
  uint32_t o[LMAX];
  bool lost = false;
#pragma unroll
  for (int k = 0; k < LMAX; ++k) {
    cs[k] = INFINITY;     // empty top
    ce[k] = -INFINITY;
    o[k] = min((uint32_t)k * olev, osat);
  }
  const int nchunk = (m + 3) >> 2;
  // shared addresses computed once (ring slots of this thread, the h table)
  const uint32_t rz_a = sh_addr(&ringz[0][0][threadIdx.x]), rk_a = sh_addr(&ringk[0][threadIdx.x]);
  const uint32_t hs_a = sh_addr(Hs);
  const uint32_t one = A.one;
  auto issue = [&](int cq) {
    if (cq < nchunk) {
      const uint32_t u = (uint32_t)(cq % LV_DC);
      const float4* src = zc + 2 * (int64_t)cq * cstr;
      cp_async16(rz_a + u * (2 * LV_T * 16), src);
      cp_async16(rz_a + u * (2 * LV_T * 16) + LV_T * 16, src + 1);
      cp_async4(rk_a + u * (LV_T * 4), kc + (int64_t)cq * cstr);
    }
    cp_async_commit();   // (empty groups too: the wait count stays uniform)
  };
#pragma unroll
  for (int t = 0; t < LV_DC - 1; ++t) issue(t);
  uint32_t kw = 0;
  uint32_t u = 0;                     // ring slot of chunk t / 4
  for (int t = 0; t < mmax; ++t) {
    if ((t & 3) == 0) {
      static_assert(LV_CLAMP == 4, "the clamp runs with the ring's 4-piece chunks");
#pragma unroll
      for (int k = 0; k < LMAX; ++k) o[k] = min(o[k], osat);
      issue((t >> 2) + LV_DC - 1);
      cp_async_wait<LV_DC - 1>();     // chunk t/4 has landed (this thread's own copies)
      kw = lds_u32(rk_a + u * (LV_T * 4));
    }
    float2 p = make_float2(0.f, 0.f);
    int nk = L1;                      // past the column's pieces: the null piece
    if (t < m) {
      p = lds_f2(rz_a + u * (2 * LV_T * 16) + (uint32_t)((t >> 1) & 1) * (LV_T * 16) + (uint32_t)(t & 1) * 8u);
      nk = (int)((kw >> (8u * (uint32_t)(t & 3))) & 0xffu);
    }
    if ((t & 3) == 3) u = u == LV_DC - 1 ? 0u : u + 1u;
    const uint32_t hrow = hs_a + (uint32_t)(nk * HS) * 4u;
    float hv[4 * NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const float4 v = lds_f4(hrow + 16u * j);
      hv[4 * j] = v.x; hv[4 * j + 1] = v.y; hv[4 * j + 2] = v.z; hv[4 * j + 3] = v.w;
    }
    // reach is monotone in k: skip when no lane's piece reaches this chunk (warp-uniform).
    // (Level 0 is in reach of every real piece and t < mmax leaves some lane a real piece, so
    // the first chunk never skips -- the test, which waits on the table load, runs from k0 > 0.)
    if (k0 > 0 && __all_sync(0xffffffffu, isnan(hv[0]))) continue;
    // the grown ends of all levels first, two levels per packed fp32 instruction (FADD2, sm_100a:
    // one issue slot for two exact fp32 additions, the same rounding as two FADDs)
    float sv[LMAX], ev[LMAX];
#pragma unroll
    for (int k = 0; k + 1 < LMAX; k += 2) {
      asm("{\n\t.reg .b64 x, y, h, r;\n\tmov.b64 x, {%4, %4};\n\tmov.b64 y, {%5, %5};\n\t"
          "mov.b64 h, {%6, %7};\n\tsub.rn.f32x2 r, x, h;\n\tmov.b64 {%0, %1}, r;\n\t"
          "add.rn.f32x2 r, y, h;\n\tmov.b64 {%2, %3}, r;\n\t}"
          : "=f"(sv[k]), "=f"(sv[k + 1]), "=f"(ev[k]), "=f"(ev[k + 1])
          : "f"(p.x), "f"(p.y), "f"(hv[k]), "f"(hv[k + 1]));
    }
    if constexpr (LMAX & 1) {
      sv[LMAX - 1] = p.x - hv[LMAX - 1];
      ev[LMAX - 1] = p.y + hv[LMAX - 1];
    }
#pragma unroll
    for (int k = 0; k < LMAX; ++k) {
      const float s = sv[k], e = ev[k];
      // push (s > ce): the top is written to its slot (the first push writes the empty top into
      // the dummy slot 0), the offset advances one slot (clamped at the next 4-piece boundary,
      // above) and the new top starts at s.  Else the top extends (cs = min(cs, s)).  Either way
      // ce = max(ce, e) (a push has e >= s > ce).  Predicated, no branch.  The step is issue-bound:
      // the moves are predicated multiply-adds by an opaque 1 and the offset a predicated add, which
      // ptxas issues on the FMA pipe (plain predicated moves become ALU selects).
      // A top extended below the end of components pushed before it (a small-kappa piece swallowing
      // a gap left by out-of-reach pieces: ~1-3 times per column per ~3000 steps on C5) is NOT merged
      // with them here: the list stays sorted by component end, every component is a union of grown
      // pieces, and pass 2 (a union) takes the components in any order -- so the sweep keeps no
      // previous-end register and no merge test (2 of ~11 instructions per (piece, level)).
      asm volatile("{\n\t.reg .pred q;\n\t.reg .b32 a, b;\n\t"
                   "setp.gt.f32 q, %3, %1;\n\t"
                   "@q st.global.v2.f32 [%4], {%0, %1};\n\t"
                   "@q add.u32 %2, %2, %5;\n\t"
                   "@!q min.f32 %0, %0, %3;\n\t"
                   "mov.b32 a, %3;\n\t"
                   "mov.b32 b, %0;\n\t"
                   "@q mad.lo.u32 b, a, %6, 0;\n\t"
                   "mov.b32 %0, b;\n\t"
                   "}"
                   : "+f"(cs[k]), "+f"(ce[k]), "+r"(o[k])
                   : "f"(s), "l"(Zd + o[k]), "r"(ostep), "r"(one) : "memory");
      ce[k] = fmaxf(ce[k], e);
    }
  }
#pragma unroll
  for (int k = 0; k < LMAX; ++k) {
    o[k] = min(o[k], osat);
    const bool top = cs[k] < ce[k];   // (the top is empty only if no piece reached this level)
    st_pred_f2(Zd + o[k], cs[k], ce[k], top);
    lost |= k0 + k <= R && o[k] == osat;   // the offset saturated: the count is lost
    const uint32_t nk_ = top ? (o[k] - (uint32_t)k * olev) / ostep : 0u;   // slots 1..n
    if (live && k0 + k <= R) {
      A.L.cnt[slot_cnt_index(A.L, row, k0 + k, i)] =
          (uint16_t)(min(nk_, (uint32_t)LV_CNT_MAX) | (q < 0 ? 0u : LV_IN_ARENA));
      tot += nk_;
      mx = max(mx, nk_);
    }
  }
  if (lost) mx = max(mx, ncap + 1);   // (ncap + 1 > the effective capacity ncap - LV_CLAMP + 1)
  if (q >= 0) tot = 0;                    // the overflow pass recounts nothing
  if (live && q >= 0 && mx > ncap) {      // a list outgrew even the arena: rerun the op
    atomicOr(A.opf + OPF_LV_RERUN, 1u);
    atomicMax(A.opf + OPF_LV_LONGEST, mx);
  }
  if (live && q < 0 && mx > (unsigned)A.L.cap) {   // hand the column to the overflow pass
    const unsigned slot = atomicAdd(A.flags + 1, 1u);
    if (slot < A.ovf_list_cap) {
      A.ovf_list[slot] = (uint32_t)c;
      A.L.ovf_idx[c] = (int32_t)slot;
    } else {                              // too many long lists: rerun the op with larger slots
      atomicOr(A.opf + OPF_LV_RERUN, 1u);
      atomicMax(A.opf + OPF_LV_LONGEST, mx);
    }
  }
  // statistics: one atomic per warp, no block barrier (warps retire independently)
  const unsigned wsum = __reduce_add_sync(0xffffffffu, tot);
  if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(A.nlev, (unsigned long long)wsum);
  }
}

}  // namespace dexel
