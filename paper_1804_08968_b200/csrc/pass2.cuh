// pass2.cuh -- pass 2 along y over the level slots, and the output compaction.
//
// out(i,j) = clip_U  U_{|dy| <= R, row j+dy in the grid}  L_|dy|(i, j+dy)      (dilate)
// A piece of M(i, j+dy) at level kappa reaches row j exactly where its power
// weight r^2 - (kappa^2 + dy^2) s^2 >= 0:
// L_|dy| of levels.cuh is that set, so pass 2 is a plain union of 2R+1 sorted
// disjoint lists per output column ("the union of both").
// Epilogues (reading R6, neutral boundary):
//   erode  E = [z_lo, z_hi] \ D_r(C)      (family A is the dilation of C)
//   shell  D_rout(S) n D_rin(C)           (= D \ E; families A = S, B = C)
//
// One thread per output column; a warp covers 32 consecutive columns of a row,
// so every list read (fixed row, level, slot t) is a coalesced 256-byte access.
// The running union lives in shared memory ([slot][thread], conflict-free) and is
// updated in place (acc_insert); a union longer than `acc` raises a flag and the
// host reruns with a larger accumulator.  Results go to a
// [t][column] staging array; compact_kernel moves them into the output CSR once
// the counts are scanned (two-phase allocation without recomputation).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "levels.cuh"

namespace dexel {

enum { OP_DILATE = 0, OP_ERODE = 1, OP_SHELL = 2 };

// In-place running union: acc[0..n) (shared memory, stride T; or global) holds sorted disjoint
// closed intervals, followed by a sentinel acc[n] = (+inf, +inf), so cursor scans need no bound
// test.  The elements of one list are inserted in order with a forward cursor p (the first
// interval whose end reaches the element's start); w caches acc[p] and n1 the next interval's start,
// so an element that is covered by w, or extends w without reaching the next interval -- the common
// cases: most of the 4R+2 lists of a column fall inside or at the edges of what L_0 and the near rows
// already cover -- costs two compares, a min / max and a store.  Anything else (a disjoint element:
// insert and shift the tail; an element reaching the next interval: merge the run) takes the
// general path.  A union longer than `cap` raises *need (the host reruns with a larger accumulator).
struct Acc {
  float2* v;   // v[t * s]: shared memory (s = T, a compile-time constant) or global (the band's columns)
  int64_t s;
  int n;
  int hw = 0;  // the most intervals it held (insertions only raise it: one max per insertion)
};

struct Cursor {
  int p;
  float2 w;    // v[p]
  float n1;    // v[p + 1].x (p < n; +inf at the sentinel)
};

__device__ __forceinline__ void cur_load(const Acc& A, Cursor& C) {
  C.w = A.v[C.p * A.s];
  C.n1 = C.p < A.n ? A.v[(C.p + 1) * A.s].x : INFINITY;
}

// one element [a, b] (clipped, a < b) of a list, cursor C of this list
__device__ __forceinline__ void acc_add(Acc& A, Cursor& C, float a, float b, int cap, unsigned* need) {
  while (C.w.y < a) {   // (the sentinel stops it)
    ++C.p;
    cur_load(A, C);
  }
  if (b >= C.w.x && b < C.n1) {   // covered by w, or extends w within the gap before the next one
    C.w = make_float2(fminf(a, C.w.x), fmaxf(b, C.w.y));
    A.v[C.p * A.s] = C.w;
    return;
  }
  if (b < C.w.x) {   // disjoint: insert before p (at p == n: append), shifting the tail and the sentinel
    if (A.n >= cap) {
      *need = max(*need, (unsigned)(A.n + 1));
      return;
    }
    for (int t = A.n; t >= C.p; --t) A.v[(t + 1) * A.s] = A.v[t * A.s];
    ++A.n;
    A.hw = max(A.hw, A.n);
    C.n1 = C.w.x;
    C.w = make_float2(a, b);
    A.v[C.p * A.s] = C.w;
    return;
  }
  // overlaps w and reaches the next interval: merge the run
  int q = C.p;
  float e = fmaxf(b, C.w.y);
  while (A.v[(q + 1) * A.s].x <= e) {   // (q + 1 <= n: the sentinel's +inf stops it)
    ++q;
    e = fmaxf(e, A.v[q * A.s].y);
  }
  C.w = make_float2(fminf(a, C.w.x), e);
  A.v[C.p * A.s] = C.w;
  const int drop = q - C.p;
  for (int t = q + 1; t <= A.n; ++t) A.v[(t - drop) * A.s] = A.v[t * A.s];   // (incl. the sentinel)
  A.n -= drop;
  C.n1 = A.v[(C.p + 1) * A.s].x;
}

#ifndef P2_R_N
#define P2_R_N 6
#endif
constexpr int P2_R = P2_R_N;   // list elements fetched per batch

// union over dy of one family's level lists for output column (i, jg): for each row offset
// dy = 0, 1, -1, 2, -2, ... the list L_|dy| of column (i, jg+dy), in lockstep across the warp (every
// list read is coalesced).  The first P2_R elements of the next list are copied into this thread's
// half of a double-buffered shared scratch with cp.async while the current list is inserted (counts
// are read one list further ahead); longer lists fetch the rest batch by batch.  Level sets are
// stored unclipped: each element is clipped to [zlo, zhi] here (clipping commutes with the union).
template <int T>
__device__ __forceinline__ void p2_family(const LevelSlots& L, int i, int jg, float zlo, float zhi, Acc& A,
                                          uint32_t scr, int cap, unsigned* need) {
  A.n = 0;
  A.v[0] = make_float2(INFINITY, INFINITY);
  const int dlo = max(-L.ry, L.row0 - jg), dhi = min(L.ry, L.row0 + L.nrows - 1 - jg);
  const int nt = 2 * L.ry + 1;
  auto dy_of = [](int t) { return (t & 1) ? ((t + 1) >> 1) : -(t >> 1); };
  // row jg's counts and level slots; row jg + dy, level k at  + dy * (one row) + k * nx
  const uint16_t* cnt0 = L.cnt + slot_cnt_index(L, jg - L.row0, 0, i);
  const int64_t crow = (int64_t)(L.R + 1) * L.nx;
  const float2* z0 = L.z + slot_z_index(L, jg - L.row0, 0, 1, i);
  const int64_t zrow = (int64_t)(L.cap + 1) * (L.R + 2) * L.nx, zslot = (int64_t)(L.R + 2) * L.nx;
  auto count = [&](int t) -> int {
    if (t >= nt) return 0;
    const int dy = dy_of(t), k = dy < 0 ? -dy : dy;
    return (dy < dlo || dy > dhi) ? 0 : (int)cnt0[(int64_t)dy * crow + k * L.nx];
  };
  // list t (count word cw != 0): its first element's address and stride, its length; the first
  // batch is copied into scratch half h
  auto open = [&](int t, int cw, const float2*& lb, int64_t& st, uint32_t h) -> int {
    const int dy = dy_of(t), k = dy < 0 ? -dy : dy;
    int nb;
    if (!(cw & LV_IN_ARENA)) {
      // (a slot list longer than cap that found no arena slot: the op reruns, read what exists)
      nb = min(cw & LV_CNT_MAX, L.cap);
      lb = z0 + (int64_t)dy * zrow + k * L.nx;
      st = zslot;
    } else {   // (rare) the column's lists live in the overflow arena
      nb = cw & LV_CNT_MAX;
      lb = L.ovf_z + ovf_z_index(L, L.ovf_idx[(size_t)(jg + dy - L.row0) * L.nx + i], k, 1);
      st = 1;
    }
    const uint32_t sb = scr + h * (uint32_t)(P2_R * T * 8);
#pragma unroll
    for (int u = 0; u < P2_R; ++u)
      if (u < nb) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sb + (uint32_t)(u * T * 8)),
                               "l"(lb + u * st));
    return nb;
  };
  int cw = count(0), cwn = count(1), n = 0;
  const float2* lb = nullptr;
  int64_t st = 0;
  uint32_t h = 0;
  if (cw & LV_CNT_MAX) n = open(0, cw, lb, st, 0);
  asm volatile("cp.async.commit_group;\n" ::);
  for (int t = 0; t < nt; ++t) {
    const int nc = n;
    const float2* lbc = lb;
    const int64_t stc = st;
    const uint32_t hc = h;
    cw = cwn;
    cwn = count(t + 2);
    h ^= 1u;
    n = (cw & LV_CNT_MAX) ? open(t + 1, cw, lb, st, h) : 0;
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 1;\n" ::);   // list t's batch has landed
    if (nc) {
      Cursor C{0, A.v[0], A.n > 0 ? A.v[A.s].x : INFINITY};
      float alast = -INFINITY;
      const uint32_t sb = scr + hc * (uint32_t)(P2_R * T * 8);
      for (int e0 = 0; e0 < nc; e0 += P2_R) {
        if (e0 > 0) {   // (a list longer than P2_R) its next batch into the same half, then wait for it
#pragma unroll
          for (int u = 0; u < P2_R; ++u)
            if (e0 + u < nc)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sb + (uint32_t)(u * T * 8)),
                           "l"(lbc + (e0 + u) * stc));
          asm volatile("cp.async.commit_group;\n" ::);
          asm volatile("cp.async.wait_group 0;\n" ::);
        }
        const int nu = min(nc - e0, P2_R);
#pragma unroll 1
        for (int u = 0; u < nu; ++u) {
          float2 v;
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(sb + (uint32_t)(u * T * 8)));
          const float lo = fmaxf(v.x, zlo), hi = fminf(v.y, zhi);
          if (lo < hi) {
            // a level list is sorted by component end; a component may start below earlier ones
            // (levels.cuh: not merged there) -- the cursor then restarts (rare)
            if (lo < alast) {
              C.p = 0;
              cur_load(A, C);
            }
            alast = lo;
            acc_add(A, C, lo, hi, cap, need);
          }
        }
      }
    }
  }
  asm volatile("cp.async.wait_all;\n" ::);
}

// output rows [row0, row0 + nrows_out) (extended-row numbering of the level slots) of a band;
// output column c_local of the band is global output column cbase + c_local; the staging
// array is [t][ncol_total]
// GACC: the accumulator lives in global memory ([acc][band columns], gacc) -- for unions longer
// than the shared memory holds; else in shared memory
template <int OP, int T, bool GACC>
__global__ void __launch_bounds__(T, 640 / T) pass2s_kernel(LevelSlots A, LevelSlots B, int nx, int row0, int nrows_out,
                                                   int64_t cbase, int64_t ncol, float zlo, float zhi, int acc,
                                                   float2* __restrict__ ostage, uint32_t* __restrict__ ocnt,
                                                   unsigned* flags, float2* __restrict__ gacc) {
  extern __shared__ __align__(16) float2 p2_smem[];
  const int tid = threadIdx.x;
  // column-tile-major block order: consecutive blocks are consecutive rows of one tile of T
  // columns, so the blocks reading a level list (output rows j +- k) run close together in time
  // and the list is read from L2 (row-major order put them ~2R rows x nx columns apart)
  const int tile = (int)(blockIdx.x / (unsigned)nrows_out), jr = (int)(blockIdx.x % (unsigned)nrows_out);
  const int i = tile * T + tid;
  if (i >= nx) return;
  const int64_t cl = (int64_t)jr * nx + i;
  const int64_t c = cbase + cl;
  const int jg = row0 + jr;
  unsigned need = 0;
  // shared memory: the accumulators [acc + 2][T] (+ the sentinel; unless global), the list scratch
  // [2][P2_R][T]
  Acc U = GACC ? Acc{gacc + cl, (int64_t)nrows_out * nx, 0} : Acc{p2_smem + tid, T, 0};
  const uint32_t scr = (uint32_t)__cvta_generic_to_shared(p2_smem + (GACC ? 0 : (size_t)(acc + 2) * T) + tid);
  p2_family<T>(A, i, jg, zlo, zhi, U, scr, acc, &need);
  uint32_t n = 0;
  if (OP == OP_DILATE) {
    for (int t = 0; t < U.n; ++t) ostage[(size_t)t * ncol + c] = U.v[t * U.s];
    n = U.n;
  } else if (OP == OP_ERODE) {
    float cur = zlo;
    for (int t = 0; t < U.n; ++t) {
      const float2 v = U.v[t * U.s];
      if (v.x > cur) ostage[(size_t)(n++) * ncol + c] = make_float2(cur, v.x);
      cur = v.y;
    }
    if (zhi > cur) ostage[(size_t)(n++) * ncol + c] = make_float2(cur, zhi);
  } else {   // shell: D_rout(S) n D_rin(C)
    // park D_rout(S) in the upper half of this column's staging slots (coalesced), reuse the
    // shared accumulator for D_rin(C), then intersect into the lower half (the result has
    // at most |U| + |V| - 1 <= 2 acc - 1 intervals and is written behind the reads)
    const int nu = U.n;
    for (int t = 0; t < nu; ++t) ostage[(size_t)(acc + t) * ncol + c] = U.v[t * U.s];
    // D_rin(C) only matters inside D_rout(S): an empty D(S) skips it, and its list elements are
    // clipped to D(S)'s hull instead of [z_lo, z_hi] (fewer insertions, a shorter accumulator)
    if (nu > 0) p2_family<T>(B, i, jg, U.v[0].x, U.v[(nu - 1) * U.s].y, U, scr, acc, &need);
    else U.n = 0;
    int p = 0, q = 0;
    float2 u = nu > 0 ? ostage[(size_t)acc * ncol + c] : make_float2(0.f, 0.f);
    while (p < nu && q < U.n) {
      const float2 v = U.v[q * U.s];
      const float lo = fmaxf(u.x, v.x), hi = fminf(u.y, v.y);
      if (lo < hi) ostage[(size_t)(n++) * ncol + c] = make_float2(lo, hi);
      if (u.y < v.y) {
        if (++p < nu) u = ostage[(size_t)(acc + p) * ncol + c];
      } else {
        ++q;
      }
    }
  }
  ocnt[c] = n;
  if (need) atomicMax(flags + OPF_P2_ACC, need);
  // the longest union of the op (one atomic per warp): the host sizes the next op's accumulator by it
  // -- a shorter accumulator is less shared memory per warp, so more resident warps for this
  // latency-bound kernel
  const unsigned am = __activemask();
  const unsigned pk = __reduce_max_sync(am, (unsigned)U.hw);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(am) - 1)) atomicMax(flags + OPF_P2_PEAK, pk);
}

inline size_t pass2_smem_bytes(int op, int acc, int T, bool gacc = false) {
  (void)op;
  return (size_t)((gacc ? 0 : acc + 2) + 2 * P2_R) * T * sizeof(float2);
}
constexpr size_t P2_SMEM_MAX = 220 * 1024;   // shared memory an accumulator block may take
inline int pass2_stage_cap(int op, int acc) { return op == OP_SHELL ? 2 * acc : acc + 1; }

// CSR compaction: out[off[c] + t] = stage[t][c] -- when the total off[ncol] fits the buffer's
// capacity; else nothing is written and the op's OPF_OUT_FIT flag asks the host to reallocate and
// compact again (the op's one readback tells it; the staging array is still alive then)
__global__ void compact_kernel(const float2* __restrict__ stage, const uint32_t* __restrict__ cnt,
                               const uint64_t* __restrict__ off, int64_t ncol, float2* __restrict__ out,
                               uint64_t cap, unsigned* __restrict__ opf) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  if (off[ncol] > cap) {
    if (c == 0) atomicOr(opf + OPF_OUT_FIT, 1u);
    return;
  }
  const uint32_t n = cnt[c];
  const uint64_t o = off[c];
  for (uint32_t t = 0; t < n; ++t) out[o + t] = stage[(size_t)t * ncol + c];
}

}  // namespace dexel
