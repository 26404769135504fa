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

// In-place running union: acc[0..n) (shared memory, stride T) holds sorted disjoint closed
// intervals.  Elements of one sorted list are inserted in order with a monotone cursor:
// an element inside an accumulator interval costs a compare (the common case -- most of
// the 4R+2 lists of a column fall inside what L_0 and the near rows already cover); an
// element that reaches outside merges the overlapped run of intervals and shifts the tail.
// Returns the new count (> cap: overflow, contents truncated).
struct Acc {
  float2* v;   // v[t * s]: shared memory (s = T, a compile-time constant) or global (the band's columns)
  int64_t s;
  int n;
};

template <int T>
__device__ __forceinline__ void acc_insert(Acc& A, int& p, float2& w, float a, float b, int cap, unsigned* need) {
  // p: first index with v[p].y >= a (monotone over one list, since the list's starts increase);
  // w caches v[p] (valid while p < n), so an element covered at the cursor costs no load
  while (p < A.n && w.y < a) {
    ++p;
    if (p < A.n) w = A.v[p * A.s];
  }
  if (p < A.n) {
    if (w.x <= a && b <= w.y) return;                 // covered
    if (w.x <= b) {                                   // overlaps [w.x, w.y]: merge the run p..q
      int q = p;
      float e = fmaxf(b, w.y);
      while (q + 1 < A.n && A.v[(q + 1) * A.s].x <= e) { ++q; e = fmaxf(e, A.v[q * A.s].y); }
      w = make_float2(fminf(a, w.x), e);
      A.v[p * A.s] = w;
      const int drop = q - p;
      if (drop) {
        for (int t = q + 1; t < A.n; ++t) A.v[(t - drop) * A.s] = A.v[t * A.s];
        A.n -= drop;
      }
      return;
    }
  }
  // disjoint from everything: insert before p (shift the tail right)
  if (A.n >= cap) { *need = max(*need, (unsigned)(A.n + 1)); return; }
  for (int t = A.n; t > p; --t) A.v[t * A.s] = A.v[(t - 1) * A.s];
  w = make_float2(a, b);
  A.v[p * A.s] = w;
  ++A.n;
}

constexpr int P2_R = 8;   // list elements loaded per batch

// insert a sorted list (element e at B[e * stride]) into the accumulator, P2_R elements at a
// time: the batch's loads are independent and issue together (unrolled), the batch is parked in
// a per-thread shared scratch and inserted by a rolled loop -- one inlined copy of acc_insert
// keeps the kernel small enough for the instruction cache.  (Level sets are stored unclipped:
// each element is clipped to [zlo, zhi] here; clipping commutes with the union.)
// one batch (<= P2_R elements) of a sorted list: element e at B[e * stride]
struct P2Batch {
  float2 x[P2_R];
  int n;
};

template <int T>
__device__ __forceinline__ void p2_load(P2Batch& X, const float2* __restrict__ B, int nb, int64_t stride) {
  X.n = min(P2_R, nb);
#pragma unroll
  for (int u = 0; u < P2_R; ++u)
    if (u < X.n) X.x[u] = B[(int64_t)u * stride];
}

// insert a loaded batch: parked in a per-thread shared scratch and inserted by a rolled loop --
// one inlined copy of acc_insert keeps the kernel small enough for the instruction cache.
// (Level sets are stored unclipped: each element is clipped to [zlo, zhi] here; clipping
// commutes with the union.)
template <int T>
__device__ __forceinline__ void p2_insert(Acc& A, int& p, float2& w, const P2Batch& X, float2* scratch, float zlo,
                                          float zhi, int cap, unsigned* need) {
#pragma unroll
  for (int u = 0; u < P2_R; ++u)
    if (u < X.n) scratch[u * T] = X.x[u];
#pragma unroll 1
  for (int u = 0; u < X.n; ++u) {
    const float2 v = scratch[u * T];
    const float lo = fmaxf(v.x, zlo), hi = fminf(v.y, zhi);
    if (lo < hi) acc_insert<T>(A, p, w, lo, hi, cap, need);
  }
}

// insert a sorted list whose first batch X is already loaded (the rare rest batch by batch)
template <int T>
__device__ __forceinline__ void acc_insert_list(Acc& A, const P2Batch& X0, const float2* __restrict__ B, int nb,
                                                int64_t stride, float2* scratch, float zlo, float zhi, int cap,
                                                unsigned* need) {
  int p = 0;
  float2 w = A.n > 0 ? A.v[0] : make_float2(0.f, 0.f);
  p2_insert<T>(A, p, w, X0, scratch, zlo, zhi, cap, need);
  for (int e0 = P2_R; e0 < nb; e0 += P2_R) {
    P2Batch X;
    p2_load<T>(X, B + (int64_t)e0 * stride, nb - e0, stride);
    p2_insert<T>(A, p, w, X, scratch, zlo, zhi, cap, need);
  }
}

// union over dy of one family's level lists for output column (i, jg): for each row
// offset dy = 0, 1, -1, 2, -2, ... the list L_|dy| of column (i, jg+dy).  The next row's
// first batch is loaded before the current row is inserted (two rows' loads in flight), and
// counts are read one row further ahead.
template <int T>
__device__ __forceinline__ void p2_family(const LevelSlots& L, int i, int jg, float zlo, float zhi, Acc& A,
                                          float2* scratch, int cap, unsigned* need) {
  A.n = 0;
  const int dlo = max(-L.ry, L.row0 - jg), dhi = min(L.ry, L.row0 + L.nrows - 1 - jg);
  const int nt = 2 * L.ry + 1;
  auto dy_of = [](int t) { return (t & 1) ? ((t + 1) >> 1) : -(t >> 1); };
  auto count = [&](int t) -> int {
    if (t >= nt) return 0;
    const int dy = dy_of(t), k = dy < 0 ? -dy : dy;
    return (dy < dlo || dy > dhi) ? 0 : (int)L.cnt[slot_cnt_index(L, jg + dy - L.row0, k, i)];
  };
  // list of row offset t (count word cw != 0): first element's address and stride, first batch
  // loaded; returns the list length
  auto open = [&](int t, int cw, const float2*& lb, int64_t& st, P2Batch& X) -> int {
    const int dy = dy_of(t), k = dy < 0 ? -dy : dy, jl = jg + dy - L.row0;
    // (a slot list longer than cap that found no arena slot: the op reruns, read what exists)
    const int nb = (cw & LV_IN_ARENA) ? (cw & LV_CNT_MAX) : min(cw & LV_CNT_MAX, L.cap);
    if (!(cw & LV_IN_ARENA)) {
      lb = L.z + slot_z_index(L, jl, k, 1, i);
      st = (int64_t)(L.R + 2) * L.nx;   // one slot
    } else {   // the column's lists live in the overflow arena
      lb = L.ovf_z + ovf_z_index(L, L.ovf_idx[(size_t)jl * L.nx + i], k, 1);
      st = 1;
    }
    p2_load<T>(X, lb, nb, st);
    return nb;
  };
  int cw = count(0), cwn = count(1), n = 0;
  const float2* lb = nullptr;
  int64_t st = 0;
  P2Batch X;
  X.n = 0;
  if (cw & LV_CNT_MAX) n = open(0, cw, lb, st, X);
  for (int t = 0; t < nt; ++t) {
    const int nc = n;
    const float2* lbc = lb;
    const int64_t stc = st;
    const P2Batch Xc = X;
    cw = cwn;
    cwn = count(t + 2);
    n = (cw & LV_CNT_MAX) ? open(t + 1, cw, lb, st, X) : 0;
    if (nc) acc_insert_list<T>(A, Xc, lbc, nc, stc, scratch, zlo, zhi, cap, need);
  }
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
  Acc U = GACC ? Acc{gacc + cl, (int64_t)nrows_out * nx, 0} : Acc{p2_smem + tid, T, 0};
  float2* scratch = p2_smem + (GACC ? 0 : (size_t)acc * T) + tid;     // [P2_R][T]
  p2_family<T>(A, i, jg, zlo, zhi, U, scratch, acc, &need);
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
    if (nu > 0) p2_family<T>(B, i, jg, U.v[0].x, U.v[(nu - 1) * U.s].y, U, scratch, acc, &need);
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
}

inline size_t pass2_smem_bytes(int op, int acc, int T, bool gacc = false) {
  (void)op;
  return (size_t)((gacc ? 0 : acc) + P2_R) * T * sizeof(float2);
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
