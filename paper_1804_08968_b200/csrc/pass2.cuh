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
// The running union lives in shared memory ([slot][thread], conflict-free),
// ping-ponged between two buffers per family; a union longer than `acc`
// raises a flag and the host reruns with a larger accumulator.  Results go to a
// [t][column] staging array; compact_kernel moves them into the output CSR once
// the counts are scanned (two-phase allocation without recomputation).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "levels.cuh"

namespace dexel {

enum { OP_DILATE = 0, OP_ERODE = 1, OP_SHELL = 2 };

// merge the running union A (smem, stride T) with sorted list B (global, element t at
// B[t * bstride]; bstride < 0 walks a list stored in descending order) into O
template <int T>
__device__ __forceinline__ int p2_merge(const float2* A, int na, const float2* __restrict__ B, int nb,
                                        int64_t bstride, float2* O, int acc) {
  int ia = 0, ib = 0, no = 0;
  float cs = 0.f, ce = 0.f;
  bool have = false;
  float2 xa = na > 0 ? A[0] : make_float2(INFINITY, INFINITY);
  float2 xb = nb > 0 ? B[0] : make_float2(INFINITY, INFINITY);
  while (ia < na || ib < nb) {
    float2 x;
    if (ib >= nb || (ia < na && xa.x <= xb.x)) {
      x = xa;
      ++ia;
      if (ia < na) xa = A[ia * T];
    } else {
      x = xb;
      ++ib;
      if (ib < nb) xb = B[(int64_t)ib * bstride];
    }
    if (!have) {
      cs = x.x; ce = x.y; have = true;
    } else if (x.x <= ce) {
      ce = fmaxf(ce, x.y);
    } else {
      if (no < acc) O[no * T] = make_float2(cs, ce);
      ++no;
      cs = x.x; ce = x.y;
    }
  }
  if (have) {
    if (no < acc) O[no * T] = make_float2(cs, ce);
    ++no;
  }
  return no;
}

// union over dy of one family's level lists for output column (i, jg): for each row
// offset, U_f(|dy|) (ascending) and U_r(|dy|) (stored descending) of column (i, jg+dy).
// Returns the count; *res = the buffer holding it (X or Y).
template <int T>
__device__ __forceinline__ int p2_family(const LevelSlots& L, int i, int jg, float2* X, float2* Y, int acc,
                                         float2** res, unsigned* need) {
  int na = 0;
  float2* cur = X;
  float2* nxt = Y;
  for (int t = 0; t <= 2 * L.R; ++t) {
    const int dy = (t & 1) ? ((t + 1) >> 1) : -(t >> 1);   // 0, 1, -1, 2, -2, ...
    const int jl = jg + dy - L.row0;
    if (jl < 0 || jl >= L.nrows) continue;
    const int k = dy < 0 ? -dy : dy;
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      const int nb = L.cnt[slot_cnt_index(L, jl, d, k, i)];
      if (nb == 0) continue;
      const float2* lb;
      int64_t stride;
      if (nb <= L.cap) {
        lb = L.z + slot_z_index(L, jl, d, k, d ? nb - 1 : 0, i);
        stride = d ? -(int64_t)L.nx : (int64_t)L.nx;
      } else {   // the column's lists live in the overflow arena
        const int q = L.ovf_idx[(size_t)jl * L.nx + i];
        lb = L.ovf_z + ovf_z_index(L, q, d, k, d ? nb - 1 : 0);
        stride = d ? -1 : 1;
      }
      const int n = p2_merge<T>(cur, na, lb, nb, stride, nxt, acc);
      if (n > acc) { *need = max(*need, (unsigned)n); na = acc; }
      else na = n;
      float2* tmp = cur; cur = nxt; nxt = tmp;
    }
  }
  *res = cur;
  return na;
}

// output rows [row0, row0 + nrows_out) (extended-row numbering of the level slots) of a band;
// output column c_local of the band is global output column cbase + c_local; the staging
// array is [t][ncol_total]
template <int OP, int T>
__global__ void __launch_bounds__(T) pass2s_kernel(LevelSlots A, LevelSlots B, int nx, int row0, int nrows_out,
                                                   int64_t cbase, int64_t ncol, float zlo, float zhi, int acc,
                                                   float2* __restrict__ ostage, uint32_t* __restrict__ ocnt,
                                                   unsigned* flags) {
  extern __shared__ __align__(16) float2 p2_smem[];
  const int tid = threadIdx.x;
  const int64_t cl = (int64_t)blockIdx.x * T + tid;
  if (cl >= (int64_t)nrows_out * nx) return;
  const int64_t c = cbase + cl;
  const int i = (int)(cl % nx), jg = row0 + (int)(cl / nx);
  float2* b0 = p2_smem + tid;
  float2* b1 = b0 + acc * T;
  float2* b2 = b1 + acc * T;
  unsigned need = 0;
  float2* ra;
  const int na = p2_family<T>(A, i, jg, b0, b1, acc, &ra, &need);
  uint32_t n = 0;
  if (OP == OP_DILATE) {
    for (int t = 0; t < na; ++t) ostage[(size_t)t * ncol + c] = ra[t * T];
    n = na;
  } else if (OP == OP_ERODE) {
    float cur = zlo;
    for (int t = 0; t < na; ++t) {
      const float2 v = ra[t * T];
      if (v.x > cur) ostage[(size_t)(n++) * ncol + c] = make_float2(cur, v.x);
      cur = v.y;
    }
    if (zhi > cur) ostage[(size_t)(n++) * ncol + c] = make_float2(cur, zhi);
  } else {
    // family B uses the two buffers not holding A's result
    float2* x = ra == b0 ? b1 : b0;
    float2* rb;
    const int nbb = p2_family<T>(B, i, jg, x, b2, acc, &rb, &need);
    int p = 0, q = 0;
    while (p < na && q < nbb) {
      const float2 u = ra[p * T], v = rb[q * T];
      const float lo = fmaxf(u.x, v.x), hi = fminf(u.y, v.y);
      if (lo < hi) ostage[(size_t)(n++) * ncol + c] = make_float2(lo, hi);
      if (u.y < v.y) ++p; else ++q;
    }
  }
  ocnt[c] = n;
  if (need) atomicMax(flags + 2, need);
}

inline size_t pass2_smem_bytes(int op, int acc, int T) {
  return (size_t)(op == OP_SHELL ? 3 : 2) * acc * T * sizeof(float2);
}
inline int pass2_stage_cap(int op, int acc) { return op == OP_SHELL ? 2 * acc : acc + 1; }

// CSR compaction: out[off[c] + t] = stage[t][c]
__global__ void compact_kernel(const float2* __restrict__ stage, const uint32_t* __restrict__ cnt,
                               const uint64_t* __restrict__ off, int64_t ncol, float2* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const uint32_t n = cnt[c];
  const uint64_t o = off[c];
  for (uint32_t t = 0; t < n; ++t) out[o + t] = stage[(size_t)t * ncol + c];
}

}  // namespace dexel
