// kernels.cuh -- common pieces of the sm_100a kernels of the separable dexel offset
// (arXiv 1804.08968): the upload check, the order-preserving keys, the rows an op reads
// (SrcRows: halo / slab / halo CSR segments), the pass-1 piece layout (PieceSlots) and the
// capsule-domination filter's thresholds.  Pass 1 is in pass1.cuh, the z-resolution in
// levels.cuh, pass 2 in pass2.cuh.
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

// offsets of a CSR slice -> offsets from 0 (dexel_pipe_run uploads row slabs of one host CSR)
__global__ void rebase_kernel(uint64_t* __restrict__ off, int64_t n, uint64_t base) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) off[c] -= base;
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

// the CSR row of extended row j: its offsets (column i at off[i]) and its segment's endpoints
// (selects, not a dynamic index into the parameter struct: that would copy it to local memory)
__device__ __forceinline__ void src_row(const SrcRows& s, int j, const uint64_t*& off, const float*& ep) {
  const bool s0 = j < s.rows[0], s2 = j >= s.rows[0] + s.rows[1];
  const int jj = s0 ? j : (s2 ? j - s.rows[0] - s.rows[1] : j - s.rows[0]);
  off = (s0 ? s.off[0] : (s2 ? s.off[2] : s.off[1])) + (size_t)jj * s.nx;
  ep = s0 ? s.ep[0] : (s2 ? s.ep[2] : s.ep[1]);
}

// Pass-1 output: the pieces of every column of a band of rows, in per-column slots of `cap`
// pieces (a multiple of 4) grouped in chunks of four: chunk q of column (row, i) holds pieces
// 4q .. 4q+3 as 32 contiguous bytes of (lo, hi) pairs, z[2 c], z[2 c + 1] with
// c = (row*NC + q)*nx + i, NC = cap/4 + 1, and their kappa bytes in the 32-bit word k[c]
// (piece 4q+u in byte u).  A lane writes whole chunks (full DRAM sectors); a warp of 32
// consecutive columns reads 1 KB contiguous per chunk.  Chunk NC-1 is a spill chunk: writes
// beyond cap are clamped there, the column is listed, and a second launch ("list mode") rewrites
// the listed columns' pieces into an arena of ovf_cap pieces (a multiple of 4) per column, with
// the same chunk layout at stride 1.
struct PieceSlots {
  float4* z;           // [nrows][NC][nx][2]  four (lo, hi) pairs per chunk
  uint32_t* k;         // [nrows][NC][nx]     four kappa bytes per chunk
  uint32_t* cnt;       // [nrows*nx]          true piece count
  int cap, nx, nrows;
  int32_t* ovf_idx;    // [nrows*nx] arena slot of an overflow column, -1 elsewhere
  float4* ovf_z;       // [n_ovf][ovf_cap/4][2]
  uint32_t* ovf_k;     // [n_ovf][ovf_cap/4]
  int ovf_cap;
  uint32_t* ovf_list;  // overflow columns (main pass appends)
  unsigned ovf_list_cap;
  uint32_t* tile_flag; // [nrows * ntiles] a tile holds an overflow column
  uint32_t* tile_list; // tiles to rerun in list mode
  unsigned* flags;     // [0] overflow columns, [2] tiles listed (device counters of this band/family)
  unsigned long long* total;   // pieces (statistics, the op's counter)
  unsigned* opf;       // the op's flag words (OpFlag): a column that does not fit asks for a rerun
  uint32_t one = 1;    // 1, opaque to the compiler (fsel: zero = one - 1, padd)
};

// The op's flag words: every capacity check of an op is deferred to ONE readback at its end
// (dexel.cu run_op_impl); a set rerun flag makes the host grow that capacity and rerun the op.
enum OpFlag {
  OPF_P1_RERUN = 0,    // a pass-1 column did not fit (slots + arena): grow the piece capacity
  OPF_P1_LONGEST = 1,  // its piece count
  OPF_LV_RERUN = 2,    // a level list did not fit (slots + arena): grow the level capacity
  OPF_LV_LONGEST = 3,
  OPF_P2_ACC = 4,      // a pass-2 union longer than the accumulator: its length
  OPF_OUT_FIT = 5,     // the output did not fit dst's buffer (compaction skipped)
  OPF_P2_PEAK = 6,     // the longest pass-2 union any column held during the op (sizes the next op's accumulator)
  OPF_WORDS = 16,      // (+ u64 statistics from word 8: n_mid, n_lev)
};

__host__ __device__ __forceinline__ size_t chunk_index(const PieceSlots& P, int row, int q, int i) {
  return ((size_t)row * (P.cap / 4 + 1) + q) * P.nx + i;
}

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
__device__ __forceinline__ bool dom_margin(float lhs, float rhs, float mabs) {
  return lhs <= rhs - 1e-6f * (1.0f + fabsf(rhs)) - mabs;
}

// Selects and conditional adds that issue on the FMA pipe.  The sweeps are ALU-pipe-bound (compares,
// min/max, bit ops and the selects ptxas makes of every ?: and predicated move all go to the ALU
// pipe, the FMA pipe idles at half the rate): a predicated multiply-add by a 0 / 1 the compiler
// cannot see through (derived from a kernel argument) is a move / add on the FMA pipe.
__device__ __forceinline__ uint32_t fsel(bool p, uint32_t a, uint32_t b, uint32_t zero) {   // p ? a : b
  // b = b * zero + a under p (zero: an opaque 0): the product involves b, so ptxas cannot share it
  // between two selects of the same value (it would compute a once and select on the ALU)
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t@q mad.lo.u32 %0, %0, %3, %2;\n\t}"
      : "+r"(b) : "r"((uint32_t)p), "r"(a), "r"(zero));
  return b;
}
__device__ __forceinline__ int fsel(bool p, int a, int b, uint32_t zero) {
  return (int)fsel(p, (uint32_t)a, (uint32_t)b, zero);
}
__device__ __forceinline__ float fsel(bool p, float a, float b, uint32_t zero) {
  return __uint_as_float(fsel(p, __float_as_uint(a), __float_as_uint(b), zero));
}
__device__ __forceinline__ uint32_t padd(bool p, uint32_t x, uint32_t d, uint32_t one) {   // p ? x + d : x
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t@q mad.lo.u32 %0, %2, %3, %0;\n\t}"
      : "+r"(x) : "r"((uint32_t)p), "r"(d), "r"(one));
  return x;
}

// shared-memory accesses through 32-bit shared addresses (computed once per kernel: a generic
// pointer into shared memory made nvcc rebuild the window address on every sweep step)
__device__ __forceinline__ uint32_t sh_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" :: "r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// capsule-domination thresholds of every (pending kappa, new kappa) pair (pass1.cuh, R <= 16)
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

}  // namespace dexel
