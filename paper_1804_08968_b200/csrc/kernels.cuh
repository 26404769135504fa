// kernels.cuh -- sm_100a kernels of the separable dexel offset (arXiv 1804.08968).
//
//   validate_kernel   upload check (strictly increasing, finite, in domain)
//   pass1_kernel      pass 1 along x: closest-parent extrusion S_In -> S_Mid
//                     (PAPER.md:494-501).  One warp per 32 output columns of a
//                     row; the warp sweeps z over the window's endpoints (merged
//                     across lanes with a REDUX min on order-preserving keys), keeps
//                     the active neighbour columns as a ballot bitmask and each lane
//                     reads its closest parent kappa = nearest set bit within R.
//   levels_kernel     the 1D half-space power diagram along z of a column's
//                     pieces (start anchors grow down, end anchors grow up, power
//                     weight W = r^2 - kappa^2 s^2; App. B) as
//                     an upper envelope F(z) = max_p [W_p - dist(z, piece_p)^2],
//                     and its superlevel sets L_k = {F >= k^2 s^2}, k = 0..R.
//                     L_k(i,j') is the 2D dilation of row j' by sqrt(r^2-k^2 s^2).
//   pass2_kernel      pass 2 along y: out(i,j) = U_{|dy|<=R} L_|dy|(i, j+dy)
//                     (a row at lateral distance dy contributes where F >= dy^2,
//                     i.e. power weight r^2 - kappa^2 - dy^2 >= 0), clipped to U,
//                     with the dilate / erode / shell epilogue.
// Every kernel runs twice (two-phase allocation): COUNT writes per-column
// counts, WRITE recomputes and writes at the scanned offsets.
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

// One warp = output columns [32*tile, 32*tile+32) of output row jr (source row j = row0 + jr).
// NW = number of 32-bit words of the window mask (window = 32 + 2R columns).
template <int NW, bool WRITE>
__global__ void __launch_bounds__(128) pass1_kernel(SrcRows src, int R, int complement, int row0, int nrows_out,
                                                    uint32_t* __restrict__ cnt, const uint64_t* __restrict__ moff,
                                                    float2* __restrict__ mz, uint8_t* __restrict__ mk) {
  const int lane = threadIdx.x & 31;
  const int ntiles = (src.nx + 31) >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= (int64_t)nrows_out * ntiles) return;  // warp-uniform
  const int jr = (int)(gw / ntiles), tile = (int)(gw % ntiles);
  const int j = row0 + jr;
  const int i0 = tile * 32;
  const int W = 32 + 2 * R;

  ColCursor cur[NW];
  uint32_t nkey[NW];
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    const int w = lane + 32 * q;
    if (w < W) col_open(src, i0 - R + w, j, complement, cur[q]);
    else { cur[q].base = 0; cur[q].n = 0; cur[q].v = 0; cur[q].vend = 0; }
    nkey[q] = cur[q].v < cur[q].vend ? fkey(col_value(src, cur[q], cur[q].v, complement)) : KEY_NONE;
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
        const bool is_start = (cur[q].v & 1u) == 0u;
        act = is_start ? (act | (1u << q)) : (act & ~(1u << q));
        cur[q].v++;
        nkey[q] = cur[q].v < cur[q].vend ? fkey(col_value(src, cur[q], cur[q].v, complement)) : KEY_NONE;
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
struct LevelTables {
  const double* Wp;    // [R+1]   W(kappa) = r^2 - kappa^2 s^2
  const double* T;     // [R+1]   T(k) = k^2 s^2
  const float* h;      // [(R+1)^2] fl32(sqrt(r^2 - (kappa^2+k^2) s^2)), -1 where negative
  int R;
  double inv_s2;
};

__device__ __forceinline__ int level_of(const LevelTables& L, double v) {
  if (!(v >= 0.0)) return -1;
  int k = (int)sqrt(v * L.inv_s2);
  if (k > L.R) k = L.R;
  while (k < L.R && __ldg(L.T + k + 1) <= v) ++k;
  while (k >= 0 && __ldg(L.T + k) > v) --k;
  return k;
}

__device__ __forceinline__ double gfun(double z, double lo, double hi, double W) {
  double d = lo - z > 0.0 ? lo - z : (z - hi > 0.0 ? z - hi : 0.0);
  return W - d * d;
}

// crossing of g_p and g_q for p below q (g_p - g_q strictly decreasing)
__device__ double crossing(double lp, double hp, double Wp, double lq, double hq, double Wq) {
  auto D = [&](double z) { return gfun(z, lp, hp, Wp) - gfun(z, lq, hq, Wq); };
  double z;
  if (D(lp) <= 0.0) {
    z = 0.5 * (lq + lp) + (Wp - Wq) / (2.0 * (lq - lp));
    z = fmin(z, lp);
  } else if (D(hp) <= 0.0) {
    double t = Wq - Wp;
    z = lq - sqrt(t > 0.0 ? t : 0.0);
    z = fmax(lp, fmin(z, hp));
  } else if (D(lq) <= 0.0) {
    z = 0.5 * (lq + hp) + (Wp - Wq) / (2.0 * (lq - hp));
    z = fmax(hp, fmin(z, lq));
  } else if (D(hq) <= 0.0) {
    double t = Wp - Wq;
    z = hp + sqrt(t > 0.0 ? t : 0.0);
    z = fmax(lq, fmin(z, hq));
  } else {
    z = 0.5 * (hp + hq) + (Wp - Wq) / (2.0 * (hq - hp));
    z = fmax(z, hq);
  }
  return z;
}

template <int MAXL>
struct LevelState {
  float open_lo[MAXL];
  float pend_lo[MAXL], pend_hi[MAXL];
  uint32_t ncnt[MAXL];
  uint32_t pend_mask_dummy;
};

template <int MAXL, bool WRITE>
struct LevelEmitter {
  LevelState<MAXL>& st;
  int lam;           // current level of the open segment (-1 = outside)
  float zlast;
  float zlo, zhi;
  int64_t c, ncol;
  const uint64_t* loff;
  float2* lz;
  uint64_t pend_bits[(MAXL + 63) / 64];

  __device__ void flush(int k) {
    uint64_t& b = pend_bits[k >> 6];
    const uint64_t bit = 1ull << (k & 63);
    if (!(b & bit)) return;
    b &= ~bit;
    float lo = fmaxf(st.pend_lo[k], zlo), hi = fminf(st.pend_hi[k], zhi);
    if (lo < hi) {
      if (WRITE) lz[loff[(int64_t)k * ncol + c] + st.ncnt[k]] = make_float2(lo, hi);
      st.ncnt[k]++;
    }
  }
  __device__ void rise(int k, float z) {  // level k becomes covered at z
    uint64_t& b = pend_bits[k >> 6];
    const uint64_t bit = 1ull << (k & 63);
    if ((b & bit) && st.pend_hi[k] >= z) {  // zero-length gap: merge (closed sets)
      b &= ~bit;
      st.open_lo[k] = st.pend_lo[k];
    } else {
      flush(k);
      st.open_lo[k] = z;
    }
  }
  __device__ void fall(int k, float z) {  // level k stops being covered at z
    flush(k);
    st.pend_lo[k] = st.open_lo[k];
    st.pend_hi[k] = z;
    pend_bits[k >> 6] |= 1ull << (k & 63);
  }
  __device__ float mono(float z) { z = fmaxf(z, zlast); zlast = z; return z; }
  __device__ void set_at(float z, int target) {  // jump to level target at z
    z = mono(z);
    while (lam < target) rise(++lam, z);
    while (lam > target) fall(lam--, z);
  }
};

// One thread per column: envelope stack over the column's pieces, then a walk
// of the envelope emitting the superlevel sets L_k, k = 0..R (clipped to U).
template <int MAXL, bool WRITE>
__global__ void __launch_bounds__(128) levels_kernel(int64_t ncol, const uint64_t* __restrict__ moff,
                                                     const float2* __restrict__ mz, const uint8_t* __restrict__ mk,
                                                     uint32_t* __restrict__ stk_p, double* __restrict__ stk_z,
                                                     LevelTables L, float zlo, float zhi,
                                                     uint32_t* __restrict__ lcnt, const uint64_t* __restrict__ loff,
                                                     float2* __restrict__ lz) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const int R = L.R;
  const uint64_t base = moff[c];
  const uint32_t m = (uint32_t)(moff[c + 1] - base);
  LevelState<MAXL> st;
  for (int k = 0; k <= R; ++k) st.ncnt[k] = 0;
  if (m > 0) {
    // ---- upper envelope of g_p (pieces sorted by z, single crossing per pair)
    int top = -1;
    for (uint32_t q = 0; q < m; ++q) {
      const float2 pq = mz[base + q];
      const double Wq = __ldg(L.Wp + mk[base + q]);
      double s = -INFINITY;
      while (top >= 0) {
        const uint32_t p = stk_p[base + top];
        const float2 pp = mz[base + p];
        const double z = crossing(pp.x, pp.y, __ldg(L.Wp + mk[base + p]), pq.x, pq.y, Wq);
        if (z <= stk_z[base + top]) {
          --top;
        } else {
          s = z;
          break;
        }
      }
      ++top;
      stk_p[base + top] = q;
      stk_z[base + top] = top == 0 ? -INFINITY : s;
    }
    // ---- walk the envelope: level crossings at the owner's candidates a -/+ h(kappa,k)
    LevelEmitter<MAXL, WRITE> E{st, -1, -INFINITY, zlo, zhi, c, ncol, loff, lz};
    for (int t = 0; t < (MAXL + 63) / 64; ++t) E.pend_bits[t] = 0;
    for (int s = 0; s <= top; ++s) {
      const uint32_t p = stk_p[base + s];
      const float2 pp = mz[base + p];
      const int kp = mk[base + p];
      const double W = __ldg(L.Wp + kp);
      const float* hrow = L.h + (size_t)kp * (R + 1);
      const double zs = stk_z[base + s];
      const double ze = s < top ? stk_z[base + s + 1] : INFINITY;
      const double lo = pp.x, hi = pp.y;
      // (a) down-arc: increasing on [zs, min(ze, lo)]
      if (zs < lo) {
        const double z1 = fmin(ze, lo);
        const int t1 = z1 >= lo ? level_of(L, W) : level_of(L, gfun(z1, lo, hi, W));
        if (t1 < E.lam) {
          E.set_at((float)zs, t1);
        } else {
          while (E.lam < t1) {
            const int k = E.lam + 1;
            double zc = (double)(pp.x - __ldg(hrow + k));
            zc = fmax(zs, fmin(zc, z1));
            E.set_at((float)zc, k);
          }
        }
      }
      // (b) plateau on [max(zs,lo), min(ze,hi)]
      if (zs < hi && ze > lo) {
        const int tp = level_of(L, W);
        if (tp != E.lam) E.set_at((float)fmax(zs, lo), tp);
      }
      // (c) up-arc: decreasing on [max(zs,hi), ze]
      if (ze > hi) {
        const double z0 = fmax(zs, hi);
        const int t1 = ze == INFINITY ? -1 : level_of(L, gfun(ze, lo, hi, W));
        if (t1 > E.lam) {
          E.set_at((float)z0, t1);
        } else {
          const int kmax = level_of(L, W);
          while (E.lam > t1) {
            const int k = E.lam;
            double zc = k <= kmax ? (double)(pp.y + __ldg(hrow + k)) : z0;
            zc = fmax(z0, fmin(zc, ze));
            E.set_at((float)zc, k - 1);
          }
        }
      }
    }
    for (int k = 0; k <= R; ++k) E.flush(k);
  }
  if (!WRITE)
    for (int k = 0; k <= R; ++k) lcnt[(int64_t)k * ncol + c] = st.ncnt[k];
}

// ------------------------------------------------------------------ levels (lanes = levels)
// Same result as levels_kernel, organised for SIMT throughput: a warp owns G
// columns (G = 32 / (R+1) for R < 32, else 1) and lane (g, k) builds the
// superlevel set L_k of column g directly as the union of the grown pieces
//   L_k = U_{p : kappa_p^2 + k^2 <= (r/s)^2} [lo_p - h(kappa_p,k), hi_p + h(kappa_p,k)]
// (capsule of PAPER.md:538-541 restricted to the row at lateral distance k).
// Pieces are read coalesced, L lanes at a time, and broadcast with shuffles;
// each lane keeps a small deque of not-yet-final union intervals in shared
// memory: an interval whose end is below lo - h(0,k) can no longer grow
// (every later piece starts at >= lo and grows by <= h(0,k)), so it is emitted.
constexpr int LV_D = 16;   // deque depth per lane and level slot

template <int NS>
struct LvCfg {
  static constexpr int WARPS = NS <= 2 ? 4 : (NS == 4 ? 2 : 1);
};

template <int NS, bool WRITE>
__global__ void __launch_bounds__(LvCfg<NS>::WARPS * 32) levels2_kernel(
    int64_t ncol, const uint64_t* __restrict__ moff, const float2* __restrict__ mz, const uint8_t* __restrict__ mk,
    const float* __restrict__ htab, int R, int h_in_smem, float zlo, float zhi, uint32_t* __restrict__ lcnt,
    const uint64_t* __restrict__ loff, float2* __restrict__ lz, int* __restrict__ overflow) {
  constexpr int WARPS = LvCfg<NS>::WARPS;
  extern __shared__ float4 lv_smem4[];
  float2* dq_all = reinterpret_cast<float2*>(lv_smem4);                 // [WARPS][NS][LV_D][32]
  float* hs = reinterpret_cast<float*>(dq_all + WARPS * NS * LV_D * 32);  // [(R+1)^2] if h_in_smem
  const int L = R + 1;
  if (h_in_smem) {
    for (int t = threadIdx.x; t < L * L; t += blockDim.x) hs[t] = htab[t];
    __syncthreads();
  }
  const float* H = h_in_smem ? hs : htab;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int G = NS == 1 ? 32 / L : 1;           // columns per warp (L <= 32 when NS == 1)
  const int LC = NS == 1 ? L : 32;              // lanes per column group
  const int g = lane / LC, u0 = lane % LC;
  const bool lane_ok = g < G;
  const int64_t c = ((int64_t)blockIdx.x * WARPS + wib) * G + g;
  const bool col_ok = lane_ok && c < ncol;
  float2* dq = dq_all + (size_t)wib * NS * LV_D * 32;

  uint64_t base = 0;
  uint32_t m = 0;
  if (col_ok) { base = moff[c]; m = (uint32_t)(moff[c + 1] - base); }
  int kk[NS], b[NS], n[NS];
  uint32_t cnt[NS];
  float Hk[NS];
  uint64_t obase[NS];
  bool ovf = false;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    kk[s] = u0 + 32 * s;
    b[s] = 0; n[s] = 0; cnt[s] = 0; obase[s] = 0;
    const bool v = col_ok && kk[s] <= R;
    Hk[s] = v ? H[kk[s]] : 0.f;                  // h(0,k): the largest growth at level k
    if (WRITE && v) obase[s] = loff[(int64_t)kk[s] * ncol + c];
  }
  auto emit = [&](int s, float2 iv) {
    const float lo = fmaxf(iv.x, zlo), hi = fminf(iv.y, zhi);
    if (lo < hi) {
      if (WRITE) lz[obase[s] + cnt[s]] = make_float2(lo, hi);
      ++cnt[s];
    }
  };
  const uint32_t mmax = __reduce_max_sync(FULL, m);
  for (uint32_t t0 = 0; t0 < mmax; t0 += LC) {
    float2 pz = make_float2(0.f, 0.f);
    int pk = 0;
    if (t0 + u0 < m) { pz = mz[base + t0 + u0]; pk = mk[base + t0 + u0]; }
    const int nu = min((uint32_t)LC, mmax - t0);
    for (int u = 0; u < nu; ++u) {
      const int srcl = g * LC + u;
      const float lo = __shfl_sync(FULL, pz.x, srcl);
      const float hi = __shfl_sync(FULL, pz.y, srcl);
      const int kap = __shfl_sync(FULL, pk, srcl);
      if (t0 + u >= m) continue;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        if (kk[s] > R) continue;
        float2* q = dq + (size_t)s * LV_D * 32 + lane;   // q[d*32]
        const float lim = lo - Hk[s];
        while (n[s] > 0 && q[b[s] * 32].y < lim) {      // final: cannot be reached by later pieces
          emit(s, q[b[s] * 32]);
          b[s] = (b[s] + 1) & (LV_D - 1);
          --n[s];
        }
        const float hv = H[kap * L + kk[s]];
        if (hv >= 0.f) {
          float s0 = lo - hv, e0 = hi + hv;
          while (n[s] > 0) {
            const int top = (b[s] + n[s] - 1) & (LV_D - 1);
            const float2 tv = q[top * 32];
            if (tv.y < s0) break;
            s0 = fminf(s0, tv.x);
            e0 = fmaxf(e0, tv.y);
            --n[s];
          }
          if (n[s] == LV_D) {
            ovf = true;
          } else {
            q[((b[s] + n[s]) & (LV_D - 1)) * 32] = make_float2(s0, e0);
            ++n[s];
          }
        }
      }
    }
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (!col_ok || kk[s] > R) continue;
    float2* q = dq + (size_t)s * LV_D * 32 + lane;
    while (n[s] > 0) {
      emit(s, q[b[s] * 32]);
      b[s] = (b[s] + 1) & (LV_D - 1);
      --n[s];
    }
    if (!WRITE) lcnt[(int64_t)kk[s] * ncol + c] = cnt[s];
  }
  if (ovf) atomicExch(overflow, 1);
}

// ------------------------------------------------------------------ pass 2
struct LevelFamily {
  const uint64_t* loff;  // [(R+1)*ncol + 1], level-major
  const float2* lz;
  int R;
  int64_t ncol;          // columns per level (rows_L * nx)
  int row0;              // global row of level row 0
  int nrows;             // rows available
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
    const int64_t idx = (int64_t)k * F.ncol + (int64_t)jl * nx + i;
    const uint64_t s0 = F.loff[idx], s1 = F.loff[idx + 1];
    if (s1 == s0) continue;
    int n = merge_union(cur, na, F.lz + s0, (int)(s1 - s0), nxt, ACC_CAP);
    if (n > ACC_CAP) { *ovf = true; n = ACC_CAP; }
    float2* tmp = cur; cur = nxt; nxt = tmp;
    na = n;
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
