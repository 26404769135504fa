// pass1.cuh -- pass 1 along x: the closest-parent extrusion S_In -> S_Mid.
//
// For output column (i, j) and every z, kappa(z) = min { |dx| <= R : z in S(i+dx, j) } (the
// "closest parent"; "keep the largest radius"); the output is the sequence of
// maximal closed runs of constant kappa, the pieces (lo, hi, kappa).  Pure selection: lo / hi
// are copies of input values and kappa is an integer, so the pieces are bitwise the oracle's P1.
//
// Two kernels, picked per R by measurement:
//
//  * p1g_kernel (R <= P1G_RMAX, "gather"): one thread per output column merges the 2R+1 sorted
//    endpoint lists of its own neighbour columns (a lane's window is tiny, so the merge is a few
//    compares per event; a warp-wide sweep would walk the 32 + 2R columns' events for each).
//
//  * p1s_kernel (larger R, "warp sweep"): one warp per 32 output columns of a row.  The window's
//    32 + 2R columns are staged in shared memory (one coalesced copy of the window's contiguous
//    CSR range, as order-preserving u32 keys); each step takes the window's next z with one REDUX
//    min, toggles the activity mask with one ballot per 32 columns, and every lane reads its
//    closest parent as the nearest set bit within R of its position.
//
// Shell: both families (S at r_out, C = U \ S at r_in, same R) come from one sweep -- C's active
// set is G & ~M (G = in-grid window columns), its first piece starts at z_lo and its last closes
// at z_hi, zero-length C pieces are dropped as complement-on-load drops them.  Erosion runs the C
// family alone.
//
// Output: the chunked piece layout of kernels.cuh (PieceSlots): a lane's consecutive pieces fill
// whole 32-byte sectors.  Capsule domination (kernels.cuh) filters the pieces before they are
// stored.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace dexel {

#ifndef P1_WARPS_N
#define P1_WARPS_N 4
#endif
constexpr int P1_WARPS = P1_WARPS_N;
constexpr int P1_STAGE = 2048;   // staged window keys per warp (larger windows read through L1)
constexpr int P1G_RMAX = 4;      // gather kernel up to this R (measured)
constexpr int P1G_T = 128;       // gather kernel block

// ------------------------------------------------------------------ per-family output state
// A lane's pieces of one family: the pending piece of the domination filter, then a 4-piece
// register buffer flushed as one chunk.
struct PFam {
  float zstart;       // start of the open run
  int kap;            // its kappa (knone: no parent within R)
  int knone;          // "no parent" (KNONE, or R + 1 in the two-word warp sweep)
  float plo, phi;     // pending (closed, filtered-later) piece
  int pk;
  uint32_t trow;      // shared address of the threshold-table row of pk (row 17: no pending piece)
  float hpk;          // H[pk] (computed-threshold mode, R > 16)
  uint32_t np;        // pieces stored
  float2* zb;         // piece 0 of this column (chunk 0)
  uint8_t* kb;
  uint32_t woff;      // offset (pieces) of the next store from zb / kb
  uint32_t cs;        // chunk stride in pieces: 4 nx (slots), 4 (arena), 0 (no output)
  uint32_t wlim;      // offset of the spill chunk: stores stay there once reached
  bool has_out;
  uint32_t one, zero; // P.one, P.one - 1 (padd, fsel)
};

// predicated store of one piece without a branch: the (lo, hi) pair and its kappa byte
__device__ __forceinline__ void st_pred_piece(float2* zp, uint8_t* kp, float lo, float hi, int k, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.global.v2.f32 [%0], {%2, %3};\n\t"
               "@q st.global.u8 [%1], %4;\n\t}"
               :: "l"(zp), "l"(kp), "f"(lo), "f"(hi), "r"(k), "r"((int)pred));
}

// out_kind: 0 = slots of column i of band row jr, 1 = arena slot `aslot`, 2 = no output (spill)
__device__ __forceinline__ void pfam_init(PFam& F, const PieceSlots& P, int jr, int i, int out_kind, int aslot,
                                          uint32_t thr, int knone = KNONE) {
  const uint32_t nc = (uint32_t)(P.cap / 4);   // chunks per column (+1: the spill chunk)
  if (out_kind == 0) {
    F.zb = reinterpret_cast<float2*>(P.z + 2 * chunk_index(P, jr, 0, i));
    F.kb = reinterpret_cast<uint8_t*>(P.k + chunk_index(P, jr, 0, i));
    F.cs = 4u * (uint32_t)P.nx;
    F.wlim = nc * F.cs;
  } else if (out_kind == 1) {
    const size_t oc = (size_t)(P.ovf_cap / 4);
    F.zb = reinterpret_cast<float2*>(P.ovf_z + 2 * (size_t)aslot * oc);
    F.kb = reinterpret_cast<uint8_t*>(P.ovf_k + (size_t)aslot * oc);
    F.cs = 4u;
    F.wlim = 4u * (uint32_t)oc;   // (arena columns hold at most ovf_cap pieces: no spill)
  } else {   // the spill chunk of column 0 of this row (never read)
    F.zb = reinterpret_cast<float2*>(P.z + 2 * chunk_index(P, jr, (int)nc, 0));
    F.kb = reinterpret_cast<uint8_t*>(P.k + chunk_index(P, jr, (int)nc, 0));
    F.cs = 0u;
    F.wlim = 0u;
  }
  // opaque per-lane base pointers (no per-store 64-bit index arithmetic from the kernel params)
  asm("mov.b64 %0, %0;" : "+l"(F.zb));
  asm("mov.b64 %0, %0;" : "+l"(F.kb));
  F.has_out = out_kind != 2;
  F.one = P.one;
  F.zero = P.one - 1u;
  F.np = 0;
  F.woff = 0;
  F.plo = F.phi = 0.f;
  F.knone = knone;
  F.pk = knone;
  F.trow = thr + 17u * 32u * 8u;
  F.hpk = 0.f;
  F.zstart = 0.f;
  F.kap = knone;
}

// append one piece (predicated): piece t goes to slot t % 4 of chunk t / 4 (clamped to the spill
// chunk).  A lane's consecutive pieces fill one 32-byte sector (and one 4-byte kappa word) within a
// few steps, so L2 sees whole sectors written (the old slot-major layout put every piece of a lane
// in another sector, shared with other lanes' pieces written at other times: DRAM read-fills).
__device__ __forceinline__ void pfam_put(PFam& F, float lo, float hi, int k, bool wr) {
  st_pred_piece(F.zb + F.woff, F.kb + F.woff, lo, hi, k, wr);
  F.np = padd(wr, F.np, 1u, F.one);
  // the next slot of the chunk, or slot 0 of the next chunk (a running offset: no index arithmetic)
  const uint32_t step = fsel((F.np & 3u) != 0u, 1u, F.cs - 3u, F.zero);
  F.woff = padd(wr && F.woff < F.wlim, F.woff, step, F.one);
}

// a piece [zs, z] at level kap closes (closed == true): the capsule-domination filter against
// the pending piece (table mode: thresholds from the (kp, kn) table; else from H = prune), then
// the pending piece is stored unless dominated, and the new one becomes pending unless dominated
template <bool TABLE, bool PRUNE>
__device__ __forceinline__ void pfam_close(PFam& F, bool closed, float zs, float z, int kap, uint32_t thr,
                                           const float* h0, float mabs) {
  if constexpr (!PRUNE) {
    pfam_put(F, zs, z, kap, closed);
    return;
  }
  bool drop_new, drop_pend;
  const bool hp = F.pk != F.knone;
  if constexpr (TABLE) {
    const float2 th = lds_f2(F.trow + 8u * (uint32_t)(kap & 31));
    drop_new = z - F.phi <= th.x;
    drop_pend = zs - F.plo <= th.y;
  } else {
    const float D = F.hpk - h0[kap & 255];                      // H[kp] - H[kn]
    drop_new = hp && F.pk <= kap && dom_margin(z - F.phi, D, mabs);
    drop_pend = kap <= F.pk && dom_margin(zs - F.plo, -D, mabs);
  }
  pfam_put(F, F.plo, F.phi, F.pk, closed && hp && !drop_new && !drop_pend);
  const bool take = closed && !drop_new;
  F.plo = fsel(take, zs, F.plo, F.zero);
  F.phi = fsel(take, z, F.phi, F.zero);
  if constexpr (TABLE) F.trow = fsel(take, thr + 256u * (uint32_t)(kap & 31), F.trow, F.zero);
  else F.hpk = take ? h0[kap & 255] : F.hpk;
  F.pk = fsel(take, kap, F.pk, F.zero);
}

// flush the pending piece; store the count; list an overflowing column (or ask for a rerun)
__device__ __forceinline__ void pfam_finish(PFam& F, const PieceSlots& P, int64_t c, int jr, int tile, int ntiles,
                                            bool list_mode) {
  pfam_put(F, F.plo, F.phi, F.pk, F.has_out && F.pk != F.knone);
  if (!list_mode) {
    if (F.has_out) {
      P.cnt[c] = F.np;
      if (F.np > (uint32_t)P.cap) {                    // hand the column to list mode
        const unsigned slot = atomicAdd(P.flags, 1u);
        if (slot >= P.ovf_list_cap || F.np > (uint32_t)P.ovf_cap) {   // does not fit: rerun the op
          atomicOr(P.opf + OPF_P1_RERUN, 1u);
          atomicMax(P.opf + OPF_P1_LONGEST, F.np);
        } else {
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
  } else if (F.has_out) {
    P.cnt[c] = F.np;                                   // the filtered count of an arena column
    atomicAdd(P.total, (unsigned long long)F.np);
  }
}

// ------------------------------------------------------------------ window bit helpers
// nearest set bit of a window mask to position p, within R (KNONE if none)
template <int NW>
__device__ __forceinline__ int nearest_bit(const uint32_t (&M)[NW], int p, int R) {
  if constexpr (NW == 2) {
    const unsigned long long m = ((unsigned long long)M[1] << 32) | M[0];
    const unsigned long long left = m & ((2ull << p) - 1ull);          // positions <= p (p <= 62)
    const unsigned long long right = m >> p;                            // positions >= p
    const int dl = left ? p - (63 - __clzll(left)) : KNONE;
    const int dr = right ? __ffsll(right) - 1 : KNONE;
    const int d = min(dl, dr);
    return d <= R ? d : KNONE;
  } else {
    int best = KNONE;
#pragma unroll
    for (int t = 0; t < NW; ++t) {
      const uint32_t w = M[t];
      const int b0 = 32 * t;
      const int sh = p - b0;
      if (sh >= 0) {  // bits at positions <= p
        const uint32_t m = sh >= 31 ? w : (w & ((2u << sh) - 1u));
        if (m) best = min(best, p - (b0 + 31 - __clz(m)));
      }
      if (sh <= 31) {  // bits at positions >= p
        const uint32_t m = sh <= 0 ? w : (w & ~((1u << sh) - 1u));
        if (m) best = min(best, b0 + __ffs(m) - 1 - p);
      }
    }
    return best <= R ? best : KNONE;
  }
}

// ------------------------------------------------------------------ common per-warp setup
// the output tile of one warp and the CSR row it reads
struct P1Tile {
  int jr, tile, j, i0;
  const uint64_t* off;   // the row's offsets (column i at off[i])
  const float* ep;       // the segment's endpoints
};

__device__ __forceinline__ P1Tile p1_tile(const SrcRows& src, int row0, int64_t tl, int ntiles) {
  P1Tile t;
  t.jr = (int)(tl / ntiles);
  t.tile = (int)(tl % ntiles);
  t.j = row0 + t.jr;
  t.i0 = t.tile * 32;
  src_row(src, t.j, t.off, t.ep);
  return t;
}

// ------------------------------------------------------------------ warp sweep (larger R)
// One warp per 32 output columns of a row: the window's keys are staged in shared memory (one
// coalesced copy of its contiguous CSR range); each step takes the next z of the whole window
// with one REDUX min, toggles the window's activity mask with one ballot per word, and every
// lane reads its closest parent as the nearest set bit within R of its own position (C: of
// G & ~M).  A step where no lane's kappa changes skips the family's filter / emission half
// (SKIP, a warp vote: pays from R = 8).  (A batched variant -- window events recorded in shared
// memory, per-lane emission only at the events that can change the lane's column -- walked fewer
// emission steps but measured 1.2-1.5x slower at R >= 8: DESIGN.md "What was tried".)
// SKIP: 0 = none, 1 = a warp vote per family and step (one vote for both families measured slower)
template <int NW, int FAMS, bool TABLE, int SKIP>
__global__ void __launch_bounds__(P1_WARPS * 32) p1s_kernel(SrcRows src, int R, int row0, int jr0, int nrows_out,
                                                             PieceSlots PS, PieceSlots PC, int64_t nlist,
                                                             const float* __restrict__ prune_s,
                                                             const float* __restrict__ prune_c) {
  extern __shared__ __align__(16) uint32_t p1_smem[];
  constexpr bool FS_ON = (FAMS & 1) != 0, FC_ON = (FAMS & 2) != 0;
  __shared__ float2 thr_s[TABLE && FS_ON ? 18 * 32 : 1], thr_c[TABLE && FC_ON ? 18 * 32 : 1];
  __shared__ float h0s[!TABLE && FS_ON ? 256 : 1], h0c[!TABLE && FC_ON ? 256 : 1];
  const bool prune = FS_ON ? prune_s != nullptr : prune_c != nullptr;
  float mabs_s = 0.f, mabs_c = 0.f;
  if (FS_ON && prune_s) {
    if constexpr (TABLE) p1_thr_init(thr_s, prune_s, R);
    else for (int t = threadIdx.x; t <= R; t += blockDim.x) h0s[t] = prune_s[t];
    mabs_s = prune_s[R + 1];
  }
  if (FC_ON && prune_c) {
    if constexpr (TABLE) p1_thr_init(thr_c, prune_c, R);
    else for (int t = threadIdx.x; t <= R; t += blockDim.x) h0c[t] = prune_c[t];
    mabs_c = prune_c[R + 1];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t one = FS_ON ? PS.one : PC.one;
  uint32_t* stage = p1_smem + (size_t)wid * (P1_STAGE + 4);
  const uint32_t stage_a = sh_addr(stage);
  const uint32_t ths = sh_addr(thr_s), thc = sh_addr(thr_c);
  const int ntiles = (src.nx + 31) >> 5;
  const bool list_mode = nlist >= 0;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t* tile_list = FS_ON ? PS.tile_list : PC.tile_list;
  const int32_t* ovf_idx = FS_ON ? PS.ovf_idx : PC.ovf_idx;
  // one warp's work: the output tile tl (row jr = tl / ntiles of the band, 32 columns)
  auto process = [&](int64_t tl) {
  __syncwarp();   // (the previous tile's reads of stage[] are done)
  const P1Tile T = p1_tile(src, row0, tl, ntiles);
  const int W = 32 + 2 * R;
  // ---- stage the window's keys: column p's list at sb[p] .. sb[p] + n - 1, then a KEY_NONE
  // sentinel (the sweep's advance needs no bound check); each lane copies its own columns with
  // 8-byte loads (a column's intervals are contiguous; the window's lanes stream one contiguous
  // CSR range between them)
  const float* ep = T.ep;
  uint32_t pos[NW], end[NW], nkey[NW], G[NW], M[NW], sb[NW];
  uint64_t cb0[NW];
  uint32_t total = 0;
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    const int p = lane + 32 * q, gi = T.i0 - R + p;
    const bool in = p < W && gi >= 0 && gi < src.nx;
    G[q] = __ballot_sync(FULL, in);
    const uint64_t a = in ? __ldg(T.off + gi) : 0ull, b = in ? __ldg(T.off + gi + 1) : 0ull;
    cb0[q] = a;
    const uint32_t nv = (uint32_t)(2 * (b - a)) + 1u;          // + the sentinel
    uint32_t incl = nv;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, d);
      if (lane >= d) incl += y;
    }
    sb[q] = total + incl - nv;
    total += __shfl_sync(FULL, incl, 31);
    pos[q] = 0u;
    end[q] = nv - 1u;
    M[q] = 0u;
  }
  const bool staged = total <= (uint32_t)P1_STAGE;
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    if (staged) {
      const float2* src2 = reinterpret_cast<const float2*>(ep) + cb0[q];
      for (uint32_t t = 0; t < end[q]; t += 2) {
        const float2 v = __ldg(src2 + (t >> 1));
        sts_u32(stage_a + 4u * (sb[q] + t), fkey(v.x));
        sts_u32(stage_a + 4u * (sb[q] + t + 1), fkey(v.y));
      }
      sts_u32(stage_a + 4u * (sb[q] + end[q]), KEY_NONE);
      pos[q] = stage_a + 4u * sb[q];             // staged: pos is the key's shared address
      end[q] = stage_a + 4u * (sb[q] + end[q]);
    }
  }
  __syncwarp();
  // unstaged windows (more keys than the staging area) read through L1: key t of column q at
  // ep[2 cb0[q] + t]
#pragma unroll
  for (int q = 0; q < NW; ++q)
    nkey[q] = pos[q] < end[q] ? (staged ? lds_u32(pos[q]) : fkey(__ldg(ep + 2 * cb0[q] + pos[q]))) : KEY_NONE;
  // ---- this lane's output column and its families
  const int knone = NW == 2 ? R + 1 : KNONE;
  const int i = T.i0 + lane;
  const bool out_ok = i < src.nx;
  const int64_t c = (int64_t)T.jr * src.nx + i;
  PFam FS, FC;
  {
    int kind = out_ok ? 0 : 2, aslot = 0;
    if (list_mode) {
      aslot = out_ok ? ovf_idx[c] : -1;
      kind = aslot >= 0 ? 1 : 2;
    }
    if (FS_ON) pfam_init(FS, PS, T.jr, out_ok ? i : 0, kind, aslot, ths, knone);
    if (FC_ON) pfam_init(FC, PC, T.jr, out_ok ? i : 0, kind, aslot, thc, knone);
  }
  const int pp = lane + R;
  // NW == 2: this lane's two 32-bit windows of the 64-bit mask, bits pp .. pp+31 (right) and
  // pp-31 .. pp with bit pp on top (left), one 64-bit funnel shift each (SHF.R.U64 /
  // SHF.L.U64.HI take shift amounts up to 63)
  const uint32_t shl = (uint32_t)(63 - pp);
  auto win_r = [&](uint32_t m0, uint32_t m1) {
    return (uint32_t)((((unsigned long long)m1 << 32) | m0) >> pp);
  };
  auto win_l = [&](uint32_t m0, uint32_t m1) {
    return (uint32_t)(((((unsigned long long)m1 << 32) | m0) << shl) >> 32);
  };
  // (NW == 2) nearest set bit within R of a lane's two windows: the windows are masked to
  // distances <= R and carry a sentinel bit at distance R + 1, so the distance is R + 1 (= knone,
  // "no parent") without a range test: one 3-input LOP per window
  const uint32_t mkl = ~((1u << (31 - R)) - 1u), skl = 1u << (30 - R);     // left: bit 31 - d
  const uint32_t mkr = (2u << R) - 1u, skr = 2u << R;                        // right: bit d
  auto nearest_w = [&](uint32_t rw, uint32_t lw) -> int {   // (rw, lw masked + sentinels)
    return min(__clz(lw), __ffs(rw) - 1);
  };
  uint32_t gr = 0u, gl = 0u;   // (NW == 2) the windows of G (masked), fixed for the sweep
  if constexpr (NW == 2) {
    gr = win_r(G[0], G[1]) & mkr;
    gl = win_l(G[0], G[1]) & mkl;
  }
  if (FC_ON) {               // before the first event every in-grid column is in C
    if constexpr (NW == 2) FC.kap = nearest_w(gr | skr, gl | skl);
    else FC.kap = nearest_bit<NW>(G, pp, R);
    FC.zstart = src.zlo;
  }
  auto sweep = [&](auto stg, auto prn) {
    constexpr bool STG = decltype(stg)::value, PRN = decltype(prn)::value;
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
        if constexpr (STG) {   // sentinel-terminated lists in shared memory
          pos[q] = padd(hit, pos[q], 4u, one);
          if (hit) nkey[q] = lds_u32(pos[q]);
        } else if (hit) {
          ++pos[q];
          nkey[q] = pos[q] < end[q] ? fkey(__ldg(ep + 2 * cb0[q] + pos[q])) : KEY_NONE;
        }
      }
      const float z = keyf(zk);
      int ks = knone, kc = knone;
      if constexpr (NW == 2) {
        const uint32_t mr = win_r(M[0], M[1]), ml = win_l(M[0], M[1]);
        if (FS_ON) ks = nearest_w((mr & mkr) | skr, (ml & mkl) | skl);
        if (FC_ON) kc = nearest_w((gr & ~mr) | skr, (gl & ~ml) | skl);
      } else {
        if (FS_ON) ks = nearest_bit<NW>(M, pp, R);
        if (FC_ON) {
          uint32_t C[NW];
#pragma unroll
          for (int q = 0; q < NW; ++q) C[q] = G[q] & ~M[q];
          kc = nearest_bit<NW>(C, pp, R);
        }
      }
      if (FS_ON) {
        const bool chg = ks != FS.kap;
        // an event changes kappa only for lanes within R of its column: a step where no lane of
        // the warp changes (often: halo events) skips the filter / emission half (warp-uniform)
        if (SKIP != 1 || __any_sync(FULL, chg)) {
          pfam_close<TABLE, PRN>(FS, chg && FS.kap != knone, FS.zstart, z, FS.kap, ths, h0s, mabs_s);
          FS.kap = fsel(chg, ks, FS.kap, FS.zero);
          FS.zstart = fsel(chg, z, FS.zstart, FS.zero);
        }
      }
      if (FC_ON) {
        const bool chg = kc != FC.kap;
        if (SKIP != 1 || __any_sync(FULL, chg)) {
          pfam_close<TABLE, PRN>(FC, chg && FC.kap != knone && FC.zstart < z, FC.zstart, z, FC.kap, thc, h0c,
                                 mabs_c);
          FC.kap = fsel(chg, kc, FC.kap, FC.zero);
          FC.zstart = fsel(chg, z, FC.zstart, FC.zero);
        }
      }
    }
  };
  // the sweep, versioned on the (warp-uniform) staging and filter decisions
  if (staged) {
    if (prune) sweep(std::true_type{}, std::true_type{});
    else sweep(std::true_type{}, std::false_type{});
  } else {
    if (prune) sweep(std::false_type{}, std::true_type{});
    else sweep(std::false_type{}, std::false_type{});
  }
  if (FC_ON) {   // C's last piece closes at z_hi
    const bool cl = FC.kap != knone && FC.zstart < src.zhi;
    if (prune) pfam_close<TABLE, true>(FC, cl, FC.zstart, src.zhi, FC.kap, thc, h0c, mabs_c);
    else pfam_close<TABLE, false>(FC, cl, FC.zstart, src.zhi, FC.kap, thc, h0c, mabs_c);
  }
  if (FS_ON) pfam_finish(FS, PS, c, T.jr, T.tile, ntiles, list_mode);
  if (FC_ON) pfam_finish(FC, PC, c, T.jr, T.tile, ntiles, list_mode);
  };
  if (!list_mode) {
    if (gw < (int64_t)nrows_out * ntiles) process(gw + (int64_t)jr0 * ntiles);   // warp-uniform
  } else {   // the listed tiles, their count read on the device (no host round trip): grid-stride
    const unsigned nl = min((unsigned)nlist, (FS_ON ? PS.flags : PC.flags)[2]);
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = gw; t < (int64_t)nl; t += nw) process((int64_t)tile_list[t]);
  }
}

constexpr size_t p1s_smem() { return (size_t)P1_WARPS * (P1_STAGE + 4) * 4; }

// ------------------------------------------------------------------ gather (small R)
// One thread per output column: merge the 2R+1 (<= 2 RM + 1) sorted endpoint lists of its
// neighbour columns (read through L1: neighbouring threads share them) and track the activity
// of each neighbour in a small mask; kappa = distance of the nearest active neighbour.
// Same families, filter, chunked store and list mode as p1s_kernel.
template <int RM, int FAMS>
__global__ void __launch_bounds__(P1G_T) p1g_kernel(SrcRows src, int R, int row0, int jr0, int nrows_out,
                                                     PieceSlots PS, PieceSlots PC, int64_t nlist,
                                                     const float* __restrict__ prune_s,
                                                     const float* __restrict__ prune_c) {
  constexpr int NC = 2 * RM + 1;
  __shared__ float2 thr_s[18 * 32], thr_c[18 * 32];
  constexpr bool FS_ON = (FAMS & 1) != 0, FC_ON = (FAMS & 2) != 0;
  const bool prune = FS_ON ? prune_s != nullptr : prune_c != nullptr;
  if (FS_ON && prune_s) p1_thr_init(thr_s, prune_s, R);
  if (FC_ON && prune_c) p1_thr_init(thr_c, prune_c, R);
  __syncthreads();
  const bool list_mode = nlist >= 0;
  const uint32_t* tile_list = FS_ON ? PS.tile_list : PC.tile_list;
  const int32_t* ovf_idx = FS_ON ? PS.ovf_idx : PC.ovf_idx;
  const int ntiles = (src.nx + 31) >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // list mode: a thread per column of the listed tiles (32 columns each), their count read on
  // the device, grid-stride (whole warps iterate together)
  const int64_t nlt = list_mode ? 32 * (int64_t)min((unsigned)nlist, (FS_ON ? PS.flags : PC.flags)[2]) : 0;
  const int64_t tstep = list_mode ? (int64_t)gridDim.x * blockDim.x : 1;   // (main mode: one pass)
  for (int64_t t = t0; list_mode ? (t - (int64_t)(threadIdx.x & 31)) < nlt : t == t0; t += tstep) {
  // (no early return of single lanes: the statistics reduction below needs whole warps)
  int jr = 0, i = 0;
  bool live;
  if (list_mode) {
    live = t < nlt;
    if (live) {
      const int64_t tl = (int64_t)tile_list[t >> 5];
      jr = (int)(tl / ntiles);
      i = (int)(tl % ntiles) * 32 + (int)(t & 31);
    }
  } else {
    live = t < (int64_t)nrows_out * src.nx;
    if (live) {
      jr = jr0 + (int)(t / src.nx);
      i = (int)(t % src.nx);
    }
  }
  live = live && i < src.nx;
  const int64_t c = (int64_t)jr * src.nx + i;
  int kind = live ? 0 : 2, aslot = 0;
  if (list_mode && live) {
    aslot = ovf_idx[c];
    kind = aslot >= 0 ? 1 : 2;
  }
  live = live && kind != 2;
  PFam FS, FC;
  const uint32_t ths = sh_addr(thr_s), thc = sh_addr(thr_c);
  if (FS_ON) pfam_init(FS, PS, jr, i, kind, aslot, ths);
  if (FC_ON) pfam_init(FC, PC, jr, i, kind, aslot, thc);
  if (live) {
    const uint64_t* off;
    const float* ep;
    src_row(src, row0 + jr, off, ep);
    // neighbour i - R + s, s = 0 .. 2R: endpoint cursor and next endpoint.  The merge compares
    // the fp32 values themselves (finite; +inf marks an exhausted list; -0 == +0 falls in one
    // step like the sweep's keys), no key conversion.
    uint32_t pos[NC], end[NC];
    float nz[NC];
    uint32_t G = 0u;
#pragma unroll
    for (int s = 0; s < NC; ++s) {
      const int gi = i - R + s;
      const bool in = s <= 2 * R && gi >= 0 && gi < src.nx;
      G |= in ? 1u << s : 0u;
      pos[s] = in ? (uint32_t)(2 * __ldg(off + gi)) : 0u;
      end[s] = in ? (uint32_t)(2 * __ldg(off + gi + 1)) : 0u;
      nz[s] = pos[s] < end[s] ? __ldg(ep + pos[s]) : INFINITY;
    }
    // kappa of an activity mask (bit s = the neighbour at distance |s - R|)
    auto kappa_of = [&](uint32_t m) -> int {
      const uint32_t left = m & ((2u << R) - 1u);   // s <= R
      const uint32_t right = m >> R;                  // s >= R
      const int dl = left ? R - (31 - __clz(left)) : KNONE;
      const int dr = right ? __ffs(right) - 1 : KNONE;
      return min(dl, dr);
    };
    uint32_t M = 0u;
    if (FC_ON) {   // before the first event every in-grid column is in C
      FC.kap = kappa_of(G);
      FC.zstart = src.zlo;
    }
    auto sweep = [&](auto prn) {
      constexpr bool PRN = decltype(prn)::value;
      for (;;) {
        float z = nz[0];
#pragma unroll
        for (int s = 1; s < NC; ++s) z = fminf(z, nz[s]);
        if (z == INFINITY) break;
#pragma unroll
        for (int s = 0; s < NC; ++s) {
          const bool hit = nz[s] == z;
          M ^= hit ? 1u << s : 0u;
          if (hit) {
            ++pos[s];
            nz[s] = pos[s] < end[s] ? __ldg(ep + pos[s]) : INFINITY;
          }
        }
        if (FS_ON) {
          const int kn = kappa_of(M);
          const bool chg = kn != FS.kap;
          pfam_close<true, PRN>(FS, chg && FS.kap != KNONE, FS.zstart, z, FS.kap, ths, nullptr, 0.f);
          FS.kap = chg ? kn : FS.kap;
          FS.zstart = chg ? z : FS.zstart;
        }
        if (FC_ON) {
          const int kn = kappa_of(G & ~M);
          const bool chg = kn != FC.kap;
          pfam_close<true, PRN>(FC, chg && FC.kap != KNONE && FC.zstart < z, FC.zstart, z, FC.kap, thc, nullptr,
                                0.f);
          FC.kap = chg ? kn : FC.kap;
          FC.zstart = chg ? z : FC.zstart;
        }
      }
    };
    if (prune) sweep(std::true_type{});
    else sweep(std::false_type{});
    if (FC_ON)   // C's last piece closes at z_hi
      if (prune) pfam_close<true, true>(FC, FC.kap != KNONE && FC.zstart < src.zhi, FC.zstart, src.zhi, FC.kap, thc,
                                        nullptr, 0.f);
      else pfam_close<true, false>(FC, FC.kap != KNONE && FC.zstart < src.zhi, FC.zstart, src.zhi, FC.kap, thc,
                                   nullptr, 0.f);
  }
  if (FS_ON) pfam_finish(FS, PS, c, jr, i >> 5, ntiles, list_mode);
  if (FC_ON) pfam_finish(FC, PC, c, jr, i >> 5, ntiles, list_mode);
  }
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
  const float2* zc = arena ? reinterpret_cast<const float2*>(P.ovf_z + 2 * (size_t)P.ovf_idx[c] * (P.ovf_cap / 4))
                           : reinterpret_cast<const float2*>(P.z + 2 * chunk_index(P, row, 0, i));
  const uint32_t* kc = arena ? P.ovf_k + (size_t)P.ovf_idx[c] * (P.ovf_cap / 4) : P.k + chunk_index(P, row, 0, i);
  const size_t cs = arena ? 1 : (size_t)P.nx;
  for (uint32_t t = 0; t < m; ++t) {
    oz[o + t] = zc[(size_t)(t >> 2) * cs * 4 + (t & 3)];
    ok[o + t] = (uint8_t)(kc[(size_t)(t >> 2) * cs] >> (8 * (t & 3)));
  }
}

}  // namespace dexel
