// scan.cuh -- two-phase allocation support: exclusive scan of u32 counts into
// u64 offsets (north star: "two-phase count, warp/block scan and write
// compaction").  Reduce-then-scan in three launches:
//   A  per-tile sums            (tile = SCAN_THREADS * SCAN_ITEMS counts)
//   B  exclusive scan of the tile sums (one CTA, chunked, carried)
//   C  per-tile block scan (warp shuffles) + tile offset -> offsets
// out[n] receives the total.  Counts are read once in A and once in C.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dexel {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint64_t t = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

// Block-wide exclusive scan of one u64 per thread; returns exclusive prefix, *total = block sum.
__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t v, uint64_t* total) {
  __shared__ uint64_t warp_sums[SCAN_THREADS / 32 + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t incl = warp_incl_scan_u64(v);
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint64_t s = lane < SCAN_THREADS / 32 ? warp_sums[lane] : 0;
    uint64_t si = warp_incl_scan_u64(s);
    if (lane < SCAN_THREADS / 32) warp_sums[lane] = si - s;
    if (lane == SCAN_THREADS / 32 - 1) warp_sums[SCAN_THREADS / 32] = si;  // slot after: total
  }
  __syncthreads();
  uint64_t res = incl - v + warp_sums[wid];
  *total = warp_sums[SCAN_THREADS / 32];
  __syncthreads();
  return res;
}

__global__ void scan_tile_sums(const uint32_t* __restrict__ cnt, uint64_t n, uint64_t* __restrict__ sums) {
  const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    uint64_t idx = base + (uint64_t)k * SCAN_THREADS + threadIdx.x;  // coalesced
    if (idx < n) s += cnt[idx];
  }
  uint64_t total;
  block_excl_scan_u64(s, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void scan_sums_exclusive(uint64_t* __restrict__ sums, uint64_t ntiles) {
  __shared__ uint64_t carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (uint64_t base = 0; base < ntiles; base += SCAN_THREADS) {
    uint64_t idx = base + threadIdx.x;
    uint64_t v = idx < ntiles ? sums[idx] : 0;
    uint64_t total;
    uint64_t ex = block_excl_scan_u64(v, &total);
    uint64_t carry = carry_s;
    if (idx < ntiles) sums[idx] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[ntiles] = carry_s;
}

__global__ void scan_tiles_write(const uint32_t* __restrict__ cnt, uint64_t n, const uint64_t* __restrict__ sums,
                                 uint64_t* __restrict__ out) {
  // each thread owns SCAN_ITEMS consecutive counts (strided staging through smem for coalescing)
  __shared__ uint32_t tile[SCAN_TILE];
  const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    uint64_t idx = base + (uint64_t)k * SCAN_THREADS + threadIdx.x;
    tile[k * SCAN_THREADS + threadIdx.x] = idx < n ? cnt[idx] : 0u;
  }
  __syncthreads();
  uint32_t v[SCAN_ITEMS];
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) { v[k] = tile[threadIdx.x * SCAN_ITEMS + k]; s += v[k]; }
  uint64_t total;
  uint64_t ex = block_excl_scan_u64(s, &total) + sums[blockIdx.x];
  __shared__ uint64_t res[SCAN_TILE];
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) { res[threadIdx.x * SCAN_ITEMS + k] = ex; ex += v[k]; }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    uint64_t idx = base + (uint64_t)k * SCAN_THREADS + threadIdx.x;   // coalesced
    if (idx < n) out[idx] = res[k * SCAN_THREADS + threadIdx.x];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = sums[gridDim.x];
}

// ---- single-launch variant: decoupled look-back (each tile publishes its aggregate, then its
// inclusive prefix, in a status word; a tile's thread 0 walks back over its predecessors'
// words).  Tiles take their index from an atomic ticket, so a tile only ever waits on tiles that
// started before it (no deadlock whatever the block scheduling).  status[0 .. ntiles) and the
// ticket (status[ntiles]) must be zero at launch.  Word: bits 62-63 = state (0 not ready,
// 1 aggregate, 2 inclusive prefix), bits 0-61 = the value.
constexpr unsigned long long SCAN_ST_A = 1ull << 62, SCAN_ST_P = 2ull << 62, SCAN_ST_V = (1ull << 62) - 1;

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_lookback(const uint32_t* __restrict__ cnt, uint64_t n,
                                                             unsigned long long* status, uint64_t* __restrict__ out) {
  __shared__ uint32_t tile[SCAN_TILE];
  __shared__ uint64_t res[SCAN_TILE];
  __shared__ unsigned long long tid_s, prefix_s;
  const uint64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (threadIdx.x == 0) tid_s = atomicAdd(status + ntiles, 1ull);
  __syncthreads();
  const uint64_t t = tid_s;
  const uint64_t base = t * SCAN_TILE;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    const uint64_t idx = base + (uint64_t)k * SCAN_THREADS + threadIdx.x;   // coalesced
    tile[k * SCAN_THREADS + threadIdx.x] = idx < n ? cnt[idx] : 0u;
  }
  __syncthreads();
  uint32_t v[SCAN_ITEMS];
  uint64_t sum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = tile[threadIdx.x * SCAN_ITEMS + k];
    sum += v[k];
  }
  uint64_t total;
  uint64_t ex = block_excl_scan_u64(sum, &total);
  if (threadIdx.x == 0) {
    unsigned long long excl = 0;
    if (t == 0) {
      st_release_u64(status, SCAN_ST_P | total);
    } else {
      st_release_u64(status + t, SCAN_ST_A | total);
      for (int64_t q = (int64_t)t - 1;;) {
        const unsigned long long w = ld_acquire_u64(status + q);
        if (!(w & ~SCAN_ST_V)) continue;   // not ready yet: spin
        excl += w & SCAN_ST_V;
        if (w & SCAN_ST_P) break;
        --q;
      }
      st_release_u64(status + t, SCAN_ST_P | (excl + total));
    }
    prefix_s = excl;
  }
  __syncthreads();
  ex += prefix_s;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    res[threadIdx.x * SCAN_ITEMS + k] = ex;
    ex += v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    const uint64_t idx = base + (uint64_t)k * SCAN_THREADS + threadIdx.x;   // coalesced
    if (idx < n) out[idx] = res[k * SCAN_THREADS + threadIdx.x];
  }
  if (t == ntiles - 1 && threadIdx.x == 0) out[n] = prefix_s + total;
}

}  // namespace dexel
