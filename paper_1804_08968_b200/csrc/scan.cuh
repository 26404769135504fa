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

}  // namespace dexel
