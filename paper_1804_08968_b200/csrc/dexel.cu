// dexel.cu -- host orchestration and C ABI (include/dexel.h) of the B200
// separable dexel offset library.  Builds libdexel.so for sm_100a.
//
// Op pipeline (one "family" per dilation; erode and shell dilate the
// complement, which pass 1 reads on the fly):
//   pass1 (slots; rare list pass)          S_In -> S_Mid (pieces lo,hi,kappa)
//   levels (forward stack sweep)           S_Mid -> level slots L_k, k = 0..R
//   pass2 (+ epilogue) -> scan -> compact  {L_k} -> S_Out (output CSR)
// Host synchronisations per family: the pass-1 total (allocation size) and the
// level kernel's capacity flags; per op: the pass-2 flags and the output total.
// A capacity overflow (piece slots, level list > cap, pass-2 union > acc) reruns that stage with a larger capacity; the sizes are kept as hints
// on the handle for later ops.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include <nccl.h>

#include "dexel.h"
#include "kernels.cuh"
#include "levels.cuh"
#include "pass1.cuh"
#include "pass2.cuh"
#include "raster.cuh"
#include "scan.cuh"

using namespace dexel;

namespace {

thread_local std::string g_err;

bool g_timing = false;

dexel_alloc_fn g_alloc = nullptr;
dexel_free_fn g_free = nullptr;
void* g_alloc_ctx = nullptr;

dexel_status fail(dexel_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(DEXEL_ECUDA, std::string(#call) + " (dexel.cu:" + std::to_string(__LINE__) + "): " + \
                                   cudaGetErrorString(e_));                                       \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  dexel_free_fn freefn = nullptr;   // the allocator that produced p (NULL: cudaMallocAsync)
  void* ctx = nullptr;
};

}  // namespace

struct dexel_grid_s {
  dexel_desc d;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int nrows = 0;        // local rows y1 - y0
  int64_t ncol = 0;     // local columns
  Buf off, ep;
  uint64_t n = 0;
  dexel_stats stats{};
  unsigned char* pin = nullptr;   // pinned host scratch for the small device->host readbacks
  // capacity hints carried between ops (grown on overflow)
  int lev_cap = 0, p2_acc = 0, p1_cap = 0;
  int p2_peak = 0;     // longest pass-2 union any op on this handle held (sizes p2_acc)
  int lev_arena = 0;   // level-list arena entries per list once lev_cap is at LV_SLOT_MAX (0: 4 lev_cap)
  // the previous input CSR after a re-upload: the next upload of a similar size fills it
  // instead of allocating (an upload must not touch the current contents until validated)
  Buf spare_off, spare_ep;
  // y-slab halos (multi-GPU): rows [y0 - hrows[0], y0) and [y1, y1 + hrows[1]) of the input
  Buf hoff[2], hep[2];
  int hrows[2] = {0, 0};
  uint64_t hn[2] = {0, 0};
  // halo transport: NCCL (desc.nccl_comm), loopback links to the
  // neighbouring slab handles of one process (dexel_link_slabs), else caller-managed halos
  // (dexel_upload_halo).  The exchange runs on its own stream; pass 1 of the slab's own rows
  // does not wait for it, the halo rows' launches wait on ev_halo.
  dexel_grid_s* link[2] = {nullptr, nullptr};
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_main = nullptr, ev_halo = nullptr;
  bool halo_pending = false;
  std::vector<int32_t> part;   // NCCL: every rank's slab rows (y0, y1), gathered on first use
  Buf hdr;                     // NCCL: interval counts sent [0..1] / received [2..3]
  // device h(kappa, k) tables of the last radii used (make_htab), with the host copies their
  // asynchronous uploads read from: a repeated op uploads nothing and waits for nothing
  struct HTab {
    float r = -1.f;
    double s = 0.0;
    Buf dev;
    std::vector<float> host;
  } htab[2];
  int htab_next = 0;
  // small-temporary arena (below WS_MIN): an op's small temporaries are carved from one block kept
  // on the handle between ops (stream-ordered reuse: the handle's ops run on its stream), instead
  // of a cudaMallocAsync / cudaFreeAsync pair each -- a dozen per op, a large share of a small
  // op's host time.  Temps nest as a stack (mark / reset); a request that does not fit falls back
  // to its own allocation and grows the arena for the next op.
  Buf arena;
  size_t arena_top = 0, arena_want = 0;
  int arena_depth = 0;
};

namespace {

// dst[t] = src[t] - src[0] + add, t in [0, n]
__global__ void rebase_offsets(const uint64_t* __restrict__ src, uint64_t n, uint64_t add, uint64_t* __restrict__ dst) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t <= n) dst[t] = src[t] - src[0] + add;
}

// host-side diagnostics (DEXEL_DEBUG): seconds spent in allocation calls and stream syncs
thread_local double g_t_alloc = 0.0, g_t_sync = 0.0, g_t_free = 0.0, g_t_info = 0.0;   // (diagnostics of the calling thread's op)
inline double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
inline cudaError_t timed_sync(cudaStream_t st) {
  const double t = now_s();
  const cudaError_t e = cudaStreamSynchronize(st);
  g_t_sync += now_s() - t;
  return e;
}

// small device->host readbacks through the handle's pinned buffer (a pageable destination makes
// cudaMemcpyAsync a staged, host-synchronous copy); offsets are bytes into the 256-byte buffer
struct Readback {
  dexel_grid g;
  cudaError_t err = cudaSuccess;
  void add(size_t off, const void* dev, size_t bytes) {
    if (err == cudaSuccess) err = cudaMemcpyAsync(g->pin + off, dev, bytes, cudaMemcpyDeviceToHost, g->stream);
  }
  cudaError_t wait() { return err != cudaSuccess ? err : timed_sync(g->stream); }
  void get(size_t off, void* dst, size_t bytes) const { std::memcpy(dst, g->pin + off, bytes); }
};

dexel_status dalloc(dexel_grid g, Buf& b, size_t bytes) {
  const double t0 = now_s();
  struct Acc { double t0; ~Acc() { g_t_alloc += now_s() - t0; } } acc_{t0};
  b.bytes = bytes;
  b.p = nullptr;
  if (bytes == 0) bytes = 16;
  b.freefn = g_free;
  b.ctx = g_alloc_ctx;
  if (g_alloc) {
    b.p = g_alloc(bytes, g->d.device, (void*)g->stream, g_alloc_ctx);
    if (!b.p) return fail(DEXEL_ENOMEM, "allocator returned NULL for " + std::to_string(bytes) + " bytes");
  } else {
    cudaError_t e = cudaMallocAsync(&b.p, bytes, g->stream);
    if (e != cudaSuccess) {
      b.p = nullptr;
      cudaGetLastError();   // (reported here: a caller that recovers must not see it again later)
      return fail(DEXEL_ENOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e) + " (" +
                                    std::to_string(bytes) + " bytes)");
    }
  }
  return DEXEL_OK;
}

void dfree(dexel_grid g, Buf& b) {
  if (!b.p) return;
  const double t0 = now_s();
  struct Acc { double t0; ~Acc() { g_t_free += now_s() - t0; } } acc_{t0};
  // free with the allocator that allocated it, even if the hook changed since
  if (b.freefn) b.freefn(b.p, b.bytes ? b.bytes : 16, g->d.device, (void*)g->stream, b.ctx);
  else cudaFreeAsync(b.p, g->stream);
  b.p = nullptr;
  b.bytes = 0;
}

// per-op kernel accounting: launch counts always, CUDA-event device times when g_timing
enum { K_P1 = 0, K_P1LIST = 1, K_LEV = 2, K_P2 = 3, K_COMPACT = 4, K_SCAN = 5, K_OTHER = 6, K_RASTER = 7 };
struct Prof {
  cudaStream_t st = nullptr;
  dexel_stats* s = nullptr;
  bool on = false;
  int curk = K_OTHER;
  cudaEvent_t cur = nullptr;
  struct Rec { int k; cudaEvent_t a, b; };
  std::vector<Rec> ev;
  void pre(int k) {
    curk = k;
    if (on) { cudaEventCreate(&cur); cudaEventRecord(cur, st); }
  }
  void post() {
    if (s) { s->launches++; s->kernel_calls[curk]++; }
    if (on) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, st);
      ev.push_back({curk, cur, e});
    }
  }
  void finish() {
    if (!ev.empty()) {
      cudaEventSynchronize(ev.back().b);
      for (auto& r : ev) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        if (s) s->kernel_ms[r.k] += ms;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
      }
      ev.clear();
    }
  }
  ~Prof() { finish(); }
};

// Device workspace: an op's large temporaries (band slot arrays, staging) stay allocated and
// are reused by size by later ops of any handle on the device; freeing them to the
// stream-ordered pool and allocating again fragments the pool once other allocations (e.g. a
// re-upload) land in the freed blocks, and the pool then remaps tens of GB per op (measured:
// 150-900 ms).  A block released on one stream and taken on another is ordered by an event.
// Idle blocks are freed when the device's last handle is destroyed, or on out-of-memory.
// The band budget lives here too (queried once per device: a driver query per op costs
// 0.2-11 ms under contention, and one budget for all handles keeps the block sizes shared).
struct WsEntry {
  Buf b;
  bool busy = false;
  cudaEvent_t ev = nullptr;      // recorded on the stream that last released the block
  cudaStream_t last = nullptr;
};
struct DevWs {
  std::mutex mu;
  std::vector<WsEntry> e;        // (indices are stable: freed entries keep an empty Buf)
  int handles = 0;
  size_t band_budget = 0;
};
DevWs& dev_ws(int device) {
  static DevWs w[64];
  return w[device & 63];
}
constexpr size_t WS_MIN = (size_t)32 << 20;   // temporaries from this size on use the workspace

// free the idle blocks of a device's workspace, ordered after their last users on stream st
void ws_trim_idle(dexel_grid g) {
  DevWs& W = dev_ws(g->d.device);
  std::lock_guard<std::mutex> lk(W.mu);
  for (auto& e : W.e)
    if (!e.busy && e.b.p) {
      // a caller allocator (e.g. torch's caching allocator) only orders the free on its own
      // allocation stream: wait for the block's last user on the host before handing it back
      if (e.ev && e.b.freefn) cudaEventSynchronize(e.ev);
      else if (e.ev && e.last != g->stream) cudaStreamWaitEvent(g->stream, e.ev, 0);
      dfree(g, e.b);
      if (e.ev) cudaEventDestroy(e.ev);
      e.ev = nullptr;
      e.last = nullptr;
    }
}

// RAII for temporaries of one op

struct Temps {
  dexel_grid g;
  std::vector<Buf> bufs;
  std::vector<int> wsi;   // workspace entries this op holds
  Prof prof;
  size_t mark = 0, top = 0;   // the handle's arena: this op's first byte, its next free byte
  explicit Temps(dexel_grid g_, dexel_stats* st = nullptr) : g(g_) {
    prof.st = g_->stream;
    prof.s = st;
    prof.on = g_timing && st != nullptr;
    if (g->arena_depth == 0 && g->arena_want > g->arena.bytes) {   // grow (no op holds it now)
      dfree(g, g->arena);
      if (dalloc(g, g->arena, g->arena_want + g->arena_want / 4 + ((size_t)64 << 10)) != DEXEL_OK) {
        g->arena = Buf{};
        g_err.clear();
      }
    }
    ++g->arena_depth;
    mark = top = g->arena_top;
  }
  ~Temps() {
    prof.finish();
    for (auto& b : bufs) dfree(g, b);
    while (!wsi.empty()) release_ws(0);
    g->arena_want = std::max(g->arena_want, top);
    g->arena_top = mark;
    --g->arena_depth;
  }
  void release_ws(size_t t) {   // hand block wsi[t] back, ordered after this op's stream work
    DevWs& W = dev_ws(g->d.device);
    std::lock_guard<std::mutex> lk(W.mu);
    WsEntry& e = W.e[wsi[t]];
    e.busy = false;
    if (!e.ev) cudaEventCreateWithFlags(&e.ev, cudaEventDisableTiming);
    if (e.ev) cudaEventRecord(e.ev, g->stream);
    e.last = g->stream;
    wsi.erase(wsi.begin() + t);
  }
  dexel_status get(size_t bytes, void** p) {
    if (bytes >= WS_MIN) {   // a free workspace block of about this size (at most 1/4 larger)
      DevWs& W = dev_ws(g->d.device);
      {
        std::lock_guard<std::mutex> lk(W.mu);
        int best = -1;
        for (int w = 0; w < (int)W.e.size(); ++w)
          if (!W.e[w].busy && W.e[w].b.p && W.e[w].b.bytes >= bytes && W.e[w].b.bytes - bytes <= bytes / 4 &&
              (best < 0 || W.e[w].b.bytes < W.e[best].b.bytes))
            best = w;
        if (best >= 0) {
          WsEntry& e = W.e[best];
          e.busy = true;
          if (e.ev && e.last != g->stream) cudaStreamWaitEvent(g->stream, e.ev, 0);
          wsi.push_back(best);
          *p = e.b.p;
          return DEXEL_OK;
        }
      }
      Buf b;
      dexel_status s = dalloc(g, b, bytes);
      if (s == DEXEL_ENOMEM) {   // drop the idle workspace and retry once
        ws_trim_idle(g);
        g_err.clear();
        s = dalloc(g, b, bytes);
      }
      if (s) return s;
      std::lock_guard<std::mutex> lk(W.mu);
      WsEntry e;
      e.b = b;
      e.busy = true;
      W.e.push_back(e);
      wsi.push_back((int)W.e.size() - 1);
      *p = b.p;
      return DEXEL_OK;
    }
    const size_t a = (bytes + 255) & ~(size_t)255;
    if (top + a <= ((size_t)256 << 20)) {   // (the arena holds at most 256 MB)
      const size_t at = top;
      top += a;
      if (g->arena.p && g->arena_top == at && top <= g->arena.bytes) {   // (innermost Temps only)
        g->arena_top = top;
        *p = (char*)g->arena.p + at;
        return DEXEL_OK;
      }
    }
    Buf b;
    dexel_status s = dalloc(g, b, bytes);
    if (s) return s;
    bufs.push_back(b);
    *p = b.p;
    return DEXEL_OK;
  }
  void release(void* p) {   // (an arena block is released with its Temps)
    for (auto& b : bufs)
      if (b.p == p) dfree(g, b);
    for (size_t t = 0; t < wsi.size(); ++t) {
      bool hit;
      {
        DevWs& W = dev_ws(g->d.device);
        std::lock_guard<std::mutex> lk(W.mu);
        hit = W.e[wsi[t]].b.p == p;
      }
      if (hit) {
        release_ws(t);
        break;
      }
    }
  }
};

#define LAUNCH(T, KID, ...) do { (T).prof.pre(KID); __VA_ARGS__; (T).prof.post(); } while (0)

// exclusive scan of cnt[0..n) into off[0..n], returns total (synchronising read)
dexel_status scan_counts(dexel_grid g, Temps& T, const uint32_t* cnt, uint64_t n, uint64_t* off, uint64_t* total) {
  const uint64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  uint64_t* sums = nullptr;
  dexel_status s = T.get(sizeof(uint64_t) * (ntiles + 2), (void**)&sums);
  if (s) return s;
  if (n == 0) {
    CK(cudaMemsetAsync(off, 0, sizeof(uint64_t), g->stream));
    *total = 0;
    T.release(sums);
    return DEXEL_OK;
  }
  LAUNCH(T, K_SCAN, scan_tile_sums<<<(unsigned)ntiles, SCAN_THREADS, 0, g->stream>>>(cnt, n, sums));
  LAUNCH(T, K_SCAN, scan_sums_exclusive<<<1, SCAN_THREADS, 0, g->stream>>>(sums, ntiles));
  LAUNCH(T, K_SCAN, scan_tiles_write<<<(unsigned)ntiles, SCAN_THREADS, 0, g->stream>>>(cnt, n, sums, off));
  CK(cudaGetLastError());
  Readback rb{g};
  rb.add(0, off + n, sizeof(uint64_t));
  CK(rb.wait());
  rb.get(0, total, sizeof(uint64_t));
  T.release(sums);
  return DEXEL_OK;
}

// exclusive scan of cnt[0..n) into off[0..n], the total at off[n] (stays on the device): one
// decoupled look-back launch (scan.cuh) whose status words -- scan_status_words(n), zeroed by
// the caller (the op zeroes them with its flag words) -- live at `status`
inline size_t scan_status_words(uint64_t n) { return (size_t)((n + SCAN_TILE - 1) / SCAN_TILE) + 1; }
dexel_status scan_counts_dev(dexel_grid g, Temps& T, const uint32_t* cnt, uint64_t n, uint64_t* off,
                             unsigned long long* status) {
  const uint64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (n == 0) {
    CK(cudaMemsetAsync(off, 0, sizeof(uint64_t), g->stream));
    return DEXEL_OK;
  }
  LAUNCH(T, K_SCAN, scan_lookback<<<(unsigned)ntiles, SCAN_THREADS, 0, g->stream>>>(cnt, n, status, off));
  CK(cudaGetLastError());
  return DEXEL_OK;
}

int radius_levels(double r, double s) {
  int R = (int)std::floor(r / s);
  while ((double)(R + 1) * s <= r) ++R;
  while (R > 0 && (double)R * s > r) --R;
  return R;
}

dexel_status check_radius(float r, double s, int* R) {
  if (!std::isfinite(r) || r < 0.f) return fail(DEXEL_EINVAL, "radius must be finite and >= 0");
  *R = radius_levels((double)r, s);
  if (*R > 255) return fail(DEXEL_EINVAL, "R = floor(r/spacing) must be <= 255");
  return DEXEL_OK;
}

// ---------------------------------------------------------------- pass 1
// one pass-1 launch of families `fams` (1 = S, 2 = C = U \ S, 3 = both, pass1.cuh): main mode
// over slot rows [jr0, jr0 + nrows_out) of a band whose slot row 0 is extended row row0; list mode
// (nlist >= 0, one family) over the listed tiles
template <int NW, int F, bool TABLE, int SKIP>
void launch_p1s_t(unsigned blocks, cudaStream_t st, const SrcRows& src, int R, int row0, int jr0, int nrows_out,
                  const PieceSlots& PS, const PieceSlots& PC, int64_t nlist, const float* ps, const float* pc) {
  const size_t smem = p1s_smem();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(p1s_kernel<NW, F, TABLE, SKIP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  p1s_kernel<NW, F, TABLE, SKIP><<<blocks, P1_WARPS * 32, smem, st>>>(src, R, row0, jr0, nrows_out, PS, PC, nlist, ps, pc);
}

template <int F>
void launch_p1_f(const SrcRows& src, int R, int row0, int jr0, int nrows_out, const PieceSlots& PS,
                 const PieceSlots& PC, int64_t nlist, const float* ps, const float* pc, cudaStream_t st,
                 int64_t list_warps = 0) {
  // (list mode, nlist >= 0: nlist is the tile list's capacity, the kernels read the live count;
  // list_warps warps walk it grid-stride)
  if (R <= P1G_RMAX) {   // gather: a thread per output column (list mode: 32 per listed tile)
    const int64_t threads = nlist >= 0 ? list_warps * 32 : (int64_t)nrows_out * src.nx;
    const unsigned blocks = (unsigned)((threads + P1G_T - 1) / P1G_T);
    if (blocks == 0) return;
#define P1G(RM) p1g_kernel<RM, F><<<blocks, P1G_T, 0, st>>>(src, R, row0, jr0, nrows_out, PS, PC, nlist, ps, pc)
    if (R <= 1) P1G(1);
    else if (R == 2) P1G(2);
    else if (R == 3) P1G(3);
    else P1G(4);
#undef P1G
    return;
  }
  // warp sweep: a warp per 32 output columns (list mode: the listed tiles)
  const int64_t warps = nlist >= 0 ? list_warps : (int64_t)nrows_out * ((src.nx + 31) / 32);
  const unsigned blocks = (unsigned)((warps + P1_WARPS - 1) / P1_WARPS);
  if (blocks == 0) return;
  const int NW = (32 + 2 * R + 31) / 32;   // window words
#define P1S(NWV, TB, SK) launch_p1s_t<NWV, F, TB, SK>(blocks, st, src, R, row0, jr0, nrows_out, PS, PC, nlist, ps, pc)
  // the step-skip vote (a warp vote per family and step) no longer pays for R <= 16 since the emission
  // half moved to the FMA pipe (measured: C4 r = 8 pass 1 4.11 -> 3.83 ms without it, C5 equal); it
  // stays for the larger windows.  DEXEL_P1_SKIP=1 forces it on (A/B).
  static const int skip_mode = [] { const char* e = std::getenv("DEXEL_P1_SKIP"); return e ? std::atoi(e) : -1; }();
  if (NW <= 2 && skip_mode != 1) P1S(2, true, 0);
  else if (NW <= 2) P1S(2, true, 1);
  else if (NW <= 3) P1S(3, false, 1);
  else if (NW <= 5) P1S(5, false, 1);
  else if (NW <= 9) P1S(9, false, 1);
  else P1S(17, false, 1);
#undef P1S
}

// single family: complement = 0 -> S into P, 1 -> C into P
void launch_p1(const SrcRows& src, int R, int complement, int row0, int jr0, int nrows_out, const PieceSlots& P,
               int64_t nlist, const float* prune, cudaStream_t st, int64_t list_warps = 0) {
  if (complement) launch_p1_f<2>(src, R, row0, jr0, nrows_out, P, P, nlist, nullptr, prune, st, list_warps);
  else launch_p1_f<1>(src, R, row0, jr0, nrows_out, P, P, nlist, prune, nullptr, st, list_warps);
}

// Pass-1 launches of band rows [row0, row0 + nrows) (extended numbering), split so that the
// slab's own rows go first and the halo rows -- still arriving on the exchange stream when
// g->halo_pending -- wait for the exchange (g->ev_halo): the transfer overlaps the interior
// pass 1.  f(jr0, count) launches slot rows [jr0, jr0 + count) of the band.
template <class F>
cudaError_t launch_rows_split(dexel_grid g, const SrcRows& src, int row0, int nrows, F&& f) {
  const int own0 = src.rows[0], own1 = src.rows[0] + src.rows[1], r1 = row0 + nrows;
  auto seg = [&](int a, int b) { if (b > a) f(a - row0, b - a); };
  if (!g->halo_pending || (row0 >= own0 && r1 <= own1)) {
    seg(row0, r1);
    return cudaGetLastError();
  }
  seg(std::max(row0, own0), std::min(r1, own1));      // the slab's own rows: no wait
  cudaError_t e = cudaStreamWaitEvent(g->stream, g->ev_halo, 0);
  if (e != cudaSuccess) return e;
  seg(row0, std::min(r1, own0));                      // halo rows below the slab
  seg(std::max(row0, own1), r1);                      // halo rows above
  return cudaGetLastError();
}

// Pass 1 over band rows [row0, row0+nrows) of src: pieces into per-column slots (one launch, split
// around the halo rows), then the list launch that recomputes the columns that outgrew their slots
// into the arena -- launched unconditionally: it reads the listed-tile count on the device, so the
// host never waits here.  A column that fits neither (too many listed, or longer than the arena
// lists) raises OPF_P1_RERUN; the op's one readback reruns it with larger slots (run_op_impl).
dexel_status p1_alloc(dexel_grid g, Temps& T, const SrcRows& src, int nrows, unsigned* opf, PieceSlots* P) {
  const int64_t ncol = (int64_t)nrows * src.nx;
  const int ntiles = (src.nx + 31) / 32;
  dexel_status s;
  *P = PieceSlots{};
  P->nx = src.nx;
  P->nrows = nrows;
  P->cap = (g->p1_cap > 0 ? (g->p1_cap + 3) / 4 * 4 : 256);   // (whole chunks of 4 pieces)
  // the arena: up to 1/64 of the columns, 4x the slot capacity each (beyond: the op reruns with
  // larger slots -- a memory trade: larger slots for every column cost more bands)
  P->ovf_list_cap = (unsigned)std::max<int64_t>(256, ncol / 64);
  P->ovf_cap = 4 * P->cap;                                    // arena pieces per listed column
  P->opf = opf;
  P->total = reinterpret_cast<unsigned long long*>(opf + 8);   // n_mid
  // the kernels address a column's chunks with 32-bit offsets (chunk * nx)
  const size_t nch = (size_t)(P->cap / 4 + 1);   // chunks per column (+ the spill chunk)
  if (nch * 4 * (size_t)src.nx >= ((size_t)1 << 31))
    return fail(DEXEL_EOVERFLOW, "pass-1 slot offsets exceed 32 bits (grid too wide for the piece capacity)");
  if ((s = T.get(sizeof(uint32_t) * (ncol + 1), (void**)&P->cnt))) return s;
  if ((s = T.get(sizeof(int32_t) * (ncol + 1), (void**)&P->ovf_idx))) return s;
  if ((s = T.get(64, (void**)&P->flags))) return s;
  if ((s = T.get(sizeof(uint32_t) * P->ovf_list_cap * 2, (void**)&P->ovf_list))) return s;
  P->tile_list = P->ovf_list + P->ovf_list_cap;
  if ((s = T.get(sizeof(uint32_t) * ((size_t)nrows * ntiles + 1), (void**)&P->tile_flag))) return s;
  if ((s = T.get(2 * sizeof(float4) * nch * ncol + 32, (void**)&P->z))) return s;
  if ((s = T.get(sizeof(uint32_t) * nch * ncol + 16, (void**)&P->k))) return s;
  const size_t na = (size_t)P->ovf_list_cap * (P->ovf_cap / 4);
  if ((s = T.get(2 * sizeof(float4) * na + 32, (void**)&P->ovf_z))) return s;
  if ((s = T.get(sizeof(uint32_t) * na + 16, (void**)&P->ovf_k))) return s;
  CK(cudaMemsetAsync(P->flags, 0, 64, g->stream));
  CK(cudaMemsetAsync(P->tile_flag, 0, sizeof(uint32_t) * ((size_t)nrows * ntiles + 1), g->stream));
  CK(cudaMemsetAsync(P->ovf_idx, 0xff, sizeof(int32_t) * (ncol + 1), g->stream));   // -1: slots
  return DEXEL_OK;
}

// the list launch: a fixed grid walks the listed tiles (count read on the device)
void p1_list_launch(Temps& T, const SrcRows& src, int R, int fams, int row0, const PieceSlots& PS,
                    const PieceSlots& PC, const float* ps, const float* pc, cudaStream_t st) {
  const unsigned nl = (fams == 2 ? PC : PS).ovf_list_cap;   // the tile list's capacity
  const int64_t cap_warps = std::min<int64_t>(nl, 148 * 16);
  T.prof.pre(K_P1LIST);
  if (fams == 1) launch_p1_f<1>(src, R, row0, 0, 0, PS, PC, (int64_t)nl, ps, pc, st, cap_warps);
  else launch_p1_f<2>(src, R, row0, 0, 0, PS, PC, (int64_t)nl, ps, pc, st, cap_warps);
  T.prof.post();
}

dexel_status run_pass1(dexel_grid g, Temps& T, const SrcRows& src, int R, int complement, int row0, int nrows,
                       unsigned* opf, PieceSlots* P, const float* prune) {
  dexel_status s;
  if ((s = p1_alloc(g, T, src, nrows, opf, P))) return s;
  CK(launch_rows_split(g, src, row0, nrows, [&](int jr0, int cnt) {
    T.prof.pre(K_P1);
    launch_p1(src, R, complement, row0, jr0, cnt, *P, -1, prune, g->stream);
    T.prof.post();
  }));
  p1_list_launch(T, src, R, complement ? 2 : 1, row0, *P, *P, complement ? nullptr : prune, complement ? prune : nullptr,
                 g->stream);
  CK(cudaGetLastError());
  return DEXEL_OK;
}

// both shell families (S at r_a, C = U \ S at r_b, the same R) in one sweep (FAMS = 3); the
// overflow columns are redone per family in list mode
dexel_status run_pass1_dual(dexel_grid g, Temps& T, const SrcRows& src, int R, int row0, int nrows, unsigned* opf,
                            PieceSlots* PA, PieceSlots* PB, const float* prune_a, const float* prune_b) {
  dexel_status s;
  if ((s = p1_alloc(g, T, src, nrows, opf, PA))) return s;
  if ((s = p1_alloc(g, T, src, nrows, opf, PB))) return s;
  CK(launch_rows_split(g, src, row0, nrows, [&](int jr0, int cnt) {
    T.prof.pre(K_P1);
    launch_p1_f<3>(src, R, row0, jr0, cnt, *PA, *PB, -1, prune_a, prune_b, g->stream);
    T.prof.post();
  }));
  p1_list_launch(T, src, R, 1, row0, *PA, *PA, prune_a, nullptr, g->stream);
  p1_list_launch(T, src, R, 2, row0, *PB, *PB, nullptr, prune_b, g->stream);
  CK(cudaGetLastError());
  return DEXEL_OK;
}

void release_pieces(Temps& T, PieceSlots& P) {
  for (void* p : {(void*)P.z, (void*)P.k, (void*)P.cnt, (void*)P.ovf_idx, (void*)P.flags, (void*)P.ovf_list,
                  (void*)P.tile_flag, (void*)P.ovf_z, (void*)P.ovf_k})
    if (p) T.release(p);
}

// h(kappa,k) = sqrt(r^2 - (kappa^2 + k^2) s^2) computed in fp64 on the host and rounded once
// to fp32 (readings R10, R20), -1 where kappa^2 + k^2 > (r/s)^2: the device never
// evaluates a square root of a weight, and which (kappa, k) contribute is decided exactly.
dexel_status make_htab(dexel_grid g, Temps& T, float r, int R, float** out, float** prune) {
  (void)T;
  const double s = g->d.spacing;
  const int n1 = R + 1;
  const char* e = std::getenv("DEXEL_NO_PRUNE");
  const bool no_prune = e && std::atoi(e);
  const size_t nh = (size_t)n1 * n1;
  for (auto& H : g->htab)   // the same radius as a recent op: nothing to build, upload or wait for
    if (H.dev.p && H.r == r && H.s == s) {
      *out = (float*)H.dev.p;
      *prune = no_prune ? nullptr : *out + nh;
      return DEXEL_OK;
    }
  dexel_grid_s::HTab& H = g->htab[g->htab_next];
  g->htab_next ^= 1;
  std::vector<float> h(nh + n1 + 1);
  const double rr = (double)r * (double)r;
  for (int a = 0; a < n1; ++a)
    for (int k = 0; k < n1; ++k) {
      const double w = rr - ((double)a * a + (double)k * k) * s * s;   // exact for fp32 r, small integers
      h[(size_t)a * n1 + k] = w >= 0.0 ? (float)std::sqrt(w) : -1.0f;
    }
  // capsule-domination table for the pass-1 filter: h(kappa, 0), rounded once to fp32
  // (DEXEL_NO_PRUNE=1 disables the filter)
  // (+ one entry: the absolute part of the domination margin, 16 r 2^-24 >= 8 ulp(r), kernels.cuh)
  for (int a = 0; a < n1; ++a) h[nh + a] = (float)std::sqrt(std::max(0.0, rr - (double)a * a * s * s));
  h[nh + n1] = (float)(16.0 * (double)r * std::ldexp(1.0, -24));
  dexel_status st;
  dfree(g, H.dev);   // (stream-ordered after the ops that used it)
  H.r = -1.f;
  if ((st = dalloc(g, H.dev, sizeof(float) * h.size() + 16))) return st;
  H.host.swap(h);
  // the host copy stays alive with the cache entry; the upload is stream-ordered, no wait
  CK(cudaMemcpyAsync(H.dev.p, H.host.data(), sizeof(float) * H.host.size(), cudaMemcpyHostToDevice, g->stream));
  H.r = r;
  H.s = s;
  *out = (float*)H.dev.p;
  *prune = no_prune ? nullptr : *out + nh;
  return DEXEL_OK;
}

// level slots of one family for level rows [lr0, lr0 + lrn) (extended-row numbering):
// pass 1 on those rows, then the level-set kernel and its overflow pass (launched unconditionally:
// it reads the listed-column count on the device); the pieces are freed on return.  A list that
// fits neither its slots nor the arena raises OPF_LV_RERUN (the op's readback reruns it with a
// larger level capacity).  (pre != nullptr: the family's pieces were computed already, by
// run_pass1_dual)
dexel_status run_levels(dexel_grid g, Temps& T, const SrcRows& src, int R, const float* htab, const float* prune,
                        int complement, int lr0, int lrn, unsigned* opf, LevelSlots* L,
                        const PieceSlots* pre = nullptr, bool slices = false) {
  // slices: only L_0 is needed (pass 2 reads dy = 0), so only the first chunk of levels runs
  const int nlev_compute = slices ? 1 : R + 1;
  dexel_status s;
  PieceSlots P;
  if (pre) P = *pre;
  else if ((s = run_pass1(g, T, src, R, complement, lr0, lrn, opf, &P, prune))) return s;
  const int64_t ncol = (int64_t)lrn * src.nx;
  unsigned* flags = nullptr;
  if ((s = T.get(128, (void**)&flags))) return s;
  unsigned long long* nlev = reinterpret_cast<unsigned long long*>(opf + 10);
  L->R = R;
  L->ry = slices ? 0 : R;
  L->nx = src.nx;
  L->nrows = lrn;
  L->row0 = lr0;
  // slots per list: the level capacity + the LV_CLAMP - 1 slots a list may run past its clamp point
  // between two clamps (levels.cuh)
  L->cap = (g->lev_cap > 0 ? g->lev_cap : 8) + LV_CLAMP - 1;
  // arena lists: 4x the slot capacity (at least 32); longer lists rerun the op with larger slots,
  // then (slots at LV_SLOT_MAX) with a larger arena
  L->ovf_cap = std::min(LV_CNT_MAX, std::max({32, 4 * L->cap, g->lev_arena}));
  const size_t nlist = (size_t)ncol * (R + 1);
  if ((s = T.get(sizeof(uint16_t) * nlist + 16, (void**)&L->cnt))) return s;
  if ((s = T.get(sizeof(int32_t) * ncol + 16, (void**)&L->ovf_idx))) return s;
  const unsigned ovf_list_cap = (unsigned)std::max<int64_t>(256, ncol / 256);
  uint32_t* ovf_list = nullptr;
  if ((s = T.get(sizeof(uint32_t) * ovf_list_cap, (void**)&ovf_list))) return s;
  const size_t nslot = (size_t)ncol * (R + 2) * (L->cap + 1);   // + the dummy slot, the spill level
  if ((size_t)(R + 2) * (L->cap + 1) * src.nx >= (1ull << 32))
    return fail(DEXEL_EOVERFLOW, "level slot offsets exceed 32 bits (grid too wide for this radius)");
  if ((s = T.get(sizeof(float2) * nslot + 16, (void**)&L->z))) return s;
  if ((s = T.get(sizeof(float2) * (size_t)ovf_list_cap * ((size_t)(R + 1) * (L->ovf_cap + 1) + LV_CLAMP) + 16,
                 (void**)&L->ovf_z)))
    return s;
  CK(cudaMemsetAsync(flags, 0, 128, g->stream));
  CK(cudaMemsetAsync(L->ovf_idx, 0xff, sizeof(int32_t) * ncol, g->stream));   // -1: no arena slot
  // levels per thread: the smallest instantiated chunk size covering R+1 in as few chunks of
  // <= max_chunk (larger chunks cost more in registers/occupancy than they save)
  static const int kChunk[] = {2, 3, 4, 5, 6, 8, 10, 12, 14, 17};
  int max_chunk = 17;   // measured on B200 (branch-free emission): 17 beats 12 at r = 16 and 32
  if (const char* e = std::getenv("DEXEL_LV_CHUNK")) max_chunk = std::max(2, std::min(17, std::atoi(e)));
  const int nchunk = (nlev_compute + max_chunk - 1) / max_chunk;
  const int per = (nlev_compute + nchunk - 1) / nchunk;
  int lmax = 17;
  for (int v : kChunk)
    if (v >= per) { lmax = v; break; }
  auto launch = [&](const LvArgs& A, int64_t nwork) {
    if (nwork <= 0) return;
    const dim3 grid((unsigned)((nwork + LV_T - 1) / LV_T), (unsigned)nchunk);
    T.prof.pre(K_LEV);
    switch (lmax) {
#define LV(V) case V: levels_kernel<V><<<grid, LV_T, 0, g->stream>>>(A); break;
      LV(2) LV(3) LV(4) LV(5) LV(6) LV(8) LV(10) LV(12) LV(14) LV(17)
#undef LV
    }
    T.prof.post();
  };
  static const bool dbg_on = std::getenv("DEXEL_DEBUG") != nullptr;
  unsigned long long* dbg = dbg_on ? (unsigned long long*)(flags + 12) : nullptr;
  LvArgs A{P, ncol, htab, src.zlo, src.zhi, *L, flags, nlev, dbg, ovf_list, ovf_list_cap, nullptr, opf};
  launch(A, ncol);
  if (dbg) {   // (diagnostics only: waits)
    unsigned long long hd[3];
    CK(cudaMemcpyAsync(hd, dbg, sizeof(hd), cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    std::fprintf(stderr, "[dexel] levels rows %d..%d main pass: %lld columns, %.2f pieces per column, "
                 "%.2f per lane (warp maxima)\n", lr0, lr0 + lrn, (long long)ncol,
                 (double)hd[2] / std::max<int64_t>(1, ncol), (double)hd[0] / std::max(1ull, hd[1]));
    CK(cudaMemsetAsync(dbg, 0, sizeof(hd), g->stream));
  }
  // the overflow pass: every listed column's lists into the arena (a fixed grid, grid-stride over
  // the count the main pass left on the device)
  LvArgs B = A;
  B.list = ovf_list;
  launch(B, std::min<int64_t>(ovf_list_cap, 148 * 8 * LV_T));
  CK(cudaGetLastError());
  if (dbg) {   // (diagnostics only: waits)
    unsigned long long hd[3];
    CK(cudaMemcpyAsync(hd, dbg, sizeof(hd), cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    std::fprintf(stderr, "[dexel] levels rows %d..%d overflow pass: %llu warps, %.1f pieces per lane\n",
                 lr0, lr0 + lrn, hd[1], (double)hd[0] / std::max(1ull, hd[1]));
  }
  release_pieces(T, P);
  T.release(ovf_list);
  T.release(flags);
  return DEXEL_OK;
}

struct P2Out {
  int64_t cbase, ncol;     // first output column of the band; staging stride (all output columns)
  int acc;
  float2* stage;
  uint32_t* ocnt;
  unsigned* flags;
  float2* gacc;            // global accumulator [acc][band columns] (unions beyond shared memory) or null
};

template <int OP, int TT>
void launch_pass2_t(const LevelSlots& A, const LevelSlots& B, int nx, int row0, int nrows, float zlo, float zhi,
                    const P2Out& O, cudaStream_t st) {
  const int acc = O.acc;
  const unsigned blocks = (unsigned)((int64_t)((nx + TT - 1) / TT) * nrows);   // (column tiles) x rows
  if (blocks == 0) return;
  if (O.gacc) {
    pass2s_kernel<OP, TT, true><<<blocks, TT, pass2_smem_bytes(OP, acc, TT, true), st>>>(
        A, B, nx, row0, nrows, O.cbase, O.ncol, zlo, zhi, acc, O.stage, O.ocnt, O.flags, O.gacc);
    return;
  }
  const size_t smem = pass2_smem_bytes(OP, acc, TT);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(pass2s_kernel<OP, TT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  pass2s_kernel<OP, TT, false><<<blocks, TT, smem, st>>>(A, B, nx, row0, nrows, O.cbase, O.ncol, zlo, zhi, acc,
                                                         O.stage, O.ocnt, O.flags, nullptr);
}

// block size: 32 threads (one warp per block: measured fastest, C5 pass 2 36.6 ms at 128 threads,
// 35.0 at 64, 34.1 at 32); the accumulators of a block always fit
inline int pass2_block(int op, int acc) {
  int TT = 32;
  while (TT > 32 && pass2_smem_bytes(op, acc, TT) > P2_SMEM_MAX) TT >>= 1;
  return TT;
}

template <int OP>
void launch_pass2_op(const LevelSlots& A, const LevelSlots& B, int nx, int row0, int nrows, float zlo, float zhi,
                     const P2Out& O, cudaStream_t st) {
  const int TT = pass2_block(OP, O.acc);
  if (TT == 128) launch_pass2_t<OP, 128>(A, B, nx, row0, nrows, zlo, zhi, O, st);
  else if (TT == 64) launch_pass2_t<OP, 64>(A, B, nx, row0, nrows, zlo, zhi, O, st);
  else launch_pass2_t<OP, 32>(A, B, nx, row0, nrows, zlo, zhi, O, st);
}

void launch_pass2(int op, const LevelSlots& A, const LevelSlots& B, int nx, int row0, int nrows, float zlo,
                  float zhi, const P2Out& O, cudaStream_t st) {
  if (op == OP_DILATE) launch_pass2_op<OP_DILATE>(A, B, nx, row0, nrows, zlo, zhi, O, st);
  else if (op == OP_ERODE) launch_pass2_op<OP_ERODE>(A, B, nx, row0, nrows, zlo, zhi, O, st);
  else launch_pass2_op<OP_SHELL>(A, B, nx, row0, nrows, zlo, zhi, O, st);
}

bool same_geometry(const dexel_desc& a, const dexel_desc& b) {
  return a.nx == b.nx && a.ny == b.ny && a.spacing == b.spacing && a.z_lo == b.z_lo && a.z_hi == b.z_hi &&
         a.device == b.device && a.y0 == b.y0 && a.y1 == b.y1 && a.rank == b.rank && a.nranks == b.nranks;
}

void set_empty(dexel_grid g) {
  g->n = 0;
  if (!g->off.p) dalloc(g, g->off, sizeof(uint64_t) * (g->ncol + 1));
  if (g->off.p) cudaMemsetAsync(g->off.p, 0, sizeof(uint64_t) * (g->ncol + 1), g->stream);
  dfree(g, g->ep);
}

// ---------------------------------------------------------------- halo exchange (multi-GPU)
#define NK(call)                                                                                  \
  do {                                                                                            \
    ncclResult_t r_ = (call);                                                                     \
    if (r_ != ncclSuccess) return fail(DEXEL_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// the boundary slices a slab sends: rows [0, sr0) to rank g-1, rows [nrows - sr1, nrows) to g+1.
// hdr[2 s] = intervals of slice s, hdr[2 s + 1] = its first interval (the offset the receiver
// subtracts)
__global__ void halo_header(const uint64_t* __restrict__ off, int64_t c_lo, int64_t c_hi0, int64_t c_end,
                            uint64_t* __restrict__ hdr) {
  hdr[0] = off[c_lo];
  hdr[1] = 0;
  hdr[2] = off[c_end] - off[c_hi0];
  hdr[3] = off[c_hi0];
}

// received offsets (absolute in the sender's CSR) -> offsets of a CSR of their own
__global__ void halo_rebase(uint64_t* __restrict__ o, uint64_t n, const uint64_t* __restrict__ base_dev,
                            uint64_t base_host) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t b = base_dev ? *base_dev : base_host;
  if (t <= n) o[t] -= b;
}

enum { HALO_CALLER = 0, HALO_NCCL = 1, HALO_LOOP = 2 };
int halo_mode(const dexel_grid g) {
  if (g->d.nranks <= 1) return HALO_CALLER;
  if (g->d.nccl_comm) return HALO_NCCL;
  if (g->link[0] || g->link[1]) return HALO_LOOP;
  return HALO_CALLER;
}

dexel_status ensure_comm_stream(dexel_grid g) {
  if (!g->comm) CK(cudaStreamCreateWithFlags(&g->comm, cudaStreamNonBlocking));
  if (!g->ev_main) CK(cudaEventCreateWithFlags(&g->ev_main, cudaEventDisableTiming));
  if (!g->ev_halo) CK(cudaEventCreateWithFlags(&g->ev_halo, cudaEventDisableTiming));
  return DEXEL_OK;
}

// the exchange stream waits for everything queued on the handle's stream so far
dexel_status comm_after_main(dexel_grid g) {
  CK(cudaEventRecord(g->ev_main, g->stream));
  CK(cudaStreamWaitEvent(g->comm, g->ev_main, 0));
  return DEXEL_OK;
}

// a halo buffer of at least `bytes` (kept on the handle between ops; reallocated when too small or
// more than twice too large).  Allocated on the handle's stream: call comm_after_main afterwards.
dexel_status halo_buf(dexel_grid g, Buf& b, size_t bytes) {
  if (b.p && b.bytes >= bytes && b.bytes <= 2 * bytes + 4096) return DEXEL_OK;
  dfree(g, b);
  return dalloc(g, b, bytes);
}

// NCCL: every rank's slab rows, gathered once per handle; the partition must tile [0, ny) in
// rank order (every rank sees the same table, so every rank takes the same decisions below)
dexel_status nccl_partition(dexel_grid g) {
  if (!g->part.empty()) return DEXEL_OK;
  ncclComm_t comm = (ncclComm_t)g->d.nccl_comm;
  const int P = g->d.nranks;
  int cnt = 0, rk = -1;
  NK(ncclCommCount(comm, &cnt));
  NK(ncclCommUserRank(comm, &rk));
  if (cnt != P || rk != g->d.rank)
    return fail(DEXEL_EINVAL, "nccl_comm has " + std::to_string(cnt) + " ranks (this is rank " + std::to_string(rk) +
                                  "), the descriptor says rank " + std::to_string(g->d.rank) + " of " +
                                  std::to_string(P));
  Buf b;
  dexel_status s = dalloc(g, b, sizeof(int32_t) * 2 * (P + 1));
  if (s) return s;
  const int32_t mine[2] = {g->d.y0, g->d.y1};
  CK(cudaMemcpyAsync((int32_t*)b.p + 2 * P, mine, sizeof(mine), cudaMemcpyHostToDevice, g->stream));
  if ((s = ensure_comm_stream(g)) || (s = comm_after_main(g))) { dfree(g, b); return s; }
  NK(ncclAllGather((int32_t*)b.p + 2 * P, b.p, 2, ncclInt32, comm, g->comm));
  std::vector<int32_t> part(2 * P);
  CK(cudaMemcpyAsync(part.data(), b.p, sizeof(int32_t) * 2 * P, cudaMemcpyDeviceToHost, g->comm));
  CK(timed_sync(g->comm));
  ncclResult_t ae = ncclSuccess;
  ncclCommGetAsyncError(comm, &ae);
  if (ae != ncclSuccess) return fail(DEXEL_ENCCL, std::string("NCCL async error: ") + ncclGetErrorString(ae));
  CK(cudaEventRecord(g->ev_main, g->comm));   // the handle's stream may free b only after the gather
  CK(cudaStreamWaitEvent(g->stream, g->ev_main, 0));
  dfree(g, b);
  for (int q = 0; q < P; ++q) {
    const bool ok = part[2 * q] < part[2 * q + 1] && (q == 0 ? part[0] == 0 : part[2 * q] == part[2 * q - 1]) &&
                    (q + 1 < P || part[2 * q + 1] == g->d.ny);
    if (!ok)
      return fail(DEXEL_EINVAL, "the ranks' slabs [y0, y1) must tile [0, ny) in rank order (rank " + std::to_string(q) +
                                    " has [" + std::to_string(part[2 * q]) + ", " + std::to_string(part[2 * q + 1]) + "))");
  }
  g->part = part;
  return DEXEL_OK;
}

// Start the op's halo exchange (SURVEY 8(e) Option A): the R input rows beyond each
// slab boundary come from ranks g-1 / g+1 into g->hoff/hep, on the exchange stream; g->ev_halo
// marks their arrival (pass 1 of the halo rows waits on it, launch_rows_split).  Two phases,
// because rows are ragged: the interval counts (one host synchronisation: allocation sizes), then
// offsets and endpoints.  Sends read the slab's own CSR in place (contiguous row ranges).
dexel_status halo_begin(dexel_grid g, int R) {
  const int mode = halo_mode(g);
  const int nx = g->d.nx, ny = g->d.ny, y0 = g->d.y0, y1 = g->d.y1;
  const int need[2] = {std::min(R, y0), std::min(R, ny - y1)};
  dexel_status s;
  if ((s = ensure_comm_stream(g))) return s;
  uint64_t recv_n[2] = {0, 0};
  if (mode == HALO_NCCL) {
    if ((s = nccl_partition(g))) return s;
    const int P = g->d.nranks, me = g->d.rank;
    // rank q sends min(R, ny - y0_q) rows down and min(R, y1_q) rows up: both must lie in its slab
    for (int q = 0; q < P; ++q) {
      const int qy0 = g->part[2 * q], qy1 = g->part[2 * q + 1], rows = qy1 - qy0;
      if ((q > 0 && std::min(R, ny - qy0) > rows) || (q + 1 < P && std::min(R, qy1) > rows))
        return fail(DEXEL_EINVAL, "slab of rank " + std::to_string(q) + " has " + std::to_string(rows) +
                                      " rows < R = " + std::to_string(R) + ": its neighbours' halos would reach past it");
    }
    ncclComm_t comm = (ncclComm_t)g->d.nccl_comm;
    const int peer[2] = {me - 1, me + 1 < P ? me + 1 : -1};
    const int sr[2] = {peer[0] >= 0 ? std::min(R, ny - y0) : 0, peer[1] >= 0 ? std::min(R, y1) : 0};
    if ((s = halo_buf(g, g->hdr, 8 * sizeof(uint64_t)))) return s;
    uint64_t* hdr = (uint64_t*)g->hdr.p;
    if ((s = comm_after_main(g))) return s;
    halo_header<<<1, 1, 0, g->comm>>>((const uint64_t*)g->off.p, (int64_t)sr[0] * nx, (int64_t)(g->nrows - sr[1]) * nx,
                                      g->ncol, hdr);
    CK(cudaGetLastError());
    NK(ncclGroupStart());
    for (int q = 0; q < 2; ++q)
      if (peer[q] >= 0) {
        NK(ncclSend(hdr + 2 * q, 2, ncclUint64, peer[q], comm, g->comm));
        NK(ncclRecv(hdr + 4 + 2 * q, 2, ncclUint64, peer[q], comm, g->comm));
      }
    NK(ncclGroupEnd());
    uint64_t h[8];
    CK(cudaMemcpyAsync(g->pin, hdr, sizeof(h), cudaMemcpyDeviceToHost, g->comm));
    CK(timed_sync(g->comm));
    std::memcpy(h, g->pin, sizeof(h));
    ncclResult_t ae = ncclSuccess;
    ncclCommGetAsyncError(comm, &ae);
    if (ae != ncclSuccess) return fail(DEXEL_ENCCL, std::string("NCCL async error: ") + ncclGetErrorString(ae));
    for (int q = 0; q < 2; ++q) {
      recv_n[q] = peer[q] >= 0 ? h[4 + 2 * q] : 0;
      if (need[q] && ((s = halo_buf(g, g->hoff[q], sizeof(uint64_t) * ((size_t)need[q] * nx + 1))) ||
                      (s = halo_buf(g, g->hep[q], sizeof(float2) * (recv_n[q] + 1)))))
        return s;
    }
    if ((s = comm_after_main(g))) return s;   // (the allocations above are ordered on the handle's stream)
    NK(ncclGroupStart());
    for (int q = 0; q < 2; ++q) {
      if (peer[q] < 0) continue;
      const uint64_t* so = (const uint64_t*)g->off.p + (q == 0 ? 0 : (size_t)(g->nrows - sr[q]) * nx);
      NK(ncclSend(so, (size_t)sr[q] * nx + 1, ncclUint64, peer[q], comm, g->comm));
      if (h[2 * q]) NK(ncclSend((const float2*)g->ep.p + h[2 * q + 1], 2 * h[2 * q], ncclFloat32, peer[q], comm, g->comm));
      NK(ncclRecv(g->hoff[q].p, (size_t)need[q] * nx + 1, ncclUint64, peer[q], comm, g->comm));
      if (recv_n[q]) NK(ncclRecv(g->hep[q].p, 2 * recv_n[q], ncclFloat32, peer[q], comm, g->comm));
    }
    NK(ncclGroupEnd());
    for (int q = 0; q < 2; ++q)
      if (need[q]) {
        const uint64_t nc = (uint64_t)need[q] * nx;
        halo_rebase<<<(unsigned)((nc + 256) / 256), 256, 0, g->comm>>>((uint64_t*)g->hoff[q].p, nc, hdr + 5 + 2 * q, 0);
      }
    CK(cudaGetLastError());
  } else {   // HALO_LOOP: the neighbouring handles of this process
    for (int q = 0; q < 2; ++q) {
      if (!need[q]) continue;
      dexel_grid nb = g->link[q];
      if (!nb) return fail(DEXEL_EINVAL, "loopback slab: no linked neighbour on side " + std::to_string(q));
      if (nb->nrows < need[q])
        return fail(DEXEL_EINVAL, "neighbouring slab has " + std::to_string(nb->nrows) + " rows < R = " + std::to_string(R));
      const int64_t c0 = q == 0 ? (int64_t)(nb->nrows - need[q]) * nx : 0, nc = (int64_t)need[q] * nx;
      uint64_t ab[2];
      CK(cudaStreamSynchronize(nb->stream));   // (its contents are final: ops are not re-entrant)
      CK(cudaMemcpy(&ab[0], (const uint64_t*)nb->off.p + c0, 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&ab[1], (const uint64_t*)nb->off.p + c0 + nc, 8, cudaMemcpyDeviceToHost));
      recv_n[q] = ab[1] - ab[0];
      if ((s = halo_buf(g, g->hoff[q], sizeof(uint64_t) * (nc + 1))) ||
          (s = halo_buf(g, g->hep[q], sizeof(float2) * (recv_n[q] + 1))))
        return s;
      if ((s = comm_after_main(g))) return s;
      CK(cudaMemcpyAsync(g->hoff[q].p, (const uint64_t*)nb->off.p + c0, sizeof(uint64_t) * (nc + 1), cudaMemcpyDefault,
                         g->comm));
      if (recv_n[q])
        CK(cudaMemcpyAsync(g->hep[q].p, (const float2*)nb->ep.p + ab[0], sizeof(float2) * recv_n[q],
                           cudaMemcpyDefault, g->comm));
      halo_rebase<<<(unsigned)((nc + 256) / 256), 256, 0, g->comm>>>((uint64_t*)g->hoff[q].p, (uint64_t)nc, nullptr, ab[0]);
      CK(cudaGetLastError());
    }
  }
  CK(cudaEventRecord(g->ev_halo, g->comm));
  g->halo_pending = true;
  for (int q = 0; q < 2; ++q) {
    g->hrows[q] = need[q];
    g->hn[q] = recv_n[q];
  }
  return DEXEL_OK;
}

// the handle's stream waits for an exchange still in flight (before any later free or reuse of the
// halo buffers on that stream)
void halo_end(dexel_grid g) {
  if (g->halo_pending) cudaStreamWaitEvent(g->stream, g->ev_halo, 0);
  g->halo_pending = false;
}

dexel_status run_op_impl(int op, dexel_grid src, float r_a, float r_b, dexel_grid dst, bool slices) {
  const double op_t0 = now_s();
  g_t_alloc = g_t_sync = g_t_free = g_t_info = 0.0;
  if (!src || !dst) return fail(DEXEL_EINVAL, "NULL handle");
  if (src == dst) return fail(DEXEL_EINVAL, "src and dst must be different handles");
  if (!same_geometry(src->d, dst->d)) return fail(DEXEL_EMISMATCH, "src and dst geometry differ");
  int Ra, Rb;
  dexel_status s;
  if ((s = check_radius(r_a, src->d.spacing, &Ra))) return s;
  if ((s = check_radius(r_b, src->d.spacing, &Rb))) return s;
  CK(cudaSetDevice(src->d.device));
  cudaStream_t st = src->stream;
  if (dst->stream != st) {  // order dst's stream after src's
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, dst->stream));
    CK(cudaStreamWaitEvent(st, ev, 0));
    cudaEventDestroy(ev);
  }
  dexel_stats stats{};
  Temps T(src, &stats);
  // halo rows (y-slabs): the op reads rows [y0 - hlo, y1 + hhi) and writes [y0, y1).
  // Slices (2D offsets of every row on its own) reach no other row: no halo, no band overlap.
  const int Rmax = slices ? 0 : (Ra > Rb ? Ra : Rb);
  const int need_lo = src->d.y0 < Rmax ? src->d.y0 : Rmax;
  const int need_hi = src->d.ny - src->d.y1 < Rmax ? src->d.ny - src->d.y1 : Rmax;
  const int hmode = halo_mode(src);
  int hlo = 0, hhi = 0;
  if (hmode != HALO_CALLER) {   // the library exchanges the halo rows itself (NCCL or loopback)
    if (Rmax > 0 && (s = halo_begin(src, Rmax))) return s;
    hlo = need_lo;
    hhi = need_hi;
  } else {
    if (src->hrows[0] < need_lo || src->hrows[1] < need_hi)
      return fail(DEXEL_EINVAL, "slab halo too small: need " + std::to_string(need_lo) + " rows below and " +
                                    std::to_string(need_hi) + " above (dexel_upload_halo)");
    hlo = slices ? 0 : src->hrows[0];
    hhi = slices ? 0 : src->hrows[1];
  }
  const int nrows_ext = hlo + src->nrows + hhi;
  SrcRows rows{{(const uint64_t*)src->hoff[0].p, (const uint64_t*)src->off.p, (const uint64_t*)src->hoff[1].p},
               {(const float*)src->hep[0].p, (const float*)src->ep.p, (const float*)src->hep[1].p},
               {hlo, src->nrows, hhi},
               src->d.nx, nrows_ext, src->d.z_lo, src->d.z_hi};
  stats.n_in = src->n;
  // h(kappa, k) tables, one per family radius
  float* htab_a = nullptr;
  float* htab_b = nullptr;
  float* prune_a = nullptr;
  float* prune_b = nullptr;
  if ((s = make_htab(src, T, r_a, Ra, &htab_a, &prune_a))) return s;
  if (op == OP_SHELL && (s = make_htab(src, T, r_b, Rb, &htab_b, &prune_b))) return s;
  // ---- row bands: level slots of (band + R-row halo) rows, then pass 2 of the band
  const int64_t ncol = src->ncol;
  const int nx = src->d.nx;
  const int nfam = op == OP_SHELL ? 2 : 1;
  int lcap = src->lev_cap > 0 ? src->lev_cap : 8;
  // the shell's two pass-1 families in one sweep (pass1.cuh, FAMS = 3) when they share R
  // (DEXEL_NO_FUSE=1 runs them separately, for testing)
  static const bool no_fuse = [] { const char* e = std::getenv("DEXEL_NO_FUSE"); return e && std::atoi(e); }();
  const bool fused = op == OP_SHELL && Ra == Rb && (prune_a != nullptr) == (prune_b != nullptr) && !no_fuse;
  // bytes per level row of a band: level slots of all families + the piece slots alive at once
  // (one family's, or both when fused)
  const int pcap = src->p1_cap > 0 ? src->p1_cap : 256;
  size_t row_bytes = (size_t)nx * ((size_t)(pcap / 4 + 1) * 36 + 8) * (fused ? 2 : 1);
  for (int f = 0; f < nfam; ++f) {
    const int Rf = f == 0 ? Ra : Rb;
    row_bytes += (size_t)nx * ((Rf + 1) * sizeof(uint16_t) + (Rf + 2) * sizeof(float2) * (size_t)(lcap + LV_CLAMP));
  }
  // slots of one band (pieces + level sets, all families): fewer, taller bands recompute fewer
  // halo rows (2R per band); the budget leaves room for the output staging and the caller
  size_t budget = (size_t)64 << 30;
  // a grid whose whole extended slot set is small (under 1 GiB) is one band without asking the
  // driver (cudaMemGetInfo costs 0.2-1.5 ms, a large share of a small op)
  const size_t whole = row_bytes * (size_t)(src->nrows + 2 * Rmax);
  if (whole > ((size_t)1 << 30) && dev_ws(src->d.device).band_budget) {
    budget = dev_ws(src->d.device).band_budget;
  } else if (whole > ((size_t)1 << 30)) {
    // free device memory plus what the stream-ordered pool holds but does not use (freed
    // temporaries of earlier ops stay reserved: the release threshold is kept at max)
    size_t fr = 0, tot = 0;
    const double ti = now_s();
    struct Acc { double t0; ~Acc() { g_t_info += now_s() - t0; } } acc_{ti};
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
      size_t pooled = 0;
      cudaMemPool_t pool;
      if (!g_alloc && cudaDeviceGetDefaultMemPool(&pool, src->d.device) == cudaSuccess) {
        uint64_t res = 0, used = 0;
        if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && res > used)
          pooled = (size_t)(res - used);
      }
      budget = std::min(budget, (fr + pooled) / 2);
    }
    dev_ws(src->d.device).band_budget = budget;
  }
  int band = (int)std::max<int64_t>(64, (int64_t)(budget / std::max<size_t>(row_bytes, 1)) - 2 * Rmax);
  if (const char* e = std::getenv("DEXEL_BAND_ROWS")) band = std::max(1, std::atoi(e));   // testing override
  band = std::min(band, src->nrows);
  {   // equal bands: every band's slot arrays then fit the blocks the first band allocated
    const int nb = (src->nrows + band - 1) / band;
    band = (src->nrows + nb - 1) / nb;
  }
  uint32_t* ocnt = nullptr;
  unsigned* opf = nullptr;   // the op's flag words and statistics (kernels.cuh OpFlag)
  if ((s = T.get(sizeof(uint32_t) * (ncol + 1), (void**)&ocnt))) return s;
  // the op's flag words, then the output scan's look-back status words: one memset per attempt
  const size_t opf_bytes = sizeof(unsigned) * OPF_WORDS + sizeof(unsigned long long) * scan_status_words((uint64_t)ncol);
  if ((s = T.get(opf_bytes, (void**)&opf))) return s;
  int acc = src->p2_acc > 0 ? src->p2_acc : 32;
  static const bool no_acc_fit = std::getenv("DEXEL_P2_ACC") != nullptr || std::getenv("DEXEL_P2_NOFIT") != nullptr;
  float2* stage = nullptr;
  // Every capacity of the op (piece slots and arena, level slots and arena, the pass-2
  // accumulator, dst's buffer) is checked ONCE, at the end: kernels raise flags instead of the
  // host reading sizes back after every launch.  The one readback (flags + statistics + the
  // output size) then either confirms the op or grows what overflowed and reruns it.
  for (int attempt = 0;; ++attempt) {
    const int nb = (src->nrows + band - 1) / band;
    if ((s = T.get(sizeof(float2) * (size_t)pass2_stage_cap(op, acc) * ncol + 16, (void**)&stage))) return s;
    // unions longer than a shared-memory accumulator holds: a global one for the band's columns
    float2* gacc = nullptr;
    if (pass2_smem_bytes(op, acc, 32) > P2_SMEM_MAX &&
        (s = T.get(sizeof(float2) * (size_t)(acc + 2) * band * nx + 16, (void**)&gacc)))
      return s;
    CK(cudaMemsetAsync(opf, 0, opf_bytes, st));
    uint32_t lev_cap_used = 0;
    for (int b0 = 0; b0 < src->nrows; b0 += band) {
      const int b1 = std::min(src->nrows, b0 + band);
      const int lr0 = std::max(0, hlo + b0 - Rmax), lr1 = std::min(nrows_ext, hlo + b1 + Rmax);
      LevelSlots LA{}, LB{};
      PieceSlots PA{}, PB{};
      if (fused && (s = run_pass1_dual(src, T, rows, Ra, lr0, lr1 - lr0, opf, &PA, &PB, prune_a, prune_b))) return s;
      // family A: S (dilate, shell r_out) or C = U \ S (erode); family B: C at r_in (shell)
      if ((s = run_levels(src, T, rows, Ra, htab_a, prune_a, op == OP_ERODE ? 1 : 0, lr0, lr1 - lr0, opf, &LA,
                          fused ? &PA : nullptr, slices)))
        return s;
      if (op == OP_SHELL) {
        if ((s = run_levels(src, T, rows, Rb, htab_b, prune_b, 1, lr0, lr1 - lr0, opf, &LB, fused ? &PB : nullptr,
                            slices)))
          return s;
      } else {
        LB = LA;
      }
      lev_cap_used = std::max<uint32_t>(lev_cap_used, std::max(LA.cap, LB.cap) - (LV_CLAMP - 1));
      const P2Out O{(int64_t)b0 * nx, ncol, acc, stage, ocnt, opf, gacc};
      LAUNCH(T, K_P2, launch_pass2(op, LA, LB, nx, hlo + b0, b1 - b0, src->d.z_lo, src->d.z_hi, O, st));
      CK(cudaGetLastError());
      for (LevelSlots* Lf : {&LA, &LB}) {
        if (Lf == &LB && op != OP_SHELL) break;
        T.release(Lf->z);
        T.release(Lf->cnt);
        T.release(Lf->ovf_idx);
        if (Lf->ovf_z) T.release(Lf->ovf_z);
      }
    }
    if (gacc) T.release(gacc);
    // output offsets (scan of the staged counts) and the compaction into dst's current buffer
    // (when the total fits it: the kernel checks on the device)
    dst->n = 0;   // (from here on dst is being replaced: an error leaves it empty, run_op)
    if (!dst->off.p && (s = dalloc(dst, dst->off, sizeof(uint64_t) * (dst->ncol + 1)))) return s;
    if ((s = scan_counts_dev(src, T, ocnt, (uint64_t)ncol, (uint64_t*)dst->off.p,
                             reinterpret_cast<unsigned long long*>(opf + OPF_WORDS))))
      return s;
    if (!dst->ep.p && (s = dalloc(dst, dst->ep, sizeof(float2) * (size_t)(2 * src->n + 1024)))) return s;
    const uint64_t ep_cap = dst->ep.bytes / sizeof(float2);
    if (ncol > 0)
      LAUNCH(T, K_COMPACT, compact_kernel<<<(unsigned)((ncol + 255) / 256), 256, 0, st>>>(
                               stage, ocnt, (const uint64_t*)dst->off.p, ncol, (float2*)dst->ep.p, ep_cap, opf));
    CK(cudaGetLastError());
    // ---- the op's one readback
    unsigned hf[OPF_WORDS];
    uint64_t nout = 0;
    {
      Readback rb{src};
      rb.add(0, opf, sizeof(hf));
      rb.add(sizeof(hf), (const uint64_t*)dst->off.p + ncol, sizeof(nout));
      CK(rb.wait());
      rb.get(0, hf, sizeof(hf));
      rb.get(sizeof(hf), &nout, sizeof(nout));
    }
    const bool p1_over = hf[OPF_P1_RERUN] != 0, lv_over = hf[OPF_LV_RERUN] != 0;
    const unsigned need = hf[OPF_P2_ACC];
    if (!p1_over && !lv_over && need == 0) {
      if (hf[OPF_OUT_FIT]) {   // the output outgrew dst's buffer: the exact size, compact again
        dfree(dst, dst->ep);
        if ((s = dalloc(dst, dst->ep, sizeof(float2) * (nout + 1)))) return s;
        CK(cudaMemsetAsync(opf + OPF_OUT_FIT, 0, sizeof(unsigned), st));
        if (ncol > 0)
          LAUNCH(T, K_COMPACT, compact_kernel<<<(unsigned)((ncol + 255) / 256), 256, 0, st>>>(
                                   stage, ocnt, (const uint64_t*)dst->off.p, ncol, (float2*)dst->ep.p, nout, opf));
        CK(cudaGetLastError());
      }
      uint64_t st64[2];
      std::memcpy(st64, hf + 8, sizeof(st64));
      stats.n_mid = st64[0];
      stats.n_lev = st64[1];
      stats.n_out = nout;
      stats.bands = (uint32_t)nb;
      stats.p2_acc = acc;
      stats.lev_cap = lev_cap_used;
      dst->n = nout;
      // size the next ops' accumulator by the longest union any op on this handle has held (rounded
      // up to a multiple of 4): a shorter accumulator is less shared memory per warp, so more resident
      // warps for the latency-bound pass 2 (measured, profiles/r02_p2_acc_times.txt: C5 needs 17-20
      // entries; 32 -> 20 runs the op 133.0 -> 127.1 ms, C4 r=16 11.35 -> 10.88).  The handle's
      // maximum, not the last op's: alternating ops do not rerun each other.
      if (acc <= (int)(P2_SMEM_MAX / (32 * sizeof(float2))) - 2 * P2_R - 2 && !no_acc_fit) {
        src->p2_peak = std::max(src->p2_peak, (int)hf[OPF_P2_PEAK]);
        src->p2_acc = std::max(8, (src->p2_peak + 3) / 4 * 4);
      }
      break;
    }
    // something overflowed: grow it (kept on the handle for later ops) and rerun the op.  Only the
    // earliest stage that overflowed is trusted: later stages ran on incomplete input.
    if (attempt >= 24) return fail(DEXEL_ECUDA, "op capacity sizing did not converge");
    if (p1_over) {
      int cap = src->p1_cap > 0 ? (src->p1_cap + 3) / 4 * 4 : 256;
      while (cap < 1 << 15 && (unsigned)cap * 2 < hf[OPF_P1_LONGEST]) cap *= 2;
      src->p1_cap = std::min(1 << 15, cap * 2);
    }
    if (lv_over && !p1_over) {
      const int cap = src->lev_cap > 0 ? src->lev_cap : 8;
      if (cap >= LV_SLOT_MAX && hf[OPF_LV_LONGEST] > (unsigned)LV_CNT_MAX)
        return fail(DEXEL_EOVERFLOW, "a column has a level list of more than " + std::to_string(LV_CNT_MAX) +
                                         " intervals (counted in 15 bits)");
      src->lev_cap = std::min(LV_SLOT_MAX, 2 * cap);
      if (cap >= LV_SLOT_MAX) {   // slots at their largest: grow the arena lists
        const int ac = std::min(LV_CNT_MAX, std::max({32, 4 * cap, src->lev_arena}));
        if (ac >= LV_CNT_MAX)
          return fail(DEXEL_EOVERFLOW, "level lists outgrow the largest slot capacity and arena");
        src->lev_arena = std::min(LV_CNT_MAX, std::max<int>(2 * ac, (int)std::min<unsigned>(hf[OPF_LV_LONGEST], LV_CNT_MAX)));
      }
    }
    if (need && !p1_over && !lv_over) {   // a pass-2 union outgrew the accumulator
      int nacc = acc;
      while (nacc < (int)need) nacc *= 2;
      // (beyond P2_SMEM_MAX the accumulator moves to global memory: slower, any length)
      acc = nacc;
      // (the handle keeps at most the largest shared-memory accumulator: one pathological op does
      // not send later ops to the global one)
      src->p2_acc = std::min(acc, (int)(P2_SMEM_MAX / (32 * sizeof(float2))) - 2 * P2_R - 2);
    }
    T.release(stage);
  }
  T.prof.finish();
  if (dst->stream != st) {
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, st));
    CK(cudaStreamWaitEvent(dst->stream, ev, 0));
    cudaEventDestroy(ev);
  }
  dst->stats = stats;
  src->stats = stats;
  if (std::getenv("DEXEL_DEBUG")) {
    CK(timed_sync(st));
    std::fprintf(stderr, "[dexel] op wall %.2f ms: allocation calls %.2f ms, frees %.2f ms, memory queries %.2f ms, "
                 "stream syncs %.2f ms\n", 1e3 * (now_s() - op_t0), 1e3 * g_t_alloc, 1e3 * g_t_free,
                 1e3 * g_t_info, 1e3 * g_t_sync);
  }
  return DEXEL_OK;
}

// an op that ran out of device memory drops the cached band budget (the next op re-queries)
dexel_status run_op(int op, dexel_grid src, float r_a, float r_b, dexel_grid dst, bool slices = false) {
  const dexel_status s = run_op_impl(op, src, r_a, r_b, dst, slices);
  if (src) halo_end(src);
  if (s == DEXEL_ENOMEM && src) dev_ws(src->d.device).band_budget = 0;
  // dst is replaced; on any error it is left empty, never partially written (dexel.h).  (src == dst
  // and NULL handles are rejected before anything is touched and leave both as they were.)
  if (s != DEXEL_OK && dst && dst != src) {
    const std::string msg = g_err;
    set_empty(dst);
    g_err = msg;
  }
  return s;
}

// Load every kernel's code now: with CUDA's lazy module loading a kernel is loaded at its first
// launch, which needs device memory -- and an op's workspace may hold most of it by then (a big
// op failed its first levels launch with "out of memory").  Once per device, at handle creation.
template <class K>
void preload_one(K* fn) {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, (const void*)fn);
}
template <int F>
void preload_p1() {
  preload_one(p1g_kernel<1, F>);
  preload_one(p1g_kernel<2, F>);
  preload_one(p1g_kernel<3, F>);
  preload_one(p1g_kernel<4, F>);
  preload_one(p1s_kernel<2, F, true, 0>);
  preload_one(p1s_kernel<2, F, true, 1>);
  preload_one(p1s_kernel<3, F, false, 1>);
  preload_one(p1s_kernel<5, F, false, 1>);
  preload_one(p1s_kernel<9, F, false, 1>);
  preload_one(p1s_kernel<17, F, false, 1>);
}
template <int OP>
void preload_p2() {
  preload_one(pass2s_kernel<OP, 32, false>);
  preload_one(pass2s_kernel<OP, 64, false>);
  preload_one(pass2s_kernel<OP, 128, false>);
  preload_one(pass2s_kernel<OP, 32, true>);
}
void preload_kernels(int device) {
  static bool done[64] = {false};
  if (device < 0 || device >= 64 || done[device]) return;
  done[device] = true;
  preload_p1<1>();
  preload_p1<2>();
  preload_p1<3>();
  preload_one(levels_kernel<2>);
  preload_one(levels_kernel<3>);
  preload_one(levels_kernel<4>);
  preload_one(levels_kernel<5>);
  preload_one(levels_kernel<6>);
  preload_one(levels_kernel<8>);
  preload_one(levels_kernel<10>);
  preload_one(levels_kernel<12>);
  preload_one(levels_kernel<14>);
  preload_one(levels_kernel<17>);
  preload_p2<OP_DILATE>();
  preload_p2<OP_ERODE>();
  preload_p2<OP_SHELL>();
  preload_one(compact_kernel);
  preload_one(scan_tile_sums);
  preload_one(scan_sums_exclusive);
  preload_one(scan_tiles_write);
  preload_one(validate_kernel);
  preload_one(rebase_offsets);
  preload_one(halo_header);
  preload_one(halo_rebase);
  preload_one(pieces_to_csr);
  preload_one(raster_bin_count);
  preload_one(raster_bin_fill);
  preload_one(raster_kernel<RS_CAP>);
  preload_one(raster_kernel<RS_CAP_BIG>);
  cudaGetLastError();
}

}  // namespace

// ================================================================ C ABI
extern "C" {

const char* dexel_last_error(void) { return g_err.c_str(); }

dexel_status dexel_set_allocator(dexel_alloc_fn alloc, dexel_free_fn free_, void* ctx) {
  if ((alloc == nullptr) != (free_ == nullptr)) return fail(DEXEL_EINVAL, "allocator: both or neither");
  g_alloc = alloc;
  g_free = free_;
  g_alloc_ctx = ctx;
  return DEXEL_OK;
}

dexel_status dexel_create(const dexel_desc* d, dexel_grid* out) {
  g_err.clear();
  if (!d || !out) return fail(DEXEL_EINVAL, "NULL argument");
  if (d->nx < 1 || d->ny < 1) return fail(DEXEL_EINVAL, "nx, ny must be >= 1");
  if (!(d->spacing > 0) || !std::isfinite(d->spacing)) return fail(DEXEL_EINVAL, "spacing must be finite and > 0");
  if (!std::isfinite(d->z_lo) || !std::isfinite(d->z_hi) || !(d->z_lo < d->z_hi))
    return fail(DEXEL_EINVAL, "domain must be finite with z_lo < z_hi");
  if (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks) return fail(DEXEL_EINVAL, "bad rank/nranks");
  if (d->y0 < 0 || d->y1 > d->ny || d->y0 >= d->y1) return fail(DEXEL_EINVAL, "bad slab rows [y0,y1)");
  if (d->nranks == 1 && (d->y0 != 0 || d->y1 != d->ny)) return fail(DEXEL_EINVAL, "single rank must own all rows");
  CK(cudaSetDevice(d->device));
  preload_kernels(d->device);
  {
    // keep freed pool memory mapped: ops allocate and free tens of GB per call
    static bool pool_set[64] = {false};
    if (d->device >= 0 && d->device < 64 && !pool_set[d->device]) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, d->device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      pool_set[d->device] = true;
    }
  }
  dexel_grid g = new dexel_grid_s();
  g->d = *d;
  // initial capacity hints (testing / tuning overrides; grown automatically on overflow)
  if (const char* e = std::getenv("DEXEL_LEV_CAP")) g->lev_cap = std::max(1, std::min(255, std::atoi(e)));
  if (const char* e = std::getenv("DEXEL_P2_ACC")) g->p2_acc = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("DEXEL_P1_CAP")) g->p1_cap = std::max(1, std::atoi(e));
  g->nrows = d->y1 - d->y0;
  g->ncol = (int64_t)g->nrows * d->nx;
  if (d->stream) {
    g->stream = (cudaStream_t)d->stream;
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete g;
      return fail(DEXEL_ECUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    g->own_stream = true;
  }
  if (cudaMallocHost((void**)&g->pin, 256) != cudaSuccess) {
    if (g->own_stream) cudaStreamDestroy(g->stream);
    delete g;
    return fail(DEXEL_ENOMEM, "cudaMallocHost (256 B readback buffer) failed");
  }
  dexel_status s = dalloc(g, g->off, sizeof(uint64_t) * (g->ncol + 1));
  if (s) {
    cudaFreeHost(g->pin);
    delete g;
    return s;
  }
  CK(cudaMemsetAsync(g->off.p, 0, sizeof(uint64_t) * (g->ncol + 1), g->stream));
  {
    DevWs& W = dev_ws(g->d.device);
    std::lock_guard<std::mutex> lk(W.mu);
    ++W.handles;
  }
  *out = g;
  return DEXEL_OK;
}

}  // extern "C"

namespace {
// copy + validate a CSR of ncol columns into fresh buffers (grid unchanged on error)
// b := the spare buffer if it holds bytes (and at most 1/4 more), else a new allocation
dexel_status take_or_alloc(dexel_grid g, Buf* spare, Buf& b, size_t bytes) {
  if (spare && spare->p && spare->bytes >= bytes && spare->bytes - bytes <= bytes / 4) {
    b = *spare;
    *spare = Buf{};
    return DEXEL_OK;
  }
  return dalloc(g, b, bytes);
}

dexel_status load_csr(dexel_grid g, const uint64_t* offsets, const float* endpoints, int64_t ncol, uint64_t n,
                      int on_dev, Buf* off_out, Buf* ep_out, Buf* spare_off = nullptr, Buf* spare_ep = nullptr,
                      bool sliced = false) {
  if (!offsets || (n > 0 && !endpoints)) return fail(DEXEL_EINVAL, "NULL argument");
  CK(cudaSetDevice(g->d.device));
  uint64_t first = 0, last = 0;
  if (on_dev) {
    CK(cudaMemcpyAsync(&first, offsets, 8, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaMemcpyAsync(&last, offsets + ncol, 8, cudaMemcpyDeviceToHost, g->stream));
    CK(timed_sync(g->stream));
  } else {
    first = offsets[0];
    last = offsets[ncol];
  }
  // sliced (dexel_pipe_run): the rows are a slice of a larger CSR -- offsets[0] = b, `endpoints` points at
  // interval b, and the device copy of the offsets is rebased to 0 before validation
  if (sliced ? (last < first || last - first != n) : (first != 0 || last != n))
    return fail(DEXEL_EINVAL, "offsets[0] must be 0 and offsets[ncols] == n_intervals");
  Buf off, ep;
  dexel_status s;
  if ((s = take_or_alloc(g, spare_off, off, sizeof(uint64_t) * (ncol + 1)))) return s;
  if ((s = take_or_alloc(g, spare_ep, ep, sizeof(float) * 2 * (n + 1)))) {
    dfree(g, off);
    return s;
  }
  const cudaMemcpyKind k = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CK(cudaMemcpyAsync(off.p, offsets, sizeof(uint64_t) * (ncol + 1), k, g->stream));
  if (n) CK(cudaMemcpyAsync(ep.p, endpoints, sizeof(float) * 2 * n, k, g->stream));
  if (sliced && first != 0)
    rebase_kernel<<<(unsigned)((ncol + 1 + 255) / 256), 256, 0, g->stream>>>((uint64_t*)off.p, ncol + 1, first);
  Temps T(g);
  unsigned long long* bad = nullptr;
  if ((s = T.get(sizeof(unsigned long long), (void**)&bad))) {
    dfree(g, off);
    dfree(g, ep);
    return s;
  }
  CK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), g->stream));
  if (ncol > 0)
    validate_kernel<<<(unsigned)((ncol + 255) / 256), 256, 0, g->stream>>>((const uint64_t*)off.p,
                                                                             (const float*)ep.p, ncol, g->d.z_lo,
                                                                             g->d.z_hi, bad);
  CK(cudaGetLastError());
  unsigned long long hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, g->stream));
  CK(timed_sync(g->stream));
  if (hbad != ~0ull) {
    dfree(g, off);
    dfree(g, ep);
    const int64_t c = (int64_t)hbad;
    return fail(DEXEL_EINVAL, "invalid column " + std::to_string(c) + " (i=" + std::to_string(c % g->d.nx) +
                                  ", local row " + std::to_string(c / g->d.nx) +
                                  "): intervals must be finite, strictly increasing and inside [z_lo, z_hi]");
  }
  *off_out = off;
  *ep_out = ep;
  return DEXEL_OK;
}
}  // namespace

extern "C" {

static dexel_status upload_impl(dexel_grid g, const uint64_t* offsets, const float* endpoints, uint64_t n, int on_dev,
                                bool sliced);
static dexel_status upload_halo_impl(dexel_grid g, int side, const uint64_t* offsets, const float* endpoints,
                                     int nrows, uint64_t n, int on_dev, bool sliced);

dexel_status dexel_upload(dexel_grid g, const uint64_t* offsets, const float* endpoints, uint64_t n, int on_dev) {
  return upload_impl(g, offsets, endpoints, n, on_dev, false);
}

static dexel_status upload_impl(dexel_grid g, const uint64_t* offsets, const float* endpoints, uint64_t n, int on_dev,
                                bool sliced) {
  g_err.clear();
  if (!g) return fail(DEXEL_EINVAL, "NULL handle");
  static const bool dbg = std::getenv("DEXEL_DEBUG") != nullptr;
  const double t0 = now_s();
  g_t_alloc = g_t_sync = 0.0;
  Buf off, ep;
  dexel_status s = load_csr(g, offsets, endpoints, g->ncol, n, on_dev, &off, &ep, &g->spare_off, &g->spare_ep,
                            sliced);
  if (s) return s;
  if (dbg)
    std::fprintf(stderr, "[dexel] upload %llu intervals: %.2f ms (allocation calls %.2f ms, stream syncs %.2f ms)\n",
                 (unsigned long long)n, 1e3 * (now_s() - t0), 1e3 * g_t_alloc, 1e3 * g_t_sync);
  // the previous contents become the spare (a larger spare from before is released)
  dfree(g, g->spare_off);
  dfree(g, g->spare_ep);
  g->spare_off = g->off;
  g->spare_ep = g->ep;
  g->off = off;
  g->ep = ep;
  g->n = n;
  return DEXEL_OK;
}

dexel_status dexel_upload_halo(dexel_grid g, int side, const uint64_t* offsets, const float* endpoints, int nrows,
                               uint64_t n, int on_dev) {
  return upload_halo_impl(g, side, offsets, endpoints, nrows, n, on_dev, false);
}

static dexel_status upload_halo_impl(dexel_grid g, int side, const uint64_t* offsets, const float* endpoints,
                                     int nrows, uint64_t n, int on_dev, bool sliced) {
  g_err.clear();
  if (!g || (side != 0 && side != 1) || nrows < 0) return fail(DEXEL_EINVAL, "bad halo arguments");
  const int avail = side == 0 ? g->d.y0 : g->d.ny - g->d.y1;
  if (nrows > avail) return fail(DEXEL_EINVAL, "halo extends past the grid");
  dfree(g, g->hoff[side]);
  dfree(g, g->hep[side]);
  g->hrows[side] = 0;
  g->hn[side] = 0;
  if (nrows == 0) return DEXEL_OK;
  Buf off, ep;
  dexel_status s = load_csr(g, offsets, endpoints, (int64_t)nrows * g->d.nx, n, on_dev, &off, &ep, nullptr, nullptr,
                            sliced);
  if (s) return s;
  g->hoff[side] = off;
  g->hep[side] = ep;
  g->hrows[side] = nrows;
  g->hn[side] = n;
  return DEXEL_OK;
}

dexel_status dexel_download_rows(dexel_grid g, int row_begin, int nrows, uint64_t* offsets, float* endpoints,
                                 uint64_t cap, uint64_t* n_out, int on_dev) {
  g_err.clear();
  if (!g || !n_out || row_begin < 0 || nrows < 0 || row_begin + nrows > g->nrows)
    return fail(DEXEL_EINVAL, "bad row range");
  CK(cudaSetDevice(g->d.device));
  const int64_t c0 = (int64_t)row_begin * g->d.nx, nc = (int64_t)nrows * g->d.nx;
  uint64_t ab[2] = {0, 0};
  CK(cudaMemcpyAsync(&ab[0], (uint64_t*)g->off.p + c0, 8, cudaMemcpyDeviceToHost, g->stream));
  CK(cudaMemcpyAsync(&ab[1], (uint64_t*)g->off.p + c0 + nc, 8, cudaMemcpyDeviceToHost, g->stream));
  CK(timed_sync(g->stream));
  const uint64_t n = ab[1] - ab[0];
  *n_out = n;
  if (!offsets) return DEXEL_OK;   // size query
  if (cap < n) return fail(DEXEL_EOVERFLOW, "capacity < intervals in the rows");
  if (!offsets || (n && !endpoints)) return fail(DEXEL_EINVAL, "NULL output buffer");
  Temps T(g);
  uint64_t* tmp = nullptr;
  dexel_status s;
  if (on_dev) {
    tmp = offsets;
  } else if ((s = T.get(sizeof(uint64_t) * (nc + 1), (void**)&tmp))) {
    return s;
  }
  rebase_offsets<<<(unsigned)((nc + 256) / 256), 256, 0, g->stream>>>((const uint64_t*)g->off.p + c0, (uint64_t)nc,
                                                                       0, tmp);
  CK(cudaGetLastError());
  const cudaMemcpyKind k = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (!on_dev) CK(cudaMemcpyAsync(offsets, tmp, sizeof(uint64_t) * (nc + 1), k, g->stream));
  if (n) CK(cudaMemcpyAsync(endpoints, (const float2*)g->ep.p + ab[0], sizeof(float2) * n, k, g->stream));
  CK(timed_sync(g->stream));
  return DEXEL_OK;
}

dexel_status dexel_dilate(dexel_grid src, float r, dexel_grid dst) {
  g_err.clear();
  return run_op(OP_DILATE, src, r, r, dst);
}

dexel_status dexel_erode(dexel_grid src, float r, dexel_grid dst) {
  g_err.clear();
  return run_op(OP_ERODE, src, r, r, dst);
}

dexel_status dexel_shell(dexel_grid src, float r_out, float r_in, dexel_grid dst) {
  g_err.clear();
  return run_op(OP_SHELL, src, r_out, r_in, dst);
}

dexel_status dexel_dilate_slices(dexel_grid src, float r, dexel_grid dst) {
  g_err.clear();
  return run_op(OP_DILATE, src, r, r, dst, true);
}

dexel_status dexel_erode_slices(dexel_grid src, float r, dexel_grid dst) {
  g_err.clear();
  return run_op(OP_ERODE, src, r, r, dst, true);
}

dexel_status dexel_shell_slices(dexel_grid src, float r_out, float r_in, dexel_grid dst) {
  g_err.clear();
  return run_op(OP_SHELL, src, r_out, r_in, dst, true);
}

}  // extern "C"

namespace {
// morphological compositions: first op into a
// temporary handle of the same geometry, second op from it into dst
dexel_status compose(int op1, int op2, dexel_grid src, float r, dexel_grid dst) {
  if (!src || !dst) return fail(DEXEL_EINVAL, "NULL handle");
  if (src == dst) return fail(DEXEL_EINVAL, "src and dst must be different handles");
  if (src->d.nranks > 1 && !src->d.nccl_comm)
    return fail(DEXEL_EINVAL, "opening/closing of a y-slab needs the intermediate's halo rows: give the slabs an "
                              "NCCL communicator (the intermediate is exchanged like any input), or compose "
                              "dexel_erode/dexel_dilate with a halo exchange in between");
  dexel_desc d = src->d;
  d.stream = (void*)src->stream;
  dexel_grid tmp = nullptr;
  dexel_status s = dexel_create(&d, &tmp);
  if (s) return s;
  tmp->lev_cap = src->lev_cap;
  tmp->lev_arena = src->lev_arena;
  tmp->p1_cap = src->p1_cap;
  tmp->p2_acc = src->p2_acc;
  s = run_op(op1, src, r, r, tmp);
  if (!s) {
    s = run_op(op2, tmp, r, r, dst);
    src->lev_cap = std::max(src->lev_cap, tmp->lev_cap);
    src->lev_arena = std::max(src->lev_arena, tmp->lev_arena);
    src->p1_cap = std::max(src->p1_cap, tmp->p1_cap);
    src->p2_acc = std::max(src->p2_acc, tmp->p2_acc);
  }
  dexel_destroy(tmp);
  return s;
}
}  // namespace

extern "C" {

dexel_status dexel_open(dexel_grid src, float r, dexel_grid dst) {
  g_err.clear();
  return compose(OP_ERODE, OP_DILATE, src, r, dst);
}

dexel_status dexel_close(dexel_grid src, float r, dexel_grid dst) {
  g_err.clear();
  return compose(OP_DILATE, OP_ERODE, src, r, dst);
}

dexel_status dexel_size(dexel_grid g, uint64_t* n) {
  if (!g || !n) return fail(DEXEL_EINVAL, "NULL argument");
  *n = g->n;
  return DEXEL_OK;
}

dexel_status dexel_download(dexel_grid g, uint64_t* offsets, float* endpoints, uint64_t cap, int on_dev) {
  g_err.clear();
  if (!g || !offsets || (g->n > 0 && !endpoints)) return fail(DEXEL_EINVAL, "NULL argument");
  if (cap < g->n) return fail(DEXEL_EOVERFLOW, "capacity " + std::to_string(cap) + " < " + std::to_string(g->n));
  CK(cudaSetDevice(g->d.device));
  const cudaMemcpyKind k = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  const double t0 = now_s();
  CK(cudaMemcpyAsync(offsets, g->off.p, sizeof(uint64_t) * (g->ncol + 1), k, g->stream));
  if (g->n) CK(cudaMemcpyAsync(endpoints, g->ep.p, sizeof(float) * 2 * g->n, k, g->stream));
  CK(timed_sync(g->stream));
  static const bool dbg = std::getenv("DEXEL_DEBUG") != nullptr;
  if (dbg)
    std::fprintf(stderr, "[dexel] download %llu intervals: %.2f ms\n", (unsigned long long)g->n, 1e3 * (now_s() - t0));
  return DEXEL_OK;
}

dexel_status dexel_rasterize_shapes(dexel_grid g, double zmin, double zmax, int nsph, const double* sph,
                                    const int32_t* sph_sign, int nbox, const double* box, const int32_t* box_sign,
                                    int src_on_device) {
  g_err.clear();
  if (!g) return fail(DEXEL_EINVAL, "NULL handle");
  if (nsph < 0 || nbox < 0 || (nsph && (!sph || !sph_sign)) || (nbox && (!box || !box_sign)))
    return fail(DEXEL_EINVAL, "invalid shape arrays");
  const double zref = 0.5 * (zmin + zmax);
  if (!(zmin < zmax) || zref != g->d.z_ref || (float)(zmin - zref) != g->d.z_lo || (float)(zmax - zref) != g->d.z_hi)
    return fail(DEXEL_EINVAL, "[zmin, zmax] must give the grid's frame: z_ref = (zmin + zmax)/2, "
                              "z_lo = fl32(zmin - z_ref), z_hi = fl32(zmax - z_ref)");
  CK(cudaSetDevice(g->d.device));
  // the shapes on the host (validation), then on the device (binning, the kernel)
  std::vector<double> hs((size_t)4 * nsph), hb((size_t)6 * nbox);
  std::vector<int32_t> hss(nsph), hbs(nbox);
  const cudaMemcpyKind k = src_on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost;
  if (nsph) {
    CK(cudaMemcpy(hs.data(), sph, sizeof(double) * hs.size(), k));
    CK(cudaMemcpy(hss.data(), sph_sign, sizeof(int32_t) * hss.size(), k));
  }
  if (nbox) {
    CK(cudaMemcpy(hb.data(), box, sizeof(double) * hb.size(), k));
    CK(cudaMemcpy(hbs.data(), box_sign, sizeof(int32_t) * hbs.size(), k));
  }
  for (double v : hs) if (!std::isfinite(v)) return fail(DEXEL_EINVAL, "non-finite sphere parameter");
  for (double v : hb) if (!std::isfinite(v)) return fail(DEXEL_EINVAL, "non-finite box parameter");
  const int nx = g->d.nx, nrows = g->nrows, y0 = g->d.y0;
  const int ntx = (nx + RT_X - 1) / RT_X, nty = (nrows + RT_Y - 1) / RT_Y;
  const int64_t ntiles = (int64_t)ntx * nty;
  const int nshape = nsph + nbox;
  dexel_status s;
  dexel_stats stats{};
  Temps T(g, &stats);
  double *dsph = nullptr, *dbox = nullptr;
  int32_t *dss = nullptr, *dbs = nullptr, *dtid = nullptr;
  uint64_t* dtoff = nullptr;
  uint32_t *tcnt = nullptr, *tcur = nullptr;
  const int64_t ncol = g->ncol;
  float2* stage = nullptr;
  uint32_t* cnt = nullptr;
  unsigned* flags = nullptr;
  if ((s = T.get(sizeof(double) * hs.size() + 16, (void**)&dsph))) return s;
  if ((s = T.get(sizeof(double) * hb.size() + 16, (void**)&dbox))) return s;
  if ((s = T.get(sizeof(int32_t) * hss.size() + 16, (void**)&dss))) return s;
  if ((s = T.get(sizeof(int32_t) * hbs.size() + 16, (void**)&dbs))) return s;
  if ((s = T.get(sizeof(uint64_t) * (ntiles + 1), (void**)&dtoff))) return s;
  if ((s = T.get(sizeof(uint32_t) * (ntiles + 1) * 2, (void**)&tcnt))) return s;
  tcur = tcnt + ntiles + 1;
  int out_cap = RS_OUT;
  if ((s = T.get(sizeof(float2) * (size_t)out_cap * ncol + 16, (void**)&stage))) return s;
  if ((s = T.get(sizeof(uint32_t) * (ncol + 1), (void**)&cnt))) return s;
  if ((s = T.get(64, (void**)&flags))) return s;
  if (nsph) {
    CK(cudaMemcpyAsync(dsph, hs.data(), sizeof(double) * hs.size(), cudaMemcpyHostToDevice, g->stream));
    CK(cudaMemcpyAsync(dss, hss.data(), sizeof(int32_t) * hss.size(), cudaMemcpyHostToDevice, g->stream));
  }
  if (nbox) {
    CK(cudaMemcpyAsync(dbox, hb.data(), sizeof(double) * hb.size(), cudaMemcpyHostToDevice, g->stream));
    CK(cudaMemcpyAsync(dbs, hbs.data(), sizeof(int32_t) * hbs.size(), cudaMemcpyHostToDevice, g->stream));
  }
  // tile binning on the device: count, scan, fill (conservative; the kernel's tests are exact)
  const RasterBin Bn{nx, nrows, y0, ntx, nsph, nshape, dsph, dbox};
  CK(cudaMemsetAsync(tcnt, 0, sizeof(uint32_t) * (ntiles + 1) * 2, g->stream));
  const unsigned sb = (unsigned)((nshape + 255) / 256);
  if (nshape) LAUNCH(T, K_RASTER, raster_bin_count<<<sb, 256, 0, g->stream>>>(Bn, tcnt));
  uint64_t nids = 0;
  if ((s = scan_counts(g, T, tcnt, (uint64_t)ntiles, dtoff, &nids))) return s;
  if ((s = T.get(sizeof(int32_t) * (nids + 1), (void**)&dtid))) return s;
  if (nshape) LAUNCH(T, K_RASTER, raster_bin_fill<<<sb, 256, 0, g->stream>>>(Bn, dtoff, tcur, dtid));
  CK(cudaGetLastError());
  CK(cudaMemsetAsync(flags, 0, 64, g->stream));
  RasterArgs A{nx, nrows, y0, zmin, zmax, zref, nsph, dsph, dss, nbox, dbox, dbs, dtoff, dtid, ntx,
               stage, cnt, flags, out_cap};
  if (ntiles > 0)
    LAUNCH(T, K_RASTER, raster_kernel<RS_CAP><<<(unsigned)ntiles, dim3(RT_X, RT_Y), 0, g->stream>>>(A));
  CK(cudaGetLastError());
  unsigned hf = 0;
  auto read_flag = [&]() -> cudaError_t {
    Readback rb{g};
    rb.add(0, flags, sizeof(hf));
    const cudaError_t e = rb.wait();   // (the host shape vectors also stay alive until here)
    rb.get(0, &hf, sizeof(hf));
    return e;
  };
  CK(read_flag());
  if (hf) {
    // a column outgrew the first attempt's capacities (64 chord intervals per sign, 32 output
    // intervals): once more with 512-entry unions in local memory and a staging array of up to 512
    // output intervals per column (at most ~8 GB: min(512, 2^30 / columns), at least 32)
    const int64_t fit = ((int64_t)1 << 30) / (ncol > 0 ? ncol : 1);
    out_cap = (int)std::max<int64_t>(RS_OUT, std::min<int64_t>(RS_CAP_BIG, fit));
    if ((s = T.get(sizeof(float2) * (size_t)out_cap * ncol + 16, (void**)&stage))) return s;
    CK(cudaMemsetAsync(flags, 0, 64, g->stream));
    A.stage = stage;
    A.out_cap = out_cap;
    LAUNCH(T, K_RASTER, raster_kernel<RS_CAP_BIG><<<(unsigned)ntiles, dim3(RT_X, RT_Y), 0, g->stream>>>(A));
    CK(cudaGetLastError());
    CK(read_flag());
    if (hf)
      return fail(DEXEL_EOVERFLOW, "a column needs more than " + std::to_string(RS_CAP_BIG) +
                                       " chord intervals per sign or " + std::to_string(out_cap) +
                                       " output intervals");
  }
  // offsets, then the endpoints: the grid is replaced only now, into its own buffers when they
  // fit (a fresh allocation per call churns the stream-ordered pool); an error from here on
  // leaves the grid empty
  if (!g->off.p && (s = dalloc(g, g->off, sizeof(uint64_t) * (ncol + 1)))) return s;
  uint64_t n = 0;
  if ((s = scan_counts(g, T, cnt, (uint64_t)ncol, (uint64_t*)g->off.p, &n))) {
    set_empty(g);
    return s;
  }
  {
    const size_t need = sizeof(float2) * (n + 1);
    if (!(g->ep.p && g->ep.bytes >= need && g->ep.bytes - need <= need / 4)) {
      dfree(g, g->ep);
      if ((s = dalloc(g, g->ep, need))) {
        set_empty(g);
        return s;
      }
    }
  }
  if (ncol > 0)
    LAUNCH(T, K_COMPACT, compact_kernel<<<(unsigned)((ncol + 255) / 256), 256, 0, g->stream>>>(
                             stage, cnt, (const uint64_t*)g->off.p, ncol, (float2*)g->ep.p, n, flags));
  CK(cudaGetLastError());
  T.prof.finish();
  CK(timed_sync(g->stream));
  g->n = n;
  stats.n_out = n;
  g->stats = stats;
  return DEXEL_OK;
}

dexel_status dexel_rasterize_gyroid(dexel_grid g, double zmin, double zmax, double period, double t, double amp,
                                    uint64_t seed) {
  g_err.clear();
  if (!g) return fail(DEXEL_EINVAL, "NULL handle");
  const double zref = 0.5 * (zmin + zmax);
  if (!(zmin < zmax) || zref != g->d.z_ref || (float)(zmin - zref) != g->d.z_lo || (float)(zmax - zref) != g->d.z_hi)
    return fail(DEXEL_EINVAL, "[zmin, zmax] must give the grid's frame: z_ref = (zmin + zmax)/2, "
                              "z_lo = fl32(zmin - z_ref), z_hi = fl32(zmax - z_ref)");
  if (!(zmin >= 0.0 && zmin == std::floor(zmin) && zmax == std::floor(zmax) && zmax - zmin <= (double)(1 << 24)))
    return fail(DEXEL_EINVAL, "gyroid: zmin and zmax must be integers, 0 <= zmin < zmax (samples at zmin + m + 1/2)");
  if (!(std::isfinite(period) && period > 0.0 && std::isfinite(t) && std::isfinite(amp) && amp >= 0.0))
    return fail(DEXEL_EINVAL, "gyroid: period > 0, finite t and amp >= 0 required");
  CK(cudaSetDevice(g->d.device));
  const int nx = g->d.nx, nrows = g->nrows, y0 = g->d.y0, z0 = (int)zmin, nz = (int)(zmax - zmin);
  // sin / cos of w (k + 1/2) from the host's libm -- the generator's own values (dexelgen.c)
  const double w = 2.0 * M_PI / period;
  const int nk = std::max({nx, g->d.ny, z0 + nz});
  std::vector<double> tab(2 * (size_t)nk);
  for (int k = 0; k < nk; ++k) {
    tab[k] = std::sin(w * (k + 0.5));
    tab[nk + k] = std::cos(w * (k + 0.5));
  }
  auto mix = [](uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
  };
  const uint64_t key = mix(mix(seed) ^ (6ULL * 0xD1B54A32D192ED03ULL));   // stream 6 (dexelgen_gyroid)
  dexel_status s;
  dexel_stats stats{};
  Temps T(g, &stats);
  const int64_t ncol = g->ncol;
  double* dtab = nullptr;
  uint32_t* cnt = nullptr;
  if ((s = T.get(sizeof(double) * tab.size() + 16, (void**)&dtab))) return s;
  if ((s = T.get(sizeof(uint32_t) * (ncol + 1), (void**)&cnt))) return s;
  CK(cudaMemcpyAsync(dtab, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice, g->stream));
  GyroidArgs A{nx, nrows, y0, nz, z0, t, amp, zref, key, dtab, dtab + nk, cnt, nullptr, nullptr};
  const unsigned blocks = (unsigned)((ncol + 255) / 256);
  if (ncol > 0) LAUNCH(T, K_RASTER, gyroid_kernel<false><<<blocks, 256, 0, g->stream>>>(A));
  CK(cudaGetLastError());
  // offsets, then the endpoints (an error from here on leaves the grid empty)
  if (!g->off.p && (s = dalloc(g, g->off, sizeof(uint64_t) * (ncol + 1)))) return s;
  uint64_t n = 0;
  if ((s = scan_counts(g, T, cnt, (uint64_t)ncol, (uint64_t*)g->off.p, &n))) {   // (synchronises: tab is read)
    set_empty(g);
    return s;
  }
  {
    const size_t need = sizeof(float2) * (n + 1);
    if (!(g->ep.p && g->ep.bytes >= need && g->ep.bytes - need <= need / 4)) {
      dfree(g, g->ep);
      if ((s = dalloc(g, g->ep, need))) {
        set_empty(g);
        return s;
      }
    }
  }
  A.off = (const uint64_t*)g->off.p;
  A.ep = (float2*)g->ep.p;
  if (ncol > 0) LAUNCH(T, K_RASTER, gyroid_kernel<true><<<blocks, 256, 0, g->stream>>>(A));
  CK(cudaGetLastError());
  T.prof.finish();
  CK(timed_sync(g->stream));
  g->n = n;
  stats.n_out = n;
  g->stats = stats;
  return DEXEL_OK;
}

dexel_status dexel_pass1(dexel_grid g, float r, int complement, uint64_t* offsets, float* z, uint8_t* kappa,
                         uint64_t cap, uint64_t* n_pieces, int on_dev) {
  g_err.clear();
  if (!g || !n_pieces) return fail(DEXEL_EINVAL, "NULL argument");
  int R;
  dexel_status s;
  if ((s = check_radius(r, g->d.spacing, &R))) return s;
  CK(cudaSetDevice(g->d.device));
  Temps T(g);
  SrcRows rows{{nullptr, (const uint64_t*)g->off.p, nullptr}, {nullptr, (const float*)g->ep.p, nullptr},
               {0, g->nrows, 0}, g->d.nx, g->nrows, g->d.z_lo, g->d.z_hi};
  PieceSlots P;
  uint64_t m = 0;
  unsigned* opf = nullptr;
  if ((s = T.get(sizeof(unsigned) * OPF_WORDS, (void**)&opf))) return s;
  // unfiltered pieces (no capsule-domination pruning): bitwise comparable with the oracle's P1
  for (int attempt = 0;; ++attempt) {
    CK(cudaMemsetAsync(opf, 0, sizeof(unsigned) * OPF_WORDS, g->stream));
    if ((s = run_pass1(g, T, rows, R, complement ? 1 : 0, 0, g->nrows, opf, &P, nullptr))) return s;
    unsigned hf[OPF_WORDS];
    Readback rb{g};
    rb.add(0, opf, sizeof(hf));
    CK(rb.wait());
    rb.get(0, hf, sizeof(hf));
    std::memcpy(&m, hf + 8, sizeof(m));
    if (!hf[OPF_P1_RERUN]) break;
    if (attempt >= 10) return fail(DEXEL_ECUDA, "pass-1 capacity sizing did not converge");
    release_pieces(T, P);
    int cap = g->p1_cap > 0 ? (g->p1_cap + 3) / 4 * 4 : 256;
    while (cap < 1 << 15 && (unsigned)cap * 2 < hf[OPF_P1_LONGEST]) cap *= 2;
    g->p1_cap = std::min(1 << 15, cap * 2);
  }
  *n_pieces = m;
  if (cap < m) return fail(DEXEL_EOVERFLOW, "capacity < pieces");
  if (!offsets || (m && (!z || !kappa))) return fail(DEXEL_EINVAL, "NULL output buffer");
  // slots -> CSR on the device (count scan + gather)
  uint64_t* off = nullptr;
  float2* oz = nullptr;
  uint8_t* ok = nullptr;
  if ((s = T.get(sizeof(uint64_t) * (g->ncol + 1), (void**)&off))) return s;
  if ((s = T.get(sizeof(float2) * (m + 1), (void**)&oz))) return s;
  if ((s = T.get(m + 16, (void**)&ok))) return s;
  uint64_t m2 = 0;
  if ((s = scan_counts(g, T, P.cnt, (uint64_t)g->ncol, off, &m2))) return s;
  if (g->ncol > 0)
    pieces_to_csr<<<(unsigned)((g->ncol + 255) / 256), 256, 0, g->stream>>>(P, g->ncol, off, oz, ok);
  CK(cudaGetLastError());
  const cudaMemcpyKind k = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  CK(cudaMemcpyAsync(offsets, off, sizeof(uint64_t) * (g->ncol + 1), k, g->stream));
  if (m) {
    CK(cudaMemcpyAsync(z, oz, sizeof(float2) * m, k, g->stream));
    CK(cudaMemcpyAsync(kappa, ok, m, k, g->stream));
  }
  CK(timed_sync(g->stream));
  return DEXEL_OK;
}

dexel_status dexel_sync(dexel_grid g) {
  if (!g) return fail(DEXEL_EINVAL, "NULL handle");
  CK(timed_sync(g->stream));
  return DEXEL_OK;
}

void dexel_destroy(dexel_grid g) {
  if (!g) return;
  cudaSetDevice(g->d.device);
  dfree(g, g->off);
  dfree(g, g->ep);
  for (int q = 0; q < 2; ++q) {
    dfree(g, g->hoff[q]);
    dfree(g, g->hep[q]);
  }
  {
    DevWs& W = dev_ws(g->d.device);
    bool last;
    {
      std::lock_guard<std::mutex> lk(W.mu);
      last = --W.handles == 0;
      if (last) W.band_budget = 0;
    }
    if (last) ws_trim_idle(g);   // the device's last handle: its workspace goes too
  }
  dfree(g, g->spare_off);
  dfree(g, g->spare_ep);
  dfree(g, g->hdr);
  dfree(g, g->arena);
  for (auto& H : g->htab) dfree(g, H.dev);
  if (g->comm) {
    cudaStreamSynchronize(g->comm);
    cudaStreamDestroy(g->comm);
  }
  if (g->ev_main) cudaEventDestroy(g->ev_main);
  if (g->ev_halo) cudaEventDestroy(g->ev_halo);
  for (int q = 0; q < 2; ++q)   // unlink from loopback neighbours
    if (g->link[q] && g->link[q]->link[1 - q] == g) g->link[q]->link[1 - q] = nullptr;
  cudaStreamSynchronize(g->stream);
  if (g->own_stream) cudaStreamDestroy(g->stream);
  if (g->pin) cudaFreeHost(g->pin);
  delete g;
}

dexel_status dexel_trim_workspace(int device) {
  g_err.clear();
  if (device < 0 || device >= 64) return fail(DEXEL_EINVAL, "device out of range");
  CK(cudaSetDevice(device));
  DevWs& W = dev_ws(device);
  std::lock_guard<std::mutex> lk(W.mu);
  for (auto& e : W.e)
    if (!e.busy && e.b.p) {
      if (e.ev) cudaEventSynchronize(e.ev);   // its last user is done
      if (e.b.freefn) e.b.freefn(e.b.p, e.b.bytes ? e.b.bytes : 16, device, nullptr, e.b.ctx);
      else cudaFree(e.b.p);
      e.b = Buf{};
      if (e.ev) cudaEventDestroy(e.ev);
      e.ev = nullptr;
      e.last = nullptr;
    }
  W.band_budget = 0;   // (re-queried by the next op)
  // the stream-ordered pool keeps freed memory reserved (release threshold: max): hand its
  // unused part back to the driver too
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, 0);
  }
  return DEXEL_OK;
}

dexel_status dexel_set_timing(int on) {
  g_timing = on != 0;
  return DEXEL_OK;
}

dexel_status dexel_last_stats(dexel_grid g, dexel_stats* out) {
  if (!g || !out) return fail(DEXEL_EINVAL, "NULL argument");
  *out = g->stats;
  return DEXEL_OK;
}

dexel_status dexel_nccl_unique_id(uint8_t id[128]) {
  g_err.clear();
  if (!id) return fail(DEXEL_EINVAL, "NULL argument");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  NK(ncclGetUniqueId(&u));
  std::memcpy(id, &u, sizeof(u));
  return DEXEL_OK;
}

dexel_status dexel_nccl_comm_init(const uint8_t id[128], int nranks, int rank, int device, void** comm) {
  g_err.clear();
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return fail(DEXEL_EINVAL, "bad communicator arguments");
  CK(cudaSetDevice(device));
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  NK(ncclCommInitRank(&c, nranks, u, rank));
  *comm = (void*)c;
  return DEXEL_OK;
}

dexel_status dexel_nccl_comm_destroy(void* comm) {
  g_err.clear();
  if (!comm) return DEXEL_OK;
  NK(ncclCommDestroy((ncclComm_t)comm));
  return DEXEL_OK;
}

dexel_status dexel_link_slabs(dexel_grid* slabs, int n) {
  g_err.clear();
  if (!slabs || n < 1) return fail(DEXEL_EINVAL, "bad slab list");
  for (int q = 0; q < n; ++q) {
    const dexel_grid g = slabs[q];
    if (!g) return fail(DEXEL_EINVAL, "NULL slab handle");
    const dexel_desc& d = g->d;
    if (d.nranks != n || d.rank != q || d.nccl_comm)
      return fail(DEXEL_EINVAL, "slab " + std::to_string(q) + " must have rank " + std::to_string(q) + " of nranks " +
                                    std::to_string(n) + " and no NCCL communicator");
    const dexel_desc& d0 = slabs[0]->d;
    if (d.nx != d0.nx || d.ny != d0.ny || d.spacing != d0.spacing || d.z_lo != d0.z_lo || d.z_hi != d0.z_hi)
      return fail(DEXEL_EINVAL, "slabs must share the grid geometry");
    if ((q == 0 && d.y0 != 0) || (q > 0 && d.y0 != slabs[q - 1]->d.y1) || (q + 1 == n && d.y1 != d.ny))
      return fail(DEXEL_EINVAL, "the slabs' rows [y0, y1) must tile [0, ny) in rank order");
  }
  for (int q = 0; q < n; ++q) {
    slabs[q]->link[0] = q > 0 ? slabs[q - 1] : nullptr;
    slabs[q]->link[1] = q + 1 < n ? slabs[q + 1] : nullptr;
  }
  return DEXEL_OK;
}

// ------------------------------------------------------------------ host pipeline
// dexel_pipe: one op from a host CSR to a host CSR, streamed in y-slabs (dexel.h).  The host holds
// every row, so each slab's halo rows are uploaded straight from the host CSR (caller-managed halo
// mode: no exchange); three host threads keep the copy engines and the SMs busy at once:
//   uploader   slab q+1: rows and halo rows host -> device (offsets rebased on the device), validation
//   caller     slab q:   the op (pass 1, levels, pass 2: the same kernels as dexel_dilate/erode/shell)
//   downloader slab q-1: result device -> host at its place in the output CSR, offsets shifted by the
//                        intervals of the slabs before it
// Each slab has its own stream; the stages hand slabs over under one mutex.
struct dexel_pipe_s {
  dexel_desc d;
  int nslabs = 0;
  std::vector<dexel_grid> src, dst;
  uint64_t h2d = 0, d2h = 0;   // bytes the last run copied (dexel_pipe_last_bytes)
};

namespace {
struct PipeSync {
  std::mutex mu;
  std::condition_variable cv;
  int uploaded = 0, computed = 0;   // slabs that left each stage
  dexel_status err = DEXEL_OK;
  std::string msg;
  void fail_with(dexel_status s) {
    std::lock_guard<std::mutex> lk(mu);
    if (err == DEXEL_OK) {
      err = s;
      msg = g_err;
    }
    cv.notify_all();
  }
};
}  // namespace

dexel_status dexel_pipe_create(const dexel_desc* d, int nslabs, dexel_pipe* out) {
  g_err.clear();
  if (!d || !out) return fail(DEXEL_EINVAL, "NULL argument");
  if (d->nranks != 1 || d->y0 != 0 || d->y1 != d->ny || d->nccl_comm)
    return fail(DEXEL_EINVAL, "the pipeline's descriptor must describe the whole grid on one device");
  if (nslabs < 1 || nslabs > d->ny) return fail(DEXEL_EINVAL, "nslabs must be in [1, ny]");
  dexel_pipe p = new dexel_pipe_s();
  p->d = *d;
  p->nslabs = nslabs;
  for (int q = 0; q < nslabs; ++q) {
    dexel_desc dq = *d;
    dq.stream = nullptr;   // a stream per slab (the stages overlap across slabs)
    dq.rank = q;
    dq.nranks = nslabs;
    // the first upload and the last download are the only copies no op hides: from 3 slabs on the
    // first and the last slab get half the rows of the others (weights 1/2, 1, ..., 1, 1/2)
    auto cut = [&](int t) -> int {   // first row of slab t
      if (t <= 0) return 0;
      if (t >= nslabs) return d->ny;
      if (nslabs < 3 || d->ny < 2 * nslabs) return (int)((int64_t)d->ny * t / nslabs);
      return (int)((int64_t)d->ny * (2 * t - 1) / (2 * (nslabs - 1)));
    };
    dq.y0 = cut(q);
    dq.y1 = cut(q + 1);
    dexel_grid a = nullptr, b = nullptr;
    dexel_status s = dexel_create(&dq, &a);
    if (s == DEXEL_OK) {
      dq.stream = a->stream;   // the result handle shares the slab's stream
      s = dexel_create(&dq, &b);
    }
    if (s != DEXEL_OK) {
      const std::string msg = g_err;
      dexel_destroy(a);
      dexel_pipe_destroy(p);
      g_err = msg;
      return s;
    }
    p->src.push_back(a);
    p->dst.push_back(b);
  }
  *out = p;
  return DEXEL_OK;
}

// Slab count for a grid and radius: slabs of at least max(512, 32 R) rows (the halo rows' pass 1 and
// levels stay under ~6% of a slab's; smaller slabs also pay the per-op fixed costs more often), at
// most 6 (with the half-size end slabs C5 r=16 runs 147.5 ms with 6, 148.7 with 8, 151.1 with 10),
// and no split below R = 8: there the op is shorter than its copies, and uploads and
// downloads running at once each slow down about 2x on this host, so overlapping them gains nothing
// (measured on B200, profiles/r02_pipe_e2e.md: C4 r=16 and r=8 best at 4 slabs; C4
// r <= 4, C4 r=64 and the 512^2 grid lose with any split -> 1).
int dexel_pipe_suggest_slabs(const dexel_desc* d, float r) {
  if (!d || d->ny < 1 || !(d->spacing > 0) || !(r >= 0)) return 1;
  const double R = std::floor((double)r / d->spacing);
  if (R < 8) return 1;
  const double rows = std::max(512.0, 32.0 * R);
  const int s = (int)((double)d->ny / rows);
  return s < 1 ? 1 : (s > 6 ? 6 : s);
}

dexel_status dexel_pipe_last_bytes(dexel_pipe p, uint64_t* h2d, uint64_t* d2h) {
  g_err.clear();
  if (!p || !h2d || !d2h) return fail(DEXEL_EINVAL, "NULL argument");
  *h2d = p->h2d;
  *d2h = p->d2h;
  return DEXEL_OK;
}

dexel_status dexel_pipe_slab_rows(dexel_pipe p, int q, int32_t* y0, int32_t* y1) {
  g_err.clear();
  if (!p || !y0 || !y1 || q < 0 || q >= p->nslabs) return fail(DEXEL_EINVAL, "bad slab index");
  *y0 = p->src[q]->d.y0;
  *y1 = p->src[q]->d.y1;
  return DEXEL_OK;
}

void dexel_pipe_destroy(dexel_pipe p) {
  if (!p) return;
  for (dexel_grid g : p->dst) dexel_destroy(g);   // (before src: they borrow its stream)
  for (dexel_grid g : p->src) dexel_destroy(g);
  delete p;
}

dexel_status dexel_pipe_run(dexel_pipe p, int op, float r_a, float r_b, const uint64_t* offsets,
                            const float* endpoints, uint64_t* out_offsets, float* out_endpoints, uint64_t cap,
                            uint64_t* n_out) {
  g_err.clear();
  if (!p || !offsets || !out_offsets || !n_out) return fail(DEXEL_EINVAL, "NULL argument");
  if (op != OP_DILATE && op != OP_ERODE && op != OP_SHELL) return fail(DEXEL_EINVAL, "op must be 0, 1 or 2");
  const int S = p->nslabs, nx = p->d.nx, ny = p->d.ny;
  const int64_t ncol = (int64_t)nx * ny;
  if (offsets[0] != 0 || (offsets[ncol] > 0 && !endpoints)) return fail(DEXEL_EINVAL, "bad input CSR");
  int Ra, Rb;
  dexel_status s;
  if ((s = check_radius(r_a, p->d.spacing, &Ra))) return s;
  if ((s = check_radius(op == OP_SHELL ? r_b : r_a, p->d.spacing, &Rb))) return s;
  const int R = Ra > Rb ? Ra : Rb;
  *n_out = 0;
  PipeSync Q;
  static const bool dbg = std::getenv("DEXEL_DEBUG") != nullptr;
  const double t_run = now_s();
  auto mark = [&](const char* what, int q, double t0) {   // DEXEL_DEBUG: the stages' timeline
    if (dbg)
      std::fprintf(stderr, "[dexel] pipe %s slab %d: %.3f .. %.3f ms\n", what, q, 1e3 * (t0 - t_run),
                   1e3 * (now_s() - t_run));
  };
  // rows [a, b) of the host CSR as a slice: offsets from a*nx, endpoints from its first interval
  auto slice = [&](int a, int b, const uint64_t*& off, const float*& ep, uint64_t& n) {
    off = offsets + (int64_t)a * nx;
    n = offsets[(int64_t)b * nx] - off[0];
    ep = endpoints ? endpoints + 2 * off[0] : nullptr;
  };
  uint64_t h2d = 0;
  std::thread up([&] {
    for (int q = 0; q < S; ++q) {
      {
        std::lock_guard<std::mutex> lk(Q.mu);
        if (Q.err) return;
      }
      const double t_up = now_s();
      dexel_grid g = p->src[q];
      const int y0 = g->d.y0, y1 = g->d.y1;
      const int lo = y0 < R ? y0 : R, hi = ny - y1 < R ? ny - y1 : R;
      const uint64_t* off;
      const float* ep;
      uint64_t n;
      slice(y0, y1, off, ep, n);
      h2d += 8 * ((uint64_t)(y1 - y0) * nx + 1) + 8 * n;
      dexel_status e = upload_impl(g, off, ep, n, 0, true);
      if (!e) {
        slice(y0 - lo, y0, off, ep, n);
        if (lo) h2d += 8 * ((uint64_t)lo * nx + 1) + 8 * n;
        e = upload_halo_impl(g, 0, off, ep, lo, n, 0, true);
      }
      if (!e) {
        slice(y1, y1 + hi, off, ep, n);
        if (hi) h2d += 8 * ((uint64_t)hi * nx + 1) + 8 * n;
        e = upload_halo_impl(g, 1, off, ep, hi, n, 0, true);
      }
      if (e) return Q.fail_with(e);
      mark("upload", q, t_up);
      std::lock_guard<std::mutex> lk(Q.mu);
      Q.uploaded = q + 1;
      Q.cv.notify_all();
    }
  });
  uint64_t total = 0, d2h = 0;
  std::thread down([&] {
    for (int q = 0; q < S; ++q) {
      {
        std::unique_lock<std::mutex> lk(Q.mu);
        Q.cv.wait(lk, [&] { return Q.computed > q || Q.err; });
        if (Q.err) return;
      }
      const double t_dn = now_s();
      dexel_grid g = p->dst[q];
      if (total + g->n > cap) {
        fail(DEXEL_EOVERFLOW, "capacity " + std::to_string(cap) + " < the result's intervals");
        return Q.fail_with(DEXEL_EOVERFLOW);
      }
      uint64_t* o = out_offsets + (int64_t)g->d.y0 * nx;
      const dexel_status e = dexel_download(g, o, out_endpoints ? out_endpoints + 2 * total : nullptr, cap - total, 0);
      if (e) return Q.fail_with(e);
      if (total)
        for (int64_t c = 0; c <= g->ncol; ++c) o[c] += total;
      total += g->n;
      d2h += 8 * ((uint64_t)g->ncol + 1) + 8 * g->n;
      mark("download", q, t_dn);
    }
  });
  for (int q = 0; q < S; ++q) {
    {
      std::unique_lock<std::mutex> lk(Q.mu);
      Q.cv.wait(lk, [&] { return Q.uploaded > q || Q.err; });
      if (Q.err) break;
    }
    const double t_op = now_s();
    const dexel_status e = run_op(op, p->src[q], r_a, op == OP_SHELL ? r_b : r_a, p->dst[q]);
    if (e) {
      Q.fail_with(e);
      break;
    }
    mark("op", q, t_op);
    std::lock_guard<std::mutex> lk(Q.mu);
    Q.computed = q + 1;
    Q.cv.notify_all();
  }
  up.join();
  down.join();
  mark("run", S, t_run);
  p->h2d = h2d;
  p->d2h = d2h;
  if (Q.err) {
    g_err = Q.msg;
    return Q.err;
  }
  *n_out = total;
  return DEXEL_OK;
}

}  // extern "C"
