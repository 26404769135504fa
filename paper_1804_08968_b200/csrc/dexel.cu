// dexel.cu -- host orchestration and C ABI (include/dexel.h) of the B200
// separable dexel offset library.  Builds libdexel.so for sm_100a.
//
// Op pipeline (one "family" per dilation; erode and shell dilate the
// complement, which pass 1 reads on the fly):
//   pass1 COUNT -> scan -> pass1 WRITE          S_In -> S_Mid (pieces lo,hi,kappa)
//   levels COUNT -> scan -> levels WRITE        S_Mid -> {L_k}, k = 0..R
//   pass2 COUNT -> scan -> pass2 WRITE          {L_k} -> S_Out (+ epilogue)
// Each scan ends with one 8-byte device->host read of the total (allocation size).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "dexel.h"
#include "kernels.cuh"
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
    if (e_ != cudaSuccess) return fail(DEXEL_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
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
  double lev_ratio = 0.0;   // n_lev / n_mid of the last op (arena sizing hint)
  // y-slab halos (multi-GPU): rows [y0 - hrows[0], y0) and [y1, y1 + hrows[1]) of the input
  Buf hoff[2], hep[2];
  int hrows[2] = {0, 0};
  uint64_t hn[2] = {0, 0};
};

namespace {

// dst[t] = src[t] - src[0] + add, t in [0, n]
__global__ void rebase_offsets(const uint64_t* __restrict__ src, uint64_t n, uint64_t add, uint64_t* __restrict__ dst) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t <= n) dst[t] = src[t] - src[0] + add;
}

dexel_status dalloc(dexel_grid g, Buf& b, size_t bytes) {
  b.bytes = bytes;
  b.p = nullptr;
  if (bytes == 0) bytes = 16;
  if (g_alloc) {
    b.p = g_alloc(bytes, g->d.device, (void*)g->stream, g_alloc_ctx);
    if (!b.p) return fail(DEXEL_ENOMEM, "allocator returned NULL for " + std::to_string(bytes) + " bytes");
  } else {
    cudaError_t e = cudaMallocAsync(&b.p, bytes, g->stream);
    if (e != cudaSuccess) {
      b.p = nullptr;
      return fail(DEXEL_ENOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e) + " (" +
                                    std::to_string(bytes) + " bytes)");
    }
  }
  return DEXEL_OK;
}

void dfree(dexel_grid g, Buf& b) {
  if (!b.p) return;
  if (g_free) g_free(b.p, b.bytes ? b.bytes : 16, g->d.device, (void*)g->stream, g_alloc_ctx);
  else cudaFreeAsync(b.p, g->stream);
  b.p = nullptr;
  b.bytes = 0;
}

// per-op kernel accounting: launch counts always, CUDA-event device times when g_timing
enum { K_P1C = 0, K_P1W = 1, K_LVC = 2, K_LVW = 3, K_P2C = 4, K_P2W = 5, K_SCAN = 6, K_OTHER = 7 };
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

// RAII for temporaries of one op
struct Temps {
  dexel_grid g;
  std::vector<Buf> bufs;
  Prof prof;
  explicit Temps(dexel_grid g_, dexel_stats* st = nullptr) : g(g_) {
    prof.st = g_->stream;
    prof.s = st;
    prof.on = g_timing && st != nullptr;
  }
  ~Temps() {
    prof.finish();
    for (auto& b : bufs) dfree(g, b);
  }
  dexel_status get(size_t bytes, void** p) {
    Buf b;
    dexel_status s = dalloc(g, b, bytes);
    if (s) return s;
    bufs.push_back(b);
    *p = b.p;
    return DEXEL_OK;
  }
  void release(void* p) {
    for (auto& b : bufs)
      if (b.p == p) dfree(g, b);
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
  CK(cudaMemcpyAsync(total, off + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  T.release(sums);
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
template <bool WRITE>
void launch_pass1(int NW, const SrcRows& src, int R, int complement, int row0, int nrows_out, uint32_t* cnt,
                  const uint64_t* moff, float2* mz, uint8_t* mk, cudaStream_t st) {
  const int64_t warps = (int64_t)nrows_out * ((src.nx + 31) / 32);
  const unsigned blocks = (unsigned)((warps + P1_WARPS - 1) / P1_WARPS);
  if (blocks == 0) return;
#define P1(NWV) pass1_kernel<NWV, WRITE><<<blocks, P1_WARPS * 32, 0, st>>>(src, R, complement, row0, nrows_out, cnt, moff, mz, mk)
  if (NW <= 2) P1(2);
  else if (NW <= 3) P1(3);
  else if (NW <= 5) P1(5);
  else if (NW <= 9) P1(9);
  else P1(17);
#undef P1
}

struct Pieces {
  uint64_t* moff = nullptr;
  float2* mz = nullptr;
  uint8_t* mk = nullptr;
  uint64_t m = 0;
};

dexel_status run_pass1(dexel_grid g, Temps& T, const SrcRows& src, int R, int complement, int row0, int nrows_out,
                       Pieces* P) {
  const int64_t ncol = (int64_t)nrows_out * src.nx;
  const int NW = (32 + 2 * R + 31) / 32;
  uint32_t* cnt = nullptr;
  dexel_status s;
  if ((s = T.get(sizeof(uint32_t) * (ncol + 1), (void**)&cnt))) return s;
  if ((s = T.get(sizeof(uint64_t) * (ncol + 1), (void**)&P->moff))) return s;
  LAUNCH(T, K_P1C, launch_pass1<false>(NW, src, R, complement, row0, nrows_out, cnt, nullptr, nullptr, nullptr, g->stream));
  CK(cudaGetLastError());
  if ((s = scan_counts(g, T, cnt, (uint64_t)ncol, P->moff, &P->m))) return s;
  T.release(cnt);
  if ((s = T.get(sizeof(float2) * (P->m + 1), (void**)&P->mz))) return s;
  if ((s = T.get(P->m + 16, (void**)&P->mk))) return s;
  LAUNCH(T, K_P1W, launch_pass1<true>(NW, src, R, complement, row0, nrows_out, nullptr, P->moff, P->mz, P->mk, g->stream));
  CK(cudaGetLastError());
  return DEXEL_OK;
}

// ---------------------------------------------------------------- levels
struct Family {
  LevelFamily F;
  uint64_t nlev = 0;
};

dexel_status make_tables(dexel_grid g, Temps& T, float r, int R, LevelTables* L, EnvTables* E) {
  const double s = g->d.spacing;
  const int n1 = R + 1;
  std::vector<float> h((size_t)n1 * n1);
  std::vector<double> W(n1), Tk(n1);
  const double rr = (double)r * (double)r;
  for (int a = 0; a < n1; ++a) {
    W[a] = rr - (double)a * a * s * s;
    Tk[a] = (double)a * a * s * s;
  }
  for (int a = 0; a < n1; ++a)
    for (int k = 0; k < n1; ++k) {
      // W(kappa) - T(k) in fp64, rounded once to fp32; valid iff T(k) <= W(kappa)
      const double w = W[a] - Tk[k];
      h[(size_t)a * n1 + k] = w >= 0.0 ? (float)std::sqrt(w) : -1.0f;
    }
  char* buf = nullptr;
  const size_t hb = sizeof(float) * h.size(), db = sizeof(double) * n1;
  dexel_status st;
  if ((st = T.get(hb + 2 * db + 64, (void**)&buf))) return st;
  double* dW = (double*)buf;
  double* dT = dW + n1;
  float* dh = (float*)(dT + n1);
  CK(cudaMemcpyAsync(dW, W.data(), db, cudaMemcpyHostToDevice, g->stream));
  CK(cudaMemcpyAsync(dT, Tk.data(), db, cudaMemcpyHostToDevice, g->stream));
  CK(cudaMemcpyAsync(dh, h.data(), hb, cudaMemcpyHostToDevice, g->stream));
  CK(cudaStreamSynchronize(g->stream));  // host vectors go out of scope
  L->h = dh;
  L->R = R;
  E->h = dh;
  E->W = dW;
  E->Tk = dT;
  E->R = R;
  E->r = (double)r;
  E->inv_s2 = 1.0 / (s * s);
  return DEXEL_OK;
}

template <int NS>
void launch_levels4_t(int R, int64_t ncol, const Pieces& P, const LevelTables& L, float zlo, float zhi,
                      const LevelOut& O, cudaStream_t st) {
  constexpr int WARPS = Lv4Cfg<NS>::WARPS;
  const int nl = R + 1;
  const int G = NS == 1 ? 32 / nl : 1;
  const int h_in_smem = sizeof(float) * nl * nl <= 64 * 1024 ? 1 : 0;
  const size_t smem = sizeof(float2) * WARPS * 2 * NS * STG_C * 32 + (h_in_smem ? sizeof(float) * nl * nl : 0);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(levels4_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const int64_t per_block = (int64_t)WARPS * G;
  const unsigned blocks = (unsigned)((ncol + per_block - 1) / per_block);
  if (blocks == 0) return;
  levels4_kernel<NS><<<blocks, WARPS * 32, smem, st>>>(ncol, P.moff, P.mz, P.mk, L, h_in_smem, zlo, zhi, O);
}

template <int LMAX>
void launch_levels5_t(int R, int64_t ncol, const Pieces& P, const LevelTables& L, float zlo, float zhi,
                      const LevelOut& O, cudaStream_t st) {
  (void)R;
  const unsigned blocks = (unsigned)((ncol + 127) / 128);
  if (blocks == 0) return;
  levels5_kernel<LMAX><<<blocks, 128, 0, st>>>(ncol, P.moff, P.mz, P.mk, L, zlo, zhi, O);
}

void launch_levels(int R, int64_t ncol, const Pieces& P, const LevelTables& L, float zlo, float zhi,
                   const LevelOut& O, cudaStream_t st) {
  const int nl = R + 1;
  // R < 17: one thread per column, 2(R+1) running unions in registers (levels5);
  // larger R: one warp per column, lanes = levels (levels4)
  if (nl <= 2) launch_levels5_t<2>(R, ncol, P, L, zlo, zhi, O, st);
  else if (nl <= 3) launch_levels5_t<3>(R, ncol, P, L, zlo, zhi, O, st);
  else if (nl <= 5) launch_levels5_t<5>(R, ncol, P, L, zlo, zhi, O, st);
  else if (nl <= 9) launch_levels5_t<9>(R, ncol, P, L, zlo, zhi, O, st);
  else if (nl <= 17) launch_levels5_t<17>(R, ncol, P, L, zlo, zhi, O, st);
  else if (nl <= 32) launch_levels4_t<1>(R, ncol, P, L, zlo, zhi, O, st);
  else if (nl <= 64) launch_levels4_t<2>(R, ncol, P, L, zlo, zhi, O, st);
  else if (nl <= 96) launch_levels4_t<3>(R, ncol, P, L, zlo, zhi, O, st);
  else if (nl <= 128) launch_levels4_t<4>(R, ncol, P, L, zlo, zhi, O, st);
  else launch_levels4_t<8>(R, ncol, P, L, zlo, zhi, O, st);
}

// level-set kernel: 1 = per-level running unions (levels5 for R < 17, levels4 above;
// default), 0 = power-diagram envelope (levels6; DEXEL_LEVELS=envelope, cross-checked
// in tests)
int levels_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("DEXEL_LEVELS");
    v = (e && std::strcmp(e, "envelope") == 0) ? 0 : 1;
  }
  return v;
}

// one dilation family: rows [row0, row0+nrows) of src (S or its complement) at radius r
dexel_status run_family(dexel_grid g, Temps& T, const SrcRows& src, float r, int complement, int row0, int nrows,
                        Family* out, uint64_t* n_mid) {
  int R;
  dexel_status s;
  if ((s = check_radius(r, g->d.spacing, &R))) return s;
  Pieces P;
  if ((s = run_pass1(g, T, src, R, complement, row0, nrows, &P))) return s;
  *n_mid += P.m;
  LevelTables L;
  EnvTables E;
  if ((s = make_tables(g, T, r, R, &L, &E))) return s;
  const int64_t ncol = (int64_t)nrows * src.nx;
  const int ndir = levels_mode() == 0 ? 1 : 2;
  const int ntask = ndir * (R + 1);
  LevelOut O;
  if ((s = T.get(sizeof(uint64_t) * (ncol + 1), (void**)&O.dbase))) return s;
  if ((s = T.get(sizeof(uint32_t) * (ncol * (ntask + 1) + 1), (void**)&O.rel))) return s;
  if ((s = T.get(sizeof(unsigned long long) * 2, (void**)&O.counter))) return s;
  // arena sized from the previous op's level/piece ratio (rerun with the exact size if it overflows)
  const double ratio = g->lev_ratio > 0 ? g->lev_ratio * 1.1 : 1.5;
  O.cap = (uint64_t)(ratio * (double)P.m) + 4096;
  for (int attempt = 0; attempt < 2; ++attempt) {
    if ((s = T.get(sizeof(float2) * (O.cap + 1), (void**)&O.arena))) return s;
    CK(cudaMemsetAsync(O.counter, 0, 2 * sizeof(unsigned long long), g->stream));
    if (ndir == 1) {
      const size_t smem = (sizeof(float) + sizeof(uint32_t)) * (R + 1) * 128;
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(levels6_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
      }
      const unsigned blocks = (unsigned)((ncol + 127) / 128);
      if (blocks) LAUNCH(T, K_LVW, levels6_kernel<<<blocks, 128, smem, g->stream>>>(ncol, P.moff, P.mz, P.mk, E,
                                                                                    src.zlo, src.zhi, O));
    } else {
      LAUNCH(T, K_LVW, launch_levels(R, ncol, P, L, src.zlo, src.zhi, O, g->stream));
    }
    CK(cudaGetLastError());
    unsigned long long used2[2] = {0, 0};
    CK(cudaMemcpyAsync(used2, O.counter, sizeof(used2), cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    const unsigned long long used = used2[0];
    if (used2[1])
      return fail(DEXEL_EOVERFLOW, ndir == 1 ? "a column's power-diagram envelope exceeds the deque capacity"
                                             : "a column has more than 65534 intervals in one level list");
    if (used <= O.cap) {
      out->nlev = used;
      break;
    }
    T.release(O.arena);
    O.cap = used;
    if (attempt == 1) return fail(DEXEL_ECUDA, "level arena sizing did not converge");
  }
  if (P.m > 0) g->lev_ratio = (double)out->nlev / (double)P.m;
  T.release(P.mz);
  T.release(P.mk);
  T.release(P.moff);
  out->F.dbase = O.dbase;
  out->F.rel = O.rel;
  out->F.arena = O.arena;
  out->F.R = R;
  out->F.ndir = ndir;
  out->F.ncol = ncol;
  out->F.row0 = row0;
  out->F.nrows = nrows;
  return DEXEL_OK;
}

template <int OP, bool WRITE>
void launch_pass2_t(const LevelFamily& A, const LevelFamily& B, int nx, int row0, int nrows, float zlo, float zhi,
                    uint32_t* ocnt, const uint64_t* ooff, float2* oz, int* ovf, cudaStream_t st) {
  const int64_t n = (int64_t)nrows * nx;
  const unsigned blocks = (unsigned)((n + 127) / 128);
  if (blocks == 0) return;
  pass2_kernel<OP, WRITE><<<blocks, 128, 0, st>>>(A, B, nx, row0, nrows, zlo, zhi, ocnt, ooff, oz, ovf);
}

template <bool WRITE>
void launch_pass2(int op, const LevelFamily& A, const LevelFamily& B, int nx, int row0, int nrows, float zlo,
                  float zhi, uint32_t* ocnt, const uint64_t* ooff, float2* oz, int* ovf, cudaStream_t st) {
  if (op == OP_DILATE) launch_pass2_t<OP_DILATE, WRITE>(A, B, nx, row0, nrows, zlo, zhi, ocnt, ooff, oz, ovf, st);
  else if (op == OP_ERODE) launch_pass2_t<OP_ERODE, WRITE>(A, B, nx, row0, nrows, zlo, zhi, ocnt, ooff, oz, ovf, st);
  else launch_pass2_t<OP_SHELL, WRITE>(A, B, nx, row0, nrows, zlo, zhi, ocnt, ooff, oz, ovf, st);
}

bool same_geometry(const dexel_desc& a, const dexel_desc& b) {
  return a.nx == b.nx && a.ny == b.ny && a.spacing == b.spacing && a.z_lo == b.z_lo && a.z_hi == b.z_hi &&
         a.device == b.device && a.y0 == b.y0 && a.y1 == b.y1 && a.rank == b.rank && a.nranks == b.nranks;
}

void set_empty(dexel_grid g) {
  if (g->off.p) cudaMemsetAsync(g->off.p, 0, sizeof(uint64_t) * (g->ncol + 1), g->stream);
  dfree(g, g->ep);
  g->n = 0;
}

dexel_status run_op(int op, dexel_grid src, float r_a, float r_b, dexel_grid dst) {
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
  // halo rows (y-slabs): the op reads rows [y0 - hlo, y1 + hhi) and writes [y0, y1)
  const int Rmax = Ra > Rb ? Ra : Rb;
  const int need_lo = src->d.y0 < Rmax ? src->d.y0 : Rmax;
  const int need_hi = src->d.ny - src->d.y1 < Rmax ? src->d.ny - src->d.y1 : Rmax;
  if (src->hrows[0] < need_lo || src->hrows[1] < need_hi)
    return fail(DEXEL_EINVAL, "slab halo too small: need " + std::to_string(need_lo) + " rows below and " +
                                  std::to_string(need_hi) + " above (dexel_upload_halo)");
  const int hlo = src->hrows[0], hhi = src->hrows[1];
  const int nrows_ext = hlo + src->nrows + hhi;
  const uint64_t* ext_off = (const uint64_t*)src->off.p;
  const float* ext_ep = (const float*)src->ep.p;
  if (hlo || hhi) {
    const int64_t nx = src->d.nx;
    const int64_t ncol_ext = (int64_t)nrows_ext * nx;
    const uint64_t next = src->hn[0] + src->n + src->hn[1];
    uint64_t* eo = nullptr;
    float2* ee = nullptr;
    if ((s = T.get(sizeof(uint64_t) * (ncol_ext + 1), (void**)&eo))) return s;
    if ((s = T.get(sizeof(float2) * (next + 1), (void**)&ee))) return s;
    const Buf* parts_off[3] = {&src->hoff[0], &src->off, &src->hoff[1]};
    const Buf* parts_ep[3] = {&src->hep[0], &src->ep, &src->hep[1]};
    const int64_t part_cols[3] = {(int64_t)hlo * nx, src->ncol, (int64_t)hhi * nx};
    const uint64_t part_n[3] = {src->hn[0], src->n, src->hn[1]};
    int64_t cbase = 0;
    uint64_t ebase = 0;
    for (int q = 0; q < 3; ++q) {
      if (part_cols[q] == 0) continue;
      rebase_offsets<<<(unsigned)((part_cols[q] + 256) / 256), 256, 0, st>>>(
          (const uint64_t*)parts_off[q]->p, (uint64_t)part_cols[q], ebase, eo + cbase);
      if (part_n[q]) CK(cudaMemcpyAsync(ee + ebase, parts_ep[q]->p, sizeof(float2) * part_n[q],
                                        cudaMemcpyDeviceToDevice, st));
      cbase += part_cols[q];
      ebase += part_n[q];
    }
    CK(cudaGetLastError());
    ext_off = eo;
    ext_ep = (const float*)ee;
  }
  SrcRows rows{ext_off, ext_ep, src->d.nx, nrows_ext, src->d.z_lo, src->d.z_hi};
  stats.n_in = src->n;
  Family FA, FB;
  // family A: dilate S (dilate, shell r_out) or C (erode)
  if ((s = run_family(src, T, rows, r_a, op == OP_ERODE ? 1 : 0, 0, nrows_ext, &FA, &stats.n_mid))) {
    set_empty(dst);
    return s;
  }
  stats.n_lev = FA.nlev;
  if (op == OP_SHELL) {
    if ((s = run_family(src, T, rows, r_b, 1, 0, nrows_ext, &FB, &stats.n_mid))) {
      set_empty(dst);
      return s;
    }
    stats.n_lev += FB.nlev;
  } else {
    FB = FA;
  }
  // pass 2
  const int64_t ncol = src->ncol;
  uint32_t* ocnt = nullptr;
  int* ovf = nullptr;
  if ((s = T.get(sizeof(uint32_t) * (ncol + 1), (void**)&ocnt))) return s;
  if ((s = T.get(sizeof(int) * 4, (void**)&ovf))) return s;
  CK(cudaMemsetAsync(ovf, 0, sizeof(int), st));
  LAUNCH(T, K_P2C, launch_pass2<false>(op, FA.F, FB.F, src->d.nx, hlo, src->nrows, src->d.z_lo, src->d.z_hi, ocnt,
                                       nullptr, nullptr, ovf, st));
  CK(cudaGetLastError());
  uint64_t nout = 0;
  // dst offsets: reuse dst->off
  if (!dst->off.p && (s = dalloc(dst, dst->off, sizeof(uint64_t) * (dst->ncol + 1)))) return s;
  if ((s = scan_counts(src, T, ocnt, (uint64_t)ncol, (uint64_t*)dst->off.p, &nout))) return s;
  int hovf = 0;
  CK(cudaMemcpy(&hovf, ovf, sizeof(int), cudaMemcpyDeviceToHost));
  if (hovf) {
    set_empty(dst);
    return fail(DEXEL_EOVERFLOW, "a column's union exceeds the pass-2 accumulator (" + std::to_string(ACC_CAP) +
                                     " intervals)");
  }
  dfree(dst, dst->ep);
  if ((s = dalloc(dst, dst->ep, sizeof(float2) * (nout + 1)))) return s;
  LAUNCH(T, K_P2W, launch_pass2<true>(op, FA.F, FB.F, src->d.nx, hlo, src->nrows, src->d.z_lo, src->d.z_hi,
                                      nullptr, (const uint64_t*)dst->off.p, (float2*)dst->ep.p, ovf, st));
  CK(cudaGetLastError());
  dst->n = nout;
  stats.n_out = nout;
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
  return DEXEL_OK;
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
  dexel_status s = dalloc(g, g->off, sizeof(uint64_t) * (g->ncol + 1));
  if (s) {
    delete g;
    return s;
  }
  CK(cudaMemsetAsync(g->off.p, 0, sizeof(uint64_t) * (g->ncol + 1), g->stream));
  *out = g;
  return DEXEL_OK;
}

}  // extern "C"

namespace {
// copy + validate a CSR of ncol columns into fresh buffers (grid unchanged on error)
dexel_status load_csr(dexel_grid g, const uint64_t* offsets, const float* endpoints, int64_t ncol, uint64_t n,
                      int on_dev, Buf* off_out, Buf* ep_out) {
  if (!offsets || (n > 0 && !endpoints)) return fail(DEXEL_EINVAL, "NULL argument");
  CK(cudaSetDevice(g->d.device));
  uint64_t first = 0, last = 0;
  if (on_dev) {
    CK(cudaMemcpyAsync(&first, offsets, 8, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaMemcpyAsync(&last, offsets + ncol, 8, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
  } else {
    first = offsets[0];
    last = offsets[ncol];
  }
  if (first != 0 || last != n) return fail(DEXEL_EINVAL, "offsets[0] must be 0 and offsets[ncols] == n_intervals");
  Buf off, ep;
  dexel_status s;
  if ((s = dalloc(g, off, sizeof(uint64_t) * (ncol + 1)))) return s;
  if ((s = dalloc(g, ep, sizeof(float) * 2 * (n + 1)))) {
    dfree(g, off);
    return s;
  }
  const cudaMemcpyKind k = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CK(cudaMemcpyAsync(off.p, offsets, sizeof(uint64_t) * (ncol + 1), k, g->stream));
  if (n) CK(cudaMemcpyAsync(ep.p, endpoints, sizeof(float) * 2 * n, k, g->stream));
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
  CK(cudaStreamSynchronize(g->stream));
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

dexel_status dexel_upload(dexel_grid g, const uint64_t* offsets, const float* endpoints, uint64_t n, int on_dev) {
  g_err.clear();
  if (!g) return fail(DEXEL_EINVAL, "NULL handle");
  Buf off, ep;
  dexel_status s = load_csr(g, offsets, endpoints, g->ncol, n, on_dev, &off, &ep);
  if (s) return s;
  dfree(g, g->off);
  dfree(g, g->ep);
  g->off = off;
  g->ep = ep;
  g->n = n;
  return DEXEL_OK;
}

dexel_status dexel_upload_halo(dexel_grid g, int side, const uint64_t* offsets, const float* endpoints, int nrows,
                               uint64_t n, int on_dev) {
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
  dexel_status s = load_csr(g, offsets, endpoints, (int64_t)nrows * g->d.nx, n, on_dev, &off, &ep);
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
  CK(cudaStreamSynchronize(g->stream));
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
  CK(cudaStreamSynchronize(g->stream));
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
  CK(cudaMemcpyAsync(offsets, g->off.p, sizeof(uint64_t) * (g->ncol + 1), k, g->stream));
  if (g->n) CK(cudaMemcpyAsync(endpoints, g->ep.p, sizeof(float) * 2 * g->n, k, g->stream));
  CK(cudaStreamSynchronize(g->stream));
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
  SrcRows rows{(const uint64_t*)g->off.p, (const float*)g->ep.p, g->d.nx, g->nrows, g->d.z_lo, g->d.z_hi};
  Pieces P;
  if ((s = run_pass1(g, T, rows, R, complement ? 1 : 0, 0, g->nrows, &P))) return s;
  *n_pieces = P.m;
  if (cap < P.m) return fail(DEXEL_EOVERFLOW, "capacity < pieces");
  if (!offsets || (P.m && (!z || !kappa))) return fail(DEXEL_EINVAL, "NULL output buffer");
  const cudaMemcpyKind k = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  CK(cudaMemcpyAsync(offsets, P.moff, sizeof(uint64_t) * (g->ncol + 1), k, g->stream));
  if (P.m) {
    CK(cudaMemcpyAsync(z, P.mz, sizeof(float2) * P.m, k, g->stream));
    CK(cudaMemcpyAsync(kappa, P.mk, P.m, k, g->stream));
  }
  CK(cudaStreamSynchronize(g->stream));
  return DEXEL_OK;
}

dexel_status dexel_sync(dexel_grid g) {
  if (!g) return fail(DEXEL_EINVAL, "NULL handle");
  CK(cudaStreamSynchronize(g->stream));
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
  cudaStreamSynchronize(g->stream);
  if (g->own_stream) cudaStreamDestroy(g->stream);
  delete g;
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

}  // extern "C"
