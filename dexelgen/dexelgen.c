/* dexelgen.c -- seeded synthetic solids -> canonical fp32 dexel CSR.
 *
 * Input generator shared by the oracle and the CUDA path (SURVEY.md 8(d),
 * "Generator").  It holds none of the method's arithmetic: it only rasterises
 * analytic solids (sphere chords, boxes, a noisy gyroid) onto the ray lattice
 * and performs the per-column CSG that *defines* the input solid
 * (PAPER.md:42 / :174 "CSG operations can be carried out easily in dexel
 * space").  Nothing here dilates or erodes.
 *
 * Conventions:
 *   - column (i,j) is the ray at lateral position ((i+1/2)s, (j+1/2)s), s = 1;
 *     linear column index j*nx + i (i fastest, SPEC.md:110 row-major order);
 *   - solids are evaluated in fp64 in world coordinates, clipped to the z
 *     domain [zmin,zmax], shifted to the local frame z - z_ref with
 *     z_ref = (zmin+zmax)/2, rounded to fp32, and canonicalised: intervals
 *     strictly increasing, touching/overlapping merged, zero-length dropped.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double lo, hi; } ivl;

/* ---- counter-based RNG (splitmix64 finaliser over a keyed counter) ---- */
static uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
uint64_t dexelgen_u64(uint64_t seed, uint64_t stream, uint64_t index) {
  return mix64(mix64(mix64(seed) ^ (stream * 0xD1B54A32D192ED03ULL)) ^ index);
}
double dexelgen_uniform(uint64_t seed, uint64_t stream, uint64_t index) {
  return (double)(dexelgen_u64(seed, stream, index) >> 11) * (1.0 / 9007199254740992.0);
}

static int cmp_ivl(const void* a, const void* b) {
  double x = ((const ivl*)a)->lo, y = ((const ivl*)b)->lo;
  return (x > y) - (x < y);
}

/* union of n intervals in place (sort + merge, gap <= 0 merges); returns count */
static int union_inplace(ivl* v, int n) {
  if (n <= 1) return n;
  qsort(v, (size_t)n, sizeof(ivl), cmp_ivl);
  int k = 0;
  for (int t = 1; t < n; ++t) {
    if (v[t].lo <= v[k].hi) {
      if (v[t].hi > v[k].hi) v[k].hi = v[t].hi;
    } else {
      v[++k] = v[t];
    }
  }
  return k + 1;
}

/* a \ b for sorted disjoint lists; writes into out (capacity na+nb+1) */
static int difference(const ivl* a, int na, const ivl* b, int nb, ivl* out) {
  int k = 0, jb = 0;
  for (int ia = 0; ia < na; ++ia) {
    double lo = a[ia].lo, hi = a[ia].hi;
    while (jb < nb && b[jb].hi <= lo) ++jb;
    int t = jb;
    while (t < nb && b[t].lo < hi) {
      if (b[t].lo > lo) out[k++] = (ivl){lo, b[t].lo};
      if (b[t].hi > lo) lo = b[t].hi;
      if (lo >= hi) break;
      ++t;
    }
    if (lo < hi) out[k++] = (ivl){lo, hi};
  }
  return k;
}

/* clip to [zmin,zmax], shift to local frame, round to fp32, canonicalise */
static int finish_column(const ivl* v, int n, double zmin, double zmax, double zref, float* dst) {
  int k = 0;
  for (int t = 0; t < n; ++t) {
    double lo = v[t].lo < zmin ? zmin : v[t].lo;
    double hi = v[t].hi > zmax ? zmax : v[t].hi;
    if (!(lo < hi)) continue;
    float a = (float)(lo - zref), b = (float)(hi - zref);
    if (k > 0 && a <= dst[2 * k - 1]) {          /* touches/overlaps after rounding */
      if (b > dst[2 * k - 1]) dst[2 * k - 1] = b;
      continue;
    }
    if (!(a < b)) continue;                       /* zero length after rounding */
    dst[2 * k] = a;
    dst[2 * k + 1] = b;
    ++k;
  }
  return k;
}

/* ------------------------------------------------------------------------ */
/* Shapes: spheres (cx,cy,cz,R) and boxes (x0,x1,y0,y1,z0,z1), each with a
 * sign (+1 solid, -1 void).  Result = (U positives) \ (U negatives).        */
typedef struct {
  int nx, ny;
  double zmin, zmax, zref;
  int nsph; const double* sph; const int* sph_sign;
  int nbox; const double* box; const int* box_sign;
  /* per-row shape lists (CSR over rows) */
  const int64_t* row_off; const int32_t* row_ids; /* ids: sphere k -> k, box k -> nsph+k */
  /* output: per-row buffers */
  float** row_ep; int32_t** row_cnt; int64_t* row_tot;
  int next_row; pthread_mutex_t mu;
} raster_job;

typedef struct { int32_t col; int32_t sign; double lo, hi; } chord;
typedef struct { chord* v; size_t n, cap; } chordvec;

static void push_chord(chordvec* cv, int col, int sign, double lo, double hi) {
  if (cv->n == cv->cap) {
    cv->cap = cv->cap ? 2 * cv->cap : 4096;
    cv->v = (chord*)realloc(cv->v, sizeof(chord) * cv->cap);
  }
  cv->v[cv->n++] = (chord){col, sign, lo, hi};
}

typedef struct {
  chordvec cv;
  int64_t* start;      /* nx+1 */
  ivl* sorted;         /* grouped by column */
  int32_t* sgn;
  size_t scap;
  ivl* P; ivl* N; ivl* tmp; float* colbuf; size_t ccap;
} raster_ws;

static void raster_row(raster_job* J, int j, raster_ws* W) {
  int nx = J->nx;
  double y = j + 0.5;
  W->cv.n = 0;
  for (int64_t t = J->row_off[j]; t < J->row_off[j + 1]; ++t) {
    int id = J->row_ids[t];
    if (id < J->nsph) {
      const double* s = J->sph + 4 * (size_t)id;
      double dy = y - s[1], R = s[3];
      double rr = R * R - dy * dy;
      if (rr <= 0) continue;
      double hx = sqrt(rr);
      int i0 = (int)ceil(s[0] - hx - 0.5), i1 = (int)floor(s[0] + hx - 0.5);
      if (i0 < 0) i0 = 0;
      if (i1 > nx - 1) i1 = nx - 1;
      for (int i = i0; i <= i1; ++i) {
        double dx = (i + 0.5) - s[0];
        double q = rr - dx * dx;
        if (q <= 0) continue;
        double h = sqrt(q);
        push_chord(&W->cv, i, J->sph_sign[id], s[2] - h, s[2] + h);
      }
    } else {
      int b = id - J->nsph;
      const double* x = J->box + 6 * (size_t)b;
      if (y < x[2] || y > x[3]) continue;
      int i0 = (int)ceil(x[0] - 0.5), i1 = (int)floor(x[1] - 0.5);
      if (i0 < 0) i0 = 0;
      if (i1 > nx - 1) i1 = nx - 1;
      for (int i = i0; i <= i1; ++i) push_chord(&W->cv, i, J->box_sign[b], x[4], x[5]);
    }
  }
  /* counting sort by column */
  for (int i = 0; i <= nx; ++i) W->start[i] = 0;
  for (size_t t = 0; t < W->cv.n; ++t) W->start[W->cv.v[t].col + 1]++;
  for (int i = 0; i < nx; ++i) W->start[i + 1] += W->start[i];
  if (W->cv.n > W->scap) {
    W->scap = W->cv.n;
    W->sorted = (ivl*)realloc(W->sorted, sizeof(ivl) * W->scap);
    W->sgn = (int32_t*)realloc(W->sgn, sizeof(int32_t) * W->scap);
  }
  {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nx + 1));
    memcpy(fill, W->start, sizeof(int64_t) * (size_t)(nx + 1));
    for (size_t t = 0; t < W->cv.n; ++t) {
      int64_t p = fill[W->cv.v[t].col]++;
      W->sorted[p] = (ivl){W->cv.v[t].lo, W->cv.v[t].hi};
      W->sgn[p] = W->cv.v[t].sign;
    }
    free(fill);
  }
  int64_t tot = 0;
  int32_t* cnt = (int32_t*)malloc(sizeof(int32_t) * (size_t)nx);
  size_t outcap = 1024;
  float* out = (float*)malloc(sizeof(float) * outcap);
  for (int i = 0; i < nx; ++i) {
    size_t m = (size_t)(W->start[i + 1] - W->start[i]);
    if (m + 2 > W->ccap) {
      W->ccap = 2 * (m + 2);
      W->P = (ivl*)realloc(W->P, sizeof(ivl) * W->ccap);
      W->N = (ivl*)realloc(W->N, sizeof(ivl) * W->ccap);
      W->tmp = (ivl*)realloc(W->tmp, sizeof(ivl) * 2 * W->ccap);
      W->colbuf = (float*)realloc(W->colbuf, sizeof(float) * 4 * W->ccap);
    }
    int np = 0, nn = 0;
    for (int64_t t = W->start[i]; t < W->start[i + 1]; ++t) {
      if (W->sgn[t] > 0) W->P[np++] = W->sorted[t]; else W->N[nn++] = W->sorted[t];
    }
    np = union_inplace(W->P, np);
    nn = union_inplace(W->N, nn);
    int nd = difference(W->P, np, W->N, nn, W->tmp);
    int k = finish_column(W->tmp, nd, J->zmin, J->zmax, J->zref, W->colbuf);
    cnt[i] = k;
    if ((size_t)(tot + k) * 2 > outcap) {
      while ((size_t)(tot + k) * 2 > outcap) outcap *= 2;
      out = (float*)realloc(out, sizeof(float) * outcap);
    }
    memcpy(out + 2 * tot, W->colbuf, sizeof(float) * 2 * (size_t)k);
    tot += k;
  }
  J->row_ep[j] = out;
  J->row_cnt[j] = cnt;
  J->row_tot[j] = tot;
}

static void* raster_worker(void* arg) {
  raster_job* J = (raster_job*)arg;
  raster_ws W;
  memset(&W, 0, sizeof(W));
  W.start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(J->nx + 1));
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int j = J->next_row++;
    pthread_mutex_unlock(&J->mu);
    if (j >= J->ny) break;
    raster_row(J, j, &W);
  }
  free(W.cv.v); free(W.start); free(W.sorted); free(W.sgn);
  free(W.P); free(W.N); free(W.tmp); free(W.colbuf);
  return NULL;
}

/* Assemble per-row outputs into one CSR (malloc'ed; free with dexelgen_free). */
static int assemble(int nx, int ny, float** row_ep, int32_t** row_cnt, int64_t* row_tot,
                    uint64_t** off_out, float** ep_out, uint64_t* n_out) {
  uint64_t n = 0;
  for (int j = 0; j < ny; ++j) n += (uint64_t)row_tot[j];
  uint64_t* off = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)nx * ny + 1));
  float* ep = (float*)malloc(sizeof(float) * (2 * (size_t)n + 2));
  if (!off || !ep) return -1;
  uint64_t o = 0;
  for (int j = 0; j < ny; ++j) {
    for (int i = 0; i < nx; ++i) { off[(size_t)j * nx + i] = o; o += (uint64_t)row_cnt[j][i]; }
    memcpy(ep + 2 * (off[(size_t)j * nx]), row_ep[j], sizeof(float) * 2 * (size_t)row_tot[j]);
    free(row_ep[j]); free(row_cnt[j]);
  }
  off[(size_t)nx * ny] = o;
  *off_out = off; *ep_out = ep; *n_out = n;
  return 0;
}

int dexelgen_shapes(int nx, int ny, double zmin, double zmax,
                    int nsph, const double* sph, const int* sph_sign,
                    int nbox, const double* box, const int* box_sign,
                    int nthreads, uint64_t** off_out, float** ep_out, uint64_t* n_out) {
  /* bin shapes by rows */
  int64_t* rc = (int64_t*)calloc((size_t)ny + 1, sizeof(int64_t));
  int nsh = nsph + nbox;
  int* r0 = (int*)malloc(sizeof(int) * (size_t)(nsh + 1));
  int* r1 = (int*)malloc(sizeof(int) * (size_t)(nsh + 1));
  for (int k = 0; k < nsh; ++k) {
    double ylo, yhi;
    if (k < nsph) { ylo = sph[4 * k + 1] - sph[4 * k + 3]; yhi = sph[4 * k + 1] + sph[4 * k + 3]; }
    else { const double* x = box + 6 * (k - nsph); ylo = x[2]; yhi = x[3]; }
    int a = (int)floor(ylo - 0.5), b = (int)ceil(yhi - 0.5);
    if (a < 0) a = 0;
    if (b > ny - 1) b = ny - 1;
    r0[k] = a; r1[k] = b;
    for (int j = a; j <= b; ++j) rc[j + 1]++;
  }
  for (int j = 0; j < ny; ++j) rc[j + 1] += rc[j];
  int32_t* ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(rc[ny] + 1));
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ny + 1));
  memcpy(fill, rc, sizeof(int64_t) * (size_t)(ny + 1));
  for (int k = 0; k < nsh; ++k)
    for (int j = r0[k]; j <= r1[k]; ++j) ids[fill[j]++] = k;
  free(fill); free(r0); free(r1);

  raster_job J;
  memset(&J, 0, sizeof(J));
  J.nx = nx; J.ny = ny; J.zmin = zmin; J.zmax = zmax; J.zref = 0.5 * (zmin + zmax);
  J.nsph = nsph; J.sph = sph; J.sph_sign = sph_sign;
  J.nbox = nbox; J.box = box; J.box_sign = box_sign;
  J.row_off = rc; J.row_ids = ids;
  J.row_ep = (float**)calloc((size_t)ny, sizeof(float*));
  J.row_cnt = (int32_t**)calloc((size_t)ny, sizeof(int32_t*));
  J.row_tot = (int64_t*)calloc((size_t)ny, sizeof(int64_t));
  pthread_mutex_init(&J.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, raster_worker, &J);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&J.mu);
  int rc2 = assemble(nx, ny, J.row_ep, J.row_cnt, J.row_tot, off_out, ep_out, n_out);
  free(J.row_ep); free(J.row_cnt); free(J.row_tot); free(rc); free(ids);
  return rc2;
}

/* ------------------------------------------------------------------------ */
/* Noisy gyroid (config C3): F = sin X cos Y + sin Y cos Z + sin Z cos X,
 * X = 2 pi x / period (same for Y, Z); solid where F + eps > t.  F + eps is
 * sampled at z = m + 1/2 (m = 0..nz-1), eps ~ U[-amp, amp] i.i.d. per
 * (column, m) from the counter RNG (stream 6), linearly interpolated in z;
 * endpoints are the linear roots between samples.  Beyond the first/last
 * sample the field is held constant (clipped to the domain).             */
typedef struct {
  int n, nz; double period, t, amp; uint64_t seed;
  float** row_ep; int32_t** row_cnt; int64_t* row_tot;
  int next_row; pthread_mutex_t mu;
} gyroid_job;

static void* gyroid_worker(void* arg) {
  gyroid_job* G = (gyroid_job*)arg;
  int n = G->n, nz = G->nz;
  double w = 2.0 * M_PI / G->period;
  double* f = (double*)malloc(sizeof(double) * (size_t)nz);
  double* sz = (double*)malloc(sizeof(double) * (size_t)nz);
  double* cz = (double*)malloc(sizeof(double) * (size_t)nz);
  for (int m = 0; m < nz; ++m) { sz[m] = sin(w * (m + 0.5)); cz[m] = cos(w * (m + 0.5)); }
  ivl* v = (ivl*)malloc(sizeof(ivl) * (size_t)(nz + 2));
  float* colbuf = (float*)malloc(sizeof(float) * (size_t)(2 * nz + 4));
  double zref = 0.5 * nz;
  for (;;) {
    pthread_mutex_lock(&G->mu);
    int j = G->next_row++;
    pthread_mutex_unlock(&G->mu);
    if (j >= n) break;
    int32_t* cnt = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    size_t outcap = 4096;
    float* out = (float*)malloc(sizeof(float) * outcap);
    int64_t tot = 0;
    double sy = sin(w * (j + 0.5)), cy = cos(w * (j + 0.5));
    for (int i = 0; i < n; ++i) {
      double sx = sin(w * (i + 0.5)), cx = cos(w * (i + 0.5));
      uint64_t col = (uint64_t)j * (uint64_t)n + (uint64_t)i;
      for (int m = 0; m < nz; ++m) {
        double eps = G->amp * (2.0 * dexelgen_uniform(G->seed, 6, col * (uint64_t)nz + (uint64_t)m) - 1.0);
        f[m] = sx * cy + sy * cz[m] + sz[m] * cx + eps - G->t;   /* solid where > 0 */
      }
      int k = 0;
      int inside = f[0] > 0;
      double start = 0.0;
      for (int m = 0; m + 1 < nz; ++m) {
        int nin = f[m + 1] > 0;
        if (nin != inside) {
          double zc = (m + 0.5) + f[m] / (f[m] - f[m + 1]);   /* linear root */
          if (nin) start = zc;
          else v[k++] = (ivl){start, zc};
          inside = nin;
        }
      }
      if (inside) v[k++] = (ivl){start, (double)nz};
      int kk = finish_column(v, k, 0.0, (double)nz, zref, colbuf);
      cnt[i] = kk;
      if ((size_t)(tot + kk) * 2 > outcap) {
        while ((size_t)(tot + kk) * 2 > outcap) outcap *= 2;
        out = (float*)realloc(out, sizeof(float) * outcap);
      }
      memcpy(out + 2 * tot, colbuf, sizeof(float) * 2 * (size_t)kk);
      tot += kk;
    }
    G->row_ep[j] = out; G->row_cnt[j] = cnt; G->row_tot[j] = tot;
  }
  free(f); free(sz); free(cz); free(v); free(colbuf);
  return NULL;
}

int dexelgen_gyroid(int n, double period, double t, double amp, uint64_t seed, int nthreads,
                    uint64_t** off_out, float** ep_out, uint64_t* n_out) {
  gyroid_job G;
  memset(&G, 0, sizeof(G));
  G.n = n; G.nz = n; G.period = period; G.t = t; G.amp = amp; G.seed = seed;
  G.row_ep = (float**)calloc((size_t)n, sizeof(float*));
  G.row_cnt = (int32_t**)calloc((size_t)n, sizeof(int32_t*));
  G.row_tot = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  pthread_mutex_init(&G.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], NULL, gyroid_worker, &G);
  for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
  free(th);
  pthread_mutex_destroy(&G.mu);
  int rc = assemble(n, n, G.row_ep, G.row_cnt, G.row_tot, off_out, ep_out, n_out);
  free(G.row_ep); free(G.row_cnt); free(G.row_tot);
  return rc;
}

void dexelgen_free(void* p) { free(p); }
