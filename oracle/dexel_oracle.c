/* dexel_oracle.c -- plain, slow, fp64 CPU oracle for the separable dexel
 * dilation / erosion / shell of arXiv 1804.08968.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this.
 * The product path (paper_1804_08968_b200/) never imports it and shares no
 * code, header, helper or table with it.
 *
 * Everything is computed in fp64 from the fp32 canonical input (upcast
 * exactly).  Closed intervals throughout (reading R5): touching
 * intervals merge, zero-length intervals are dropped.
 *
 *  O1  oracle_dilate(method=0): brute force, the definition.
 *      PAPER.md:235-238 (Eq. 1, D_r(S) = points at distance <= r of S)
 *      restricted to the ray lattice, as in the paper's own baseline
 *      PAPER.md:592-594 ("each segment ... generates an explicit list of
 *      dilated segments in a disk of radius r around it, and all overlapping
 *      segments are merged").  For output column c and every lattice column
 *      c' with |c-c'|^2 s^2 <= r^2, each interval [a,b] of c' grows to
 *      [a-h, b+h], h = sqrt(r^2 - |c-c'|^2 s^2); sort, merge, clip to U.
 *
 *  O2  oracle_dilate(method=1): the paper's two passes in plain gather form.
 *      P1 ("extruded, not dilated"; closest parent, P:500;
 *      occlusion P:467-469; expiry at distance r P:470): for output column
 *      (i,j) gather columns (i+dx, j), |dx| <= R, sweep their endpoints in z
 *      order counting active intervals per level |dx|, and emit maximal runs
 *      of the minimum active level kappa as closed pieces (lo, hi, kappa).
 *      P2 (PAPER.md:498-500, 504-510, 538-541, 556-560 + App. B):
 *      each piece of M(i, j+dy) is a segment with power weight
 *      W = r^2 - (kappa^2 + dy^2) s^2 (the printed "sqrt(d^2-r^2)" P:212/500
 *      and "w_i := r_i" P:505 are read as sqrt(r^2-d^2) and r^2, DESIGN.md
 *      readings R1/R2); its dilation along the second axis is the capsule
 *      [lo - sqrt(W), hi + sqrt(W)] (box + endpoint half-disks);
 *      sort, merge, clip.
 *
 *  Erosion  = U \ D_r(C), C = U \ S   (neutral boundary R6)
 *  Shell    = D_rout(S) \ E_rin(S) = D_rout(S) n D_rin(C)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double lo, hi; } iv;
typedef struct { double lo, hi; int k; } piece;

typedef struct {
  int nx, ny;
  const uint64_t* off;
  const float* ep;
  double zlo, zhi, r, s;
  int R;
} grid_in;

/* ---- dynamic arrays ---- */
typedef struct { iv* v; size_t n, cap; } ivec;
static void ivec_push(ivec* a, double lo, double hi) {
  if (a->n == a->cap) { a->cap = a->cap ? 2 * a->cap : 64; a->v = (iv*)realloc(a->v, a->cap * sizeof(iv)); }
  a->v[a->n].lo = lo; a->v[a->n].hi = hi; a->n++;
}
typedef struct { piece* v; size_t n, cap; } pvec;
static void pvec_push(pvec* a, double lo, double hi, int k) {
  if (a->n == a->cap) { a->cap = a->cap ? 2 * a->cap : 64; a->v = (piece*)realloc(a->v, a->cap * sizeof(piece)); }
  a->v[a->n].lo = lo; a->v[a->n].hi = hi; a->v[a->n].k = k; a->n++;
}

static int in_grid(const grid_in* g, int i, int j) { return i >= 0 && i < g->nx && j >= 0 && j < g->ny; }

/* Column (i,j) of S or of its complement C = [zlo,zhi] \ S (closed
 * representation, zero-length pieces dropped), in fp64. */
static void get_column(const grid_in* g, int i, int j, int complement, ivec* out) {
  out->n = 0;
  size_t c = (size_t)j * (size_t)g->nx + (size_t)i;
  uint64_t a = g->off[c], b = g->off[c + 1];
  if (!complement) {
    for (uint64_t t = a; t < b; ++t) ivec_push(out, (double)g->ep[2 * t], (double)g->ep[2 * t + 1]);
    return;
  }
  double cur = g->zlo;
  for (uint64_t t = a; t < b; ++t) {
    double lo = (double)g->ep[2 * t], hi = (double)g->ep[2 * t + 1];
    if (lo > cur) ivec_push(out, cur, lo);
    cur = hi;
  }
  if (g->zhi > cur) ivec_push(out, cur, g->zhi);
}

static int cmp_iv(const void* x, const void* y) {
  double a = ((const iv*)x)->lo, b = ((const iv*)y)->lo;
  if (a < b) return -1;
  if (a > b) return 1;
  double c = ((const iv*)x)->hi, d = ((const iv*)y)->hi;
  return (c > d) - (c < d);
}

/* sort by start, merge (gap <= 0 merges), clip to [zlo,zhi], drop zero-length */
static void union_clip(ivec* v, double zlo, double zhi) {
  if (v->n == 0) return;
  qsort(v->v, v->n, sizeof(iv), cmp_iv);
  size_t k = 0;
  for (size_t t = 1; t < v->n; ++t) {
    if (v->v[t].lo <= v->v[k].hi) {
      if (v->v[t].hi > v->v[k].hi) v->v[k].hi = v->v[t].hi;
    } else {
      v->v[++k] = v->v[t];
    }
  }
  size_t n = k + 1, m = 0;
  for (size_t t = 0; t < n; ++t) {
    double lo = v->v[t].lo < zlo ? zlo : v->v[t].lo;
    double hi = v->v[t].hi > zhi ? zhi : v->v[t].hi;
    if (lo < hi) { v->v[m].lo = lo; v->v[m].hi = hi; ++m; }
  }
  v->n = m;
}

/* power weight W = r^2 - (a^2 + b^2) s^2, one expression shared by O1 and O2 */
static double weight(const grid_in* g, int a, int b) {
  return g->r * g->r - ((double)a * a + (double)b * b) * g->s * g->s;
}

/* ---------------- O1: brute force ---------------- */
static void dilate_brute_col(const grid_in* g, int i, int j, int complement, ivec* out, ivec* col) {
  out->n = 0;
  for (int dy = -g->R; dy <= g->R; ++dy)
    for (int dx = -g->R; dx <= g->R; ++dx) {
      if (!in_grid(g, i + dx, j + dy)) continue;
      double W = weight(g, dx, dy);
      if (W < 0) continue;
      double h = sqrt(W);
      get_column(g, i + dx, j + dy, complement, col);
      for (size_t t = 0; t < col->n; ++t) ivec_push(out, col->v[t].lo - h, col->v[t].hi + h);
    }
  union_clip(out, g->zlo, g->zhi);
}

/* ---------------- O2 pass 1: closest-parent extrusion ---------------- */
typedef struct { double z; int level; int delta; } event;
static int cmp_ev(const void* x, const void* y) {
  double a = ((const event*)x)->z, b = ((const event*)y)->z;
  return (a > b) - (a < b);
}

static void pass1_col(const grid_in* g, int i, int j, int complement, pvec* out, ivec* col,
                      event** evbuf, size_t* evcap, int* cnt) {
  out->n = 0;
  size_t ne = 0;
  for (int dx = -g->R; dx <= g->R; ++dx) {
    if (!in_grid(g, i + dx, j)) continue;
    if (weight(g, dx, 0) < 0) continue;
    get_column(g, i + dx, j, complement, col);
    int level = dx < 0 ? -dx : dx;
    for (size_t t = 0; t < col->n; ++t) {
      if (ne + 2 > *evcap) { *evcap = *evcap ? 2 * *evcap : 256; *evbuf = (event*)realloc(*evbuf, *evcap * sizeof(event)); }
      (*evbuf)[ne++] = (event){col->v[t].lo, level, +1};
      (*evbuf)[ne++] = (event){col->v[t].hi, level, -1};
    }
  }
  if (ne == 0) return;
  event* ev = *evbuf;
  qsort(ev, ne, sizeof(event), cmp_ev);
  for (int l = 0; l <= g->R; ++l) cnt[l] = 0;
  int cur = -1;            /* current min active level, -1 = none */
  double start = 0.0;
  size_t t = 0;
  while (t < ne) {
    double z = ev[t].z;
    while (t < ne && ev[t].z == z) { cnt[ev[t].level] += ev[t].delta; ++t; }
    int k = -1;
    for (int l = 0; l <= g->R; ++l) if (cnt[l] > 0) { k = l; break; }
    if (k != cur) {
      if (cur >= 0) pvec_push(out, start, z, cur);   /* z > start: groups have distinct z */
      cur = k;
      start = z;
    }
  }
}

/* ---------------- O2 pass 2: power dilation of pieces along y ---------------- */
static void pass2_col(const grid_in* g, pvec* const* M /* per dy+R, NULL if outside */,
                      ivec* out) {
  out->n = 0;
  for (int dy = -g->R; dy <= g->R; ++dy) {
    const pvec* p = M[dy + g->R];
    if (!p) continue;
    for (size_t t = 0; t < p->n; ++t) {
      double W = weight(g, p->v[t].k, dy);
      if (W < 0) continue;
      double h = sqrt(W);
      ivec_push(out, p->v[t].lo - h, p->v[t].hi + h);
    }
  }
  union_clip(out, g->zlo, g->zhi);
}

/* ---------------- per-column set operations ---------------- */
static void complement_within(const ivec* a, double zlo, double zhi, ivec* out) {
  out->n = 0;
  double cur = zlo;
  for (size_t t = 0; t < a->n; ++t) {
    if (a->v[t].lo > cur) ivec_push(out, cur, a->v[t].lo);
    cur = a->v[t].hi;
  }
  if (zhi > cur) ivec_push(out, cur, zhi);
}

static void intersect(const ivec* a, const ivec* b, ivec* out) {
  out->n = 0;
  size_t p = 0, q = 0;
  while (p < a->n && q < b->n) {
    double lo = a->v[p].lo > b->v[q].lo ? a->v[p].lo : b->v[q].lo;
    double hi = a->v[p].hi < b->v[q].hi ? a->v[p].hi : b->v[q].hi;
    if (lo < hi) ivec_push(out, lo, hi);
    if (a->v[p].hi < b->v[q].hi) ++p; else ++q;
  }
}

/* ---------------- driver ---------------- */
enum { OP_DILATE = 0, OP_ERODE = 1, OP_SHELL = 2, OP_PASS1 = 3 };

typedef struct {
  grid_in g, g2;            /* g2: second radius (shell r_in) */
  int op, method, complement;
  const int64_t* cols; int64_t ncols;
  /* P1 cache for O2: per column pointer (NULL = not needed) */
  pvec** P1a; pvec** P1b;   /* for S (or C) with g, and C with g2 (shell) */
  int64_t* need; int64_t nneed;
  /* outputs */
  ivec* res; pvec* pres;
  volatile int64_t next;
  int phase;
} job;

static void compute_p1_cache(job* J, int64_t t, ivec* col, event** eb, size_t* ec, int* cnt) {
  int64_t c = J->need[t];
  int i = (int)(c % J->g.nx), j = (int)(c / J->g.nx);
  /* P1a: dilate -> S (or C if complement), erode -> C, shell -> S (radius r_out) */
  int compA = J->op == OP_DILATE ? J->complement : (J->op == OP_ERODE ? 1 : 0);
  if (J->P1a) pass1_col(&J->g, i, j, compA, J->P1a[c], col, eb, ec, cnt);
  /* P1b: shell only -> C (radius r_in) */
  if (J->P1b) pass1_col(&J->g2, i, j, 1, J->P1b[c], col, eb, ec, cnt);
}

static void dilate_sep(job* J, const grid_in* g, pvec** P1, int i, int j, ivec* out) {
  pvec* M[512];
  for (int dy = -g->R; dy <= g->R; ++dy)
    M[dy + g->R] = in_grid(g, i, j + dy) ? P1[(size_t)(j + dy) * g->nx + i] : NULL;
  pass2_col(g, M, out);
  (void)J;
}

static void* worker(void* arg) {
  job* J = (job*)arg;
  ivec col = {0}, d1 = {0}, d2 = {0};
  event* eb = NULL; size_t ec = 0;
  int* cnt = (int*)malloc(sizeof(int) * 600);
  for (;;) {
    int64_t t = __sync_fetch_and_add(&J->next, 64);
    int64_t lim = J->phase == 0 ? J->nneed : J->ncols;
    if (t >= lim) break;
    int64_t e = t + 64 < lim ? t + 64 : lim;
    for (; t < e; ++t) {
      if (J->phase == 0) { compute_p1_cache(J, t, &col, &eb, &ec, cnt); continue; }
      int64_t c = J->cols[t];
      int i = (int)(c % J->g.nx), j = (int)(c / J->g.nx);
      if (J->op == OP_PASS1) {
        pass1_col(&J->g, i, j, J->complement, &J->pres[t], &col, &eb, &ec, cnt);
        continue;
      }
      ivec* out = &J->res[t];
      if (J->op == OP_DILATE) {
        if (J->method == 0) dilate_brute_col(&J->g, i, j, J->complement, out, &col);
        else dilate_sep(J, &J->g, J->P1a, i, j, out);
      } else if (J->op == OP_ERODE) {
        if (J->method == 0) dilate_brute_col(&J->g, i, j, 1, &d1, &col);
        else dilate_sep(J, &J->g, J->P1a, i, j, &d1);
        complement_within(&d1, J->g.zlo, J->g.zhi, out);
      } else { /* shell */
        if (J->method == 0) {
          dilate_brute_col(&J->g, i, j, 0, &d1, &col);
          dilate_brute_col(&J->g2, i, j, 1, &d2, &col);
        } else {
          dilate_sep(J, &J->g, J->P1a, i, j, &d1);
          dilate_sep(J, &J->g2, J->P1b, i, j, &d2);
        }
        intersect(&d1, &d2, out);
      }
    }
  }
  free(col.v); free(d1.v); free(d2.v); free(eb); free(cnt);
  return NULL;
}

static void run_threads(job* J, int nthreads) {
  pthread_t th[256];
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  J->next = 0;
  for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], NULL, worker, J);
  for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
}

static int radius_levels(double r, double s) {
  int R = (int)floor(r / s);
  while ((double)(R + 1) * s <= r) ++R;          /* guard floor() rounding */
  while (R > 0 && (double)R * s > r) --R;
  return R;
}

/* op: 0 dilate, 1 erode, 2 shell, 3 pass1.  method: 0 brute force (O1), 1 separable (O2).
 * cols: output column ids (NULL -> all).  Results malloc'ed, free with oracle_free.
 * Returns 0, or -1 on invalid arguments (R > 255 or r < 0). */
int oracle_run(int op, int method, int nx, int ny, const uint64_t* off, const float* ep,
               double zlo, double zhi, double r, double r2, double s, int complement,
               const int64_t* cols, int64_t ncols, int nthreads,
               uint64_t** out_off, double** out_z, uint8_t** out_k, uint64_t* out_n) {
  if (!(r >= 0) || !(r2 >= 0) || !(s > 0)) return -1;
  job J;
  memset(&J, 0, sizeof(J));
  J.g = (grid_in){nx, ny, off, ep, zlo, zhi, r, s, radius_levels(r, s)};
  J.g2 = (grid_in){nx, ny, off, ep, zlo, zhi, r2, s, radius_levels(r2, s)};
  if (J.g.R > 255 || J.g2.R > 255) return -1;
  J.op = op; J.method = method; J.complement = complement;
  int64_t ncol = (int64_t)nx * ny;
  int64_t* all = NULL;
  if (!cols) {
    all = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ncol > 0 ? ncol : 1));
    for (int64_t c = 0; c < ncol; ++c) all[c] = c;
    cols = all; ncols = ncol;
  }
  J.cols = cols; J.ncols = ncols;
  if (op == OP_PASS1) J.pres = (pvec*)calloc((size_t)(ncols > 0 ? ncols : 1), sizeof(pvec));
  else J.res = (ivec*)calloc((size_t)(ncols > 0 ? ncols : 1), sizeof(ivec));

  if (method == 1 && op != OP_PASS1) {
    /* O2: pass 1 once for every column some requested output needs (row neighbours). */
    uint8_t* mark = (uint8_t*)calloc((size_t)ncol, 1);
    int Rm = J.g.R > J.g2.R ? J.g.R : J.g2.R;
    int64_t nneed = 0;
    for (int64_t t = 0; t < ncols; ++t) {
      int i = (int)(cols[t] % nx), j = (int)(cols[t] / nx);
      for (int dy = -Rm; dy <= Rm; ++dy)
        if (j + dy >= 0 && j + dy < ny) {
          size_t c = (size_t)(j + dy) * nx + i;
          if (!mark[c]) { mark[c] = 1; ++nneed; }
        }
    }
    J.need = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nneed > 0 ? nneed : 1));
    int64_t q = 0;
    for (int64_t c = 0; c < ncol; ++c) if (mark[c]) J.need[q++] = c;
    J.nneed = nneed;
    J.P1a = (pvec**)calloc((size_t)ncol, sizeof(pvec*));
    pvec* storeA = (pvec*)calloc((size_t)(nneed > 0 ? nneed : 1), sizeof(pvec));
    pvec* storeB = NULL;
    for (int64_t t = 0; t < nneed; ++t) J.P1a[J.need[t]] = &storeA[t];
    if (op == OP_SHELL) {
      J.P1b = (pvec**)calloc((size_t)ncol, sizeof(pvec*));
      storeB = (pvec*)calloc((size_t)(nneed > 0 ? nneed : 1), sizeof(pvec));
      for (int64_t t = 0; t < nneed; ++t) J.P1b[J.need[t]] = &storeB[t];
    }
    free(mark);
    J.phase = 0;
    run_threads(&J, nthreads);
    J.phase = 1;
    run_threads(&J, nthreads);
    for (int64_t t = 0; t < nneed; ++t) { free(storeA[t].v); if (storeB) free(storeB[t].v); }
    free(storeA); free(storeB); free(J.P1a); free(J.P1b); free(J.need);
  } else {
    J.phase = 1;
    run_threads(&J, nthreads);
  }

  uint64_t tot = 0;
  for (int64_t t = 0; t < ncols; ++t) tot += op == OP_PASS1 ? J.pres[t].n : J.res[t].n;
  uint64_t* o = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(ncols + 1));
  double* z = (double*)malloc(sizeof(double) * (2 * tot + 2));
  uint8_t* kk = op == OP_PASS1 ? (uint8_t*)malloc(tot + 1) : NULL;
  uint64_t w = 0;
  for (int64_t t = 0; t < ncols; ++t) {
    o[t] = w;
    if (op == OP_PASS1) {
      for (size_t u = 0; u < J.pres[t].n; ++u) {
        z[2 * w] = J.pres[t].v[u].lo; z[2 * w + 1] = J.pres[t].v[u].hi; kk[w] = (uint8_t)J.pres[t].v[u].k; ++w;
      }
      free(J.pres[t].v);
    } else {
      for (size_t u = 0; u < J.res[t].n; ++u) { z[2 * w] = J.res[t].v[u].lo; z[2 * w + 1] = J.res[t].v[u].hi; ++w; }
      free(J.res[t].v);
    }
  }
  o[ncols] = w;
  free(J.res); free(J.pres); free(all);
  *out_off = o; *out_z = z; if (out_k) *out_k = kk; else free(kk); *out_n = tot;
  return 0;
}

void oracle_free(void* p) { free(p); }
