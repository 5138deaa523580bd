/*
 * synth/gen.c — seeded synthetic graph generators shared by the CUDA path's
 * tests/bench and by the oracle's tests.
 *
 * This module holds NONE of the method's arithmetic (no matvec, no BFS, no
 * direction rule).  It only builds input graphs in CSR form, following the
 * paper's preprocessing (Sec. 7.1): "All datasets have been
 * converted to undirected graphs. Self-loops and duplicated edges are removed."
 *
 * Generators
 *   - RMAT / Kronecker with Graph500 parameters (a,b,c,d) = (.57,.19,.19,.05)
 *     (the paper does not state them; this reproduces Table 3's
 *     nnz within 0.5%, SURVEY.md pin P1).  Counter-based RNG (splitmix64 keyed
 *     by (seed, edge index)), so every edge can be regenerated independently,
 *     in parallel, bit-identically on any machine.  Optional seeded bijective
 *     vertex scramble.
 *   - 2-D 4-neighbour grid (config C4) and a bond-percolated grid restricted to
 *     its giant component (the road-like variant of C4).
 *   - Generic edge-list preprocessing (self-loop removal, optional
 *     symmetrisation, dedup, sorted rows).
 *
 * Output: CSR with int64 row offsets (n+1) and uint32 column ids (sorted,
 * unique within each row).  For the symmetric graphs generated here CSR == CSC.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef struct {
  int64_t n;
  int64_t nnz;
  int64_t* off;  /* n+1 */
  uint32_t* idx; /* nnz */
} synth_graph;

static inline uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* uniform double in [0,1) from 53 high bits */
static inline double u01(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

/* Bijective scramble of [0, 2^scale): alternating odd-multiply (mod 2^s) and
 * xor-shift rounds, keyed by the seed.  Each round is a bijection on s bits. */
typedef struct { uint64_t mask; int s; uint64_t m1, a1, m2, a2, m3; } scrambler;

static scrambler make_scrambler(int scale, uint64_t seed) {
  scrambler q;
  q.s = scale;
  q.mask = (scale >= 64) ? ~0ull : ((1ull << scale) - 1);
  q.m1 = sm64(seed ^ 0x1234567ull) | 1ull;
  q.a1 = sm64(seed ^ 0x2345678ull);
  q.m2 = sm64(seed ^ 0x3456789ull) | 1ull;
  q.a2 = sm64(seed ^ 0x456789Aull);
  q.m3 = sm64(seed ^ 0x56789ABull) | 1ull;
  return q;
}

static inline uint64_t scramble(const scrambler* q, uint64_t x) {
  int h = q->s / 2 + 1;
  if (q->s == 0) return 0;
  x = (x * q->m1 + q->a1) & q->mask;
  x ^= x >> h;
  x = (x * q->m2 + q->a2) & q->mask;
  x ^= x >> h;
  x = (x * q->m3) & q->mask;
  x ^= x >> (h > 1 ? h - 1 : 1);
  return x & q->mask;
}

/* One RMAT edge: `scale` recursive quadrant choices.  Each splitmix64 draw
 * supplies two 32-bit uniforms; the quadrant thresholds are a, a+b, a+b+c
 * scaled to 2^32 (quantisation 2^-32). */
static inline void rmat_edge(uint64_t seed, uint64_t k, int scale, uint64_t ta, uint64_t tab, uint64_t tabc,
                             uint64_t* pu, uint64_t* pv) {
  uint64_t st = sm64(seed * 0x100000001B3ull ^ (k * 0xD1B54A32D192ED03ull));
  uint64_t u = 0, v = 0, r64 = 0;
  for (int l = 0; l < scale; ++l) {
    uint64_t r;
    if ((l & 1) == 0) { st = sm64(st + (uint64_t)l); r64 = st; r = r64 >> 32; }
    else r = r64 & 0xFFFFFFFFull;
    uint64_t bu = (r >= tab), bv = (r >= ta && r < tab) || (r >= tabc);
    u = (u << 1) | bu;
    v = (v << 1) | bv;
  }
  *pu = u;
  *pv = v;
}

static void sort_u32(uint32_t* a, int64_t len) {
  while (len > 24) {
    uint32_t x = a[0], y = a[len / 2], z = a[len - 1];
    uint32_t piv = (x < y) ? ((y < z) ? y : (x < z ? z : x)) : ((x < z) ? x : (y < z ? z : y));
    int64_t i = 0, j = len - 1;
    while (i <= j) {
      while (a[i] < piv) ++i;
      while (a[j] > piv) --j;
      if (i <= j) { uint32_t t = a[i]; a[i] = a[j]; a[j] = t; ++i; --j; }
    }
    /* recurse on the smaller part, loop on the larger */
    if (j + 1 < len - i) { sort_u32(a, j + 1); a += i; len -= i; }
    else { sort_u32(a + i, len - i); len = j + 1; }
  }
  for (int64_t i = 1; i < len; ++i) {
    uint32_t t = a[i];
    int64_t j = i - 1;
    while (j >= 0 && a[j] > t) { a[j + 1] = a[j]; --j; }
    a[j + 1] = t;
  }
}

/* Sort + dedup every row in place; returns the compacted graph (buckets freed). */
static synth_graph* finish_rows(int64_t n, int64_t* start, int64_t* fill, uint32_t* buf) {
  int64_t* deg = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i) {
    uint32_t* r = buf + start[i];
    int64_t len = fill[i] - start[i];
    if (len > 1) sort_u32(r, len);
    int64_t w = 0;
    for (int64_t j = 0; j < len; ++j)
      if (w == 0 || r[j] != r[w - 1]) r[w++] = r[j];
    deg[i] = w;
  }
  synth_graph* g = (synth_graph*)calloc(1, sizeof(synth_graph));
  g->n = n;
  g->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  g->off[0] = 0;
  for (int64_t i = 0; i < n; ++i) g->off[i + 1] = g->off[i] + deg[i];
  g->nnz = g->off[n];
  g->idx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(g->nnz > 0 ? g->nnz : 1));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i)
    memcpy(g->idx + g->off[i], buf + start[i], sizeof(uint32_t) * (size_t)deg[i]);
  free(deg);
  return g;
}

/* RMAT/Kronecker graph, symmetrised, self-loops and duplicates removed. */
synth_graph* synth_rmat(int scale, int64_t edgefactor, uint64_t seed, int do_scramble,
                        double a, double b, double c) {
  int64_t n = (int64_t)1 << scale;
  int64_t E = edgefactor * n;
  const double two32 = 4294967296.0;
  uint64_t ta = (uint64_t)(a * two32), tab = (uint64_t)((a + b) * two32), tabc = (uint64_t)((a + b + c) * two32);
  scrambler q = make_scrambler(scale, seed ^ 0xC0FFEEull);
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < E; ++k) {
    uint64_t u, v;
    rmat_edge(seed, (uint64_t)k, scale, ta, tab, tabc, &u, &v);
    if (u == v) continue;
    if (do_scramble) { u = scramble(&q, u); v = scramble(&q, v); }
    __atomic_fetch_add(&cnt[u], 1, __ATOMIC_RELAXED);
    __atomic_fetch_add(&cnt[v], 1, __ATOMIC_RELAXED);
  }
  int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  start[0] = 0;
  for (int64_t i = 0; i < n; ++i) start[i + 1] = start[i] + cnt[i];
  int64_t* fill = cnt; /* reuse as fill cursor */
  memcpy(fill, start, sizeof(int64_t) * (size_t)n);
  uint32_t* buf = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(start[n] > 0 ? start[n] : 1));
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < E; ++k) {
    uint64_t u, v;
    rmat_edge(seed, (uint64_t)k, scale, ta, tab, tabc, &u, &v);
    if (u == v) continue;
    if (do_scramble) { u = scramble(&q, u); v = scramble(&q, v); }
    int64_t pu = __atomic_fetch_add(&fill[u], 1, __ATOMIC_RELAXED);
    int64_t pv = __atomic_fetch_add(&fill[v], 1, __ATOMIC_RELAXED);
    buf[pu] = (uint32_t)v;
    buf[pv] = (uint32_t)u;
  }
  synth_graph* g = finish_rows(n, start, fill, buf);
  free(buf);
  free(start);
  free(cnt);
  return g;
}

/* rows x cols 4-neighbour grid; vertex id = y*cols + x. */
synth_graph* synth_grid(int64_t rows, int64_t cols) {
  int64_t n = rows * cols;
  synth_graph* g = (synth_graph*)calloc(1, sizeof(synth_graph));
  g->n = n;
  g->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  g->off[0] = 0;
  for (int64_t v = 0; v < n; ++v) {
    int64_t y = v / cols, x = v % cols;
    g->off[v + 1] = g->off[v] + (y > 0) + (x > 0) + (x + 1 < cols) + (y + 1 < rows);
  }
  g->nnz = g->off[n];
  g->idx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(g->nnz > 0 ? g->nnz : 1));
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) {
    int64_t y = v / cols, x = v % cols;
    int64_t p = g->off[v];
    if (y > 0) g->idx[p++] = (uint32_t)(v - cols);
    if (x > 0) g->idx[p++] = (uint32_t)(v - 1);
    if (x + 1 < cols) g->idx[p++] = (uint32_t)(v + 1);
    if (y + 1 < rows) g->idx[p++] = (uint32_t)(v + cols);
  }
  return g;
}

/* Random geometric graph (rgg_n_2_24_s0 shape, Table 3): 2^scale points
 * uniform in the unit square, an edge between every pair at Euclidean distance <= r with
 * r = factor * sqrt(ln n / n).  Point k's coordinates come from the splitmix64 stream keyed by
 * (seed, 2k) and (seed, 2k+1).  Vertex ids are assigned in cell-major order over a grid of
 * cells of side >= r (row-major cells, points of a cell by generation index), so every
 * neighbour lies in the 3x3 surrounding cells and scanning those cells in order emits each
 * row already sorted.  Symmetric by construction (the distance test is symmetric). */
synth_graph* synth_rgg(int scale, double factor, uint64_t seed) {
  const int64_t n = (int64_t)1 << scale;
  const double r = factor * sqrt(log((double)n) / (double)n), r2 = r * r;
  int64_t C = (int64_t)floor(1.0 / r);
  if (C < 1) C = 1;
  const int64_t ncell = C * C;
  double* x0 = (double*)malloc(sizeof(double) * (size_t)n);
  double* y0 = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* cell = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* cstart = (int64_t*)calloc((size_t)ncell + 1, sizeof(int64_t));
  const uint64_t key = seed * 0x100000001B3ull;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < n; ++k) {
    x0[k] = u01(sm64(key ^ (uint64_t)(2 * k)));
    y0[k] = u01(sm64(key ^ (uint64_t)(2 * k + 1)));
    int64_t cx = (int64_t)(x0[k] * (double)C), cy = (int64_t)(y0[k] * (double)C);
    if (cx >= C) cx = C - 1;
    if (cy >= C) cy = C - 1;
    cell[k] = cy * C + cx;
  }
  for (int64_t k = 0; k < n; ++k) cstart[cell[k] + 1]++;
  for (int64_t c = 0; c < ncell; ++c) cstart[c + 1] += cstart[c];
  double* px = (double*)malloc(sizeof(double) * (size_t)n);
  double* py = (double*)malloc(sizeof(double) * (size_t)n);
  {
    int64_t* fillc = (int64_t*)malloc(sizeof(int64_t) * (size_t)ncell);
    memcpy(fillc, cstart, sizeof(int64_t) * (size_t)ncell);
    for (int64_t k = 0; k < n; ++k) {  /* stable: generation order inside a cell */
      const int64_t id = fillc[cell[k]]++;
      px[id] = x0[k];
      py[id] = y0[k];
    }
    free(fillc);
  }
  free(x0);
  free(y0);
  free(cell);
  synth_graph* g = (synth_graph*)calloc(1, sizeof(synth_graph));
  g->n = n;
  g->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* deg = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  for (int pass = 0; pass < 2; ++pass) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t cy = 0; cy < C; ++cy)
      for (int64_t cx = 0; cx < C; ++cx)
        for (int64_t i = cstart[cy * C + cx]; i < cstart[cy * C + cx + 1]; ++i) {
          int64_t cntv = 0, p = pass ? g->off[i] : 0;
          for (int64_t ny = cy - 1; ny <= cy + 1; ++ny) {
            if (ny < 0 || ny >= C) continue;
            for (int64_t nx = cx - 1; nx <= cx + 1; ++nx) {
              if (nx < 0 || nx >= C) continue;
              const int64_t c = ny * C + nx;
              for (int64_t j = cstart[c]; j < cstart[c + 1]; ++j) {
                if (j == i) continue;
                const double dx = px[i] - px[j], dy = py[i] - py[j];
                if (dx * dx + dy * dy <= r2) {
                  if (pass) g->idx[p++] = (uint32_t)j;
                  else ++cntv;
                }
              }
            }
          }
          if (!pass) deg[i] = cntv;
        }
    if (!pass) {
      g->off[0] = 0;
      for (int64_t i = 0; i < n; ++i) g->off[i + 1] = g->off[i] + deg[i];
      g->nnz = g->off[n];
      g->idx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(g->nnz > 0 ? g->nnz : 1));
    }
  }
  free(deg);
  free(px);
  free(py);
  free(cstart);
  return g;
}

static int64_t uf_find(int64_t* par, int64_t x) {
  while (par[x] != x) { par[x] = par[par[x]]; x = par[x]; }
  return x;
}

/* Bond-percolated grid: each grid edge kept with probability p (seeded hash
 * of the edge id); only the largest connected component is kept, relabelled
 * in increasing original id order (road-like variant of config C4). */
synth_graph* synth_percolated_grid(int64_t rows, int64_t cols, double p, uint64_t seed) {
  int64_t n = rows * cols;
  /* edge e = 2*v (right neighbour), 2*v+1 (down neighbour) */
  int64_t* par = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t v = 0; v < n; ++v) par[v] = v;
  for (int64_t v = 0; v < n; ++v) {
    int64_t y = v / cols, x = v % cols;
    if (x + 1 < cols && u01(sm64(seed * 0x9E37ull ^ (uint64_t)(2 * v))) < p) {
      int64_t a = uf_find(par, v), b = uf_find(par, v + 1);
      if (a != b) par[a < b ? b : a] = a < b ? a : b;
    }
    if (y + 1 < rows && u01(sm64(seed * 0x9E37ull ^ (uint64_t)(2 * v + 1))) < p) {
      int64_t a = uf_find(par, v), b = uf_find(par, v + cols);
      if (a != b) par[a < b ? b : a] = a < b ? a : b;
    }
  }
  int64_t* size = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  for (int64_t v = 0; v < n; ++v) size[uf_find(par, v)]++;
  int64_t best = 0;
  for (int64_t v = 0; v < n; ++v) if (size[v] > size[best]) best = v;
  int64_t* id = size; /* reuse: new id or -1 */
  int64_t m = 0;
  for (int64_t v = 0; v < n; ++v) id[v] = (uf_find(par, v) == best) ? m++ : -1;
  synth_graph* g = (synth_graph*)calloc(1, sizeof(synth_graph));
  g->n = m;
  g->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  int64_t cap = 4 * m;
  g->idx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(cap > 0 ? cap : 1));
  int64_t p_ = 0, r = 0;
  g->off[0] = 0;
  for (int64_t v = 0; v < n; ++v) {
    if (id[v] < 0) continue;
    int64_t y = v / cols, x = v % cols;
    /* neighbours in increasing id order: up, left, right, down */
    if (y > 0 && u01(sm64(seed * 0x9E37ull ^ (uint64_t)(2 * (v - cols) + 1))) < p) g->idx[p_++] = (uint32_t)id[v - cols];
    if (x > 0 && u01(sm64(seed * 0x9E37ull ^ (uint64_t)(2 * (v - 1)))) < p) g->idx[p_++] = (uint32_t)id[v - 1];
    if (x + 1 < cols && u01(sm64(seed * 0x9E37ull ^ (uint64_t)(2 * v))) < p) g->idx[p_++] = (uint32_t)id[v + 1];
    if (y + 1 < rows && u01(sm64(seed * 0x9E37ull ^ (uint64_t)(2 * v + 1))) < p) g->idx[p_++] = (uint32_t)id[v + cols];
    g->off[++r] = p_;
  }
  g->nnz = p_;
  free(par);
  free(size);
  return g;
}

/* Generic preprocessing of an edge list: drop self-loops,
 * optionally symmetrise, dedup, sort rows.  Edges (src[k] -> dst[k]). */
synth_graph* synth_from_edges(int64_t n, int64_t m, const uint32_t* src, const uint32_t* dst,
                              int symmetrize, int keep_self_loops) {
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t k = 0; k < m; ++k) {
    if (src[k] == dst[k] && !keep_self_loops) continue;
    cnt[src[k]]++;
    if (symmetrize && src[k] != dst[k]) cnt[dst[k]]++;
  }
  int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  start[0] = 0;
  for (int64_t i = 0; i < n; ++i) start[i + 1] = start[i] + cnt[i];
  memcpy(cnt, start, sizeof(int64_t) * (size_t)n);
  uint32_t* buf = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(start[n] > 0 ? start[n] : 1));
  for (int64_t k = 0; k < m; ++k) {
    if (src[k] == dst[k] && !keep_self_loops) continue;
    buf[cnt[src[k]]++] = dst[k];
    if (symmetrize && src[k] != dst[k]) buf[cnt[dst[k]]++] = src[k];
  }
  synth_graph* g = finish_rows(n, start, cnt, buf);
  free(buf);
  free(start);
  free(cnt);
  return g;
}

/* Transpose a CSR (rows -> columns), producing sorted rows. */
synth_graph* synth_transpose(int64_t n, const int64_t* off, const uint32_t* idx) {
  int64_t nnz = off[n];
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t e = 0; e < nnz; ++e) cnt[idx[e]]++;
  synth_graph* g = (synth_graph*)calloc(1, sizeof(synth_graph));
  g->n = n;
  g->nnz = nnz;
  g->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  g->off[0] = 0;
  for (int64_t i = 0; i < n; ++i) g->off[i + 1] = g->off[i] + cnt[i];
  memcpy(cnt, g->off, sizeof(int64_t) * (size_t)n);
  g->idx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(nnz > 0 ? nnz : 1));
  for (int64_t i = 0; i < n; ++i) /* rows visited in increasing i => columns sorted */
    for (int64_t e = off[i]; e < off[i + 1]; ++e) g->idx[cnt[idx[e]]++] = (uint32_t)i;
  free(cnt);
  return g;
}

void synth_free(synth_graph* g) {
  if (!g) return;
  free(g->off);
  free(g->idx);
  free(g);
}

/* splitmix64 exposed so Python-side samplers use the same counter-based stream */
uint64_t synth_splitmix64(uint64_t x) { return sm64(x); }

int synth_num_threads(void) { return omp_get_max_threads(); }
