/*
 * oracle/oracle.c — plain, slow, single-thread CPU oracle for the hot path of
 * Yang, Buluç, Owens, "Implementing Push-Pull Efficiently in GraphBLAS"
 * (ICPP'18, arXiv 1804.03327).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_1804_03327_b200/), and neither side includes the other.
 *
 * Citations: P:n = /root/reference/PAPER.md line n.
 *
 * Functions (each is the plain definition, no blocking/fusion/reordering):
 *   O1 oracle_bfs        textbook FIFO-queue BFS; Alg. 1 depth convention
 *                        (source depth 1, unreached 0).
 *   O2 oracle_parents    canonical min-id parent at depth-1 (R14);
 *      oracle_parents_ordered  the same under a vertex order (first in the order).
 *   O3 oracle_mxv        definitional Boolean masked matvec, Eq. 2/4 (P:91-96,
 *                        123-125) with structural complement, accumulate
 *                        and replace (R5, R6).  No early exit, no
 *                        direction: every row, every stored entry.
 *   O4 oracle_direction  one push/pull decision (R10, R11).
 *      oracle_trace      the per-level direction sequence and counters that the
 *                        decision rule implies for a given depth vector.
 * Pins: tests/test_oracle_pins.py (brute force, closed forms, scipy, the paper's
 * and SPEC's worked examples).  Nothing here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------------------
 * O1: BFS depths.  A is n x n in CSR (row u lists the out-neighbours w of u,
 * i.e. (u,w) in E; P:51 read as "w is a child of u iff (u,w) in E", R21).
 * depth[s] = 1 (Alg. 1 line 2: d <- 1 and v <- f*d + v with f = e_s);
 * depth[w] = depth[u] + 1 on first visit; unreached = 0.
 * Returns the number of BFS levels executed by Alg. 1's while-loop, i.e. the
 * maximum depth reached (the last level discovers nothing), or -1 on bad input.
 * ------------------------------------------------------------------------------------- */
int64_t oracle_bfs(int64_t n, const int64_t* off, const uint32_t* idx, int64_t s, int32_t* depth) {
  if (s < 0 || s >= n) return -1;
  int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) depth[i] = 0;
  int64_t head = 0, tail = 0, maxd = 1;
  depth[s] = 1;
  queue[tail++] = s;
  while (head < tail) {
    int64_t u = queue[head++];
    for (int64_t e = off[u]; e < off[u + 1]; ++e) {
      uint32_t w = idx[e];
      if (depth[w] == 0) {
        depth[w] = depth[u] + 1;
        if (depth[w] > maxd) maxd = depth[w];
        queue[tail++] = w;
      }
    }
  }
  free(queue);
  return maxd;
}

/* ---------------------------------------------------------------------------------------
 * O2: canonical parents.  coff/cidx = CSC of A (row v lists in-neighbours u,
 * (u,v) in E).  parent[v] = min{ u in N-(v) : depth[u] = depth[v]-1 };
 * parent[s] = s; unreached -> -1.  The paper computes no parents (Alg. 1 returns
 * depths only); this is the reading DESIGN.md R14 fixes.
 * ------------------------------------------------------------------------------------- */
int oracle_parents(int64_t n, const int64_t* coff, const uint32_t* cidx, const int32_t* depth,
                   int64_t s, int32_t* parent) {
  for (int64_t v = 0; v < n; ++v) {
    parent[v] = -1;
    if (depth[v] == 0) continue;
    if (v == s) { parent[v] = (int32_t)s; continue; }
    int64_t best = -1;
    for (int64_t e = coff[v]; e < coff[v + 1]; ++e) {
      uint32_t u = cidx[e];
      if (depth[u] == depth[v] - 1 && (best < 0 || (int64_t)u < best)) best = u;
    }
    if (best < 0) return -1; /* depth vector is not a BFS result */
    parent[v] = (int32_t)best;
  }
  return 0;
}

/* O2 under a vertex order (PP_GRAPH_RELABEL, R14): the same set of valid
 * parents { u in N-(v) : depth[u] = depth[v]-1 }, the canonical one being the u with the
 * smallest key[u] (key = a permutation of 0..n-1: the position of u in the order).
 * key[u] = u gives oracle_parents. */
int oracle_parents_ordered(int64_t n, const int64_t* coff, const uint32_t* cidx,
                           const int32_t* depth, int64_t s, const uint32_t* key, int32_t* parent) {
  for (int64_t v = 0; v < n; ++v) {
    parent[v] = -1;
    if (depth[v] == 0) continue;
    if (v == s) { parent[v] = (int32_t)s; continue; }
    int64_t best = -1;
    for (int64_t e = coff[v]; e < coff[v + 1]; ++e) {
      uint32_t u = cidx[e];
      if (depth[u] == depth[v] - 1 && (best < 0 || key[u] < key[best])) best = u;
    }
    if (best < 0) return -1;
    parent[v] = (int32_t)best;
  }
  return 0;
}

/* ---------------------------------------------------------------------------------------
 * O3: masked matvec over the Boolean semiring ({0,1}, AND, OR, 0)
 * (Alg. 1 caption P:204: "x = AND, + = OR"; R3).
 *
 * The operator M (n_rows x n_cols) is given in CSR: row i lists the j with
 * M(i,j) != 0.  For BFS traversal w = A^T u, the caller passes M = A^T, i.e.
 * the CSC of A ("f' = A^T f .* !v").
 *
 *   t(i)    = OR_{j : M(i,j) != 0} ( M(i,j) AND u(j) )         Eq. 2
 *   pass(i) = mask == NULL ? 1 : ((mask(i) != 0) XOR scmp)     P:152, Alg. 2 line 3
 *   z(i)    = accum ? (w_in(i) OR t(i)) : t(i)                 Alg. 2 line 10 (R6)
 *   w(i)    = pass(i) ? z(i) : (replace ? 0 : w_in(i))         Eq. 4, P:125 (R5)
 *
 * u, mask, w_in, w_out are dense 0/1 byte vectors.  w_in may be NULL when
 * accum == 0 and replace == 1 (it is then never read).  Returns 0, or -1 on
 * invalid arguments (complement without a mask, R9; w_in missing).
 * ------------------------------------------------------------------------------------- */
int oracle_mxv(int64_t n_rows, const int64_t* off, const uint32_t* idx, const uint8_t* u,
               const uint8_t* mask, int scmp, int accum, int replace, const uint8_t* w_in,
               uint8_t* w_out) {
  if (mask == NULL && scmp) return -1;
  if (w_in == NULL && (accum || !replace)) return -1;
  for (int64_t i = 0; i < n_rows; ++i) {
    uint8_t t = 0;
    for (int64_t e = off[i]; e < off[i + 1]; ++e) t = (uint8_t)(t | (u[idx[e]] != 0));
    int pass = (mask == NULL) ? 1 : ((mask[i] != 0) ^ (scmp != 0));
    uint8_t z = accum ? (uint8_t)((w_in[i] != 0) | t) : t;
    w_out[i] = pass ? z : (replace ? 0 : (uint8_t)(w_in[i] != 0));
  }
  return 0;
}

/* ---------------------------------------------------------------------------------------
 * O4: direction decision, made after level k from integer counters.
 *   dir: 0 = push, 1 = pull.  rule: 0 = edge-count rule (Beamer, P:366 first
 *   sentence; R11), 1 = the paper's r-rule (R10).
 *   c_old = |frontier expanded at level k|, c_new = |frontier it discovered|,
 *   m_f = sum of out-degrees over the new frontier (Eq. 1),
 *   m_u = sum of in-degrees over vertices still unvisited, n = #rows (M).
 *
 *   edge rule : push->pull iff c_new > c_old and m_f * alpha > m_u     (alpha default 15)
 *               pull->push iff c_new < c_old and c_new * beta < n      (beta default 18)
 *   paper rule: r = c_new / n; push->pull iff r increasing and r > alpha;
 *               pull->push iff r decreasing and r < beta                (alpha=beta=0.01)
 *   otherwise keep the current direction (ties hold).
 * All comparisons in IEEE double on exactly-representable integer operands.
 * ------------------------------------------------------------------------------------- */
int oracle_direction(int rule, int dir, int64_t c_old, int64_t c_new, int64_t m_f, int64_t m_u,
                     int64_t n, double alpha, double beta) {
  if (rule == 0) {
    if (dir == 0) return (c_new > c_old && (double)m_f * alpha > (double)m_u) ? 1 : 0;
    return (c_new < c_old && (double)c_new * beta < (double)n) ? 0 : 1;
  } else {
    double cn = (double)c_new, nn = (double)n;
    if (dir == 0) return (c_new > c_old && cn > alpha * nn) ? 1 : 0;
    return (c_new < c_old && cn < beta * nn) ? 0 : 1;
  }
}

/* ---------------------------------------------------------------------------------------
 * O4: the per-level trace implied by a depth vector.
 *   mode: 0 = direction-optimised, 1 = push only, 2 = pull only.
 *   Level k (k = 1..L) expands F_k = {v : depth v = k}; after it,
 *   c[k-1] = |F_{k+1}|, m_f[k-1] = sum outdeg(F_{k+1}),
 *   m_u[k-1] = sum indeg over {v : depth v = 0 or depth v > k+1},
 *   dir[k-1] = direction used by level k.  Level 1 is push in DO mode
 *   (SPEC S:366).  Returns L (number of levels), or -1 if cap < L.
 * outdeg from off (CSR of A), indeg from coff (CSC of A).
 * ------------------------------------------------------------------------------------- */
int64_t oracle_trace(int64_t n, const int64_t* off, const int64_t* coff, const int32_t* depth,
                     int mode, int rule, double alpha, double beta, int64_t cap, int8_t* dir,
                     int64_t* c, int64_t* m_f, int64_t* m_u) {
  int64_t L = 0;
  for (int64_t v = 0; v < n; ++v) if (depth[v] > L) L = depth[v];
  if (L > cap) return -1;
  int64_t* cnt = (int64_t*)calloc((size_t)L + 2, sizeof(int64_t));
  int64_t* out_sum = (int64_t*)calloc((size_t)L + 2, sizeof(int64_t));
  int64_t* in_sum = (int64_t*)calloc((size_t)L + 2, sizeof(int64_t));
  int64_t in_total = 0;
  for (int64_t v = 0; v < n; ++v) {
    int64_t od = off[v + 1] - off[v], id = coff[v + 1] - coff[v];
    in_total += id;
    cnt[depth[v]] += 1;
    out_sum[depth[v]] += od;
    in_sum[depth[v]] += id;
  }
  int cur = (mode == 2) ? 1 : 0;
  int64_t visited_in = in_sum[1];
  for (int64_t k = 1; k <= L; ++k) {
    dir[k - 1] = (int8_t)cur;
    int64_t cn = (k + 1 <= L) ? cnt[k + 1] : 0;
    int64_t mf = (k + 1 <= L) ? out_sum[k + 1] : 0;
    visited_in += (k + 1 <= L) ? in_sum[k + 1] : 0;
    c[k - 1] = cn;
    m_f[k - 1] = mf;
    m_u[k - 1] = in_total - visited_in;
    if (mode == 0 && cn > 0) cur = oracle_direction(rule, cur, cnt[k], cn, mf, in_total - visited_in, n, alpha, beta);
  }
  free(cnt);
  free(out_sum);
  free(in_sum);
  return L;
}
