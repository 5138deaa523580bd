// bfs.cu — persistent, device-resident direction-optimised BFS (Algorithm 1).
//
// One cooperative launch runs the whole traversal: every level is one phase
// separated by a software grid barrier, and every CTA evaluates the push/pull
// decision redundantly from the same level counters, so no host round trip or
// relaunch happens between levels.
//
//   push level  (Alg. 3; Eq. 5):  f' = A^T f .* !v, column-based: the
//               frontier's CSR rows are expanded (light vertices warp-balanced by a
//               warp scan of degrees; heavy vertices as fixed-size edge chunks);
//               the mask test !v happens BEFORE the OR-merge, which is an atomicOr
//               on the visited bitmap (replaces the radix sort + segmented reduction
//               of P:360-362; exact because OR is idempotent).
//   pull level  (Alg. 2; Eq. 4): f' = A^T v .* !v (operand reuse P:284),
//               only rows with !v(i) are touched (masking P:270), each stops at its
//               first visited in-neighbour (early exit P:278).  Reads a snapshot of v
//               and writes v' = v | f' into the other bitmap (no intra-level races).
//   convert     (Dense2sparse) only on a pull->push switch: the new
//               frontier v' & !v becomes the light list / heavy chunks.
//   assign+reduce (Alg. 1 lines 7-8) are fused: depth is written at discovery and
//               c, m_f are warp-aggregated counters.
#include <cooperative_groups.h>

#include "pp_device.cuh"

namespace pp {

template <typename Off>
struct BfsArgs {
  int64_t n;
  int64_t nnz;
  uint32_t nwords;
  const Off* __restrict__ off;       // CSR (push rows, out-degree)
  const uint32_t* __restrict__ idx;
  const Off* __restrict__ coff;      // CSC (pull rows, in-degree)
  const uint32_t* __restrict__ cidx;
  int symmetric;
  const uint32_t* __restrict__ isolated;
  uint32_t* vis0;
  uint32_t* vis1;
  uint32_t* L0;
  uint32_t* L1;
  uint2* H0;
  uint2* H1;
  int32_t* depth;
  uint32_t* parent;
  LevelCtr* ctr;
  LevelStat* stats;
  int stats_cap;
  GridBarrier* bar;
  BfsStatus* status;
  uint32_t source;
  int mode;  // 0 DO, 1 push only, 2 pull only
  int rule;  // 0 edges, 1 paper r
  double alpha, beta;
  uint32_t toggles;
  int max_levels;
};

constexpr unsigned long long kWatchdogNs = 4000000000ull;  // 4 s per barrier wait

// Software grid barrier (all CTAs co-resident: cooperative launch).  The gpu-scope
// fences around the arrival/wait order every CTA's writes before the release and
// invalidate this SM's L1 after the acquire, so post-barrier loads see them.
__device__ __forceinline__ bool grid_barrier(GridBarrier* b, BfsStatus* st) {
  __shared__ int s_ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    int ok = 1;
    const unsigned nblocks = gridDim.x;
    unsigned g = ld_acquire_gpu(&b->gen);
    __threadfence();
    unsigned arrived = atomicAdd(&b->count, 1u);
    if (arrived == nblocks - 1) {
      atomicExch(&b->count, 0u);
      __threadfence();
      st_release_gpu(&b->gen, g + 1);
    } else {
      unsigned long long t0 = global_timer_ns();
      while (ld_acquire_gpu(&b->gen) == g) {
        __nanosleep(32);
        if (global_timer_ns() - t0 > kWatchdogNs) {
          ok = 0;
          atomicExch(&st->error, (int)PP_ERR_TIMEOUT);
          break;
        }
      }
    }
    __threadfence();
    if (ld_relaxed_s32(&st->error) != 0) ok = 0;
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// Per-lane accumulators of a level's counters, flushed once per phase.
struct Acc {
  unsigned long long c, mf, mfin;
};

__device__ __forceinline__ void flush_acc(Acc& acc, LevelCtr* out) {
  unsigned long long c = warp_sum(acc.c), mf = warp_sum(acc.mf), mfin = warp_sum(acc.mfin);
  if (lane_id() == 0 && c) {
    atomicAdd(&out->c, c);
    atomicAdd(&out->m_f, mf);
    atomicAdd(&out->m_fin, mfin);
  }
  acc.c = acc.mf = acc.mfin = 0;
}

// Append newly discovered vertex v (valid lanes) to the next frontier: light list if
// 0 < deg < kHeavy, else ceil(deg/kChunk) heavy chunks.  Warp-collective.
template <typename Off>
__device__ __forceinline__ void append_frontier(bool valid, uint32_t v, Off deg, uint32_t* Lout,
                                                uint2* Hout, LevelCtr* out) {
  const unsigned lane = lane_id();
  bool heavy = valid && deg >= (Off)kHeavy;
  bool light = valid && deg > 0 && !heavy;
  unsigned lm = __ballot_sync(kFull, light);
  if (lm) {
    unsigned leader = __ffs(lm) - 1, base = 0;
    if (lane == leader) base = atomicAdd(&out->nL, (unsigned)__popc(lm));
    base = __shfl_sync(kFull, base, leader);
    if (light) Lout[base + __popc(lm & lanemask_lt())] = v;
  }
  unsigned hm = __ballot_sync(kFull, heavy);
  if (hm) {
    unsigned nch = heavy ? (unsigned)((deg + (Off)kChunk - 1) / (Off)kChunk) : 0u;
    unsigned incl = warp_incl_scan(nch);
    unsigned tot = __shfl_sync(kFull, incl, 31), base = 0;
    if (lane == 0) base = atomicAdd(&out->nH, tot);
    base = __shfl_sync(kFull, base, 0);
    for (unsigned k = 0; k < nch; ++k) Hout[base + incl - nch + k] = make_uint2(v, k);
  }
}

// Push visit of edge (u, w): the mask test (w unvisited) precedes the OR-merge
// (atomicOr).  Parents: atomicMin over every edge whose head was unvisited when the
// level started: bit clear in a post-barrier read, or depth still 0
// or newdepth (i.e. discovered during this level).
template <bool PARENTS>
__device__ __forceinline__ bool push_visit(uint32_t* vis, int32_t* depth, uint32_t* parent,
                                           uint32_t u, uint32_t w, int newdepth) {
  const uint32_t wi = w >> 5, bit = 1u << (w & 31u);
  const uint32_t cur = vis[wi];
  bool disc = false;
  if (!(cur & bit)) {
    uint32_t old = atomicOr(&vis[wi], bit);
    disc = !(old & bit);
  }
  if (disc) depth[w] = newdepth;
  if (PARENTS) {
    bool fresh = disc || !(cur & bit);
    if (!fresh) {
      int dw = ld_relaxed_s32(&depth[w]);
      fresh = (dw == 0 || dw == newdepth);
    }
    if (fresh) atomicMin(&parent[w], u);
  }
  return disc;
}

template <typename Off, bool PARENTS>
__device__ __forceinline__ void push_edge_batch(const BfsArgs<Off>& a, bool valid, uint32_t u,
                                                uint32_t w, uint32_t* vis, int newdepth,
                                                uint32_t* Lout, uint2* Hout, LevelCtr* out,
                                                Acc& acc) {
  bool disc = valid && push_visit<PARENTS>(vis, a.depth, a.parent, u, w, newdepth);
  if (__ballot_sync(kFull, disc) == 0) return;
  Off deg = 0, degin = 0;
  if (disc) {
    Off b = a.off[w], e = a.off[w + 1];
    deg = e - b;
    degin = a.symmetric ? deg : (Off)(a.coff[w + 1] - a.coff[w]);
    acc.c += 1;
    acc.mf += (unsigned long long)deg;
    acc.mfin += (unsigned long long)degin;
  }
  append_frontier<Off>(disc, w, deg, Lout, Hout, out);
}

// Column-based masked mxv over the frontier (light list + heavy chunks).
template <typename Off, bool PARENTS>
__device__ void push_phase(const BfsArgs<Off>& a, const uint32_t* Lin, unsigned nL,
                           const uint2* Hin, unsigned nH, uint32_t* Lout, uint2* Hout,
                           LevelCtr* out, uint32_t* vis, int newdepth, Acc& acc) {
  const unsigned lane = lane_id();
  const unsigned nRounds = (nL + 31u) / 32u;
  const unsigned total = nH + nRounds;
  for (;;) {
    const unsigned item = warp_grab(&out->work);
    if (item >= total) break;
    if (item < nH) {
      // heavy chunk: kChunk consecutive edges of one vertex, fully coalesced
      const uint2 h = Hin[item];
      const uint32_t u = h.x;
      const Off rb = a.off[u], re = a.off[u + 1];
      const Off b = rb + (Off)h.y * (Off)kChunk;
      const Off e = min(re, b + (Off)kChunk);
      for (Off base = b; base < e; base += 32) {
        const Off p = base + lane;
        const bool valid = p < e;
        const uint32_t w = valid ? a.idx[p] : 0u;
        push_edge_batch<Off, PARENTS>(a, valid, u, w, vis, newdepth, Lout, Hout, out, acc);
      }
    } else {
      // light round: 32 frontier vertices, edges balanced across lanes by a warp scan
      const unsigned i = (item - nH) * 32u + lane;
      uint32_t u = 0;
      Off b = 0;
      unsigned deg = 0;
      if (i < nL) {
        u = Lin[i];
        b = a.off[u];
        deg = (unsigned)(a.off[u + 1] - b);
      }
      const unsigned incl = warp_incl_scan(deg);
      const unsigned excl = incl - deg;
      const unsigned tot = __shfl_sync(kFull, incl, 31);
      for (unsigned base = 0; base < tot; base += 32) {
        const unsigned e = base + lane;
        const unsigned j = warp_owner(incl, e);
        const uint32_t uj = __shfl_sync(kFull, u, j);
        const Off bj = __shfl_sync(kFull, b, j);
        const unsigned xj = __shfl_sync(kFull, excl, j);
        const bool valid = e < tot;
        const uint32_t w = valid ? a.idx[bj + (Off)(e - xj)] : 0u;
        push_edge_batch<Off, PARENTS>(a, valid, uj, w, vis, newdepth, Lout, Hout, out, acc);
      }
    }
  }
}

constexpr int kLaneProbe = 8;  // indices per lane-probe round (one 32 B sector)
constexpr int kLaneRounds = 2;

// Row-based masked mxv with early exit over the complement of the visited snapshot.
// Warp item = 32 bitmap words (1024 rows); candidates are enumerated warp-balanced.
template <typename Off, bool PARENTS>
__device__ void pull_phase(const BfsArgs<Off>& a, const uint32_t* __restrict__ vin,
                           uint32_t* __restrict__ vout, LevelCtr* out, int d, Acc& acc,
                           uint32_t* sfound) {
  const unsigned lane = lane_id();
  const unsigned nchunks = a.nwords / 32u;
  const bool early_exit = !(a.toggles & PP_OPT_NO_EARLYEXIT);
  const bool no_mask = (a.toggles & PP_OPT_NO_MASKING) != 0;
  const bool no_reuse = (a.toggles & PP_OPT_NO_REUSE) != 0;
  for (;;) {
    const unsigned item = warp_grab(&out->work);
    if (item >= nchunks) break;
    const unsigned wbase = item * 32u;
    const uint32_t vw = vin[wbase + lane];
    const uint32_t unvisited = ~vw;
    // Masking (Opt. 2): only rows with !v(i) are computed.  Without it every
    // non-isolated row is computed and the result filtered afterwards.
    const uint32_t cand = no_mask ? ~a.isolated[wbase + lane] : unvisited;
    sfound[lane] = 0u;
    __syncwarp();
    const unsigned cnt = __popc(cand);
    const unsigned incl = warp_incl_scan(cnt);
    const unsigned excl = incl - cnt;
    const unsigned tot = __shfl_sync(kFull, incl, 31);
    for (unsigned base = 0; base < tot; base += 32) {
      const unsigned k = base + lane;
      const bool valid = k < tot;
      const unsigned j = warp_owner(incl, k);
      const uint32_t mj = __shfl_sync(kFull, cand, j);
      const unsigned xj = __shfl_sync(kFull, excl, j);
      const uint32_t uj = __shfl_sync(kFull, unvisited, j);
      const unsigned bitpos = valid ? __fns(mj, 0, (int)(k - xj) + 1) : 0u;
      const uint32_t i = (wbase + j) * 32u + bitpos;
      Off p = 0, e = 0, rb = 0;
      bool found = false;
      uint32_t par = 0;
      if (valid) {
        rb = p = a.coff[i];
        e = a.coff[i + 1];
        // Lane probes: up to kLaneRounds sector-aligned groups of indices, loaded
        // together, tested together; the first hit in sorted order is the parent.
        for (int r = 0; r < kLaneRounds && p < e && !(found && early_exit); ++r) {
          const Off lim = min(e, (p | (Off)(kLaneProbe - 1)) + 1);
          uint32_t x[kLaneProbe];
#pragma unroll
          for (int t = 0; t < kLaneProbe; ++t) x[t] = (p + t < lim) ? a.cidx[p + t] : 0u;
#pragma unroll
          for (int t = 0; t < kLaneProbe; ++t) {
            if (p + t < lim) {
              const bool hit = no_reuse ? (a.depth[x[t]] == d) : bit_test(vin, x[t]);
              if (hit && !found) {
                found = true;
                par = x[t];
              }
            }
          }
          p = lim;
        }
      }
      // Warp-cooperative continuation for rows still unresolved: 128 indices per
      // step (4 coalesced loads per lane), ballot early exit.
      const bool deferred = valid && p < e && (!found || !early_exit);
      unsigned dm = __ballot_sync(kFull, deferred);
      while (dm) {
        const unsigned l = __ffs(dm) - 1;
        dm &= dm - 1;
        const Off pb = __shfl_sync(kFull, p, l), pe = __shfl_sync(kFull, e, l);
        bool f = __shfl_sync(kFull, found ? 1 : 0, l) != 0;
        uint32_t fx = __shfl_sync(kFull, par, l);
        for (Off q0 = pb; q0 < pe; q0 += 128) {
          uint32_t x[4];
          bool h[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const Off q = q0 + (Off)(t * 32) + lane;
            x[t] = q < pe ? a.cidx[q] : 0u;
          }
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const Off q = q0 + (Off)(t * 32) + lane;
            h[t] = q < pe && (no_reuse ? (a.depth[x[t]] == d) : bit_test(vin, x[t]));
          }
          bool stop = false;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const unsigned bm = __ballot_sync(kFull, h[t]);
            if (bm && !f) {
              f = true;
              fx = __shfl_sync(kFull, x[t], __ffs(bm) - 1);
            }
            stop = stop || (f && early_exit);
          }
          if (stop) break;
        }
        if (lane == l) {
          found = f;
          par = fx;
        }
      }
      if (found && ((uj >> bitpos) & 1u)) {
        atomicOr(&sfound[j], 1u << bitpos);
        a.depth[i] = d + 1;
        if (PARENTS) a.parent[i] = par;
        const Off degin = e - rb;
        const Off deg = a.symmetric ? degin : (Off)(a.off[i + 1] - a.off[i]);
        acc.c += 1;
        acc.mf += (unsigned long long)deg;
        acc.mfin += (unsigned long long)degin;
      }
    }
    __syncwarp();
    vout[wbase + lane] = vw | sfound[lane];
    __syncwarp();
  }
}

// Dense2sparse of the new frontier v' & !v after a pull level (pull->push switch).
template <typename Off>
__device__ void convert_phase(const BfsArgs<Off>& a, const uint32_t* vnew, const uint32_t* vold,
                              uint32_t* Lout, uint2* Hout, LevelCtr* out) {
  const unsigned lane = lane_id();
  const unsigned nchunks = a.nwords / 32u;
  for (;;) {
    const unsigned item = warp_grab(&out->work2);
    if (item >= nchunks) break;
    const unsigned w = item * 32u + lane;
    uint32_t diff = vnew[w] & ~vold[w];
    while (__ballot_sync(kFull, diff != 0u)) {
      const bool valid = diff != 0u;
      uint32_t v = 0;
      Off deg = 0;
      if (valid) {
        const unsigned b = __ffs(diff) - 1;
        diff &= diff - 1;
        v = w * 32u + b;
        deg = a.off[v + 1] - a.off[v];
      }
      append_frontier<Off>(valid, v, deg, Lout, Hout, out);
    }
  }
}

__device__ __forceinline__ int decide(int rule, int dir, long long c_old, long long c_new,
                                      long long m_f, long long m_u, long long n, double alpha,
                                      double beta) {
  // DESIGN.md R10/R11; identical arithmetic to oracle_direction (IEEE double).
  if (rule == 0) {
    if (dir == 0) return (c_new > c_old && (double)m_f * alpha > (double)m_u) ? 1 : 0;
    return (c_new < c_old && (double)c_new * beta < (double)n) ? 0 : 1;
  }
  const double cn = (double)c_new, nn = (double)n;
  if (dir == 0) return (c_new > c_old && cn > __dmul_rn(alpha, nn)) ? 1 : 0;
  return (c_new < c_old && cn < __dmul_rn(beta, nn)) ? 0 : 1;
}

template <typename Off, bool PARENTS>
__global__ void __launch_bounds__(kBlock, 4) bfs_persistent(BfsArgs<Off> a) {
  __shared__ uint32_t sfound[kWarps][32];
  const unsigned warp = threadIdx.x >> 5;
  const unsigned long long gtid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long gsize = (unsigned long long)gridDim.x * blockDim.x;
  const uint32_t s = a.source;

  // ---- Alg. 1 lines 2-4: d <- 1, f <- e_s, v <- 0 (depth 0 = unvisited) ----
  for (unsigned long long v = gtid; v < (unsigned long long)a.n; v += gsize) {
    a.depth[v] = (v == s) ? 1 : 0;
    if (PARENTS) a.parent[v] = (v == s) ? s : 0xFFFFFFFFu;
  }
  // visited starts as {s} plus the isolated / padding vertices, which no pull may
  // compute and no push can reach (they have no edges).
  for (unsigned long long w = gtid; w < a.nwords; w += gsize)
    a.vis0[w] = a.isolated[w] | ((w == (s >> 5)) ? (1u << (s & 31u)) : 0u);
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t < kRing * (int)(sizeof(LevelCtr) / 4); t += blockDim.x)
      reinterpret_cast<unsigned*>(a.ctr)[t] = 0u;
    __syncthreads();
    const Off deg = a.off[s + 1] - a.off[s];
    if (deg >= (Off)kHeavy) {
      const unsigned nch = (unsigned)((deg + (Off)kChunk - 1) / (Off)kChunk);
      for (unsigned k = threadIdx.x; k < nch; k += blockDim.x) a.H0[k] = make_uint2(s, k);
      if (threadIdx.x == 0) a.ctr[0].nH = nch;
    } else if (deg > 0 && threadIdx.x == 0) {
      a.L0[0] = s;
      a.ctr[0].nL = 1;
    }
  }
  if (!grid_barrier(a.bar, a.status)) return;

  int dir = (a.mode == 2) ? 1 : 0;
  int cur = 0;  // visited bitmap in use
  int sel = 0;  // frontier list / chunk buffers holding the current frontier
  long long c_old = 1;
  const Off indeg_s = a.coff[s + 1] - a.coff[s];
  long long m_u = a.nnz - (long long)indeg_s;
  long long reached = 1;
  Acc acc{0, 0, 0};
  int d = 1;
  for (;; ++d) {
    LevelCtr* in = &a.ctr[(d - 1) & (kRing - 1)];
    LevelCtr* out = &a.ctr[d & (kRing - 1)];
    if (blockIdx.x == 0 && threadIdx.x < sizeof(LevelCtr) / 4)
      reinterpret_cast<unsigned*>(&a.ctr[(d + 1) & (kRing - 1)])[threadIdx.x] = 0u;
    uint32_t* vis = cur ? a.vis1 : a.vis0;
    uint32_t* vis_other = cur ? a.vis0 : a.vis1;
    if (dir == 0) {
      const unsigned nL = ld_relaxed_u32(&in->nL), nH = ld_relaxed_u32(&in->nH);
      push_phase<Off, PARENTS>(a, sel ? a.L1 : a.L0, nL, sel ? a.H1 : a.H0, nH,
                               sel ? a.L0 : a.L1, sel ? a.H0 : a.H1, out, vis, d + 1, acc);
    } else {
      pull_phase<Off, PARENTS>(a, vis, vis_other, out, d, acc, sfound[warp]);
    }
    flush_acc(acc, out);
    if (!grid_barrier(a.bar, a.status)) return;
    const long long c_new = (long long)ld_relaxed_u64(&out->c);
    const long long mf = (long long)ld_relaxed_u64(&out->m_f);
    const long long mfin = (long long)ld_relaxed_u64(&out->m_fin);
    if (dir == 1) cur ^= 1;
    else sel ^= 1;
    m_u -= a.symmetric ? mf : mfin;
    reached += c_new;
    if (blockIdx.x == 0 && threadIdx.x == 0 && d - 1 < a.stats_cap) {
      LevelStat st;
      st.dir = dir;
      st.pad = 0;
      st.c = c_new;
      st.m_f = mf;
      st.m_u = m_u;
      a.stats[d - 1] = st;
    }
    if (c_new == 0 || d >= a.max_levels) break;
    int next = dir;
    if (a.mode == 0) next = decide(a.rule, dir, c_old, c_new, mf, m_u, a.n, a.alpha, a.beta);
    if (dir == 1 && next == 0) {
      // pull -> push: Dense2sparse of the frontier just discovered
      uint32_t* vnew = cur ? a.vis1 : a.vis0;
      uint32_t* vold = cur ? a.vis0 : a.vis1;
      convert_phase<Off>(a, vnew, vold, sel ? a.L1 : a.L0, sel ? a.H1 : a.H0, out);
      if (!grid_barrier(a.bar, a.status)) return;
    }
    dir = next;
    c_old = c_new;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.status->levels = d;
    a.status->reached = reached;
  }
}

template <typename Off, bool PARENTS>
static int grid_for() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bfs_persistent<Off, PARENTS>, kBlock, 0);
    cached = sms * (per > 0 ? per : 1);
  }
  return cached;
}

int bfs_grid_size(pp_graph g, bool parents) {
  if (g->off64) return parents ? grid_for<uint64_t, true>() : grid_for<uint64_t, false>();
  return parents ? grid_for<uint32_t, true>() : grid_for<uint32_t, false>();
}

template <typename Off, bool PARENTS>
static cudaError_t launch_t(pp_graph g, const BfsArgs<Off>& args) {
  const int grid = grid_for<Off, PARENTS>();
  void* params[] = {(void*)&args};
  g->ctx->launches += 1;
  return cudaLaunchCooperativeKernel((const void*)bfs_persistent<Off, PARENTS>, dim3(grid),
                                     dim3(kBlock), params, 0, g->ctx->stream);
}

template <typename Off>
static cudaError_t launch_off(pp_graph g, uint32_t source, int mode, int rule, double alpha,
                              double beta, uint32_t toggles, int32_t* depth, uint32_t* parent,
                              int max_levels) {
  BfsArgs<Off> a;
  a.n = g->n;
  a.nnz = g->nnz;
  a.nwords = g->nwords;
  a.off = (const Off*)g->off;
  a.idx = g->idx;
  a.coff = (const Off*)g->coff;
  a.cidx = g->cidx;
  a.symmetric = g->symmetric ? 1 : 0;
  a.isolated = g->isolated;
  a.vis0 = g->vis[0];
  a.vis1 = g->vis[1];
  a.L0 = g->L[0];
  a.L1 = g->L[1];
  a.H0 = g->H[0];
  a.H1 = g->H[1];
  a.depth = depth;
  a.parent = parent;
  a.ctr = g->ctr;
  a.stats = g->stats;
  a.stats_cap = g->stats_cap;
  a.bar = g->bar;
  a.status = g->status;
  a.source = source;
  a.mode = mode;
  a.rule = rule;
  a.alpha = alpha;
  a.beta = beta;
  a.toggles = toggles;
  a.max_levels = max_levels;
  if (parent) return launch_t<Off, true>(g, a);
  return launch_t<Off, false>(g, a);
}

cudaError_t launch_bfs(pp_graph g, uint32_t source, int mode, int rule, double alpha, double beta,
                       uint32_t toggles, int32_t* depth, uint32_t* parent, int max_levels) {
  if (g->off64)
    return launch_off<uint64_t>(g, source, mode, rule, alpha, beta, toggles, depth, parent,
                                max_levels);
  return launch_off<uint32_t>(g, source, mode, rule, alpha, beta, toggles, depth, parent,
                              max_levels);
}

}  // namespace pp
