#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
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
  uint32_t* fr;  // frontier bitmap written by pull levels (push-from-bitmap)
  const uint32_t* __restrict__ drec;  // PP_DENSE: 32-byte rows {6 in-neighbours, caller, in-degree}
  long long n_noniso;                 // rows not pre-marked visited (isolated / padding)
  uint32_t* sumv;      // visited summary: bit per 2^sum_shift vertices, isolated excluded
  int sum_shift;
  uint32_t sum_words;
  uint4* L0;  // light frontier entries {v, deg, begin_lo, begin_hi}
  uint4* L1;
  uint2* H0;
  uint2* H1;
  unsigned hcap;  // entries of H0 / H1 (chunk descriptors grow up, hub blocks down)
  int32_t* depth;       // caller ids (PP_GRAPH_RELABEL: index through perm)
  uint32_t* parent;     // internal ids (the caller's array, or pint on a relabelled graph)
  uint32_t* pout;       // relabelled graph with parents: the caller's parent array
  const uint32_t* __restrict__ perm;  // internal -> caller id, nullptr = identity
  const uint32_t* __restrict__ rank;  // caller -> internal id
  const uint4* __restrict__ vrec;     // relabelled: {begin lo, hi, out-degree, caller id}
  LevelCtr* ctr;
  LevelStat* stats;
  int stats_cap;
  GridBarrier* bar;
  BfsStatus* status;
  int narrow;  // 1: this launch is one thread-block cluster running the small levels
  int resume;  // 1: continue the loop state a narrow launch handed over (bar->rs)
  int stop_before;  // > 0: hand the loop state over (bar->rs) before level stop_before
                    // (pp_bfs_debug_level: one level alone in its own launch, for ncu)
  uint32_t source;  // caller id
  int mode;  // 0 DO, 1 push only, 2 pull only
  int rule;  // 0 edges, 1 paper r
  double alpha, beta;
  uint32_t toggles;
  int max_levels;
  long long* dbg;  // optional: per level, per CTA work duration (ns) of the level's phase
  int dbg_levels;
  // CTAs of this rank in the launch: [cta_base, cta_base + ncta) (a single-device team runs
  // its ranks as CTA groups of one cooperative launch; otherwise 0 and gridDim.x)
  int cta_base, ncta;
  unsigned* gwork;  // [kRing][kMaxCtas] per-CTA pull item counters (PP_STEAL)
  // ---- multi-rank (1D row partition; D-template instantiations only) ----
  // rank owns vertices [lo, hi) = bitmap words [wlo, wlo + wcnt); off/idx = push structure
  // (global rows, owned targets), coff/cidx/head = CSC rows of the block (local row v - lo),
  // depth/parent = the block's slices.  Each level's discoveries are OR-ed into xfr[d & 1]
  // and the owned words are stored into every peer's copy (pfr), the per-rank counters into
  // every peer's record slot (pcnt), then one release flag per peer (pflag).
  int64_t lo, hi;
  uint32_t wlo, wcnt;
  int me, nranks;  // this rank's index, ranks in the group
  uint32_t* xfr0;
  uint32_t* xfr1;
  unsigned long long* xcnt;   // own [2][kMaxRanks][8]
  uint32_t* xlst0;            // own id-list receive areas (parity 0 / 1; sender q at q*wcnt)
  uint32_t* xlst1;
  uint32_t* xown;             // this rank's push discoveries of the level (first wcnt ids)
  uint32_t* plst[kMaxRanks][2];
  unsigned long long* xflag;  // own [kMaxRanks]
  uint32_t* pfr[kMaxRanks][2];
  unsigned long long* pcnt[kMaxRanks];
  unsigned long long* pflag[kMaxRanks];
  unsigned long long xseq;  // flag epoch base of this BFS (monotone across calls)
  const uint32_t* __restrict__ odeg;  // directed: global out-degree of the owned rows
  long long in_total;                 // sum of in-degrees over all ranks
};

constexpr unsigned long long kWatchdogNs = 4000000000ull;  // 4 s per barrier wait

// Software grid barrier (all CTAs co-resident: cooperative launch).  One 64-bit counter
// grows monotonically through the BFS: barrier number `epoch` is complete when it reaches
// epoch * gridDim.  Arrival is a single atom.add.acq_rel.gpu (releases this CTA's prior
// writes, published to thread 0 by __syncthreads; the last arriver acquires everyone's),
// waiting is ld.acquire.gpu polling (which invalidates this SM's L1), and the closing
// __syncthreads hands the acquire to the CTA's other threads — no trailing fence (the
// release-arrival + fence.sc form is PP_BAR_ACQREL=0).  Bit 63 is the abort flag (watchdog),
// which releases every waiter.
constexpr unsigned long long kAbortBit = 1ull << 63;
#ifndef PP_BAR_SLEEP
#define PP_BAR_SLEEP 16  // ns of back-off between barrier polls
#endif
#ifndef PP_BAR_ACQREL
#define PP_BAR_ACQREL 1  // measured: C4 7.09 -> 6.63 us per level, C2 +3%
#endif


__device__ __forceinline__ bool grid_barrier(GridBarrier* b, BfsStatus* st, unsigned& epoch,
                                             unsigned ncta) {
  __shared__ int s_ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned long long target = (unsigned long long)epoch * ncta;
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(&b->count);
#if PP_BAR_ACQREL
    // arrival with acquire-release semantics (the last arriver acquires too) and acquire
    // polling: no trailing fence
    unsigned long long v;
    asm volatile("atom.add.acq_rel.gpu.u64 %0, [%1], 1;" : "=l"(v) : "l"(cnt) : "memory");
    v += 1ull;
#else
    unsigned long long v = atom_add_release_u64(cnt, 1ull) + 1ull;
#endif
    if (v < target) {
      unsigned long long t0 = global_timer_ns();
      while ((v = ld_acquire_u64(cnt)) < target) {
        if (PP_BAR_SLEEP) __nanosleep(PP_BAR_SLEEP);
        if (global_timer_ns() - t0 > kWatchdogNs) {
          atomicExch(&st->error, (int)PP_ERR_TIMEOUT);
          atomicOr(cnt, kAbortBit);
          v = kAbortBit;
          break;
        }
      }
    }
    if (!PP_BAR_ACQREL) __threadfence();
    s_ok = (v & kAbortBit) ? 0 : 1;
  }
  __syncthreads();
  return s_ok != 0;
}

// Narrow mode: the whole launch is ONE thread-block cluster, so the level barrier is the
// hardware cluster barrier (release/acquire at cluster scope, which also orders the
// global-memory writes of the level) instead of the software grid barrier.
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ bool level_barrier(bool narrow, GridBarrier* b, BfsStatus* st,
                                              unsigned& epoch, unsigned ncta) {
  if (narrow) {
    __syncthreads();
    cluster_barrier();
    return true;
  }
  return grid_barrier(b, st, epoch, ncta);
}

// Per-lane accumulators of a level's counters, flushed once per phase.
struct Acc {
  unsigned long long c, mf, mfin, big, cand;  // cand: rows a pull computed (pp_bfs_stats.cand)
};

// CTA-level reduction, then one set of atomics per CTA (single-address L2 atomics
// serialise; per-warp flushing cost ~3 x #warps atomics per level).
__device__ __forceinline__ void flush_acc(Acc& acc, LevelCtr* out,
                                          unsigned long long (*red)[5]) {
  const unsigned warp = threadIdx.x >> 5;
  unsigned long long c = 0, mf = 0, mfin = 0, big = 0, cd = 0;
  // a warp with nothing to report (most warps of a small level) skips its 25 shuffles
  if (__any_sync(kFull, (acc.c | acc.mf | acc.mfin | acc.big | acc.cand) != 0ull)) {
    c = warp_sum(acc.c);
    mf = warp_sum(acc.mf);
    mfin = warp_sum(acc.mfin);
    big = warp_sum(acc.big);
    cd = warp_sum(acc.cand);
  }
  if (lane_id() == 0) {
    red[warp][0] = c;
    red[warp][1] = mf;
    red[warp][2] = mfin;
    red[warp][3] = big;
    red[warp][4] = cd;
  }
  __syncthreads();
  if (warp == 0) {  // warp 0 reduces the CTA's per-warp partials, lane 0 publishes
    const unsigned l = lane_id();
    const bool in = l < (unsigned)kBfsWarps;
    const unsigned long long x0 = in ? red[l][0] : 0ull, x1 = in ? red[l][1] : 0ull,
                             x2 = in ? red[l][2] : 0ull, x3 = in ? red[l][3] : 0ull,
                             x4 = in ? red[l][4] : 0ull;
    unsigned long long tc = 0, tm = 0, ti = 0, tb = 0, td = 0;
    if (__any_sync(kFull, (x0 | x1 | x2 | x3 | x4) != 0ull)) {
      tc = warp_sum(x0);
      tm = warp_sum(x1);
      ti = warp_sum(x2);
      tb = warp_sum(x3);
      td = warp_sum(x4);
    }
    if (l == 0) {
      if (tc) {
        atomicAdd(&out->c, tc);
        atomicAdd(&out->m_f, tm);
        atomicAdd(&out->m_fin, ti);
      }
      if (tb) atomicAdd(&out->nbig, tb);
      if (td) atomicAdd(&out->cand, td);
    }
  }
  acc.c = acc.mf = acc.mfin = acc.big = acc.cand = 0;
}

// Work assignment: CTA b owns items b, b+G, b+2G, ... (interleaved, so every CTA sees the
// same mix of heavy and light items) and its warps grab them dynamically through a
// shared-memory counter (reset to 0 before each phase by read_level), which balances the
// irregular per-item cost inside the CTA without any global atomics.
template <typename Off>
__device__ __forceinline__ unsigned cta_of(const BfsArgs<Off>& a) { return blockIdx.x - a.cta_base; }
template <typename Off>
__device__ __forceinline__ unsigned cta_grab(const BfsArgs<Off>& a, unsigned* sctr) {
  unsigned j = 0;
  if (lane_id() == 0) j = atomicAdd(sctr, 1u);
  j = __shfl_sync(kFull, j, 0);
  return cta_of(a) + j * (unsigned)a.ncta;
}
// A phase's FIRST grab is static: warp w takes the CTA's item w, and the shared counter starts
// at kBfsWarps (set by read_level), so the 32 warps do not serialise on one shared-memory
// atomic at the start of every level (~1 us on a small level).
__device__ __forceinline__ unsigned first_j() { return threadIdx.x >> 5; }
template <typename Off>
__device__ __forceinline__ unsigned cta_first(const BfsArgs<Off>& a) {
  return cta_of(a) + first_j() * (unsigned)a.ncta;
}
template <typename Off>
__device__ __forceinline__ unsigned nwarps(const BfsArgs<Off>& a) { return (unsigned)a.ncta * kBfsWarps; }



// Light frontier entry: the discovering thread already loaded the row's offsets, so the
// next push reads {v, deg, begin} in one 16-byte load instead of a list load followed by
// a dependent offsets load.
template <typename Off>
__device__ __forceinline__ uint4 light_entry(uint32_t v, Off deg, Off begin) {
  return make_uint4(v, (uint32_t)deg, (uint32_t)begin, (uint32_t)((unsigned long long)begin >> 32));
}
template <typename Off>
__device__ __forceinline__ Off light_begin(const uint4& e) {
  return (Off)(((unsigned long long)e.w << 32) | e.z);
}

// Heavy frontier vertices (out-degree >= kHeavy) are expanded as kChunk-edge chunks.  A
// vertex with <= kSelfChunks chunks gets one descriptor {v, k} per chunk (bottom of H); a
// hub gets one descriptor {v, k0} per 32 chunks (top of H, growing down: H[hcap-1-j]), and
// the next push maps its hub items (32 per block) back to chunks.  Descriptor writes are
// O(degree / 4096) for a hub, so no warp stalls emitting them whichever hubs it discovers
// (with PP_GRAPH_RELABEL the first chunk of a row holds the highest-degree neighbours).
// cs / cb: this lane's chunk / block descriptor counts; warp-collective.
__device__ __forceinline__ void heavy_counts(unsigned nch, unsigned& cs, unsigned& cb) {
  const bool hub = nch > kSelfChunks;
  cs = hub ? 0u : nch;
  cb = hub ? (nch + 31u) / 32u : 0u;
}
__device__ __forceinline__ void heavy_bases(unsigned CS, unsigned CB, LevelCtr* out, unsigned& s0,
                                            unsigned& b0) {
  const unsigned is = warp_incl_scan(CS), ib = warp_incl_scan(CB);
  const unsigned ts = __shfl_sync(kFull, is, 31), tb = __shfl_sync(kFull, ib, 31);
  unsigned bs = 0, bb = 0;
  if (lane_id() == 0) {
    if (ts) bs = atomicAdd(&out->nH, ts);
    if (tb) bb = atomicAdd(&out->nB, tb);
  }
  s0 = __shfl_sync(kFull, bs, 0) + is - CS;
  b0 = __shfl_sync(kFull, bb, 0) + ib - CB;
}
__device__ __forceinline__ void heavy_write(uint32_t v, unsigned cs, unsigned cb, uint2* H,
                                            unsigned hcap, unsigned& s0, unsigned& b0) {
  for (unsigned k = 0; k < cs; ++k) H[s0 + k] = make_uint2(v, k);
  for (unsigned j = 0; j < cb; ++j) H[hcap - 1u - (b0 + j)] = make_uint2(v, 32u * j);
  s0 += cs;
  b0 += cb;
}

// Append newly discovered vertex v (valid lanes) to the next frontier: light list if
// 0 < deg < kHeavy, else heavy chunks.  Warp-collective.
template <typename Off>
__device__ __forceinline__ void append_frontier(bool valid, uint32_t v, Off deg, Off begin, uint4* Lout,
                                                uint2* Hout, unsigned hcap, LevelCtr* out) {
  const unsigned lane = lane_id();
  bool heavy = valid && deg >= (Off)kHeavy;
  bool light = valid && deg > 0 && !heavy;
  unsigned lm = __ballot_sync(kFull, light);
  if (lm) {
    unsigned leader = __ffs(lm) - 1, base = 0;
    if (lane == leader) base = atomicAdd(&out->nL, (unsigned)__popc(lm));
    base = __shfl_sync(kFull, base, leader);
    if (light) Lout[base + __popc(lm & lanemask_lt())] = light_entry<Off>(v, deg, begin);
  }
  if (__any_sync(kFull, heavy)) {
    unsigned cs, cb, s0, b0;
    heavy_counts(heavy ? (unsigned)((deg + (Off)kChunk - 1) / (Off)kChunk) : 0u, cs, cb);
    heavy_bases(cs, cb, out, s0, b0);
    heavy_write(v, cs, cb, Hout, hcap, s0, b0);
  }
}

#ifndef PP_PUSH_KU
#define PP_PUSH_KU 2  // measured: +7% on C2, -14% per C4 level vs 4 (half the spills)
#endif
constexpr int kU = PP_PUSH_KU;  // edges (push) in flight per lane
#ifndef PP_LOWLAT_VREC
#define PP_LOWLAT_VREC 1  // round 2b: C4 7.41 -> 7.35 us per level, C2 equal; with
#endif                    // kU = 2 and the smaller kernel it costs 60 B of spills, not 670
#ifndef PP_PF_ROWS
#define PP_PF_ROWS 0  // measured neutral
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// The same for kU candidates per lane, with one atomic per list per warp.
template <typename Off>
__device__ __forceinline__ void append_frontier4(const bool (&disc)[kU], const uint32_t (&w)[kU],
                                                 const Off (&deg)[kU], const Off (&beg)[kU],
                                                 uint4* Lout, uint2* Hout, unsigned hcap,
                                                 LevelCtr* out) {
  const unsigned lane = lane_id();
  unsigned lm[kU], ltot = 0, hsum = 0;
#pragma unroll
  for (int t = 0; t < kU; ++t) {
    const bool light = disc[t] && deg[t] > 0 && deg[t] < (Off)kHeavy;
    lm[t] = __ballot_sync(kFull, light);
    ltot += __popc(lm[t]);
    if (disc[t] && deg[t] >= (Off)kHeavy) hsum += (unsigned)((deg[t] + (Off)kChunk - 1) / (Off)kChunk);
  }
  if (ltot) {
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(&out->nL, ltot);
    base = __shfl_sync(kFull, base, 0);
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      if ((lm[t] >> lane) & 1u)
        Lout[base + __popc(lm[t] & lanemask_lt())] = light_entry<Off>(w[t], deg[t], beg[t]);
      base += __popc(lm[t]);
    }
  }
  if (__any_sync(kFull, hsum != 0)) {
    unsigned cs[kU], cb[kU], CS = 0, CB = 0;
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      heavy_counts((disc[t] && deg[t] >= (Off)kHeavy)
                       ? (unsigned)((deg[t] + (Off)kChunk - 1) / (Off)kChunk) : 0u, cs[t], cb[t]);
      CS += cs[t];
      CB += cb[t];
    }
    unsigned s0, b0;
    heavy_bases(CS, CB, out, s0, b0);
#pragma unroll
    for (int t = 0; t < kU; ++t) heavy_write(w[t], cs[t], cb[t], Hout, hcap, s0, b0);
  }
}

// Push visit of kU edges (u, w) per lane, all loads issued before use.  The mask test
// (w unvisited) precedes the OR-merge (atomicOr on the visited bitmap).  Parents:
// atomicMin over every edge whose head was unvisited when the level started
// (SURVEY.md G14): bit clear in a post-barrier read, or depth 0 / newdepth.
//
// Multi-rank (D): every target w is owned (the push structure holds only owned targets);
// a discovery writes the block's depth slot w - lo and ORs w into the level's frontier
// bitmap `frout` (exchanged after the level) instead of appending to the local lists, and
// counts the GLOBAL out-degree of w for m_f (the decision needs global sums).
template <typename Off, bool PARENTS, bool D>
__device__ __forceinline__ void push_visit4(const BfsArgs<Off>& a, const bool (&valid)[kU],
                                            const uint32_t (&u)[kU], const uint32_t (&w)[kU],
                                            uint32_t* vis, int newdepth, uint4* Lout,
                                            uint2* Hout, LevelCtr* out, Acc& acc, bool lowlat,
                                            uint32_t* frout, bool& xfull) {
  uint32_t cur[kU];
  bool disc[kU];
  Off sb[kU], se[kU];
  uint32_t sp[kU];  // lowlat + relabelled: the caller id, from the same speculative record
  if (lowlat) {
    // small level: latency matters more than traffic — atomicOr without the pre-test, and
    // the head's offsets (relabelled graph: its whole 16-byte vertex record, offsets AND
    // caller id) loaded speculatively in parallel: one round trip instead of three
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      cur[t] = 0xFFFFFFFFu;
      sb[t] = se[t] = 0;
      sp[t] = w[t];
      if (valid[t]) {
        cur[t] = atomicOr(&vis[w[t] >> 5], 1u << (w[t] & 31u));
        if (PP_LOWLAT_VREC && !D && a.vrec) {
          const uint4 r = __ldg(a.vrec + w[t]);
          sb[t] = (Off)(((unsigned long long)r.y << 32) | r.x);
          se[t] = sb[t] + (Off)r.z;
          sp[t] = r.w;
        } else {
          sb[t] = a.off[w[t]];
          se[t] = a.off[w[t] + 1];
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kU; ++t) disc[t] = valid[t] && !((cur[t] >> (w[t] & 31u)) & 1u);
  } else {
#pragma unroll
    for (int t = 0; t < kU; ++t) cur[t] = valid[t] ? vis[w[t] >> 5] : 0xFFFFFFFFu;
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      const uint32_t bit = 1u << (w[t] & 31u);
      disc[t] = false;
      if (!(cur[t] & bit)) {
        const uint32_t old = atomicOr(&vis[w[t] >> 5], bit);
        disc[t] = !(old & bit);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < kU; ++t) {
    if (disc[t] && kSumWordsMax && !D) {
      const uint32_t gi = w[t] >> a.sum_shift;
      atomicOr(&a.sumv[gi >> 5], 1u << (gi & 31u));
    }
  }
  if (PARENTS) {
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      if (!valid[t]) continue;
      bool fresh = disc[t] || !((cur[t] >> (w[t] & 31u)) & 1u);
      const uint32_t slot = D ? w[t] - (uint32_t)a.lo : w[t];
      if (!fresh) {
        const int dw = ld_relaxed_s32(&a.depth[D ? slot : (a.perm ? a.perm[w[t]] : w[t])]);
        fresh = (dw == 0 || dw == newdepth);
      }
      if (fresh) atomicMin(&a.parent[slot], u[t]);
    }
  }
  bool any = false;
#pragma unroll
  for (int t = 0; t < kU; ++t) any = any || disc[t];
  if (!__any_sync(kFull, any)) return;
  if (D) {
    // the id list the exchange sends instead of the bitmap slice when it is shorter: slots are
    // reserved with ONE atomic per warp step (a per-discovery atomic on one counter serialised
    // in one L2 slice: C5's big push level took 4.7 ms instead of 0.4)
    unsigned dm[kU], ndisc = 0;
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      dm[t] = __ballot_sync(kFull, disc[t]);
      ndisc += __popc(dm[t]);
    }
    // once this warp has seen the list overflow the slice, it stops counting (nX only has to
    // be exact below wcnt: the exchange sends the list only then)
    unsigned xbase = a.wcnt;
    if (!xfull) {
      if (lane_id() == 0) xbase = atomicAdd(&out->nX, ndisc);
      xbase = __shfl_sync(kFull, xbase, 0);
      xfull = xbase + ndisc >= a.wcnt;
    }
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      const unsigned slot = xbase + __popc(dm[t] & lanemask_lt());
      xbase += __popc(dm[t]);
      if (!disc[t]) continue;
      const uint32_t r = w[t] - (uint32_t)a.lo;  // local row of the owned target
      const Off degin = a.coff[r + 1] - a.coff[r];
      const Off dg = a.symmetric ? degin : (Off)a.odeg[r];
      a.depth[r] = newdepth;
      atomicOr(&frout[w[t] >> 5], 1u << (w[t] & 31u));
      if (slot < a.wcnt) a.xown[slot] = w[t];
      acc.c += 1;
      acc.mf += (unsigned long long)dg;
      acc.mfin += (unsigned long long)degin;
      acc.big += dg >= (Off)kBig ? 1u : 0u;
    }
    return;
  }
  Off deg[kU], beg[kU];
  uint32_t dpos[kU];  // where the discovery's depth goes (caller id)
#pragma unroll
  for (int t = 0; t < kU; ++t) {
    deg[t] = 0;
    beg[t] = 0;
    dpos[t] = w[t];
    if (disc[t]) {
      if (a.vrec && !lowlat) {  // one 16-byte record: offsets + caller id
        const uint4 r = __ldg(a.vrec + w[t]);
        beg[t] = (Off)(((unsigned long long)r.y << 32) | r.x);
        deg[t] = (Off)r.z;
        dpos[t] = r.w;
      } else if (PP_LOWLAT_VREC && a.vrec) {  // lowlat: the speculative record
        beg[t] = sb[t];
        deg[t] = se[t] - sb[t];
        dpos[t] = sp[t];
      } else {
        if (a.perm) dpos[t] = a.perm[w[t]];  // loaded in the same batch as the offsets
        beg[t] = lowlat ? sb[t] : a.off[w[t]];
        deg[t] = (lowlat ? se[t] : a.off[w[t] + 1]) - beg[t];
      }
      const Off degin = a.symmetric ? deg[t] : (Off)(a.coff[w[t] + 1] - a.coff[w[t]]);
      acc.c += 1;
      acc.mf += (unsigned long long)deg[t];
      acc.mfin += (unsigned long long)degin;
      // the next push (if any) reads this row: pull its first ids into L2 now, off the
      // critical path of the next level's dependent chain (entry -> ids -> visited word)
      if (PP_PF_ROWS && deg[t] > 0) prefetch_l2(a.idx + beg[t]);
    }
  }
#pragma unroll
  for (int t = 0; t < kU; ++t)
    if (disc[t]) a.depth[dpos[t]] = newdepth;
  append_frontier4<Off>(disc, w, deg, beg, Lout, Hout, a.hcap, out);
}

// Edges of up to 32 light frontier vertices (lane l holds v, row begin b, degree deg),
// balanced over lanes by a warp scan of the degrees, kU edges in flight per lane.
template <typename Off, bool PARENTS, bool D>
__device__ __forceinline__ void push_round(const BfsArgs<Off>& a, uint32_t v, Off b, unsigned deg,
                                           uint4* Lout, uint2* Hout, LevelCtr* out,
                                           uint32_t* vis, int newdepth, Acc& acc, bool lowlat,
                                           uint32_t* frout, bool& xfull) {
  const unsigned lane = lane_id();
  const unsigned incl = warp_incl_scan(deg);
  const unsigned excl = incl - deg;
  const unsigned tot = __shfl_sync(kFull, incl, 31);
  bool valid[kU];
  uint32_t u[kU], w[kU];
  for (unsigned base = 0; base < tot; base += 32 * kU) {
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      const unsigned e = base + t * 32 + lane;
      const unsigned j = warp_owner(incl, e);
      u[t] = __shfl_sync(kFull, v, j);
      const Off bj = __shfl_sync(kFull, b, j);
      const unsigned xj = __shfl_sync(kFull, excl, j);
      valid[t] = e < tot;
      w[t] = valid[t] ? a.idx[bj + (Off)(e - xj)] : 0u;
    }
    push_visit4<Off, PARENTS, D>(a, valid, u, w, vis, newdepth, Lout, Hout, out, acc, lowlat,
                                 frout, xfull);
  }
}

#ifndef PP_PULL_WORDS
#define PP_PULL_WORDS 8
#endif
constexpr unsigned kPW = PP_PULL_WORDS;  // bitmap words per warp item (32*kPW rows)

// Column-based masked mxv over the frontier (Alg. 3 re-designed).  The frontier is
// either (list mode) a light list + heavy chunks, or (bitmap mode, right after a pull
// level whose discoveries all have out-degree < kBig) the pull's frontier bitmap `fr`,
// which skips the Dense2sparse conversion and its grid barrier.  Heavy chunk = kChunk =
// 128 consecutive edges = one warp iteration with 4 coalesced loads per lane.  Light
// round = R frontier vertices (R = 32, or fewer when the frontier is too small to occupy
// every warp), their edges balanced over lanes by a warp scan of degrees.
template <typename Off, bool PARENTS, bool D>
__device__ void push_phase(const BfsArgs<Off>& a, const uint4* Lin, unsigned nL,
                           const uint2* Hin, unsigned nH, unsigned nB, const uint32_t* fr,
                           uint4* Lout,
                           uint2* Hout, LevelCtr* out, uint32_t* vis, int newdepth, Acc& acc,
                           unsigned* sctr, bool lowlat, uint32_t* frout) {
  const unsigned lane = lane_id();
  const unsigned NW = nwarps(a);
  bool xfull = false;  // multi-rank: this warp saw the level's id list overflow its slice
  unsigned R = 32;
  while (R > 1 && (nL + R / 2 - 1) / (R / 2) <= NW) R >>= 1;
  const unsigned nRounds = fr ? a.nwords / kPW : (nL + R - 1) / R;
  const unsigned nHC = nH + 32u * nB;  // chunk items: descriptors, then 32 per hub block
  const unsigned total = nHC + nRounds;
  for (unsigned item = cta_first(a); item < total; item = cta_grab(a, sctr)) {
    if (item < nHC) {
      bool valid[kU];
      uint32_t u[kU], w[kU];
      uint2 h;
      if (item < nH) {
        h = Hin[item];
      } else {
        const unsigned q = item - nH;
        h = Hin[a.hcap - 1u - (q >> 5)];
        h.y += q & 31u;
      }
      const Off rb = a.off[h.x], re = a.off[h.x + 1];
      const Off b = rb + (Off)h.y * (Off)kChunk;  // past the row end for a hub's last slots
      const Off e = min(re, b + (Off)kChunk);
      static_assert(kChunk % (32 * kU) == 0, "chunk = whole warp iterations");
      for (Off sb = b; sb < e; sb += (Off)(32 * kU)) {
#pragma unroll
        for (int t = 0; t < kU; ++t) {
          const Off p = sb + (Off)(t * 32) + lane;
          valid[t] = p < e;
          u[t] = h.x;
          w[t] = valid[t] ? a.idx[p] : 0u;
        }
        push_visit4<Off, PARENTS, D>(a, valid, u, w, vis, newdepth, Lout, Hout, out, acc, lowlat,
                                     frout, xfull);
      }
    } else if (!fr) {
      const unsigned i = (item - nHC) * R + lane;
      uint32_t v = 0;
      Off b = 0;
      unsigned deg = 0;
      if (lane < R && i < nL) {
        const uint4 le = Lin[i];
        v = le.x;
        deg = le.y;
        b = light_begin<Off>(le);
      }
      push_round<Off, PARENTS, D>(a, v, b, deg, Lout, Hout, out, vis, newdepth, acc, lowlat, frout,
                                  xfull);
    } else {
      const unsigned wbase = (item - nHC) * kPW;
      const uint32_t fw = lane < kPW ? fr[wbase + lane] : 0u;
      const unsigned cnt = __popc(fw);
      const unsigned incl = warp_incl_scan(cnt);
      const unsigned excl = incl - cnt;
      const unsigned tot = __shfl_sync(kFull, incl, 31);
      for (unsigned base = 0; base < tot; base += 32) {
        const unsigned k = base + lane;
        const unsigned j = warp_owner(incl, k);
        const uint32_t mj = __shfl_sync(kFull, fw, j);
        const unsigned xj = __shfl_sync(kFull, excl, j);
        uint32_t v = 0;
        Off b = 0;
        unsigned deg = 0;
        if (k < tot) {
          v = (wbase + j) * 32u + nth_set_bit(mj, k - xj);
          b = a.off[v];
          deg = (unsigned)(a.off[v + 1] - b);
        }
        push_round<Off, PARENTS, D>(a, v, b, deg, Lout, Hout, out, vis, newdepth, acc, lowlat,
                                    frout, xfull);
      }
    }
  }
}

#ifndef PP_DENSE_DIST
#define PP_DENSE_DIST 0  // dense pull on multi-rank blocks: measured slower (their rows are not
#endif                   // degree-ordered: the first record id rarely decides)
#ifndef PP_PULL_KC
#define PP_PULL_KC 1
#endif
#ifndef PP_SUM_RESID
#define PP_SUM_RESID 0  // with PP_SUM_WORDS > 0: the summary serves the residual tiers only
#endif
#ifndef PP_STEAL
#define PP_STEAL 0    // > 0: per-CTA item counters in global memory; a warp whose CTA ran out
                      // of items claims items of up to PP_STEAL other CTAs (tail balance)
#endif
constexpr int kC = PP_PULL_KC;  // candidates in flight per lane
constexpr int kLaneMax = 16;    // residual rows with <= this many ids left: one lane each
constexpr int kGroupMax = 512;   // <= this many: 8-lane groups; longer: the whole warp
#ifndef PP_RQ_EXTRA
#define PP_RQ_EXTRA 32
#endif
// residual-queue entries per warp: a round parks at most 32*kC rows on top of <= 31 left over
// (shared memory is carved out of L1, whose hits serve the visited-bitmap probes: keep it small)
constexpr int kQ = 32 * kC + PP_RQ_EXTRA;
static_assert(PP_RQ_EXTRA >= 31, "residual queue: 31 + 32*kC entries must fit");
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kRelP = 0x80000000u;  // ResidualQ::rem flag: p is relative to coff[i]

// Rows whose first sector did not decide them, parked per warp in shared memory and
// processed 32 at a time so no lane idles behind one long row.
template <typename Off>
struct ResidualQ {
  uint32_t i[kQ];
  uint32_t par[kQ];  // kNone = not found yet (else: committed, scan continues w/o early exit)
  Off p[kQ];
  uint32_t rem[kQ];
  uint32_t degin[kQ];
};

__device__ __forceinline__ uint4 ld_nc_u4(const uint32_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

// One 32-byte sector of column ids in a single 256-bit load (LDG.E.ENL2.256 on sm_100a).
struct V8 {
  uint32_t x[8];
};
__device__ __forceinline__ V8 ld_nc_v8(const uint32_t* p) {
  V8 v;
#ifdef PP_IDX_NOALLOC
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#else
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#endif
               : "=r"(v.x[0]), "=r"(v.x[1]), "=r"(v.x[2]), "=r"(v.x[3]), "=r"(v.x[4]),
                 "=r"(v.x[5]), "=r"(v.x[6]), "=r"(v.x[7])
               : "l"(p));
  return v;
}

template <typename Off, bool PARENTS, bool D>
struct PullCtx {
  const BfsArgs<Off>& a;
  const uint32_t* __restrict__ vin;
  uint32_t* __restrict__ vout;
  int d;
  bool early_exit, no_reuse;
  Acc& acc;
  uint32_t* sfound;
  ResidualQ<Off>& q;
  const uint32_t* ssum;  // shared-memory copy of the visited summary (snapshot)
  uint2* hubs;           // no early exit: long-row chunk descriptors (2 uint2 each) ...
  unsigned* hub_count;   // ... and their count
  uint32_t* fr;          // the level's frontier bitmap (multi-rank: the exchanged xfr[d & 1])

  // Visited test of a probed neighbour.  The summary in shared memory rejects most
  // unvisited neighbours without a global access (false positives only: a set summary
  // bit is confirmed against the exact snapshot bitmap).
  __device__ __forceinline__ bool hit(uint32_t x) const {
    if (!D && no_reuse) return a.depth[a.perm ? a.perm[x] : x] == d;
#ifdef PP_KO_PROBE  // timing-only knockout: every probed neighbour counts as visited
    return x != 0xFFFFFFFFu;
#endif
    if (kSumWordsMax && !PP_SUM_RESID && !D) {
      const uint32_t gi = x >> a.sum_shift;
      if (!((ssum[gi >> 5] >> (gi & 31u)) & 1u)) return false;
    }
    return bit_test(vin, x);
  }
  // The residual tiers' probe (rows the 8-id head did not decide, mostly rows with no visited
  // in-neighbour at all, whose every probe is negative): with PP_SUM_RESID the shared-memory
  // summary answers "not visited" for a whole 2^sum_shift-vertex group without a global load.
  __device__ __forceinline__ bool hit_res(uint32_t x) const {
    if (!D && no_reuse) return a.depth[a.perm ? a.perm[x] : x] == d;
    if (kSumWordsMax && !D) {
      const uint32_t gi = x >> a.sum_shift;
      if (!((ssum[gi >> 5] >> (gi & 31u)) & 1u)) return false;
    }
    return bit_test(vin, x);
  }
  // Ids [q0, q0+8) (q0 8-aligned: one 32-byte sector, a single 256-bit load) clipped to
  // [rb, e).  The first valid id is probed alone and the others only if it misses:
  // every probe is a scattered visited-bitmap load, and most rows hit at their first
  // id.  First hit in sorted order = parent.
  __device__ __forceinline__ void test8(const V8& v, Off q0, Off rb, Off e, bool& found,
                                        uint32_t& par) const {
    const Off f0 = rb > q0 ? rb - q0 : (Off)0;  // first valid slot (0..7)
    if (q0 + f0 >= e || (found && early_exit)) return;
    uint32_t xf = v.x[0];
#pragma unroll
    for (int t = 1; t < 8; ++t)
      if ((Off)t == f0) xf = v.x[t];
    if (hit_res(xf)) {
      if (!found) {
        found = true;
        par = xf;
      }
      if (early_exit) return;
    }
    bool h[8];
#pragma unroll
    for (int t = 1; t < 8; ++t) h[t] = (Off)t > f0 && q0 + (Off)t < e && hit_res(v.x[t]);
#pragma unroll
    for (int t = 1; t < 8; ++t) {
      if (h[t] && !found) {
        found = true;
        par = v.x[t];
      }
    }
  }
  __device__ __forceinline__ void probe8(Off q0, Off rb, Off e, bool& found, uint32_t& par) const {
    const V8 v = ld_nc_v8(a.cidx + q0);
    test8(v, q0, rb, e, found, par);
  }
  // discovery of row i (found this level): Alg. 1 lines 7-8 fused
  __device__ __forceinline__ void commit(uint32_t i, uint32_t par, Off degin, unsigned wbase,
                                         bool in_item, uint32_t dpos) const {
    const uint32_t bit = 1u << (i & 31u);
    if (in_item) {
      atomicOr(&sfound[(i >> 5) - wbase], bit);
    } else {
      atomicOr(&vout[i >> 5], bit);
      atomicOr(&fr[i >> 5], bit);
    }
#ifndef PP_KO_DEPTH  // timing-only knockout: results invalid when defined
    a.depth[dpos] = d + 1;  // caller id of i (multi-rank: the block's slot i - lo)
#endif
    if (PARENTS) a.parent[D ? i - (uint32_t)a.lo : i] = par;
    if (kSumWordsMax && !D && !in_item) {  // in-item finds reach the summary at item close
      const uint32_t gi = i >> a.sum_shift;
      atomicOr(&a.sumv[gi >> 5], 1u << (gi & 31u));
    }
    const Off deg = a.symmetric ? degin
                    : (D ? (Off)a.odeg[i - (uint32_t)a.lo] : (Off)(a.off[i + 1] - a.off[i]));
    acc.c += 1;
    acc.mf += (unsigned long long)deg;
    acc.mfin += (unsigned long long)degin;
    acc.big += deg >= (Off)kBig ? 1u : 0u;
  }
  // process the top `cnt` (<= 32) residual rows, one per lane
  __device__ void residual_batch(int& qn, int cnt, unsigned wbase, unsigned pw) const {
    const unsigned lane = lane_id();
    const int slot = qn - cnt + (int)lane;
    const bool valid = (int)lane < cnt;
    uint32_t i = 0, par = kNone, degin = 0;
    Off p = 0, e = 0;
    if (valid) {
      i = q.i[slot];
      par = q.par[slot];
      p = q.p[slot];
      uint32_t rem = q.rem[slot];
      if (rem & kRelP) {  // dense pull: p is relative to the row's begin
        rem &= ~kRelP;
        p += a.coff[D ? i - (uint32_t)a.lo : i];
      }
      e = p + (Off)rem;
      degin = q.degin[slot];
    }
    __syncwarp();
    qn -= cnt;
    const bool committed = par != kNone;
    bool found = committed;
    // tier 0: short remainders, one lane per row, 8 ids per step
    while (true) {
      const bool act = valid && p < e && !(found && early_exit) && (e - p) <= (Off)kLaneMax;
      if (!__any_sync(kFull, act)) break;
      if (act) {
        const Off q0 = p & ~(Off)7;
        probe8(q0, p, e, found, par);
        p = q0 + 8;
      }
    }
    // tier 1: medium remainders, 8-lane groups (64 ids per step), 4 rows at once
    unsigned m1 = __ballot_sync(kFull, valid && p < e && !(found && early_exit) &&
                                           (e - p) <= (Off)kGroupMax);
    const unsigned g = lane >> 3, sub = lane & 7u;
    while (m1) {
      unsigned pick = 0, mm = m1;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        pick |= mm & (0u - mm);  // lowest set bit
        mm &= mm - 1;
      }
      m1 &= ~pick;
      const bool has = g < (unsigned)__popc(pick);
      const unsigned rl = has ? nth_set_bit(pick, g) : 0u;
      Off gp = __shfl_sync(kFull, p, rl);
      const Off ge = __shfl_sync(kFull, e, rl);
      bool gf = __shfl_sync(kFull, found ? 1 : 0, rl) != 0;
      uint32_t gx = __shfl_sync(kFull, par, rl);
      while (true) {
        const bool gact = has && gp < ge && !(gf && early_exit);
        if (!__any_sync(kFull, gact)) break;
        bool lf = false;
        uint32_t lx = 0;
        const Off qq = (gp & ~(Off)7) + (Off)(sub * 8u);
        if (gact && qq < ge) probe8(qq, gp, ge, lf, lx);
        const unsigned bm = __ballot_sync(kFull, lf) & (0xFFu << (g * 8u));
        const uint32_t fx = __shfl_sync(kFull, lx, bm ? (unsigned)(__ffs(bm) - 1) : lane);
        if (gact && bm && !gf) {
          gf = true;
          gx = fx;
        }
        if (gact) gp = (gp & ~(Off)7) + 64;
      }
      const bool mine = (pick >> lane) & 1u;
      const unsigned src = mine ? (unsigned)__popc(pick & lanemask_lt()) * 8u : lane;
      const bool rf = __shfl_sync(kFull, gf ? 1 : 0, src) != 0;
      const uint32_t rx = __shfl_sync(kFull, gx, src);
      const Off rp = __shfl_sync(kFull, gp, src);
      if (mine) {
        found = rf;
        par = rx;
        p = rp;
      }
    }
    // tier 2: long remainders, whole warp (256 ids per step: 8 per lane), ballot early exit.
    // Without early exit (the Table-2 ablation arms) a remainder longer than kHubSplit is
    // not scanned here: it becomes kHubSplit-id chunk descriptors that every warp of the
    // grid processes after the item loop (pull_hub_chunks), so the relabelled hubs, which
    // share the first items, do not serialise in one warp.
    unsigned dm = __ballot_sync(kFull, valid && p < e && !(found && early_exit));
    while (dm) {
      const unsigned l = __ffs(dm) - 1;
      dm &= dm - 1;
      const Off pb = __shfl_sync(kFull, p, l), pe = __shfl_sync(kFull, e, l);
      if (!early_exit && pe - pb > (Off)kHubSplit) {
        const unsigned nch = (unsigned)((pe - pb + (Off)kHubSplit - 1) / (Off)kHubSplit);
        unsigned base = 0;
        // capacity: 3*ceil(rem/2048) <= deg/128 for deg > 2048, and hcap >= sum ceil(deg/128)
        if (lane == 0) base = atomicAdd(hub_count, nch);
        base = __shfl_sync(kFull, base, 0);
        // row id (valid only when the row may still commit: unvisited, not yet found)
        const uint32_t ri = __shfl_sync(kFull, i, l);
        const bool may = __shfl_sync(kFull, (i < kNone - 1u && !committed) ? 1 : 0, l) != 0;
        const uint32_t flags = __shfl_sync(kFull, degin & 0x7FFFFFFFu, l) | (may ? 0x80000000u : 0u);
        for (unsigned j = lane; j < nch; j += 32) {
          const Off q0 = pb + (Off)j * (Off)kHubSplit;
          const unsigned len = (unsigned)min((Off)kHubSplit, pe - q0);
          uint2* h = hubs + 3u * (base + j);
          h[0] = make_uint2(ri, flags);
          h[1] = make_uint2((uint32_t)q0, (uint32_t)((unsigned long long)q0 >> 32));
          h[2] = make_uint2(len, 0u);
        }
        if (lane == l) p = e;  // handed over; `found` stays as it was (committed rows only)
        continue;
      }
      bool f = __shfl_sync(kFull, found ? 1 : 0, l) != 0;
      uint32_t fx = __shfl_sync(kFull, par, l);
      for (Off q0 = pb & ~(Off)7; q0 < pe; q0 += 256) {
        bool lf = false;
        uint32_t lx = 0;
        const Off qq = q0 + (Off)(lane * 8u);
        if (qq < pe) probe8(qq, pb, pe, lf, lx);
        const unsigned bm = __ballot_sync(kFull, lf);
        if (bm && !f) {
          f = true;
          fx = __shfl_sync(kFull, lx, __ffs(bm) - 1);
        }
        if (f && early_exit) break;
      }
      if (lane == l) {
        found = f;
        par = fx;
      }
    }
    if (valid && found && !committed) {
      const bool in_item = (i >> 5) >= wbase && (i >> 5) < wbase + pw;
      commit(i, par, (Off)degin, wbase, in_item,
             D ? i - (uint32_t)a.lo : (a.perm ? a.perm[i] : i));
    }
  }
};

// Row-based masked mxv with early exit over the complement of the visited snapshot
// (Alg. 2 re-designed).  Warp item = kPW bitmap words (256 rows); candidates (zero bits)
// are enumerated warp-balanced and processed kC per lane at a time with every stage's
// loads in flight together: offsets (for dense items one coalesced load of the item's
// 257 offsets into shared memory), then each row's aligned 4-id block (ld.global.nc.v4),
// then the first valid id's visited bit, then the block's other ids only for rows that
// missed.  First hit in sorted order = min-id parent (R14).  Rows the block does not
// decide are parked in the warp's residual queue and finished 32 at a time (lane / 8-lane
// group / warp tiers).  Found bits are OR-ed in shared memory; the owning lane writes
// v' = v | found and the frontier bitmap; rows resolved after their item closed use
// atomicOr.
//
// Multi-rank (D): the items cover the owned words [wlo, wlo + wcnt) only; the rows' CSC
// data is local (row i - lo), the probed in-neighbour ids are global and test the
// replicated visited snapshot.
template <typename Off, bool PARENTS, bool D, bool ABL>
__device__ void pull_phase(const BfsArgs<Off>& a, const uint32_t* __restrict__ vin,
                           uint32_t* __restrict__ vout, LevelCtr* out, int d, Acc& acc,
                           uint32_t* sfound, ResidualQ<Off>& rq, const uint32_t* ssum,
                           unsigned* sctr, uint32_t* fr, unsigned* gwork) {
  const unsigned lane = lane_id();
  const unsigned nitems = (D ? a.wcnt : a.nwords) / kPW;
  const unsigned wb0 = D ? a.wlo : 0u;
  const uint32_t lo = D ? (uint32_t)a.lo : 0u;
  // ABL: the Table-2 ablation kernel; the default kernel compiles the toggles out
  const bool no_mask = ABL && (a.toggles & PP_OPT_NO_MASKING) != 0;
  PullCtx<Off, PARENTS, D> C{a, vin, vout, d, !ABL || !(a.toggles & PP_OPT_NO_EARLYEXIT),
                             ABL && (a.toggles & PP_OPT_NO_REUSE) != 0, acc, sfound, rq, ssum,
                             a.H0, &out->work2, fr};
  int qn = 0;
  unsigned wbase = 0;
  // CTA b owns items b, b+G, ... (G = grid, interleaved so every CTA sees the same mix of
  // heavy and light items); its warps grab them in order through the shared-memory counter.
  // The warp grabs one step ahead and loads the next item's visited words meanwhile.
  // (Handing a CTA's last items out one word at a time, or smaller items, measured slower:
  // DESIGN.md §11.)
  const unsigned G = (unsigned)a.ncta;
  const unsigned cta = cta_of(a);
  const unsigned K = nitems > cta ? (nitems - cta + G - 1) / G : 0u;
  auto map = [&](unsigned k, unsigned& w0, unsigned& pw) {
    w0 = wb0 + (cta + k * G) * kPW;
    pw = kPW;
  };
#if PP_STEAL
  // claims an item: own CTA's counter first, then up to PP_STEAL victims' (an item is claimed
  // by exactly one atomicAdd that returns j < K_v, so a thief may give up at any time: the
  // owner processes whatever nobody claimed)
  unsigned vic = cta, tries = 0;
  auto grab = [&]() {
    unsigned it = ~0u;
    if (lane == 0) {
      while (tries <= (unsigned)PP_STEAL) {
        const unsigned j = atomicAdd(&gwork[vic], 1u);
        const unsigned Kv = nitems > vic ? (nitems - vic + G - 1) / G : 0u;
        if (j < Kv) {
          it = vic + j * G;
          break;
        }
        ++tries;
        vic = (vic + 1u + tries * 37u) % G;
      }
    }
    return __shfl_sync(kFull, it, 0);
  };
  auto mapi = [&](unsigned it, unsigned& w0, unsigned& pw) {
    w0 = wb0 + it * kPW;
    pw = kPW;
  };
  unsigned k = grab(), w0n = 0, pwn = 0;
  if (k != ~0u) mapi(k, w0n, pwn);
  uint32_t vw_next = (k != ~0u && lane < pwn) ? vin[w0n + lane] : 0xFFFFFFFFu;
  while (k != ~0u) {
    wbase = w0n;
    const unsigned pw = pwn;
    const bool own = lane < pw;
    const uint32_t vw = vw_next;
    k = grab();
    if (k != ~0u) mapi(k, w0n, pwn);
    vw_next = (k != ~0u && lane < pwn) ? vin[w0n + lane] : 0xFFFFFFFFu;
#else
  (void)gwork;
  bool first = true;  // the first grab is static (first_j)
  auto grab = [&]() {
    if (first) {
      first = false;
      return first_j();
    }
    unsigned j = 0;
    if (lane == 0) j = atomicAdd(sctr, 1u);
    return __shfl_sync(kFull, j, 0);
  };
  unsigned k = grab(), w0n = 0, pwn = 0;
  if (k < K) map(k, w0n, pwn);
  uint32_t vw_next = (k < K && lane < pwn) ? vin[w0n + lane] : 0xFFFFFFFFu;
  while (k < K) {
    wbase = w0n;
    const unsigned pw = pwn;
    const bool own = lane < pw;
    const uint32_t vw = vw_next;
    k = grab();
    if (k < K) map(k, w0n, pwn);
    vw_next = (k < K && lane < pwn) ? vin[w0n + lane] : 0xFFFFFFFFu;
#endif
    const uint32_t unvisited = ~vw;
    // Masking (Opt. 2): only rows with !v(i) are computed.  Without it every
    // non-isolated row is computed and the result filtered afterwards.
    const uint32_t cand = no_mask ? (own ? ~a.isolated[wbase + lane] : 0u) : unvisited;
    sfound[lane] = 0u;
    const unsigned cnt = __popc(cand);
    acc.cand += cnt;
    const unsigned incl = warp_incl_scan(cnt);
    const unsigned excl = incl - cnt;
    const unsigned tot = __shfl_sync(kFull, incl, 31);
    __syncwarp();
    for (unsigned base = 0; base < tot; base += 32 * kC) {
      bool valid[kC], fresh[kC], found[kC];
      uint32_t i[kC], par[kC];
      Off rb[kC], e[kC], p[kC];
#pragma unroll
      for (int t = 0; t < kC; ++t) {
        const unsigned k = base + t * 32 + lane;
        valid[t] = k < tot;
        const unsigned j = warp_owner(incl, k);
        const uint32_t mj = __shfl_sync(kFull, cand, j);
        const unsigned xj = __shfl_sync(kFull, excl, j);
        const uint32_t uj = __shfl_sync(kFull, unvisited, j);
        const unsigned bitpos = valid[t] ? nth_set_bit(mj, k - xj) : 0u;
        const unsigned r = j * 32u + bitpos;  // row within the item
        i[t] = wbase * 32u + r;
        fresh[t] = valid[t] && ((uj >> bitpos) & 1u);
        found[t] = false;
        par[t] = kNone;
        rb[t] = e[t] = 0;
      }
      // stage: the row's 32-byte record {first 6 in-neighbours, caller id (multi-rank: block
      // slot), in-degree}: one 256-bit load from a row-contiguous array (an ELL head in front of
      // the CSR tail); positions are row-relative [0, deg) until a parked row needs its begin
      V8 hd[kC];
      uint32_t dpos[kC];  // where the row's depth goes
#pragma unroll
      for (int t = 0; t < kC; ++t) {
        const uint32_t li = i[t] - lo;  // row of the CSC block (lo = 0 on one GPU)
        dpos[t] = li;
        if (valid[t]) {
          hd[t] = ld_nc_v8(a.drec + (size_t)li * 8u);
          dpos[t] = hd[t].x[6];
          rb[t] = 0;
          e[t] = (Off)hd[t].x[7];
        }
      }
      // stage: probe the first neighbour, then the other head ids of rows that missed
#pragma unroll
      for (int t = 0; t < kC; ++t) {
        const Off deg = e[t] - rb[t];
        if (valid[t] && deg > 0 && C.hit(hd[t].x[0])) {
          found[t] = true;
          par[t] = hd[t].x[0];
        }
      }
#pragma unroll
      for (int t = 0; t < kC; ++t) {
        const Off deg = e[t] - rb[t];
        if (valid[t] && deg > 1 && !(found[t] && C.early_exit)) {
          bool h[kDenseHead];
#pragma unroll
          for (int q = 1; q < kDenseHead; ++q) h[q] = deg > (Off)q && C.hit(hd[t].x[q]);
#pragma unroll
          for (int q = 1; q < kDenseHead; ++q) {
            if (h[q] && !found[t]) {
              found[t] = true;
              par[t] = hd[t].x[q];
            }
          }
        }
        p[t] = (valid[t] && deg > (Off)kDenseHead) ? (Off)kDenseHead : e[t];  // tail continues in idx
      }
#pragma unroll
      for (int t = 0; t < kC; ++t) {
        if (found[t] && fresh[t]) C.commit(i[t], par[t], e[t] - rb[t], wbase, true, dpos[t]);
        // park undecided rows (and, without early exit, rows with ids left)
        const bool park = valid[t] && p[t] < e[t] && !(found[t] && C.early_exit) &&
                          (fresh[t] || !found[t]);
        const unsigned pm = __ballot_sync(kFull, park);
        if (park) {
          const int slot = qn + __popc(pm & lanemask_lt());
          rq.i[slot] = fresh[t] ? i[t] : kNone - 1;  // visited rows (no masking) never commit
          rq.par[slot] = (found[t] || !fresh[t]) ? (found[t] ? par[t] : 0u) : kNone;
          // p is row-relative: the batch adds the row begin (rows that cannot commit, i.e.
          // visited rows of the no-masking ablation, carry no row id: made absolute here)
          rq.p[slot] = fresh[t] ? p[t] : a.coff[i[t] - lo] + p[t];
          rq.rem[slot] = (uint32_t)(e[t] - p[t]) | (fresh[t] ? kRelP : 0u);
          rq.degin[slot] = (uint32_t)(e[t] - rb[t]);
        }
        qn += __popc(pm);
      }
      __syncwarp();
#ifdef PP_KO_RESID  // timing-only knockout: undecided rows are dropped
      qn = 0;
#endif
      while (qn >= 32) C.residual_batch(qn, 32, wbase, pw);
    }
    if (qn > 0) C.residual_batch(qn, qn, wbase, pw);
    __syncwarp();
    const uint32_t fw = own ? sfound[lane] : 0u;
    if (own) {
      vout[wbase + lane] = vw | fw;
      fr[wbase + lane] = fw;
    }
    if (kSumWordsMax && !D && a.sum_shift >= 5) {
      // the item's rows map into one summary word: one aggregated atomic per item
      const uint32_t gi = ((wbase + lane) * 32u) >> a.sum_shift;
      const uint32_t bits = __reduce_or_sync(kFull, fw ? (1u << (gi & 31u)) : 0u);
      if (lane == 0 && bits) atomicOr(&a.sumv[(((wbase * 32u) >> a.sum_shift)) >> 5], bits);
    } else if (kSumWordsMax && !D && fw) {
      for (uint32_t x = fw; x; x &= x - 1) {
        const uint32_t gi = ((wbase + lane) * 32u + (__ffs(x) - 1)) >> a.sum_shift;
        atomicOr(&a.sumv[gi >> 5], 1u << (gi & 31u));
      }
    }
    __syncwarp();
  }
}

// ---- dense pull (PP_DENSE) ---------------------------------------------------------------
// A pull level whose candidates are a large fraction of the rows (C2's heavy levels: ~100% and
// 15-40% of the non-isolated rows) is bound by how many bytes of row data each SM keeps in
// flight, not by the bytes themselves (one row per lane in flight, ~44 B, left
// the heavy pull at ~2.6 TB/s even with every probe knocked out).  Here the row data is a
// 32-byte record per row {in-neighbours 0..5, caller id, in-degree} streamed by the copy
// engine: every warp owns a ring of kDenseR one-KB slots in shared memory; one lane issues a
// cp.async.bulk of a bitmap word's 32 records into a free slot (completion counted on the
// slot's mbarrier), so kDenseR KB per warp are in flight without holding registers.  Words
// whose rows are all visited (or isolated / padding, pre-marked) are never fetched.  A step
// takes the next landed word: lane l owns row l, probes the visited snapshot for the
// record's first in-neighbour, then (on a miss) the other five (Alg. 2 with masking, early
// exit and operand reuse; first hit in sorted order = min-id parent, R14); rows
// longer than 6 that no record id decides go to the residual tiers.  The word's found bits
// come from one ballot, so v' and the frontier bitmap are written as whole words.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
      " selp.u32 %0, 1, 0, P;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

// Per-warp ring (shared memory): kDenseR slots of 32 records, their mbarriers, and the word
// index / visited word each slot holds.
struct DenseRing {
  uint32_t* rec;             // [kDenseR][256]
  unsigned long long* bar;   // [kDenseR]
  uint32_t* word;            // [kDenseR]
  uint32_t* vw;              // [kDenseR]
  unsigned* seq;             // bulk copies this warp issued (= consumed between phases)
};
// The calling warp's ring, from the dynamic shared memory layout (recomputed where used, so no
// ring state stays live in registers across the level loop).  Layout: dense_ring_offset(),
// then kBfsWarps*kDenseR slots of 1 KB, their mbarriers, words, visited words, and one
// sequence counter per warp.
template <typename Off>
__device__ __forceinline__ DenseRing dense_ring(unsigned char* dyn, size_t off) {
  const unsigned warp = threadIdx.x >> 5;
  unsigned char* rb = dyn + off;
  unsigned char* mb = rb + (size_t)kBfsWarps * kDenseR * 1024;
  uint32_t* meta = reinterpret_cast<uint32_t*>(mb + (size_t)kBfsWarps * kDenseR * 8);
  DenseRing r;
  r.rec = reinterpret_cast<uint32_t*>(rb) + (size_t)warp * kDenseR * 256;
  r.bar = reinterpret_cast<unsigned long long*>(mb) + (size_t)warp * kDenseR;
  r.word = meta + (size_t)warp * kDenseR;
  r.vw = meta + (size_t)kBfsWarps * kDenseR + (size_t)warp * kDenseR;
  r.seq = meta + (size_t)2 * kBfsWarps * kDenseR + warp;
  return r;
}

template <typename Off, bool PARENTS, bool D>
__device__ void pull_dense(const BfsArgs<Off>& a, const uint32_t* __restrict__ vin,
                           uint32_t* __restrict__ vout, LevelCtr* out, int d, Acc& acc,
                           uint32_t* sfound, ResidualQ<Off>& rq, unsigned* sctr, uint32_t* fr,
                           const DenseRing& R) {
  const unsigned lane = lane_id();
  PullCtx<Off, PARENTS, D> C{a, vin, vout, d, true, false, acc, sfound, rq, nullptr,
                             a.H0, &out->work2, fr};
  int qn = 0;
  // multi-rank (D): the items cover the owned words [wlo, wlo + wcnt), whose records are the
  // block's (row i - lo); one GPU: all words, wlo = lo = 0
  const unsigned wb0 = D ? a.wlo : 0u;
  const uint32_t lo = D ? (uint32_t)a.lo : 0u;
  const unsigned nitems = (D ? a.wcnt : a.nwords) / kDenseIW;
  const unsigned G = (unsigned)a.ncta;
  const unsigned cta = cta_of(a);
  const unsigned K = nitems > cta ? (nitems - cta + G - 1) / G : 0u;
  // producer: the item whose words are being issued (CTA-interleaved items, grabbed by the
  // CTA's warps in order), the words of it still to fetch, and their visited words (lane j < kPW)
  unsigned pk = 0, pbase = 0, pneed = 0;
  uint32_t pvw = 0xFFFFFFFFu;
  bool more = true;
  const unsigned seq0 = *R.seq;
  unsigned issued = seq0, cons = seq0;
  // the item after the producer's is grabbed, and its visited words loaded, one item ahead
  bool first = true;  // the first grab is static (first_j)
  auto grab_item = [&](uint32_t& vw_out) {
    unsigned j = first_j();
    if (!first) {
      if (lane == 0) j = atomicAdd(sctr, 1u);
      j = __shfl_sync(kFull, j, 0);
    }
    first = false;
    vw_out = (j < K && lane < kDenseIW) ? vin[wb0 + (cta + j * G) * kDenseIW + lane] : 0xFFFFFFFFu;
    return j;
  };
  uint32_t nvw;
  unsigned nk = grab_item(nvw);
  auto next_item = [&]() {  // warp-uniform; false when the CTA has no items left
    while (pneed == 0) {
      if (nk >= K) return false;
      pk = nk;
      pbase = wb0 + (cta + pk * G) * kDenseIW;
      pvw = nvw;
      nk = grab_item(nvw);
      const bool need = pvw != 0xFFFFFFFFu;
      pneed = __ballot_sync(kFull, need);
      if (lane < kDenseIW && !need) {  // nothing to compute: v' = v, no discoveries
        vout[pbase + lane] = 0xFFFFFFFFu;
        fr[pbase + lane] = 0u;
      }
    }
    return true;
  };
  auto issue = [&]() {  // fills the free slots; warp-uniform
    while (kDenseR > 0 && more && issued - cons < (unsigned)kDenseR) {
      if (pneed == 0 && !next_item()) {
        more = false;
        break;
      }
      const unsigned j = __ffs(pneed) - 1;
      pneed &= pneed - 1;
      const uint32_t vwj = __shfl_sync(kFull, pvw, j);
      const unsigned slot = issued % (unsigned)(kDenseR > 0 ? kDenseR : 1);
      if (lane == 0) {
        R.word[slot] = pbase + j;
        R.vw[slot] = vwj;
        mbar_arrive_tx(&R.bar[slot], 1024u);
        bulk_g2s(R.rec + slot * 256u, a.drec + (size_t)(pbase + j - wb0) * 256u, 1024u, &R.bar[slot]);
      }
      ++issued;
    }
    __syncwarp();
  };
  // one bitmap word: lane l owns row w*32 + l, its record is {x0..x5 | x0..x4 + begin, caller, deg}
  auto process = [&](uint32_t w, uint32_t vw, const uint4& r0, const uint4& r1) {
    const bool cand = !((vw >> lane) & 1u);
    acc.cand += cand ? 1u : 0u;
    const uint32_t dg = r1.w;
    bool found = cand && dg > 0u && C.hit(r0.x);
    uint32_t par = r0.x;
    // the other record ids only for rows whose first id missed (probing all six in one round
    // measured slower: DESIGN.md §11)
    if (cand && !found && dg > 1u) {
      const uint32_t x[5] = {r0.y, r0.z, r0.w, r1.x, r1.y};
      constexpr int kX = kDenseHead - 1;  // ids after the first in the record
      bool h[kX];
#pragma unroll
      for (int q = 0; q < kX; ++q) h[q] = dg > (uint32_t)(q + 1) && C.hit(x[q]);
#pragma unroll
      for (int q = kX - 1; q >= 0; --q)
        if (h[q]) {
          found = true;
          par = x[q];
        }
    }
    const uint32_t fb = __ballot_sync(kFull, found);
    if (lane == 0) {
      vout[w] = vw | fb;
      fr[w] = fb;
    }
    const uint32_t i = w * 32u + lane;
    if (found) {
      a.depth[r1.z] = d + 1;  // caller id (multi-rank: the block slot i - lo)
      if (PARENTS) a.parent[i - lo] = par;
      const Off odg = a.symmetric ? (Off)dg
                                  : (D ? (Off)a.odeg[i - lo] : (Off)(a.off[i + 1] - a.off[i]));
      acc.c += 1;
      acc.mf += (unsigned long long)odg;
      acc.mfin += (unsigned long long)dg;
      acc.big += odg >= (Off)kBig ? 1u : 0u;
    }
    // rows longer than the record that no record id decided: the residual tiers
    const bool park = cand && !found && dg > (uint32_t)kDenseHead;
    const unsigned pm = __ballot_sync(kFull, park);
    if (park) {
      const int slot = qn + __popc(pm & lanemask_lt());
      rq.i[slot] = i;
      rq.par[slot] = kNone;
      rq.p[slot] = (Off)kDenseHead;  // relative: the batch adds coff[i] (one round trip per
      rq.rem[slot] = (dg - (uint32_t)kDenseHead) | kRelP;  // batch, not per step)
      rq.degin[slot] = dg;
    }
    qn += __popc(pm);
    __syncwarp();
    while (qn >= 32) C.residual_batch(qn, 32, 0u, 0u);
  };
  {
    issue();
    while (cons != issued) {
      const unsigned slot = cons % (unsigned)kDenseR;
      const unsigned par = (cons / (unsigned)kDenseR) & 1u;
      if (!mbar_try(&R.bar[slot], par)) {
        const unsigned long long t0 = global_timer_ns();
        while (!mbar_try(&R.bar[slot], par))
          if (global_timer_ns() - t0 > kWatchdogNs) __trap();  // a lost copy: fail, never hang
      }
      const uint32_t w = R.word[slot], vw = R.vw[slot];
      const uint4* rp = reinterpret_cast<const uint4*>(R.rec + slot * 256u) + 2 * lane;
      const uint4 r0 = rp[0], r1 = rp[1];
      ++cons;
      __syncwarp();  // every lane has its records: the slot may be refilled
      issue();
      process(w, vw, r0, r1);
    }
  }
  if (qn > 0) C.residual_batch(qn, qn, 0u, 0u);
  if (lane == 0) *R.seq = issued;
  __syncwarp();
}

// No-early-exit pull, second part: the long-row chunks emitted by tier 2, grabbed by every
// warp of the grid (global counter: few chunks).  A chunk scans its ids in full (no early
// exit), takes its first hit in sorted order, and the row's commit happens once, by the
// chunk whose atomicOr on v' flips the bit (the item owning the row has closed); the
// min-id parent is the atomicMin of the chunks' first hits (R14).
template <typename Off, bool PARENTS>
__device__ void pull_hub_chunks(const BfsArgs<Off>& a, const uint32_t* __restrict__ vin,
                                uint32_t* __restrict__ vout, LevelCtr* out, unsigned nch, int d,
                                Acc& acc, ResidualQ<Off>& rq) {
  const unsigned lane = lane_id();
  PullCtx<Off, PARENTS, false> C{a, vin, vout, d, false, (a.toggles & PP_OPT_NO_REUSE) != 0,
                                 acc, nullptr, rq, nullptr, a.H0, nullptr, a.fr};
  while (true) {
    unsigned j = 0;
    if (lane == 0) j = atomicAdd(&out->work, 1u);
    j = __shfl_sync(kFull, j, 0);
    if (j >= nch) break;
    const uint2 h0 = a.H0[3u * j], h1 = a.H0[3u * j + 1u], h2 = a.H0[3u * j + 2u];
    const uint32_t i = h0.x;
    const bool may = (h0.y >> 31) != 0;  // row unvisited and not found yet (else: scan only)
    const Off degin = (Off)(h0.y & 0x7FFFFFFFu);
    const Off q0 = (Off)(((unsigned long long)h1.y << 32) | h1.x);
    const Off e = q0 + (Off)h2.x;
    bool f = false;
    uint32_t fx = 0;
    for (Off qb = q0 & ~(Off)7; qb < e; qb += 256) {
      bool lf = false;
      uint32_t lx = 0;
      const Off qq = qb + (Off)(lane * 8u);
      if (qq < e) C.probe8(qq, q0, e, lf, lx);
      const unsigned bm = __ballot_sync(kFull, lf);
      if (bm && !f) {
        f = true;
        fx = __shfl_sync(kFull, lx, __ffs(bm) - 1);
      }
    }
    if (f && may && lane == 0) {
      if (PARENTS) atomicMin(&a.parent[i], fx);
      const uint32_t bit = 1u << (i & 31u);
      const uint32_t old = atomicOr(&vout[i >> 5], bit);
      if (!(old & bit)) {
        atomicOr(&a.fr[i >> 5], bit);
        a.depth[a.perm ? a.perm[i] : i] = d + 1;
        const Off deg = a.symmetric ? degin : (Off)(a.off[i + 1] - a.off[i]);
        acc.c += 1;
        acc.mf += (unsigned long long)deg;
        acc.mfin += (unsigned long long)degin;
        acc.big += deg >= (Off)kBig ? 1u : 0u;
      }
    }
  }
}

// Dense2sparse of the new frontier v' & !v after a pull level (pull->push switch).
template <typename Off>
__device__ void convert_phase(const BfsArgs<Off>& a, const uint32_t* vnew, const uint32_t* vold,
                              uint4* Lout, uint2* Hout, LevelCtr* out, unsigned* sctr) {
  const unsigned lane = lane_id();
  const unsigned nchunks = a.nwords / 32u;
  for (unsigned item = cta_first(a); item < nchunks; item = cta_grab(a, sctr)) {
    const unsigned w = item * 32u + lane;
    uint32_t diff = vold ? (vnew[w] & ~vold[w]) : vnew[w];  // multi-rank: vnew = frontier
    while (__ballot_sync(kFull, diff != 0u)) {
      const bool valid = diff != 0u;
      uint32_t v = 0;
      Off deg = 0, beg = 0;
      if (valid) {
        const unsigned b = __ffs(diff) - 1;
        diff &= diff - 1;
        v = w * 32u + b;
        beg = a.off[v];
        deg = a.off[v + 1] - beg;
      }
      append_frontier<Off>(valid, v, deg, beg, Lout, Hout, a.hcap, out);
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

template <typename Off>
struct BfsShared {  // static part; the residual queues live in dynamic shared memory
  uint32_t sfound[kBfsWarps][32];
  unsigned long long red[kBfsWarps][5];
  long long lvl[8];  // c, m_f, m_fin, nL, nH, nbig, nB, cand of the level just finished
  unsigned work;     // CTA-local work counter (cta_grab)
  unsigned xlmask;   // multi-rank: senders whose last exchange was an id list ...
  unsigned xlen[kMaxRanks];  // ... and the lists' lengths
};



// thread 0 reads a level's counters once (post-barrier) and broadcasts them via smem
template <typename Off>
__device__ __forceinline__ void read_level(const LevelCtr* out, BfsShared<Off>& sh) {
  if (threadIdx.x == 0) {
    sh.lvl[0] = (long long)ld_relaxed_u64(&out->c);
    sh.lvl[1] = (long long)ld_relaxed_u64(&out->m_f);
    sh.lvl[2] = (long long)ld_relaxed_u64(&out->m_fin);
    sh.lvl[3] = (long long)ld_relaxed_u32(&out->nL);
    sh.lvl[4] = (long long)ld_relaxed_u32(&out->nH);
    sh.lvl[5] = (long long)ld_relaxed_u64(&out->nbig);
    sh.lvl[6] = (long long)ld_relaxed_u32(&out->nB);
    sh.lvl[7] = (long long)ld_relaxed_u64(&out->cand);
    sh.work = (unsigned)kBfsWarps;  // item j < kBfsWarps is warp j's static first grab
  }
  __syncthreads();
}

__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Multi-rank: one cross-rank rendezvous.  Thread 0 of CTA 0 stores `tag` into its slot of
// every peer's flag array (release, system scope: the rank's earlier peer stores, fenced by
// every CTA and collected by the rank-local barrier before this call, become visible first);
// thread 0 of every CTA then waits (acquire, system scope) until every peer's flag in its own
// array reached `tag`.  Watchdog as in grid_barrier.
template <typename Off>
__device__ __forceinline__ bool rank_rendezvous(const BfsArgs<Off>& a, unsigned long long tag) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    int ok = 1;
    if (cta_of(a) == 0)
      for (int q = 0; q < a.nranks; ++q)
        if (q != a.me) st_release_sys_u64(a.pflag[q] + a.me, tag);
    const unsigned long long t0 = global_timer_ns();
    for (int q = 0; q < a.nranks && ok; ++q) {
      if (q == a.me) continue;
      while (ld_acquire_sys_u64(a.xflag + q) < tag) {
        __nanosleep(32);
        if (global_timer_ns() - t0 > kWatchdogNs) {
          atomicExch(&a.status->error, (int)PP_ERR_TIMEOUT);
          atomicOr(reinterpret_cast<unsigned long long*>(&a.bar->count), kAbortBit);
          ok = 0;
          break;
        }
      }
    }
    __threadfence();
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// Multi-rank exchange after level d (SURVEY.md §8e, NEXT-1 "exchange fused into the level
// kernel over NVLink").  Entered by every CTA of the rank right after the level barrier;
// sh.lvl holds this rank's counter sums.  (1) the owned words of the level's frontier bitmap
// go straight into every peer's copy (16-byte peer stores); (2) the rank's counter record
// (c, m_f, m_fin, big) goes into its slot of every rank's table; (3) system-scope fence,
// rank-local barrier, one release flag per peer and the wait for the peers' flags;
// (4) every CTA sums the P records, so every rank continues with identical global counters
// and takes the identical direction decision (R10/R11) without any host round trip.
template <typename Off>
__device__ bool exchange(const BfsArgs<Off>& a, BfsShared<Off>& sh, const uint32_t* frout, int d,
                         unsigned& epoch, long long extra_mfin, unsigned long long gtid,
                         unsigned long long gsize, bool was_push, const LevelCtr* out) {
  const int P = a.nranks, me = a.me;
  const unsigned par = (unsigned)d & 1u;
  // hybrid encoding: after a push level whose discoveries are fewer than
  // the slice's words, the id list (4 bytes per discovery) replaces the bitmap slice
  const unsigned nx = was_push ? ld_relaxed_u32(&out->nX) : ~0u;
  const bool lst = was_push && nx < a.wcnt;
  if (P > 1) {
    if (lst) {
      const unsigned long long tot = (unsigned long long)nx * (unsigned)(P - 1);
      for (unsigned long long k = gtid; k < tot; k += gsize) {
        const int qi = (int)(k / nx);
        const unsigned j = (unsigned)(k - (unsigned long long)qi * nx);
        const int q = qi >= me ? qi + 1 : qi;
        a.plst[q][par][(size_t)me * a.wcnt + j] = a.xown[j];
      }
    } else {
      const unsigned nv = a.wcnt / 4u;
      const uint4* src = reinterpret_cast<const uint4*>(frout + a.wlo);
      const unsigned long long tot = (unsigned long long)nv * (unsigned)(P - 1);
      for (unsigned long long k = gtid; k < tot; k += gsize) {
        const int qi = (int)(k / nv);
        const unsigned j = (unsigned)(k - (unsigned long long)qi * nv);
        const int q = qi >= me ? qi + 1 : qi;
        reinterpret_cast<uint4*>(a.pfr[q][par] + a.wlo)[j] = src[j];
      }
    }
  }
  if (cta_of(a) == 0 && threadIdx.x < (unsigned)P) {
    unsigned long long* rec = a.pcnt[threadIdx.x] + ((size_t)par * kMaxRanks + (size_t)me) * 8u;
    rec[0] = (unsigned long long)sh.lvl[0];
    rec[1] = (unsigned long long)sh.lvl[1];
    rec[2] = (unsigned long long)(sh.lvl[2] + extra_mfin);
    rec[3] = (unsigned long long)sh.lvl[5];
    rec[4] = lst ? (unsigned long long)nx : ~0ull;  // list length, or ~0: bitmap slice
    rec[5] = (unsigned long long)sh.lvl[7];
  }
  if (cta_of(a) == 0 && threadIdx.x == 0 && P > 1)
    a.status->xbytes += (long long)(P - 1) * ((lst ? 4ll * nx : 4ll * a.wcnt) + 40);
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
  if (!grid_barrier(a.bar, a.status, epoch, (unsigned)a.ncta)) return false;
  if (P > 1 && !rank_rendezvous(a, a.xseq + (unsigned long long)d)) return false;
  if (threadIdx.x == 0) {
    long long c = 0, mf = 0, mfin = 0, big = 0, cd = 0;
    unsigned lmask = 0;
    for (int q = 0; q < P; ++q) {
      const unsigned long long* rec = a.xcnt + ((size_t)par * kMaxRanks + (size_t)q) * 8u;
      c += (long long)ld_relaxed_u64(rec + 0);
      mf += (long long)ld_relaxed_u64(rec + 1);
      mfin += (long long)ld_relaxed_u64(rec + 2);
      big += (long long)ld_relaxed_u64(rec + 3);
      cd += (long long)ld_relaxed_u64(rec + 5);
      const unsigned long long ln = ld_relaxed_u64(rec + 4);
      if (q != me && ln != ~0ull) {
        lmask |= 1u << q;
        sh.xlen[q] = (unsigned)ln;
      }
    }
    sh.lvl[0] = c;
    sh.lvl[1] = mf;
    sh.lvl[2] = mfin;
    sh.lvl[5] = big;
    sh.lvl[7] = cd;
    sh.xlmask = lmask;
  }
  __syncthreads();
  return true;
}

// dynamic shared memory: residual queues, visited summary, then (PP_DENSE, 128-byte aligned)
// the warps' bulk-copy rings, their mbarriers and slot metadata
template <typename Off>
__host__ __device__ constexpr size_t dense_ring_offset() {
  return (sizeof(ResidualQ<Off>) * kBfsWarps + sizeof(uint32_t) * kSumWordsMax + 127) & ~(size_t)127;
}
template <typename Off, bool D = false>
__host__ __device__ constexpr size_t dyn_smem_bytes() {  // multi-rank: rings only with PP_DENSE_DIST
  return (kDenseR && (!D || PP_DENSE_DIST))
             ? dense_ring_offset<Off>() + (size_t)kBfsWarps * (kDenseR * (1024 + 8 + 4 + 4) + 4)
             : sizeof(ResidualQ<Off>) * kBfsWarps + sizeof(uint32_t) * kSumWordsMax;
}

// The BFS loop (Algorithm 1) run by the CTAs of one rank.  D = multi-rank (1D
// row partition): the same push / pull / convert phases over the rank's block, plus the
// exchange after every level and a merge of the peers' discoveries into the visited bitmap.
template <typename Off, bool PARENTS, bool D, bool ABL = false>
__device__ __forceinline__ void bfs_body(const BfsArgs<Off>& a) {
  __shared__ BfsShared<Off> sh;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  ResidualQ<Off>* rqs = reinterpret_cast<ResidualQ<Off>*>(dyn_smem);
  uint32_t* ssum = reinterpret_cast<uint32_t*>(dyn_smem + sizeof(ResidualQ<Off>) * kBfsWarps);
  const unsigned warp = threadIdx.x >> 5;
  if constexpr (kDenseR > 0 && (!D || PP_DENSE_DIST)) {
    if (a.drec) {
      const DenseRing ring = dense_ring<Off>(dyn_smem, dense_ring_offset<Off>());
      if (lane_id() == 0) {
        for (int r = 0; r < kDenseR; ++r) mbar_init(&ring.bar[r], 1u);
        *ring.seq = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      __syncwarp();
    }
  }
  const unsigned cta = cta_of(a);
  const unsigned long long gtid = (unsigned long long)cta * blockDim.x + threadIdx.x;
  const unsigned long long gsize = (unsigned long long)a.ncta * blockDim.x;
  // internal id of the source (relabelled graph) / its global id (multi-rank)
  const uint32_t s = (!D && a.rank) ? a.rank[a.source] : a.source;
  if (a.resume && a.bar->rs.done) return;  // the narrow launch finished the BFS
  if (!a.resume && cta == 0 && threadIdx.x == 0)
    a.status->t_start = (long long)global_timer_ns();
  unsigned epoch = 0;  // grid barriers passed (thread 0)
  // multi-rank: the owned block and the source's slot in it
  const bool own_s = D && (int64_t)s >= a.lo && (int64_t)s < a.hi;
  const unsigned long long nloc = D ? (unsigned long long)(a.hi - a.lo) : (unsigned long long)a.n;
  const unsigned long long srcl = D ? (own_s ? (unsigned long long)(s - (uint32_t)a.lo) : ~0ull)
                                    : (unsigned long long)a.source;

  int dir = (a.mode == 2) ? 1 : 0;
  int cur = 0;  // visited bitmap in use
  int sel = 0;  // frontier list / chunk buffers holding the current frontier
  long long c_old = 1;
  long long m_u, indeg_s_own = 0;
  if (D) {
    // m_u starts at the global in-degree mass; the source's owner adds indeg(s) to its
    // level-1 m_fin record, so every rank subtracts it after level 1
    m_u = a.in_total;
    if (own_s) indeg_s_own = (long long)(a.coff[s - (uint32_t)a.lo + 1] - a.coff[s - (uint32_t)a.lo]);
  } else {
    const Off indeg_s = a.coff[s + 1] - a.coff[s];
    m_u = a.nnz - (long long)indeg_s;
  }
  long long reached = 1;
  Acc acc{0, 0, 0, 0, 0};
  bool from_bits = false;  // next push reads the previous level's frontier bitmap
  // edges the next push expands (a latency heuristic only; multi-rank: this rank's part)
  long long mf_last = (long long)(a.off[s + 1] - a.off[s]);
  int d = 1;
  unsigned nL = 0, nH = 0, nB = 0;
  if (a.resume) {  // continue where the narrow cluster stopped (stream-ordered after it)
    const BfsResume& r = a.bar->rs;
    d = r.d;
    dir = r.dir;
    cur = r.cur;
    sel = r.sel;
    from_bits = r.from_bits != 0;
    nL = r.nL;
    nH = r.nH;
    nB = r.nB;
    c_old = r.c_old;
    m_u = r.m_u;
    reached = r.reached;
    mf_last = r.mf_last;
    if (threadIdx.x == 0) sh.work = (unsigned)kBfsWarps;
    __syncthreads();
  } else {
  // ---- Alg. 1 lines 2-4: d <- 1, f <- e_s, v <- 0 (depth 0 = unvisited) ----
  if (kInitVec && !PARENTS && (reinterpret_cast<uintptr_t>(a.depth) & 15u) == 0) {
    // 16-byte stores: a quarter of the store instructions of the scalar loop
    const unsigned long long n4 = nloc / 4u;
    int4* d4 = reinterpret_cast<int4*>(a.depth);
    for (unsigned long long q = gtid; q < n4; q += gsize) {
      const unsigned long long v0 = q * 4u;
      d4[q] = make_int4(v0 == srcl, v0 + 1 == srcl, v0 + 2 == srcl, v0 + 3 == srcl);
    }
    for (unsigned long long v = n4 * 4u + gtid; v < nloc; v += gsize)
      a.depth[v] = (v == srcl) ? 1 : 0;
  } else {
    for (unsigned long long v = gtid; v < nloc; v += gsize) {
      a.depth[v] = (v == srcl) ? 1 : 0;                              // caller ids / block slots
      if (PARENTS) a.parent[v] = (v == (D ? srcl : (unsigned long long)s)) ? s : 0xFFFFFFFFu;
    }
  }
  // visited starts as {s} plus the isolated / padding vertices, which no pull may
  // compute and no push can reach (they have no edges).  Multi-rank: the isolated words of
  // other blocks are 0 here (never tested), and the level-0 frontier {s} is xfr0.
  const uint32_t sbit_w = s >> 5, sbit = 1u << (s & 31u);
  for (unsigned long long w = gtid; w < a.nwords; w += gsize) {
    a.vis0[w] = a.isolated[w] | ((w == sbit_w) ? sbit : 0u);
    if (D) {
      a.xfr0[w] = (w == sbit_w) ? sbit : 0u;
      if (w >= a.wlo && w < (unsigned long long)a.wlo + a.wcnt) a.xfr1[w] = 0u;
    }
  }
  {
    const uint32_t gs = s >> a.sum_shift;
    for (unsigned long long w = gtid; w < a.sum_words; w += gsize)
      a.sumv[w] = (w == (gs >> 5)) ? (1u << (gs & 31u)) : 0u;
  }
  if (cta == 0) {
    for (int t = threadIdx.x; t < kRing * (int)(sizeof(LevelCtr) / 4); t += blockDim.x)
      reinterpret_cast<unsigned*>(a.ctr)[t] = 0u;
    if (PP_STEAL)
      for (int t = threadIdx.x; t < kRing * kMaxCtas; t += blockDim.x) a.gwork[t] = 0u;
    __syncthreads();
    const Off deg = a.off[s + 1] - a.off[s];  // multi-rank: s's edges into this block
    if (deg >= (Off)kHeavy) {
      const unsigned nch = (unsigned)((deg + (Off)kChunk - 1) / (Off)kChunk);
      if (nch <= kSelfChunks) {
        for (unsigned k = threadIdx.x; k < nch; k += blockDim.x) a.H0[k] = make_uint2(s, k);
        if (threadIdx.x == 0) a.ctr[0].nH = nch;
      } else {
        const unsigned nb = (nch + 31u) / 32u;
        for (unsigned j = threadIdx.x; j < nb; j += blockDim.x)
          a.H0[a.hcap - 1u - j] = make_uint2(s, 32u * j);
        if (threadIdx.x == 0) a.ctr[0].nB = nb;
      }
    } else if (deg > 0 && threadIdx.x == 0) {
      a.L0[0] = light_entry<Off>(s, deg, a.off[s]);
      a.ctr[0].nL = 1;
    }
  }
  if (!level_barrier(a.narrow, a.bar, a.status, epoch, (unsigned)a.ncta)) return;
  read_level(&a.ctr[0], sh);
  if (cta == 0 && threadIdx.x == 0) a.status->t_init = (long long)global_timer_ns();
  nL = (unsigned)sh.lvl[3];
  nH = (unsigned)sh.lvl[4];
  nB = (unsigned)sh.lvl[6];
  }
  for (;; ++d) {
    if ((a.narrow && (dir == 1 || (unsigned long long)mf_last > kNarrowMaxEdges)) ||
        (a.stop_before > 0 && d >= a.stop_before)) {
      // this level is too wide for one cluster: hand the loop to the whole grid
      if (cta == 0 && threadIdx.x == 0) {
        BfsResume& r = a.bar->rs;
        r.d = d;
        r.dir = dir;
        r.cur = cur;
        r.sel = sel;
        r.from_bits = from_bits ? 1 : 0;
        r.nL = nL;
        r.nH = nH;
        r.nB = nB;
        r.c_old = c_old;
        r.m_u = m_u;
        r.reached = reached;
        r.mf_last = mf_last;
        r.valid = 1;
      }
      return;
    }
    const long long t_lvl = (a.dbg && threadIdx.x == 0) ? (long long)global_timer_ns() : 0;
    LevelCtr* out = &a.ctr[d & (kRing - 1)];
    if (cta == 0 && threadIdx.x < (unsigned)(sizeof(LevelCtr) / 4))
      reinterpret_cast<unsigned*>(&a.ctr[(d + 1) & (kRing - 1)])[threadIdx.x] = 0u;
    if (PP_STEAL && cta == 0 && threadIdx.x < (unsigned)kMaxCtas)
      a.gwork[(size_t)((d + 1) & (kRing - 1)) * kMaxCtas + threadIdx.x] = 0u;
    uint32_t* vis = cur ? a.vis1 : a.vis0;
    uint32_t* vis_other = cur ? a.vis0 : a.vis1;
    // frontier bitmap this level writes (pull; multi-rank also push) and the previous one
    uint32_t* frout = D ? ((d & 1) ? a.xfr1 : a.xfr0) : a.fr;
    uint32_t* frin = D ? ((d & 1) ? a.xfr0 : a.xfr1) : a.fr;
    if (dir == 0) {
      push_phase<Off, PARENTS, D>(a, sel ? a.L1 : a.L0, from_bits ? 0u : nL, sel ? a.H1 : a.H0,
                                  from_bits ? 0u : nH, from_bits ? 0u : nB, from_bits ? frin : nullptr,
                                  sel ? a.L0 : a.L1, sel ? a.H0 : a.H1, out, vis, d + 1, acc,
                                  &sh.work, (unsigned long long)mf_last <= kLowLatEdges, frout);
      from_bits = false;
    } else {
      if (kSumWordsMax) {
        for (unsigned t = threadIdx.x; t < a.sum_words; t += blockDim.x) ssum[t] = a.sumv[t];
        __syncthreads();
      }
      bool dense = false;
      if constexpr (kDense && (!D || PP_DENSE_DIST))
        dense = !ABL && a.drec != nullptr && !a.narrow &&
                (a.n_noniso - reached) * 8 >= a.n_noniso * (long long)PP_DENSE_MIN8;
      if (dense) {
        if constexpr (kDense)
          pull_dense<Off, PARENTS, D>(a, vis, vis_other, out, d, acc, sh.sfound[warp], rqs[warp],
                                   &sh.work, frout,
                                   dense_ring<Off>(dyn_smem, dense_ring_offset<Off>()));
      } else {
        pull_phase<Off, PARENTS, D, ABL>(a, vis, vis_other, out, d, acc, sh.sfound[warp], rqs[warp],
                                    ssum, &sh.work, frout, a.gwork + (size_t)(d & (kRing - 1)) * kMaxCtas);
      }
      if (!D && ABL && (a.toggles & PP_OPT_NO_EARLYEXIT)) {  // ablation arms: long rows grid-wide
        if (!level_barrier(a.narrow, a.bar, a.status, epoch, (unsigned)a.ncta)) return;
        const unsigned nch = ld_relaxed_u32(&out->work2);
        if (nch) pull_hub_chunks<Off, PARENTS>(a, vis, vis_other, out, nch, d, acc, rqs[warp]);
      }
    }
    if (a.dbg && threadIdx.x == 0 && d - 1 < a.dbg_levels)
      a.dbg[(size_t)(d - 1) * a.ncta + cta] = (long long)global_timer_ns() - t_lvl;
    flush_acc(acc, out, sh.red);
    // debug phases (pp_bfs_debug_phases): plane 1 = every warp of the CTA done (counters
    // flushed), plane 2 = the grid barrier released; ns from the level's loop top
    const bool dbgp = a.dbg && threadIdx.x == 0 && d - 1 < a.dbg_levels;
    const size_t dplane = (size_t)a.dbg_levels * (size_t)a.ncta, dslot = (size_t)(d - 1) * a.ncta + cta;
    if (dbgp) a.dbg[dplane + dslot] = (long long)global_timer_ns() - t_lvl;
    if (!level_barrier(a.narrow, a.bar, a.status, epoch, (unsigned)a.ncta)) return;
    if (dbgp) a.dbg[2 * dplane + dslot] = (long long)global_timer_ns() - t_lvl;
    read_level(out, sh);
    if (D && !exchange<Off>(a, sh, frout, d, epoch, (d == 1) ? indeg_s_own : 0, gtid, gsize,
                            dir == 0, out))
      return;
    const long long c_new = sh.lvl[0], mf = sh.lvl[1], mfin = sh.lvl[2];
    nL = (unsigned)sh.lvl[3];
    nH = (unsigned)sh.lvl[4];
    nB = (unsigned)sh.lvl[6];
    const int dir_done = dir;
    if (dir == 1) cur ^= 1;
    else if (!D) sel ^= 1;  // multi-rank pushes append nothing (the frontier is exchanged)
    m_u -= (D || !a.symmetric) ? mfin : mf;
    reached += c_new;
    if (cta == 0 && threadIdx.x == 0 && d - 1 < a.stats_cap) {
      LevelStat st;
      st.dir = dir;
      st.pad = 0;
      st.c = c_new;
      st.m_f = mf;
      st.m_u = m_u;
      st.cand = dir ? sh.lvl[7] : c_old;  // pull: rows computed; push: frontier expanded
      st.t_ns = (long long)global_timer_ns();
      a.stats[d - 1] = st;
    }
    const bool done = c_new == 0 || d >= a.max_levels;
    int next = dir;
    if (!done && a.mode == 0)
      next = decide(a.rule, dir, c_old, c_new, mf, m_u, a.n, a.alpha, a.beta);
    if (done) break;
    if (D) {
      // merge the peers' discoveries into the visited bitmap the next level reads (the owned
      // words are already final), clear the owned words of the next push's output bitmap,
      // and build this rank's push frontier from the exchanged bitmap: straight from the
      // bitmap when no frontier vertex is big, else Dense2sparse into light list / chunks
      uint32_t* vbase = dir_done ? vis : vis;        // pull: the snapshot; push: updated in place
      uint32_t* vnext = cur ? a.vis1 : a.vis0;       // bitmap the next level reads
      uint32_t* frnext = (d & 1) ? a.xfr0 : a.xfr1;  // output of level d + 1
      const unsigned long long wlo = a.wlo, whi = (unsigned long long)a.wlo + a.wcnt;
      const unsigned lmask = sh.xlmask;
      for (unsigned long long w = gtid; w < a.nwords; w += gsize) {
        if (w >= wlo && w < whi) {
          if (next == 0) frnext[w] = 0u;
        } else if ((lmask >> (unsigned)(w / a.wcnt)) & 1u) {
          frout[w] = 0u;  // this sender sent an id list: its slice is rebuilt below
        } else {
          vnext[w] = vbase[w] | frout[w];
        }
      }
      if (lmask) {  // id lists: set their bits in the frontier and visited bitmaps
        if (!level_barrier(false, a.bar, a.status, epoch, (unsigned)a.ncta)) return;
        const uint32_t* lst = (d & 1) ? a.xlst1 : a.xlst0;
        for (int q = 0; q < a.nranks; ++q) {
          if (!((lmask >> q) & 1u)) continue;
          const unsigned len = sh.xlen[q];
          for (unsigned long long k = gtid; k < len; k += gsize) {
            const uint32_t v = lst[(size_t)q * a.wcnt + k];
            const uint32_t bit = 1u << (v & 31u);
            atomicOr(&frout[v >> 5], bit);
            atomicOr(&vnext[v >> 5], bit);
          }
        }
        // every list bit must be in place before the convert below reads the bitmap
        if (!level_barrier(false, a.bar, a.status, epoch, (unsigned)a.ncta)) return;
      }
      if (next == 0 && sh.lvl[5] != 0) {
        convert_phase<Off>(a, frout, nullptr, sel ? a.L1 : a.L0, sel ? a.H1 : a.H0, out, &sh.work);
        if (!level_barrier(a.narrow, a.bar, a.status, epoch, (unsigned)a.ncta)) return;
        read_level(out, sh);
        nL = (unsigned)sh.lvl[3];
        nH = (unsigned)sh.lvl[4];
        nB = (unsigned)sh.lvl[6];
      } else {
        from_bits = next == 0;
        if (!level_barrier(a.narrow, a.bar, a.status, epoch, (unsigned)a.ncta)) return;
      }
    } else if (dir == 1 && next == 0 && sh.lvl[5] == 0) {
      from_bits = true;  // every new frontier vertex is light: push straight from `fr`
    } else if (dir == 1 && next == 0) {
      // pull -> push with a high-degree vertex in the frontier: Dense2sparse into the
      // light list / heavy chunks so the hub's edges are split across warps
      uint32_t* vnew = cur ? a.vis1 : a.vis0;
      uint32_t* vold = cur ? a.vis0 : a.vis1;
      convert_phase<Off>(a, vnew, vold, sel ? a.L1 : a.L0, sel ? a.H1 : a.H0, out, &sh.work);
      if (!level_barrier(a.narrow, a.bar, a.status, epoch, (unsigned)a.ncta)) return;
      read_level(out, sh);
      nL = (unsigned)sh.lvl[3];
      nH = (unsigned)sh.lvl[4];
      nB = (unsigned)sh.lvl[6];
    }
    dir = next;
    c_old = c_new;
    mf_last = mf;
  }
  if ((a.narrow || a.stop_before > 0) && cta == 0 && threadIdx.x == 0) a.bar->rs.done = 1;
  if (cta == 0 && threadIdx.x == 0) {
    a.status->levels = d;
    a.status->reached = reached;
    a.status->reached_nnz = (D ? a.in_total : a.nnz) - m_u;  // in-degree mass of the reached
  }
  if (D && a.nranks > 1) {
    // no rank leaves while a peer may still read its own buffers for this BFS: a fast rank's
    // next BFS writes into the peers' exchange buffers
    if (!grid_barrier(a.bar, a.status, epoch, (unsigned)a.ncta)) return;
    if (cta == 0) rank_rendezvous(a, a.xseq + 0xFFFFFFFFull);
  }
  if (!D && PARENTS && a.perm) {  // relabelled graph: internal parents -> caller ids (after
    for (unsigned long long i = gtid; i < (unsigned long long)a.n; i += gsize) {  // last barrier)
      const uint32_t p = a.parent[i];
      a.pout[a.perm[i]] = p == 0xFFFFFFFFu ? p : a.perm[p];
    }
  }
}

// One GPU: the whole grid runs one BFS; the arguments are a kernel parameter.
template <typename Off, bool PARENTS, bool ABL>
__global__ void __launch_bounds__(kBfsBlock, 1) bfs_persistent(BfsArgs<Off> a) {
  bfs_body<Off, PARENTS, false, ABL>(a);
}

// Multi-rank: `all` holds one argument block per rank of this launch, rank r running on the
// CTAs [all[r].cta_base, all[r].cta_base + all[r].ncta).  One process per GPU launches with
// nranks = 1 (the whole grid); a single-device team launches its P ranks as P CTA groups of
// one cooperative launch, so every rank is co-resident and the cross-rank flags cannot
// deadlock.
template <typename Off, bool PARENTS>
__global__ void __launch_bounds__(kBfsBlock, 1) bfs_ranks(const BfsArgs<Off>* __restrict__ all,
                                                          int nranks) {
  __shared__ BfsArgs<Off> sa;
  if (threadIdx.x == 0) {
    int r = 0;
    while (r + 1 < nranks && (int)blockIdx.x >= all[r + 1].cta_base) ++r;
    sa = all[r];
  }
  __syncthreads();
  bfs_body<Off, PARENTS, true>(sa);
}



// Cooperative grid size per (device, kernel) (and the dynamic shared-memory attribute, which
// is per device too): computed once, guarded by a mutex.
static int coop_grid(const void* fn, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, fn});
  if (it != cache.end()) return it->second;
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kBfsBlock, smem);
  const int g = sms * (per > 0 ? per : 1);
  cache[{dev, fn}] = g;
  return g;
}

template <typename Off, bool PARENTS, bool ABL = false>
static int grid_for() {
  return coop_grid((const void*)bfs_persistent<Off, PARENTS, ABL>, dyn_smem_bytes<Off>());
}
// the default kernel (toggles compiled out) or the ablation kernel
template <typename Off, bool PARENTS>
static const void* bfs_kernel(bool abl) {
  return abl ? (const void*)bfs_persistent<Off, PARENTS, true>
             : (const void*)bfs_persistent<Off, PARENTS, false>;
}

int bfs_grid_size(pp_graph g, bool parents) {
  if (g->off64) return parents ? grid_for<uint64_t, true>() : grid_for<uint64_t, false>();
  return parents ? grid_for<uint32_t, true>() : grid_for<uint32_t, false>();
}

template <typename Off, bool PARENTS>
static cudaError_t launch_t(pp_graph g, BfsArgs<Off> args) {
  const bool abl = args.toggles != 0u;
  const int grid = abl ? grid_for<Off, PARENTS, true>() : grid_for<Off, PARENTS, false>();
  args.cta_base = 0;
  args.ncta = grid;
  void* params[] = {(void*)&args};
  g->ctx->launches += 1;
  return cudaLaunchCooperativeKernel(bfs_kernel<Off, PARENTS>(abl), dim3(grid),
                                     dim3(kBfsBlock), params, dyn_smem_bytes<Off>(),
                                     g->ctx->stream);
}

// Narrow launch: ONE thread-block cluster of kNarrowCtas CTAs runs init and the levels while
// they stay small, then hands the loop state to the cooperative whole-grid launch queued
// right behind it on the stream (which returns at once if the cluster finished the BFS).
template <typename Off, bool PARENTS>
static cudaError_t launch_narrow(pp_graph g, BfsArgs<Off> args) {
  args.cta_base = 0;
  args.ncta = kNarrowCtas;
  const bool abl = args.toggles != 0u;
  (void)(abl ? grid_for<Off, PARENTS, true>() : grid_for<Off, PARENTS, false>());  // smem attribute
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kNarrowCtas);
  cfg.blockDim = dim3(kBfsBlock);
  cfg.dynamicSmemBytes = dyn_smem_bytes<Off>();
  cfg.stream = g->ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kNarrowCtas;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  g->ctx->launches += 1;
  void* params[] = {(void*)&args};
  return cudaLaunchKernelExC(&cfg, bfs_kernel<Off, PARENTS>(abl), params);
}

// PP_NARROW unset or 0: never; 1: always (tests of the hand-over on any graph);
// 2: for graphs with max out-degree <= kNarrowMaxDeg.
static bool use_narrow(pp_graph g, int mode) {
  if (mode == 2) return false;
  // Measured slower than the whole grid on C4 and RGG24, so opt-in only.
  const char* e = getenv("PP_NARROW");
  if (e && e[0] == '1') return true;
  if (e && e[0] == '2') return g->max_out_deg <= kNarrowMaxDeg;
  return false;
}

template <typename Off>
static cudaError_t launch_off(pp_graph g, uint32_t source, int mode, int rule, double alpha,
                              double beta, uint32_t toggles, int32_t* depth, uint32_t* parent,
                              int max_levels, int split_level) {
  BfsArgs<Off> a;
  memset(&a, 0, sizeof(a));
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
  a.fr = g->fr;
  a.sumv = g->sumv;
  a.drec = g->drec;
  a.n_noniso = g->n_noniso;
  a.sum_shift = g->sum_shift;
  a.sum_words = g->sum_words;
  a.L0 = reinterpret_cast<uint4*>(g->L[0]);
  a.L1 = reinterpret_cast<uint4*>(g->L[1]);
  a.H0 = g->H[0];
  a.H1 = g->H[1];
  a.hcap = (unsigned)g->hcap;
  a.depth = depth;
  a.parent = (parent && g->perm) ? g->pint : parent;
  a.pout = parent;
  a.perm = g->perm;
  a.rank = g->rank;
  a.vrec = g->vrec;
  a.ctr = g->ctr;
  a.gwork = g->gwork;
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
  a.dbg = g->dbg;
  a.dbg_levels = g->dbg_levels;
  a.narrow = 0;
  a.resume = 0;
  if (use_narrow(g, mode)) {
    a.narrow = 1;
    const cudaError_t e = parent ? launch_narrow<Off, true>(g, a) : launch_narrow<Off, false>(g, a);
    if (e != cudaSuccess) return e;
    a.narrow = 0;
    a.resume = 1;
  }
  if (split_level > 0) {
    // debug split: levels 1 .. split_level-1 in one launch, then level split_level alone in a
    // second launch that resumes the handed-over loop state (its grid-barrier count restarts)
    a.stop_before = split_level;
    cudaError_t e = parent ? launch_t<Off, true>(g, a) : launch_t<Off, false>(g, a);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(&g->bar->count, 0, sizeof(g->bar->count), g->ctx->stream);
    if (e != cudaSuccess) return e;
    a.stop_before = 0;
    a.resume = 1;
    a.max_levels = split_level;
  }
  if (parent) return launch_t<Off, true>(g, a);
  return launch_t<Off, false>(g, a);
}

cudaError_t launch_bfs(pp_graph g, uint32_t source, int mode, int rule, double alpha, double beta,
                       uint32_t toggles, int32_t* depth, uint32_t* parent, int max_levels,
                       int split_level) {
  if (g->off64)
    return launch_off<uint64_t>(g, source, mode, rule, alpha, beta, toggles, depth, parent,
                                max_levels, split_level);
  return launch_off<uint32_t>(g, source, mode, rule, alpha, beta, toggles, depth, parent,
                              max_levels, split_level);
}

}  // namespace pp

namespace pp {

template <typename Off, bool PARENTS>
static cudaError_t launch_ranks_t(pp_graph* gs, int P, uint32_t source, int mode, int rule,
                                  double alpha, double beta, int32_t* const* depth,
                                  uint32_t* const* parent) {
  pp_graph g0 = gs[0];
  const void* fn = (const void*)bfs_ranks<Off, PARENTS>;
  const int grid = coop_grid(fn, dyn_smem_bytes<Off, true>());
  if (grid < P) return cudaErrorInvalidConfiguration;
  BfsArgs<Off> h[kMaxRanks];
  memset(h, 0, sizeof(h));
  for (int r = 0; r < P; ++r) {
    pp_graph g = gs[r];
    BfsArgs<Off>& a = h[r];
    a.n = g->n;
    a.nnz = g->nnz;
    a.nwords = g->nwords;
    a.off = (const Off*)g->off;
    a.idx = g->idx;
    a.coff = (const Off*)g->coff;
    a.cidx = g->cidx;
    a.symmetric = g->symmetric ? 1 : 0;
    a.drec = g->drec;
    a.n_noniso = g->n_noniso;  // all ranks' (dense-pull decision)
    a.isolated = g->isolated;
    a.vis0 = g->vis[0];
    a.vis1 = g->vis[1];
    a.fr = g->xfr[0];
    a.sumv = nullptr;
    a.sum_shift = 3;
    a.sum_words = 0;
    a.L0 = reinterpret_cast<uint4*>(g->L[0]);
    a.L1 = reinterpret_cast<uint4*>(g->L[1]);
    a.H0 = g->H[0];
    a.H1 = g->H[1];
    a.hcap = (unsigned)g->hcap;
    a.depth = depth[r];
    a.parent = parent ? parent[r] : nullptr;
    a.pout = a.parent;
    a.ctr = g->ctr;
    a.gwork = g->gwork;
    a.stats = g->stats;
    a.stats_cap = g->stats_cap;
    a.bar = g->bar;
    a.status = g->status;
    a.source = source;
    a.mode = mode;
    a.rule = rule;
    a.alpha = alpha;
    a.beta = beta;
    a.toggles = 0;
    a.max_levels = (int)std::min<int64_t>(g->n + 1, 0x7FFFFFFF);
    a.cta_base = (int)((int64_t)r * grid / P);
    a.ncta = (int)((int64_t)(r + 1) * grid / P) - a.cta_base;
    a.lo = g->row_lo;
    a.hi = g->row_hi;
    a.wlo = (uint32_t)(g->me * g->chunk_words);
    a.wcnt = (uint32_t)g->chunk_words;
    a.me = g->me;
    a.nranks = g->nranks;
    a.xfr0 = g->xfr[0];
    a.xfr1 = g->xfr[1];
    a.xcnt = g->xcnt;
    a.xflag = g->xflag;
    a.xlst0 = g->xlst[0];
    a.xlst1 = g->xlst[1];
    a.xown = g->xown;
    for (int q = 0; q < kMaxRanks; ++q) {
      a.pfr[q][0] = g->pfr[q][0];
      a.pfr[q][1] = g->pfr[q][1];
      a.pcnt[q] = g->pcnt[q];
      a.plst[q][0] = g->plst[q][0];
      a.plst[q][1] = g->plst[q][1];
      a.pflag[q] = g->pflag[q];
    }
    g->xseq += 1;  // identical on every rank: pp_bfs is collective
    a.xseq = g->xseq << 32;
    a.odeg = g->odeg;
    a.in_total = g->in_total;
  }
  cudaStream_t st = g0->ctx->stream;
  // pageable source: the runtime stages it before returning, so `h` may go out of scope
  cudaError_t e = cudaMemcpyAsync(g0->dargs, h, sizeof(BfsArgs<Off>) * P, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  const BfsArgs<Off>* dall = (const BfsArgs<Off>*)g0->dargs;
  void* params[] = {(void*)&dall, (void*)&P};
  g0->ctx->launches += 1;
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBfsBlock), params, dyn_smem_bytes<Off, true>(), st);
}

cudaError_t launch_bfs_ranks(pp_graph* graphs, int nranks, uint32_t source, int mode, int rule,
                             double alpha, double beta, int32_t* const* depth,
                             uint32_t* const* parent) {
  if (graphs[0]->off64)
    return parent ? launch_ranks_t<uint64_t, true>(graphs, nranks, source, mode, rule, alpha, beta, depth, parent)
                  : launch_ranks_t<uint64_t, false>(graphs, nranks, source, mode, rule, alpha, beta, depth, parent);
  return parent ? launch_ranks_t<uint32_t, true>(graphs, nranks, source, mode, rule, alpha, beta, depth, parent)
                : launch_ranks_t<uint32_t, false>(graphs, nranks, source, mode, rule, alpha, beta, depth, parent);
}

size_t bfs_args_bytes() { return sizeof(BfsArgs<uint64_t>) * kMaxRanks; }

}  // namespace pp
