// sssp.cu — SURVEY NEXT-4: the paper's generality claim (Sec. 5.6): SSSP as
// Bellman-Ford over the min-plus semiring through the same push / pull matvec shapes, with
// the "simple 2-phase direction-optimized traversal": unmasked column-based (push) mxv
// while the active set is small, ONE switch to row-based (pull) mxv once nnz(f)/n > alpha.
// No mask and no early exit (Boolean-only); operand reuse in the pull: the
// row reads all of d instead of f.  Jacobi iteration (R28):
//   t = d_k;  t(j) = min(t(j), d_k(i) + A(i,j)) over the step's edges;  f_{k+1} = {t < d_k};
//   d_{k+1} = t.
// Distances and non-negative weights are fp32 (R30); non-negative floats order like their
// int32 bit patterns, so the push's min-reduction is a plain atomicMin on the bits.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <map>
#include <mutex>

#include "pp_device.cuh"

namespace {

using namespace pp;

constexpr int kT = 256;                 // threads per CTA (prologue kernels)
constexpr int kLoopT = 1024;            // threads per CTA of the persistent loop
constexpr unsigned kInfBits = 0x7f800000u;

__global__ void k_sssp_init(int64_t n, int64_t s, float* __restrict__ d, float* __restrict__ t,
                            uint32_t* __restrict__ list, unsigned* __restrict__ cnt) {
  const float inf = __int_as_float(kInfBits);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = i == s ? 0.f : inf;
    d[i] = v;
    t[i] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    list[0] = (uint32_t)s;
    cnt[0] = 0;  // next-frontier length
    cnt[1] = 0;  // error flag (negative / NaN weight)
    cnt[2] = 0;  // heavy active vertices of the step (push)
    cnt[3] = 0;  // heavy rows of A^T (pull), counted once
    cnt[4] = 0;  // their chunk descriptors
  }
}

// negative weights are rejected (NaN fails w >= 0 too).
__global__ void k_sssp_check(int64_t nnz, const float* __restrict__ w, unsigned* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    if (!(w[e] >= 0.f)) cnt[1] = 1;
}

#ifndef PP_SSSP_G
#define PP_SSSP_G 4
#endif
constexpr int kG = PP_SSSP_G;           // lanes per light vertex / row (32/kG groups per warp)
#ifndef PP_SSSP_HEAVY
#define PP_SSSP_HEAVY 256
#endif
constexpr int64_t kHeavyDeg = PP_SSSP_HEAVY;  // longer rows / out-lists: kChunk-edge warp chunks

__device__ __forceinline__ unsigned group_mask() {
  return ((1u << kG) - 1u) << ((threadIdx.x & 31) & ~(kG - 1));
}

// t(v) <- min(t(v), nd); the thread whose atomicMin moves t(v) off d(v) appends v.
__device__ __forceinline__ void relax(uint32_t v, float nd, const float* __restrict__ d, float* t,
                                      uint32_t* __restrict__ next, unsigned* __restrict__ cnt) {
  if (nd < t[v]) {
    const int old = atomicMin(reinterpret_cast<int*>(t) + v, __float_as_int(nd));
    if (__float_as_int(nd) < old && old == __float_as_int(d[v])) next[atomicAdd(cnt, 1u)] = v;
  }
}

constexpr int64_t kChunk = 2048;        // heavy rows / out-lists are cut into chunks of this
                                        // many edges, one warp each (no serial hub tail)

// The iteration loop runs in ONE persistent cooperative kernel (k_sssp_loop): the phases
// below are grid-stride device functions separated by a software grid barrier, the frontier
// size is read on the device after each barrier and the push -> pull switch (R29) is decided
// on the device, so a whole SSSP is one launch after the prologue with no host round trip per
// iteration (as bfs_persistent does for BFS).

// Column-based step (push, Alg. 3 shape P:370): a kG-lane group per active vertex u scatters
// d(u) + A(u, v) into t(v); a vertex with more than kHeavyDeg out-edges is cut into kChunk-edge
// chunk descriptors {u, chunk} for push_heavy.
__device__ void push_light(const uint32_t* __restrict__ f, unsigned nf, const int64_t* __restrict__ off,
                           const uint32_t* __restrict__ idx, const float* __restrict__ w,
                           const float* __restrict__ d, float* __restrict__ t,
                           uint32_t* __restrict__ next, unsigned* __restrict__ ncnt,
                           uint2* __restrict__ chunks, unsigned* __restrict__ ccnt) {
  const unsigned lane = threadIdx.x & (kG - 1);
  const unsigned gpb = blockDim.x / kG;
  for (unsigned k = blockIdx.x * gpb + threadIdx.x / kG; k < nf; k += gridDim.x * gpb) {
    const uint32_t u = f[k];
    const int64_t b = off[u], e = off[u + 1];
    if (e - b > kHeavyDeg) {
      const unsigned nch = (unsigned)((e - b + kChunk - 1) / kChunk);
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(ccnt, nch);
      base = __shfl_sync(group_mask(), base, 0, kG);
      for (unsigned c = lane; c < nch; c += kG) chunks[base + c] = make_uint2(u, c);
      continue;
    }
    const float du = d[u];
    for (int64_t j = b + lane; j < e; j += kG) relax(__ldg(idx + j), du + __ldg(w + j), d, t, next, ncnt);
  }
}

// Heavy out-lists of this step: one warp per kChunk-edge chunk.
__device__ void push_heavy(const uint2* __restrict__ chunks, unsigned nc, const int64_t* __restrict__ off,
                           const uint32_t* __restrict__ idx, const float* __restrict__ w,
                           const float* __restrict__ d, float* __restrict__ t,
                           uint32_t* __restrict__ next, unsigned* __restrict__ ncnt) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned nw = gridDim.x * (blockDim.x >> 5);
  for (unsigned k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < nc; k += nw) {
    const uint2 c = chunks[k];
    const float du = d[c.x];
    const int64_t b = off[c.x] + (int64_t)c.y * kChunk;
    const int64_t e = min(off[c.x + 1], b + kChunk);
    for (int64_t j = b + lane; j < e; j += 32) relax(__ldg(idx + j), du + __ldg(w + j), d, t, next, ncnt);
  }
}

// Row-based step (pull, Alg. 2 shape P:320 without mask / early exit): a kG-lane group per
// row j of A^T reduces min_i d(i) + A(i, j) over the in-edges (operand reuse: all of d).
// Rows longer than kHeavyDeg are left to pull_heavy / pull_finish.
__device__ void pull_light(int64_t n, const int64_t* __restrict__ coff, const uint32_t* __restrict__ cidx,
                           const float* __restrict__ cw, const float* __restrict__ d,
                           float* __restrict__ t, uint32_t* __restrict__ next, unsigned* __restrict__ ncnt) {
  const unsigned lane = threadIdx.x & (kG - 1);
  const unsigned gm = group_mask();
  const int64_t gpb = blockDim.x / kG;
  for (int64_t j = blockIdx.x * gpb + threadIdx.x / kG; j < n; j += (int64_t)gridDim.x * gpb) {
    const int64_t b = coff[j], e = coff[j + 1];
    if (e - b > kHeavyDeg) continue;
    float m = __int_as_float(kInfBits);
    for (int64_t q = b + lane; q < e; q += kG) m = fminf(m, d[__ldg(cidx + q)] + __ldg(cw + q));
#pragma unroll
    for (int o = kG / 2; o; o >>= 1) m = fminf(m, __shfl_xor_sync(gm, m, o));
    if (lane == 0 && m < d[j]) {
      t[j] = m;
      next[atomicAdd(ncnt, 1u)] = (uint32_t)j;
    }
  }
}

// Heavy rows: one warp per kChunk-edge chunk (descriptors built once per call), partial min
// folded into cand(j) with atomicMin on the fp32 bits.
__device__ void pull_heavy(const uint2* __restrict__ chunks, unsigned nc,
                           const int64_t* __restrict__ coff, const uint32_t* __restrict__ cidx,
                           const float* __restrict__ cw, const float* __restrict__ d,
                           float* __restrict__ cand) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned nw = gridDim.x * (blockDim.x >> 5);
  for (unsigned k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < nc; k += nw) {
    const uint2 c = chunks[k];
    const int64_t b = coff[c.x] + (int64_t)c.y * kChunk;
    const int64_t e = min(coff[c.x + 1], b + kChunk);
    float m = __int_as_float(kInfBits);
    int64_t q = b + lane;
    for (; q + 96 < e; q += 128) {  // 4 independent gathers in flight per lane
      uint32_t i0 = __ldg(cidx + q), i1 = __ldg(cidx + q + 32), i2 = __ldg(cidx + q + 64),
               i3 = __ldg(cidx + q + 96);
      float w0 = __ldg(cw + q), w1 = __ldg(cw + q + 32), w2 = __ldg(cw + q + 64), w3 = __ldg(cw + q + 96);
      m = fminf(fminf(m, fminf(d[i0] + w0, d[i1] + w1)), fminf(d[i2] + w2, d[i3] + w3));
    }
    for (; q < e; q += 32) m = fminf(m, d[__ldg(cidx + q)] + __ldg(cw + q));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0 && m < cand[c.x]) atomicMin(reinterpret_cast<int*>(cand) + c.x, __float_as_int(m));
  }
}

// Heavy rows: t(j) = cand(j) where it improves d(j); cand reset to +inf for the next step.
__device__ void pull_finish(const uint32_t* __restrict__ hrows, unsigned nh, const float* __restrict__ d,
                            float* __restrict__ t, float* __restrict__ cand,
                            uint32_t* __restrict__ next, unsigned* __restrict__ ncnt) {
  for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < nh; k += gridDim.x * blockDim.x) {
    const uint32_t j = hrows[k];
    const float m = cand[j];
    cand[j] = __int_as_float(kInfBits);
    if (m < d[j]) {
      t[j] = m;
      next[atomicAdd(ncnt, 1u)] = j;
    }
  }
}

// Once per call: list the heavy rows of A^T and cut them into chunk descriptors.
__global__ void k_sssp_heavy_rows(int64_t n, const int64_t* __restrict__ coff, uint32_t* __restrict__ hrows,
                                  uint2* __restrict__ chunks, float* __restrict__ cand,
                                  unsigned* __restrict__ cnt) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    cand[j] = __int_as_float(kInfBits);
    const int64_t deg = coff[j + 1] - coff[j];
    if (deg > kHeavyDeg) {
      hrows[atomicAdd(cnt + 3, 1u)] = (uint32_t)j;
      const unsigned nch = (unsigned)((deg + kChunk - 1) / kChunk);
      const unsigned base = atomicAdd(cnt + 4, nch);
      for (unsigned c = 0; c < nch; ++c) chunks[base + c] = make_uint2((uint32_t)j, c);
    }
  }
}

// Device control block of the persistent loop (in the workspace, zeroed before the launch).
struct SsspCtl {
  unsigned long long bar;        // grid barrier: monotone arrivals, bit 63 = abort (watchdog)
  unsigned pad[30];
  unsigned cnt[3][4];            // per iteration mod 3: [0] next-frontier length, [1] push chunks
  long long it, push_it, pull_it, sw;  // stats, written by block 0 at the end
  int error;                     // PP_ERR_TIMEOUT if a barrier wait timed out
};

constexpr unsigned long long kSsspAbort = 1ull << 63;
constexpr unsigned long long kSsspWatchdogNs = 4000000000ull;

__device__ __forceinline__ bool sssp_barrier(SsspCtl* c, unsigned& epoch) {
  __shared__ int s_ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned long long target = (unsigned long long)epoch * gridDim.x;
    // acq_rel arrival (the last arriver acquires too), acquire polling, no trailing fence:
    // the same protocol as bfs.cu's grid barrier
    unsigned long long v;
    asm volatile("atom.add.acq_rel.gpu.u64 %0, [%1], 1;" : "=l"(v) : "l"(&c->bar) : "memory");
    v += 1ull;
    if (v < target) {
      const unsigned long long t0 = global_timer_ns();
      while ((v = ld_acquire_u64(&c->bar)) < target) {
        __nanosleep(32);
        if (global_timer_ns() - t0 > kSsspWatchdogNs) {
          atomicExch(&c->error, (int)PP_ERR_TIMEOUT);
          atomicOr(&c->bar, kSsspAbort);
          v = kSsspAbort;
          break;
        }
      }
    }
    s_ok = (v & kSsspAbort) ? 0 : 1;
  }
  __syncthreads();
  return s_ok != 0;
}

struct SsspArgs {
  int64_t n;
  double alpha;
  const int64_t *off, *coff;
  const uint32_t *idx, *cidx;
  const float *w, *cw;
  float *d, *t, *cand;
  uint32_t *la, *lb, *hrows;
  uint2 *pch, *hch;
  const unsigned* flags;  // prologue counters: [1] bad weight, [3] heavy rows, [4] their chunks
  SsspCtl* ctl;
};

// The whole 2-phase traversal in one cooperative launch: per iteration the step's
// phase(s), a grid barrier, the commit d = t on the changed list, a grid barrier; the next
// frontier's length decides termination and the single push -> pull switch identically in
// every CTA (R28, R29).
__global__ void __launch_bounds__(kLoopT, 2) k_sssp_loop(SsspArgs a) {
  SsspCtl* c = a.ctl;
  if (a.flags[1]) return;  // a negative or NaN weight: the host reports PP_ERR_GRAPH
  const unsigned nh = a.flags[3], nhc = a.flags[4];
  unsigned epoch = 0;
  long long it = 0, push_it = 0, pull_it = 0, sw = -1;
  int dir = 0;
  unsigned nf = 1;
  uint32_t *f = a.la, *nx = a.lb;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x, gsize = gridDim.x * blockDim.x;
  while (nf > 0) {
    if (dir == 0 && (double)nf / (double)a.n > a.alpha) {  // the one switch (R29)
      dir = 1;
      sw = it;
    }
    unsigned* cc = c->cnt[it % 3];
    // the counters of iteration it+1 were last read in iteration it-2: two barriers ago
    if (blockIdx.x == 0 && threadIdx.x < 4) c->cnt[(it + 1) % 3][threadIdx.x] = 0u;
    if (dir == 0) {
      push_light(f, nf, a.off, a.idx, a.w, a.d, a.t, nx, &cc[0], a.pch, &cc[1]);
      if (!sssp_barrier(c, epoch)) return;
      push_heavy(a.pch, ld_relaxed_u32(&cc[1]), a.off, a.idx, a.w, a.d, a.t, nx, &cc[0]);
      ++push_it;
    } else {
      pull_light(a.n, a.coff, a.cidx, a.cw, a.d, a.t, nx, &cc[0]);
      if (nhc) pull_heavy(a.hch, nhc, a.coff, a.cidx, a.cw, a.d, a.cand);
      if (!sssp_barrier(c, epoch)) return;
      if (nh) pull_finish(a.hrows, nh, a.d, a.t, a.cand, nx, &cc[0]);
      ++pull_it;
    }
    if (!sssp_barrier(c, epoch)) return;
    const unsigned nn = ld_relaxed_u32(&cc[0]);
    for (unsigned k = gtid; k < nn; k += gsize) {  // d_{k+1} = t on the changed set
      const uint32_t v = nx[k];
      a.d[v] = a.t[v];
    }
    if (!sssp_barrier(c, epoch)) return;
    nf = nn;
    uint32_t* tmp = f;
    f = nx;
    nx = tmp;
    ++it;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c->it = it;
    c->push_it = push_it;
    c->pull_it = pull_it;
    c->sw = sw;
  }
}

unsigned grid_for(int64_t work, int per_block, int cap) {
  int64_t g = (work + per_block - 1) / per_block;
  return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

using namespace pp;

#define SS_CK(call, what)                                        \
  do {                                                           \
    cudaError_t _e = (call);                                     \
    if (_e != cudaSuccess) { st = cuda_fail(_e, what); goto out; } \
  } while (0)

extern "C" pp_status pp_sssp(pp_ctx ctx, int64_t n, int64_t nnz, const int64_t* csr_off,
                             const uint32_t* csr_idx, const float* csr_w, const int64_t* csc_off,
                             const uint32_t* csc_idx, const float* csc_w, int64_t source,
                             double alpha, float* dist, pp_sssp_stats* stats) {
  if (!ctx || !csr_off || !csc_off || !dist || (nnz > 0 && (!csr_idx || !csr_w || !csc_idx || !csc_w))) {
    set_error("pp_sssp: NULL argument");
    return PP_ERR_ARG;
  }
  if (n <= 0 || nnz < 0 || n >= (int64_t)UINT32_MAX) {
    set_error("pp_sssp: n=%lld nnz=%lld invalid", (long long)n, (long long)nnz);
    return PP_ERR_ARG;
  }
  if (source < 0 || source >= n) {
    set_error("pp_sssp: source %lld out of range [0, %lld)", (long long)source, (long long)n);
    return PP_ERR_RANGE;
  }
  if (!(alpha >= 0.0)) {
    set_error("pp_sssp: alpha must be >= 0");
    return PP_ERR_ARG;
  }
  pp_status st = PP_OK;
  cudaStream_t s = ctx->stream;
  const int cap = ctx->num_sms * 8;
  float* t = nullptr;
  uint32_t *la = nullptr, *lb = nullptr;
  uint32_t* hrows = nullptr;
  uint2 *pch = nullptr, *hch = nullptr;  // push / pull chunk descriptors
  float* cand = nullptr;
  const int64_t nch_max = nnz / kHeavyDeg + 1;  // ceil(deg/kChunk) <= deg/kHeavyDeg for heavy rows
  unsigned* cnt = nullptr;
  SsspCtl* ctl = nullptr;
  unsigned h[5] = {0, 0, 0, 0, 0};
  SsspCtl hc;
  SS_CK(cudaSetDevice(ctx->device), "pp_sssp: cudaSetDevice");
  {  // structural check of the caller's arrays: off[0] = 0 and off[n] = nnz on both sides
    int64_t ends[4] = {-1, -1, -1, -1};
    SS_CK(cudaMemcpyAsync(&ends[0], csr_off, 8, cudaMemcpyDeviceToHost, s), "pp_sssp: read csr_off[0]");
    SS_CK(cudaMemcpyAsync(&ends[1], csr_off + n, 8, cudaMemcpyDeviceToHost, s), "pp_sssp: read csr_off[n]");
    SS_CK(cudaMemcpyAsync(&ends[2], csc_off, 8, cudaMemcpyDeviceToHost, s), "pp_sssp: read csc_off[0]");
    SS_CK(cudaMemcpyAsync(&ends[3], csc_off + n, 8, cudaMemcpyDeviceToHost, s), "pp_sssp: read csc_off[n]");
    SS_CK(cudaStreamSynchronize(s), "pp_sssp: read offsets");
    if (ends[0] != 0 || ends[1] != nnz || ends[2] != 0 || ends[3] != nnz) {
      set_error("pp_sssp: offsets off[0]=%lld off[n]=%lld coff[0]=%lld coff[n]=%lld, expected 0 and "
                "nnz=%lld", (long long)ends[0], (long long)ends[1], (long long)ends[2],
                (long long)ends[3], (long long)nnz);
      st = PP_ERR_GRAPH;
      goto out;
    }
  }
  {  // workspace cached in the context (grown on demand, freed by pp_ctx_destroy): no
     // per-call allocation and no change to any process-wide allocator state
    const size_t need = sizeof(float) * n * 2 + sizeof(uint32_t) * n * 3 +
                        sizeof(uint2) * (size_t)nch_max * 2 + 256 * 9 + sizeof(SsspCtl) + 256;
    if (ctx->sssp_ws_bytes < need) {
      if (ctx->sssp_ws) cudaFree(ctx->sssp_ws);
      ctx->sssp_ws = nullptr;
      ctx->sssp_ws_bytes = 0;
      SS_CK(cudaMalloc(&ctx->sssp_ws, need), "pp_sssp: workspace");
      ctx->sssp_ws_bytes = need;
    }
    char* p = static_cast<char*>(ctx->sssp_ws);
    auto carve = [&](size_t bytes) {
      char* r = p;
      p += (bytes + 255) & ~(size_t)255;
      return (void*)r;
    };
    t = (float*)carve(sizeof(float) * n);
    cand = (float*)carve(sizeof(float) * n);
    la = (uint32_t*)carve(sizeof(uint32_t) * n);
    lb = (uint32_t*)carve(sizeof(uint32_t) * n);
    hrows = (uint32_t*)carve(sizeof(uint32_t) * n);
    pch = (uint2*)carve(sizeof(uint2) * nch_max);
    hch = (uint2*)carve(sizeof(uint2) * nch_max);
    cnt = (unsigned*)carve(sizeof(unsigned) * 8);
    ctl = (SsspCtl*)carve(sizeof(SsspCtl));
  }
  k_sssp_init<<<grid_for(n, kT, cap), kT, 0, s>>>(n, source, dist, t, la, cnt);
  ctx->launches++;
  if (nnz > 0) {
    k_sssp_check<<<grid_for(nnz, kT, cap), kT, 0, s>>>(nnz, csr_w, cnt);
    k_sssp_check<<<grid_for(nnz, kT, cap), kT, 0, s>>>(nnz, csc_w, cnt);
    ctx->launches += 2;
  }
  k_sssp_heavy_rows<<<grid_for(n, kT, cap), kT, 0, s>>>(n, csc_off, hrows, hch, cand, cnt);
  ctx->launches++;
  SS_CK(cudaMemsetAsync(ctl, 0, sizeof(SsspCtl), s), "pp_sssp: reset control block");
  {  // the iteration loop: one persistent cooperative launch, then one synchronisation
    static std::mutex mu;
    static std::map<int, int> grid_cache;  // per device: co-resident CTAs of k_sssp_loop
    int grid = 0;
    {
      std::lock_guard<std::mutex> lock(mu);
      auto itg = grid_cache.find(ctx->device);
      if (itg == grid_cache.end()) {
        int per = 0;
        SS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sssp_loop, kLoopT, 0),
              "pp_sssp: occupancy");
        grid_cache[ctx->device] = ctx->num_sms * (per > 0 ? per : 1);
      }
      grid = grid_cache[ctx->device];
    }
    SsspArgs args{n, alpha, csr_off, csc_off, csr_idx, csc_idx, csr_w, csc_w, dist, t, cand,
                  la, lb, hrows, pch, hch, cnt, ctl};
    void* params[] = {(void*)&args};
    SS_CK(cudaLaunchCooperativeKernel((const void*)k_sssp_loop, dim3(grid), dim3(kLoopT), params, 0, s),
          "pp_sssp: persistent loop");
    ctx->launches++;
  }
  SS_CK(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s), "pp_sssp: read flags");
  SS_CK(cudaMemcpyAsync(&hc, ctl, sizeof(SsspCtl), cudaMemcpyDeviceToHost, s), "pp_sssp: read stats");
  SS_CK(cudaStreamSynchronize(s), "pp_sssp: run");
  if (h[1]) {
    set_error("pp_sssp: negative or NaN edge weight (SPEC S:342)");
    st = PP_ERR_GRAPH;
    goto out;
  }
  if (hc.error) {
    set_error("pp_sssp: a grid barrier timed out (watchdog)");
    st = (pp_status)hc.error;
    goto out;
  }
  if (stats) {
    stats->iterations = hc.it;
    stats->push_iterations = hc.push_it;
    stats->pull_iterations = hc.pull_it;
    stats->switch_iteration = hc.sw;
  }
out:
  return st;
}
