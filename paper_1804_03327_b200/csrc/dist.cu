// dist.cu — multi-GPU direction-optimised BFS over a 1D row partition (
// the paper names distributed GPUs as future work).
//
// One process per GPU.  Rank p owns the vertex block [lo_p, hi_p) (boundaries aligned to
// 1024 vertices = 32 bitmap words).  Every rank keeps the whole graph resident (s26 is
// ~9 GB, far inside 180 GB) and, for push, the sub-range of every row's sorted ids that
// falls inside its block, so a push expands the *global* frontier but discovers only owned
// vertices (no all-to-all).  Pull scans owned unvisited rows against the replicated
// visited bitmap.  Each level ends with one in-place ncclAllGather of the owned slices of
// the next-frontier bitmap over NVLink/NVSwitch; a finish kernel then ORs it into the
// replicated visited bitmap and counts c, m_f, m_fin, so every rank takes the identical
// push/pull decision (R10/R11) with no further communication.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>

#include "pp_device.cuh"

namespace pp {

// ---------------------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

static NcclApi g_nccl;

// libnccl.so.2 is resolved at run time (torch.distributed has usually loaded it already),
// so libpushpull.so loads and serves single-GPU calls on systems without NCCL.
bool nccl_load(const char** why) {
  if (g_nccl.loaded) return true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* nm : names)
    if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
  if (!h) {
    *why = "libnccl.so.2 not found (load torch.distributed first or set LD_LIBRARY_PATH)";
    return false;
  }
  g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.allGather = (decltype(g_nccl.allGather))dlsym(h, "ncclAllGather");
  g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.getErrorString = (decltype(g_nccl.getErrorString))dlsym(h, "ncclGetErrorString");
  if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.allGather || !g_nccl.commDestroy ||
      !g_nccl.getErrorString) {
    *why = "libnccl.so.2 lacks a required symbol";
    return false;
  }
  g_nccl.loaded = true;
  return true;
}

int nccl_unique_id(void* out128, const char** why) {
  if (!nccl_load(why)) return -1;
  ncclUniqueId id;
  ncclResult_t r = g_nccl.getUniqueId(&id);
  if (r != ncclSuccess) {
    *why = g_nccl.getErrorString(r);
    return -1;
  }
  memcpy(out128, &id, sizeof(id));
  return 0;
}

int nccl_comm_init(void** comm, int nranks, const void* id128, int rank, const char** why) {
  if (!nccl_load(why)) return -1;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  ncclResult_t r = g_nccl.commInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) {
    *why = g_nccl.getErrorString(r);
    return -1;
  }
  *comm = c;
  return 0;
}

void nccl_comm_destroy(void* comm) {
  if (comm && g_nccl.loaded) g_nccl.commDestroy((ncclComm_t)comm);
}

// 1D partition: rank p owns words [p*cw, min((p+1)*cw, W)) with cw = ceil(W/32/P)*32,
// W = ceil(n/32) rounded up to 32 words; vertices = words*32 clipped to n.
void partition(int64_t n, int rank, int nranks, int64_t* lo, int64_t* hi, int64_t* chunk_words) {
  const int64_t W = ((n + 31) / 32 + 31) / 32 * 32;
  const int64_t cw = ((W / 32 + nranks - 1) / nranks) * 32;
  int64_t l = (int64_t)rank * cw * 32, h = (int64_t)(rank + 1) * cw * 32;
  if (l > n) l = n;
  if (h > n) h = n;
  *lo = l;
  *hi = h;
  *chunk_words = cw;
}

// ---------------------------------------------------------------------------- kernels ----

// Push ranges: positions [pb[u], pe[u]) of row u's sorted ids that lie in [lo, hi).
template <typename Off>
__global__ void k_push_ranges(const Off* __restrict__ off, const uint32_t* __restrict__ idx,
                              int64_t n, uint32_t lo, uint32_t hi, Off* __restrict__ pb,
                              Off* __restrict__ pe) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    Off b = off[u], e = off[u + 1];
    Off l = b, r = e;  // first id >= lo
    while (l < r) {
      const Off m = l + (r - l) / 2;
      if (idx[m] < lo) l = m + 1;
      else r = m;
    }
    const Off s = l;
    r = e;  // first id >= hi
    while (l < r) {
      const Off m = l + (r - l) / 2;
      if (idx[m] < hi) l = m + 1;
      else r = m;
    }
    pb[u] = s;
    pe[u] = l;
  }
}

// Init: visited = {s}, frontier = {s}, next = {}; owned depth/parent slices.
__global__ void k_dist_init(uint32_t* vis, uint32_t* fr, uint32_t* nxt, int64_t W, uint32_t s,
                            int32_t* depth, uint32_t* parent, int64_t lo, int64_t hi) {
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = t0; w < W; w += gs) {
    const uint32_t b = (w == (int64_t)(s >> 5)) ? (1u << (s & 31u)) : 0u;
    vis[w] = b;
    fr[w] = b;
    nxt[w] = 0u;
  }
  for (int64_t v = lo + t0; v < hi; v += gs) {
    depth[v - lo] = (v == (int64_t)s) ? 1 : 0;
    if (parent) parent[v - lo] = (v == (int64_t)s) ? s : 0xFFFFFFFFu;
  }
}

// Push level: every frontier vertex u (global bitmap `fr`), edges into the owned block only.
// Warp per frontier word; each frontier vertex's owned range is walked by its lane, or by
// the whole warp when longer than 32.
template <typename Off, bool PARENTS>
__global__ void __launch_bounds__(kBlock) k_dist_push(
    const uint32_t* __restrict__ fr, uint32_t* vis, uint32_t* nxt, int64_t W,
    const Off* __restrict__ pb, const Off* __restrict__ pe, const uint32_t* __restrict__ idx,
    int64_t lo, int32_t* depth, uint32_t* parent, int newdepth) {
  const unsigned lane = lane_id();
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  for (int64_t w = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); w < W; w += nw) {
    const uint32_t word = fr[w];
    if (!word) continue;
    auto visit = [&](uint32_t u, uint32_t x) {
      const uint32_t wi = x >> 5, bit = 1u << (x & 31u);
      const uint32_t cur = vis[wi];
      bool disc = false;
      if (!(cur & bit)) disc = !(atomicOr(&vis[wi], bit) & bit);
      if (disc) {
        depth[x - lo] = newdepth;
        atomicOr(&nxt[wi], bit);
      }
      if (PARENTS) {
        bool fresh = disc || !(cur & bit);
        if (!fresh) {
          const int dx = ld_relaxed_s32(&depth[x - lo]);
          fresh = dx == 0 || dx == newdepth;
        }
        if (fresh) atomicMin(&parent[x - lo], u);
      }
    };
    // lanes take the word's vertices; short owned ranges lane-serial, long ones by the warp
    const bool mine = (word >> lane) & 1u;
    const uint32_t u = (uint32_t)w * 32u + lane;
    Off b = 0, e = 0;
    if (mine) {
      b = pb[u];
      e = pe[u];
    }
    const bool longr = mine && (e - b) > (Off)32;
    if (mine && !longr)
      for (Off p = b; p < e; ++p) visit(u, idx[p]);
    unsigned lm = __ballot_sync(kFull, longr);
    while (lm) {
      const unsigned l = __ffs(lm) - 1;
      lm &= lm - 1;
      const Off lb = __shfl_sync(kFull, b, l), le = __shfl_sync(kFull, e, l);
      const uint32_t lu = (uint32_t)w * 32u + l;
      for (Off p = lb + lane; p < le; p += 32) visit(lu, idx[p]);
    }
  }
}

// Pull level: owned unvisited non-isolated rows scan their in-neighbours (global ids) against
// the replicated visited snapshot; first hit in sorted order = parent (early exit).
template <typename Off, bool PARENTS>
__global__ void __launch_bounds__(kBlock) k_dist_pull(
    const uint32_t* __restrict__ vis, const uint32_t* __restrict__ iso, uint32_t* nxt,
    int64_t w_lo, int64_t w_hi, const Off* __restrict__ coff, const uint32_t* __restrict__ cidx,
    int64_t lo, int64_t n, int32_t* depth, uint32_t* parent, int newdepth) {
  const unsigned lane = lane_id();
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  for (int64_t w = w_lo + (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); w < w_hi; w += nw) {
    uint32_t cand = ~vis[w] & ~iso[w];
    uint32_t found = 0;
    while (cand) {  // one candidate per lane per round
      const unsigned cnt = __popc(cand);
      const bool act = lane < cnt;
      const unsigned bit = act ? __fns(cand, 0, (int)lane + 1) : 0u;
      const int64_t i = (int64_t)w * 32 + bit;
      bool f = false;
      uint32_t par = 0;
      if (act && i < n) {
        const Off b = coff[i], e = coff[i + 1];
        for (Off p = b; p < e; ++p) {
          const uint32_t x = cidx[p];
          if (bit_test(vis, x)) {
            f = true;
            par = x;
            break;
          }
        }
      }
      if (f) {
        depth[i - lo] = newdepth;
        if (PARENTS) parent[i - lo] = par;
      }
      found |= __reduce_or_sync(kFull, f ? (1u << bit) : 0u);
      // drop the (up to 32) candidates handled this round
      uint32_t handled = 0, c2 = cand;
      for (unsigned k = 0; k < 32 && c2; ++k) {
        handled |= c2 & (0u - c2);
        c2 &= c2 - 1;
      }
      cand &= ~handled;
    }
    if (lane == 0 && found) nxt[w] = found;
  }
}

// Finish: vis |= nxt; fr = nxt; nxt = 0; counters c, m_f (out-degree), m_fin (in-degree).
template <typename Off>
__global__ void __launch_bounds__(kBlock) k_dist_finish(
    uint32_t* vis, uint32_t* fr, uint32_t* nxt, int64_t W, const Off* __restrict__ off,
    const Off* __restrict__ coff, unsigned long long* cnt) {
  unsigned long long c = 0, mf = 0, mfin = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = nxt[w];
    fr[w] = x;
    if (x) {
      vis[w] |= x;
      nxt[w] = 0u;
      c += __popc(x);
      while (x) {
        const int64_t v = w * 32 + (__ffs(x) - 1);
        x &= x - 1;
        mf += (unsigned long long)(off[v + 1] - off[v]);
        mfin += (unsigned long long)(coff[v + 1] - coff[v]);
      }
    }
  }
  c = warp_sum(c);
  mf = warp_sum(mf);
  mfin = warp_sum(mfin);
  if (lane_id() == 0 && c) {
    atomicAdd(&cnt[0], c);
    atomicAdd(&cnt[1], mf);
    atomicAdd(&cnt[2], mfin);
  }
}

// ---------------------------------------------------------------------------- host -------

template <typename Off>
static cudaError_t ranges_t(pp_graph g) {
  const int blocks = g->ctx->num_sms * 8;
  g->ctx->launches += 1;
  k_push_ranges<Off><<<blocks, kBlock, 0, g->ctx->stream>>>(
      (const Off*)g->off, g->idx, g->n, (uint32_t)g->row_lo, (uint32_t)g->row_hi, (Off*)g->pbeg,
      (Off*)g->pend);
  return cudaGetLastError();
}

cudaError_t launch_push_ranges(pp_graph g) {
  return g->off64 ? ranges_t<uint64_t>(g) : ranges_t<uint32_t>(g);
}

static int host_decide(int rule, int dir, long long c_old, long long c_new, long long m_f,
                       long long m_u, long long n, double alpha, double beta) {
  // identical arithmetic to the device decide() and oracle_direction (IEEE double)
  if (rule == 0) {
    if (dir == 0) return (c_new > c_old && (double)m_f * alpha > (double)m_u) ? 1 : 0;
    return (c_new < c_old && (double)c_new * beta < (double)n) ? 0 : 1;
  }
  const double cn = (double)c_new, nn = (double)n;
  if (dir == 0) return (c_new > c_old && cn > alpha * nn) ? 1 : 0;
  return (c_new < c_old && cn < beta * nn) ? 0 : 1;
}

template <typename Off, bool PARENTS>
static int bfs_dist_t(pp_graph g, uint32_t s, int mode, int rule, double alpha, double beta,
                      int32_t* depth, uint32_t* parent, DistLevel* levels, int cap,
                      int* nlevels, long long* reached, const char** why) {
  cudaStream_t st = g->ctx->stream;
  const int blocks = g->ctx->num_sms * 4;
  const int64_t W = g->dist_words;
  const int64_t cw = g->chunk_words;
  const int rank = g->ctx->rank;
  uint64_t& L = g->ctx->launches;
  L += 1;
  k_dist_init<<<blocks, kBlock, 0, st>>>(g->dvis, g->dfr, g->dnxt, W, s, depth, parent, g->row_lo,
                                         g->row_hi);
  const Off* off = (const Off*)g->off;
  const Off* coff = (const Off*)g->coff;
  long long indeg_s = 0;
  {
    Off h[2];
    cudaMemcpyAsync(h, coff + s, 2 * sizeof(Off), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    indeg_s = (long long)(h[1] - h[0]);
  }
  long long m_u = g->nnz - indeg_s, c_old = 1, reach = 1;
  int dir = mode == 2 ? 1 : 0;
  int d = 1;
  for (;; ++d) {
    cudaMemsetAsync(g->dcnt, 0, 4 * sizeof(unsigned long long), st);
    L += 1;
    if (dir == 0)
      k_dist_push<Off, PARENTS><<<blocks, kBlock, 0, st>>>(g->dfr, g->dvis, g->dnxt, W,
                                                           (const Off*)g->pbeg, (const Off*)g->pend,
                                                           g->idx, g->row_lo, depth, parent, d + 1);
    else
      k_dist_pull<Off, PARENTS><<<blocks, kBlock, 0, st>>>(
          g->dvis, g->diso, g->dnxt, g->row_lo / 32, (g->row_hi + 31) / 32, coff, g->cidx,
          g->row_lo, g->n, depth, parent, d + 1);
    // exchange: in-place all-gather of every rank's owned slice of the next bitmap
    ncclResult_t r = g_nccl.allGather(g->dnxt + (size_t)rank * cw, g->dnxt, (size_t)cw * 4,
                                      ncclUint8, (ncclComm_t)g->ctx->comm, st);
    if (r != ncclSuccess) {
      *why = g_nccl.getErrorString(r);
      return -2;
    }
    L += 1;
    k_dist_finish<Off><<<blocks, kBlock, 0, st>>>(g->dvis, g->dfr, g->dnxt, W, off, coff, g->dcnt);
    cudaMemcpyAsync(g->dcnt_host, g->dcnt, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                    st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      *why = cudaGetErrorString(e);
      return -1;
    }
    const long long c_new = (long long)g->dcnt_host[0], mf = (long long)g->dcnt_host[1],
                    mfin = (long long)g->dcnt_host[2];
    m_u -= g->symmetric ? mf : mfin;
    reach += c_new;
    if (d - 1 < cap) levels[d - 1] = DistLevel{dir, c_new, mf, m_u};
    if (c_new == 0 || d >= g->n + 1) break;
    int next = dir;
    if (mode == 0) next = host_decide(rule, dir, c_old, c_new, mf, m_u, g->n, alpha, beta);
    dir = next;
    c_old = c_new;
  }
  *nlevels = d;
  *reached = reach;
  return 0;
}

int launch_bfs_dist(pp_graph g, uint32_t source, int mode, int rule, double alpha, double beta,
                    int32_t* depth, uint32_t* parent, DistLevel* levels, int cap, int* nlevels,
                    long long* reached, const char** why) {
  if (g->off64)
    return parent ? bfs_dist_t<uint64_t, true>(g, source, mode, rule, alpha, beta, depth, parent,
                                               levels, cap, nlevels, reached, why)
                  : bfs_dist_t<uint64_t, false>(g, source, mode, rule, alpha, beta, depth, parent,
                                                levels, cap, nlevels, reached, why);
  return parent ? bfs_dist_t<uint32_t, true>(g, source, mode, rule, alpha, beta, depth, parent,
                                             levels, cap, nlevels, reached, why)
                : bfs_dist_t<uint32_t, false>(g, source, mode, rule, alpha, beta, depth, parent,
                                              levels, cap, nlevels, reached, why);
}

}  // namespace pp
