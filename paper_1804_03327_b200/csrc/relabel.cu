// relabel.cu — optional degree-ordered vertex relabelling at graph upload (PP_GRAPH_RELABEL).
//
// Internal id = rank of the vertex in order of decreasing degree (out + in; ties by
// increasing caller id).  The graph's rows are renumbered and each row re-sorted, so:
//  - the non-isolated vertices form a dense prefix and the still-unvisited candidates of a
//    pull level sit in few, dense bitmap items: their row records stream from HBM instead
//    of being scattered 32-byte sectors;
//  - every pull row lists its highest-degree in-neighbours first, which are the ones
//    visited earliest, so the early exit fires at the first probe far more often;
//  - the visited bits the pull probes most (hubs) share a few cache lines.
// Upload-time preprocessing, excluded from BFS timing like the CSR build.  Results
// are reported in the caller's ids (bfs.cu maps them through perm / rank).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "pp_device.cuh"

namespace pp {

__global__ void k_relabel_keys(const int64_t* __restrict__ off, const int64_t* __restrict__ coff,
                               int symmetric, int64_t n, uint32_t* __restrict__ key,
                               uint32_t* __restrict__ iota) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = off[v + 1] - off[v];
    if (!symmetric) d += coff[v + 1] - coff[v];
    const uint32_t dc = d > 0xFFFFFFFFll ? 0xFFFFFFFFu : (uint32_t)d;
    key[v] = ~dc;  // ascending radix sort of ~deg = decreasing degree, stable in v
    iota[v] = (uint32_t)v;
  }
}

__global__ void k_relabel_rank(const uint32_t* __restrict__ perm, int64_t n, uint32_t* __restrict__ rank) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    rank[perm[i]] = (uint32_t)i;
}

// new row i = old row perm[i]: degree (for the offsets scan)
__global__ void k_relabel_deg(const int64_t* __restrict__ off, const uint32_t* __restrict__ perm,
                              int64_t n, int64_t* __restrict__ ndeg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = perm[i];
    ndeg[i] = off[v + 1] - off[v];
  }
}

// one warp per new row: copy the old row's ids mapped to internal ids (unsorted)
__global__ void k_relabel_rows(const int64_t* __restrict__ off, const uint32_t* __restrict__ idx,
                               const int64_t* __restrict__ noff, const uint32_t* __restrict__ perm,
                               const uint32_t* __restrict__ rank, int64_t n, uint32_t* __restrict__ nidx) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; i < n; i += warps) {
    const uint32_t v = perm[i];
    const int64_t b = off[v], d = off[v + 1] - b, nb = noff[i];
    for (int64_t p = lane_id(); p < d; p += 32) nidx[nb + p] = rank[idx[b + p]];
  }
}

namespace {
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t b) { return cudaMalloc(&p, b > 0 ? b : 1); }
};
#define RL_CK(x)                        \
  do {                                  \
    cudaError_t _e = (x);               \
    if (_e != cudaSuccess) return _e;   \
  } while (0)

// Renumber one side (CSR or CSC): new int64 offsets into noff[n+1], sorted rows into *idx
// (replaced: the old id array is reused as the sort output).
cudaError_t relabel_side(cudaStream_t st, int blocks, int64_t n, int64_t nnz, const int64_t* off,
                         uint32_t* idx, const uint32_t* perm, const uint32_t* rank, int64_t* noff) {
  DevBuf ndeg, tmp, nidx;
  RL_CK(ndeg.alloc(sizeof(int64_t) * n));
  k_relabel_deg<<<blocks, kBlock, 0, st>>>(off, perm, n, (int64_t*)ndeg.p);
  RL_CK(cudaMemsetAsync(noff, 0, sizeof(int64_t), st));
  size_t tb = 0;
  RL_CK(cub::DeviceScan::InclusiveSum(nullptr, tb, (int64_t*)ndeg.p, noff + 1, (int)n, st));
  RL_CK(tmp.alloc(tb));
  RL_CK(cub::DeviceScan::InclusiveSum(tmp.p, tb, (int64_t*)ndeg.p, noff + 1, (int)n, st));
  if (nnz == 0) return cudaGetLastError();
  RL_CK(nidx.alloc(sizeof(uint32_t) * nnz));
  k_relabel_rows<<<blocks, kBlock, 0, st>>>(off, idx, noff, perm, rank, n, (uint32_t*)nidx.p);
  size_t sb = 0;
  RL_CK(cub::DeviceSegmentedSort::SortKeys(nullptr, sb, (const uint32_t*)nidx.p, idx, (int)nnz,
                                           (int)n, noff, noff + 1, st));
  DevBuf stmp;
  RL_CK(stmp.alloc(sb));
  RL_CK(cub::DeviceSegmentedSort::SortKeys(stmp.p, sb, (const uint32_t*)nidx.p, idx, (int)nnz,
                                           (int)n, noff, noff + 1, st));
  RL_CK(cudaStreamSynchronize(st));  // temporaries are freed on return
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_relabel(pp_graph g, const int64_t* d_off64, const int64_t* d_coff64,
                           int64_t* new_off64, int64_t* new_coff64, uint64_t* launches) {
  cudaStream_t st = g->ctx->stream;
  const int blocks = g->ctx->num_sms * 8;
  const int64_t n = g->n;
  DevBuf keys, keys2, iota;
  RL_CK(keys.alloc(sizeof(uint32_t) * n));
  RL_CK(keys2.alloc(sizeof(uint32_t) * n));
  RL_CK(iota.alloc(sizeof(uint32_t) * n));
  k_relabel_keys<<<blocks, kBlock, 0, st>>>(d_off64, d_coff64, g->symmetric ? 1 : 0, n,
                                            (uint32_t*)keys.p, (uint32_t*)iota.p);
  size_t tb = 0;
  RL_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, (const uint32_t*)keys.p, (uint32_t*)keys2.p,
                                        (const uint32_t*)iota.p, g->perm, (int)n, 0, 32, st));
  DevBuf tmp;
  RL_CK(tmp.alloc(tb));
  RL_CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, (const uint32_t*)keys.p, (uint32_t*)keys2.p,
                                        (const uint32_t*)iota.p, g->perm, (int)n, 0, 32, st));
  k_relabel_rank<<<blocks, kBlock, 0, st>>>(g->perm, n, g->rank);
  *launches += 6;
  RL_CK(relabel_side(st, blocks, n, g->nnz, d_off64, g->idx, g->perm, g->rank, new_off64));
  if (!g->symmetric) {
    *launches += 4;
    RL_CK(relabel_side(st, blocks, n, g->nnz, d_coff64, g->cidx, g->perm, g->rank, new_coff64));
  }
  RL_CK(cudaStreamSynchronize(st));
  return cudaGetLastError();
}

// Vector permutations for pp_mxv on a relabelled graph (gather form, no atomics):
// to_internal: out bit i = in bit perm[i]; to_caller: out bit v = in bit rank[v].
__global__ void k_permute_bits(const uint32_t* __restrict__ in, const uint32_t* __restrict__ map,
                               int64_t n, uint32_t nwords, uint32_t* __restrict__ out) {
  const int64_t total = (int64_t)nwords * 32;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool b = false;
    if (i < n) {
      const uint32_t j = map[i];
      b = (in[j >> 5] >> (j & 31u)) & 1u;
    }
    const uint32_t word = __ballot_sync(kFull, b);
    if (lane_id() == 0) out[i >> 5] = word;
  }
}

cudaError_t launch_permute_bits(pp_graph g, const uint32_t* in, bool to_internal, uint32_t* out) {
  const int blocks = g->ctx->num_sms * 8;
  g->ctx->launches += 1;
  k_permute_bits<<<blocks, kBlock, 0, g->ctx->stream>>>(in, to_internal ? g->perm : g->rank, g->n,
                                                        g->nwords, out);
  return cudaGetLastError();
}

}  // namespace pp
