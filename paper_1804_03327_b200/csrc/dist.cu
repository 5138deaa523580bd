// dist.cu — multi-rank graph residency for the 1D row partition (the paper
// names distributed GPUs as future work).  DESIGN.md §7.
//
// Rank p of P owns the vertex block [lo_p, hi_p) (bitmap words [p*cw, (p+1)*cw), cw a
// multiple of 32 words, so blocks are 1024-vertex aligned) and keeps ONLY:
//   - the CSC rows of its block (in-neighbours, global ids) + their 8-id row heads: pull;
//   - the PUSH structure: for every global vertex u, the out-neighbours of u inside the
//     block — the transpose of the CSC block, built here on the device (count, scan,
//     scatter, per-row sort) — so a push expands the global frontier but discovers only
//     owned vertices (no all-to-all);
//   - the global out-degree of its rows (directed graphs; m_f of the direction rule);
//   - replicated bitmaps (visited x2, frontier x2: n/8 bytes each) and an exchange buffer
//     that the peers write into: frontier bitmaps, per-level counter records, flags.
// Graph bytes per rank ~ (2 * 4 * nnz + 4 n) / P + 4 n: the graph is partitioned, only the
// O(n) push offsets and bitmaps are replicated.
//
// The peers' exchange buffers are mapped into every rank's address space: through CUDA IPC
// handles exchanged over the NCCL communicator (one process per GPU), or directly for a
// single-device team (pp_team_create, same device).  The BFS kernel (bfs.cu, D = true)
// writes the peers' copies itself — no host-issued collective on the data path.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
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
// so libpushpull.so loads and serves single-GPU calls on systems without NCCL.  NCCL is the
// bootstrap of the multi-rank path only (exchange of the IPC handles at upload).
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

// All-gather of a small host record (bootstrap only), staged through device memory:
// recv receives nranks * bytes.
int nccl_allgather_host(void* comm, const void* send, void* recv, size_t bytes, int nranks,
                        cudaStream_t st, const char** why) {
  char* d = nullptr;
  if (cudaMalloc((void**)&d, bytes * (size_t)(nranks + 1)) != cudaSuccess) {
    cudaGetLastError();
    *why = "cudaMalloc (bootstrap buffer)";
    return -1;
  }
  int rc = 0;
  if (cudaMemcpyAsync(d, send, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) {
    *why = "cudaMemcpyAsync (bootstrap)";
    rc = -1;
  }
  if (!rc) {
    const ncclResult_t r = g_nccl.allGather(d, d + bytes, bytes, ncclUint8, (ncclComm_t)comm, st);
    if (r != ncclSuccess) {
      *why = g_nccl.getErrorString(r);
      rc = -2;
    }
  }
  if (!rc && (cudaMemcpyAsync(recv, d + bytes, bytes * (size_t)nranks, cudaMemcpyDeviceToHost, st) !=
                  cudaSuccess ||
              cudaStreamSynchronize(st) != cudaSuccess)) {
    *why = "cudaMemcpy (bootstrap)";
    rc = -1;
  }
  cudaStreamSynchronize(st);
  cudaFree(d);
  cudaGetLastError();
  return rc;
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

// in-edge count per global source u over the block's CSC ids (push-structure row lengths)
__global__ void k_count_src(const uint32_t* __restrict__ cidx, int64_t m,
                            unsigned long long* __restrict__ cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[cidx[e]], 1ull);
}

// scatter: CSC entry (u -> lo + r) of local row r lands in push row u (warp per row)
__global__ void k_fill_push(const int64_t* __restrict__ coff, const uint32_t* __restrict__ cidx,
                            int64_t rows, uint32_t lo, unsigned long long* __restrict__ cursor,
                            uint32_t* __restrict__ pidx) {
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < rows; r += nw) {
    const int64_t b = coff[r], e = coff[r + 1];
    for (int64_t p = b + lane_id(); p < e; p += 32) {
      const unsigned long long pos = atomicAdd(&cursor[cidx[p]], 1ull);
      pidx[pos] = lo + (uint32_t)r;
    }
  }
}

// isolated / padding bits of the owned words: local row >= rows (past the block or n), or no
// in- and no out-edges
__global__ void k_iso_block(const int64_t* __restrict__ off, const int64_t* __restrict__ coff,
                            int64_t rows, uint32_t wlo, uint32_t cw, uint32_t* __restrict__ iso,
                            unsigned long long* __restrict__ niso) {
  unsigned long long cnt = 0;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < cw; w += gridDim.x * blockDim.x) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t r = (int64_t)w * 32 + b;
      bool isolated = true;
      if (r < rows) isolated = (off[r + 1] == off[r]) && (coff[r + 1] == coff[r]);
      bits |= (isolated ? 1u : 0u) << b;
    }
    iso[wlo + w] = bits;
    cnt += (unsigned long long)__popc(bits);
  }
  if (cnt) atomicAdd(niso, cnt);
}

__global__ void k_odeg(const int64_t* __restrict__ off, int64_t rows, uint32_t* __restrict__ od) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    od[r] = (uint32_t)(off[r + 1] - off[r]);
}

// ---------------------------------------------------------------------------- launchers --

struct DTmp {  // scratch device buffer freed on scope exit
  void* p = nullptr;
  ~DTmp() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t b) { return cudaMalloc(&p, b < 1 ? 1 : b); }
};

#define DS_CK(x)                              \
  do {                                        \
    cudaError_t _e = (x);                     \
    if (_e != cudaSuccess) return _e;         \
  } while (0)

// Push structure of the block: poff64[n+1] (int64) and pidx[m] (global ids, rows sorted).
cudaError_t launch_push_structure(pp_graph g, const int64_t* d_coff64, int64_t rows, int64_t m,
                                  int64_t* poff64, uint32_t* pidx) {
  cudaStream_t st = g->ctx->stream;
  const int blocks = g->ctx->num_sms * 8;
  const int64_t n = g->n;
  DTmp cnt, cursor, tmp, pidx2;
  DS_CK(cnt.alloc(sizeof(unsigned long long) * (size_t)(n + 1)));
  DS_CK(cursor.alloc(sizeof(unsigned long long) * (size_t)(n + 1)));
  DS_CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * (size_t)(n + 1), st));
  g->ctx->launches += 3;
  k_count_src<<<blocks, kBlock, 0, st>>>(g->cidx, m, (unsigned long long*)cnt.p);
  size_t tb = 0;
  DS_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, (unsigned long long*)cnt.p,
                                      (unsigned long long*)poff64, (int)(n + 1), st));
  DS_CK(tmp.alloc(tb));
  DS_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, (unsigned long long*)cnt.p,
                                      (unsigned long long*)poff64, (int)(n + 1), st));
  DS_CK(cudaMemcpyAsync(cursor.p, poff64, sizeof(int64_t) * (size_t)(n + 1),
                        cudaMemcpyDeviceToDevice, st));
  k_fill_push<<<blocks, kBlock, 0, st>>>(d_coff64, g->cidx, rows, (uint32_t)g->row_lo,
                                         (unsigned long long*)cursor.p, pidx);
  DS_CK(cudaGetLastError());
  // sorted rows (ascending owned ids): deterministic layout, sequential visited words
  if (m > 1 && m < (int64_t)0x7FFFFFFF && n < (int64_t)0x7FFFFFFF) {
    DS_CK(pidx2.alloc(sizeof(uint32_t) * (size_t)m));
    DS_CK(cudaMemcpyAsync(pidx2.p, pidx, sizeof(uint32_t) * (size_t)m, cudaMemcpyDeviceToDevice, st));
    size_t sb = 0;
    DS_CK(cub::DeviceSegmentedSort::SortKeys(nullptr, sb, (const uint32_t*)pidx2.p, pidx, (int)m,
                                             (int)n, poff64, poff64 + 1, st));
    DTmp stmp;
    DS_CK(stmp.alloc(sb));
    DS_CK(cub::DeviceSegmentedSort::SortKeys(stmp.p, sb, (const uint32_t*)pidx2.p, pidx, (int)m,
                                             (int)n, poff64, poff64 + 1, st));
    DS_CK(cudaStreamSynchronize(st));  // scratch freed on return
  } else {
    DS_CK(cudaStreamSynchronize(st));
  }
  return cudaSuccess;
}

cudaError_t launch_block_prepare(pp_graph g, const int64_t* d_off64, const int64_t* d_coff64,
                                 int64_t rows) {
  cudaStream_t st = g->ctx->stream;
  const int blocks = g->ctx->num_sms * 8;
  g->ctx->launches += 1;
  k_iso_block<<<blocks, kBlock, 0, st>>>(d_off64, d_coff64, rows,
                                         (uint32_t)(g->me * g->chunk_words),
                                         (uint32_t)g->chunk_words, g->isolated, g->scount + 5);
  if (g->odeg) {
    g->ctx->launches += 1;
    k_odeg<<<blocks, kBlock, 0, st>>>(d_off64, rows, g->odeg);
  }
  return cudaGetLastError();
}

}  // namespace pp
