// graph.cu — graph residency: offset narrowing, the isolated /
// padding bitmap (vertices no traversal can touch), heavy-chunk capacity, validation.
#include "pp_device.cuh"

namespace pp {

template <typename Off>
__global__ void k_off_narrow(const int64_t* __restrict__ in, Off* __restrict__ out, int64_t m) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (Off)in[i];
}

// bit v of word w: 1 when v >= n (padding) or v has neither in- nor out-edges.
__global__ void k_isolated(const int64_t* __restrict__ off, const int64_t* __restrict__ coff,
                           int64_t n, uint32_t nwords, uint32_t* __restrict__ iso,
                           unsigned long long* __restrict__ niso) {
  unsigned long long cnt = 0;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += gridDim.x * blockDim.x) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t v = (int64_t)w * 32 + b;
      bool isolated = true;
      if (v < n) isolated = (off[v + 1] == off[v]) && (coff[v + 1] == coff[v]);
      bits |= (isolated ? 1u : 0u) << b;
    }
    iso[w] = bits;
    cnt += (unsigned long long)__popc(bits);
  }
  if (cnt) atomicAdd(niso, cnt);
}

// Pull row record {in-neighbours 0..5 (0xFFFFFFFF-padded), caller id (perm == nullptr: the row
// itself, i.e. the block slot of a multi-rank block), in-degree}, 32 bytes: the sparse pull's
// one load per candidate (an ELL head in front of the CSR tail); one 1 KB bulk copy brings a
// bitmap word's 32 rows to the dense pull.  Rows >= n
// (padding of the last words) stay zero (in-degree 0; they are pre-marked visited anyway).
__global__ void k_drec(const int64_t* __restrict__ coff, const uint32_t* __restrict__ cidx,
                       const uint32_t* __restrict__ perm, int64_t n, uint32_t* __restrict__ drec) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = coff[v], d = coff[v + 1] - b;
    uint4 r0, r1;
    r0.x = d > 0 ? cidx[b] : 0xFFFFFFFFu;
    r0.y = d > 1 ? cidx[b + 1] : 0xFFFFFFFFu;
    r0.z = d > 2 ? cidx[b + 2] : 0xFFFFFFFFu;
    r0.w = d > 3 ? cidx[b + 3] : 0xFFFFFFFFu;
    r1.x = d > 4 ? cidx[b + 4] : 0xFFFFFFFFu;
    r1.y = d > 5 ? cidx[b + 5] : 0xFFFFFFFFu;
    r1.z = perm ? perm[v] : (uint32_t)v;
    r1.w = (uint32_t)d;
    reinterpret_cast<uint4*>(drec)[2 * v] = r0;
    reinterpret_cast<uint4*>(drec)[2 * v + 1] = r1;
  }
}

// Heavy-chunk capacity: sum over rows with degree >= kHeavy of ceil(deg / kChunk).
__global__ void k_hcap(const int64_t* __restrict__ off, int64_t n, unsigned long long* out,
                       unsigned long long* maxdeg) {
  unsigned long long c = 0, m = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = off[v + 1] - off[v];
    if (d >= (int64_t)kHeavy) c += (unsigned long long)((d + kChunk - 1) / kChunk);
    m = max(m, (unsigned long long)d);
  }
  c = warp_sum(c);
  for (int o = 16; o >= 1; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
  if (lane_id() == 0 && c) atomicAdd(out, c);
  if (lane_id() == 0 && m) atomicMax(maxdeg, m);
}

// First offending row (or none): non-monotone offsets, id >= n, unsorted / duplicate.
// rows = rows given (a rank's block in a multi-rank upload), n = bound on the ids.
__global__ void k_validate(const int64_t* __restrict__ off, const uint32_t* __restrict__ idx,
                           int64_t rows, int64_t n, unsigned long long* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = off[i], e = off[i + 1];
    bool ok = b <= e;
    for (int64_t p = b; ok && p < e; ++p) {
      const uint32_t x = idx[p];
      if ((int64_t)x >= n) ok = false;
      if (p > b && idx[p - 1] >= x) ok = false;
    }
    if (!ok) atomicMin(bad, (unsigned long long)i);
  }
}

cudaError_t launch_graph_validate(pp_graph g, const int64_t* d_off64, const uint32_t* d_idx,
                                  unsigned long long* d_bad, uint64_t* launches, int64_t rows) {
  const int blocks = g->ctx->num_sms * 8;
  *launches += 1;
  k_validate<<<blocks, kBlock, 0, g->ctx->stream>>>(d_off64, d_idx, rows < 0 ? g->n : rows, g->n,
                                                     d_bad);
  return cudaGetLastError();
}

// ---- pieces of the multi-rank (1D row partition) upload, dist.cu -------------------------
cudaError_t launch_off_narrow(pp_graph g, const int64_t* in, void* out, int64_t m) {
  const int blocks = g->ctx->num_sms * 8;
  g->ctx->launches += 1;
  if (g->off64) k_off_narrow<uint64_t><<<blocks, kBlock, 0, g->ctx->stream>>>(in, (uint64_t*)out, m);
  else k_off_narrow<uint32_t><<<blocks, kBlock, 0, g->ctx->stream>>>(in, (uint32_t*)out, m);
  return cudaGetLastError();
}
cudaError_t launch_drec(pp_graph g, const int64_t* coff, const uint32_t* cidx, int64_t rows) {
  g->ctx->launches += 1;
  k_drec<<<g->ctx->num_sms * 8, kBlock, 0, g->ctx->stream>>>(coff, cidx, nullptr, rows, g->drec);
  return cudaGetLastError();
}
cudaError_t launch_hcap(pp_graph g, const int64_t* off, int64_t rows, unsigned long long* d_cap,
                        unsigned long long* d_max) {
  g->ctx->launches += 1;
  k_hcap<<<g->ctx->num_sms * 8, kBlock, 0, g->ctx->stream>>>(off, rows, d_cap, d_max);
  return cudaGetLastError();
}

// Relabelled graph: one 16-byte record per vertex {row begin lo, hi, out-degree, caller id}
// so a push discovery gets its offsets and the caller id of its depth slot in ONE scattered
// access instead of two (offsets, perm).
__global__ void k_vrec(const int64_t* __restrict__ off, const uint32_t* __restrict__ perm, int64_t n,
                       uint4* __restrict__ vrec) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = off[v];
    vrec[v] = make_uint4((uint32_t)b, (uint32_t)((uint64_t)b >> 32), (uint32_t)(off[v + 1] - b), perm[v]);
  }
}

cudaError_t launch_graph_prepare(pp_graph g, const int64_t* d_off64, const int64_t* d_coff64,
                                 unsigned long long* d_scratch, uint64_t* launches) {
  cudaStream_t st = g->ctx->stream;
  const int blocks = g->ctx->num_sms * 8;
  if (g->off64) {
    *launches += 1;
    k_off_narrow<uint64_t><<<blocks, kBlock, 0, st>>>(d_off64, (uint64_t*)g->off, g->n + 1);
    if (!g->symmetric) {
      *launches += 1;
      k_off_narrow<uint64_t><<<blocks, kBlock, 0, st>>>(d_coff64, (uint64_t*)g->coff, g->n + 1);
    }
  } else {
    *launches += 1;
    k_off_narrow<uint32_t><<<blocks, kBlock, 0, st>>>(d_off64, (uint32_t*)g->off, g->n + 1);
    if (!g->symmetric) {
      *launches += 1;
      k_off_narrow<uint32_t><<<blocks, kBlock, 0, st>>>(d_coff64, (uint32_t*)g->coff, g->n + 1);
    }
  }
  if (g->vrec) {
    *launches += 1;
    k_vrec<<<blocks, kBlock, 0, st>>>(d_off64, g->perm, g->n, g->vrec);
  }
  *launches += 3;
  if (g->drec) {
    *launches += 1;
    k_drec<<<blocks, kBlock, 0, st>>>(d_coff64, g->cidx, g->perm, g->n, g->drec);
  }
  k_isolated<<<blocks, kBlock, 0, st>>>(d_off64, d_coff64, g->n, g->nwords, g->isolated,
                                        d_scratch + 4);
  k_hcap<<<blocks, kBlock, 0, st>>>(d_off64, g->n, d_scratch + 0, d_scratch + 2);
  k_hcap<<<blocks, kBlock, 0, st>>>(d_coff64, g->n, d_scratch + 1, d_scratch + 3);
  return cudaGetLastError();
}

}  // namespace pp
