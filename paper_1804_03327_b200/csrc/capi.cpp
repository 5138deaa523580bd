// capi.cpp — the C ABI of include/pushpull.h: argument validation, ownership, device
// residency and the host side of pp_mxv / pp_bfs.  Every compute step runs in the
// CUDA kernels of bfs.cu / mxv.cu / graph.cu; there is no CPU path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pp_internal.h"

namespace pp {
static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

pp_status cuda_fail(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  cudaGetLastError();  // clear sticky-free errors
  return e == cudaErrorMemoryAllocation ? PP_ERR_OOM : PP_ERR_CUDA;
}
}  // namespace pp

using namespace pp;

#define PP_CK(call, what)                                 \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return pp::cuda_fail(_e, what); \
  } while (0)

#define PP_FAIL(code, ...)  \
  do {                      \
    set_error(__VA_ARGS__); \
    return code;            \
  } while (0)

namespace {

template <typename T>
pp_status dalloc(T** p, size_t count, int64_t* bytes, const char* what) {
  size_t b = sizeof(T) * std::max<size_t>(count, 1);
  cudaError_t e = cudaMalloc((void**)p, b);
  if (e != cudaSuccess) {
    *p = nullptr;
    return cuda_fail(e, what);
  }
  *bytes += (int64_t)b;
  return PP_OK;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void free_graph(pp_graph g) {
  if (!g) return;
  // multi-rank: unmap the peers' exchange buffers first (CUDA IPC, multi-process only)
  for (int q = 0; q < kMaxRanks; ++q)
    if (g->ipc_base[q]) cudaIpcCloseMemHandle(g->ipc_base[q]);
  const bool alias = g->dist ? false : g->symmetric;  // multi-rank: coff/off are distinct
  void* ptrs[] = {g->off, g->idx, alias ? nullptr : g->coff,
                  (alias || g->cidx == g->idx) ? nullptr : (void*)g->cidx, g->isolated,
                  g->vis[0], g->vis[1], g->fr, g->sumv,
                  g->L[0], g->L[1], g->H[0], g->H[1], g->ctr, g->stats, g->bar,
                  g->sbits[0], g->sbits[1], g->sbits[2], g->sbits[3], g->sblock, g->hubq, g->scount,
                  g->dtmp[0], g->dtmp[1], g->dbg, g->perm, g->rank, g->pint, g->vrec,
                  g->rbits[0], g->rbits[1], g->rbits[2], g->rbits[3],
                  g->odeg, g->xbuf, g->dargs, g->gwork, g->drec};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (g->status_host) cudaFreeHost(g->status_host);
  if (g->scount_host) cudaFreeHost(g->scount_host);
  if (g->hargs) cudaFreeHost(g->hargs);
  delete g;
}

struct Guard {  // frees a half-built graph on early return
  pp_graph g;
  ~Guard() { free_graph(g); }
};

// ---- multi-rank residency (dist.cu) -----------------------------------------
// Layout of the exchange buffer every peer writes into (identical on every rank).
struct XLayout {
  size_t fr0, fr1, l0, l1, cnt, flag, own, bytes;
};
XLayout xlayout(int64_t nwords) {
  XLayout L;
  const size_t fb = sizeof(uint32_t) * (size_t)nwords;  // multiple of 128 bytes
  L.fr0 = 0;
  L.fr1 = fb;
  L.l0 = 2 * fb;  // id lists, same geometry as the bitmap slices (a list is sent only when it
  L.l1 = 3 * fb;  // is shorter than the sender's slice in words)
  L.cnt = 4 * fb;
  L.flag = L.cnt + sizeof(unsigned long long) * 2 * kMaxRanks * 8;
  L.own = L.flag + sizeof(unsigned long long) * kMaxRanks;
  L.bytes = L.own + fb;  // own list (local only), >= one slice
  return L;
}

void set_peer(pp_graph g, int q, char* base, const XLayout& L) {
  g->pfr[q][0] = (uint32_t*)(base + L.fr0);
  g->pfr[q][1] = (uint32_t*)(base + L.fr1);
  g->plst[q][0] = (uint32_t*)(base + L.l0);
  g->plst[q][1] = (uint32_t*)(base + L.l1);
  g->pcnt[q] = (unsigned long long*)(base + L.cnt);
  g->pflag[q] = (unsigned long long*)(base + L.flag);
}

// Bootstrap record of one rank (all-gathered over the NCCL communicator).
struct BootRec {
  cudaIpcMemHandle_t h;  // 64 bytes: the rank's exchange buffer
  int64_t n, lo, hi, nnz;
  int32_t rank, nranks, off64, symmetric;
  int64_t noniso;  // the block's non-isolated rows (dense-pull decision needs the global sum)
  char pad[8];
};
static_assert(sizeof(BootRec) == 128, "BootRec layout");

// This rank's bootstrap record.
pp_status make_record(pp_graph g, BootRec* me) {
  memset(me, 0, sizeof(*me));
  if (g->nranks > 1) PP_CK(cudaIpcGetMemHandle(&me->h, g->xbuf), "cudaIpcGetMemHandle");
  me->n = g->n;
  me->lo = g->row_lo;
  me->hi = g->row_hi;
  me->nnz = g->nnz;
  me->noniso = g->n_noniso_block;
  me->rank = g->me;
  me->nranks = g->nranks;
  me->off64 = g->off64 ? 1 : 0;
  me->symmetric = g->symmetric ? 1 : 0;
  return PP_OK;
}

// Check that the ranks agree on the graph and tile it, then map every peer's exchange buffer
// (CUDA IPC: NVLink / NVSwitch peer memory, or the same device).
pp_status attach_records(pp_graph g, const BootRec* all) {
  const int P = g->nranks;
  const XLayout L = xlayout(g->nwords);
  int64_t in_total = 0, noniso = 0;
  for (int q = 0; q < P; ++q) {
    const BootRec& r = all[q];
    int64_t lo, hi, cw;
    partition(g->n, q, P, &lo, &hi, &cw);
    if (r.n != g->n || r.rank != q || r.nranks != P || r.lo != lo || r.hi != hi ||
        r.off64 != (g->off64 ? 1 : 0) || r.symmetric != (g->symmetric ? 1 : 0))
      PP_FAIL(PP_ERR_ARG, "pp_graph_upload: rank %d disagrees on the graph or its block (n=%lld, "
              "rows [%lld, %lld), offsets %s, %s)", q, (long long)r.n, (long long)r.lo,
              (long long)r.hi, r.off64 ? "64-bit" : "32-bit", r.symmetric ? "symmetric" : "directed");
    in_total += r.nnz;
    noniso += r.noniso;
  }
  for (int q = 0; q < P; ++q) {
    if (q == g->me || g->ipc_base[q]) continue;
    void* base = nullptr;
    PP_CK(cudaIpcOpenMemHandle(&base, all[q].h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    g->ipc_base[q] = base;
    set_peer(g, q, (char*)base, L);
  }
  g->in_total = in_total;
  g->n_noniso = noniso;
  g->attached = true;
  return PP_OK;
}

// One process per GPU with an NCCL communicator: all-gather the records over NCCL.
pp_status bootstrap_ipc(pp_graph g) {
  pp_ctx ctx = g->ctx;
  const int P = ctx->nranks;
  BootRec me;
  pp_status s = make_record(g, &me);
  if (s != PP_OK) return s;
  BootRec all[kMaxRanks];
  const char* why = "";
  const int rc = nccl_allgather_host(ctx->comm, &me, all, sizeof(BootRec), P, ctx->stream, &why);
  if (rc != 0) PP_FAIL(rc == -2 ? PP_ERR_NCCL : PP_ERR_CUDA, "pp_graph_upload: bootstrap: %s", why);
  return attach_records(g, all);
}

// pp_graph_upload on a multi-rank context: the rank's CSR / CSC rows [row_lo, row_hi) with
// global column ids (offsets row-local: row_hi - row_lo + 1 entries starting at 0).
pp_status upload_block(pp_ctx ctx, int64_t n, int64_t row_lo, int64_t row_hi, int64_t nnz,
                       const int64_t* csr_off, const uint32_t* csr_idx, const int64_t* csc_off,
                       const uint32_t* csc_idx, uint32_t flags, pp_graph* out) {
  const bool symmetric = (flags & PP_GRAPH_SYMMETRIC) != 0;
  if (flags & PP_GRAPH_RELABEL)
    PP_FAIL(PP_ERR_UNSUPPORTED, "pp_graph_upload: PP_GRAPH_RELABEL is single-GPU only");
  if (ctx->nranks > kMaxRanks)
    PP_FAIL(PP_ERR_UNSUPPORTED, "pp_graph_upload: %d ranks (at most %d)", ctx->nranks, kMaxRanks);
  if (n < 1 || n >= (int64_t)0xFFFFFFFFll)
    PP_FAIL(PP_ERR_UNSUPPORTED, "pp_graph_upload: n=%lld outside [1, 2^32-1)", (long long)n);
  int64_t lo, hi, cw;
  partition(n, ctx->rank, ctx->nranks, &lo, &hi, &cw);
  if (row_lo != lo || row_hi != hi)
    PP_FAIL(PP_ERR_ARG, "pp_graph_upload: rank %d of %d owns rows [%lld, %lld) (pp_partition), got "
            "[%lld, %lld)", ctx->rank, ctx->nranks, (long long)lo, (long long)hi,
            (long long)row_lo, (long long)row_hi);
  if (symmetric) {
    csc_off = csr_off;
    csc_idx = csr_idx;
  }
  if (!csc_off) PP_FAIL(PP_ERR_ARG, "pp_graph_upload: CSC rows required unless PP_GRAPH_SYMMETRIC");
  const int64_t len = hi - lo;
  PP_CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = ctx->stream;
  pp_graph g = new pp_graph_s;
  Guard guard{g};
  g->ctx = ctx;
  g->dist = true;
  g->n = n;
  g->symmetric = symmetric;
  g->me = ctx->rank;
  g->nranks = ctx->nranks;
  g->row_lo = lo;
  g->row_hi = hi;
  g->chunk_words = cw;
  g->nwords = (uint32_t)(cw * ctx->nranks);
  int64_t& bytes = g->device_bytes;
  pp_status s;
  const bool dev = (flags & PP_GRAPH_DEVICE) != 0;
  int64_t junk = 0;
  // block offsets staged as int64 on the device
  if ((s = dalloc(&g->dtmp[0], (size_t)(len + 1) * 2, &junk, "offset staging")) != PP_OK) return s;
  int64_t* d_off = g->dtmp[0];
  int64_t* d_coff = g->dtmp[0] + (len + 1);
  PP_CK(cudaMemcpyAsync(d_off, csr_off, sizeof(int64_t) * (len + 1),
                        dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st), "copy offsets");
  PP_CK(cudaMemcpyAsync(d_coff, csc_off, sizeof(int64_t) * (len + 1),
                        dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st), "copy offsets");
  int64_t ends[4];
  PP_CK(cudaMemcpyAsync(&ends[0], d_off, 8, cudaMemcpyDeviceToHost, st), "read off[0]");
  PP_CK(cudaMemcpyAsync(&ends[1], d_off + len, 8, cudaMemcpyDeviceToHost, st), "read off[len]");
  PP_CK(cudaMemcpyAsync(&ends[2], d_coff, 8, cudaMemcpyDeviceToHost, st), "read coff[0]");
  PP_CK(cudaMemcpyAsync(&ends[3], d_coff + len, 8, cudaMemcpyDeviceToHost, st), "read coff[len]");
  PP_CK(cudaStreamSynchronize(st), "sync");
  if (ends[0] != 0 || ends[1] != nnz)
    PP_FAIL(PP_ERR_GRAPH, "pp_graph_upload: CSR block off[0]=%lld off[len]=%lld, expected 0 and nnz=%lld",
            (long long)ends[0], (long long)ends[1], (long long)nnz);
  const int64_t m = ends[3];  // in-edges of the block (CSC entries)
  if (ends[2] != 0 || m < 0) PP_FAIL(PP_ERR_GRAPH, "pp_graph_upload: CSC block offsets malformed");
  if (m > 0 && !csc_idx) PP_FAIL(PP_ERR_ARG, "pp_graph_upload: CSC ids missing");
  g->nnz = m;
  g->off64 = m >= (int64_t)0xFFFFFFFFll || (flags & PP_GRAPH_OFF64);
  if ((s = dalloc(&g->cidx, (size_t)m + 8, &bytes, "csc idx")) != PP_OK) return s;
  PP_CK(cudaMemsetAsync(g->cidx + m, 0, 8 * sizeof(uint32_t), st), "pad csc idx");
  if (m) PP_CK(cudaMemcpyAsync(g->cidx, csc_idx, sizeof(uint32_t) * m, cudaMemcpyDefault, st), "copy csc idx");
  if ((s = dalloc(&g->scount, 8, &bytes, "counters")) != PP_OK) return s;
  PP_CK(cudaMallocHost((void**)&g->scount_host, 8 * sizeof(unsigned long long)), "pinned counters");
  PP_CK(cudaMallocHost((void**)&g->status_host, sizeof(BfsStatus)), "pinned status");
  if (flags & PP_GRAPH_VALIDATE) {
    PP_CK(cudaMemsetAsync(g->scount, 0xFF, sizeof(unsigned long long), st), "memset");
    PP_CK(launch_graph_validate(g, d_coff, g->cidx, g->scount, &ctx->launches, len), "validate");
    PP_CK(cudaMemcpyAsync(g->scount_host, g->scount, 8, cudaMemcpyDeviceToHost, st), "copy");
    PP_CK(cudaStreamSynchronize(st), "sync");
    if (g->scount_host[0] != ~0ull)
      PP_FAIL(PP_ERR_GRAPH, "pp_graph_upload: CSC row %llu of the block is malformed (offsets "
              "decrease, an id >= n, or the row is not strictly increasing)",
              (unsigned long long)(g->scount_host[0] + (unsigned long long)lo));
  }
  const size_t offb = g->off64 ? 8 : 4;
  // CSC rows of the block (pull), narrowed offsets padded like the single-GPU layout
  {
    void* p = nullptr;
    const size_t cnt = (size_t)cw * 32 + 16;
    PP_CK(cudaMalloc(&p, offb * cnt), "block offsets");
    PP_CK(cudaMemsetAsync(p, 0, offb * cnt, st), "memset");
    g->coff = p;
    bytes += (int64_t)(offb * cnt);
    PP_CK(launch_off_narrow(g, d_coff, g->coff, len + 1), "narrow offsets");
    // rows past the block end keep offset m (empty rows; they are padding, pre-visited)
    if (cnt > (size_t)(len + 1)) {
      // fill the tail with m so coff[r+1]-coff[r] = 0 there
      std::vector<char> tail(offb * (cnt - (size_t)(len + 1)));
      for (size_t k = 0; k < cnt - (size_t)(len + 1); ++k) {
        if (offb == 8) reinterpret_cast<uint64_t*>(tail.data())[k] = (uint64_t)m;
        else reinterpret_cast<uint32_t*>(tail.data())[k] = (uint32_t)m;
      }
      PP_CK(cudaMemcpyAsync((char*)p + offb * (len + 1), tail.data(), tail.size(),
                            cudaMemcpyHostToDevice, st), "offsets tail");
      PP_CK(cudaStreamSynchronize(st), "sync");
    }
  }
  {  // pull row records of the block's rows (ids global, caller id = block slot), padded to the
     // owned words
    const size_t words = (size_t)std::max<int64_t>(g->chunk_words, 1) * 32 * 8;
    if ((s = dalloc(&g->drec, words, &bytes, "pull row records")) != PP_OK) return s;
    PP_CK(cudaMemsetAsync(g->drec, 0, words * 4, st), "memset row records");
    PP_CK(launch_drec(g, d_coff, g->cidx, len), "row records");
  }
  if ((s = dalloc(&g->isolated, g->nwords, &bytes, "isolated")) != PP_OK) return s;
  PP_CK(cudaMemsetAsync(g->isolated, 0, sizeof(uint32_t) * g->nwords, st), "memset");
  if (!symmetric && (s = dalloc(&g->odeg, (size_t)std::max<int64_t>(len, 1), &bytes, "out-degrees")) != PP_OK)
    return s;
  PP_CK(cudaMemsetAsync(g->scount + 5, 0, sizeof(unsigned long long), st), "memset");
  PP_CK(launch_block_prepare(g, d_off, d_coff, len), "block prepare");
  // push structure: transpose of the CSC block (global rows u, owned targets)
  {
    int64_t* poff64 = nullptr;
    if ((s = dalloc(&poff64, (size_t)n + 1, &junk, "push offsets staging")) != PP_OK) return s;
    g->dtmp[1] = poff64;
    if ((s = dalloc(&g->idx, (size_t)m + 8, &bytes, "push ids")) != PP_OK) return s;
    PP_CK(cudaMemsetAsync(g->idx + m, 0, 8 * sizeof(uint32_t), st), "pad push ids");
    PP_CK(launch_push_structure(g, d_coff, len, m, poff64, g->idx), "push structure");
    void* p = nullptr;
    const size_t cnt = (size_t)g->nwords * 32 + 16;
    PP_CK(cudaMalloc(&p, offb * cnt), "push offsets");
    PP_CK(cudaMemsetAsync(p, 0, offb * cnt, st), "memset");
    g->off = p;
    bytes += (int64_t)(offb * cnt);
    PP_CK(launch_off_narrow(g, poff64, g->off, n + 1), "narrow push offsets");
    PP_CK(cudaMemsetAsync(g->scount, 0, 4 * sizeof(unsigned long long), st), "memset");
    PP_CK(launch_hcap(g, poff64, n, g->scount, g->scount + 2), "chunk capacity");
    PP_CK(cudaMemcpyAsync(g->scount_host, g->scount, 48, cudaMemcpyDeviceToHost, st), "copy");
    PP_CK(cudaStreamSynchronize(st), "sync");
    g->hcap = (int64_t)g->scount_host[0];
    g->max_out_deg = (int64_t)g->scount_host[2];
    g->n_noniso_block = g->chunk_words * 32 - (int64_t)g->scount_host[5];
    g->n_noniso = g->n_noniso_block;  // the global count after the bootstrap / team setup
    cudaFree(poff64);
    g->dtmp[1] = nullptr;
  }
  cudaFree(g->dtmp[0]);
  g->dtmp[0] = nullptr;
  // working set: replicated bitmaps, local frontier lists, exchange buffer
  for (int k = 0; k < 2; ++k) {
    if ((s = dalloc(&g->vis[k], g->nwords, &bytes, "visited")) != PP_OK) return s;
    if ((s = dalloc(&g->L[k], (size_t)n * 4, &bytes, "frontier list")) != PP_OK) return s;
    if ((s = dalloc(&g->H[k], (size_t)std::max<int64_t>(g->hcap, 1), &bytes, "heavy chunks")) != PP_OK)
      return s;
  }
  if ((s = dalloc(&g->ctr, kRing, &bytes, "level counters")) != PP_OK) return s;
  if ((s = dalloc(&g->gwork, (size_t)kRing * kMaxCtas, &bytes, "work counters")) != PP_OK) return s;
  g->stats_cap = (int)std::min<int64_t>(n + 1, 1 << 16);
  if ((s = dalloc(&g->stats, (size_t)g->stats_cap, &bytes, "level stats")) != PP_OK) return s;
  if ((s = dalloc(&g->bar, 2, &bytes, "barrier")) != PP_OK) return s;
  g->status = reinterpret_cast<BfsStatus*>(g->bar + 1);
  PP_CK(cudaMemsetAsync(g->bar, 0, sizeof(GridBarrier) * 2, st), "memset");
  const XLayout L = xlayout(g->nwords);
  PP_CK(cudaMalloc(&g->xbuf, L.bytes), "exchange buffer");
  bytes += (int64_t)L.bytes;
  PP_CK(cudaMemsetAsync(g->xbuf, 0, L.bytes, st), "memset exchange buffer");
  g->xfr[0] = (uint32_t*)((char*)g->xbuf + L.fr0);
  g->xfr[1] = (uint32_t*)((char*)g->xbuf + L.fr1);
  g->xcnt = (unsigned long long*)((char*)g->xbuf + L.cnt);
  g->xflag = (unsigned long long*)((char*)g->xbuf + L.flag);
  g->xlst[0] = (uint32_t*)((char*)g->xbuf + L.l0);
  g->xlst[1] = (uint32_t*)((char*)g->xbuf + L.l1);
  g->xown = (uint32_t*)((char*)g->xbuf + L.own);
  set_peer(g, g->me, (char*)g->xbuf, L);
  PP_CK(cudaMalloc(&g->dargs, bfs_args_bytes()), "kernel arguments");
  PP_CK(cudaStreamSynchronize(st), "sync");
  g->in_total = m;
  if (ctx->team) {
    ctx->team->graphs[ctx->rank] = g;
  } else if (ctx->comm) {  // one process per GPU: map the peers now (collective)
    if ((s = bootstrap_ipc(g)) != PP_OK) return s;
  } else if (ctx->nranks == 1) {  // a single rank has no peers
    BootRec me;
    if ((s = make_record(g, &me)) != PP_OK) return s;
    if ((s = attach_records(g, &me)) != PP_OK) return s;
  }  // else: external bootstrap (pp_graph_export / pp_graph_import)
  guard.g = nullptr;
  ctx->refs += 1;
  *out = g;
  return PP_OK;
}

}  // namespace

extern "C" {

const char* pp_last_error(void) { return g_err.c_str(); }
const char* pp_version(void) { return "pushpull-b200 0.1 (sm_100a)"; }

pp_status pp_ctx_create(int device, void* cuda_stream, pp_ctx* out) {
  if (!out) PP_FAIL(PP_ERR_ARG, "pp_ctx_create: out is NULL");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    PP_FAIL(PP_ERR_CUDA, "pp_ctx_create: no CUDA device (%s); there is no CPU fallback",
            e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
  }
  if (device < 0 || device >= count) PP_FAIL(PP_ERR_ARG, "pp_ctx_create: device %d of %d", device, count);
  PP_CK(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop;
  PP_CK(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    PP_FAIL(PP_ERR_UNSUPPORTED, "pp_ctx_create: built for sm_100a (B200), device is sm_%d%d",
            prop.major, prop.minor);
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
  if (!coop) PP_FAIL(PP_ERR_UNSUPPORTED, "pp_ctx_create: device lacks cooperative launch");
  pp_ctx c = new pp_ctx_s;
  c->device = device;
  c->stream = (cudaStream_t)cuda_stream;
  c->num_sms = prop.multiProcessorCount;
  *out = c;
  return PP_OK;
}

static void ctx_release(pp_ctx ctx) {
  if (--ctx->refs == 0) {
    if (ctx->team && --ctx->team->refs == 0) delete ctx->team;
    if (ctx->comm) nccl_comm_destroy(ctx->comm);
    if (ctx->sssp_ws) {
      cudaSetDevice(ctx->device);
      cudaFree(ctx->sssp_ws);
    }
    delete ctx;
  }
}

pp_status pp_nccl_unique_id(void* out128) {
  if (!out128) PP_FAIL(PP_ERR_ARG, "pp_nccl_unique_id: NULL output");
  const char* why = "";
  if (nccl_unique_id(out128, &why) != 0) PP_FAIL(PP_ERR_NCCL, "pp_nccl_unique_id: %s", why);
  return PP_OK;
}

pp_status pp_ctx_create_dist(int device, void* cuda_stream, const void* nccl_unique_id_,
                             int rank, int nranks, pp_ctx* out) {
  if (!out) PP_FAIL(PP_ERR_ARG, "pp_ctx_create_dist: NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks || nranks > kMaxRanks)
    PP_FAIL(PP_ERR_ARG, "pp_ctx_create_dist: rank %d of %d (at most %d ranks)", rank, nranks, kMaxRanks);
  pp_status s = pp_ctx_create(device, cuda_stream, out);
  if (s != PP_OK) return s;
  const char* why = "";
  void* comm = nullptr;
  if (nccl_unique_id_ && nccl_comm_init(&comm, nranks, nccl_unique_id_, rank, &why) != 0) {
    delete *out;
    *out = nullptr;
    PP_FAIL(PP_ERR_NCCL, "pp_ctx_create_dist: ncclCommInitRank: %s", why);
  }
  (*out)->comm = comm;
  (*out)->rank = rank;
  (*out)->nranks = nranks;
  return PP_OK;
}

pp_status pp_partition(int64_t n, int32_t rank, int32_t nranks, int64_t* row_lo, int64_t* row_hi) {
  if (!row_lo || !row_hi || n < 1 || nranks < 1 || rank < 0 || rank >= nranks)
    PP_FAIL(PP_ERR_ARG, "pp_partition: bad arguments");
  int64_t cw;
  partition(n, rank, nranks, row_lo, row_hi, &cw);
  return PP_OK;
}

pp_status pp_ctx_destroy(pp_ctx ctx) {
  if (!ctx) PP_FAIL(PP_ERR_ARG, "pp_ctx_destroy: NULL ctx");
  ctx_release(ctx);  // graphs still alive keep the context until they are freed
  return PP_OK;
}

pp_status pp_ctx_launch_count(pp_ctx ctx, uint64_t* out) {
  if (!ctx || !out) PP_FAIL(PP_ERR_ARG, "pp_ctx_launch_count: NULL argument");
  *out = ctx->launches;
  return PP_OK;
}

pp_status pp_graph_upload(pp_ctx ctx, int64_t n, int64_t row_lo, int64_t row_hi, int64_t nnz,
                          const int64_t* csr_off, const uint32_t* csr_idx, const int64_t* csc_off,
                          const uint32_t* csc_idx, uint32_t flags, pp_graph* out) {
  if (!ctx || !out || !csr_off || (nnz > 0 && !csr_idx))
    PP_FAIL(PP_ERR_ARG, "pp_graph_upload: NULL argument");
  *out = nullptr;
  if (ctx->nranks > 0)
    return upload_block(ctx, n, row_lo, row_hi, nnz, csr_off, csr_idx, csc_off, csc_idx, flags, out);
  if (row_lo != 0 || row_hi != n)
    PP_FAIL(PP_ERR_ARG, "pp_graph_upload: rows [%lld, %lld) on a single-GPU context (must be [0, n))",
            (long long)row_lo, (long long)row_hi);
  const bool symmetric = (flags & PP_GRAPH_SYMMETRIC) != 0;
  if (!symmetric && (!csc_off || (nnz > 0 && !csc_idx)))
    PP_FAIL(PP_ERR_ARG, "pp_graph_upload: CSC required unless PP_GRAPH_SYMMETRIC");
  if (symmetric) {
    csc_off = csr_off;
    csc_idx = csr_idx;
  }
  if (n < 1 || n >= (int64_t)0xFFFFFFFFll)
    PP_FAIL(PP_ERR_UNSUPPORTED, "pp_graph_upload: n=%lld outside [1, 2^32-1)", (long long)n);
  if (nnz < 0) PP_FAIL(PP_ERR_ARG, "pp_graph_upload: nnz < 0");
  PP_CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = ctx->stream;

  pp_graph g = new pp_graph_s;
  Guard guard{g};
  g->ctx = ctx;
  g->n = n;
  g->nnz = nnz;
  g->symmetric = symmetric;
  g->off64 = nnz >= (int64_t)0xFFFFFFFFll || (flags & PP_GRAPH_OFF64);
  const int64_t words = (n + 31) / 32;
  g->nwords = (uint32_t)(((words + 31) / 32) * 32);
  int64_t& bytes = g->device_bytes;
  pp_status s;

  // int64 offsets staged on device (host input copied, device input used in place)
  const bool dev = (flags & PP_GRAPH_DEVICE) != 0;
  const int64_t* d_off64 = csr_off;
  const int64_t* d_coff64 = csc_off;
  if (!dev) {
    int64_t junk = 0;
    if ((s = dalloc(&g->dtmp[0], (size_t)(n + 1) * 2, &junk, "offset staging")) != PP_OK) return s;
    PP_CK(cudaMemcpyAsync(g->dtmp[0], csr_off, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st),
          "copy offsets");
    d_off64 = (const int64_t*)g->dtmp[0];
    if (symmetric) {
      d_coff64 = d_off64;
    } else {
      PP_CK(cudaMemcpyAsync((int64_t*)g->dtmp[0] + (n + 1), csc_off, sizeof(int64_t) * (n + 1),
                            cudaMemcpyHostToDevice, st),
            "copy csc offsets");
      d_coff64 = (const int64_t*)g->dtmp[0] + (n + 1);
    }
  }
  // offsets boundary values
  int64_t ends[4];
  PP_CK(cudaMemcpyAsync(&ends[0], d_off64, 8, cudaMemcpyDefault, st), "read off[0]");
  PP_CK(cudaMemcpyAsync(&ends[1], d_off64 + n, 8, cudaMemcpyDefault, st), "read off[n]");
  PP_CK(cudaMemcpyAsync(&ends[2], d_coff64, 8, cudaMemcpyDefault, st), "read coff[0]");
  PP_CK(cudaMemcpyAsync(&ends[3], d_coff64 + n, 8, cudaMemcpyDefault, st), "read coff[n]");
  PP_CK(cudaStreamSynchronize(st), "sync");
  if (ends[0] != 0 || ends[1] != nnz)
    PP_FAIL(PP_ERR_GRAPH, "pp_graph_upload: CSR off[0]=%lld off[n]=%lld, expected 0 and nnz=%lld",
            (long long)ends[0], (long long)ends[1], (long long)nnz);
  if (ends[2] != 0 || ends[3] != nnz)
    PP_FAIL(PP_ERR_GRAPH, "pp_graph_upload: CSC off[0]=%lld off[n]=%lld, expected 0 and nnz=%lld",
            (long long)ends[2], (long long)ends[3], (long long)nnz);

  // column ids
  // ids padded by 8 zero entries: the pull kernel reads aligned 16-byte blocks
  if ((s = dalloc(&g->idx, (size_t)nnz + 8, &bytes, "csr idx")) != PP_OK) return s;
  PP_CK(cudaMemsetAsync(g->idx + nnz, 0, 8 * sizeof(uint32_t), st), "pad idx");
  if (nnz) PP_CK(cudaMemcpyAsync(g->idx, csr_idx, sizeof(uint32_t) * nnz, cudaMemcpyDefault, st), "copy idx");
  if (symmetric) {
    g->cidx = g->idx;
  } else {
    if ((s = dalloc(&g->cidx, (size_t)nnz + 8, &bytes, "csc idx")) != PP_OK) return s;
    PP_CK(cudaMemsetAsync(g->cidx + nnz, 0, 8 * sizeof(uint32_t), st), "pad csc idx");
    if (nnz)
      PP_CK(cudaMemcpyAsync(g->cidx, csc_idx, sizeof(uint32_t) * nnz, cudaMemcpyDefault, st),
            "copy csc idx");
  }
  // small control buffers
  if ((s = dalloc(&g->scount, 8, &bytes, "counters")) != PP_OK) return s;
  PP_CK(cudaMallocHost((void**)&g->scount_host, 8 * sizeof(unsigned long long)), "pinned counters");
  PP_CK(cudaMallocHost((void**)&g->status_host, sizeof(BfsStatus)), "pinned status");

  if (flags & PP_GRAPH_VALIDATE) {
    for (int side = 0; side < (symmetric ? 1 : 2); ++side) {
      PP_CK(cudaMemsetAsync(g->scount, 0xFF, sizeof(unsigned long long), st), "memset");
      PP_CK(launch_graph_validate(g, side ? d_coff64 : d_off64, side ? g->cidx : g->idx, g->scount,
                                  &ctx->launches),
            "validate kernel");
      PP_CK(cudaMemcpyAsync(g->scount_host, g->scount, 8, cudaMemcpyDeviceToHost, st), "copy");
      PP_CK(cudaStreamSynchronize(st), "sync");
      if (g->scount_host[0] != ~0ull)
        PP_FAIL(PP_ERR_GRAPH,
                "pp_graph_upload: %s row %llu is malformed (offsets decrease, an id >= n, or the "
                "row is not strictly increasing)",
                side ? "CSC" : "CSR", (unsigned long long)g->scount_host[0]);
    }
  }

  // optional degree-ordered relabelling (relabel.cu): rows renumbered and re-sorted; the
  // prepare kernels below then see only internal ids
  if (flags & PP_GRAPH_RELABEL) {
    if (nnz >= (int64_t)0x7FFFFFFF || n >= (int64_t)0x7FFFFFFF)
      PP_FAIL(PP_ERR_UNSUPPORTED, "pp_graph_upload: PP_GRAPH_RELABEL needs nnz, n < 2^31");
    if ((s = dalloc(&g->perm, (size_t)n, &bytes, "relabel perm")) != PP_OK) return s;
    if ((s = dalloc(&g->rank, (size_t)n, &bytes, "relabel rank")) != PP_OK) return s;
    if ((s = dalloc(&g->pint, (size_t)n, &bytes, "internal parents")) != PP_OK) return s;
    if (kVrec && (s = dalloc(&g->vrec, (size_t)n, &bytes, "vertex records")) != PP_OK) return s;
    for (int k = 0; k < 4; ++k)
      if ((s = dalloc(&g->rbits[k], g->nwords, &bytes, "relabel scratch bitmap")) != PP_OK) return s;
    int64_t junk = 0;
    int64_t* noff = nullptr;
    if ((s = dalloc(&noff, (size_t)(n + 1) * 2, &junk, "relabel offsets")) != PP_OK) return s;
    const cudaError_t e = launch_relabel(g, d_off64, d_coff64, noff, noff + (n + 1), &ctx->launches);
    if (g->dtmp[0]) cudaFree(g->dtmp[0]);
    g->dtmp[0] = noff;  // freed with the other staging below
    if (e != cudaSuccess) return cuda_fail(e, "relabel");
    d_off64 = noff;
    d_coff64 = symmetric ? noff : noff + (n + 1);
  }

  // narrowed offsets, isolated bitmap, heavy-chunk capacities
  // offsets padded to nwords*32 + 16 entries: the pull kernel loads an item's 257
  // offsets with aligned vector loads (padding rows are never candidates)
  const size_t offb = g->off64 ? 8 : 4;
  const size_t noff = (size_t)g->nwords * 32 + 16;
  {
    void* p = nullptr;
    PP_CK(cudaMalloc(&p, offb * noff), "offsets");
    PP_CK(cudaMemsetAsync(p, 0, offb * noff, st), "memset offsets");
    g->off = p;
    bytes += (int64_t)(offb * noff);
    if (symmetric) {
      g->coff = g->off;
    } else {
      PP_CK(cudaMalloc(&p, offb * noff), "csc offsets");
      PP_CK(cudaMemsetAsync(p, 0, offb * noff, st), "memset csc offsets");
      g->coff = p;
      bytes += (int64_t)(offb * noff);
    }
  }
  if ((s = dalloc(&g->isolated, g->nwords, &bytes, "isolated")) != PP_OK) return s;
  // pull row data: one 32-byte record per row {first 6 in-neighbours, caller id, in-degree},
  // read by the sparse pull per candidate and streamed by the dense pull per bitmap word
  {
    const size_t words = (size_t)g->nwords * 32 * 8;  // 32 B per row incl. padding rows
    if ((s = dalloc(&g->drec, words, &bytes, "dense pull records")) != PP_OK) return s;
    PP_CK(cudaMemsetAsync(g->drec, 0, words * 4, st), "memset dense records");
  }
  PP_CK(cudaMemsetAsync(g->scount, 0, 5 * sizeof(unsigned long long), st), "memset");
  PP_CK(launch_graph_prepare(g, d_off64, d_coff64, g->scount, &ctx->launches), "prepare kernels");
  PP_CK(cudaMemcpyAsync(g->scount_host, g->scount, 40, cudaMemcpyDeviceToHost, st), "copy");
  PP_CK(cudaStreamSynchronize(st), "sync");
  g->hcap = (int64_t)std::max(g->scount_host[0], g->scount_host[1]);
  g->max_out_deg = (int64_t)g->scount_host[2];
  g->n_noniso = (int64_t)g->nwords * 32 - (int64_t)g->scount_host[4];
  if (g->scount_host[3] >= (1ull << 31))  // residual queue: 31-bit remaining lengths
    PP_FAIL(PP_ERR_UNSUPPORTED, "pp_graph_upload: a row of A^T has %llu >= 2^31 entries",
            (unsigned long long)g->scount_host[3]);

  // BFS / mxv working set
  for (int k = 0; k < 2; ++k) {
    if ((s = dalloc(&g->vis[k], g->nwords, &bytes, "visited")) != PP_OK) return s;
    // 16-byte light entries {v, deg, begin} (BFS); mxv reuses it as a uint32 list
    if ((s = dalloc(&g->L[k], (size_t)n * 4, &bytes, "frontier list")) != PP_OK) return s;
    if ((s = dalloc(&g->H[k], (size_t)g->hcap, &bytes, "heavy chunks")) != PP_OK) return s;
  }
  if ((s = dalloc(&g->fr, g->nwords, &bytes, "frontier bitmap")) != PP_OK) return s;
  // visited summary: group size 2^shift >= 8 vertices, at most kSumWordsMax words
  g->sum_shift = 3;
  while (((n + ((int64_t)1 << g->sum_shift) - 1) >> g->sum_shift) > (int64_t)std::max(kSumWordsMax, 1u) * 32)
    ++g->sum_shift;
  g->sum_words = (uint32_t)((((n + ((int64_t)1 << g->sum_shift) - 1) >> g->sum_shift) + 31) / 32);
  if ((s = dalloc(&g->sumv, g->sum_words, &bytes, "visited summary")) != PP_OK) return s;
  if ((s = dalloc(&g->ctr, kRing, &bytes, "level counters")) != PP_OK) return s;
  if ((s = dalloc(&g->gwork, (size_t)kRing * kMaxCtas, &bytes, "work counters")) != PP_OK) return s;
  g->stats_cap = (int)std::min<int64_t>(n + 1, 1 << 16);
  if ((s = dalloc(&g->stats, (size_t)g->stats_cap, &bytes, "level stats")) != PP_OK) return s;
  if ((s = dalloc(&g->bar, 2, &bytes, "barrier")) != PP_OK) return s;  // [bar][status]
  g->status = reinterpret_cast<BfsStatus*>(g->bar + 1);
  for (int k = 0; k < 4; ++k)
    if ((s = dalloc(&g->sbits[k], g->nwords, &bytes, "scratch bitmap")) != PP_OK) return s;
  if ((s = dalloc(&g->sblock, g->nwords / 256 + 1, &bytes, "scan blocks")) != PP_OK) return s;
  // long-row chunk queue of the row mxv: at most 2*nnz/1024 + 1 chunks
  if ((s = dalloc(&g->hubq, (size_t)(2 * (nnz / 1024) + 2), &bytes, "row-mxv hub chunks")) != PP_OK)
    return s;
  PP_CK(cudaMemsetAsync(g->bar, 0, sizeof(GridBarrier) * 2, st), "memset");
  PP_CK(cudaStreamSynchronize(st), "sync");
  if (g->dtmp[0]) {
    cudaFree(g->dtmp[0]);
    g->dtmp[0] = nullptr;
  }
  g->bfs_grid = bfs_grid_size(g, false);
  guard.g = nullptr;
  ctx->refs += 1;
  *out = g;
  return PP_OK;
}

pp_status pp_graph_free(pp_graph g) {
  if (!g) PP_FAIL(PP_ERR_ARG, "pp_graph_free: NULL graph");
  pp_ctx ctx = g->ctx;
  if (ctx->team && ctx->team->graphs[ctx->rank] == g) ctx->team->graphs[ctx->rank] = nullptr;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  free_graph(g);
  ctx_release(ctx);
  return PP_OK;
}

pp_status pp_graph_partition(pp_graph g, int64_t* row_lo, int64_t* row_hi) {
  if (!g || !row_lo || !row_hi) PP_FAIL(PP_ERR_ARG, "pp_graph_partition: NULL argument");
  *row_lo = g->dist ? g->row_lo : 0;
  *row_hi = g->dist ? g->row_hi : g->n;
  return PP_OK;
}

pp_status pp_graph_export(pp_graph g, void* record128) {
  if (!g || !record128 || !g->dist) PP_FAIL(PP_ERR_ARG, "pp_graph_export: NULL or not a multi-rank graph");
  PP_CK(cudaSetDevice(g->ctx->device), "cudaSetDevice");
  BootRec me;
  pp_status s = make_record(g, &me);
  if (s != PP_OK) return s;
  memcpy(record128, &me, sizeof(me));
  return PP_OK;
}

pp_status pp_graph_import(pp_graph g, const void* records) {
  if (!g || !records || !g->dist || g->ctx->team)
    PP_FAIL(PP_ERR_ARG, "pp_graph_import: NULL, not a multi-rank graph, or a team member");
  PP_CK(cudaSetDevice(g->ctx->device), "cudaSetDevice");
  std::vector<BootRec> all((size_t)g->nranks);
  memcpy(all.data(), records, sizeof(BootRec) * (size_t)g->nranks);
  return attach_records(g, all.data());
}

pp_status pp_team_create(int device, void* cuda_stream, int32_t nranks, pp_ctx* ctxs) {
  if (!ctxs || nranks < 1 || nranks > kMaxRanks)
    PP_FAIL(PP_ERR_ARG, "pp_team_create: nranks %d outside [1, %d]", nranks, kMaxRanks);
  pp_team_s* t = new pp_team_s;
  t->device = device;
  t->nranks = nranks;
  for (int r = 0; r < nranks; ++r) {
    pp_status s = pp_ctx_create(device, cuda_stream, &ctxs[r]);
    if (s != PP_OK) {
      for (int q = 0; q < r; ++q) {
        ctxs[q]->team = nullptr;
        delete ctxs[q];
        ctxs[q] = nullptr;
      }
      delete t;
      return s;
    }
    ctxs[r]->rank = r;
    ctxs[r]->nranks = nranks;
    ctxs[r]->team = t;
    t->ctx[r] = ctxs[r];
    t->refs += 1;
  }
  return PP_OK;
}

pp_status pp_graph_info(pp_graph g, int64_t* n, int64_t* nnz, int64_t* device_bytes) {
  if (!g) PP_FAIL(PP_ERR_ARG, "pp_graph_info: NULL graph");
  if (n) *n = g->n;
  if (nnz) *nnz = g->nnz;
  if (device_bytes) *device_bytes = g->device_bytes;
  return PP_OK;
}

pp_status pp_descriptor_default(pp_descriptor* d) {
  if (!d) PP_FAIL(PP_ERR_ARG, "pp_descriptor_default: NULL");
  memset(d, 0, sizeof(*d));
  d->mask = nullptr;
  d->semiring = PP_SR_LOR_LAND;
  d->replace = 1;
  d->direction = PP_DIR_AUTO;
  d->early_exit = 1;
  d->transpose = 1;
  d->want_nnz = 1;
  d->switchpoint = 0.01;
  d->prev_nnz = -1;
  return PP_OK;
}

pp_status pp_bfs_options_default(pp_bfs_options* o) {
  if (!o) PP_FAIL(PP_ERR_ARG, "pp_bfs_options_default: NULL");
  memset(o, 0, sizeof(*o));
  o->heuristic = PP_HEUR_EDGES;
  o->mode = PP_MODE_DO;
  o->alpha = 0;
  o->beta = 0;
  o->want_parents = 0;
  o->toggles = 0;
  return PP_OK;
}

static pp_status check_vec(const pp_vector* v, int64_t n, const char* name) {
  if (!v) PP_FAIL(PP_ERR_ARG, "pp_mxv: %s is NULL", name);
  if (v->n != n) PP_FAIL(PP_ERR_DIM, "pp_mxv: %s has length %lld, graph has n=%lld", name, (long long)v->n, (long long)n);
  if (v->format != PP_VEC_LIST && v->format != PP_VEC_BITMAP)
    PP_FAIL(PP_ERR_DIM, "pp_mxv: %s has unknown format %d", name, v->format);
  if (!v->data && !(v->format == PP_VEC_LIST && v->nnz == 0 && v->capacity == 0))
    PP_FAIL(PP_ERR_ARG, "pp_mxv: %s data is NULL", name);
  if (v->format == PP_VEC_LIST && (v->nnz < 0 || v->nnz > v->capacity))
    PP_FAIL(PP_ERR_DIM, "pp_mxv: %s list nnz=%lld invalid", name, (long long)v->nnz);
  return PP_OK;
}

pp_status pp_mxv(pp_graph g, pp_vector* w, const pp_descriptor* desc, const pp_vector* u) {
  if (!g || !desc) PP_FAIL(PP_ERR_ARG, "pp_mxv: NULL graph or descriptor");
  if (g->dist) PP_FAIL(PP_ERR_UNSUPPORTED, "pp_mxv: multi-rank graphs run pp_bfs only");
  pp_status s;
  if ((s = check_vec(u, g->n, "u")) != PP_OK) return s;
  if ((s = check_vec(w, g->n, "w")) != PP_OK) return s;
  if (desc->semiring != PP_SR_LOR_LAND)
    PP_FAIL(PP_ERR_UNSUPPORTED, "pp_mxv: semiring %d unsupported (Boolean LOR.LAND only)", desc->semiring);
  if (!desc->mask && desc->complement)
    PP_FAIL(PP_ERR_ARG, "pp_mxv: structural complement without a mask");
  if (desc->mask && (s = check_vec(desc->mask, g->n, "mask")) != PP_OK) return s;
  if (desc->direction < PP_DIR_AUTO || desc->direction > PP_DIR_PULL)
    PP_FAIL(PP_ERR_ARG, "pp_mxv: direction %d", desc->direction);
  PP_CK(cudaSetDevice(g->ctx->device), "cudaSetDevice");
  cudaStream_t st = g->ctx->stream;
  unsigned long long* bad = g->scount + 2;
  PP_CK(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), st), "memset");
  const bool need_win = desc->accum || !desc->replace;

  // Convert — AUTO picks the kernel by nnz(u)/n with hysteresis (R25)
  int64_t unnz = u->nnz;
  int pull;
  if (desc->direction == PP_DIR_AUTO) {
    if (unnz < 0) {  // bitmap of unknown count
      PP_CK(launch_popcount(g, (const uint32_t*)u->data, g->scount), "popcount");
      PP_CK(cudaMemcpyAsync(g->scount_host, g->scount, 8, cudaMemcpyDeviceToHost, st), "copy");
      PP_CK(cudaStreamSynchronize(st), "sync");
      unnz = (int64_t)g->scount_host[0];
    }
    const double r = (double)unnz / (double)g->n;
    const int64_t prev = desc->prev_nnz;
    if (u->format == PP_VEC_LIST) pull = (r > desc->switchpoint && (prev < 0 || unnz > prev)) ? 1 : 0;
    else pull = (r < desc->switchpoint && (prev < 0 || unnz < prev)) ? 0 : 1;
  } else {
    pull = desc->direction == PP_DIR_PULL ? 1 : 0;
  }

  MxvPlan p;
  memset(&p, 0, sizeof(p));
  p.pull = pull;
  p.transpose = desc->transpose ? 1 : 0;
  p.complement = desc->complement ? 1 : 0;
  p.accum = desc->accum ? 1 : 0;
  p.replace = desc->replace ? 1 : 0;
  p.early_exit = desc->early_exit ? 1 : 0;
  if (pull) {
    if (u->format == PP_VEC_BITMAP) {
      p.u_bits = (const uint32_t*)u->data;
    } else {
      PP_CK(launch_list_to_bitmap(g, (const uint32_t*)u->data, u->nnz, g->sbits[1], bad), "u list->bitmap");
      p.u_bits = g->sbits[1];
    }
  } else {
    if (u->format == PP_VEC_LIST) {
      p.u_list = (const uint32_t*)u->data;
      p.u_nnz = u->nnz;
    } else {
      p.u_bits = (const uint32_t*)u->data;
    }
  }
  if (desc->mask) {
    if (desc->mask->format == PP_VEC_BITMAP) {
      p.mask_bits = (const uint32_t*)desc->mask->data;
    } else {
      PP_CK(launch_list_to_bitmap(g, (const uint32_t*)desc->mask->data, desc->mask->nnz, g->sbits[2], bad),
            "mask list->bitmap");
      p.mask_bits = g->sbits[2];
    }
  }
  if (w->format == PP_VEC_BITMAP) {
    p.out_bits = (uint32_t*)w->data;
    p.win_bits = (const uint32_t*)w->data;
  } else {
    p.out_bits = g->sbits[3];
    if (need_win) {
      PP_CK(launch_list_to_bitmap(g, (const uint32_t*)w->data, w->nnz, g->sbits[3], bad), "w list->bitmap");
    }
    p.win_bits = g->sbits[3];
  }
  uint32_t* out_caller = p.out_bits;
  if (g->perm) {
    // relabelled graph: every operand as an internal-id bitmap, result mapped back
    const uint32_t* ub = p.u_bits;
    if (!ub) {
      PP_CK(launch_list_to_bitmap(g, p.u_list, p.u_nnz, g->sbits[1], bad), "u list->bitmap");
      ub = g->sbits[1];
    }
    PP_CK(launch_permute_bits(g, ub, true, g->rbits[0]), "permute u");
    p.u_bits = g->rbits[0];
    p.u_list = nullptr;
    p.u_nnz = 0;
    if (p.mask_bits) {
      PP_CK(launch_permute_bits(g, p.mask_bits, true, g->rbits[1]), "permute mask");
      p.mask_bits = g->rbits[1];
    }
    if (need_win) PP_CK(launch_permute_bits(g, p.win_bits, true, g->rbits[2]), "permute w_in");
    p.win_bits = need_win ? g->rbits[2] : g->rbits[3];
    p.out_bits = g->rbits[3];
  }
  PP_CK(launch_mxv(g, p), "mxv kernels");
  if (g->perm) PP_CK(launch_permute_bits(g, g->rbits[3], false, out_caller), "permute w");

  if (w->format == PP_VEC_LIST) {
    PP_CK(launch_bitmap_to_list(g, g->sbits[3], (uint32_t*)w->data, w->capacity, g->scount), "bitmap->list");
  } else if (desc->want_nnz) {
    PP_CK(launch_popcount(g, (const uint32_t*)w->data, g->scount), "popcount");
  }
  if (w->format == PP_VEC_LIST || desc->want_nnz) {
    PP_CK(cudaMemcpyAsync(g->scount_host, g->scount, 24, cudaMemcpyDeviceToHost, st), "copy");
    PP_CK(cudaStreamSynchronize(st), "sync");
    if (g->scount_host[2] != ~0ull)
      PP_FAIL(PP_ERR_RANGE, "pp_mxv: input list entry %llu holds an id >= n or breaks the strictly increasing order",
              (unsigned long long)g->scount_host[2]);
    w->nnz = (int64_t)g->scount_host[0];
    if (w->format == PP_VEC_LIST && w->nnz > w->capacity)
      PP_FAIL(PP_ERR_DIM, "pp_mxv: output list needs %lld entries, capacity %lld", (long long)w->nnz,
              (long long)w->capacity);
  } else {
    w->nnz = -1;
  }
  return PP_OK;
}

// After a BFS launch: optional sync, device status check and the per-level stats.
static pp_status finish_bfs(pp_graph g, pp_bfs_stats* stats, bool sync) {
  cudaStream_t st = g->ctx->stream;
  if (!sync) return PP_OK;
  PP_CK(cudaMemcpyAsync(g->status_host, g->status, sizeof(BfsStatus), cudaMemcpyDeviceToHost, st),
        "copy status");
  PP_CK(cudaStreamSynchronize(st), "bfs sync");
  if (g->status_host->error)
    PP_FAIL((pp_status)g->status_host->error, "pp_bfs: device watchdog fired (barrier wait > 4 s)");
  if (stats) {
    stats->levels = g->status_host->levels;
    stats->init_ns = g->status_host->t_init - g->status_host->t_start;
    stats->reached = g->status_host->reached;
    stats->reached_nnz = g->status_host->reached_nnz;
    stats->exchanged_bytes = g->dist ? g->status_host->xbytes : 0;
    const int m = std::min(std::min(stats->capacity, g->status_host->levels), g->stats_cap);
    if (m > 0) {
      std::vector<LevelStat> hs((size_t)m);
      PP_CK(cudaMemcpy(hs.data(), g->stats, sizeof(LevelStat) * m, cudaMemcpyDeviceToHost), "copy stats");
      for (int k = 0; k < m; ++k) {
        if (stats->ns) stats->ns[k] = hs[k].t_ns - (k ? hs[k - 1].t_ns : g->status_host->t_init);
        if (stats->dir) stats->dir[k] = (int8_t)hs[k].dir;
        if (stats->c) stats->c[k] = hs[k].c;
        if (stats->m_f) stats->m_f[k] = hs[k].m_f;
        if (stats->m_u) stats->m_u[k] = hs[k].m_u;
        if (stats->cand) stats->cand[k] = hs[k].cand;
      }
    }
  }
  return PP_OK;
}

pp_status pp_bfs(pp_graph g, int64_t source, const pp_bfs_options* opts, int32_t* depth,
                 int32_t* parent, pp_bfs_stats* stats) {
  if (!g || !depth) PP_FAIL(PP_ERR_ARG, "pp_bfs: NULL graph or depth");
  if (source < 0 || source >= g->n)
    PP_FAIL(PP_ERR_RANGE, "pp_bfs: source %lld out of range [0, %lld)", (long long)source, (long long)g->n);
  pp_bfs_options o;
  if (opts) o = *opts;
  else pp_bfs_options_default(&o);
  if (o.heuristic != PP_HEUR_EDGES && o.heuristic != PP_HEUR_PAPER_R)
    PP_FAIL(PP_ERR_ARG, "pp_bfs: heuristic %d", o.heuristic);
  if (o.mode < PP_MODE_DO || o.mode > PP_MODE_PULL_ONLY) PP_FAIL(PP_ERR_ARG, "pp_bfs: mode %d", o.mode);
  if (o.toggles & ~7u) PP_FAIL(PP_ERR_ARG, "pp_bfs: unknown toggles 0x%x", o.toggles);
  double alpha = o.alpha, beta = o.beta;
  if (alpha <= 0) alpha = (o.heuristic == PP_HEUR_EDGES) ? 15.0 : 0.01;
  if (beta <= 0) beta = (o.heuristic == PP_HEUR_EDGES) ? 18.0 : 0.01;
  if (!o.want_parents) parent = nullptr;
  PP_CK(cudaSetDevice(g->ctx->device), "cudaSetDevice");
  cudaStream_t st = g->ctx->stream;

  // Host outputs (end-to-end path): compute into device staging, copy back in the call.
  const bool host_depth = !is_device_ptr(depth);
  const bool host_parent = parent && !is_device_ptr(parent);
  int32_t* d_depth = depth;
  uint32_t* d_parent = (uint32_t*)parent;
  pp_status s;
  if (host_depth) {
    if (!g->dtmp[0] && (s = dalloc(&g->dtmp[0], (size_t)(g->n + 1) / 2 + 1, &g->device_bytes, "depth staging")) != PP_OK)
      return s;
    d_depth = (int32_t*)g->dtmp[0];
  }
  if (host_parent) {
    if (!g->dtmp[1] && (s = dalloc(&g->dtmp[1], (size_t)(g->n + 1) / 2 + 1, &g->device_bytes, "parent staging")) != PP_OK)
      return s;
    d_parent = (uint32_t*)g->dtmp[1];
  }
  if (g->dist && o.toggles)
    PP_FAIL(PP_ERR_UNSUPPORTED, "pp_bfs: ablation toggles are single-GPU only");
  if (g->dist && g->ctx->team)
    PP_FAIL(PP_ERR_ARG, "pp_bfs: a team member's graph runs through pp_bfs_team");
  if (g->dist && !g->attached)
    PP_FAIL(PP_ERR_ARG, "pp_bfs: the peers' exchange buffers are not mapped (pp_graph_import)");
  if (g->dist) {  // collective 1D-partitioned BFS; depth/parent are the block's slices
    PP_CK(cudaMemsetAsync(g->bar, 0, sizeof(GridBarrier) + sizeof(BfsStatus), st), "memset control");
    uint32_t* pp_ = (uint32_t*)d_parent;
    PP_CK(launch_bfs_ranks(&g, 1, (uint32_t)source, o.mode, o.heuristic, alpha, beta, &d_depth,
                           pp_ ? &pp_ : nullptr),
          "bfs kernel launch");
    const int64_t len = g->row_hi - g->row_lo;
    if (host_depth && len)
      PP_CK(cudaMemcpyAsync(depth, d_depth, sizeof(int32_t) * len, cudaMemcpyDeviceToHost, st), "copy");
    if (host_parent && len)
      PP_CK(cudaMemcpyAsync(parent, d_parent, sizeof(int32_t) * len, cudaMemcpyDeviceToHost, st), "copy");
    return finish_bfs(g, stats, stats || host_depth || host_parent);
  }
  PP_CK(cudaMemsetAsync(g->bar, 0, sizeof(GridBarrier) + sizeof(BfsStatus), st), "memset control");
  const int max_levels = (int)std::min<int64_t>(g->n + 1, 0x7FFFFFFF);
  PP_CK(launch_bfs(g, (uint32_t)source, o.mode, o.heuristic, alpha, beta, o.toggles, d_depth, d_parent,
                   max_levels),
        "bfs kernel launch");
  if (host_depth)
    PP_CK(cudaMemcpyAsync(depth, d_depth, sizeof(int32_t) * g->n, cudaMemcpyDeviceToHost, st), "copy depth");
  if (host_parent)
    PP_CK(cudaMemcpyAsync(parent, d_parent, sizeof(int32_t) * g->n, cudaMemcpyDeviceToHost, st), "copy parent");
  return finish_bfs(g, stats, stats || host_depth || host_parent);
}

pp_status pp_bfs_team(const pp_graph* graphs, int32_t nranks, int64_t source,
                      const pp_bfs_options* opts, int32_t* const* depth, int32_t* const* parent,
                      pp_bfs_stats* stats) {
  if (!graphs || !depth || nranks < 1 || nranks > kMaxRanks)
    PP_FAIL(PP_ERR_ARG, "pp_bfs_team: NULL argument or nranks %d outside [1, %d]", nranks, kMaxRanks);
  pp_team_s* team = nullptr;
  for (int r = 0; r < nranks; ++r) {
    pp_graph g = graphs[r];
    if (!g || !g->dist || !g->ctx->team || g->ctx->rank != r || !depth[r])
      PP_FAIL(PP_ERR_ARG, "pp_bfs_team: graphs[%d] is not rank %d of a team (or depth[%d] is NULL)", r, r, r);
    if (r == 0) team = g->ctx->team;
    if (g->ctx->team != team || team->nranks != nranks || g->n != graphs[0]->n ||
        g->off64 != graphs[0]->off64 || g->symmetric != graphs[0]->symmetric)
      PP_FAIL(PP_ERR_ARG, "pp_bfs_team: graphs[%d] belongs to another team or graph", r);
    if (!is_device_ptr(depth[r]) || (parent && parent[r] && !is_device_ptr(parent[r])))
      PP_FAIL(PP_ERR_ARG, "pp_bfs_team: depth / parent slices must be device memory");
  }
  pp_graph g0 = graphs[0];
  if (source < 0 || source >= g0->n)
    PP_FAIL(PP_ERR_RANGE, "pp_bfs_team: source %lld out of range [0, %lld)", (long long)source, (long long)g0->n);
  pp_bfs_options o;
  if (opts) o = *opts;
  else pp_bfs_options_default(&o);
  if (o.heuristic != PP_HEUR_EDGES && o.heuristic != PP_HEUR_PAPER_R)
    PP_FAIL(PP_ERR_ARG, "pp_bfs_team: heuristic %d", o.heuristic);
  if (o.mode < PP_MODE_DO || o.mode > PP_MODE_PULL_ONLY) PP_FAIL(PP_ERR_ARG, "pp_bfs_team: mode %d", o.mode);
  if (o.toggles) PP_FAIL(PP_ERR_UNSUPPORTED, "pp_bfs_team: ablation toggles are single-GPU only");
  double alpha = o.alpha, beta = o.beta;
  if (alpha <= 0) alpha = (o.heuristic == PP_HEUR_EDGES) ? 15.0 : 0.01;
  if (beta <= 0) beta = (o.heuristic == PP_HEUR_EDGES) ? 18.0 : 0.01;
  const bool want_parents = o.want_parents && parent;
  // the peers' exchange buffers are on this device: map them directly
  const XLayout L = xlayout(g0->nwords);
  int64_t in_total = 0, noniso = 0;
  for (int r = 0; r < nranks; ++r) {
    in_total += graphs[r]->nnz;
    noniso += graphs[r]->n_noniso_block;
  }
  for (int r = 0; r < nranks; ++r) {
    for (int q = 0; q < nranks; ++q) set_peer(graphs[r], q, (char*)graphs[q]->xbuf, L);
    graphs[r]->in_total = in_total;
    graphs[r]->n_noniso = noniso;
  }
  PP_CK(cudaSetDevice(g0->ctx->device), "cudaSetDevice");
  cudaStream_t st = g0->ctx->stream;
  for (int r = 0; r < nranks; ++r)
    PP_CK(cudaMemsetAsync(graphs[r]->bar, 0, sizeof(GridBarrier) + sizeof(BfsStatus), st), "memset control");
  std::vector<pp_graph> gs(graphs, graphs + nranks);
  PP_CK(launch_bfs_ranks(gs.data(), nranks, (uint32_t)source, o.mode, o.heuristic, alpha, beta, depth,
                         want_parents ? (uint32_t* const*)parent : nullptr),
        "bfs kernel launch");
  for (int r = 1; r < nranks; ++r) {  // every rank's status (each has its own watchdog)
    pp_status s = finish_bfs(graphs[r], nullptr, true);
    if (s != PP_OK) return s;
  }
  pp_status s = finish_bfs(g0, stats, true);
  if (s != PP_OK) return s;
  for (int r = 1; r < nranks; ++r)
    if (graphs[r]->status_host->levels != g0->status_host->levels ||
        graphs[r]->status_host->reached != g0->status_host->reached)
      PP_FAIL(PP_ERR_CUDA, "pp_bfs_team: ranks disagree (levels %d vs %d)", graphs[r]->status_host->levels,
              g0->status_host->levels);
  return PP_OK;
}

pp_status pp_bfs_debug_phases(pp_graph g, int64_t* out_ns) {
  if (!g || !out_ns || !g->dbg) PP_FAIL(PP_ERR_ARG, "pp_bfs_debug_phases: NULL or not enabled");
  PP_CK(cudaSetDevice(g->ctx->device), "cudaSetDevice");
  PP_CK(cudaStreamSynchronize(g->ctx->stream), "sync");
  PP_CK(cudaMemcpy(out_ns, g->dbg, sizeof(long long) * (size_t)g->dbg_levels * g->bfs_grid * 3,
                   cudaMemcpyDeviceToHost), "copy debug phases");
  return PP_OK;
}

pp_status pp_bfs_debug_level(pp_graph g, int64_t source, int32_t level, const pp_bfs_options* opts,
                             int32_t* depth) {
  if (!g || !depth || level < 1) PP_FAIL(PP_ERR_ARG, "pp_bfs_debug_level: NULL graph/depth or level < 1");
  if (g->dist) PP_FAIL(PP_ERR_UNSUPPORTED, "pp_bfs_debug_level: single-GPU graphs only");
  if (source < 0 || source >= g->n)
    PP_FAIL(PP_ERR_RANGE, "pp_bfs_debug_level: source %lld out of range", (long long)source);
  if (!is_device_ptr(depth)) PP_FAIL(PP_ERR_ARG, "pp_bfs_debug_level: depth must be device memory");
  pp_bfs_options o;
  if (opts) o = *opts;
  else pp_bfs_options_default(&o);
  if (o.toggles & ~7u) PP_FAIL(PP_ERR_ARG, "pp_bfs_debug_level: unknown toggles 0x%x", o.toggles);
  double alpha = o.alpha, beta = o.beta;
  if (alpha <= 0) alpha = (o.heuristic == PP_HEUR_EDGES) ? 15.0 : 0.01;
  if (beta <= 0) beta = (o.heuristic == PP_HEUR_EDGES) ? 18.0 : 0.01;
  PP_CK(cudaSetDevice(g->ctx->device), "cudaSetDevice");
  cudaStream_t st = g->ctx->stream;
  PP_CK(cudaMemsetAsync(g->bar, 0, sizeof(GridBarrier) + sizeof(BfsStatus), st), "memset control");
  const int max_levels = (int)std::min<int64_t>(g->n + 1, 0x7FFFFFFF);
  PP_CK(launch_bfs(g, (uint32_t)source, o.mode, o.heuristic, alpha, beta, o.toggles, depth, nullptr,
                   max_levels, level),
        "bfs kernel launch");
  return finish_bfs(g, nullptr, true);
}

pp_status pp_bfs_debug_times(pp_graph g, int32_t levels, int64_t* out_ns, int32_t* nctas) {
  if (!g) PP_FAIL(PP_ERR_ARG, "pp_bfs_debug_times: NULL graph");
  if (g->dist) PP_FAIL(PP_ERR_UNSUPPORTED, "pp_bfs_debug_times: single-GPU graphs only");
  PP_CK(cudaSetDevice(g->ctx->device), "cudaSetDevice");
  if (nctas) *nctas = g->bfs_grid;
  if (levels > 0 && !g->dbg) {
    pp_status s = dalloc(&g->dbg, (size_t)levels * g->bfs_grid * 3, &g->device_bytes, "debug times");
    if (s != PP_OK) return s;
    PP_CK(cudaMemset(g->dbg, 0, sizeof(long long) * (size_t)levels * g->bfs_grid * 3), "memset");
    g->dbg_levels = levels;
    return PP_OK;
  }
  if (out_ns && g->dbg) {
    PP_CK(cudaStreamSynchronize(g->ctx->stream), "sync");
    PP_CK(cudaMemcpy(out_ns, g->dbg, sizeof(long long) * (size_t)g->dbg_levels * g->bfs_grid,
                     cudaMemcpyDeviceToHost), "copy debug times");
  }
  return PP_OK;
}

}  // extern "C"
