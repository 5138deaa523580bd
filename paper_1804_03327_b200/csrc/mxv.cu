// mxv.cu — stand-alone masked Boolean matvec GrB_mxv and the
// sparse<->dense vector conversions (Sparse2dense / Dense2sparse).
//
//   row-based (PULL, Alg. 2 / Eq. 2, 4):  rows with pass(i) only (masking); each row
//       folds OR over its entries and stops at the first true term when early_exit
//       (legal because the semiring's add is OR).  The warp owning a bitmap
//       word writes w directly: no atomics, accumulate/replace fused.
//   column-based (PUSH, Alg. 3 / Eq. 3, 5): the rows of the transposed operator of
//       every u(j) != 0 are expanded load-balanced (light vertices by a warp scan,
//       heavy ones as fixed-size chunks); the mask filter is applied before the
//       OR-merge, which is an atomicOr into a scratch bitmap t; a combine pass applies
//       accumulate / replace.  Output order is by construction sorted (bitmap scan).
#include "pp_device.cuh"

namespace pp {

constexpr int kGridPerSM = 4;
#ifndef PP_STREAM_U
#define PP_STREAM_U 8
#endif
constexpr int kStreamU = PP_STREAM_U;  // row mxv without early exit: id loads in flight per lane
constexpr unsigned kHubIds = 1024;  // row-mxv rows with more ids left go to k_mxv_pull_hubs

static int grid_blocks(pp_graph g) { return g->ctx->num_sms * kGridPerSM; }

__device__ __forceinline__ uint32_t valid_bits(int64_t n, uint32_t w) {
  const int64_t lo = (int64_t)w * 32;
  if (lo + 32 <= n) return 0xFFFFFFFFu;
  if (lo >= n) return 0u;
  return (1u << (unsigned)(n - lo)) - 1u;
}

__device__ __forceinline__ uint32_t pass_word(const uint32_t* mask, int complement, int64_t n,
                                              uint32_t w) {
  const uint32_t vb = valid_bits(n, w);
  if (!vb) return 0u;  // beyond ceil(n/32): never touch caller buffers there
  uint32_t p = mask ? mask[w] : 0xFFFFFFFFu;
  if (complement) p = ~p;
  return p & vb;
}

// ---------------------------------------------------------------------------- conversions --

__global__ void k_list_to_bitmap(const uint32_t* __restrict__ list, int64_t m,
                                 uint32_t* __restrict__ bits, int64_t n,
                                 unsigned long long* bad) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = list[k];
    if ((int64_t)x >= n || (k > 0 && list[k - 1] >= x)) {  // id range; sorted unique (R15)
      atomicMin(bad, (unsigned long long)k);
      continue;
    }
    atomicOr(&bits[x >> 5], 1u << (x & 31u));
  }
}

__global__ void k_popcount(const uint32_t* __restrict__ bits, uint32_t nwords,
                           unsigned long long* out) {
  unsigned long long c = 0;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += gridDim.x * blockDim.x)
    c += __popc(bits[w]);
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(out, c);
}

// Dense2sparse (sorted): 1) per-block popcounts, 2) exclusive scan of the block sums
// in one CTA, 3) each block re-scans its words and writes ascending ids.
constexpr int kB2LWords = kBlock;  // words per block

__global__ void k_b2l_count(const uint32_t* __restrict__ bits, uint32_t nwords,
                            uint32_t* __restrict__ bsum) {
  __shared__ unsigned s[kWarps];
  const uint32_t w = blockIdx.x * kB2LWords + threadIdx.x;
  unsigned c = w < nwords ? __popc(bits[w]) : 0u;
  c = warp_sum(c);
  if (lane_id() == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int i = 0; i < kWarps; ++i) t += s[i];
    bsum[blockIdx.x] = t;
  }
}

__global__ void k_b2l_scan(uint32_t* __restrict__ bsum, uint32_t nblk,
                           unsigned long long* total) {
  __shared__ unsigned long long s[32];  // launched with 1024 threads
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < nblk; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const unsigned v = i < nblk ? bsum[i] : 0u;
    unsigned incl = warp_incl_scan(v);
    if (lane_id() == 31) s[threadIdx.x >> 5] = incl;
    __syncthreads();
    unsigned long long wpre = 0;
    for (unsigned k = 0; k < (threadIdx.x >> 5); ++k) wpre += s[k];
    const unsigned long long excl = carry + wpre + incl - v;
    __syncthreads();
    if (i < nblk) bsum[i] = (uint32_t)excl;  // exclusive prefix (fits: ids < 2^32)
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void k_b2l_write(const uint32_t* __restrict__ bits, uint32_t nwords,
                            const uint32_t* __restrict__ boff, uint32_t* __restrict__ list,
                            int64_t capacity) {
  __shared__ unsigned s[kWarps];
  const uint32_t w = blockIdx.x * kB2LWords + threadIdx.x;
  uint32_t word = w < nwords ? bits[w] : 0u;
  const unsigned c = __popc(word);
  const unsigned incl = warp_incl_scan(c);
  if (lane_id() == 31) s[threadIdx.x >> 5] = incl;
  __syncthreads();
  unsigned wpre = 0;
  for (unsigned k = 0; k < (threadIdx.x >> 5); ++k) wpre += s[k];
  uint64_t pos = (uint64_t)boff[blockIdx.x] + wpre + incl - c;
  while (word) {
    const unsigned b = __ffs(word) - 1;
    word &= word - 1;
    if ((int64_t)pos < capacity) list[pos] = w * 32u + b;
    ++pos;
  }
}

// ---------------------------------------------------------------------------- row-based ----

template <typename Off>
__global__ void __launch_bounds__(kBlock) k_mxv_pull(
    int64_t n, uint32_t nwords, const Off* __restrict__ roff, const uint32_t* __restrict__ ridx,
    const uint32_t* __restrict__ ubits, const uint32_t* __restrict__ mask, int complement,
    int accum, int replace, int early_exit, const uint32_t* win, uint32_t* out, uint4* hubq,
    unsigned* nhub) {
  __shared__ uint32_t st[kWarps][32];
  uint32_t* tword = st[threadIdx.x >> 5];
  const unsigned lane = lane_id();
  const unsigned nchunks = nwords / 32u;
  const unsigned wstride = gridDim.x * kWarps;
  for (unsigned item = blockIdx.x * kWarps + (threadIdx.x >> 5); item < nchunks; item += wstride) {
    const uint32_t w = item * 32u + lane;
    const uint32_t pass = pass_word(mask, complement, n, w);
    tword[lane] = 0u;
    __syncwarp();
    const unsigned cnt = __popc(pass);
    const unsigned incl = warp_incl_scan(cnt);
    const unsigned excl = incl - cnt;
    const unsigned tot = __shfl_sync(kFull, incl, 31);
    for (unsigned base = 0; base < tot; base += 32) {
      const unsigned k = base + lane;
      const bool valid = k < tot;
      const unsigned j = warp_owner(incl, k);
      const uint32_t mj = __shfl_sync(kFull, pass, j);
      const unsigned xj = __shfl_sync(kFull, excl, j);
      const unsigned bitpos = valid ? nth_set_bit(mj, k - xj) : 0u;
      const uint32_t i = (item * 32u + j) * 32u + bitpos;
      Off p = 0, e = 0;
      bool t = false;
      if (valid) {
        p = roff[i];
        e = roff[i + 1];
        const Off lim = min(e, (p | (Off)7) + 1);
        uint32_t x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = (p + q < lim) ? ridx[p + q] : 0u;
#pragma unroll
        for (int q = 0; q < 8; ++q) t = t || ((p + q < lim) && bit_test(ubits, x[q]));
        p = lim;
      }
      const bool deferred = valid && p < e && !(t && early_exit);
      unsigned dm = __ballot_sync(kFull, deferred);
      while (dm) {
        const unsigned l = __ffs(dm) - 1;
        dm &= dm - 1;
        const Off pb = __shfl_sync(kFull, p, l), pe = __shfl_sync(kFull, e, l);
        bool f = false;
        if (!early_exit && pe - pb > (Off)kHubIds) {
          // long row: split into kHubIds-id chunks for k_mxv_pull_hubs (the whole grid);
          // its bit is OR-ed into `out` there (exact: OR is idempotent and commutative)
          const uint32_t il = __shfl_sync(kFull, i, l);
          const unsigned nch = (unsigned)((pe - pb + (Off)kHubIds - 1) / (Off)kHubIds);
          unsigned base = 0;
          if (lane == 0) base = atomicAdd(nhub, nch);
          base = __shfl_sync(kFull, base, 0);
          for (unsigned c = lane; c < nch; c += 32) {
            const Off st = pb + (Off)c * (Off)kHubIds;
            const Off len = min((Off)kHubIds, pe - st);
            hubq[base + c] = make_uint4(il, (uint32_t)len, (uint32_t)st,
                                        (uint32_t)((unsigned long long)st >> 32));
          }
          continue;
        }
        for (Off q0 = pb; q0 < pe; q0 += 128) {
          bool h = false;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const Off q = q0 + (Off)(s * 32) + lane;
            h = h || (q < pe && bit_test(ubits, ridx[q]));
          }
          f = __any_sync(kFull, h) || f;
          if (f && early_exit) break;
        }
        if (lane == l) t = t || f;
      }
      if (valid && t) atomicOr(&tword[j], 1u << bitpos);
    }
    __syncwarp();
    if ((int64_t)w * 32 < n) {
      const uint32_t tw = tword[lane];
      const uint32_t wi = (accum || !replace) ? win[w] : 0u;
      const uint32_t z = accum ? (wi | tw) : tw;
      const uint32_t keep = replace ? 0u : wi;
      out[w] = ((pass & z) | (~pass & keep)) & valid_bits(n, w);
    }
    __syncwarp();
  }
}

// Row-based mxv WITHOUT early exit (Eq. 2 / Eq. 4 evaluated in full): every passing row's
// ids must be read.  Warp item = ONE 32-row bitmap word (so every warp of the grid has work:
// n/32 items), its passing rows' ids streamed as one packed, warp-balanced sequence (warp
// scan of the degrees, kStreamU coalesced id loads per lane in flight per step), hits OR-ed
// per row by a warp reduction; the next item's pass word and offsets are loaded while the
// current one streams (one dependent step less per item).  Rows longer than kHubIds go to
// k_mxv_pull_hubs.  (Round 1's item of 32 words processed them one after another on only
// n/1024 warps: a 32-deep chain per warp, 14% of the copy peak.)
template <typename Off>
__global__ void __launch_bounds__(kBlock) k_mxv_pull_stream(
    int64_t n, uint32_t nwords, const Off* __restrict__ roff, const uint32_t* __restrict__ ridx,
    const uint32_t* __restrict__ ubits, const uint32_t* __restrict__ mask, int complement,
    int accum, int replace, const uint32_t* win, uint32_t* out, uint4* hubq, unsigned* nhub) {
  const unsigned lane = lane_id();
  const unsigned wstride = gridDim.x * kWarps;
  unsigned w = blockIdx.x * kWarps + (threadIdx.x >> 5);
  // item state one step ahead: pass word (all lanes), row offsets (lane = row)
  auto load = [&](unsigned wn, uint32_t& pass, Off& b, Off& e) {
    pass = 0u;
    b = e = 0;
    if (wn < nwords) {
      pass = pass_word(mask, complement, n, wn);
      if ((pass >> lane) & 1u) {
        const uint32_t i = wn * 32u + lane;
        b = roff[i];
        e = roff[i + 1];
      }
    }
  };
  uint32_t pass_n;
  Off b_n, e_n;
  load(w, pass_n, b_n, e_n);
  for (; w < nwords; w += wstride) {
    const uint32_t pass = pass_n;
    const Off b = b_n, e = e_n;
    load(w + wstride, pass_n, b_n, e_n);
    const uint32_t i = w * 32u + lane;
    const bool mine = (pass >> lane) & 1u;
    uint32_t t = 0;
    if (pass) {
      const bool hub = mine && (e - b) > (Off)kHubIds;
      const unsigned hm = __ballot_sync(kFull, hub);
      if (hm) {  // hub rows: chunks for the grid-wide kernel
        const unsigned nch = hub ? (unsigned)((e - b + (Off)kHubIds - 1) / (Off)kHubIds) : 0u;
        const unsigned incl = warp_incl_scan(nch);
        const unsigned tot = __shfl_sync(kFull, incl, 31);
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(nhub, tot);
        base = __shfl_sync(kFull, base, 0) + incl - nch;
        for (unsigned c = 0; c < nch; ++c) {
          const Off st = b + (Off)c * (Off)kHubIds;
          const Off len = min((Off)kHubIds, e - st);
          hubq[base + c] = make_uint4(i, (uint32_t)len, (uint32_t)st,
                                      (uint32_t)((unsigned long long)st >> 32));
        }
      }
      const unsigned deg = (mine && !hub) ? (unsigned)(e - b) : 0u;
      const unsigned incl = warp_incl_scan(deg);
      const unsigned excl = incl - deg;
      const unsigned tot = __shfl_sync(kFull, incl, 31);
      // kStreamU coalesced id loads per lane in flight per step, then their probes
      for (unsigned base = 0; base < tot; base += 32u * kStreamU) {
        uint32_t x[kStreamU];
        unsigned jj[kStreamU];
        bool ok[kStreamU];
#pragma unroll
        for (int s2 = 0; s2 < kStreamU; ++s2) {
          const unsigned q = base + (unsigned)s2 * 32u + lane;
          const unsigned j = warp_owner(incl, q);
          const Off bj = __shfl_sync(kFull, b, j);
          const unsigned xj = __shfl_sync(kFull, excl, j);
          jj[s2] = j;
          ok[s2] = q < tot;
          x[s2] = ok[s2] ? ridx[bj + (Off)(q - xj)] : 0u;
        }
#pragma unroll
        for (int s2 = 0; s2 < kStreamU; ++s2) {
          const bool hit = ok[s2] && bit_test(ubits, x[s2]);
          t |= __reduce_or_sync(kFull, hit ? (1u << jj[s2]) : 0u);
        }
      }
    }
    if (lane == 0) {
      const uint32_t wi = (accum || !replace) ? win[w] : 0u;
      const uint32_t z = accum ? (wi | t) : t;
      const uint32_t keep = replace ? 0u : wi;
      out[w] = ((pass & z) | (~pass & keep)) & valid_bits(n, w);
    }
  }
}

// Long rows of k_mxv_pull, kHubIds ids per chunk, spread over the whole grid (warp per chunk,
// 128 ids per step, ballot early exit inside the chunk).
template <typename Off>
__global__ void __launch_bounds__(kBlock) k_mxv_pull_hubs(const uint4* __restrict__ hubq,
                                                         const unsigned* __restrict__ nhub,
                                                         const uint32_t* __restrict__ ridx,
                                                         const uint32_t* __restrict__ ubits,
                                                         int early_exit, uint32_t* out) {
  const unsigned lane = lane_id();
  const unsigned total = *nhub;
  for (unsigned c = blockIdx.x * kWarps + (threadIdx.x >> 5); c < total; c += gridDim.x * kWarps) {
    const uint4 h = hubq[c];
    const Off st = (Off)(((unsigned long long)h.w << 32) | h.z), en = st + (Off)h.y;
    bool f = false;
    for (Off q0 = st; q0 < en; q0 += 128) {
      bool hit = false;
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        const Off q = q0 + (Off)(s2 * 32) + lane;
        hit = hit || (q < en && bit_test(ubits, ridx[q]));
      }
      f = __any_sync(kFull, hit) || f;
      if (f && early_exit) break;
    }
    if (f && lane == 0) atomicOr(&out[h.x >> 5], 1u << (h.x & 31u));
  }
}

// ---------------------------------------------------------------------------- column-based -

// Split the frontier u (a list, or a bitmap when list == nullptr) into light vertices and
// heavy chunks of kChunk edges of the expanded operator rows (roff).
template <typename Off>
__global__ void __launch_bounds__(kBlock) k_classify(int64_t n, const uint32_t* __restrict__ list, int64_t m,
                                                    const uint32_t* __restrict__ bits,
                                                    uint32_t nwords, const Off* __restrict__ roff,
                                                    uint32_t* L, uint2* H, LevelCtr* ctr,
                                                    unsigned long long* bad) {
  const unsigned lane = lane_id();
  const int64_t nitems = list ? (m + 31) / 32 : (n + 31) / 32;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  for (int64_t item = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); item < nitems;
       item += wstride) {
    uint32_t pending = 0;
    uint32_t single = 0;
    bool has_single = false;
    if (list) {
      const int64_t k = item * 32 + lane;
      if (k < m) {
        single = list[k];
        has_single = (int64_t)single < n;
        // the same PP_ERR_RANGE as the pull side's list->bitmap, and a duplicate or unsorted
        // id (which would overflow the chunk buffers) is rejected too
        if (!has_single || (k > 0 && list[k - 1] >= single)) {
          has_single = false;
          atomicMin(bad, (unsigned long long)k);
        }
      }
    } else {
      pending = bits[item];  // word `item`: lane b takes vertex item*32+b
    }
    // bitmap mode: the warp processes one word; lane b takes bit b
    if (!list) {
      single = (uint32_t)item * 32u + lane;
      has_single = ((pending >> lane) & 1u) && (int64_t)single < n;
    }
    Off deg = 0;
    if (has_single) deg = roff[single + 1] - roff[single];
    const bool heavy = has_single && deg >= (Off)kHeavy;
    const bool light = has_single && deg > 0 && !heavy;
    const unsigned lm = __ballot_sync(kFull, light);
    if (lm) {
      const unsigned leader = __ffs(lm) - 1;
      unsigned base = 0;
      if (lane == leader) base = atomicAdd(&ctr->nL, (unsigned)__popc(lm));
      base = __shfl_sync(kFull, base, leader);
      if (light) L[base + __popc(lm & lanemask_lt())] = single;
    }
    const unsigned hm = __ballot_sync(kFull, heavy);
    if (hm) {
      const unsigned nch = heavy ? (unsigned)((deg + (Off)kChunk - 1) / (Off)kChunk) : 0u;
      const unsigned incl = warp_incl_scan(nch);
      const unsigned excl = incl - nch;
      const unsigned tot = __shfl_sync(kFull, incl, 31);
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(&ctr->nH, tot);
      base = __shfl_sync(kFull, base, 0);
      for (unsigned c0 = 0; c0 < tot; c0 += 32) {  // 32 descriptors per step
        const unsigned c = c0 + lane;
        const unsigned j = warp_owner(incl, c);
        const uint32_t vj = __shfl_sync(kFull, single, j);
        const unsigned xj = __shfl_sync(kFull, excl, j);
        if (c < tot) H[base + c] = make_uint2(vj, c - xj);
      }
    }
  }
}

__device__ __forceinline__ void push_or(uint32_t* t, const uint32_t* mask, int complement,
                                        bool valid, uint32_t x) {
  if (!valid) return;
  const uint32_t wi = x >> 5, bit = 1u << (x & 31u);
  if (mask) {
    const bool m = (mask[wi] & bit) != 0;
    if (m == (complement != 0)) return;  // filtered by the mask (Alg. 3 lines 17-24)
  }
  if (!(t[wi] & bit)) atomicOr(&t[wi], bit);
}

template <typename Off>
__global__ void __launch_bounds__(kBlock) k_mxv_push(const Off* __restrict__ roff,
                                                    const uint32_t* __restrict__ ridx,
                                                    const uint32_t* L, const uint2* H,
                                                    LevelCtr* ctr, const uint32_t* mask,
                                                    int complement, uint32_t* t) {
  const unsigned lane = lane_id();
  const unsigned nL = ld_relaxed_u32(&ctr->nL), nH = ld_relaxed_u32(&ctr->nH);
  const unsigned total = nH + (nL + 31u) / 32u;
  for (;;) {
    const unsigned item = warp_grab(&ctr->work);
    if (item >= total) break;
    if (item < nH) {
      const uint2 h = H[item];
      const Off b = roff[h.x] + (Off)h.y * (Off)kChunk;
      const Off e = min(roff[h.x + 1], b + (Off)kChunk);
      for (Off p = b + lane; p < e; p += 32) push_or(t, mask, complement, true, ridx[p]);
    } else {
      const unsigned i = (item - nH) * 32u + lane;
      Off b = 0;
      unsigned deg = 0;
      if (i < nL) {
        const uint32_t u = L[i];
        b = roff[u];
        deg = (unsigned)(roff[u + 1] - b);
      }
      const unsigned incl = warp_incl_scan(deg);
      const unsigned excl = incl - deg;
      const unsigned tot = __shfl_sync(kFull, incl, 31);
      for (unsigned base = 0; base < tot; base += 32) {
        const unsigned e = base + lane;
        const unsigned j = warp_owner(incl, e);
        const Off bj = __shfl_sync(kFull, b, j);
        const unsigned xj = __shfl_sync(kFull, excl, j);
        const bool valid = e < tot;
        push_or(t, mask, complement, valid, valid ? ridx[bj + (Off)(e - xj)] : 0u);
      }
    }
  }
}

__global__ void k_combine(int64_t n, uint32_t nwords, const uint32_t* __restrict__ t,
                          const uint32_t* __restrict__ mask, int complement, int accum,
                          int replace, const uint32_t* win, uint32_t* out) {
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += gridDim.x * blockDim.x) {
    const uint32_t pass = pass_word(mask, complement, n, w);
    const uint32_t tw = t[w];
    const uint32_t wi = (accum || !replace) ? win[w] : 0u;
    const uint32_t z = accum ? (wi | tw) : tw;
    const uint32_t keep = replace ? 0u : wi;
    out[w] = ((pass & z) | (~pass & keep)) & valid_bits(n, w);
  }
}

// ---------------------------------------------------------------------------- launchers ----

static uint32_t uwords(pp_graph g) { return (uint32_t)((g->n + 31) / 32); }

cudaError_t launch_list_to_bitmap(pp_graph g, const uint32_t* list, int64_t m, uint32_t* bits,
                                  unsigned long long* d_bad) {
  cudaStream_t st = g->ctx->stream;
  cudaError_t e = cudaMemsetAsync(bits, 0, sizeof(uint32_t) * uwords(g), st);
  if (e != cudaSuccess || m == 0) return e;
  int blocks = (int)std::min<int64_t>((m + kBlock - 1) / kBlock, (int64_t)grid_blocks(g));
  g->ctx->launches += 1;
  k_list_to_bitmap<<<blocks, kBlock, 0, st>>>(list, m, bits, g->n, d_bad);
  return cudaGetLastError();
}

cudaError_t launch_popcount(pp_graph g, const uint32_t* bits, unsigned long long* d_out) {
  cudaStream_t st = g->ctx->stream;
  cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  int blocks = (int)std::min<int64_t>((uwords(g) + kBlock - 1) / kBlock, (int64_t)grid_blocks(g));
  g->ctx->launches += 1;
  k_popcount<<<blocks, kBlock, 0, st>>>(bits, uwords(g), d_out);
  return cudaGetLastError();
}

cudaError_t launch_bitmap_to_list(pp_graph g, const uint32_t* bits, uint32_t* list,
                                  int64_t capacity, unsigned long long* d_count) {
  cudaStream_t st = g->ctx->stream;
  const uint32_t nblk = (uwords(g) + kB2LWords - 1) / kB2LWords;
  g->ctx->launches += 3;
  k_b2l_count<<<nblk, kBlock, 0, st>>>(bits, uwords(g), g->sblock);
  k_b2l_scan<<<1, 1024, 0, st>>>(g->sblock, nblk, d_count);
  k_b2l_write<<<nblk, kBlock, 0, st>>>(bits, uwords(g), g->sblock, list, capacity);
  return cudaGetLastError();
}

template <typename Off>
static cudaError_t mxv_t(pp_graph g, const MxvPlan& p) {
  cudaStream_t st = g->ctx->stream;
  // Op rows: pull scans rows of the operator (A^T -> CSC, A -> CSR); push expands the
  // rows of its transpose (A^T u -> CSR rows of each u(j), A u -> CSC rows).
  const bool use_csc_rows = p.pull ? (p.transpose != 0) : (p.transpose == 0);
  const Off* roff = (const Off*)(use_csc_rows ? g->coff : g->off);
  const uint32_t* ridx = use_csc_rows ? g->cidx : g->idx;
  const int blocks = grid_blocks(g);
  if (p.pull) {
    g->ctx->launches += 1;
    // Without early exit, rows longer than kHubIds are split into chunks that a second
    // kernel spreads over the grid; with early exit rows stay in their warp (most resolve in
    // their first sector) and no second launch is needed.
    unsigned* nhub = reinterpret_cast<unsigned*>(g->scount + 4);
    if (!p.early_exit) {
      cudaError_t e0 = cudaMemsetAsync(g->scount + 4, 0, sizeof(unsigned long long), st);
      if (e0 != cudaSuccess) return e0;
    }
    g->ctx->launches += 1;
    if (p.early_exit)
      k_mxv_pull<Off><<<blocks, kBlock, 0, st>>>(g->n, g->nwords, roff, ridx, p.u_bits, p.mask_bits,
                                                 p.complement, p.accum, p.replace, p.early_exit,
                                                 p.win_bits, p.out_bits, g->hubq, nhub);
    else
      k_mxv_pull_stream<Off><<<g->ctx->num_sms * 8, kBlock, 0, st>>>(g->n, (uint32_t)((g->n + 31) / 32), roff,
                                                        ridx, p.u_bits, p.mask_bits, p.complement,
                                                        p.accum, p.replace, p.win_bits, p.out_bits,
                                                        g->hubq, nhub);
    if (!p.early_exit) {
      g->ctx->launches += 1;
      k_mxv_pull_hubs<Off><<<blocks, kBlock, 0, st>>>(g->hubq, nhub, ridx, p.u_bits, p.early_exit,
                                                      p.out_bits);
    }
    return cudaGetLastError();
  }
  uint32_t* t = g->sbits[0];
  cudaError_t e = cudaMemsetAsync(t, 0, sizeof(uint32_t) * uwords(g), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(g->ctr, 0, sizeof(LevelCtr), st);
  if (e != cudaSuccess) return e;
  g->ctx->launches += 3;
  k_classify<Off><<<blocks, kBlock, 0, st>>>(g->n, p.u_list, p.u_nnz, p.u_bits, g->nwords, roff,
                                             g->L[0], g->H[0], g->ctr, g->scount + 2);
  k_mxv_push<Off><<<blocks, kBlock, 0, st>>>(roff, ridx, g->L[0], g->H[0], g->ctr, p.mask_bits,
                                             p.complement, t);
  k_combine<<<blocks, kBlock, 0, st>>>(g->n, uwords(g), t, p.mask_bits, p.complement, p.accum,
                                       p.replace, p.win_bits, p.out_bits);
  return cudaGetLastError();
}

cudaError_t launch_mxv(pp_graph g, const MxvPlan& p) {
  return g->off64 ? mxv_t<uint64_t>(g, p) : mxv_t<uint32_t>(g, p);
}

}  // namespace pp
