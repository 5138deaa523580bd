// pp_device.cuh — warp-level building blocks shared by the BFS and mxv kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pp_internal.h"

namespace pp {

constexpr unsigned kFull = 0xFFFFFFFFu;
#ifndef PP_FAST_NTH
#define PP_FAST_NTH 1
#endif

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned warp_incl_scan(unsigned v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    unsigned t = __shfl_up_sync(kFull, v, d);
    if (lane >= (unsigned)d) v += t;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  return v;
}

// Owner lane of item e given the warp's inclusive scan `incl` of per-lane counts:
// the number of lanes whose inclusive prefix is <= e (<= 31 whenever e < total).
__device__ __forceinline__ unsigned warp_owner(unsigned incl, unsigned e) {
  unsigned j = 0;
#pragma unroll
  for (unsigned s = 16; s >= 1; s >>= 1) {
    unsigned v = __shfl_sync(kFull, incl, j + s - 1);
    if (v <= e) j += s;
  }
  return j;
}

// One dynamic work item per warp (lane 0 grabs, broadcast).
__device__ __forceinline__ unsigned warp_grab(unsigned* ctr) {
  unsigned x = 0;
  if (lane_id() == 0) x = atomicAdd(ctr, 1u);
  return __shfl_sync(kFull, x, 0);
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_add_release_u64(unsigned long long* p,
                                                                   unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.release.gpu.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_timer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Read-only (non-coherent) loads for data that no thread writes during the kernel.
template <typename T>
__device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

// Position of the k-th (0-based) set bit of m, k < popc(m): a branch-free 5-step popcount
// search.  (__fns compiles to a ~50-instruction sequence with divergent branches on sm_100a;
// the warp-balanced candidate enumerations call this once per candidate.)
__device__ __forceinline__ unsigned nth_set_bit(uint32_t m, unsigned k) {
#if PP_FAST_NTH
  unsigned pos = 0, c;
  c = __popc(m & 0xFFFFu);
  if (k >= c) { k -= c; m >>= 16; pos += 16; }
  c = __popc(m & 0xFFu);
  if (k >= c) { k -= c; m >>= 8; pos += 8; }
  c = __popc(m & 0xFu);
  if (k >= c) { k -= c; m >>= 4; pos += 4; }
  c = __popc(m & 0x3u);
  if (k >= c) { k -= c; m >>= 2; pos += 2; }
  c = m & 1u;
  if (k >= c) pos += 1;
  return pos;
#else
  return __fns(m, 0, (int)k + 1);
#endif
}

// Bit test in a bitmap.
__device__ __forceinline__ bool bit_test(const uint32_t* bits, uint32_t x) {
  return (bits[x >> 5] >> (x & 31u)) & 1u;
}

}  // namespace pp
