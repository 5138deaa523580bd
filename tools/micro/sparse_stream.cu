// Sparse-ascending record reads on B200: the pull's access pattern.  An array of N 32-byte
// records; a warp walks an item of 1024 consecutive records and loads (one 256-bit load per
// lane) only those passing a hashed Bernoulli(p) mask, 32 at a time in ascending order.
// Reports records/s and sector GB/s for several densities p, plus the same with the
// records permuted (fully random order) for reference.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

__global__ void k_sparse(const uint4* __restrict__ rec, uint32_t n, uint32_t thresh, int randomize,
                         unsigned* ctr, uint32_t* out) {
  const unsigned lane = threadIdx.x & 31;
  uint32_t acc = 0;
  const uint32_t nitems = n / 1024;
  for (;;) {
    unsigned item = 0;
    if (lane == 0) item = atomicAdd(ctr, 1u);
    item = __shfl_sync(~0u, item, 0);
    if (item >= nitems) break;
    for (uint32_t w = 0; w < 32; ++w) {
      const uint32_t r = item * 1024 + w * 32 + lane;
      const bool take = hash(r * 2654435761u + 17) < thresh;
      uint32_t idx = randomize ? (hash(r) % n) : r;
      if (take) {
        uint32_t a0, a1, a2, a3, a4, a5, a6, a7;
        asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3), "=r"(a4), "=r"(a5), "=r"(a6), "=r"(a7)
                     : "l"(rec + 2 * (size_t)idx));
        acc += a0 ^ a7;
      }
    }
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  const uint32_t n = 1u << 22;  // 4.2M records = 134 MB
  uint4* rec;
  cudaMalloc(&rec, (size_t)n * 32);
  cudaMemset(rec, 1, (size_t)n * 32);
  unsigned* ctr;
  uint32_t* out;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&out, 4);
  char* flush;
  cudaMalloc(&flush, 256 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double ps[] = {1.0, 0.57, 0.33, 0.2, 0.1, 0.05};
  for (int rnd = 0; rnd < 2; ++rnd)
    for (double p : ps)
      for (int threads : {512, 1024}) {
        const uint32_t thresh = (uint32_t)(p * 4294967295.0);
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaMemset(flush, rep, 256 << 20);
          cudaMemset(ctr, 0, 4);
          cudaEventRecord(e0);
          k_sparse<<<sms, threads>>>(rec, n, thresh, rnd, ctr, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        const double recs = p * n;
        printf("%s p=%.2f threads/SM=%4d: %7.1f us  %6.1f G rec/s  %7.1f GB/s\n",
               rnd ? "random   " : "ascending", p, threads, best * 1e3, recs / best / 1e6,
               recs * 32 / best / 1e6);
      }
  return 0;
}
