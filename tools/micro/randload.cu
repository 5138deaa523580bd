// Random-access throughput microbenchmark on B200 (Little's-law calibration for the pull).
// Each thread issues K independent random loads per iteration (hashed addresses), ITERS
// iterations; reports requests/s and sectors/s for DRAM-sized and L2-sized targets.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int K, int W>  // W = words per load (1 = 4B, 8 = 32B)
__global__ void k_rand(const uint32_t* __restrict__ a, uint32_t mask, int iters, uint32_t* out) {
  uint32_t acc = 0;
  uint32_t seed = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    uint32_t v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      uint32_t idx = (hash(seed * 131u + it * 7919u + k) & mask) & ~(uint32_t)(W - 1);
      if (W == 1) {
        v[k] = __ldg(a + idx);
      } else {
        uint32_t r0, r1, r2, r3, r4, r5, r6, r7;
        asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(r4), "=r"(r5), "=r"(r6), "=r"(r7)
                     : "l"(a + idx));
        v[k] = r0 ^ r7;
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc += v[k];
    seed += acc & 1;  // serialize iterations lightly (dependence on loaded data)
  }
  if (acc == 0x12345678) out[0] = acc;
}

template <int K, int W>
void run(const uint32_t* a, uint32_t mask, int threads, const char* tag) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, 4);
  int iters = 200;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_rand<K, W><<<sms, threads>>>(a, mask, 10, out);
  cudaEventRecord(e0);
  k_rand<K, W><<<sms, threads>>>(a, mask, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double req = (double)sms * threads * iters * K;
  printf("%-6s K=%2d W=%d threads/SM=%4d : %7.2f G req/s  %7.1f GB/s(sector)  %.1f req/SM/us\n", tag, K, W,
         threads, req / ms / 1e6, req * 32 / ms / 1e6, req / ms * 1e-3 / sms);
  cudaFree(out);
}

int main() {
  size_t big = (size_t)512 << 20;  // 512 MB: DRAM
  uint32_t* a; cudaMalloc(&a, big); cudaMemset(a, 1, big);
  uint32_t mbig = (uint32_t)(big / 4 - 1), msmall = (512 * 1024) / 4 - 1;  // 512 KB: L2
  for (int th : {256, 512, 1024}) {
    run<1, 1>(a, mbig, th, "DRAM"); run<4, 1>(a, mbig, th, "DRAM"); run<8, 1>(a, mbig, th, "DRAM");
    run<16, 1>(a, mbig, th, "DRAM");
    run<1, 8>(a, mbig, th, "DRAM"); run<4, 8>(a, mbig, th, "DRAM"); run<8, 8>(a, mbig, th, "DRAM");
    run<1, 1>(a, msmall, th, "L2"); run<4, 1>(a, msmall, th, "L2"); run<8, 1>(a, msmall, th, "L2");
    run<16, 1>(a, msmall, th, "L2");
  }
  return 0;
}
