// gridbar.cu — decomposes the per-level fixed cost of bfs_persistent:
// software grid-barrier variants on one CTA per SM (148 x 1024 threads, cooperative launch),
// timed over many back-to-back barriers with CUDA events.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o gridbar gridbar.cu
//   ./gridbar [iters]
//
// Variants (V = template id):
//   0  bfs.cu today: bar.sync; t0: atom.add.release.gpu; poll ld.acquire.gpu + nanosleep(16);
//      fence.sc.gpu; bar.sync
//   1  as 0 without the nanosleep
//   2  as 0 without the trailing fence.sc.gpu (the acquire poll orders the CTA)
//   3  red.release.gpu arrival (no return) + acquire poll, no trailing fence
//   4  an empty BFS level: flush_acc (warp sums, bar.sync, 3 counter atomics per CTA) +
//      variant-0 barrier + read_level (thread 0 reads 7 counters, bar.sync) + ring reset
//   5  as 4 with the variant-3 barrier and the counters read by 7 lanes of warp 0 at once
//   6  two-level: cluster of 2 CTAs (barrier.cluster), one arrival per cluster, poll, cluster
//      barrier
//   7  same with clusters of 4
//   8  bar.sync only (lower bound of the CTA-local part)
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));         \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

struct Ctr {
  unsigned long long c, m_f, m_fin, nbig;
  unsigned nL, nH, work, work2;
  unsigned long long pad[2];
};

__device__ __forceinline__ unsigned long long atom_add_release(unsigned long long* p, unsigned long long v) {
  unsigned long long o;
  asm volatile("atom.add.release.gpu.u64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(v) : "memory");
  return o;
}
__device__ __forceinline__ void red_add_release(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned nclusters() {
  unsigned r;
  asm("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}

template <int V>
__device__ __forceinline__ void barrier(unsigned long long* cnt, unsigned& epoch) {
  if (V == 8) {
    __syncthreads();
    return;
  }
  if (V == 6 || V == 7) {
    __syncthreads();
    cluster_sync();
    if (cluster_ctarank() == 0 && threadIdx.x == 0) {
      ++epoch;
      const unsigned long long target = (unsigned long long)epoch * nclusters();
      red_add_release(cnt, 1ull);
      while (ld_acquire(cnt) < target) {
      }
    }
    cluster_sync();
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned long long target = (unsigned long long)epoch * gridDim.x;
    unsigned long long v;
    if (V == 3 || V == 5) {
      red_add_release(cnt, 1ull);
      v = 0;
    } else {
      v = atom_add_release(cnt, 1ull) + 1ull;
    }
    while (v < target) {
      v = ld_acquire(cnt);
      if (V == 0 || V == 2 || V == 4) __nanosleep(16);
    }
    if (V == 0 || V == 1 || V == 4) __threadfence();
  }
  __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(1024, 1) k_bar(unsigned long long* cnt, Ctr* ring, int iters,
                                                 unsigned long long* sink) {
  __shared__ unsigned long long red[32][4];
  __shared__ long long lvl[8];
  unsigned epoch = 0;
  unsigned long long acc = threadIdx.x & 1;  // every CTA contributes (a level's counters)
  long long keep = 0;
  for (int it = 0; it < iters; ++it) {
    Ctr* out = &ring[it & 3];
    if (V == 4 || V == 5) {
      // flush_acc: warp sums -> smem -> warp 0 -> 3 atomics per CTA
      unsigned long long c = acc;
      for (int d = 16; d >= 1; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][0] = c;
      __syncthreads();
      if (threadIdx.x < 32) {
        unsigned long long t = red[threadIdx.x][0];
        for (int d = 16; d >= 1; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
        if (threadIdx.x == 0) {
          atomicAdd(&out->c, t);
          atomicAdd(&out->m_f, t);
          atomicAdd(&out->m_fin, t);
        }
      }
      if (blockIdx.x == 0 && threadIdx.x < 16)
        reinterpret_cast<unsigned*>(&ring[(it + 1) & 3])[threadIdx.x] = 0u;
    }
    barrier<V>(cnt, epoch);
    if (V == 4) {
      if (threadIdx.x == 0) {
        lvl[0] = (long long)ld_relaxed(&out->c);
        lvl[1] = (long long)ld_relaxed(&out->m_f);
        lvl[2] = (long long)ld_relaxed(&out->m_fin);
        lvl[3] = (long long)ld_relaxed(&out->nbig);
        lvl[4] = (long long)*(volatile unsigned*)&out->nL;
        lvl[5] = (long long)*(volatile unsigned*)&out->nH;
        lvl[6] = (long long)*(volatile unsigned*)&out->work;
      }
      __syncthreads();
      keep += lvl[0] + lvl[6];
    } else if (V == 5) {
      if (threadIdx.x < 7) {
        const unsigned long long* p = reinterpret_cast<const unsigned long long*>(out);
        lvl[threadIdx.x] = (long long)ld_relaxed(p + threadIdx.x);
      }
      __syncthreads();
      keep += lvl[0] + lvl[6];
    }
  }
  if (threadIdx.x == 0 && keep == 12345) sink[0] = keep;
}

template <int V>
static float run(int iters, int cluster) {
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  unsigned long long *cnt, *sink;
  Ctr* ring;
  CK(cudaMalloc(&cnt, 256));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&ring, 4 * sizeof(Ctr)));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaMemset(cnt, 0, 256));
    CK(cudaMemset(ring, 0, 4 * sizeof(Ctr)));
    cudaLaunchConfig_t cfg = {};
    int grid = sms;
    if (cluster > 1) grid = sms / cluster * cluster;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(1024);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    int na = 1;
    if (cluster > 1) {
      at[1].id = cudaLaunchAttributeClusterDimension;
      at[1].val.clusterDim.x = cluster;
      at[1].val.clusterDim.y = 1;
      at[1].val.clusterDim.z = 1;
      na = 2;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    CK(cudaEventRecord(a));
    CK(cudaLaunchKernelEx(&cfg, k_bar<V>, cnt, ring, iters, sink));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  cudaFree(cnt);
  cudaFree(sink);
  cudaFree(ring);
  return best * 1000.f / iters;
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 4000;
  printf("us per barrier (best of 5 launches, %d barriers each, 1 CTA x 1024 thr per SM)\n", iters);
  printf("V0 bfs.cu today (atom.release, acquire poll + nanosleep, fence.sc)   %.3f\n", run<0>(iters, 1));
  printf("V1 V0 without nanosleep                                              %.3f\n", run<1>(iters, 1));
  printf("V2 V0 without trailing fence.sc                                      %.3f\n", run<2>(iters, 1));
  printf("V3 red.release arrival, acquire poll, no fence                       %.3f\n", run<3>(iters, 1));
  printf("V4 empty level today: flush_acc + V0 + read_level                    %.3f\n", run<4>(iters, 1));
  printf("V5 empty level: flush_acc + V3 + parallel counter read               %.3f\n", run<5>(iters, 1));
  printf("V6 cluster-2 two-level barrier                                       %.3f\n", run<6>(iters, 2));
  printf("V7 cluster-4 two-level barrier                                       %.3f\n", run<7>(iters, 4));
  printf("V8 bar.sync only                                                     %.3f\n", run<8>(iters, 1));
  return 0;
}
