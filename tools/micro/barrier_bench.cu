// Micro-benchmark (B200): cost of one grid-wide barrier in a persistent cooperative kernel.
//   (a) arrival tree: one arrival per CTA on 16 sub-counters + top, acquire spin on a generation word
//   (c) counter barrier (the library's grid_barrier since r01_s)
//   (b) cluster-hierarchical: barrier.cluster, then one arrival per cluster, then barrier.cluster
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../include -o barrier_bench barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2001_01158_b200/csrc/lc_internal.cuh"

namespace cg = cooperative_groups;
using namespace lc;

// (a) the arrival tree + generation word (the library's barrier before it moved to the counter form)
__device__ __forceinline__ void tree_barrier(GridBar* gb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x, b = blockIdx.x;
    const unsigned g0 = ld_acquire_u32(&gb->gen);
    __threadfence();
    bool last = false;
    if (nb <= 64) {
      last = atomicAdd(&gb->top, 1u) == nb - 1;
    } else {
      const unsigned k = b % kBarSub;
      const unsigned nk = (nb - k + kBarSub - 1) / kBarSub;
      if (atomicAdd(&gb->sub[k][0], 1u) == nk - 1) {
        gb->sub[k][0] = 0;
        __threadfence();
        last = atomicAdd(&gb->top, 1u) == (unsigned)kBarSub - 1;
      }
    }
    if (last) {
      gb->top = 0;
      st_release_u32(&gb->gen, g0 + 1);
    } else {
      while (ld_acquire_u32(&gb->gen) == g0) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}
__global__ void k_flat(GridBar* gb, int iters) {
  for (int i = 0; i < iters; ++i) tree_barrier(gb);
}

__device__ __forceinline__ void cluster_grid_barrier(GridBar* gb) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    const unsigned nclu = gridDim.x / cl.num_blocks();
    const unsigned g0 = ld_acquire_u32(&gb->gen);
    __threadfence();
    if (atomicAdd(&gb->top, 1u) == nclu - 1) {
      gb->top = 0;
      st_release_u32(&gb->gen, g0 + 1);
    } else {
      while (ld_acquire_u32(&gb->gen) == g0) {
      }
    }
    __threadfence();
  }
  cl.sync();
}

// (c) counter barrier: every CTA adds 1 (red.release, no round trip) and polls until the counter reaches
// its target k * nb (relaxed polling, one acquire fence after) -- one one-way trip + one poll
__device__ __forceinline__ void counter_barrier(unsigned long long* ctr, unsigned long long& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned long long v;
    do {
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
    } while (v < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
__global__ void k_counter(unsigned long long* ctr, int iters) {
  unsigned long long target = 0;
  for (int i = 0; i < iters; ++i) counter_barrier(ctr, target);
}

// (f) K counters on separate lines: CTA b adds to counter b % K, polls all K (sum >= target)
template <int K>
__device__ __forceinline__ void multi_counter_barrier(unsigned long long* ctr, unsigned long long& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr + 16 * (blockIdx.x % K)) : "memory");
    unsigned long long tot;
    do {
      tot = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr + 16 * k) : "memory");
        tot += v;
      }
    } while (tot < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
template <int K>
__global__ void k_mcounter(unsigned long long* ctr, int iters) {
  unsigned long long target = 0;
  for (int i = 0; i < iters; ++i) multi_counter_barrier<K>(ctr, target);
}
// (e) counter with a short sleep between polls
__global__ void k_counter_sleep(unsigned long long* ctr, int iters) {
  unsigned long long target = 0;
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
      unsigned long long v;
      for (;;) {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        if (v >= target) break;
        __nanosleep(64);
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
  }
}

__global__ void k_cluster(GridBar* gb, int iters) {
  for (int i = 0; i < iters; ++i) cluster_grid_barrier(gb);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  GridBar* gb;
  cudaMalloc(&gb, sizeof(GridBar));
  const int iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int per_sm : {1, 2, 4}) {
    int nb = sms * per_sm;
    cudaMemset(gb, 0, sizeof(GridBar));
    void* args[] = {&gb, (void*)&iters};
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k_flat, dim3(nb), dim3(256), args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("flat    %4d CTAs: %s %.3f us/barrier\n", nb, cudaGetErrorString(e), 1e3 * ms / iters);
    {
      unsigned long long* ctr = (unsigned long long*)gb;
      cudaMemset(gb, 0, sizeof(GridBar));
      void* a2[] = {&ctr, (void*)&iters};
      cudaEventRecord(e0);
      e = cudaLaunchCooperativeKernel((void*)k_counter, dim3(nb), dim3(256), a2, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("counter %4d CTAs: %s %.3f us/barrier\n", nb, cudaGetErrorString(e), 1e3 * ms / iters);
      void* fns[4] = {(void*)k_counter_sleep, (void*)k_mcounter<2>, (void*)k_mcounter<4>, (void*)k_mcounter<8>};
      const char* nm[4] = {"sleep64", "multi2", "multi4", "multi8"};
      for (int f = 0; f < 4; ++f) {
        cudaMemset(gb, 0, sizeof(GridBar));
        cudaEventRecord(e0);
        e = cudaLaunchCooperativeKernel(fns[f], dim3(nb), dim3(256), a2, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%s %4d CTAs: %s %.3f us/barrier\n", nm[f], nb, cudaGetErrorString(e), 1e3 * ms / iters);
      }
    }
    for (int csz : {2, 4, 8}) {
      int nbc = (nb / csz) * csz;
      cudaMemset(gb, 0, sizeof(GridBar));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nbc);
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative;
      at[1].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      cudaEventRecord(e0);
      e = cudaLaunchKernelEx(&cfg, k_cluster, gb, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("cluster %4d CTAs (x%d): %s %.3f us/barrier\n", nbc, csz, cudaGetErrorString(e), 1e3 * ms / iters);
      cudaGetLastError();
    }
  }
  return 0;
}
