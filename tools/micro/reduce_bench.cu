// Micro-benchmark (B200): one REDUCING grid barrier of a persistent cooperative kernel -- every CTA contributes T
// doubles, every CTA leaves with the T fixed-order sums over all CTAs (what a batched PCG pass needs for its G
// segments, T = 2G).  Device time per barrier, 2000 barriers, 256-thread CTAs, 4 per SM:
//   (t) tree_reduce_barrier (the library's batched barrier): 16 sub-group reducers + a done counter
//   (d) counter barrier, then every CTA sums all nCTA x T partials itself (the G = 1 form, generalised)
//   (c) CL-CTA clusters: the cluster's partials summed through DSMEM by its rank-0 CTA, one arrival per cluster on
//       a counter, every CTA sums the nCTA / CL cluster partials itself
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o reduce_bench reduce_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2001_01158_b200/csrc/lc_internal.cuh"

namespace cg = cooperative_groups;
using namespace lc;

constexpr int kT = 256;
constexpr int kNW = kT / 32;
constexpr int kTMax = 128;

// every CTA: out[t] = sum over members m < M of part[m * T + t] in a fixed order: warp w takes the values
// t = w, w + NW, ...; lane l adds members l, l + 32, ... in order (8 loads in flight), then a butterfly warp sum
__device__ __forceinline__ void sum_all(const double* part, int M, int T, double* s_chunk, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  (void)s_chunk;
  for (int t = warp; t < T; t += kNW) {
    double a = 0.0;
    for (int m0 = lane; m0 < M; m0 += 32 * 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = m0 + 32 * q < M ? __ldcg(part + (size_t)(m0 + 32 * q) * T + t) : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (m0 + 32 * q < M) a += v[q];
    }
    a = warp_sum(a);
    if (lane == 0) out[t] = a;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kT, 4) k_tree(GridBar* gb, double* part, double* subred, int T, int iters,
                                                 double* sink) {
  __shared__ double s_tmp[kNW][kTMax];
  __shared__ double s_out[kTMax];
  unsigned epoch = 0;
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < T) part[(size_t)blockIdx.x * T + threadIdx.x] = blockIdx.x + i + threadIdx.x;
    tree_reduce_barrier<kNW, kTMax>(gb, part, subred, s_out, T, s_tmp, epoch);
    acc += s_out[0];
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = acc;
}

__global__ void __launch_bounds__(kT, 4) k_direct(GridBar* gb, double* part, int T, int iters, double* sink) {
  __shared__ double s_chunk[kT];
  __shared__ double s_out[kTMax];
  unsigned long long epoch = 0;
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    double* pt = part + (size_t)(i & 1) * gridDim.x * T;
    if (threadIdx.x < T) pt[(size_t)blockIdx.x * T + threadIdx.x] = blockIdx.x + i + threadIdx.x;
    grid_barrier(gb, epoch);
    sum_all(pt, gridDim.x, T, s_chunk, s_out);
    acc += s_out[0];
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = acc;
}

__global__ void __launch_bounds__(kT, 4) k_clus(GridBar* gb, double* part, int T, int iters, double* sink) {
  __shared__ double s_chunk[kT];
  __shared__ double s_out[kTMax];
  __shared__ double s_mine[2][kTMax];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned CL = cl.num_blocks(), rank = cl.block_rank();
  const unsigned ncl = gridDim.x / CL, cid = blockIdx.x / CL;
  unsigned long long target = 0;
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    const int b = i & 1;
    if (threadIdx.x < T) s_mine[b][threadIdx.x] = blockIdx.x + i + threadIdx.x;
    cl.sync();                                           // the cluster's partials are in place
    double* pt = part + (size_t)b * ncl * T;
    target += ncl;
    if (rank == 0) {
      if (threadIdx.x < T) {
        double v[16];
#pragma unroll
        for (unsigned r = 0; r < 16; ++r) v[r] = r < CL ? cl.map_shared_rank(&s_mine[b][0], r)[threadIdx.x] : 0.0;
        double a = 0.0;
#pragma unroll
        for (unsigned r = 0; r < 16; ++r)
          if (r < CL) a += v[r];
        pt[(size_t)cid * T + threadIdx.x] = a;
      }
      __syncthreads();
      if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&gb->ctr) : "memory");
    }
    if (threadIdx.x == 0) {
      unsigned long long v;
      do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&gb->ctr) : "memory");
      } while (v < target);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    sum_all(pt, ncl, T, s_chunk, s_out);
    acc += s_out[0];
  }
  cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  GridBar* gb;
  double *part, *subred, *sink;
  cudaMalloc(&gb, sizeof(GridBar));
  cudaMalloc(&part, sizeof(double) * 2 * 1024 * kTMax);
  cudaMalloc(&subred, sizeof(double) * 2 * kBarSub * kTMax);
  cudaMalloc(&sink, 64);
  const int iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int nb = 4 * sms;
  for (int T : {2, 8, 40}) {
    float ms = 0;
    cudaMemset(gb, 0, sizeof(GridBar));
    cudaEventRecord(e0);
    {
      void* a[] = {&gb, &part, &subred, (void*)&T, (void*)&iters, &sink};
      cudaError_t e = cudaLaunchCooperativeKernel((void*)k_tree, dim3(nb), dim3(kT), a, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("T=%2d tree    %4d CTAs: %s %.3f us/barrier\n", T, nb, cudaGetErrorString(e), 1e3 * ms / iters);
    }
    cudaMemset(gb, 0, sizeof(GridBar));
    cudaEventRecord(e0);
    {
      void* a[] = {&gb, &part, (void*)&T, (void*)&iters, &sink};
      cudaError_t e = cudaLaunchCooperativeKernel((void*)k_direct, dim3(nb), dim3(kT), a, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("T=%2d direct  %4d CTAs: %s %.3f us/barrier\n", T, nb, cudaGetErrorString(e), 1e3 * ms / iters);
    }
    for (int csz : {4, 8, 16}) {
      int maxc = 0;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((nb / csz) * csz);
      cfg.blockDim = dim3(kT);
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative;
      at[1].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (csz > 8) cudaFuncSetAttribute((void*)k_clus, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaOccupancyMaxActiveClusters(&maxc, (void*)k_clus, &cfg);
      const int nbc = (maxc * csz < nb ? maxc * csz : (nb / csz) * csz);
      cfg.gridDim = dim3(nbc);
      cfg.numAttrs = 2;
      cudaMemset(gb, 0, sizeof(GridBar));
      cudaEventRecord(e0);
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_clus, gb, part, T, iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("T=%2d cluster %4d CTAs (x%d, max active clusters %d): %s %.3f us/barrier\n", T, nbc, csz, maxc,
             cudaGetErrorString(e), 1e3 * ms / iters);
      cudaGetLastError();
    }
  }
  return 0;
}
