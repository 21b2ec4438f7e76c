// common.cu -- error plumbing, stream-ordered allocation, the decoupled
// look-back scan / stream compaction, SELL slice maps.
#include <atomic>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <cstdio>
#include <cstring>

#include "lc_internal.cuh"

namespace lc {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
lc_status cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  if (e == cudaErrorMemoryAllocation) return LC_ERR_OOM;
  return LC_ERR_CUDA;
}
void count_launch(int n) { g_launches += n; }

// ---- per-device state (one process may drive several GPUs from several host threads) ----
static std::mutex g_dev_mu;
static std::set<int> g_pool_dev;                                        // pools set to keep memory
static std::map<int, int> g_sms;                                        // SM count per device
static std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;  // co-resident CTAs per (dev, fn, thr, smem)
static std::map<std::tuple<int, const void*, int>, int> g_attr;         // function attributes set per device

static lc_status device_of_caller(int* dev) {
  LC_CUDA(cudaGetDevice(dev));
  return LC_OK;
}

lc_status dalloc(void** p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  lc_status st = device_of_caller(&dev);
  if (st) return st;
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (!g_pool_dev.count(dev)) {
      cudaMemPool_t pool;
      LC_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
      uint64_t thr = UINT64_MAX;
      LC_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
      g_pool_dev.insert(dev);
    }
  }
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMallocAsync(p, bytes, s);
  if (e != cudaSuccess) {
    *p = nullptr;
    return cuda_fail(e, "cudaMallocAsync");
  }
  return LC_OK;
}
void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}
int num_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_sms.find(dev);
  if (it != g_sms.end()) return it->second;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms < 1) sms = 1;
  g_sms[dev] = sms;
  return sms;
}

const lc_tuning& tuning();
static std::map<int, int64_t> g_l2;                                     // L2 bytes per device
int64_t l2_bytes() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_l2.find(dev);
  if (it != g_l2.end()) return it->second;
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev);
  g_l2[dev] = v;
  return v;
}
bool stream_policy_wanted(int64_t matrix_bytes, int64_t vector_bytes) {
  const int f = tuning().l2_stream_hint;
  if (f >= 0) return f != 0;
  const int64_t l2 = l2_bytes();
  return l2 > 0 && 4 * (matrix_bytes + vector_bytes) > 3 * l2 && vector_bytes <= 2 * l2;
}

lc_status func_attr(const void* fn, cudaFuncAttribute attr, int value) {
  int dev = 0;
  lc_status st = device_of_caller(&dev);
  if (st) return st;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  const auto key = std::make_tuple(dev, fn, (int)attr);
  auto it = g_attr.find(key);
  // the dynamic shared-memory limit only ever grows (a smaller later request keeps the larger opt-in)
  if (it != g_attr.end() && (it->second == value ||
                             (attr == cudaFuncAttributeMaxDynamicSharedMemorySize && it->second >= value)))
    return LC_OK;
  LC_CUDA(cudaFuncSetAttribute(fn, attr, value));
  g_attr[key] = value;
  return LC_OK;
}

lc_status max_coresident(const void* fn, int threads, size_t dsmem, int64_t* ctas) {
  int dev = 0;
  lc_status st = device_of_caller(&dev);
  if (st) return st;
  const auto key = std::make_tuple(dev, fn, threads, dsmem);
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) { *ctas = it->second; return LC_OK; }
  }
  if (dsmem > 0) {                 // static + dynamic above 48 KB needs the opt-in: always opt in to `dsmem`
    st = func_attr(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem);
    if (st) return st;
  }
  int per_sm = 0;
  LC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, dsmem));
  if (per_sm < 1) { set_error("kernel does not fit on an SM"); return LC_ERR_CUDA; }
  const int v = per_sm * num_sms();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  g_occ[key] = v;
  *ctas = v;
  return LC_OK;
}

static std::map<std::tuple<int, const void*, int, size_t, int>, int> g_occ_cl;   // clusters per (dev, fn, thr, smem, cl)

lc_status max_clusters(const void* fn, int threads, size_t dsmem, int cl, int64_t* clusters) {
  int dev = 0;
  lc_status st = device_of_caller(&dev);
  if (st) return st;
  const auto key = std::make_tuple(dev, fn, threads, dsmem, cl);
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_occ_cl.find(key);
    if (it != g_occ_cl.end()) { *clusters = it->second; return LC_OK; }
  }
  if (dsmem > 0 && (st = func_attr(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem))) return st;
  if (cl > 8 && (st = func_attr(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1))) return st;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cl);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = dsmem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  LC_CUDA(cudaOccupancyMaxActiveClusters(&n, fn, &cfg));
  std::lock_guard<std::mutex> lk(g_dev_mu);
  g_occ_cl[key] = n;
  *clusters = n;
  return LC_OK;
}

// ---- completion of a Krylov launch (immediate / deferred, lc_internal.cuh) ----
SolveClock::SolveClock(Pending* pend) {
  if (pend && pend->e0 && pend->e1) { e0 = pend->e0; e1 = pend->e1; return; }
  own = true;
  if (cudaEventCreate(&e0) != cudaSuccess) { e0 = nullptr; cudaGetLastError(); }
  if (cudaEventCreate(&e1) != cudaSuccess) { e1 = nullptr; cudaGetLastError(); }
}
SolveClock::~SolveClock() {
  if (!own) return;
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
}

static lc_status worst_of(const int32_t* stt, int G) {
  lc_status worst = LC_OK;
  for (int g = 0; g < G; ++g) {
    if (stt[g] < 0) worst = (lc_status)stt[g];
    else if (stt[g] == LC_NOT_CONVERGED && worst == LC_OK) worst = LC_NOT_CONVERGED;
  }
  if (worst < 0) set_error("Krylov solve: breakdown or non-finite value (see lc_solve_info.status)");
  return worst;
}

static void fill_info(lc_solve_info* info, int G, const int32_t* it, const int32_t* stt, const double* rr, float ms,
                      int kernel, int lazy) {
  if (!info) return;
  for (int g = 0; g < G; ++g) {
    info[g].iterations = it[g];
    info[g].status = stt[g];
    info[g].rel_residual = rr[g];
    info[g].seconds = ms * 1e-3;
    info[g].kernel = kernel;
    info[g].lazy_x_depth = lazy;
  }
}

lc_status solve_finish(cudaError_t e, SolveClock& clk, Pending* pend, int G, const int* d_it, const int* d_stt,
                       const double* d_rr, int kernel, int lazy, cudaStream_t s, lc_solve_info* info,
                       const char* what) {
  if (G > kMaxSegs) { set_error("solve: at most 64 segments"); return LC_ERR_DIMENSION; }
  if (pend) {
    pend->G = G; pend->kernel = kernel; pend->lazy = lazy; pend->armed = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(pend->it, d_it, 4 * G, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pend->stt, d_stt, 4 * G, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pend->rr, d_rr, 8 * G, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e, what);
    pend->armed = 1;
    return LC_OK;
  }
  int32_t it[kMaxSegs], stt[kMaxSegs];
  double rr[kMaxSegs];
  if (e == cudaSuccess) e = cudaMemcpyAsync(it, d_it, 4 * G, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(stt, d_stt, 4 * G, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(rr, d_rr, 8 * G, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  float ms = 0.f;
  if (e == cudaSuccess && clk.e0 && clk.e1) cudaEventElapsedTime(&ms, clk.e0, clk.e1);
  if (e != cudaSuccess) return cuda_fail(e, what);
  fill_info(info, G, it, stt, rr, ms, kernel, lazy);
  return worst_of(stt, G);
}

lc_status pending_info(const Pending& pend, lc_solve_info* info) {
  if (!pend.armed) return LC_OK;
  float ms = 0.f;
  if (pend.e0 && pend.e1) cudaEventElapsedTime(&ms, pend.e0, pend.e1);
  fill_info(info, pend.G, pend.it, pend.stt, pend.rr, ms, pend.kernel, pend.lazy);
  return worst_of(pend.stt, pend.G);
}

// ---- tuning (include/lc.h): thread-local, explicit, no environment variables ----
static lc_tuning defaults_() {
  lc_tuning t;
  t.stencil_layout = 1; t.symmetric_layout = 0; t.pcg_cluster_resident = 2; t.pcg_cluster = 1; t.pcg_tma = 1;
  t.lazy_x_depth = 3; t.batched_schedule = -1; t.pcg_max_ctas = 0; t.sub_repr = -1; t.gmres_exact_cgs2 = 0;
  t.gs_lines = 1;
  t.spmv_csr_tma = 1;
  t.spmv_tma = 1;
  t.batched_cluster = 0;
  t.block_dcoup = 1;
  t.l2_stream_hint = -1;
  return t;
}
static thread_local lc_tuning g_tune = defaults_();
const lc_tuning& tuning() { return g_tune; }

void Sell::release(cudaStream_t s) {
  dfree(slice_ptr, s); dfree(slice_row0, s); dfree(slice_seg, s); dfree(seg_unit0, s); dfree(seg_slice0, s);
  dfree(col, s); dfree(val, s); dfree(rowlen, s); dfree(dinv, s); dfree(mask, s); dfree(cval, s);
  mask = nullptr; cval = nullptr;
  slice_ptr = nullptr; slice_row0 = slice_seg = seg_unit0 = nullptr; seg_slice0 = nullptr;
  col = nullptr; val = nullptr; rowlen = nullptr; dinv = nullptr;
}

// ---------------------------------------------------------------------------
// Decoupled look-back (single pass, dynamic tile ids for forward progress).
// Status word: bits 62-63 = 0 invalid / 1 aggregate / 2 inclusive prefix.
// ---------------------------------------------------------------------------
constexpr unsigned long long kFlagA = 1ull << 62, kFlagP = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// called by all 32 lanes of warp 0; returns the exclusive prefix of `tile` (broadcast to all lanes)
__device__ long long lookback(unsigned long long* status, long long tile, long long aggregate) {
  int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_release(&status[0], kFlagP | (unsigned long long)aggregate);
    return 0;
  }
  if (lane == 0) st_release(&status[tile], kFlagA | (unsigned long long)aggregate);
  long long acc = 0, pred = tile - 1;
  for (;;) {
    long long t = pred - lane;
    unsigned long long w = (t >= 0) ? ld_acquire(&status[t]) : kFlagP;
    while (__any_sync(0xffffffffu, (w >> 62) == 0)) {
      if ((w >> 62) == 0) w = ld_acquire(&status[t]);
    }
    unsigned pm = __ballot_sync(0xffffffffu, (w >> 62) == 2);
    if (pm) {
      int first = __ffs(pm) - 1;
      acc += warp_sum_ll(lane <= first ? (long long)(w & kValMask) : 0);
      break;
    }
    acc += warp_sum_ll((long long)(w & kValMask));
    pred -= 32;
  }
  if (lane == 0) st_release(&status[tile], kFlagP | (unsigned long long)(acc + aggregate));
  return acc;
}

constexpr int kCtThreads = 256, kCtItems = 16, kCtTile = kCtThreads * kCtItems;

// Stable stream compaction of {u : flag[u] != 255}: warp ballot/popc counts, CTA scan, look-back.
__global__ void __launch_bounds__(kCtThreads) k_compact(const uint8_t* __restrict__ flag, int64_t m,
                                                        int32_t* __restrict__ idx, int32_t* __restrict__ inv,
                                                        unsigned long long* status, unsigned* tile_counter,
                                                        int64_t* count_out, int64_t ntiles) {
  __shared__ unsigned s_tile;
  __shared__ int s_warp[kCtThreads / 32];
  __shared__ long long s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const long long tile = s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // item k of thread t covers unit tile*4096 + k*256 + t: each warp-wide load is coalesced and the
  // ballot of item k gives the warp's 32 consecutive units in order.
  const int64_t base = tile * kCtTile;
  unsigned masks[kCtItems];
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < kCtItems; ++k) {
    int64_t u = base + k * kCtThreads + threadIdx.x;
    bool in = (u < m) && (flag[u] != 255);
    masks[k] = __ballot_sync(0xffffffffu, in);
    cnt += __popc(masks[k]);   // warp-level count (same in all lanes)
  }
  // per (item k, warp w) offsets: order = k major, then warp, then lane
  __shared__ int s_cnt[kCtItems][kCtThreads / 32];
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kCtItems; ++k) s_cnt[k][warp] = __popc(masks[k]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int k = 0; k < kCtItems; ++k)
      for (int w = 0; w < kCtThreads / 32; ++w) { int c = s_cnt[k][w]; s_cnt[k][w] = run; run += c; }
    s_warp[0] = run;
  }
  __syncthreads();
  const int total = s_warp[0];
  if (warp == 0) {
    long long ex = lookback(status, tile, total);
    if (lane == 0) s_excl = ex;
  }
  __syncthreads();
  const long long ex = s_excl;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < kCtItems; ++k) {
    int64_t u = base + k * kCtThreads + threadIdx.x;
    if (u < m) {
      bool in = (masks[k] >> lane) & 1u;
      if (in) {
        long long pos = ex + s_cnt[k][warp] + __popc(masks[k] & lt);
        idx[pos] = (int32_t)u;
        inv[u] = (int32_t)pos;
      } else {
        inv[u] = -1;
      }
    }
  }
  if (tile == ntiles - 1 && threadIdx.x == 0) *count_out = ex + total;
  (void)cnt;
}

lc_status compact_flags(const uint8_t* flag, int64_t m, int32_t* idx, int32_t* inv, int64_t* count_dev,
                        cudaStream_t s) {
  if (m == 0) {
    LC_CUDA(cudaMemsetAsync(count_dev, 0, sizeof(int64_t), s));
    return LC_OK;
  }
  int64_t ntiles = (m + kCtTile - 1) / kCtTile;
  void* ws = nullptr;
  size_t bytes = sizeof(unsigned long long) * ntiles + 16;
  lc_status st = dalloc(&ws, bytes, s);
  if (st) return st;
  LC_CUDA(cudaMemsetAsync(ws, 0, bytes, s));
  unsigned long long* status = (unsigned long long*)ws;
  unsigned* counter = (unsigned*)((char*)ws + sizeof(unsigned long long) * ntiles);
  k_compact<<<(unsigned)ntiles, kCtThreads, 0, s>>>(flag, m, idx, inv, status, counter, count_dev, ntiles);
  LC_LAUNCHED();
  dfree(ws, s);
  return LC_OK;
}

// Exclusive scan of int64 (slice widths -> slice_ptr).  out has n+1 entries.
constexpr int kScItems = 8, kScTile = kCtThreads * kScItems;
__global__ void __launch_bounds__(kCtThreads) k_scan_i64(const int64_t* __restrict__ in, int64_t* __restrict__ out,
                                                         int64_t n, unsigned long long* status,
                                                         unsigned* tile_counter, int64_t ntiles) {
  __shared__ unsigned s_tile;
  __shared__ long long s_w[kCtThreads / 32];
  __shared__ long long s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const long long tile = s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = tile * kScTile + (int64_t)threadIdx.x * kScItems;
  long long v[kScItems], sum = 0;
#pragma unroll
  for (int k = 0; k < kScItems; ++k) { v[k] = (base + k < n) ? in[base + k] : 0; sum += v[k]; }
  long long incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  long long woff = 0, total = 0;
  for (int w = 0; w < kCtThreads / 32; ++w) { if (w < warp) woff += s_w[w]; total += s_w[w]; }
  if (warp == 0) {
    long long ex = lookback(status, tile, total);
    if (lane == 0) s_excl = ex;
  }
  __syncthreads();
  long long run = s_excl + woff + incl - sum;
#pragma unroll
  for (int k = 0; k < kScItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
  if (tile == ntiles - 1 && threadIdx.x == 0) out[n] = s_excl + total;
}

lc_status scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  if (n == 0) {
    LC_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
    return LC_OK;
  }
  int64_t ntiles = (n + kScTile - 1) / kScTile;
  void* ws = nullptr;
  size_t bytes = sizeof(unsigned long long) * ntiles + 16;
  lc_status st = dalloc(&ws, bytes, s);
  if (st) return st;
  LC_CUDA(cudaMemsetAsync(ws, 0, bytes, s));
  k_scan_i64<<<(unsigned)ntiles, kCtThreads, 0, s>>>(in, out, n, (unsigned long long*)ws,
                                                      (unsigned*)((char*)ws + sizeof(unsigned long long) * ntiles),
                                                      ntiles);
  LC_LAUNCHED();
  dfree(ws, s);
  return LC_OK;
}

// slice -> (first unit, segment) from the per-segment unit / slice offsets
__global__ void k_slice_map(int64_t nslices, int nseg, const int32_t* __restrict__ seg_unit0,
                            const int64_t* __restrict__ seg_slice0, int32_t* row0, int32_t* sseg) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nslices) return;
  int lo = 0, hi = nseg - 1;   // last g with seg_slice0[g] <= s
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (seg_slice0[mid] <= s) lo = mid; else hi = mid - 1;
  }
  row0[s] = seg_unit0[lo] + (int32_t)(32 * (s - seg_slice0[lo]));
  sseg[s] = lo;
}

lc_status build_slice_map(Sell& M, cudaStream_t s) {
  if (M.nslices == 0) return LC_OK;
  k_slice_map<<<(unsigned)((M.nslices + 255) / 256), 256, 0, s>>>(M.nslices, M.nseg, M.seg_unit0, M.seg_slice0,
                                                                   M.slice_row0, M.slice_seg);
  LC_LAUNCHED();
  return LC_OK;
}

lc_status check_matrix(const lc_matrix_s* M, const char* where) {
  if (!M) { set_error(std::string(where) + ": null matrix"); return LC_ERR_INVALID_ARG; }
  if (!M->valid) {
    set_error(std::string(where) + ": the matrix holds half-written values after a failed lc_update_values "
              "(call lc_update_values again with valid values, or recreate it)");
    return LC_ERR_INVALID_ARG;
  }
  return LC_OK;
}

}  // namespace lc

void lc_domain_s::release(cudaStream_t s) {
  lc::dfree(flag, s); lc::dfree(idx, s); lc::dfree(inv, s); lc::dfree(crit, s); lc::dfree(adm, s);
  lc::dfree(r, s); lc::dfree(seg_base, s);
  flag = nullptr; idx = inv = nullptr; crit = adm = r = nullptr; seg_base = nullptr;
}
void lc_sub_s::release(cudaStream_t s) {
  B.release(s);
  lc::dfree(idx, s); lc::dfree(bsub, s); lc::dfree(xB0, s);
  lc::dfree(bs, s); lc::dfree(xm0, s); lc::dfree(omega, s); lc::dfree(slist, s); lc::dfree(nlist, s); lc::dfree(lseg, s);
  idx = nullptr; bsub = xB0 = nullptr; bs = xm0 = nullptr; omega = nullptr; slist = nullptr; nlist = nullptr; lseg = nullptr;
}

extern "C" const char* lc_last_error(void) { return lc::g_err.c_str(); }
extern "C" int64_t lc_kernel_launches(void) { return (int64_t)lc::g_launches.load(); }

extern "C" void lc_tuning_defaults(lc_tuning* t) {
  if (t) *t = lc::defaults_();
}
extern "C" lc_status lc_set_tuning(const lc_tuning* t) {
  if (!t) { lc::g_tune = lc::defaults_(); return LC_OK; }
  auto bin = [](int32_t v) { return v == 0 || v == 1; };
  if (!bin(t->stencil_layout) || !bin(t->symmetric_layout) || t->pcg_cluster_resident < 0 || t->pcg_cluster_resident > 2 || !bin(t->pcg_cluster) ||
      !bin(t->pcg_tma) || t->lazy_x_depth < 0 || t->lazy_x_depth > 3 || t->batched_schedule < -1 ||
      t->batched_schedule > 2 || t->pcg_max_ctas < 0 || t->sub_repr < -1 || t->sub_repr > 1 ||
      !bin(t->gmres_exact_cgs2) || !bin(t->gs_lines) || !bin(t->spmv_csr_tma) || t->spmv_tma < 0 || t->spmv_tma > 2 ||
      t->batched_cluster < 0 || t->batched_cluster == 1 || t->batched_cluster > 16 || !bin(t->block_dcoup) ||
      t->l2_stream_hint < -1 || t->l2_stream_hint > 1) {
    lc::set_error("lc_set_tuning: field out of range");
    return LC_ERR_INVALID_ARG;
  }
  lc::g_tune = *t;
  return LC_OK;
}
extern "C" lc_status lc_get_tuning(lc_tuning* t) {
  if (!t) { lc::set_error("lc_get_tuning: null argument"); return LC_ERR_INVALID_ARG; }
  *t = lc::g_tune;
  return LC_OK;
}
