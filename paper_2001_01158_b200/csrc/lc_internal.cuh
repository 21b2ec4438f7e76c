// lc_internal.cuh -- internal types and device helpers of liblc.so (sm_100a).
//
// Layout in HBM:
//   SELL-C-sigma with C = 32 (one warp per slice), sigma = 1 (row order kept, so
//   every per-row sum runs over the stored ascending column order, R22).  Slice s
//   covers units [slice_row0[s], slice_row0[s] + 32) of segment slice_seg[s];
//   lanes past the segment end are padding.  Slot k of lane l in slice s lives at
//   slot = slice_ptr[s] + 32 k + l: col[slot] (int32), and
//     block = 1: val[slot] (f64);
//     block = 3: val[9 (slice_ptr[s] + 32 k) + 32 q + l], q = 3 alpha + beta
//   so that each warp-wide load of one slot / one block component is 256 B
//   contiguous.  Padding slots hold col = own unit, value 0 (they contribute
//   +0 to fma chains and are skipped by pattern walks via rowlen).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/lc.h"

namespace lc {

constexpr int kWarp = 32;

// ---------------------------------------------------------------- errors ----
void set_error(const std::string& msg);
lc_status cuda_fail(cudaError_t e, const char* what);
void count_launch(int n = 1);

#define LC_CUDA(call)                                                  \
  do {                                                                 \
    cudaError_t _e = (call);                                           \
    if (_e != cudaSuccess) return ::lc::cuda_fail(_e, #call);          \
  } while (0)

#define LC_LAUNCHED()                                                  \
  do {                                                                 \
    ::lc::count_launch();                                              \
    cudaError_t _e = cudaGetLastError();                               \
    if (_e != cudaSuccess) return ::lc::cuda_fail(_e, "kernel launch"); \
  } while (0)

// stream-ordered device allocation (pool with unlimited release threshold)
lc_status dalloc(void** p, size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);
int num_sms();

// ------------------------------------------------------------------ SELL ----
struct Sell {
  int block = 1;            // 1 (scalar rows) or 3 (3x3 cell blocks)
  int64_t nunits = 0;       // rows or cells
  int64_t nslices = 0;
  int64_t nslots = 0;       // slice_ptr[nslices]
  int maxw = 0;             // max stored entries (blocks) per row (cell)
  int nseg = 1;
  int64_t* slice_ptr = nullptr;   // [nslices+1]
  int32_t* slice_row0 = nullptr;  // [nslices]
  int32_t* slice_seg = nullptr;   // [nslices]
  int32_t* seg_unit0 = nullptr;   // [nseg+1]
  int64_t* seg_slice0 = nullptr;  // [nseg+1]
  int32_t* col = nullptr;         // [nslots]
  double* val = nullptr;          // [nslots * block*block]
  uint8_t* rowlen = nullptr;      // [nunits]
  double* dinv = nullptr;         // [nunits * block*block]: 1/a_ii or the inverse cell block (row-major)
  std::vector<int32_t> h_seg_unit0;
  std::vector<int64_t> h_seg_slice0;
  void release(cudaStream_t s);
};

// Device view passed by value to kernels
struct SellView {
  int block;
  int64_t nslices;
  int nseg;
  const int64_t* slice_ptr;
  const int32_t* slice_row0;
  const int32_t* slice_seg;
  const int32_t* seg_unit0;
  const int64_t* seg_slice0;
  const int32_t* col;
  const double* val;
  const uint8_t* rowlen;
  const double* dinv;
};
inline SellView view(const Sell& m) {
  return SellView{m.block, m.nslices, m.nseg, m.slice_ptr, m.slice_row0, m.slice_seg, m.seg_unit0,
                  m.seg_slice0, m.col, m.val, m.rowlen, m.dinv};
}

// --------------------------------------------------------------- handles ----
}  // namespace lc

struct lc_matrix_s {
  int64_t n = 0;            // units (rows or cells)
  int32_t block = 1, batch = 1;
  int64_t nnz = 0;          // stored blocks / scalars of the input
  int32_t seg_units = 0;    // n / batch
  lc::Sell A;
};

struct lc_domain_s {
  lc_matrix_s* A = nullptr;
  int64_t m = 0;            // units
  int32_t nseg = 1;
  int64_t K_units = 0;      // total units in Omega
  uint8_t* flag = nullptr;  // [m] stage at which the unit entered Omega, 255 = not in Omega
  int32_t* idx = nullptr;   // [K_units] ascending units
  int32_t* inv = nullptr;   // [m] rank in idx or -1
  double* crit = nullptr;   // [m] criterion c_u
  double* adm = nullptr;    // [m] admission value (NaN if never a neighbour)
  double* r = nullptr;      // [n*block] residual (residual criterion), kept for the admission sums
  int32_t* seg_base = nullptr;  // [nseg+1] rank offsets (device)
  std::vector<int64_t> h_seg_base;   // [nseg+1] (units)
  std::vector<double> h_tau;         // [nseg]
  void release(cudaStream_t s);
};

struct lc_sub_s {
  int32_t block = 1, nseg = 1;
  int64_t K_units = 0;
  lc::Sell B;               // K_units rows/cells, segments = ranks [seg_base[g], seg_base[g+1])
  int32_t* idx = nullptr;   // [K_units] global units (owned copy)
  double* bsub = nullptr;   // [K_units*block]
  double* xB0 = nullptr;    // [K_units*block]
  std::vector<int64_t> h_seg_base;
  void release(cudaStream_t s);
};

namespace lc {

// ------------------------------------------------------------ reductions ----
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// double-double helpers (R23): (hi, lo) accumulation of sums of squares
__device__ __forceinline__ void dd_add(double& hi, double& lo, double bh, double bl) {
  double s = hi + bh;
  double bp = s - hi;
  double e = (hi - (s - bp)) + (bh - bp);
  e += lo + bl;
  double t = s + e;
  lo = e - (t - s);
  hi = t;
}
__device__ __forceinline__ void dd_add_sq(double& hi, double& lo, double v) {
  double p = v * v;
  double pe = __fma_rn(v, v, -p);
  dd_add(hi, lo, p, pe);
}
__device__ __forceinline__ void warp_dd_sum(double& hi, double& lo) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double oh = __shfl_xor_sync(0xffffffffu, hi, o), ol = __shfl_xor_sync(0xffffffffu, lo, o);
    dd_add(hi, lo, oh, ol);
  }
}

// packed (flag, value) status words for decoupled look-back
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------------------------------ launchers -----
// exclusive scan of int64 values in place: out[i] = sum_{j<i} in[j], returns total on device at out[n]
lc_status scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);
// stable compaction of units with flag[u] != 255: idx (ascending), inv, total at *count_dev
lc_status compact_flags(const uint8_t* flag, int64_t m, int32_t* idx, int32_t* inv, int64_t* count_dev,
                        cudaStream_t s);
// build slice_row0/slice_seg from seg_unit0/seg_slice0 (device)
lc_status build_slice_map(Sell& M, cudaStream_t s);

}  // namespace lc
