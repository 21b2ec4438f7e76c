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
constexpr int kMaxOff = 16;  // stencil layout: at most 16 slots (offsets) per row (9-point 2-D, 15-point 3-D)
constexpr int kMaxOffDist = 8;  // the row-partitioned form (NEXT-4): its kernels hold <= 8 slots

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

// Completion of one Krylov launch.  Every solver kernel leaves (iterations, status, relative residual) per
// segment in device memory; the host copies them out behind the launch.  Immediate mode (the lc_solve_* entry
// points) synchronises the stream and fills lc_solve_info.  Deferred mode (lc_local_method, Alg. 1 in one call)
// copies them into a Pending record in pinned host memory and returns at once; the caller reads it after its one
// synchronisation at the end (pending_info).
constexpr int kMaxSegs = 64;
struct Pending {
  int32_t it[kMaxSegs];
  int32_t stt[kMaxSegs];
  double rr[kMaxSegs];
  cudaEvent_t e0 = nullptr, e1 = nullptr;   // bracket the launch (timing events, owned by the record)
  int G = 0, kernel = 0, lazy = 1, armed = 0;
};
// events bracketing a solve launch: the Pending record's when deferred, else created (and destroyed) here
struct SolveClock {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  bool own = false;
  explicit SolveClock(Pending* pend);
  ~SolveClock();
  SolveClock(const SolveClock&) = delete;
  SolveClock& operator=(const SolveClock&) = delete;
};
// after the launch (clk.e1 recorded, launch error in e): copy the G per-segment outputs behind it.  Immediate
// (pend == nullptr): synchronise, fill info[0..G) and return the worst status (errors set lc_last_error).
// Deferred: return LC_OK unless the copies could not be enqueued.
lc_status solve_finish(cudaError_t e, SolveClock& clk, Pending* pend, int G, const int* d_it, const int* d_stt,
                       const double* d_rr, int kernel, int lazy, cudaStream_t s, lc_solve_info* info,
                       const char* what);
// a deferred record after the caller's synchronisation -> info[0..G), worst status
lc_status pending_info(const Pending& pend, lc_solve_info* info);

// one Krylov solve for run_pcg (pcg.cu)
struct Sell;
struct PcgJob {
  const Sell* M = nullptr;        // operator layout
  const double* b = nullptr;      // right-hand side in M's numbering
  double* x = nullptr;            // iterate updated in place (x_init == nullptr)
  const double* x_init = nullptr; // else: solve on a workspace copy of x_init
  const int32_t* slist = nullptr; // optional active-slice list, device count at nlist_dev
  const int64_t* nlist_dev = nullptr;
  const int64_t* lseg = nullptr;  // [G+1] start of each segment's run in slist
  int64_t nlist_max = 0;          // host upper bound of the list length
  const uint8_t* omega = nullptr; // masked solve: rows with omega[u] != 255
  const int32_t* scatter_idx = nullptr;  // explicit local solve: x_full[scatter_idx[l]] = x[l]
  double* x_full = nullptr;
  double* x_user = nullptr;       // masked local solve: x_user[u] = x[u] on Omega
  int reg_units = 0, spg = 0;     // equal segments of reg_units units with spg slices each (A), else 0
  int64_t rows_hint = -1;         // rows the solve works on (masked: K), -1 = all; picks team mode for G > 1
  Pending* defer = nullptr;       // deferred completion (lc_local_method), else immediate
};

// small single-segment stencil systems: the cluster-resident PCG (pcg_dsmem.cu)
bool pcg_dsmem_eligible(const PcgJob& job);
lc_status run_pcg_dsmem(const PcgJob& job, const lc_solver_params* p, cudaStream_t s, lc_solve_info* info);

// stream-ordered device allocation (pool with unlimited release threshold)
lc_status dalloc(void** p, size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);
int num_sms();                                   // SMs of the calling thread's current device (cached per device)
int64_t l2_bytes();                              // L2 cache size of the current device (cached per device)
// whether a solve whose passes stream `matrix_bytes` once and re-read `vector_bytes` should mark the matrix
// stream evict_first (see l2_evict_first_policy): lc_tuning.l2_stream_hint -1 = this rule, 0 / 1 force
bool stream_policy_wanted(int64_t matrix_bytes, int64_t vector_bytes);
// co-resident CTAs (occupancy x SMs) of `fn` on the current device, cached per (device, fn, threads, smem); opts the
// function into > 48 KB of dynamic shared memory on that device first when needed
lc_status max_coresident(const void* fn, int threads, size_t dsmem, int64_t* ctas);
// co-resident clusters of `cl` CTAs of `fn` (cudaOccupancyMaxActiveClusters), cached like max_coresident
lc_status max_clusters(const void* fn, int threads, size_t dsmem, int cl, int64_t* clusters);
// cudaFuncSetAttribute once per (device, fn, attribute) (function attributes are per device context)
lc_status func_attr(const void* fn, cudaFuncAttribute attr, int value);
// the calling thread's tuning (lc_set_tuning; defaults otherwise)
const lc_tuning& tuning();
// scoped stream-ordered workspace: freed on every return path (also the early LC_CUDA error returns)
struct DevBuf {
  void* p = nullptr;
  cudaStream_t s;
  explicit DevBuf(cudaStream_t st) : s(st) {}
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { dfree(p, s); }
  lc_status alloc(size_t bytes) { return dalloc(&p, bytes, s); }
};

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
  // stencil layout: every row's column offsets (col - row) lie in one sorted set off[0..W);
  // slot k of a row holds the entry at column row + off[k] or a zero "hole"; no col array is stored.
  int stencil = 0;
  int32_t off[kMaxOff] = {0};
  uint16_t* mask = nullptr;       // [nunits] bit k = slot k holds a stored entry (stencil layout)
  // symmetric stencil layout (block 1, a_uv == a_vu bitwise): only slots k >= kd (diagonal + upper offsets)
  // are stored, vw = W - kd per slice; a lower slot's value is read from the mirror row's upper slot mir[k]
  int sym = 0, kd = 0, vw = 0;
  int32_t mir[kMaxOff] = {0};
  int reg_units = 0, spg = 0;     // equal segments (matrices from lc_create_csr)
  int uniform = 0;                // SELL with every slice maxw slots wide (slice_ptr[s] = 32 maxw s): explicit B
  // block 3 stencil layout whose off-diagonal 3x3 blocks are diagonal (the 3T couplings): a compact
  // copy of the values without the blocks' explicit zeros for the Krylov SpMVs -- per slice, the diagonal block's 9
  // components, then 3 per off-diagonal slot in slot order (cw = 9 + 3 (W - 1) doubles per lane); kdiag = the slot
  // with offset 0.  Skipping exact zeros leaves every fma chain bitwise unchanged (the chains never hold -0).
  double* cval = nullptr;
  int cw = 0, kdiag = -1;
  std::vector<int32_t> h_seg_unit0;
  std::vector<int64_t> h_seg_slice0;
  void release(cudaStream_t s);
};

// Device view passed by value to kernels
struct SellView {
  int block;
  int stencil;              // 1: col(u, k) = u + off[k] (clamped), real(u, k) = mask[u] bit k
  int W;                    // stencil width (= maxw)
  int32_t off[kMaxOff];
  const uint16_t* mask;
  int64_t nunits;
  int sym, kd, vw;          // symmetric stencil storage (see Sell)
  int32_t mir[kMaxOff];
  int ru, spg;
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
  const double* cval;       // compact diagonal-coupling values (block 3 stencil) or nullptr
  int cw, kdiag;
};
inline SellView view(const Sell& m) {
  SellView v;
  v.block = m.block; v.stencil = m.stencil; v.W = m.maxw;
  for (int k = 0; k < kMaxOff; ++k) v.off[k] = m.off[k];
  v.mask = m.mask; v.nunits = m.nunits;
  v.sym = m.sym; v.kd = m.kd; v.vw = m.stencil ? (m.sym ? m.vw : m.maxw) : (m.uniform ? m.maxw : 0);
  for (int k = 0; k < kMaxOff; ++k) v.mir[k] = m.mir[k];
  v.ru = m.reg_units; v.spg = m.spg;
  v.nslices = m.nslices; v.nseg = m.nseg; v.slice_ptr = m.slice_ptr; v.slice_row0 = m.slice_row0;
  v.slice_seg = m.slice_seg; v.seg_unit0 = m.seg_unit0; v.seg_slice0 = m.seg_slice0; v.col = m.col;
  v.val = m.val; v.rowlen = m.rowlen; v.dinv = m.dinv;
  v.cval = m.cval; v.cw = m.cw; v.kdiag = m.kdiag;
  return v;
}

// column of slot k of unit u (lane offset pl = slice_ptr[s] + lane); stencil: u + off[k] clamped to [0, n)
__device__ __forceinline__ int64_t sv_col(const SellView& A, int64_t pl, int k, int64_t u) {
  if (A.stencil) {
    int64_t c = u + A.off[k];
    return c < 0 ? 0 : (c >= A.nunits ? A.nunits - 1 : c);
  }
  return A.col[pl + 32ll * k];
}
// value of scalar slot k of unit u (pl = slice_ptr[s] + lane, as for sv_col)
__device__ __forceinline__ double sv_val(const SellView& A, int64_t pl, int k, int64_t u) {
  if (!A.sym) return A.val[pl + 32ll * k];
  if (k >= A.kd) return A.val[pl + 32ll * (k - A.kd)];
  const int64_t v = u + A.off[k];              // mirror entry a_vu (row v, upper slot mir[k])
  if (v < 0) return 0.0;
  const int64_t g = v / A.ru, lv = v - g * A.ru;
  const int64_t sv = g * A.spg + (lv >> 5);
  return A.val[32ll * A.vw * sv + 32ll * A.mir[k] + (lv & 31)];
}
// slot k of unit u holds a stored entry (not padding, not a hole)
__device__ __forceinline__ bool sv_real(const SellView& A, int k, int64_t u) {
  return A.stencil ? ((A.mask[u] >> k) & 1) : (k < A.rowlen[u]);
}
// number of slots to walk for unit u
__device__ __forceinline__ int sv_len(const SellView& A, int64_t u) { return A.stencil ? A.W : A.rowlen[u]; }

// --------------------------------------------------------------- handles ----
// The last stream a handle was used on: every entry point records an event there when it returns, and the
// destroy call makes the legacy stream wait for it before the stream-ordered frees, so a handle destroyed
// while a non-synchronising call (lc_spmv, lc_extract_sub) is still running on a side stream keeps its
// memory until that work is done -- without a host synchronisation.
struct LastUse {
  cudaEvent_t ev = nullptr;
  void mark(cudaStream_t s) {
    if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) { ev = nullptr; cudaGetLastError(); }
    if (ev) cudaEventRecord(ev, s);
  }
  void order_free() {
    if (ev) { cudaStreamWaitEvent(0, ev, 0); cudaEventDestroy(ev); ev = nullptr; }
  }
};
struct Touch {               // marks `u` on scope exit (all return paths)
  LastUse& u;
  cudaStream_t s;
  Touch(LastUse& use, cudaStream_t st) : u(use), s(st) {}
  ~Touch() { u.mark(s); }
};
}  // namespace lc

struct lc_matrix_s {
  int64_t n = 0;            // units (rows or cells)
  int32_t block = 1, batch = 1;
  int64_t nnz = 0;          // stored blocks / scalars of the input
  int32_t seg_units = 0;    // n / batch
  lc::Sell A;
  int valid = 1;            // 0 after a failed lc_update_values (values half-written): calls refuse the handle
  int pattern_sym = -1;     // structural symmetry of the pattern (lc_smooth_gs, general layout): -1 unknown
  lc::LastUse use;
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
  lc::LastUse use;
  void release(cudaStream_t s);
};

struct lc_sub_s {
  int32_t block = 1, nseg = 1;
  int64_t K_units = 0;
  // masked representation (stencil-layout A, block 1): B = A[Omega, Omega] applied implicitly on A's layout
  int masked = 0;
  lc_matrix_s* A = nullptr;       // the matrix handle (must outlive the sub)
  double* bs = nullptr;           // [n] b_sub on Omega rows (global numbering), 0 elsewhere
  double* xm0 = nullptr;          // [n] x0 on Omega rows, 0 elsewhere
  uint8_t* omega = nullptr;       // [n] copy of the domain flags (255 = outside Omega)
  int32_t* slist = nullptr;       // active slices of A (ascending), count at *nlist
  int64_t* nlist = nullptr;
  int64_t* lseg = nullptr;        // [nseg+1] start of segment g's slices in slist
  // explicit representation (otherwise)
  lc::Sell B;               // K_units rows/cells, segments = ranks [seg_base[g], seg_base[g+1])
  int32_t* idx = nullptr;   // [K_units] global units (owned copy)
  double* bsub = nullptr;   // [K_units*block]
  double* xB0 = nullptr;    // [K_units*block]
  std::vector<int64_t> h_seg_base;
  lc::LastUse use;
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

// Grid-wide barriers for cooperative (co-resident) launches.  The whole struct must be zero at launch.
//
// grid_barrier: a counter barrier.  Each CTA adds 1 to one 64-bit counter with a fire-and-forget
// red.release (no round trip) and polls it with relaxed loads until it reaches epoch x gridDim.x, then one
// acquire fence: one one-way trip plus one poll on the critical path.  Measured on B200 (tools/micro/
// barrier_bench.cu): 2.2 us per barrier at 592 CTAs, 1.4 us at 296, 1.3 us at 148, against 3.3-3.6 us for
// the arrival-tree + generation-word form below, whose last arriver needs its atomic's result back before
// it can release the others.  `epoch` is the caller's per-CTA barrier count (start at 0, same sequence of
// barriers in every CTA).
//
// The arrival tree (sub-counters, top counter, generation word) is kept for tree_reduce_barrier, which
// reduces partials inside it.  Two-level arrival: CTA b arrives on sub-counter b % kBarSub (each on its own
// 128-B line), the last arriver of each sub-group arrives on the top counter, the last of those releases
// the generation.
constexpr int kBarSub = 16;
struct GridBar {
  unsigned sub[kBarSub][32];
  unsigned top;
  unsigned gen;
  unsigned pad[30];
  unsigned long long ctr;       // counter barrier
  unsigned long long pad2[15];
  unsigned long long done;      // tree_reduce_barrier: sub-group sums published
  unsigned long long pad3[15];
};
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void grid_barrier(GridBar* gb, unsigned long long& epoch) {
  __syncthreads();                                    // the CTA's writes precede thread 0's release (bar.sync)
  epoch += gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&gb->ctr) : "memory");
    unsigned long long v;
    do {
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&gb->ctr) : "memory");
    } while (v < epoch);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

// the same counter barrier over `count` co-resident CTAs of a team (its own counter; epoch as above)
__device__ __forceinline__ void team_barrier(unsigned long long* ctr, unsigned long long& epoch, unsigned count) {
  __syncthreads();
  epoch += count;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned long long v;
    do {
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
    } while (v < epoch);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

// out[t] = sum over the members m_i = first + i step (i < count, ascending) of part[m_i T + t], t < T <= 128:
// warp w sums a contiguous range of members, then the NW warp sums are added in warp order (fixed order);
// the block has NW warps.  A lane issues the loads of up to 8 members at once and then adds them in order, so
// a range costs one L2 round trip instead of one per member (on the barrier's critical path).
template <int NW, int TMAX>
__device__ __forceinline__ void sum_members(const double* part, int T, unsigned first, unsigned step, unsigned count,
                                            double* out, double (*s_tmp)[TMAX]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned per = (count + NW - 1) / NW;
  const unsigned i0 = warp * per, i1 = min(count, i0 + per);
  for (int t = lane; t < T; t += 32) {
    double a = 0.0;
    for (unsigned ib = i0; ib < i1; ib += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        v[q] = ib + q < i1 ? __ldcg(part + (size_t)(first + (ib + q) * step) * T + t) : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (ib + q < i1) a += v[q];
    }
    s_tmp[warp][t] = a;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += NW * 32) {
    double a = 0.0;
    for (int w = 0; w < NW; ++w) a += s_tmp[w][t];
    out[t] = a;
  }
}

// Grid barrier that also reduces the per-CTA partials part[b][0..T) (batched solves, G > 1), with no atomic
// round trip on its critical path: CTA b announces its arrival on sub-group counter k = b % kBarSub with a
// fire-and-forget red.release; CTA k (the sub-group's reducer) polls that counter until all its members arrived,
// sums their partials in CTA order into subred[epoch & 1][k] and announces it on the `done` counter; every CTA
// polls `done` until all reducers finished and sums the kBarSub sub-group sums in order itself, into s_out[t]
// (shared memory).  Counters are monotonic (epoch = the caller's count of these barriers, from 0); subred is
// double-buffered by epoch (a reducer can only start epoch e + 2 after every CTA has left epoch e + 1, hence read
// epoch e).  Fixed order everywhere, so every CTA holds bitwise identical sums.  The earlier form (last arriver
// of each sub-group found by an atomicAdd, a second atomic level, a generation word) took 7.8 us from the last
// arrival to the first CTA out on config 3 (per-CTA timeline, tools/tl_cta.py); see DESIGN s6.
template <int NW, int TMAX>
__device__ void tree_reduce_barrier(GridBar* gb, const double* part, double* subred, double* s_out, int T,
                                    double (*s_tmp)[TMAX], unsigned& epoch) {
  const unsigned nb = gridDim.x, b = blockIdx.x;
  const unsigned nsub = nb < (unsigned)kBarSub ? nb : (unsigned)kBarSub;
  const unsigned e = ++epoch;
  double* sr = subred + (size_t)(e & 1) * kBarSub * T;
  __syncthreads();                                    // the CTA's partials precede thread 0's release (bar.sync)
  if (threadIdx.x == 0) {
    unsigned long long* c = reinterpret_cast<unsigned long long*>(&gb->sub[b % kBarSub][0]);
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(c) : "memory");
  }
  if (b < nsub) {                                     // reducer of sub-group b
    const unsigned nk = (nb - b + kBarSub - 1) / kBarSub;
    if (threadIdx.x == 0) {
      const unsigned long long* c = reinterpret_cast<const unsigned long long*>(&gb->sub[b][0]);
      const unsigned long long want = (unsigned long long)e * nk;
      unsigned long long v;
      do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(c) : "memory");
      } while (v < want);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    sum_members<NW, TMAX>(part, T, b, kBarSub, nk, sr + (size_t)b * T, s_tmp);
    __syncthreads();                                  // the sums precede thread 0's release
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&gb->done) : "memory");
  }
  if (threadIdx.x == 0) {
    const unsigned long long want = (unsigned long long)e * nsub;
    unsigned long long v;
    do {
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&gb->done) : "memory");
    } while (v < want);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += NW * 32) {
    double v[kBarSub];
#pragma unroll
    for (int k = 0; k < kBarSub; ++k) v[k] = k < (int)nsub ? __ldcg(sr + (size_t)k * T + t) : 0.0;
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < kBarSub; ++k)
      if (k < (int)nsub) a += v[k];
    s_out[t] = a;
  }
  __syncthreads();
}

// Reducing grid barrier for a cooperative launch in thread-block clusters of CL CTAs (batched PCG, G > 1): the
// cluster's CTA partials s_mine[0..T) are summed in rank order through distributed shared memory by its rank-0 CTA
// (one barrier.cluster, CL DSMEM loads in flight per value), which stores the cluster partial into
// part[e & 1][cluster] and arrives on the counter with a fire-and-forget red.release; every CTA polls the counter
// until all nclu clusters arrived and sums the cluster partials itself into s_out (fixed order: thread (c, t) adds
// the members of chunk c of value t in order, then the chunk sums in order), so every CTA holds bitwise identical
// sums.  One level of global latency instead of tree_reduce_barrier's two (sub-group reducers, then a done
// counter): 4.5 vs 6.8 us per barrier at T = 40 on B200 (tools/micro/reduce_bench.cu).  part is double-buffered
// by epoch: a cluster writes epoch e + 2 only after every cluster arrived at e + 1, i.e. after every CTA finished
// reading epoch e.  A CTA's s_mine is read by its rank 0 before that rank arrives, and no CTA leaves the barrier
// before every rank 0 arrived, so s_mine may be rewritten right after the barrier.  `ctr_target` is the caller's
// running target (start 0); the kernel must end with a cluster sync (DSMEM lifetime).
template <int NT, int TMAX>
__device__ void cluster_reduce_barrier(GridBar* gb, double* part, const double* s_mine, double* s_out, int T,
                                       double* s_chunk, unsigned long long& ctr_target, unsigned& epoch) {
  namespace cgx = cooperative_groups;
  cgx::cluster_group cl = cgx::this_cluster();
  const unsigned CL = cl.num_blocks(), rank = cl.block_rank();
  const unsigned nclu = gridDim.x / CL, cid = blockIdx.x / CL;
  const unsigned e = epoch++;
  double* pt = part + (size_t)(e & 1) * nclu * T;
  cl.sync();                                          // the cluster's partials are in place (release / acquire)
  ctr_target += nclu;
  if (rank == 0) {
    for (int t = threadIdx.x; t < T; t += NT) {
      double v[16];
#pragma unroll
      for (unsigned r = 0; r < 16; ++r) v[r] = r < CL ? cl.map_shared_rank(s_mine, r)[t] : 0.0;
      double a = 0.0;
#pragma unroll
      for (unsigned r = 0; r < 16; ++r)
        if (r < CL) a += v[r];
      pt[(size_t)cid * T + t] = a;
    }
    __syncthreads();                                  // the cluster partial precedes thread 0's release
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&gb->ctr) : "memory");
  }
  if (threadIdx.x == 0) {
    unsigned long long v;
    do {
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&gb->ctr) : "memory");
    } while (v < ctr_target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
  // chunks of >= 4 members per thread, consecutive threads on consecutive values (coalesced rows of pt)
  int C = NT / T;
  const int cmax = ((int)nclu + 3) / 4;
  if (C > cmax) C = cmax;
  if (C < 1) C = 1;
  const int per = ((int)nclu + C - 1) / C;
  for (int i = threadIdx.x; i < C * T; i += NT) {
    const int c = i / T, t = i - c * T;
    const int m0 = c * per, m1 = min((int)nclu, m0 + per);
    double a = 0.0;
    for (int mb = m0; mb < m1; mb += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = mb + q < m1 ? __ldcg(pt + (size_t)(mb + q) * T + t) : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (mb + q < m1) a += v[q];
    }
    s_chunk[i] = a;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += NT) {
    double a = 0.0;
    for (int c = 0; c < C; ++c) a += s_chunk[c * T + t];
    s_out[t] = a;
  }
  __syncthreads();
}

// ---- TMA (bulk async copy) + mbarrier helpers (sm_90+ PTX; SASS UBLKCP / SYNCS) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// L2 eviction policy for the streams that are read once per pass (matrix values, column indices).  The vectors
// of a Krylov iteration are re-read within the iteration and, when they fit L2, across iterations; the matrix
// stream is not, and marked evict_first it stops displacing them.  The launchers decide (stream_policy_wanted):
// the hint pays when the whole working set exceeds L2 but the vectors are of about its size (config 2 global
// PCG 24.6 -> 23.0 us per iteration, config 5's explicit local subsystem 4.91 -> 4.31 ms, config 3 batched
// global 37.7 -> 35.7 ms); it changes nothing for systems far larger than L2 (config 5 global: +0.5%) and
// L2-resident ones keep plain loads (config 3's local teams were 3.5% slower with hinted loads).
// the policy word of a kernel's matrix stream: evict_first when `stream`, else evict_normal (what a plain load
// gets) -- one register pair per thread, so the loads below are single instructions whatever the choice
__device__ __forceinline__ unsigned long long l2_stream_policy(bool stream) {
  unsigned long long a, b;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(a));
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(b));
  return stream ? a : b;
}
// read-only value load with an L2 policy word
__device__ __forceinline__ double ldg_pol(const double* p, unsigned long long pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
// 1-D bulk copy global -> shared, completing `bytes` of transaction count on `bar` (16-B aligned, multiple of 16)
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// the same copy with an L2 policy word
__device__ __forceinline__ void tma_bulk_g2s_pol(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                                 unsigned long long pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
      ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// ------------------------------------------------------------ launchers -----
// exclusive scan of int64 values in place: out[i] = sum_{j<i} in[j], returns total on device at out[n]
lc_status scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);
// stable compaction of units with flag[u] != 255: idx (ascending), inv, total at *count_dev
lc_status compact_flags(const uint8_t* flag, int64_t m, int32_t* idx, int32_t* inv, int64_t* count_dev,
                        cudaStream_t s);
// build slice_row0/slice_seg from seg_unit0/seg_slice0 (device)
lc_status build_slice_map(Sell& M, cudaStream_t s);
// LC_ERR_INVALID_ARG (with a message naming `where`) for a null handle or one a failed lc_update_values left
// half-written
lc_status check_matrix(const lc_matrix_s* M, const char* where);
// block 3 stencil layout: (re)build A.cval from A.val and raise *d_bad if an off-diagonal block holds a nonzero
// off-diagonal entry (the caller reads *d_bad after its sync and drops cval then: drop_dcoup)
lc_status build_dcoup(Sell& A, unsigned* d_bad, cudaStream_t s);
void drop_dcoup(Sell& A, cudaStream_t s);
// NEXT-4: stencil layout of the rank slab [row0, row0 + n) of an nglob-row matrix (sell.cu)
lc_status build_slab(int64_t nglob, int64_t row0, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                     const double* values, int on_device, cudaStream_t s, Sell& A, int64_t* nnz_out);

}  // namespace lc
