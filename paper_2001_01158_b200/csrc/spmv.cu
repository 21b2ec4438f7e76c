// spmv.cu -- lc_spmv: y = A x (Eq. 1's operator; the product inside the residual of Alg. 3 l.4, P:670,
// and inside every Krylov iteration).  Per row the canonical chain of DESIGN.md R22: stored slots in
// ascending column order, explicit fma, so y equals the oracle's or_spmv bitwise.  One thread per row,
// one warp per 32-row slice: the stencil layout with a compile-time width (5 or 7) issues all value loads
// and gathers of a row together (the SpMV at the HBM rate, profiles/r01_v); other layouts walk the slots.
#include "lc_internal.cuh"

namespace lc {

constexpr int kVT = 256;

template <int WM>
__global__ void __launch_bounds__(kVT) k_spmv_stencil(SellView A, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t s = (blockIdx.x * (int64_t)kVT + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= A.nslices) return;
  const int g = A.slice_seg[s];
  const int64_t u = A.slice_row0[s] + lane;
  if (u >= A.seg_unit0[g + 1]) return;
  const int n1 = (int)A.nunits - 1, ui = (int)u;
  const double* vp = A.val + 32ll * WM * s + lane;
  double v[WM], xv[WM];
#pragma unroll
  for (int k = 0; k < WM; ++k) {
    int c = ui + A.off[k];
    c = c < 0 ? 0 : (c > n1 ? n1 : c);
    v[k] = __ldg(vp + 32 * k);
    xv[k] = __ldg(x + c);
  }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < WM; ++k) acc = __fma_rn(v[k], xv[k], acc);
  y[u] = acc;
}

// SELL-32 (explicit columns), block 1: the slots in groups of 4 -- the group's columns and values load
// together, then its 4 gathers, then the 4 fma of the chain in slot order (padding slots add +0).
__global__ void __launch_bounds__(kVT) k_spmv_sell(SellView A, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t s = (blockIdx.x * (int64_t)kVT + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= A.nslices) return;
  const int g = A.slice_seg[s];
  const int64_t u = A.slice_row0[s] + lane;
  if (u >= A.seg_unit0[g + 1]) return;
  const int64_t p0 = A.slice_ptr[s];
  const int w = (int)((A.slice_ptr[s + 1] - p0) >> 5);
  const int32_t* cp = A.col + p0 + lane;
  const double* vp = A.val + p0 + lane;
  double acc = 0.0;
  for (int k0 = 0; k0 < w; k0 += 4) {
    int c[4];
    double v[4], xv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool ok = k0 + j < w;
      c[j] = ok ? __ldg(cp + 32 * (k0 + j)) : 0;
      v[j] = ok ? __ldg(vp + 32 * (k0 + j)) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) xv[j] = __ldg(x + c[j]);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (k0 + j < w) acc = __fma_rn(v[j], xv[j], acc);
  }
  y[u] = acc;
}

template <int BS>
__global__ void __launch_bounds__(kVT) k_spmv(SellView A, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t s = (blockIdx.x * (int64_t)kVT + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= A.nslices) return;
  const int g = A.slice_seg[s];
  const int64_t u = A.slice_row0[s] + lane;
  if (u >= A.seg_unit0[g + 1]) return;
  const int64_t p0 = A.slice_ptr[s];
  const int w = A.stencil ? A.W : (int)((A.slice_ptr[s + 1] - p0) >> 5);
  double acc[BS];
#pragma unroll
  for (int a = 0; a < BS; ++a) acc[a] = 0.0;
  for (int k = 0; k < w; ++k) {
    const int64_t c = sv_col(A, p0 + lane, k, u);
    if (BS == 1) {
      acc[0] = __fma_rn(sv_val(A, p0 + lane, k, u), __ldg(x + c), acc[0]);
    } else {
      const double* vb = A.val + 9 * (p0 + 32ll * k) + lane;
      const double y0 = __ldg(x + 3 * c), y1 = __ldg(x + 3 * c + 1), y2 = __ldg(x + 3 * c + 2);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        acc[a] = __fma_rn(vb[32 * (3 * a)], y0, acc[a]);
        acc[a] = __fma_rn(vb[32 * (3 * a + 1)], y1, acc[a]);
        acc[a] = __fma_rn(vb[32 * (3 * a + 2)], y2, acc[a]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < BS; ++a) y[BS * u + a] = acc[a];
}

// ---- lc_spmv with the slice stream staged by TMA (stencil and SELL-32 layouts, block 1): persistent CTAs take
// chunks of kSC = 8 consecutive slices (warp w of the CTA computes slice w of the chunk, lane l its row).  The
// chunk's slots [slice_ptr[s0], slice_ptr[s0 + 8]) are contiguous and 256-byte aligned in both layouts, so thread 0
// copies its values (and, SELL, its int32 columns) into a stage of a 2-deep shared-memory ring with one or two
// cp.async.bulk per chunk, completing on the stage's mbarrier; the warps read their slots from shared memory
// (lane-consecutive, conflict-free) and gather x.  SELL chunks wider than a stage read from global memory.
constexpr int kSC = 8;                         // slices per chunk (= warps per CTA)
constexpr int kSSlots = 8 * 32 * 8;            // staged slots per chunk (8 slots per row)
constexpr int kSStage = kSSlots * 12;          // values + columns

template <int ST, int WM>
__global__ void __launch_bounds__(kVT) k_spmv_tma(SellView A, const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char ssm[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ int64_t s_p0[2];                  // first slot of the staged chunk, -1 = not staged
  const int64_t nch = (A.nslices + kSC - 1) / kSC;
  const int64_t bid = blockIdx.x, nCTA = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int64_t t) {
    const int64_t c = bid + t * nCTA;
    if (c >= nch) return;
    const int st = (int)(t & 1);
    const int64_t s0 = c * kSC, s1 = s0 + kSC < A.nslices ? s0 + kSC : A.nslices;
    const int64_t p0 = ST ? 32ll * WM * s0 : A.slice_ptr[s0];
    const int64_t p1 = ST ? 32ll * WM * s1 : A.slice_ptr[s1];
    if (p1 - p0 > kSSlots) {
      s_p0[st] = -1;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bars[st])) : "memory");
      return;
    }
    s_p0[st] = p0;
    unsigned char* sb = ssm + (size_t)st * kSStage;
    const unsigned bv = (unsigned)((p1 - p0) * 8), bc = ST ? 0u : (unsigned)((p1 - p0) * 4);
    mbar_expect_tx(&bars[st], bv + bc);
    tma_bulk_g2s(sb, A.val + p0, bv, &bars[st]);
    if (!ST) tma_bulk_g2s(sb + (size_t)kSSlots * 8, A.col + p0, bc, &bars[st]);
  };
  if (threadIdx.x == 0) { issue(0); issue(1); }
  const int n1 = (int)A.nunits - 1;
#pragma unroll 1
  for (int64_t t = 0;; ++t) {
    const int64_t c = bid + t * nCTA;
    if (c >= nch) break;
    const int st = (int)(t & 1);
    mbar_wait(&bars[st], (unsigned)((t >> 1) & 1));
    const int64_t s = c * kSC + warp;
    if (s < A.nslices) {
      const int g = A.slice_seg[s];
      const int64_t u = A.slice_row0[s] + lane;
      if (u < A.seg_unit0[g + 1]) {
        const int64_t p0 = s_p0[st];
        const int64_t ps = ST ? 32ll * WM * s : A.slice_ptr[s];
        const int w = ST ? WM : (int)((A.slice_ptr[s + 1] - ps) >> 5);
        const unsigned char* sb = ssm + (size_t)st * kSStage;
        const double* sv = p0 >= 0 ? reinterpret_cast<const double*>(sb) + (ps - p0) + lane : A.val + ps + lane;
        const int32_t* sc = p0 >= 0 ? reinterpret_cast<const int32_t*>(sb + (size_t)kSSlots * 8) + (ps - p0) + lane
                                    : A.col + ps + lane;
        double acc = 0.0;
        if (ST) {
          double v[WM > 0 ? WM : 1], xv[WM > 0 ? WM : 1];
#pragma unroll
          for (int k = 0; k < WM; ++k) {
            int cc = (int)u + A.off[k];
            cc = cc < 0 ? 0 : (cc > n1 ? n1 : cc);
            v[k] = sv[32 * k];
            xv[k] = __ldg(x + cc);
          }
#pragma unroll
          for (int k = 0; k < WM; ++k) acc = __fma_rn(v[k], xv[k], acc);
        } else {
          for (int k0 = 0; k0 < w; k0 += 4) {
            int cc[4];
            double v[4], xv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const bool ok = k0 + j < w;
              cc[j] = ok ? sc[32 * (k0 + j)] : 0;
              v[j] = ok ? sv[32 * (k0 + j)] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) xv[j] = __ldg(x + cc[j]);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (k0 + j < w) acc = __fma_rn(v[j], xv[j], acc);
          }
        }
        y[u] = acc;
      }
    }
    __syncthreads();                               // every warp is done with stage st
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();
      issue(t + 2);
    }
  }
}

// ---- CSR row-slab SpMV (SURVEY 8(a) kernel notes; the format the handles do NOT keep -- DESIGN.md s5):
// a warp owns a slab of 32 consecutive rows; its lanes copy the slab's values and columns
// [rp[r0], rp[r0 + 32]) into the warp's shared-memory slot with coalesced loads (no block-wide barrier),
// then lane l walks row r0 + l in stored order (the R22 chain, bit-exact with or_spmv) with the gathers of
// x issued in groups of 8.  Slabs with more than kCWE entries read their rows straight from global memory.
// Three dependent memory round trips per slab: the row pointers (each lane loads rp[u], rp[u + 1]; the slab's
// span comes from lanes 0 and 31 by shuffle), the slab copy (all of a lane's loads issued before its shared-memory
// stores), the x gathers.
constexpr int kCT = 256;        // threads per CTA (8 warps)
constexpr int kCWE = 256;       // staged entries per warp slab (8 per row on average)
__global__ void __launch_bounds__(kCT) k_spmv_csr(int64_t n, const int64_t* __restrict__ rp,
                                                  const int32_t* __restrict__ ci, const double* __restrict__ va,
                                                  const double* __restrict__ x, double* __restrict__ y) {
  __shared__ __align__(16) double s_v[kCT / 32][kCWE];
  __shared__ __align__(16) int32_t s_c[kCT / 32][kCWE];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * (kCT / 32) + warp) * 32;
  if (r0 >= n) return;
  const int64_t r1 = r0 + 32 < n ? r0 + 32 : n;
  const int64_t u = r0 + lane;
  const int last = (int)(r1 - r0) - 1;
  const int64_t ru0 = u < r1 ? __ldg(rp + u) : 0, ru1 = u < r1 ? __ldg(rp + u + 1) : 0;
  const int64_t e0 = __shfl_sync(0xffffffffu, ru0, 0), e1 = __shfl_sync(0xffffffffu, ru1, last);
  const int64_t ne = e1 - e0;
  double acc = 0.0;
  if (ne > kCWE) {                                        // dense slab: rows straight from global memory
    if (u < r1)
      for (int64_t k = ru0; k < ru1; ++k) acc = __fma_rn(__ldg(va + k), __ldg(x + ci[k]), acc);
  } else {
    double* sv = s_v[warp];
    int32_t* sc = s_c[warp];
    const int ni = (int)ne;
#pragma unroll
    for (int q = 0; q < kCWE / 32; q += 8) {                // 8 entries per lane in flight, then stored
      double v[8];
      int32_t c[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = lane + 32 * (q + j);
        v[j] = k < ni ? __ldg(va + e0 + k) : 0.0;
        c[j] = k < ni ? __ldg(ci + e0 + k) : 0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = lane + 32 * (q + j);
        if (k < ni) { sv[k] = v[j]; sc[k] = c[j]; }
      }
      if (32 * (q + 8) >= ni) break;
    }
    __syncwarp();
    if (u < r1) {
      const int k0 = (int)(ru0 - e0), k1 = (int)(ru1 - e0);
      for (int kb = k0; kb < k1; kb += 8) {
        double xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) xv[j] = kb + j < k1 ? __ldg(x + sc[kb + j]) : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (kb + j < k1) acc = __fma_rn(sv[kb + j], xv[j], acc);
      }
    }
  }
  if (u < r1) y[u] = acc;
}

// ---- CSR SpMV with the slab stream staged by TMA (the default when the three arrays are 16-byte aligned):
// persistent CTAs take chunks c = b + t nCTA of kCR = 256 consecutive rows (one row per thread).  Thread 0 keeps
// kCS chunks in flight: per chunk three cp.async.bulk copies into a shared-memory stage -- the chunk's row pointers
// rp[r0 .. r0 + 258), its values and its columns [rp[r0], rp[r0 + 256]) widened to 16-byte boundaries -- completing
// on the stage's mbarrier; the chunk's bounds rp[r0], rp[r0 + 256] are loaded one chunk earlier, so the copies never
// wait on them.  Each thread then walks its row in the stage (the R22 chain in stored order, gathers of x in groups
// of 8), so the DRAM stream of values / columns / row pointers no longer waits on any warp's gather latency.
// Chunks whose widened span exceeds a stage, or that touch the arrays' ends, read their rows from global memory.
constexpr int kCR = 256;                       // rows per chunk (= threads per CTA)
constexpr int kCE = 2048;                      // staged entries per chunk (8 per row on average)
constexpr int kCS = 2;                         // stages
constexpr int kStVal = (kCE + 4) * 8;          // bytes: values (span widened by up to 3 + 1 entries)
constexpr int kStCol = (kCE + 4) * 4;          // columns
constexpr int kStRp = (kCR + 2) * 8;           // row pointers rp[r0 .. r0 + kCR + 2)
constexpr int kStage = kStVal + kStCol + kStRp;
static_assert(kStVal % 16 == 0 && kStCol % 16 == 0 && kStRp % 16 == 0, "16-B stage parts");

__global__ void __launch_bounds__(kCR) k_spmv_csr_tma(int64_t n, const int64_t* __restrict__ rp,
                                                      const int32_t* __restrict__ ci, const double* __restrict__ va,
                                                      const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char csm[];
  __shared__ __align__(8) uint64_t bars[kCS];
  __shared__ int64_t s_e0[kCS];                 // widened first entry of the staged chunk, -1 = not staged
  const int64_t nch = (n + kCR - 1) / kCR;
  const int64_t bid = blockIdx.x, nCTA = gridDim.x;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int st = 0; st < kCS; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int64_t nnz = 0, b0 = 0, b1 = 0;              // thread 0: nnz and the next chunk's bounds
  auto bounds = [&](int64_t t, int64_t& e0, int64_t& e1) {
    const int64_t c = bid + t * nCTA;
    if (c >= nch) { e0 = e1 = 0; return; }
    const int64_t r0 = c * kCR, r1 = r0 + kCR < n ? r0 + kCR : n;
    e0 = __ldg(rp + r0);
    e1 = __ldg(rp + r1);
  };
  auto issue = [&](int64_t t, int64_t e0, int64_t e1) {
    const int64_t c = bid + t * nCTA;
    if (c >= nch) return;
    const int st = (int)(t % kCS);
    unsigned char* sb = csm + (size_t)st * kStage;
    const int64_t r0 = c * kCR;
    const int64_t e0a = e0 & ~(int64_t)3, e1v = (e1 + 1) & ~(int64_t)1, e1c = (e1 + 3) & ~(int64_t)3;
    const bool ok = e1c - e0a <= kCE + 4 && e1c <= nnz && r0 + kCR + 2 <= n + 1;
    if (!ok) {
      s_e0[st] = -1;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bars[st])) : "memory");
      return;
    }
    s_e0[st] = e0a;
    const unsigned bv = (unsigned)((e1v - e0a) * 8), bc = (unsigned)((e1c - e0a) * 4);
    mbar_expect_tx(&bars[st], bv + bc + kStRp);
    tma_bulk_g2s(sb + kStVal + kStCol, rp + r0, kStRp, &bars[st]);
    if (bv) tma_bulk_g2s(sb, va + e0a, bv, &bars[st]);
    if (bc) tma_bulk_g2s(sb + kStVal, ci + e0a, bc, &bars[st]);
  };
  if (tid == 0) {
    nnz = __ldg(rp + n);
    for (int t = 0; t < kCS; ++t) {
      int64_t e0, e1;
      bounds(t, e0, e1);
      issue(t, e0, e1);
    }
    bounds(kCS, b0, b1);
  }
#pragma unroll 1
  for (int64_t t = 0;; ++t) {
    const int64_t c = bid + t * nCTA;
    if (c >= nch) break;
    const int st = (int)(t % kCS);
    mbar_wait(&bars[st], (unsigned)((t / kCS) & 1));
    const int64_t u = c * kCR + tid;
    const unsigned char* sb = csm + (size_t)st * kStage;
    const int64_t e0a = s_e0[st];
    if (u < n) {
      double acc = 0.0;
      if (e0a >= 0) {
        const double* sv = reinterpret_cast<const double*>(sb);
        const int32_t* sc = reinterpret_cast<const int32_t*>(sb + kStVal);
        const int64_t* srp = reinterpret_cast<const int64_t*>(sb + kStVal + kStCol);
        const int k0 = (int)(srp[tid] - e0a), k1 = (int)(srp[tid + 1] - e0a);
        for (int kb = k0; kb < k1; kb += 8) {
          double xv[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) xv[j] = kb + j < k1 ? __ldg(x + sc[kb + j]) : 0.0;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (kb + j < k1) acc = __fma_rn(sv[kb + j], xv[j], acc);
        }
      } else {
        const int64_t k0 = __ldg(rp + u), k1 = __ldg(rp + u + 1);
        for (int64_t k = k0; k < k1; ++k) acc = __fma_rn(__ldg(va + k), __ldg(x + __ldg(ci + k)), acc);
      }
      y[u] = acc;
    }
    __syncthreads();                               // every thread is done with stage st
    if (tid == 0) {
      fence_proxy_async_smem();                    // generic reads of st before the async-proxy refill
      issue(t + kCS, b0, b1);
      bounds(t + kCS + 1, b0, b1);
    }
  }
}

}  // namespace lc

using namespace lc;

extern "C" lc_status lc_spmv(lc_matrix M, const double* x, double* y, void* stream) {
  if (!M || !x || !y) { set_error("lc_spmv: null argument"); return LC_ERR_INVALID_ARG; }
  if (x == y) { set_error("lc_spmv: x and y must not alias"); return LC_ERR_INVALID_ARG; }
  if (lc_status cs = check_matrix(M, "lc_spmv")) return cs;
  const Sell& A = M->A;
  cudaStream_t s = (cudaStream_t)stream;
  Touch tA(M->use, s);
  const unsigned nb = (unsigned)((A.nslices * 32 + kVT - 1) / kVT);
  const SellView V = view(A);
  // SELL-32 (block 1): the slice stream staged by TMA, 298 -> 289 us at 256^3 (5.66 -> 5.82 TB/s); the stencil layout
  // keeps plain loads (179 us with them, 222 us staged: its 8-byte slots leave too little in flight per stage,
  // profiles/r02_d_spmv_tma.jsonl).  lc_tuning.spmv_tma = 0: plain loads everywhere; 2: the stencil layout staged too
  if (M->block == 1 && !A.sym && tuning().spmv_tma && (!A.stencil || (tuning().spmv_tma == 2 &&
                                                                      (A.maxw == 5 || A.maxw == 7)))) {
    const void* fn = !A.stencil ? (const void*)k_spmv_tma<0, 0>
                                : A.maxw == 7 ? (const void*)k_spmv_tma<1, 7> : (const void*)k_spmv_tma<1, 5>;
    int64_t ctas = 0;
    const size_t dsm = 2 * (size_t)kSStage;
    if (lc_status st = max_coresident(fn, kVT, dsm, &ctas)) return st;
    const int64_t nch = (A.nslices + kSC - 1) / kSC;
    const unsigned grid = (unsigned)(nch < ctas ? nch : ctas);
    if (!A.stencil) k_spmv_tma<0, 0><<<grid, kVT, dsm, s>>>(V, x, y);
    else if (A.maxw == 7) k_spmv_tma<1, 7><<<grid, kVT, dsm, s>>>(V, x, y);
    else k_spmv_tma<1, 5><<<grid, kVT, dsm, s>>>(V, x, y);
    LC_LAUNCHED();
    return LC_OK;
  }
  if (M->block == 1 && A.stencil && !A.sym && A.maxw == 7)
    k_spmv_stencil<7><<<nb, kVT, 0, s>>>(V, x, y);
  else if (M->block == 1 && A.stencil && !A.sym && A.maxw == 5)
    k_spmv_stencil<5><<<nb, kVT, 0, s>>>(V, x, y);
  else if (M->block == 1 && !A.stencil)
    k_spmv_sell<<<nb, kVT, 0, s>>>(V, x, y);
  else if (M->block == 1)
    k_spmv<1><<<nb, kVT, 0, s>>>(V, x, y);
  else
    k_spmv<3><<<nb, kVT, 0, s>>>(V, x, y);
  LC_LAUNCHED();
  return LC_OK;
}

extern "C" lc_status lc_spmv_csr(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                                 const double* x, double* y, void* stream) {
  if (n < 0 || (n > 0 && (!row_ptr || !col_idx || !values || !x || !y))) {
    set_error("lc_spmv_csr: null argument or n < 0");
    return LC_ERR_INVALID_ARG;
  }
  if (x == y) { set_error("lc_spmv_csr: x and y must not alias"); return LC_ERR_INVALID_ARG; }
  if (n == 0) return LC_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const bool aligned = ((((uintptr_t)row_ptr) | ((uintptr_t)col_idx) | ((uintptr_t)values)) & 15) == 0;
  if (aligned && tuning().spmv_csr_tma) {
    int64_t ctas = 0;
    const size_t dsm = (size_t)kCS * kStage;
    if (lc_status st = max_coresident((const void*)k_spmv_csr_tma, kCR, dsm, &ctas)) return st;
    const int64_t nch = (n + kCR - 1) / kCR;
    const unsigned nb = (unsigned)(nch < ctas ? nch : ctas);
    k_spmv_csr_tma<<<nb, kCR, dsm, s>>>(n, row_ptr, col_idx, values, x, y);
    LC_LAUNCHED();
    return LC_OK;
  }
  const unsigned nb = (unsigned)((n + kCT - 1) / kCT);
  k_spmv_csr<<<nb, kCT, 0, s>>>(n, row_ptr, col_idx, values, x, y);
  LC_LAUNCHED();
  return LC_OK;
}
