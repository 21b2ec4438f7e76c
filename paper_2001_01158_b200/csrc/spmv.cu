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

}  // namespace lc

using namespace lc;

extern "C" lc_status lc_spmv(lc_matrix M, const double* x, double* y, void* stream) {
  if (!M || !x || !y) { set_error("lc_spmv: null argument"); return LC_ERR_INVALID_ARG; }
  if (x == y) { set_error("lc_spmv: x and y must not alias"); return LC_ERR_INVALID_ARG; }
  const Sell& A = M->A;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned nb = (unsigned)((A.nslices * 32 + kVT - 1) / kVT);
  const SellView V = view(A);
  if (M->block == 1 && A.stencil && !A.sym && A.maxw == 7)
    k_spmv_stencil<7><<<nb, kVT, 0, s>>>(V, x, y);
  else if (M->block == 1 && A.stencil && !A.sym && A.maxw == 5)
    k_spmv_stencil<5><<<nb, kVT, 0, s>>>(V, x, y);
  else if (M->block == 1)
    k_spmv<1><<<nb, kVT, 0, s>>>(V, x, y);
  else
    k_spmv<3><<<nb, kVT, 0, s>>>(V, x, y);
  LC_LAUNCHED();
  return LC_OK;
}
