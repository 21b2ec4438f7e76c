// domain.cu -- lc_select_domain / lc_domain_export.
//
//   a1  residual criterion  r = b - A x0 (Alg. 3 l.4), c_u = |r| (max over a cell, R16),
//       fused with the per-slice max|r| and the double-double ||b||^2 partials (Eq. 7, R23)
//   a2  gradient criterion  g_i = sum_{j != i stored} |x0_i - x0_j| (Eq. 5) + max
//   a3  threshold           tau = eps ||b||/sqrt(N) | theta max c | nearest-rank percentile (radix select)
//   a4  mark + compact      c_u > tau (strict), ballot/popc + decoupled look-back (common.cu)
//   a5  growth              Alg. 3 expansion rounds (Eq. 8) / unconditional dilation (R15)
//
// Every per-row sum runs over the stored ascending column order with the same
// operations as the oracle (fma chain for A x, plain adds of |.| otherwise), so
// the index sets are bit-exact up to the tau rounding window (R22/R23).
#include <cmath>
#include <cstring>

#include "lc_internal.cuh"

namespace lc {

constexpr int kTB = 256;               // threads per CTA for slice kernels (8 warps)
constexpr uint8_t kOut = 255;          // flag value: not in Omega

// ---------------------------------------------------------------- a1 -------
// warp per slice; per-slice partials: cmax[s], bb_hi[s], bb_lo[s]
template <int BS>
__global__ void __launch_bounds__(kTB) k_residual_crit(SellView A, const double* __restrict__ b,
                                                       const double* __restrict__ x, double* __restrict__ r,
                                                       double* __restrict__ crit, double* __restrict__ p_max,
                                                       double* __restrict__ p_hi, double* __restrict__ p_lo) {
  int64_t s = (blockIdx.x * (int64_t)kTB + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (s >= A.nslices) return;
  int g = A.slice_seg[s];
  int64_t u = A.slice_row0[s] + lane;
  bool valid = u < A.seg_unit0[g + 1];
  int64_t p0 = A.slice_ptr[s];
  int w = A.stencil ? A.W : (int)((A.slice_ptr[s + 1] - p0) >> 5);
  double cmax = 0.0, hi = 0.0, lo = 0.0;
  if (BS == 1) {
    double acc = 0.0;
    for (int k = 0; k < w; ++k) acc = __fma_rn(sv_val(A, p0 + lane, k, u), __ldg(x + sv_col(A, p0 + lane, k, u)), acc);
    if (valid) {
      double bi = b[u];
      double ri = bi - acc;
      r[u] = ri;
      cmax = fabs(ri);
      crit[u] = cmax;
      dd_add_sq(hi, lo, bi);
    }
  } else {
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (int k = 0; k < w; ++k) {
      int64_t c = sv_col(A, p0 + lane, k, u);
      const double* vb = A.val + 9 * (p0 + 32ll * k) + lane;
      double y0 = __ldg(x + 3 * c), y1 = __ldg(x + 3 * c + 1), y2 = __ldg(x + 3 * c + 2);
      acc0 = __fma_rn(vb[0], y0, acc0); acc0 = __fma_rn(vb[32], y1, acc0); acc0 = __fma_rn(vb[64], y2, acc0);
      acc1 = __fma_rn(vb[96], y0, acc1); acc1 = __fma_rn(vb[128], y1, acc1); acc1 = __fma_rn(vb[160], y2, acc1);
      acc2 = __fma_rn(vb[192], y0, acc2); acc2 = __fma_rn(vb[224], y1, acc2); acc2 = __fma_rn(vb[256], y2, acc2);
    }
    if (valid) {
      double b0 = b[3 * u], b1 = b[3 * u + 1], b2 = b[3 * u + 2];
      double r0 = b0 - acc0, r1 = b1 - acc1, r2 = b2 - acc2;
      r[3 * u] = r0; r[3 * u + 1] = r1; r[3 * u + 2] = r2;
      cmax = fabs(r0);
      if (fabs(r1) > cmax) cmax = fabs(r1);
      if (fabs(r2) > cmax) cmax = fabs(r2);
      crit[u] = cmax;
      dd_add_sq(hi, lo, b0); dd_add_sq(hi, lo, b1); dd_add_sq(hi, lo, b2);
    }
  }
  cmax = warp_max(cmax);
  warp_dd_sum(hi, lo);
  if (lane == 0) { p_max[s] = cmax; p_hi[s] = hi; p_lo[s] = lo; }
}

// a1 for the (non-symmetric-storage) stencil layout, block 1, width WM known at compile time: the same
// per-row fma chain over slots k = 0..W-1 (holes add exact zeros), with every value load and gather of a
// row issued before the chain (no runtime slot loop), so the kernel streams at the HBM rate.
template <int WM>
__global__ void __launch_bounds__(kTB) k_residual_stencil(SellView A, const double* __restrict__ b,
                                                          const double* __restrict__ x, double* __restrict__ r,
                                                          double* __restrict__ crit, double* __restrict__ p_max,
                                                          double* __restrict__ p_hi, double* __restrict__ p_lo) {
  const int64_t s = (blockIdx.x * (int64_t)kTB + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= A.nslices) return;
  const int g = A.slice_seg[s];
  const int64_t u = A.slice_row0[s] + lane;
  const bool valid = u < A.seg_unit0[g + 1];
  const int n1 = (int)A.nunits - 1, ui = (int)u;
  const double* vp = A.val + 32ll * WM * s + lane;
  double v[WM], y[WM];
#pragma unroll
  for (int k = 0; k < WM; ++k) {
    int c = ui + A.off[k];
    c = c < 0 ? 0 : (c > n1 ? n1 : c);
    v[k] = __ldg(vp + 32 * k);
    y[k] = __ldg(x + c);
  }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < WM; ++k) acc = __fma_rn(v[k], y[k], acc);
  double cmax = 0.0, hi = 0.0, lo = 0.0;
  if (valid) {
    const double bi = b[u];
    const double ri = bi - acc;
    r[u] = ri;
    cmax = fabs(ri);
    crit[u] = cmax;
    dd_add_sq(hi, lo, bi);
  }
  cmax = warp_max(cmax);
  warp_dd_sum(hi, lo);
  if (lane == 0) { p_max[s] = cmax; p_hi[s] = hi; p_lo[s] = lo; }
}

// ---------------------------------------------------------------- a2 -------
__global__ void __launch_bounds__(kTB) k_gradient(SellView A, const double* __restrict__ x,
                                                  double* __restrict__ crit, double* __restrict__ p_max) {
  int64_t s = (blockIdx.x * (int64_t)kTB + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (s >= A.nslices) return;
  int g = A.slice_seg[s];
  int64_t u = A.slice_row0[s] + lane;
  bool valid = u < A.seg_unit0[g + 1];
  int64_t p0 = A.slice_ptr[s];
  int w = A.stencil ? A.W : (int)((A.slice_ptr[s + 1] - p0) >> 5);
  double gmax = 0.0;
  if (valid) {
    double xi = x[u], acc = 0.0;
    for (int k = 0; k < w; ++k) {
      if (!sv_real(A, k, u)) continue;                    // padding / stencil holes
      int64_t c = sv_col(A, p0 + lane, k, u);
      if (c != u) acc = acc + fabs(xi - __ldg(x + c));
    }
    crit[u] = acc;
    gmax = acc;
  }
  gmax = warp_max(gmax);
  if (lane == 0) p_max[s] = gmax;
}

// ---------------------------------------------------------------- a3 -------
// fixed-order two-level reduction of the slice partials -> tau_cmp[g], tau_rep[g]
constexpr int kTauParts = 64;
__global__ void __launch_bounds__(256) k_tau_part(SellView A, int mode, const double* __restrict__ p_max,
                                                  const double* __restrict__ p_hi, const double* __restrict__ p_lo,
                                                  double* __restrict__ q) {
  int g = blockIdx.x / kTauParts, j = blockIdx.x % kTauParts;
  int64_t s0 = A.seg_slice0[g], s1 = A.seg_slice0[g + 1];
  int64_t len = s1 - s0;
  int64_t a = s0 + len * j / kTauParts, b = s0 + len * (j + 1) / kTauParts;
  double mx = 0.0, hi = 0.0, lo = 0.0;
#pragma unroll 4
  for (int64_t s = a + threadIdx.x; s < b; s += blockDim.x) {
    mx = fmax(mx, p_max[s]);
    if (mode == LC_THR_PAPER) dd_add(hi, lo, p_hi[s], p_lo[s]);
  }
  __shared__ double sm[8], sh[8], sl[8];
  mx = warp_max(mx);
  warp_dd_sum(hi, lo);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { sm[w] = mx; sh[w] = hi; sl[w] = lo; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 8; ++i) { mx = fmax(mx, sm[i]); }
    hi = sh[0]; lo = sl[0];
    for (int i = 1; i < 8; ++i) dd_add(hi, lo, sh[i], sl[i]);
    q[3 * blockIdx.x] = mx; q[3 * blockIdx.x + 1] = hi; q[3 * blockIdx.x + 2] = lo;
  }
}

__global__ void k_tau(SellView A, int mode, double param, const double* __restrict__ q, double* tau_cmp,
                      double* tau_rep) {
  int g = blockIdx.x;
  int lane = threadIdx.x;   // blockDim = 64 = kTauParts
  const double* qq = q + 3 * (g * kTauParts + lane);
  double mx = qq[0], hi = qq[1], lo = qq[2];
  __shared__ double sm[2], sh[2], sl[2];
  mx = warp_max(mx);
  warp_dd_sum(hi, lo);
  if ((lane & 31) == 0) { sm[lane >> 5] = mx; sh[lane >> 5] = hi; sl[lane >> 5] = lo; }
  __syncthreads();
  if (lane == 0) {
    mx = fmax(sm[0], sm[1]);
    hi = sh[0]; lo = sl[0];
    dd_add(hi, lo, sh[1], sl[1]);
    double t, tc;
    if (mode == LC_THR_PAPER) {
      int64_t N = (int64_t)(A.seg_unit0[g + 1] - A.seg_unit0[g]) * A.block;   // scalar unknowns
      double nb = sqrt(hi + lo);
      t = param * nb / sqrt((double)N);                                        // Eq. 7
      tc = t;
    } else {
      t = param * mx;                                                          // Alg. 2 l.10
      tc = (param == 0.0) ? -1.0 : t;                                          // alpha = 0 => Omega (R11)
    }
    tau_cmp[g] = tc;
    tau_rep[g] = t;
  }
}

// percentile: radix select of the k-th smallest f64 bit pattern (c >= 0 => monotone), 8 x 8-bit digits
struct RadixState { unsigned long long prefix, mask; long long k; };

__global__ void k_radix_init(SellView A, double p, RadixState* st) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= A.nseg) return;
  long long m = A.seg_unit0[g + 1] - A.seg_unit0[g];
  long long k = (long long)ceil(p * (double)m) - 1;     // nearest rank (R14)
  if (k < 0) k = 0;
  if (k > m - 1) k = m - 1;
  st[g] = RadixState{0ull, 0ull, k};
}

__global__ void __launch_bounds__(kTB) k_radix_hist(const double* __restrict__ crit, int64_t m, int seg_units,
                                                    const RadixState* __restrict__ st, int shift,
                                                    unsigned* __restrict__ hist) {
  __shared__ unsigned sh[256];
  sh[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * (kTB * 8);
  int64_t last = min(base + kTB * 8, m) - 1;
  int g0 = (int)(base / seg_units), g1 = (int)(last / seg_units);
  bool one = (g0 == g1);
  for (int t = 0; t < 8; ++t) {
    int64_t u = base + t * kTB + threadIdx.x;
    if (u >= m) break;
    int g = one ? g0 : (int)(u / seg_units);
    unsigned long long key = (unsigned long long)__double_as_longlong(crit[u]);
    RadixState S = st[g];
    if ((key & S.mask) != S.prefix) continue;
    unsigned d = (unsigned)(key >> shift) & 255u;
    if (one) atomicAdd(&sh[d], 1u); else atomicAdd(&hist[g * 256 + d], 1u);
  }
  __syncthreads();
  if (one && sh[threadIdx.x]) atomicAdd(&hist[g0 * 256 + threadIdx.x], sh[threadIdx.x]);
}

__global__ void k_radix_digit(RadixState* st, unsigned* hist, int shift, double* tau_cmp, double* tau_rep,
                              int final_pass) {
  int g = blockIdx.x;
  __shared__ unsigned h[256];
  h[threadIdx.x] = hist[g * 256 + threadIdx.x];
  hist[g * 256 + threadIdx.x] = 0;   // ready for the next pass
  __syncthreads();
  if (threadIdx.x == 0) {
    RadixState S = st[g];
    long long cum = 0;
    int d = 0;
    for (; d < 255; ++d) {
      if (S.k < cum + (long long)h[d]) break;
      cum += h[d];
    }
    S.k -= cum;
    S.prefix |= (unsigned long long)d << shift;
    S.mask |= 255ull << shift;
    st[g] = S;
    if (final_pass) {
      double t = __longlong_as_double((long long)S.prefix);
      tau_cmp[g] = t;
      tau_rep[g] = t;
    }
  }
}

// a2 for the stencil layout with a compile-time width: the mask decides which slots are stored neighbours;
// all gathers of a row issue together.  Same plain adds in slot (ascending column) order as k_gradient.
template <int WM>
__global__ void __launch_bounds__(kTB) k_gradient_stencil(SellView A, const double* __restrict__ x,
                                                          double* __restrict__ crit, double* __restrict__ p_max) {
  const int64_t s = (blockIdx.x * (int64_t)kTB + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= A.nslices) return;
  const int g = A.slice_seg[s];
  const int64_t u = A.slice_row0[s] + lane;
  const bool valid = u < A.seg_unit0[g + 1];
  double gmax = 0.0;
  if (valid) {
    const int n1 = (int)A.nunits - 1, ui = (int)u;
    const unsigned m = A.mask[u];
    const double xi = __ldg(x + u);
    double y[WM];
#pragma unroll
    for (int k = 0; k < WM; ++k) {
      int c = ui + A.off[k];
      c = c < 0 ? 0 : (c > n1 ? n1 : c);
      y[k] = __ldg(x + c);
    }
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < WM; ++k)
      if (((m >> k) & 1) && A.off[k] != 0) acc = acc + fabs(xi - y[k]);
    crit[u] = acc;
    gmax = acc;
  }
  gmax = warp_max(gmax);
  if (lane == 0) p_max[s] = gmax;
}

// ---------------------------------------------------------------- a4 -------
__global__ void k_mark(const double* __restrict__ crit, int64_t m, int seg_units, const double* __restrict__ tau_cmp,
                       uint8_t* __restrict__ flag) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= m) return;
  flag[u] = (crit[u] > tau_cmp[u / seg_units]) ? 0 : kOut;      // strict (R10)
}

// ---------------------------------------------------------------- a5 -------
// Alg. 3 round `stage` (1-based): unit u not in Omega with a stored neighbour in Omega is admitted iff
// |r_u| + sum_{l in Omega, ascending} |a_ul x0_l| > tau (Eq. 8).  In Omega at round start <=> flag < stage;
// admissions write flag = stage, so the round is simultaneous.  If the previous round admitted nothing the
// kernel exits at once (l.22 break).
template <int BS>
__global__ void __launch_bounds__(kTB) k_expand(SellView A, const double* __restrict__ r,
                                                const double* __restrict__ x0, uint8_t* __restrict__ flag,
                                                const double* __restrict__ tau_cmp, int stage,
                                                double* __restrict__ adm, unsigned* counters) {
  if (stage > 1 && counters[stage - 1] == 0) return;
  int64_t s = (blockIdx.x * (int64_t)kTB + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (s >= A.nslices) return;
  int g = A.slice_seg[s];
  int64_t u = A.slice_row0[s] + lane;
  if (u >= A.seg_unit0[g + 1]) return;
  if (flag[u] < stage) return;
  int64_t p0 = A.slice_ptr[s];
  int len = sv_len(A, u);
  bool nb = false;
  double best;
  if (BS == 1) {
    double sum = 0.0;
    for (int k = 0; k < len; ++k) {
      if (!sv_real(A, k, u)) continue;
      int64_t c = sv_col(A, p0 + lane, k, u);
      if (flag[c] < stage) { nb = true; sum = sum + fabs(sv_val(A, p0 + lane, k, u) * x0[c]); }
    }
    best = fabs(r[u]) + sum;
  } else {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < len; ++k) {
      if (!sv_real(A, k, u)) continue;
      int64_t c = sv_col(A, p0 + lane, k, u);
      if (flag[c] < stage) {
        nb = true;
        const double* vb = A.val + 9 * (p0 + 32ll * k) + lane;
        double y0 = x0[3 * c], y1 = x0[3 * c + 1], y2 = x0[3 * c + 2];
        s0 = s0 + fabs(vb[0] * y0); s0 = s0 + fabs(vb[32] * y1); s0 = s0 + fabs(vb[64] * y2);
        s1 = s1 + fabs(vb[96] * y0); s1 = s1 + fabs(vb[128] * y1); s1 = s1 + fabs(vb[160] * y2);
        s2 = s2 + fabs(vb[192] * y0); s2 = s2 + fabs(vb[224] * y1); s2 = s2 + fabs(vb[256] * y2);
      }
    }
    best = fabs(r[3 * u]) + s0;
    double v1 = fabs(r[3 * u + 1]) + s1, v2 = fabs(r[3 * u + 2]) + s2;
    if (v1 > best) best = v1;
    if (v2 > best) best = v2;
  }
  if (!nb) return;
  if (adm) adm[u] = best;
  if (best > tau_cmp[g]) {
    flag[u] = (uint8_t)stage;
    atomicAdd(&counters[stage], 1u);
  }
}

// a5 expansion round for the stencil layout, block 1, compile-time width (see k_expand): flags, values
// and x0 of the row's stored neighbours are gathered together; admission sum in slot order.
template <int WM>
__global__ void __launch_bounds__(kTB) k_expand_stencil(SellView A, const double* __restrict__ r,
                                                        const double* __restrict__ x0, uint8_t* __restrict__ flag,
                                                        const double* __restrict__ tau_cmp, int stage,
                                                        double* __restrict__ adm, unsigned* counters) {
  if (stage > 1 && counters[stage - 1] == 0) return;
  const int64_t s = (blockIdx.x * (int64_t)kTB + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= A.nslices) return;
  const int g = A.slice_seg[s];
  const int64_t u = A.slice_row0[s] + lane;
  if (u >= A.seg_unit0[g + 1]) return;
  if (flag[u] < stage) return;
  const unsigned m = A.mask[u];
  const int n1 = (int)A.nunits - 1, ui = (int)u;
  const double* vp = A.val + 32ll * WM * s + lane;
  bool nb = false;
  double sum = 0.0;
  uint8_t fl[WM];
  int cc[WM];
#pragma unroll
  for (int k = 0; k < WM; ++k) {
    int c = ui + A.off[k];
    cc[k] = c < 0 ? 0 : (c > n1 ? n1 : c);
    fl[k] = flag[cc[k]];
  }
#pragma unroll
  for (int k = 0; k < WM; ++k)
    if (((m >> k) & 1) && fl[k] < stage) { nb = true; sum = sum + fabs(__ldg(vp + 32 * k) * x0[cc[k]]); }
  if (!nb) return;
  const double best = fabs(r[u]) + sum;
  if (adm) adm[u] = best;
  if (best > tau_cmp[g]) {
    flag[u] = (uint8_t)stage;
    atomicAdd(&counters[stage], 1u);
  }
}

// unconditional dilation hop: u not in Omega with a stored neighbour (!= u) in Omega joins
__global__ void __launch_bounds__(kTB) k_dilate(SellView A, uint8_t* __restrict__ flag, int stage) {
  int64_t s = (blockIdx.x * (int64_t)kTB + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (s >= A.nslices) return;
  int g = A.slice_seg[s];
  int64_t u = A.slice_row0[s] + lane;
  if (u >= A.seg_unit0[g + 1]) return;
  if (flag[u] < stage) return;
  int64_t p0 = A.slice_ptr[s];
  int len = sv_len(A, u);
  for (int k = 0; k < len; ++k) {
    if (!sv_real(A, k, u)) continue;
    int64_t c = sv_col(A, p0 + lane, k, u);
    if (c != u && flag[c] < stage) { flag[u] = (uint8_t)stage; return; }
  }
}

// segment bases: seg_base[g] = #{Omega units < seg_unit0[g]} (binary search on the ascending idx)
__global__ void k_seg_base(const int32_t* __restrict__ idx, const int64_t* __restrict__ K, int nseg,
                           const int32_t* __restrict__ seg_unit0, int32_t* seg_base) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > nseg) return;
  int64_t lo = 0, hi = *K;
  int32_t key = seg_unit0[g];
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (idx[mid] < key) lo = mid + 1; else hi = mid;
  }
  seg_base[g] = (int32_t)lo;
}

__global__ void k_expand_idx(const int32_t* __restrict__ idx, int64_t K, int bs, int32_t* out) {
  int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (l >= K) return;
  for (int a = 0; a < bs; ++a) out[l * bs + a] = idx[l] * bs + a;
}

__global__ void k_fill_nan(double* p, int64_t m) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u < m) p[u] = __longlong_as_double(0x7ff8000000000000ll);
}

}  // namespace lc

using namespace lc;

extern "C" lc_status lc_select_domain(lc_matrix M, const double* b, const double* x0, const lc_domain_params* p,
                                      void* stream, lc_domain* out, int64_t* K_host) {
  if (!out) { set_error("lc_select_domain: out is NULL"); return LC_ERR_INVALID_ARG; }
  *out = nullptr;
  if (!M || !b || !x0 || !p || !K_host) { set_error("lc_select_domain: null argument"); return LC_ERR_INVALID_ARG; }
  if (lc_status cs = check_matrix(M, "lc_select_domain")) return cs;
  const int bs = M->block;
  if (p->criterion != LC_CRIT_RESIDUAL && p->criterion != LC_CRIT_GRADIENT) {
    set_error("lc_select_domain: bad criterion"); return LC_ERR_INVALID_ARG;
  }
  if (p->criterion == LC_CRIT_GRADIENT && bs != 1) {
    set_error("lc_select_domain: the gradient criterion (Eq. 5) needs block = 1"); return LC_ERR_INVALID_ARG;
  }
  if (p->threshold == LC_THR_PAPER ? !(p->param > 0)
      : p->threshold == LC_THR_REL_MAX ? !(p->param >= 0 && p->param <= 1)
      : p->threshold == LC_THR_PERCENTILE ? !(p->param > 0 && p->param < 1) : true) {
    set_error("lc_select_domain: bad threshold / param (eps > 0, theta in [0,1], p in (0,1))");
    return LC_ERR_INVALID_ARG;
  }
  if (p->expand_rounds < 0 || p->expand_rounds > 64 || p->dilate_hops < 0 || p->dilate_hops > 64 ||
      (p->expand_rounds > 0 && p->criterion != LC_CRIT_RESIDUAL)) {
    set_error("lc_select_domain: expand_rounds in [0,64] (residual criterion only), dilate_hops in [0,64]");
    return LC_ERR_INVALID_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  Touch tA(M->use, s);
  const Sell& A = M->A;
  SellView V = view(A);
  const int64_t m = M->n, ns = A.nslices;
  const int G = M->batch;
  lc_domain_s* D = new lc_domain_s();
  D->A = M; D->m = m; D->nseg = G;
  lc_status st = LC_OK;
  void* ws = nullptr;
  double *p_max, *p_hi, *p_lo, *tau_cmp, *tau_rep;
  unsigned* counters;
  int64_t* Kdev;
  RadixState* rst;
  unsigned* hist;
  size_t off = 0;
  auto carve = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
  size_t o_pmax = carve(8 * ns), o_phi = carve(8 * ns), o_plo = carve(8 * ns), o_tc = carve(8 * G),
         o_tr = carve(8 * G), o_cnt = carve(4 * 256), o_K = carve(8), o_rst = carve(sizeof(RadixState) * G),
         o_hist = carve(4 * 256 * G), o_tq = carve(8 * 3 * kTauParts * G);
  std::vector<int32_t> h_base(G + 1);
  const unsigned nb_sl = (unsigned)((ns * 32 + kTB - 1) / kTB);
  const unsigned nb_u = (unsigned)((m + 255) / 256);
#define CK(x) do { st = (x); if (st) goto fail; } while (0)
#define CKC(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { st = cuda_fail(_e, #x); goto fail; } } while (0)
#define CKL() do { count_launch(); cudaError_t _e = cudaGetLastError(); if (_e != cudaSuccess) { st = cuda_fail(_e, "launch"); goto fail; } } while (0)
  CK(dalloc(&ws, off, s));
  p_max = (double*)((char*)ws + o_pmax); p_hi = (double*)((char*)ws + o_phi); p_lo = (double*)((char*)ws + o_plo);
  tau_cmp = (double*)((char*)ws + o_tc); tau_rep = (double*)((char*)ws + o_tr);
  counters = (unsigned*)((char*)ws + o_cnt); Kdev = (int64_t*)((char*)ws + o_K);
  rst = (RadixState*)((char*)ws + o_rst); hist = (unsigned*)((char*)ws + o_hist);
  CKC(cudaMemsetAsync(counters, 0, 4 * 256, s));
  CKC(cudaMemsetAsync(hist, 0, 4 * 256 * G, s));
  CK(dalloc((void**)&D->flag, m + 16, s));
  CK(dalloc((void**)&D->inv, sizeof(int32_t) * m, s));
  CK(dalloc((void**)&D->crit, sizeof(double) * m, s));
  CK(dalloc((void**)&D->adm, sizeof(double) * m, s));
  CK(dalloc((void**)&D->seg_base, sizeof(int32_t) * (G + 1), s));
  if (p->criterion == LC_CRIT_RESIDUAL) {
    CK(dalloc((void**)&D->r, sizeof(double) * m * bs, s));
    if (bs == 1 && A.stencil && !A.sym && A.maxw == 7)
      k_residual_stencil<7><<<nb_sl, kTB, 0, s>>>(V, b, x0, D->r, D->crit, p_max, p_hi, p_lo);
    else if (bs == 1 && A.stencil && !A.sym && A.maxw == 5)
      k_residual_stencil<5><<<nb_sl, kTB, 0, s>>>(V, b, x0, D->r, D->crit, p_max, p_hi, p_lo);
    else if (bs == 1)
      k_residual_crit<1><<<nb_sl, kTB, 0, s>>>(V, b, x0, D->r, D->crit, p_max, p_hi, p_lo);
    else
      k_residual_crit<3><<<nb_sl, kTB, 0, s>>>(V, b, x0, D->r, D->crit, p_max, p_hi, p_lo);
    CKL();
  } else {
    if (A.stencil && !A.sym && A.maxw == 7)
      k_gradient_stencil<7><<<nb_sl, kTB, 0, s>>>(V, x0, D->crit, p_max);
    else if (A.stencil && !A.sym && A.maxw == 5)
      k_gradient_stencil<5><<<nb_sl, kTB, 0, s>>>(V, x0, D->crit, p_max);
    else
      k_gradient<<<nb_sl, kTB, 0, s>>>(V, x0, D->crit, p_max);
    CKL();
  }
  k_fill_nan<<<nb_u, 256, 0, s>>>(D->adm, m);
  CKL();
  if (p->threshold == LC_THR_PERCENTILE) {
    k_radix_init<<<(G + 63) / 64, 64, 0, s>>>(V, p->param, rst);
    CKL();
    const unsigned nb_h = (unsigned)((m + kTB * 8 - 1) / (kTB * 8));
    for (int pass = 0; pass < 8; ++pass) {
      int shift = 56 - 8 * pass;
      k_radix_hist<<<nb_h, kTB, 0, s>>>(D->crit, m, M->seg_units, rst, shift, hist);
      CKL();
      k_radix_digit<<<G, 256, 0, s>>>(rst, hist, shift, tau_cmp, tau_rep, pass == 7);
      CKL();
    }
  } else {
    double* tq = (double*)((char*)ws + o_tq);
    k_tau_part<<<G * kTauParts, 256, 0, s>>>(V, p->threshold, p_max, p_hi, p_lo, tq);
    CKL();
    k_tau<<<G, kTauParts, 0, s>>>(V, p->threshold, p->param, tq, tau_cmp, tau_rep);
    CKL();
  }
  k_mark<<<nb_u, 256, 0, s>>>(D->crit, m, M->seg_units, tau_cmp, D->flag);
  CKL();
  {
    int stage = 1;
    for (int rd = 0; rd < p->expand_rounds; ++rd, ++stage) {
      if (bs == 1 && A.stencil && !A.sym && A.maxw == 7)
        k_expand_stencil<7><<<nb_sl, kTB, 0, s>>>(V, D->r, x0, D->flag, tau_cmp, stage, D->adm, counters);
      else if (bs == 1 && A.stencil && !A.sym && A.maxw == 5)
        k_expand_stencil<5><<<nb_sl, kTB, 0, s>>>(V, D->r, x0, D->flag, tau_cmp, stage, D->adm, counters);
      else if (bs == 1)
        k_expand<1><<<nb_sl, kTB, 0, s>>>(V, D->r, x0, D->flag, tau_cmp, stage, D->adm, counters);
      else
        k_expand<3><<<nb_sl, kTB, 0, s>>>(V, D->r, x0, D->flag, tau_cmp, stage, D->adm, counters);
      CKL();
    }
    for (int h = 0; h < p->dilate_hops; ++h, ++stage) {
      k_dilate<<<nb_sl, kTB, 0, s>>>(V, D->flag, stage);
      CKL();
    }
  }
  CK(dalloc((void**)&D->idx, sizeof(int32_t) * m, s));
  CK(compact_flags(D->flag, m, D->idx, D->inv, Kdev, s));
  k_seg_base<<<(G + 1 + 63) / 64, 64, 0, s>>>(D->idx, Kdev, G, A.seg_unit0, D->seg_base);
  CKL();
  D->h_tau.resize(G);
  CKC(cudaMemcpyAsync(h_base.data(), D->seg_base, sizeof(int32_t) * (G + 1), cudaMemcpyDeviceToHost, s));
  CKC(cudaMemcpyAsync(D->h_tau.data(), tau_rep, sizeof(double) * G, cudaMemcpyDeviceToHost, s));
  dfree(ws, s);
  ws = nullptr;
  CKC(cudaStreamSynchronize(s));
  D->h_seg_base.resize(G + 1);
  for (int g = 0; g <= G; ++g) D->h_seg_base[g] = h_base[g];
  D->K_units = h_base[G];
  for (int g = 0; g < G; ++g) K_host[g] = (int64_t)(h_base[g + 1] - h_base[g]) * bs;
  D->use.mark(s);
  *out = D;
  return LC_OK;
fail:
  dfree(ws, s);
  D->release(s);
  cudaStreamSynchronize(s);
  delete D;
  return st;
#undef CK
#undef CKC
#undef CKL
}

namespace lc {
// Omega's ascending scalar rows into idx_dev (device, [K_units * block]), enqueued on s without a sync
lc_status domain_rows_out(const lc_domain_s* D, int32_t* idx_dev, cudaStream_t s) {
  if (D->K_units == 0) return LC_OK;
  k_expand_idx<<<(unsigned)((D->K_units + 255) / 256), 256, 0, s>>>(D->idx, D->K_units, D->A->block, idx_dev);
  LC_LAUNCHED();
  return LC_OK;
}
}  // namespace lc

extern "C" lc_status lc_domain_export(lc_domain D, int32_t* idx_dev, double* tau_host, double* crit_dev,
                                      double* adm_dev, void* stream) {
  if (!D) { set_error("lc_domain_export: NULL handle"); return LC_ERR_INVALID_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  Touch tD(D->use, s);
  int bs = D->A->block;
  if (idx_dev && D->K_units > 0) {
    k_expand_idx<<<(unsigned)((D->K_units + 255) / 256), 256, 0, s>>>(D->idx, D->K_units, bs, idx_dev);
    LC_LAUNCHED();
  }
  if (crit_dev) LC_CUDA(cudaMemcpyAsync(crit_dev, D->crit, sizeof(double) * D->m, cudaMemcpyDeviceToDevice, s));
  if (adm_dev) LC_CUDA(cudaMemcpyAsync(adm_dev, D->adm, sizeof(double) * D->m, cudaMemcpyDeviceToDevice, s));
  if (tau_host) memcpy(tau_host, D->h_tau.data(), sizeof(double) * D->nseg);
  LC_CUDA(cudaStreamSynchronize(s));
  return LC_OK;
}

extern "C" void lc_destroy_domain(lc_domain D) {
  if (!D) return;
  D->use.order_free();
  D->release(0);
  delete D;
}
