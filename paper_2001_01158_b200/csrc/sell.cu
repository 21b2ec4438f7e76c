// sell.cu -- lc_create_csr: CSR/BSR input -> SELL-32 (sigma = 1) on the device,
// with on-device pattern validation and the (block-)Jacobi inverse diagonal.
#include <climits>
#include <cstdlib>
#include <cstring>

#include "lc_internal.cuh"

namespace lc {

enum : unsigned { kErrPattern = 1u, kErrZeroDiag = 2u, kErrRowLen = 4u, kErrNotStencil = 8u };

__device__ bool inv3(const double* A, double* Ai);

struct Offsets { int W; int32_t off[kMaxOff]; };
// the host-visible scratch words of lc_create_csr / lc_update_values / build_slab
constexpr int kErrOff = 64;                             // byte offset of the candidate Offsets
constexpr size_t kErrBytes = kErrOff + ((sizeof(Offsets) + 63) & ~(size_t)63);

// first row whose length equals the maximal row length (its offsets are the stencil candidate); one
// atomic per warp (most rows of a stencil have the maximal length)
__global__ void k_first_maxrow(int64_t n, const int64_t* __restrict__ rp, int maxw, int* best) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int cand = (u < n && rp[u + 1] - rp[u] == maxw) ? (int)u : INT32_MAX;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, o));
  __shared__ int s_c[32];
  if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = cand;
  __syncthreads();
  if (threadIdx.x == 0) {                    // one candidate per CTA; no atomic once a smaller one is known
    int c = INT32_MAX;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) c = min(c, s_c[i]);
    if (c != INT32_MAX && c < *(volatile int*)best) atomicMin(best, c);
  }
}

// the candidate offsets (those of the first longest row, *best) into *O, on the device (no host round trip)
__global__ void k_candidate(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, const int* best, int W,
                            Offsets* O) {
  const int k = threadIdx.x;
  const int u = *best;
  if (k < kMaxOff) O->off[k] = (k < W && u != INT32_MAX) ? ci[rp[u] + k] - u : 0;
  if (k == 0) O->W = W;
}

// every stored (u, c) must have c - u in the candidate offset set
__global__ void k_check_stencil(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const Offsets* __restrict__ Od, unsigned* err) {
  __shared__ int s_off[kMaxOff];
  __shared__ int s_w;
  if (threadIdx.x < kMaxOff) s_off[threadIdx.x] = Od->off[threadIdx.x];
  if (threadIdx.x == 0) s_w = Od->W;
  __syncthreads();
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  // the row's offsets and the candidate set are both ascending: one merge walk
  const int W = s_w;
  int k = 0;
  for (int64_t e = rp[u]; e < rp[u + 1]; ++e) {
    const int64_t d = (int64_t)ci[e] - u;
    while (k < W && s_off[k] < d) ++k;
    if (k == W || s_off[k] != d) { atomicOr(err, kErrNotStencil); return; }
    ++k;
  }
}

// stencil layout fill: thread per unit; slot k of the row = the entry at column u + off[k] (holes stay 0)
template <int BS>
__global__ void k_fill_stencil(int64_t n, int seg_units, int spg, const int64_t* __restrict__ rp,
                               const int32_t* __restrict__ ci, const double* __restrict__ va, Offsets O,
                               double* __restrict__ val, uint16_t* __restrict__ mask, double* __restrict__ dinv,
                               unsigned* err) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  int64_t g = u / seg_units, lu = u - g * seg_units;
  int64_t s = g * spg + (lu >> 5);
  int lane = (int)(lu & 31);
  unsigned m = 0;
  double D[BS * BS];
#pragma unroll
  for (int q = 0; q < BS * BS; ++q) D[q] = 0.0;
  int k = 0;
  for (int64_t e = rp[u]; e < rp[u + 1]; ++e) {
    int64_t d = (int64_t)ci[e] - u;
    while (k < O.W && O.off[k] != d) ++k;     // offsets and columns are both ascending
    m |= 1u << k;
    int64_t base = (s * O.W + k) * 32;
    if (BS == 1) {
      val[base + lane] = va[e];
      if (d == 0) D[0] = va[e];
    } else {
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        val[9 * base + 32 * q + lane] = va[9 * e + q];
        if (d == 0) D[q] = va[9 * e + q];
      }
    }
  }
  mask[u] = (uint16_t)m;
  if (BS == 1) {
    if (D[0] == 0.0) atomicOr(err, kErrZeroDiag);
    dinv[u] = 1.0 / D[0];
  } else {
    double Ai[9];
    if (!inv3(D, Ai)) atomicOr(err, kErrZeroDiag);
#pragma unroll
    for (int q = 0; q < 9; ++q) dinv[9 * u + q] = Ai[q];
  }
}

// value symmetry on the full stencil layout: every lower slot equals its mirror (row u + off[k], upper slot
// of -off[k]); a lower slot whose mirror row lies outside the segment must be a zero hole.
// compact diagonal-coupling copy of a block 3 stencil layout (Sell::cval): thread per (slice, lane)
__global__ void k_dcoup_fill(int64_t nslices, int W, int kd, const double* __restrict__ val, double* __restrict__ cval,
                             unsigned* bad) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t sl = t >> 5;
  const int lane = (int)(t & 31);
  if (sl >= nslices) return;
  const int cw = 9 + 3 * (W - 1);
  double* cb = cval + 32ll * cw * sl + lane;
  unsigned nz = 0;
  int o = 0;
  for (int k = 0; k < W; ++k) {
    const double* vb = val + 9 * (32ll * W * sl + 32ll * k) + lane;
    if (k == kd) {
#pragma unroll
      for (int q = 0; q < 9; ++q) cb[32 * q] = vb[32 * q];
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) cb[32 * (9 + 3 * o + a)] = vb[32 * (4 * a)];
#pragma unroll
      for (int q = 0; q < 9; ++q)
        if (q % 4 != 0 && vb[32 * q] != 0.0) nz = 1;
      ++o;
    }
  }
  if (nz) atomicOr(bad, 1u);
}

__global__ void k_check_sym(int64_t n, int seg_units, int spg, Offsets O, int kd, const double* __restrict__ val,
                            unsigned* bad) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t g = u / seg_units, lu = u - g * seg_units;
  const int64_t s = g * spg + (lu >> 5);
  const int lane = (int)(lu & 31);
  for (int k = 0; k < kd; ++k) {
    const double a = val[(s * O.W + k) * 32 + lane];
    const int64_t v = u + O.off[k];
    const int64_t gv = v >= 0 ? v / seg_units : -1;
    double m = 0.0;
    if (v >= 0 && gv == g) {
      const int64_t lv = v - g * seg_units, sv = g * spg + (lv >> 5);
      m = val[(sv * O.W + (O.W - 1 - k)) * 32 + (lv & 31)];
    }
    if (__double_as_longlong(a) != __double_as_longlong(m)) { atomicOr(bad, 1u); return; }
  }
}

__global__ void k_compact_upper(int64_t nslices, int W, int kd, const double* __restrict__ full,
                                double* __restrict__ up) {
  const int vw = W - kd;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nslices * vw * 32) return;
  const int64_t s = t / (vw * 32);
  const int r = (int)(t - s * vw * 32);
  up[t] = full[(s * W + kd) * 32 + r];
}

__global__ void k_uniform_slice_ptr(int64_t nslices, int W, int64_t* slice_ptr) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s <= nslices) slice_ptr[s] = 32ll * W * s;
}

// one warp per slice: validate rows, record rowlen, slice width (in slots * 32)
__global__ void k_slice_width(int64_t nslices, int seg_units, int spg, const int64_t* __restrict__ rp,
                              const int32_t* __restrict__ ci, int64_t* __restrict__ widths,
                              uint8_t* __restrict__ rowlen, unsigned* err, int* maxw) {
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  int len = 0;
  if (s < nslices) {
    const int64_t g = s / spg;
    const int64_t lu = (s - g * spg) * 32 + lane;
    const int64_t seg0 = g * (int64_t)seg_units, seg1 = seg0 + seg_units;
    if (lu < seg_units) {
      const int64_t u = seg0 + lu;
      const int64_t k0 = rp[u], k1 = rp[u + 1];
      const int64_t l = k1 - k0;
      unsigned e = 0;
      if (l < 1 || l > 255) e |= kErrRowLen;
      bool diag = false;
      int prev = -1;
      for (int64_t k = k0; k < k1 && !(e & kErrRowLen); ++k) {
        const int c = ci[k];
        if (c <= prev || c < seg0 || c >= seg1) e |= kErrPattern;
        if (c == u) diag = true;
        prev = c;
      }
      if (!diag) e |= kErrPattern;
      if (e) atomicOr(err, e);
      len = (l > 255) ? 255 : (int)l;
      rowlen[u] = (uint8_t)len;
    }
  }
  int w = len;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
  if (lane == 0 && s < nslices) widths[s] = 32ll * w;
  // one atomic per CTA for the maximal width
  __shared__ int s_w[32];
  if (lane == 0) s_w[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    int mw = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mw = max(mw, s_w[i]);
    atomicMax(maxw, mw);
  }
}

__device__ bool inv3(const double* A, double* Ai) {
  // LU without pivoting (diagonally dominant cell blocks), then solve for each unit vector
  double L10, L20, L21, U[9];
  for (int i = 0; i < 9; ++i) U[i] = A[i];
  if (U[0] == 0.0) return false;
  L10 = U[3] / U[0]; L20 = U[6] / U[0];
  U[4] -= L10 * U[1]; U[5] -= L10 * U[2];
  U[7] -= L20 * U[1]; U[8] -= L20 * U[2];
  if (U[4] == 0.0) return false;
  L21 = U[7] / U[4];
  U[8] -= L21 * U[5];
  if (U[8] == 0.0) return false;
  for (int c = 0; c < 3; ++c) {
    double y0 = (c == 0), y1 = (c == 1) - L10 * y0, y2 = (c == 2) - L20 * y0 - L21 * y1;
    double x2 = y2 / U[8];
    double x1 = (y1 - U[5] * x2) / U[4];
    double x0 = (y0 - U[1] * x1 - U[2] * x2) / U[0];
    Ai[c] = x0; Ai[3 + c] = x1; Ai[6 + c] = x2;
  }
  return isfinite(Ai[0]) && isfinite(Ai[4]) && isfinite(Ai[8]);
}

// one warp per slice: scatter rows into SELL slots (pad with col = own unit, value 0)
template <int BS>
__global__ void k_fill(int64_t nslices, int seg_units, int spg, const int64_t* __restrict__ rp,
                       const int32_t* __restrict__ ci, const double* __restrict__ va,
                       const int64_t* __restrict__ slice_ptr, int32_t* __restrict__ col, double* __restrict__ val,
                       double* __restrict__ dinv, unsigned* err) {
  int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  int64_t g = s / spg;
  int64_t lu = (s - g * spg) * 32 + lane;
  bool valid = lu < seg_units;
  int64_t u = g * (int64_t)seg_units + lu;
  int64_t p0 = slice_ptr[s];
  int w = (int)((slice_ptr[s + 1] - p0) >> 5);
  int64_t k0 = valid ? rp[u] : 0, k1 = valid ? rp[u + 1] : 0;
  double D[BS * BS];
#pragma unroll
  for (int q = 0; q < BS * BS; ++q) D[q] = 0.0;
  for (int k = 0; k < w; ++k) {
    int64_t slot = p0 + 32ll * k + lane;
    int64_t e = k0 + k;
    bool real = valid && e < k1;
    int c = real ? ci[e] : (valid ? (int)u : 0);
    col[slot] = c;
    if (BS == 1) {
      double v = real ? va[e] : 0.0;
      val[slot] = v;
      if (real && c == u) D[0] = v;
    } else {
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        double v = real ? va[9 * e + q] : 0.0;
        val[9 * (p0 + 32ll * k) + 32 * q + lane] = v;
        if (real && c == u) D[q] = v;
      }
    }
  }
  if (!valid) return;
  if (BS == 1) {
    if (D[0] == 0.0) atomicOr(err, kErrZeroDiag);
    dinv[u] = 1.0 / D[0];
  } else {
    double Ai[9];
    if (!inv3(D, Ai)) atomicOr(err, kErrZeroDiag);
#pragma unroll
    for (int q = 0; q < 9; ++q) dinv[9 * u + q] = Ai[q];
  }
}

// ------------------------------------------------------------------ slabs ----
// NEXT-4 (Alg. 4/5): rank slab = rows [row0, row0 + n) of an nglob-row matrix.  Each row must be
// ascending, inside [0, nglob), with its diagonal and at most kMaxOff entries; cs = ci - row0 (slab-relative
// columns, may leave [0, n): the halo owned by the neighbour slabs).
__global__ void k_slab_check(int64_t n, int64_t row0, int64_t nglob, const int64_t* __restrict__ rp,
                             const int32_t* __restrict__ ci, int32_t* __restrict__ cs, unsigned* err, int* maxw) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t k0 = rp[u], k1 = rp[u + 1], l = k1 - k0;
  unsigned e = 0;
  if (l < 1 || l > kMaxOffDist) e |= kErrRowLen;
  bool diag = false;
  int64_t prev = -1;
  for (int64_t k = k0; k < k1 && !(e & kErrRowLen); ++k) {
    const int64_t c = ci[k];
    if (c <= prev || c >= nglob) e |= kErrPattern;
    if (c == row0 + u) diag = true;
    prev = c;
    cs[k] = (int32_t)(c - row0);
  }
  if (!diag) e |= kErrPattern;
  if (e) atomicOr(err, e);
  atomicMax(maxw, (int)(l > 255 ? 255 : l));
}

lc_status build_slab(int64_t nglob, int64_t row0, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                     const double* values, int on_device, cudaStream_t s, Sell& A, int64_t* nnz_out) {
  lc_status st = LC_OK;
  int64_t nnz = 0, rp0 = 0;
  if (on_device) {
    LC_CUDA(cudaMemcpyAsync(&rp0, row_ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaMemcpyAsync(&nnz, row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
  } else {
    rp0 = row_ptr[0];
    nnz = row_ptr[n];
  }
  if (rp0 != 0 || nnz < n || nnz > (int64_t)kMaxOffDist * n) {
    set_error("lc_dist_create: row_ptr must start at 0 with 1..8 entries per row");
    return LC_ERR_PATTERN;
  }
  *nnz_out = nnz;
  void *t_rp = nullptr, *t_ci = nullptr, *t_va = nullptr, *t_cs = nullptr, *t_err = nullptr;
  const int64_t* d_rp = row_ptr;
  const int32_t* d_ci = col_idx;
  const double* d_va = values;
  unsigned h_err = 0;
  int h_maxw = 0;
  Offsets O;
  const unsigned nb = (unsigned)((n + 255) / 256);
#define CK(x) do { st = (x); if (st) goto done; } while (0)
#define CKC(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { st = cuda_fail(_e, #x); goto done; } } while (0)
  if (!on_device) {
    CK(dalloc(&t_rp, sizeof(int64_t) * (n + 1), s));
    CK(dalloc(&t_ci, sizeof(int32_t) * nnz, s));
    CK(dalloc(&t_va, sizeof(double) * nnz, s));
    CKC(cudaMemcpyAsync(t_rp, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    CKC(cudaMemcpyAsync(t_ci, col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s));
    CKC(cudaMemcpyAsync(t_va, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    d_rp = (const int64_t*)t_rp; d_ci = (const int32_t*)t_ci; d_va = (const double*)t_va;
  }
  CK(dalloc(&t_cs, sizeof(int32_t) * nnz, s));
  CK(dalloc(&t_err, kErrBytes, s));           // [0] error bits, [4] asymmetry, [8] max width, [12] row,
  CKC(cudaMemsetAsync(t_err, 0, kErrBytes, s)); // [16] 3T couplings not diagonal, [64] candidate offsets
  k_slab_check<<<nb, 256, 0, s>>>(n, row0, nglob, d_rp, d_ci, (int32_t*)t_cs, (unsigned*)t_err,
                                  (int*)((char*)t_err + 8));
  count_launch();
  CKC(cudaGetLastError());
  CKC(cudaMemcpyAsync(&h_err, t_err, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  CKC(cudaMemcpyAsync(&h_maxw, (char*)t_err + 8, sizeof(int), cudaMemcpyDeviceToHost, s));
  CKC(cudaStreamSynchronize(s));
  if (h_err) {
    st = LC_ERR_PATTERN;
    set_error("lc_dist_create: rows need 1..8 strictly ascending columns in [0, n_global) with the diagonal");
    goto done;
  }
  // stencil offsets: those of the slab's first longest row; every entry must match one (else not a stencil)
  {
    int big = INT32_MAX;
    CKC(cudaMemcpyAsync((char*)t_err + 12, &big, sizeof(int), cudaMemcpyHostToDevice, s));
    k_first_maxrow<<<nb, 256, 0, s>>>(n, d_rp, h_maxw, (int*)((char*)t_err + 12));
    count_launch();
    k_candidate<<<1, 32, 0, s>>>(d_rp, (const int32_t*)t_cs, (const int*)((char*)t_err + 12), h_maxw,
                                 (Offsets*)((char*)t_err + kErrOff));
    count_launch();
  }
  k_check_stencil<<<nb, 256, 0, s>>>(n, d_rp, (const int32_t*)t_cs, (const Offsets*)((char*)t_err + kErrOff),
                                     (unsigned*)t_err);
  count_launch();
  CKC(cudaMemcpyAsync(&h_err, t_err, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  CKC(cudaMemcpyAsync(&O, (char*)t_err + kErrOff, sizeof(Offsets), cudaMemcpyDeviceToHost, s));
  CKC(cudaStreamSynchronize(s));
  if (h_err & kErrNotStencil) {
    st = LC_ERR_PATTERN;
    set_error("lc_dist_create: the slab is not a constant-offset stencil (<= 8 offsets); the row-partitioned "
              "path needs the stencil layout");
    goto done;
  }
  A.block = 1; A.nunits = n; A.nseg = 1; A.maxw = h_maxw; A.stencil = 1;
  A.spg = (int)((n + 31) / 32); A.nslices = A.spg; A.reg_units = (int)n;
  for (int k = 0; k < kMaxOff; ++k) A.off[k] = O.off[k];
  A.nslots = 32ll * h_maxw * A.nslices;
  CK(dalloc((void**)&A.val, sizeof(double) * A.nslots, s));
  CK(dalloc((void**)&A.mask, sizeof(uint16_t) * n, s));
  CK(dalloc((void**)&A.dinv, sizeof(double) * n, s));
  CKC(cudaMemsetAsync(A.val, 0, sizeof(double) * A.nslots, s));
  k_fill_stencil<1><<<nb, 256, 0, s>>>(n, (int)n, A.spg, d_rp, (const int32_t*)t_cs, d_va, O, A.val, A.mask, A.dinv,
                                       (unsigned*)t_err);
  count_launch();
  CKC(cudaGetLastError());
  CKC(cudaMemcpyAsync(&h_err, t_err, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  CKC(cudaStreamSynchronize(s));
  if (h_err & kErrZeroDiag) { st = LC_ERR_ZERO_DIAGONAL; set_error("lc_dist_create: zero diagonal"); }
done:
  dfree(t_rp, s); dfree(t_ci, s); dfree(t_va, s); dfree(t_cs, s); dfree(t_err, s);
  if (st) { A.release(s); cudaStreamSynchronize(s); }
  return st;
#undef CK
#undef CKC
}

lc_status build_dcoup(Sell& A, unsigned* d_bad, cudaStream_t s) {
  if (A.block != 3 || !A.stencil || A.sym) return LC_OK;
  if (!tuning().block_dcoup) { drop_dcoup(A, s); return LC_OK; }
  int kd = -1;
  for (int k = 0; k < A.maxw; ++k)
    if (A.off[k] == 0) kd = k;
  if (kd < 0) return LC_OK;
  const int cw = 9 + 3 * (A.maxw - 1);
  if (!A.cval) {
    lc_status st = dalloc((void**)&A.cval, sizeof(double) * 32ll * cw * A.nslices, s);
    if (st) return st;
  }
  A.cw = cw;
  A.kdiag = kd;
  const unsigned nb = (unsigned)((A.nslices * 32 + 255) / 256);
  k_dcoup_fill<<<nb, 256, 0, s>>>(A.nslices, A.maxw, kd, A.val, A.cval, d_bad);
  LC_LAUNCHED();
  return LC_OK;
}
void drop_dcoup(Sell& A, cudaStream_t s) {
  dfree(A.cval, s);
  A.cval = nullptr;
  A.cw = 0;
  A.kdiag = -1;
}

}  // namespace lc

using namespace lc;

extern "C" lc_status lc_create_csr(int64_t n, int32_t block, int32_t batch, const int64_t* row_ptr,
                                   const int32_t* col_idx, const double* values, int32_t inputs_on_device,
                                   int32_t fmt, void* stream, lc_matrix* out) {
  if (!out) { set_error("lc_create_csr: out is NULL"); return LC_ERR_INVALID_ARG; }
  *out = nullptr;
  if (!row_ptr || !col_idx || !values) { set_error("lc_create_csr: null array"); return LC_ERR_INVALID_ARG; }
  if (fmt != LC_FMT_SELL32) { set_error("lc_create_csr: fmt must be LC_FMT_SELL32"); return LC_ERR_INVALID_ARG; }
  if (block != 1 && block != 3) { set_error("lc_create_csr: block must be 1 or 3"); return LC_ERR_DIMENSION; }
  if (batch < 1 || batch > 64 || n < 1 || n % batch != 0 || n / batch > (int64_t)INT32_MAX - 64 ||
      n > (int64_t)INT32_MAX - 64) {
    set_error("lc_create_csr: need n >= 1, 1 <= batch <= 64, batch | n, n < 2^31");
    return LC_ERR_DIMENSION;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int bb = block * block;
  // row_ptr end -> nnz
  // (device inputs: nnz = row_ptr[n] is read back with the validation flags below, one round trip for both)
  int64_t nnz = inputs_on_device ? n : row_ptr[n];
  if (nnz < n || nnz > (int64_t)INT32_MAX * 4) { set_error("lc_create_csr: bad nnz"); return LC_ERR_PATTERN; }

  lc_matrix_s* M = new lc_matrix_s();
  M->n = n; M->block = block; M->batch = batch; M->nnz = nnz; M->seg_units = (int32_t)(n / batch);
  Sell& A = M->A;
  A.block = block; A.nunits = n; A.nseg = batch;
  int spg = (M->seg_units + 31) / 32;
  A.nslices = (int64_t)spg * batch;
  lc_status st = LC_OK;
  const int64_t* d_rp = row_ptr;
  const int32_t* d_ci = col_idx;
  const double* d_va = values;
  void *t_rp = nullptr, *t_ci = nullptr, *t_va = nullptr, *t_w = nullptr, *t_err = nullptr;
  unsigned h_err = 0, h_bad_dc = 0;
  int h_maxw = 0;
#define CK(x) do { st = (x); if (st) goto fail; } while (0)
#define CKC(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { st = cuda_fail(_e, #x); goto fail; } } while (0)
  if (!inputs_on_device) {
    CK(dalloc(&t_rp, sizeof(int64_t) * (n + 1), s));
    CK(dalloc(&t_ci, sizeof(int32_t) * nnz, s));
    CK(dalloc(&t_va, sizeof(double) * nnz * bb, s));
    CKC(cudaMemcpyAsync(t_rp, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    CKC(cudaMemcpyAsync(t_ci, col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s));
    CKC(cudaMemcpyAsync(t_va, values, sizeof(double) * nnz * bb, cudaMemcpyHostToDevice, s));
    d_rp = (const int64_t*)t_rp; d_ci = (const int32_t*)t_ci; d_va = (const double*)t_va;
  }
  CK(dalloc(&t_w, sizeof(int64_t) * (A.nslices + 1), s));
  CK(dalloc(&t_err, kErrBytes, s));           // [0] error bits, [4] asymmetry, [8] max width, [12] row,
  CKC(cudaMemsetAsync(t_err, 0, kErrBytes, s)); // [16] 3T couplings not diagonal, [64] candidate offsets
  CK(dalloc((void**)&A.rowlen, n, s));
  CK(dalloc((void**)&A.slice_ptr, sizeof(int64_t) * (A.nslices + 1), s));
  {
    unsigned blocks = (unsigned)((A.nslices * 32 + 255) / 256);
    k_slice_width<<<blocks, 256, 0, s>>>(A.nslices, M->seg_units, spg, d_rp, d_ci, (int64_t*)t_w, A.rowlen,
                                         (unsigned*)t_err, (int*)((char*)t_err + 8));
    count_launch();
    CKC(cudaGetLastError());
  }
  CK(scan_exclusive_i64((const int64_t*)t_w, A.slice_ptr, A.nslices, s));
  CKC(cudaMemcpyAsync(&A.nslots, A.slice_ptr + A.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CKC(cudaMemcpyAsync(&h_err, t_err, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  CKC(cudaMemcpyAsync(&h_maxw, (char*)t_err + 8, sizeof(int), cudaMemcpyDeviceToHost, s));
  if (inputs_on_device) CKC(cudaMemcpyAsync(&nnz, row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CKC(cudaStreamSynchronize(s));
  if (inputs_on_device) {
    if (nnz < n || nnz > (int64_t)INT32_MAX * 4) { st = LC_ERR_PATTERN; set_error("lc_create_csr: bad nnz"); goto fail; }
    M->nnz = nnz;
  }
  if (h_err) {
    st = (h_err & kErrRowLen) ? LC_ERR_PATTERN : LC_ERR_PATTERN;
    set_error(h_err & kErrRowLen ? "lc_create_csr: row length must be in [1, 255]"
                                 : "lc_create_csr: columns must be strictly ascending, inside the row's "
                                   "segment, with the diagonal stored");
    goto fail;
  }
  A.maxw = h_maxw;
  CK(dalloc((void**)&A.dinv, sizeof(double) * n * bb, s));
  {
    // ---- stencil detection: candidate offsets = those of the first longest row
    if (h_maxw <= kMaxOff && tuning().stencil_layout) {
      int big = INT32_MAX;
      CKC(cudaMemcpyAsync((char*)t_err + 12, &big, sizeof(int), cudaMemcpyHostToDevice, s));
      unsigned nb = (unsigned)((n + 255) / 256);
      k_first_maxrow<<<nb, 256, 0, s>>>(n, d_rp, h_maxw, (int*)((char*)t_err + 12));
      count_launch();
      // candidate offsets gathered and checked on the device: one host round trip for the layout decision
      k_candidate<<<1, 32, 0, s>>>(d_rp, d_ci, (const int*)((char*)t_err + 12), h_maxw, (Offsets*)((char*)t_err + kErrOff));
      count_launch();
      k_check_stencil<<<nb, 256, 0, s>>>(n, d_rp, d_ci, (const Offsets*)((char*)t_err + kErrOff), (unsigned*)t_err);
      count_launch();
      Offsets O;
      CKC(cudaMemcpyAsync(&h_err, t_err, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
      CKC(cudaMemcpyAsync(&O, (char*)t_err + kErrOff, sizeof(Offsets), cudaMemcpyDeviceToHost, s));
      CKC(cudaStreamSynchronize(s));
      if (!(h_err & kErrNotStencil)) {
        A.stencil = 1;
        for (int k = 0; k < kMaxOff; ++k) A.off[k] = O.off[k];
        A.nslots = 32ll * h_maxw * A.nslices;
        CK(dalloc((void**)&A.val, sizeof(double) * A.nslots * bb, s));
        CK(dalloc((void**)&A.mask, sizeof(uint16_t) * n, s));
        CKC(cudaMemsetAsync(A.val, 0, sizeof(double) * A.nslots * bb, s));
        k_uniform_slice_ptr<<<(unsigned)((A.nslices + 256) / 256), 256, 0, s>>>(A.nslices, h_maxw, A.slice_ptr);
        count_launch();
        if (block == 1)
          k_fill_stencil<1><<<nb, 256, 0, s>>>(n, M->seg_units, spg, d_rp, d_ci, d_va, O, A.val, A.mask, A.dinv,
                                               (unsigned*)t_err);
        else
          k_fill_stencil<3><<<nb, 256, 0, s>>>(n, M->seg_units, spg, d_rp, d_ci, d_va, O, A.val, A.mask, A.dinv,
                                               (unsigned*)t_err);
        count_launch();
        CKC(cudaGetLastError());
        // ---- symmetric stencil?  offsets symmetric and values equal to their mirrors (block 1)
        bool offsym = (h_maxw % 2 == 1) && block == 1;
        for (int k = 0; k < h_maxw && offsym; ++k) offsym = (O.off[k] == -O.off[h_maxw - 1 - k]);
        if (offsym && tuning().symmetric_layout) {       // opt-in (slower in the PCG)
          const int kd = h_maxw / 2;
          unsigned bad = 0;
          CKC(cudaMemsetAsync((char*)t_err + 4, 0, 4, s));
          k_check_sym<<<nb, 256, 0, s>>>(n, M->seg_units, spg, O, kd, A.val, (unsigned*)((char*)t_err + 4));
          count_launch();
          CKC(cudaMemcpyAsync(&bad, (char*)t_err + 4, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
          CKC(cudaStreamSynchronize(s));
          if (!bad) {
            const int vw = h_maxw - kd;
            double* up = nullptr;
            CK(dalloc((void**)&up, sizeof(double) * 32 * vw * A.nslices, s));
            const int64_t tot = 32ll * vw * A.nslices;
            k_compact_upper<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(A.nslices, h_maxw, kd, A.val, up);
            count_launch();
            k_uniform_slice_ptr<<<(unsigned)((A.nslices + 256) / 256), 256, 0, s>>>(A.nslices, vw, A.slice_ptr);
            count_launch();
            CKC(cudaGetLastError());
            dfree(A.val, s);
            A.val = up;
            A.sym = 1; A.kd = kd; A.vw = vw;
            A.nslots = tot;
            for (int k = 0; k < kd; ++k) A.mir[k] = (h_maxw - 1 - k) - kd;
          }
        }
      } else {
        h_err = 0;
        CKC(cudaMemsetAsync(t_err, 0, sizeof(unsigned), s));
      }
    }
  }
  if (!A.stencil) {
    CK(dalloc((void**)&A.col, sizeof(int32_t) * A.nslots, s));
    CK(dalloc((void**)&A.val, sizeof(double) * A.nslots * bb, s));
    unsigned blocks = (unsigned)((A.nslices * 32 + 255) / 256);
    if (block == 1)
      k_fill<1><<<blocks, 256, 0, s>>>(A.nslices, M->seg_units, spg, d_rp, d_ci, d_va, A.slice_ptr, A.col, A.val,
                                       A.dinv, (unsigned*)t_err);
    else
      k_fill<3><<<blocks, 256, 0, s>>>(A.nslices, M->seg_units, spg, d_rp, d_ci, d_va, A.slice_ptr, A.col, A.val,
                                       A.dinv, (unsigned*)t_err);
    count_launch();
    CKC(cudaGetLastError());
  }
  A.reg_units = M->seg_units;
  A.spg = spg;
  // segment maps
  A.h_seg_unit0.resize(batch + 1);
  A.h_seg_slice0.resize(batch + 1);
  for (int g = 0; g <= batch; ++g) { A.h_seg_unit0[g] = g * M->seg_units; A.h_seg_slice0[g] = (int64_t)g * spg; }
  CK(dalloc((void**)&A.seg_unit0, sizeof(int32_t) * (batch + 1), s));
  CK(dalloc((void**)&A.seg_slice0, sizeof(int64_t) * (batch + 1), s));
  CKC(cudaMemcpyAsync(A.seg_unit0, A.h_seg_unit0.data(), sizeof(int32_t) * (batch + 1), cudaMemcpyHostToDevice, s));
  CKC(cudaMemcpyAsync(A.seg_slice0, A.h_seg_slice0.data(), sizeof(int64_t) * (batch + 1), cudaMemcpyHostToDevice, s));
  CK(dalloc((void**)&A.slice_row0, sizeof(int32_t) * A.nslices, s));
  CK(dalloc((void**)&A.slice_seg, sizeof(int32_t) * A.nslices, s));
  CK(build_slice_map(A, s));
  if (A.stencil && block == 3) CK(build_dcoup(A, (unsigned*)((char*)t_err + 16), s));   // 3T couplings
  CKC(cudaMemcpyAsync(&h_err, t_err, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  CKC(cudaMemcpyAsync(&h_bad_dc, (char*)t_err + 16, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  CKC(cudaStreamSynchronize(s));
  if (h_err & kErrZeroDiag) {
    st = LC_ERR_ZERO_DIAGONAL;
    set_error("lc_create_csr: zero diagonal (or singular 3x3 cell block)");
    goto fail;
  }
  if (h_bad_dc) drop_dcoup(A, s);                // an off-diagonal block is not diagonal: full blocks only
  dfree(t_rp, s); dfree(t_ci, s); dfree(t_va, s); dfree(t_w, s); dfree(t_err, s);
  M->use.mark(s);
  *out = M;
  return LC_OK;
fail:
  dfree(t_rp, s); dfree(t_ci, s); dfree(t_va, s); dfree(t_w, s); dfree(t_err, s);
  A.release(s);
  cudaStreamSynchronize(s);
  delete M;
  return st;
#undef CK
#undef CKC
}

extern "C" lc_status lc_matrix_info(lc_matrix A, int64_t* n_unknowns, int64_t* nnz, int32_t* batch,
                                    int64_t* nslices, int32_t* max_row, int32_t* layout, int64_t* matrix_bytes) {
  if (!A) { set_error("lc_matrix_info: NULL handle"); return LC_ERR_INVALID_ARG; }
  const int bb = A->block * A->block;
  if (layout) *layout = A->A.sym ? LC_LAYOUT_SYMSTENCIL : A->A.stencil ? LC_LAYOUT_STENCIL : LC_LAYOUT_SELL;
  if (matrix_bytes)
    *matrix_bytes = A->A.cval ? (int64_t)8 * 32 * A->A.cw * A->A.nslices    // compact 3T couplings (GMRES)
                  : A->A.stencil ? (int64_t)8 * bb * A->A.nslots
                                 : (int64_t)(8 * bb + 4) * A->A.nslots + 8 * (A->A.nslices + 1) + 8 * A->A.nslices;
  if (n_unknowns) *n_unknowns = A->n * A->block;
  if (nnz) *nnz = A->nnz * A->block * A->block;
  if (batch) *batch = A->batch;
  if (nslices) *nslices = A->A.nslices;
  if (max_row) *max_row = A->A.maxw;
  return LC_OK;
}

extern "C" void lc_destroy_matrix(lc_matrix A) {
  if (!A) return;
  A->use.order_free();
  A->A.release(0);
  delete A;
}

// New values for the pattern A was created with (the systems of a time-step / Picard sequence share their
// mesh): refills the layout in place, skipping pattern validation and layout detection.
extern "C" lc_status lc_update_values(lc_matrix M, const int64_t* row_ptr, const int32_t* col_idx,
                                      const double* values, int32_t inputs_on_device, void* stream) {
  if (!M || !row_ptr || !col_idx || !values) { set_error("lc_update_values: null argument"); return LC_ERR_INVALID_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  Touch tA(M->use, s);
  Sell& A = M->A;
  const int64_t n = M->n;
  const int bb = M->block * M->block;
  const int spg = (M->seg_units + 31) / 32;
  const int64_t nnz = M->nnz;
  const int64_t* d_rp = row_ptr;
  const int32_t* d_ci = col_idx;
  const double* d_va = values;
  void *t_rp = nullptr, *t_ci = nullptr, *t_va = nullptr, *t_err = nullptr, *t_full = nullptr;
  lc_status st = LC_OK;
  unsigned h_err = 0;
#define CK(x) do { st = (x); if (st) goto fail; } while (0)
#define CKC(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { st = cuda_fail(_e, #x); goto fail; } } while (0)
  if (!inputs_on_device) {
    CK(dalloc(&t_rp, sizeof(int64_t) * (n + 1), s));
    CK(dalloc(&t_ci, sizeof(int32_t) * nnz, s));
    CK(dalloc(&t_va, sizeof(double) * nnz * bb, s));
    CKC(cudaMemcpyAsync(t_rp, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    CKC(cudaMemcpyAsync(t_ci, col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s));
    CKC(cudaMemcpyAsync(t_va, values, sizeof(double) * nnz * bb, cudaMemcpyHostToDevice, s));
    d_rp = (const int64_t*)t_rp; d_ci = (const int32_t*)t_ci; d_va = (const double*)t_va;
  }
  CK(dalloc(&t_err, kErrBytes, s));           // [0] error bits, [4] asymmetry, [8] max width, [12] row,
  CKC(cudaMemsetAsync(t_err, 0, kErrBytes, s)); // [16] 3T couplings not diagonal, [64] candidate offsets
  M->valid = 0;                 // the fill below overwrites the live layout; valid again once the checks pass
  {
    const unsigned nb = (unsigned)((n + 255) / 256);
    if (A.stencil) {
      Offsets O;
      O.W = A.maxw;
      for (int k = 0; k < kMaxOff; ++k) O.off[k] = A.off[k];
      double* dst = A.val;
      if (A.sym) {                                  // refill a full-width buffer, check symmetry, compact
        CK(dalloc(&t_full, sizeof(double) * 32ll * A.maxw * A.nslices, s));
        CKC(cudaMemsetAsync(t_full, 0, sizeof(double) * 32ll * A.maxw * A.nslices, s));
        dst = (double*)t_full;
      }
      if (M->block == 1)
        k_fill_stencil<1><<<nb, 256, 0, s>>>(n, M->seg_units, spg, d_rp, d_ci, d_va, O, dst, A.mask, A.dinv,
                                             (unsigned*)t_err);
      else
        k_fill_stencil<3><<<nb, 256, 0, s>>>(n, M->seg_units, spg, d_rp, d_ci, d_va, O, dst, A.mask, A.dinv,
                                             (unsigned*)t_err);
      count_launch();
      CKC(cudaGetLastError());
      if (A.sym) {
        k_check_sym<<<nb, 256, 0, s>>>(n, M->seg_units, spg, O, A.kd, dst, (unsigned*)((char*)t_err + 4));
        count_launch();
        const int64_t tot = 32ll * A.vw * A.nslices;
        k_compact_upper<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(A.nslices, A.maxw, A.kd, dst, A.val);
        count_launch();
        CKC(cudaGetLastError());
      }
    } else {
      const unsigned blocks = (unsigned)((A.nslices * 32 + 255) / 256);
      if (M->block == 1)
        k_fill<1><<<blocks, 256, 0, s>>>(A.nslices, M->seg_units, spg, d_rp, d_ci, d_va, A.slice_ptr, A.col, A.val,
                                         A.dinv, (unsigned*)t_err);
      else
        k_fill<3><<<blocks, 256, 0, s>>>(A.nslices, M->seg_units, spg, d_rp, d_ci, d_va, A.slice_ptr, A.col, A.val,
                                         A.dinv, (unsigned*)t_err);
      count_launch();
      CKC(cudaGetLastError());
    }
  }
  if (A.stencil && M->block == 3) CK(build_dcoup(A, (unsigned*)((char*)t_err + 16), s));
  {
    unsigned e2[2] = {0, 0}, bad_dc = 0;
    CKC(cudaMemcpyAsync(e2, t_err, 8, cudaMemcpyDeviceToHost, s));
    CKC(cudaMemcpyAsync(&bad_dc, (char*)t_err + 16, 4, cudaMemcpyDeviceToHost, s));
    CKC(cudaStreamSynchronize(s));
    h_err = e2[0] | (e2[1] ? kErrNotStencil : 0u);
    if (bad_dc) drop_dcoup(A, s);
  }
  if (h_err & kErrZeroDiag) { st = LC_ERR_ZERO_DIAGONAL; set_error("lc_update_values: zero diagonal"); goto fail; }
  if (h_err & kErrNotStencil) {
    st = LC_ERR_PATTERN;
    set_error("lc_update_values: values no longer symmetric (symmetric stencil layout); recreate the matrix");
    goto fail;
  }
  M->valid = 1;
fail:
  dfree(t_rp, s); dfree(t_ci, s); dfree(t_va, s); dfree(t_err, s); dfree(t_full, s);
  if (st) cudaStreamSynchronize(s);
  return st;
#undef CK
#undef CKC
}
