// extract.cu -- lc_extract_sub: B = A[Omega, Omega] in local numbering
// (Eq. 2), b_sub = b_B - E x_C^(0) (Eq. 3), x_B0 = x0[Omega], and B's
// (block-)Jacobi inverse diagonal, in one gather pass.  B is stored as SELL-32 with
// the uniform width of A's longest row, so no count pass is needed; each segment of
// a batched system keeps its own slices (local ranks [seg_base[g], seg_base[g+1])).
#include <cstring>

#include <cstdlib>

#include "lc_internal.cuh"

namespace lc {

constexpr int kTB = 256;

// out[l] = v[idx[l]] (masked subsystems keep b_sub / x_B0 in A's row numbering)
__global__ void k_gather_rows(const double* __restrict__ v, const int32_t* __restrict__ idx, int64_t K,
                              double* __restrict__ out) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l < K) out[l] = v[idx[l]];
}

template <int BS>
__global__ void __launch_bounds__(kTB) k_extract(SellView A, SellView B, int W, const int32_t* __restrict__ idx,
                                                 const int32_t* __restrict__ inv, const double* __restrict__ b,
                                                 const double* __restrict__ x0, int32_t* __restrict__ Bcol,
                                                 double* __restrict__ Bval, uint8_t* __restrict__ Browlen,
                                                 double* __restrict__ Bdinv, double* __restrict__ bsub,
                                                 double* __restrict__ xB0, int64_t* __restrict__ Bslice_ptr) {
  int64_t sB = (blockIdx.x * (int64_t)kTB + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (sB >= B.nslices) return;
  if (lane == 0) {
    Bslice_ptr[sB] = 32ll * W * sB;
    if (sB == B.nslices - 1) Bslice_ptr[sB + 1] = 32ll * W * (sB + 1);
  }
  int g = B.slice_seg[sB];
  int64_t row0 = B.slice_row0[sB];
  int64_t l = row0 + lane;
  bool valid = l < B.seg_unit0[g + 1];
  const int64_t pB = 32ll * W * sB;
  int kb = 0;
  if (valid) {
    int64_t i = idx[l];
    int64_t lu = i - A.seg_unit0[g];
    int64_t sA = A.seg_slice0[g] + (lu >> 5);
    int laneA = (int)(lu & 31);
    int64_t pA = A.slice_ptr[sA];
    int len = sv_len(A, i);
    double acc[BS];
#pragma unroll
    for (int a = 0; a < BS; ++a) acc[a] = 0.0;
    for (int k = 0; k < len; ++k) {
      if (!sv_real(A, k, i)) continue;                 // padding / stencil holes
      int64_t c = sv_col(A, pA + laneA, k, i);
      int ic = inv[c];
      if (ic >= 0) {                                   // B block: column in local numbering
        int64_t slotB = pB + 32ll * kb + lane;
        Bcol[slotB] = ic;
        if (BS == 1) {
          Bval[slotB] = sv_val(A, pA + laneA, k, i);
        } else {
#pragma unroll
          for (int q = 0; q < 9; ++q)
            Bval[9 * (pB + 32ll * kb) + 32 * q + lane] = A.val[9 * (pA + 32ll * k) + 32 * q + laneA];
        }
        ++kb;
      } else {                                         // E x_C^(0): fma chain, ascending columns
        if (BS == 1) {
          acc[0] = __fma_rn(sv_val(A, pA + laneA, k, i), x0[c], acc[0]);
        } else {
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int be = 0; be < 3; ++be)
              acc[a] = __fma_rn(A.val[9 * (pA + 32ll * k) + 32 * (3 * a + be) + laneA], x0[3 * c + be], acc[a]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < BS; ++a) {
      bsub[BS * l + a] = b[BS * i + a] - acc[a];
      xB0[BS * l + a] = x0[BS * i + a];
    }
#pragma unroll
    for (int q = 0; q < BS * BS; ++q) Bdinv[BS * BS * l + q] = A.dinv[BS * BS * i + q];
    Browlen[l] = (uint8_t)kb;
  }
  int padc = valid ? (int)l : (int)row0;
  for (int k = kb; k < W; ++k) {
    int64_t slotB = pB + 32ll * k + lane;
    Bcol[slotB] = padc;
    if (BS == 1) {
      Bval[slotB] = 0.0;
    } else {
#pragma unroll
      for (int q = 0; q < 9; ++q) Bval[9 * (pB + 32ll * k) + 32 * q + lane] = 0.0;
    }
  }
}

// Masked representation (stencil-layout A, block 1): per Omega row i (global numbering)
//   bs[i]  = b_i - (fma chain over stored columns outside Omega, ascending)   (Eq. 3)
//   xm0[i] = x0_i,  and the slice of i is marked active.
__global__ void __launch_bounds__(kTB) k_bsub_masked(SellView A, int seg_units, int spg,
                                                     const int32_t* __restrict__ idx, int64_t K,
                                                     const int32_t* __restrict__ inv, const double* __restrict__ b,
                                                     const double* __restrict__ x0, double* __restrict__ bs,
                                                     double* __restrict__ xm0, uint8_t* __restrict__ sflag) {
  int64_t l = blockIdx.x * (int64_t)kTB + threadIdx.x;
  if (l >= K) return;
  int64_t i = idx[l];
  int64_t g = i / seg_units, lu = i - g * seg_units;
  int64_t s = g * spg + (lu >> 5);
  int laneA = (int)(lu & 31);
  int64_t pA = A.slice_ptr[s];
  double acc = 0.0;
  for (int k = 0; k < A.W; ++k) {
    if (!sv_real(A, k, i)) continue;
    int64_t c = sv_col(A, pA + laneA, k, i);
    if (inv[c] < 0) acc = __fma_rn(sv_val(A, pA + laneA, k, i), x0[c], acc);
  }
  bs[i] = b[i] - acc;
  xm0[i] = x0[i];
  sflag[s] = 0;
}

// lseg[g] = first position in the ascending slice list with slice >= g * spg (segment runs)
__global__ void k_seg_list_start(const int32_t* __restrict__ slist, const int64_t* __restrict__ nlist, int G,
                                 int spg, int64_t* lseg) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > G) return;
  int64_t lo = 0, hi = *nlist;
  int64_t key = (int64_t)g * spg;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (slist[mid] < key) lo = mid + 1; else hi = mid;
  }
  lseg[g] = lo;
}

}  // namespace lc

using namespace lc;

extern "C" lc_status lc_extract_sub(lc_matrix M, lc_domain D, const double* b, const double* x0, void* stream,
                                    lc_sub* out) {
  if (!out) { set_error("lc_extract_sub: out is NULL"); return LC_ERR_INVALID_ARG; }
  *out = nullptr;
  if (!M || !D || !b || !x0 || D->A != M) {
    set_error("lc_extract_sub: null argument or domain of another matrix");
    return LC_ERR_INVALID_ARG;
  }
  if (lc_status cs = check_matrix(M, "lc_extract_sub")) return cs;
  cudaStream_t s = (cudaStream_t)stream;
  Touch tA(M->use, s), tD(D->use, s);
  const int bs = M->block, G = M->batch, bb = bs * bs;
  lc_sub_s* S = new lc_sub_s();
  S->block = bs; S->nseg = G; S->K_units = D->K_units; S->h_seg_base = D->h_seg_base;
  Sell& B = S->B;
  B.block = bs; B.nunits = D->K_units; B.nseg = G; B.maxw = M->A.maxw;
  B.h_seg_unit0.resize(G + 1);
  B.h_seg_slice0.resize(G + 1);
  int64_t nsl = 0;
  for (int g = 0; g <= G; ++g) {
    B.h_seg_unit0[g] = (int32_t)D->h_seg_base[g];
    B.h_seg_slice0[g] = nsl;
    if (g < G) nsl += (D->h_seg_base[g + 1] - D->h_seg_base[g] + 31) / 32;
  }
  B.nslices = nsl;
  B.nslots = 32ll * B.maxw * nsl;
  B.uniform = 1;                 // every slice maxw slots wide (k_extract pads with zero slots)
  if (S->K_units == 0) { S->use.mark(s);
  *out = S; return LC_OK; }
  lc_status st = LC_OK;
  const int64_t K = S->K_units;
  const int64_t n = M->n;
#define CK(x) do { st = (x); if (st) goto fail; } while (0)
#define CKC(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { st = cuda_fail(_e, #x); goto fail; } } while (0)
  // Stencil layouts: the masked representation (below) sweeps A's slices that hold Omega rows, so its cost
  // follows the slices' fill; an Omega of at most half the rows that is too large for the cluster-resident
  // kernel gets the explicit B instead (SELL, 12 B/nnz, only Omega rows): config 5 method2 (eta 0.093, slices
  // 54% filled) local solve 8.70 -> 6.07 ms, config 2 method1 2.31 -> 1.92 ms, config 3 (20 groups) 4.27 ->
  // 3.78 ms; near-full domains (config 5 method1: 44 vs 62 ms) and small ones keep the masked form.
  // lc_tuning.sub_repr = 0 / 1 forces either.
  bool masked = M->A.stencil && bs == 1;
  if (masked && 2 * K <= n && K >= 65536) masked = false;
  if (tuning().sub_repr == 0) masked = false;
  if (tuning().sub_repr == 1 && M->A.stencil && bs == 1) masked = true;
  if (masked) {
    // ---- masked representation: B = A[Omega, Omega] applied implicitly on A's stencil layout
    S->masked = 1;
    S->A = M;
    const int64_t nsA = M->A.nslices;
    const int spg = (M->seg_units + 31) / 32;
    void* t = nullptr;
    CK(dalloc((void**)&S->bs, sizeof(double) * n, s));
    CK(dalloc((void**)&S->xm0, sizeof(double) * n, s));
    CK(dalloc((void**)&S->omega, n, s));
    CK(dalloc((void**)&S->slist, sizeof(int32_t) * nsA, s));
    CK(dalloc((void**)&S->nlist, sizeof(int64_t), s));
    CK(dalloc(&t, (sizeof(int32_t) + 1) * nsA + 16, s));
    CKC(cudaMemsetAsync(S->bs, 0, sizeof(double) * n, s));
    CKC(cudaMemsetAsync(S->xm0, 0, sizeof(double) * n, s));
    CKC(cudaMemcpyAsync(S->omega, D->flag, n, cudaMemcpyDeviceToDevice, s));
    CK(dalloc((void**)&S->idx, sizeof(int32_t) * K, s));                 // Omega's rows, for lc_sub_export
    CKC(cudaMemcpyAsync(S->idx, D->idx, sizeof(int32_t) * K, cudaMemcpyDeviceToDevice, s));
    {
      uint8_t* sflag = (uint8_t*)t;
      int32_t* sinv = (int32_t*)((char*)t + ((nsA + 15) & ~(int64_t)15));
      CKC(cudaMemsetAsync(sflag, 255, nsA, s));
      k_bsub_masked<<<(unsigned)((K + kTB - 1) / kTB), kTB, 0, s>>>(view(M->A), M->seg_units, spg, D->idx, K, D->inv,
                                                                   b, x0, S->bs, S->xm0, sflag);
      count_launch();
      CKC(cudaGetLastError());
      CK(compact_flags(sflag, nsA, S->slist, sinv, S->nlist, s));
      CK(dalloc((void**)&S->lseg, sizeof(int64_t) * (G + 1), s));
      k_seg_list_start<<<(G + 1 + 63) / 64, 64, 0, s>>>(S->slist, S->nlist, G, spg, S->lseg);
      count_launch();
      CKC(cudaGetLastError());
    }
    dfree(t, s);
    S->use.mark(s);
  *out = S;
    return LC_OK;
  }
  CK(dalloc((void**)&B.seg_unit0, sizeof(int32_t) * (G + 1), s));
  CK(dalloc((void**)&B.seg_slice0, sizeof(int64_t) * (G + 1), s));
  CKC(cudaMemcpyAsync(B.seg_unit0, D->seg_base, sizeof(int32_t) * (G + 1), cudaMemcpyDeviceToDevice, s));
  CKC(cudaMemcpyAsync(B.seg_slice0, B.h_seg_slice0.data(), sizeof(int64_t) * (G + 1), cudaMemcpyHostToDevice, s));
  CK(dalloc((void**)&B.slice_row0, sizeof(int32_t) * nsl, s));
  CK(dalloc((void**)&B.slice_seg, sizeof(int32_t) * nsl, s));
  CK(build_slice_map(B, s));
  CK(dalloc((void**)&B.slice_ptr, sizeof(int64_t) * (nsl + 1), s));
  CK(dalloc((void**)&B.col, sizeof(int32_t) * B.nslots, s));
  CK(dalloc((void**)&B.val, sizeof(double) * B.nslots * bb, s));
  CK(dalloc((void**)&B.rowlen, K, s));
  CK(dalloc((void**)&B.dinv, sizeof(double) * K * bb, s));
  CK(dalloc((void**)&S->bsub, sizeof(double) * K * bs, s));
  CK(dalloc((void**)&S->xB0, sizeof(double) * K * bs, s));
  CK(dalloc((void**)&S->idx, sizeof(int32_t) * K, s));
  CKC(cudaMemcpyAsync(S->idx, D->idx, sizeof(int32_t) * K, cudaMemcpyDeviceToDevice, s));
  {
    unsigned nb = (unsigned)((nsl * 32 + kTB - 1) / kTB);
    SellView VA = view(M->A), VB = view(B);
    if (bs == 1)
      k_extract<1><<<nb, kTB, 0, s>>>(VA, VB, B.maxw, D->idx, D->inv, b, x0, B.col, B.val, B.rowlen, B.dinv, S->bsub,
                                      S->xB0, B.slice_ptr);
    else
      k_extract<3><<<nb, kTB, 0, s>>>(VA, VB, B.maxw, D->idx, D->inv, b, x0, B.col, B.val, B.rowlen, B.dinv, S->bsub,
                                      S->xB0, B.slice_ptr);
    count_launch();
    CKC(cudaGetLastError());
  }
  S->use.mark(s);
  *out = S;
  return LC_OK;
fail:
  S->release(s);
  cudaStreamSynchronize(s);
  delete S;
  return st;
#undef CK
#undef CKC
}

extern "C" lc_status lc_sub_export(lc_sub S, double* bsub_dev, double* xB0_dev, void* stream) {
  if (!S) { set_error("lc_sub_export: NULL handle"); return LC_ERR_INVALID_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  Touch tS(S->use, s);
  const int64_t len = S->K_units * S->block;
  if (len > 0) {
    if (S->masked) {                       // global numbering on A's rows: gather the Omega rows in order
      if (bsub_dev) {
        k_gather_rows<<<(unsigned)((len + kTB - 1) / kTB), kTB, 0, s>>>(S->bs, S->idx, len, bsub_dev);
        LC_LAUNCHED();
      }
      if (xB0_dev) {
        k_gather_rows<<<(unsigned)((len + kTB - 1) / kTB), kTB, 0, s>>>(S->xm0, S->idx, len, xB0_dev);
        LC_LAUNCHED();
      }
    } else {
      if (bsub_dev) LC_CUDA(cudaMemcpyAsync(bsub_dev, S->bsub, sizeof(double) * len, cudaMemcpyDeviceToDevice, s));
      if (xB0_dev) LC_CUDA(cudaMemcpyAsync(xB0_dev, S->xB0, sizeof(double) * len, cudaMemcpyDeviceToDevice, s));
    }
  }
  LC_CUDA(cudaStreamSynchronize(s));
  return LC_OK;
}

extern "C" void lc_destroy_sub(lc_sub S) {
  if (!S) return;
  S->use.order_free();
  S->release(0);
  delete S;
}
