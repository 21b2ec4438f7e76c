// pcg.cu -- Jacobi-preconditioned CG as ONE persistent cooperative kernel
// (SURVEY 8(a) a7 local solve, a8 assembly, a9 global solve, a10 method0).
//
// The Krylov loop never returns to the host: scalars live in shared memory,
// reductions are fixed-order (per-CTA partials, then every CTA that needs a
// segment's scalar sums that segment's partials in the same order), and two
// grid-wide barriers separate the two fused passes of an iteration:
//
//   pass A  q = A p with the p-update p = z + beta p_old applied on the fly to
//           every operand (own row written to the other p buffer), fused with
//           the p^T q partials;                    [or r = b - A x for INIT/CONFIRM]
//   pass B  x += alpha p, r -= alpha q, z = D^-1 r, fused with r^T z and r^T r.
//
// Step order and the true-residual confirmation follow the oracle (or_pcg):
// tolerance eps ||b||_2 (Eq. 6), recursive test then the true
// residual (R19); iterations = SpMVs with p (R30).  Batched block-diagonal
// systems (config 3) carry one state machine per segment; converged segments
// drop out of both passes while the others continue.
#include <cmath>

#include "lc_internal.cuh"

namespace cg = cooperative_groups;

namespace lc {

constexpr int kPT = 256;             // threads per CTA
constexpr int kPW = kPT / 32;        // warps per CTA
constexpr int kMaxSeg = 64;

enum Mode : int { M_INIT = 0, M_RESET, M_FIRST, M_NORMAL, M_UPDATE, M_CONFIRM, M_DONE };

struct PcgArgs {
  SellView A;
  const double* b;
  double* x;            // iterate (n)
  double* r;
  double* z;
  double* q;
  double* p0;
  double* p1;
  double* part;         // [(nCTA + nseg) * 2]
  int* n_active;
  int* out_iters;       // [nseg]
  int* out_status;
  double* out_relres;
  const int32_t* scatter_idx;   // local solve: x_full[scatter_idx[l]] = x[l] at exit
  double* x_full;
  double eps;
  int max_iters;
  int interleave;       // 1: slices strided over all warps of the grid (single segment)
  int vec2;             // 1: single segment and 16-byte aligned vectors -> flat double2 update pass
  int64_t chunk;        // contiguous slices per CTA (interleave == 0)
};

struct SegState {
  int mode, par, it, final_;
  double rho, alpha, beta, tgt, nb;
};

__device__ __forceinline__ void flush(double (*acc)[kMaxSeg][2], int warp, int gi, double a0, double a1) {
  a0 = warp_sum(a0);
  a1 = warp_sum(a1);
  if ((threadIdx.x & 31) == 0) { acc[warp][gi][0] += a0; acc[warp][gi][1] += a1; }
}

// One SELL row (lane of slice) dotted with an operand y(c) given by `ld`.  WM > 0: the slice width is
// at most WM, the loop is fully unrolled so all column/value loads issue before the dependent gathers
// (memory-level parallelism); slots k >= w are predicated off.  WM == 0: generic loop.
template <int WM, class Ld>
__device__ __forceinline__ double sell_row(const int32_t* __restrict__ cp, const double* __restrict__ vp, int w,
                                           Ld ld) {
  double acc = 0.0;
  if (WM > 0) {
    constexpr int WA = WM > 0 ? WM : 1;
    int c[WA];
    double v[WA], y[WA];
#pragma unroll
    for (int k = 0; k < WM; ++k) {
      c[k] = (k < w) ? __ldg(cp + 32 * k) : 0;
      v[k] = (k < w) ? __ldg(vp + 32 * k) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < WM; ++k) y[k] = (k < w) ? ld(c[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < WM; ++k)
      if (k < w) acc = __fma_rn(v[k], y[k], acc);
  } else {
    for (int k = 0; k < w; ++k) acc = __fma_rn(__ldg(vp + 32 * k), ld(__ldg(cp + 32 * k)), acc);
  }
  return acc;
}

template <int WM>
__global__ void __launch_bounds__(kPT) k_pcg(PcgArgs P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ SegState S[kMaxSeg];
  __shared__ double s_acc[kPW][kMaxSeg][2];
  __shared__ double s_red[kPW][2];
  __shared__ int s_exit;
  const SellView& A = P.A;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nCTA = gridDim.x, bid = blockIdx.x;
  int64_t s_begin, s_lim, s_step;
  int g_lo, g_hi;
  if (P.interleave) {
    s_begin = bid * kPW + warp; s_lim = A.nslices; s_step = nCTA * kPW;
    g_lo = 0; g_hi = 0;
  } else {
    int64_t c0 = bid * P.chunk, c1 = min(A.nslices, c0 + P.chunk);
    s_begin = c0 + warp; s_lim = c1; s_step = kPW;
    if (c0 < c1) { g_lo = A.slice_seg[c0]; g_hi = A.slice_seg[c1 - 1]; } else { g_lo = 1; g_hi = 0; }
  }
  const int nsegs_here = g_hi - g_lo + 1;
  if (threadIdx.x < kMaxSeg) {
    S[threadIdx.x].mode = M_INIT; S[threadIdx.x].par = 0; S[threadIdx.x].it = 0; S[threadIdx.x].final_ = 0;
  }
  __syncthreads();

  // partial sums of segment g of this CTA go to part[(bid + g)*2 + {0,1}]
  auto write_partials = [&]() {
    __syncthreads();
    for (int t = threadIdx.x; t < nsegs_here * 2; t += kPT) {
      int gi = t >> 1, j = t & 1;
      double v = 0.0;
      for (int w = 0; w < kPW; ++w) v += s_acc[w][gi][j];
      P.part[(bid + g_lo + gi) * 2 + j] = v;
    }
  };
  auto clear_acc = [&]() {
    for (int t = threadIdx.x; t < kPW * kMaxSeg * 2; t += kPT) (&s_acc[0][0][0])[t] = 0.0;
    __syncthreads();
  };
  // fixed-order sum of segment g's partials over the CTAs that touch it
  auto seg_sum = [&](int g, double& o0, double& o1) {
    int64_t c_lo, c_hi;
    if (P.interleave) { c_lo = 0; c_hi = nCTA - 1; }
    else { c_lo = A.seg_slice0[g] / P.chunk; c_hi = (A.seg_slice0[g + 1] - 1) / P.chunk; }
    double a0 = 0.0, a1 = 0.0;
    for (int64_t c = c_lo + threadIdx.x; c <= c_hi; c += kPT) {
      a0 += P.part[(c + g) * 2]; a1 += P.part[(c + g) * 2 + 1];
    }
    a0 = warp_sum(a0); a1 = warp_sum(a1);
    __syncthreads();
    if (lane == 0) { s_red[warp][0] = a0; s_red[warp][1] = a1; }
    __syncthreads();
    o0 = 0.0; o1 = 0.0;
    for (int w = 0; w < kPW; ++w) { o0 += s_red[w][0]; o1 += s_red[w][1]; }
  };
  auto owner = [&](int g) -> bool {
    if (P.interleave) return bid == 0;
    return bid == A.seg_slice0[g] / P.chunk;
  };
  auto finish = [&](int g, int status, double rn) {
    SegState& T = S[g];
    T.mode = M_DONE;
    if (owner(g)) {
      P.out_iters[g] = T.it;
      P.out_status[g] = status;
      P.out_relres[g] = T.nb > 0 ? rn / T.nb : rn;
      atomicSub(P.n_active, 1);
    }
  };

  for (;;) {
    // ------------------------------------------------------------ pass A ----
    clear_acc();
    {
      int gcur = -1, mode = M_DONE;
      double a0 = 0.0, a1 = 0.0, beta = 0.0;
      const double *pold = nullptr;
      double* pnew = nullptr;
      for (int64_t s = s_begin; s < s_lim; s += s_step) {
        int g = A.slice_seg[s];
        if (g != gcur) {
          if (gcur >= 0) flush(s_acc, warp, gcur - g_lo, a0, a1);
          a0 = a1 = 0.0;
          gcur = g;
          mode = S[g].mode;
          beta = S[g].beta;
          pold = S[g].par ? P.p1 : P.p0;
          pnew = S[g].par ? P.p0 : P.p1;
        }
        if (mode == M_DONE || mode == M_RESET) continue;
        int64_t u = A.slice_row0[s] + lane;
        if (u >= A.seg_unit0[g + 1]) continue;
        int64_t p0 = A.slice_ptr[s];
        int w = (int)((A.slice_ptr[s + 1] - p0) >> 5);
        const int32_t* cp = A.col + p0 + lane;
        const double* vp = A.val + p0 + lane;
        if (mode == M_INIT || mode == M_CONFIRM) {
          const double* xx = P.x;
          double acc = sell_row<WM>(cp, vp, w, [&](int c) { return xx[c]; });
          double bi = P.b[u];
          double ri = bi - acc;
          P.r[u] = ri;
          a0 = __fma_rn(ri, ri, a0);
          if (mode == M_INIT) a1 = __fma_rn(bi, bi, a1);
        } else if (mode == M_FIRST) {
          const double* zz = P.z;
          double acc = sell_row<WM>(cp, vp, w, [&](int c) { return zz[c]; });
          double pi = zz[u];
          pnew[u] = pi;
          P.q[u] = acc;
          a0 = __fma_rn(pi, acc, a0);
        } else {  // M_NORMAL: p = z + beta p_old on the fly
          const double* zz = P.z;
          double acc = sell_row<WM>(cp, vp, w, [&](int c) { return __fma_rn(beta, pold[c], zz[c]); });
          double pi = __fma_rn(beta, pold[u], zz[u]);
          pnew[u] = pi;
          P.q[u] = acc;
          a0 = __fma_rn(pi, acc, a0);
        }
      }
      if (gcur >= 0) flush(s_acc, warp, gcur - g_lo, a0, a1);
    }
    write_partials();
    grid.sync();
    // ---------------------------------------------------- pass A scalars ----
    for (int g = g_lo; g <= g_hi; ++g) {
      double s0, s1;
      seg_sum(g, s0, s1);
      if (threadIdx.x == 0) {
        SegState& T = S[g];
        if (T.mode == M_INIT) {
          T.nb = sqrt(s1);
          T.tgt = T.nb > 0 ? P.eps * T.nb : P.eps;
          double rn = sqrt(s0);
          if (!isfinite(rn)) finish(g, LC_ERR_NONFINITE, rn);
          else if (rn <= T.tgt) finish(g, LC_OK, rn);
          else T.mode = M_RESET;
        } else if (T.mode == M_FIRST || T.mode == M_NORMAL) {
          double pq = s0;
          if (!(pq > 0)) finish(g, isfinite(pq) ? LC_ERR_BREAKDOWN : LC_ERR_NONFINITE, NAN);
          else { T.alpha = T.rho / pq; T.mode = M_UPDATE; T.par ^= 1; }
        } else if (T.mode == M_CONFIRM) {
          double rn = sqrt(s0);
          if (!isfinite(rn)) finish(g, LC_ERR_NONFINITE, rn);
          else if (rn <= T.tgt) finish(g, LC_OK, rn);
          else if (T.final_) finish(g, LC_NOT_CONVERGED, rn);
          else T.mode = M_RESET;
        }
      }
      __syncthreads();
    }
    // ------------------------------------------------------------ pass B ----
    clear_acc();
    if (P.vec2) {
      // single segment: flat grid-stride over row pairs with 16-byte loads/stores
      const int mode = S[0].mode;
      double a0 = 0.0, a1 = 0.0;
      if (mode == M_UPDATE || mode == M_RESET) {
        const double alpha = S[0].alpha;
        const double2* pp = reinterpret_cast<const double2*>(S[0].par ? P.p1 : P.p0);
        double2* x2 = reinterpret_cast<double2*>(P.x);
        double2* r2 = reinterpret_cast<double2*>(P.r);
        double2* z2 = reinterpret_cast<double2*>(P.z);
        const double2* q2 = reinterpret_cast<const double2*>(P.q);
        const double2* d2 = reinterpret_cast<const double2*>(A.dinv);
        const int64_t n = A.seg_unit0[1], npair = n >> 1;
        const int64_t gt = bid * kPT + threadIdx.x, gs = nCTA * kPT;
        if (mode == M_UPDATE) {
#pragma unroll 2
          for (int64_t i = gt; i < npair; i += gs) {
            double2 xv = x2[i], pv = pp[i], rv = r2[i], qv = q2[i], dv = d2[i];
            xv.x = __fma_rn(alpha, pv.x, xv.x); xv.y = __fma_rn(alpha, pv.y, xv.y);
            rv.x = __fma_rn(-alpha, qv.x, rv.x); rv.y = __fma_rn(-alpha, qv.y, rv.y);
            double2 zv = make_double2(rv.x * dv.x, rv.y * dv.y);
            x2[i] = xv; r2[i] = rv; z2[i] = zv;
            a0 = __fma_rn(rv.x, zv.x, a0); a0 = __fma_rn(rv.y, zv.y, a0);
            a1 = __fma_rn(rv.x, rv.x, a1); a1 = __fma_rn(rv.y, rv.y, a1);
          }
          if ((n & 1) && gt == 0) {
            const double* p1 = S[0].par ? P.p1 : P.p0;
            int64_t u = n - 1;
            double xi = __fma_rn(alpha, p1[u], P.x[u]);
            double ri = __fma_rn(-alpha, P.q[u], P.r[u]);
            double zi = ri * A.dinv[u];
            P.x[u] = xi; P.r[u] = ri; P.z[u] = zi;
            a0 = __fma_rn(ri, zi, a0); a1 = __fma_rn(ri, ri, a1);
          }
        } else {
#pragma unroll 2
          for (int64_t i = gt; i < npair; i += gs) {
            double2 rv = r2[i], dv = d2[i];
            double2 zv = make_double2(rv.x * dv.x, rv.y * dv.y);
            z2[i] = zv;
            a0 = __fma_rn(rv.x, zv.x, a0); a0 = __fma_rn(rv.y, zv.y, a0);
          }
          if ((n & 1) && gt == 0) {
            int64_t u = n - 1;
            double zi = P.r[u] * A.dinv[u];
            P.z[u] = zi;
            a0 = __fma_rn(P.r[u], zi, a0);
          }
        }
      }
      flush(s_acc, warp, 0, a0, a1);
    } else {
      int gcur = -1, mode = M_DONE;
      double a0 = 0.0, a1 = 0.0, alpha = 0.0;
      const double* pp = nullptr;
      for (int64_t s = s_begin; s < s_lim; s += s_step) {
        int g = A.slice_seg[s];
        if (g != gcur) {
          if (gcur >= 0) flush(s_acc, warp, gcur - g_lo, a0, a1);
          a0 = a1 = 0.0;
          gcur = g;
          mode = S[g].mode;
          alpha = S[g].alpha;
          pp = S[g].par ? P.p1 : P.p0;
        }
        if (mode != M_UPDATE && mode != M_RESET) continue;
        int64_t u = A.slice_row0[s] + lane;
        if (u >= A.seg_unit0[g + 1]) continue;
        double di = A.dinv[u];
        if (mode == M_UPDATE) {
          double xi = __fma_rn(alpha, pp[u], P.x[u]);
          double ri = __fma_rn(-alpha, P.q[u], P.r[u]);
          double zi = ri * di;
          P.x[u] = xi; P.r[u] = ri; P.z[u] = zi;
          a0 = __fma_rn(ri, zi, a0);
          a1 = __fma_rn(ri, ri, a1);
        } else {
          double ri = P.r[u];
          double zi = ri * di;
          P.z[u] = zi;
          a0 = __fma_rn(ri, zi, a0);
        }
      }
      if (gcur >= 0) flush(s_acc, warp, gcur - g_lo, a0, a1);
    }
    write_partials();
    grid.sync();
    // ---------------------------------------------------- pass B scalars ----
    if (threadIdx.x == 0) s_exit = (atomicAdd(P.n_active, 0) == 0);
    for (int g = g_lo; g <= g_hi; ++g) {
      double s0, s1;
      seg_sum(g, s0, s1);
      if (threadIdx.x == 0) {
        SegState& T = S[g];
        if (T.mode == M_UPDATE) {
          T.it += 1;
          double rz = s0, rr = s1;
          if (!isfinite(rr) || sqrt(rr) <= T.tgt || T.it >= P.max_iters) {
            T.mode = M_CONFIRM;
            T.final_ = (T.it >= P.max_iters) || !isfinite(rr);
          } else {
            T.beta = rz / T.rho;
            T.rho = rz;
            T.mode = M_NORMAL;
          }
        } else if (T.mode == M_RESET) {
          T.rho = s0;
          T.mode = M_FIRST;
        }
      }
      __syncthreads();
    }
    __syncthreads();
    if (s_exit) break;
  }
  // a8: x~[Omega] = xbar_B (Eq. 4), fused into the local solve's exit
  if (P.scatter_idx) {
    for (int64_t s = s_begin; s < s_lim; s += s_step) {
      int g = A.slice_seg[s];
      int64_t u = A.slice_row0[s] + lane;
      if (u < A.seg_unit0[g + 1]) P.x_full[P.scatter_idx[u]] = P.x[u];
    }
  }
}

// ---------------------------------------------------------------- host ----
static int g_pcg_max_ctas[3] = {0, 0, 0};

lc_status run_pcg(const Sell& M, const double* b, double* x, const int32_t* scatter_idx, double* x_full,
                  const double* x_init, const lc_solver_params* p, cudaStream_t s, lc_solve_info* info) {
  const int G = M.nseg;
  if (G > kMaxSeg) { set_error("PCG: at most 64 segments"); return LC_ERR_DIMENSION; }
  if (M.block != 1) { set_error("PCG: needs block = 1 (use LC_GMRES for block systems)"); return LC_ERR_INVALID_ARG; }
  std::vector<int> it(G, 0), stt(G, LC_OK);
  std::vector<double> rr(G, 0.0);
  int n_active = 0;
  for (int g = 0; g < G; ++g) if (M.h_seg_slice0[g + 1] > M.h_seg_slice0[g]) ++n_active;
  float ms = 0.f;
  if (n_active > 0) {
    const int wi = M.maxw <= 5 ? 0 : M.maxw <= 7 ? 1 : 2;
    void* fn = wi == 0 ? (void*)k_pcg<5> : wi == 1 ? (void*)k_pcg<7> : (void*)k_pcg<0>;
    if (!g_pcg_max_ctas[wi]) {
      int per_sm = 0;
      LC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPT, 0));
      if (per_sm < 1) { set_error("PCG kernel does not fit on an SM"); return LC_ERR_CUDA; }
      g_pcg_max_ctas[wi] = per_sm * num_sms();
    }
    const int64_t n = M.nunits;
    int64_t nCTA = std::min<int64_t>(g_pcg_max_ctas[wi], (M.nslices + kPW - 1) / kPW);
    if (nCTA < 1) nCTA = 1;
    int interleave = (G == 1) ? 1 : 0;
    int64_t chunk = (M.nslices + nCTA - 1) / nCTA;
    if (!interleave) nCTA = (M.nslices + chunk - 1) / chunk;
    void* ws = nullptr;
    size_t vec = sizeof(double) * (size_t)n;
    size_t vbytes = (vec + 255) & ~(size_t)255;
    size_t bytes = vbytes * (scatter_idx ? 6 : 5) + sizeof(double) * 2 * (nCTA + G + 1) + 64 + 16 * G + 64;
    lc_status st = dalloc(&ws, bytes, s);
    if (st) return st;
    char* w = (char*)ws;
    PcgArgs a;
    a.A = view(M);
    a.b = b;
    a.r = (double*)w; w += vbytes;
    a.z = (double*)w; w += vbytes;
    a.q = (double*)w; w += vbytes;
    a.p0 = (double*)w; w += vbytes;
    a.p1 = (double*)w; w += vbytes;
    if (scatter_idx) {
      a.x = (double*)w; w += vbytes;
      cudaError_t e = cudaMemcpyAsync(a.x, x_init, vec, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) { dfree(ws, s); return cuda_fail(e, "cudaMemcpyAsync"); }
    } else {
      a.x = x;
    }
    a.part = (double*)w; w += sizeof(double) * 2 * (nCTA + G + 1);
    a.n_active = (int*)w; w += 64;
    a.out_iters = (int*)w; w += 4 * G;
    a.out_status = (int*)w; w += 4 * G;
    a.out_relres = (double*)((((uintptr_t)w) + 7) & ~(uintptr_t)7);
    a.scatter_idx = scatter_idx;
    a.x_full = x_full;
    a.eps = p->rel_tol;
    a.max_iters = p->max_iters;
    a.interleave = interleave;
    a.vec2 = (interleave && ((((uintptr_t)a.x) | ((uintptr_t)a.r) | ((uintptr_t)a.z) | ((uintptr_t)a.q) |
                              ((uintptr_t)a.p0) | ((uintptr_t)a.p1) | ((uintptr_t)M.dinv)) & 15) == 0) ? 1 : 0;
    a.chunk = chunk;
    cudaError_t e = cudaMemcpyAsync(a.n_active, &n_active, sizeof(int), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.out_iters, 0, 8 * G, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.out_relres, 0, 8 * G, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    void* args[] = {&a};
    if (e == cudaSuccess) e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)nCTA), dim3(kPT), args, 0, s);
    count_launch();
    cudaEventRecord(e1, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(it.data(), a.out_iters, 4 * G, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(stt.data(), a.out_status, 4 * G, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(rr.data(), a.out_relres, 8 * G, cudaMemcpyDeviceToHost, s);
    dfree(ws, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    if (e != cudaSuccess) return cuda_fail(e, "PCG kernel");
  }
  lc_status worst = LC_OK;
  for (int g = 0; g < G; ++g) {
    if (M.h_seg_slice0[g + 1] == M.h_seg_slice0[g]) { it[g] = 0; stt[g] = LC_OK; rr[g] = 0.0; }
    if (info) {
      info[g].iterations = it[g];
      info[g].status = stt[g];
      info[g].rel_residual = rr[g];
      info[g].seconds = ms * 1e-3;
    }
    if (stt[g] < 0) worst = (lc_status)stt[g];
    else if (stt[g] == LC_NOT_CONVERGED && worst == LC_OK) worst = LC_NOT_CONVERGED;
  }
  if (worst < 0) set_error("PCG: breakdown or non-finite value (see lc_solve_info.status)");
  return worst;
}

}  // namespace lc
