// gmres.cu -- right-preconditioned (block-)Jacobi GMRES(m) with CGS2 as ONE
// persistent cooperative kernel (SURVEY 8(a) a7/a9 for the nonsymmetric 3T
// systems of config 4; readings R20/R21/R33).
//
// One Arnoldi step of the default (Gram-form CGS2, R39) kernel = two grid-synchronised passes:
//   A  w = A t (BSR-in-SELL SpMV, t = M^-1 U_j from the previous pass) fused with the dots h_i = V_i^T w and
//      the new Gram column V_i^T V_j, i <= j
//   B  w <- w - V (h + h2) with h2 = h - (V^T V) h from the scalars, U_{j+1} = w, t = M^-1 U_{j+1}, ||w||^2
// (lc_tuning.gmres_exact_cgs2 keeps the textbook form: normalise, SpMV + dots, project + dots, project + norm.)
// Memory-level parallelism is what the passes live on (a warp owns 1-2 slices, every pass is ~20 us):
// the five-point 3T row is branch-free (block_row_dcoup5), the basis loads of the dot and update blocks are
// clamped instead of guarded so that they all issue before their first use, the update pass walks the basis
// downwards so each pass starts on what the previous one left in L2, the matrix and preconditioner values load
// with L2 evict_first and the basis with evict_last: config 4 Arnoldi step 63.5 -> 50 us (profiles/r02_p).
// The Hessenberg column, Givens rotations and the residual estimate |g_{j+1}|
// are computed redundantly (bitwise identically) by every CTA from the same
// fixed-order reductions, so control flow is grid-uniform without any host
// round trip.  End of cycle: x += M^-1 (V y), then the true residual (R19).
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "lc_internal.cuh"

namespace cg = cooperative_groups;

namespace lc {

#ifndef LC_GMRES_GT
#define LC_GMRES_GT 512
#endif
constexpr int kGT = LC_GMRES_GT;             // threads per CTA (1024 / kGT CTAs per SM)
#ifndef LC_GMRES_MINB
#define LC_GMRES_MINB (1024 / LC_GMRES_GT)
#endif
constexpr int kGMinB = LC_GMRES_MINB;        // CTAs per SM the kernel is compiled (registers) and launched for
constexpr int kGW = kGT / 32;
constexpr int kMaxM = 40;
constexpr int kMaxQ = 2 * (kMaxM + 1) + 2;   // reduced quantities per phase
#ifndef LC_GMRES_CC
#define LC_GMRES_CC 2
#endif
constexpr int kCC = LC_GMRES_CC;             // slices per warp chunk in the SpMV + dots pass (with kIB = 2: 1: 78.2,
                                             // 2: 69.0, 3: 81.3 us/step)
#ifndef LC_GMRES_IB
#define LC_GMRES_IB 1
#endif
// basis vectors per block of the dot / update loops.  With guarded loads (rounds 1-2: one memory round trip per
// vector whatever the block) 1 or 3 won by a few percent (profiles/r01_ar, r02_k).  With the clamped, branch-free
// loads of this round every block's loads issue together and the blocks overlap: 1 (49.7 us per config 4 Arnoldi
// step) <= 2 (50.2) <= 4 (50.6) <= 3 (51.4); kCC 2 stays (kCC 1: 50.6) -- profiles/r02_p
constexpr int kIB = LC_GMRES_IB;
#ifndef LC_GMRES_REV
#define LC_GMRES_REV 0
#endif
// 1: the update pass sweeps the slices in reverse, starting on the rows the SpMV + dots pass read last (L2 reuse
// of the basis): config 4 Arnoldi step 67.2 -> 68.3 us, not adopted (the update pass already runs above the DRAM
// rate, 19 us for 145 MB at j = 15, tools/tl_gmres.py)
constexpr bool kGRev = LC_GMRES_REV != 0;
#ifndef LC_GMRES_RED1
#define LC_GMRES_RED1 1
#endif
#ifndef LC_GMRES_VREV
#define LC_GMRES_VREV 1
#endif
// 1: the update pass walks the basis from V_j down to V_0, so it starts on the vectors the SpMV + dots pass read
// last and ends on V_0, V_1, ... where the next step's dots begin: each pass finds in L2 what the previous one
// touched last (both ascending, a cycle's basis (j + 1) x 6.3 MB streams through the 126 MB L2 in LRU order and
// every access misses once it no longer fits)
#ifndef LC_GMRES_HINT
#define LC_GMRES_HINT 2
#endif
// 1: the matrix values and preconditioner blocks (read once per step) load with L2 evict_first; 2: also the basis
// with evict_last
__device__ __forceinline__ double ld_first(const double* p) {
#if LC_GMRES_HINT >= 1
  unsigned long long pol;
  double v;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
#else
  return *p;
#endif
}
__device__ __forceinline__ double ld_last(const double* p) {
#if LC_GMRES_HINT >= 2
  unsigned long long pol;
  double v;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
#else
  return *p;
#endif
}

struct GmresArgs {
  SellView A;
  const double* b;
  double* x;
  double* r;
  double* w;
  double* t;
  double* V;            // (m+1) vectors of n scalars
  double* part;         // [(m+2) * nCTA]
  GridBar* bar;
  int* out;             // [0] iters, [1] status
  double* out_relres;
  const int32_t* scatter_idx;
  double* x_full;
  int64_t n;            // scalar unknowns
  double eps;
  int m;
  int max_iters;
  int exact_cgs2;       // 1: textbook two-pass CGS2 (4 barriers, 4 passes over V per step); 0: Gram form (R39)
};

// the 3T SpMV row (cell u of slice s) on the compact diagonal-coupling values (Sell::cval): slots in ascending
// column order, the diagonal block's 9-term chain, 1 term per component for a diagonal coupling block -- the
// same chains as the full 3x3 blocks minus their exact-zero terms, bitwise (an fma chain that starts at +0 never
// holds -0, so adding 0 * y is the identity)
__device__ __forceinline__ void block_row_dcoup(const SellView& A, int64_t s, int lane, int wd, int64_t u,
                                                const double* __restrict__ y, double* acc) {
  const double* cb = A.cval + 32ll * A.cw * s + lane;
  int o = 0;
#pragma unroll 5
  for (int k = 0; k < wd; ++k) {
    const int64_t c = sv_col(A, 0, k, u);
    const double y0 = y[3 * c], y1 = y[3 * c + 1], y2 = y[3 * c + 2];
    if (k == A.kdiag) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        acc[a] = __fma_rn(cb[32 * (3 * a)], y0, acc[a]);
        acc[a] = __fma_rn(cb[32 * (3 * a + 1)], y1, acc[a]);
        acc[a] = __fma_rn(cb[32 * (3 * a + 2)], y2, acc[a]);
      }
    } else {
      const double* cd = cb + 32 * (9 + 3 * o);
      acc[0] = __fma_rn(cd[0], y0, acc[0]);
      acc[1] = __fma_rn(cd[32], y1, acc[1]);
      acc[2] = __fma_rn(cd[64], y2, acc[2]);
      ++o;
    }
  }
}

// the same row for the five-point cell stencil (W = 5, the diagonal in slot 2: offsets {-nx, -1, 0, 1, nx}): no
// branch on the slot and no slot loop, so the row's 15 gathers and 21 values all issue before the chains (the slot
// loop above takes one memory round trip per slot: config 4's SpMV part of an Arnoldi step ran at 3 TB/s,
// profiles/r02_g).  Same chains in the same slot order, so bitwise the results of block_row_dcoup.
#ifndef LC_GMRES_SPMV5
#define LC_GMRES_SPMV5 1
#endif
__device__ __forceinline__ void block_row_dcoup5(const SellView& A, int64_t s, int lane, int64_t u,
                                                 const double* __restrict__ y, double* acc) {
  const double* cb = A.cval + 32ll * 21 * s + lane;
  const int64_t n1 = A.nunits - 1;
  double yy[5][3], dv[9], cv[4][3];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    int64_t c = u + A.off[k];
    c = c < 0 ? 0 : (c > n1 ? n1 : c);
#pragma unroll
    for (int a = 0; a < 3; ++a) yy[k][a] = y[3 * c + a];
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) dv[q] = ld_first(cb + 32 * q);
#pragma unroll
  for (int o = 0; o < 4; ++o)
#pragma unroll
    for (int a = 0; a < 3; ++a) cv[o][a] = ld_first(cb + 32 * (9 + 3 * o + a));
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    if (k == 2) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        acc[a] = __fma_rn(dv[3 * a], yy[2][0], acc[a]);
        acc[a] = __fma_rn(dv[3 * a + 1], yy[2][1], acc[a]);
        acc[a] = __fma_rn(dv[3 * a + 2], yy[2][2], acc[a]);
      }
    } else {
      const int o = k < 2 ? k : k - 1;
#pragma unroll
      for (int a = 0; a < 3; ++a) acc[a] = __fma_rn(cv[o][a], yy[k][a], acc[a]);
    }
  }
}
// The explicit 3T subsystems (SELL-32 of uniform width, full 3x3 blocks): for width 5 the five column indices
// load first and every slot's gathers and values follow without a loop guard between them (the slot loop took
// two dependent round trips per slot: column, then gather).  Padding slots hold their own row and zeros.  Same
// chains in the same order as the loop.
__device__ __forceinline__ void block_row_sell5(const SellView& A, int64_t p0, int lane, const double* __restrict__ y,
                                                double* acc) {
  int32_t c[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) c[k] = A.col[p0 + lane + 32 * k];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const double* vb = A.val + 9 * (p0 + 32ll * k) + lane;
    const double y0 = y[3 * c[k]], y1 = y[3 * c[k] + 1], y2 = y[3 * c[k] + 2];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      acc[a] = __fma_rn(ld_first(vb + 32 * (3 * a)), y0, acc[a]);
      acc[a] = __fma_rn(ld_first(vb + 32 * (3 * a + 1)), y1, acc[a]);
      acc[a] = __fma_rn(ld_first(vb + 32 * (3 * a + 2)), y2, acc[a]);
    }
  }
}
// dispatch: the branch-free row when the layout is the five-point one
__device__ __forceinline__ void block_row_dc(const SellView& A, int64_t s, int lane, int wd, int64_t u,
                                             const double* __restrict__ y, double* acc) {
  if (LC_GMRES_SPMV5 && wd == 5 && A.kdiag == 2) block_row_dcoup5(A, s, lane, u, y, acc);
  else block_row_dcoup(A, s, lane, wd, u, y, acc);
}

template <int BS>
__device__ __forceinline__ void block_apply(const double* __restrict__ Mi, const double* v, double* t) {
#pragma unroll
  for (int a = 0; a < BS; ++a) {
    double s = 0.0;
#pragma unroll
    for (int be = 0; be < BS; ++be) s = __fma_rn(ld_first(Mi + a * BS + be), v[be], s);
    t[a] = s;
  }
}

#ifdef LC_DEBUG_TIMELINE
__device__ unsigned long long g_tlg[16384];
#define TLG(k) do { if (blockIdx.x == 0 && threadIdx.x == 0 && (k) < 16384) { unsigned long long _t; \
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t)); g_tlg[(k)] = _t; } ++(k); } while (0)
#else
#define TLG(k) (void)0
#endif

// sums of N (a power of two <= 32) per-lane values over the warp with N - 1 + log2(32 / N) shuffles instead of
// 5 N: at each of the first log2 N levels a lane keeps one half of its values and sends the other half to its
// partner; afterwards lane l holds the warp's sum of v[l % N].  Fixed order, so deterministic.
template <int N>
__device__ __forceinline__ double warp_sum_multi(double* v, int lane) {
#pragma unroll
  for (int half = N / 2, bit = 1; half >= 1; half >>= 1, bit <<= 1) {
    const bool up = lane & bit;
#pragma unroll
    for (int q = 0; q < half; ++q) {
      const double keep = up ? v[2 * q + 1] : v[2 * q];
      const double send = up ? v[2 * q] : v[2 * q + 1];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
    }
  }
  double r = v[0];
#pragma unroll
  for (int o = N; o < 32; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

template <int BS, int IB>
__global__ void __launch_bounds__(kGT, kGMinB) k_gmres(GmresArgs P) {
  unsigned long long bar_epoch = 0;
#ifdef LC_DEBUG_TIMELINE
  int tk = 0;
#endif
  const SellView& A = P.A;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nCTA = gridDim.x, bid = blockIdx.x;
  const int64_t s_begin = bid * kGW + warp, s_step = nCTA * kGW;
  const int64_t nunits = A.seg_unit0[1];
  const int64_t n = P.n;
  const int m = P.m;
  __shared__ double H[(kMaxM + 1) * kMaxM];
  __shared__ double gv[kMaxM + 1], cs[kMaxM], sn[kMaxM], yv[kMaxM];
  __shared__ double sig[kMaxM + 1];   // basis scales: V_i = sig_i U_i (U stored; all 1 in the exact-CGS2 mode)
  __shared__ double red[kMaxQ];
  __shared__ double s_acc[kGW][kMaxQ];
  __shared__ double Gm[(kMaxM + 1) * (kMaxM + 1)];   // Gram matrix V^T V (low-sync CGS2, R39)

  constexpr int kNP = 2 * IB <= 2 ? 2 : 2 * IB <= 4 ? 4 : 2 * IB <= 8 ? 8 : 16;   // the dots block's sums, padded
  // per-lane accumulators -> per-warp smem -> CTA partial part[q*nCTA + bid]
  auto clear = [&](int nq) {
    for (int t = threadIdx.x; t < kGW * kMaxQ; t += kGT) (&s_acc[0][0])[t] = 0.0;
    __syncthreads();
    (void)nq;
  };
  // the partials are double-buffered by reduction (ppar): a CTA leaving a barrier early may publish its next
  // partials before a slower CTA has read these (short passes)
  int ppar = 0;
  auto publish = [&](int nq) {
    __syncthreads();
    double* pt = P.part + (size_t)ppar * kMaxQ * nCTA;
    for (int q = threadIdx.x; q < nq; q += kGT) {
      double v = 0.0;
      for (int w = 0; w < kGW; ++w) v += s_acc[w][q];
      pt[q * nCTA + bid] = v;
    }
  };
  // fixed-order reduction of nq quantities over all CTAs into red[]
  auto reduce = [&](int nq) {
    const double* pt = P.part + (size_t)ppar * kMaxQ * nCTA;
    ppar ^= 1;
#if LC_GMRES_RED1
    // two quantities per warp at a time, 5 partial loads each in flight (one quantity after the other with 8
    // loads: +1.4 us per Arnoldi step; 10 + 10 loads in flight, inline or out of line: spills / +4.5 us)
    for (int q0 = warp; q0 < nq; q0 += 2 * kGW) {
      const int q1 = q0 + kGW;
      const bool two = q1 < nq;
      double v0 = 0.0, v1 = 0.0;
      for (int64_t c0 = lane; c0 < nCTA; c0 += 32 * 5) {
        double t0[5], t1[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const bool in = c0 + 32 * k < nCTA;
          t0[k] = in ? pt[q0 * nCTA + c0 + 32 * k] : 0.0;
          t1[k] = in && two ? pt[q1 * nCTA + c0 + 32 * k] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 5; ++k)
          if (c0 + 32 * k < nCTA) { v0 += t0[k]; v1 += t1[k]; }
      }
      v0 = warp_sum(v0);
      v1 = warp_sum(v1);
      if (lane == 0) { red[q0] = v0; if (two) red[q1] = v1; }
    }
#else
    for (int q = warp; q < nq; q += kGW) {
      // a lane's partials (CTAs lane, lane + 32, ...) are loaded 8 at a time and added in that order
      double v = 0.0;
      for (int64_t c0 = lane; c0 < nCTA; c0 += 32 * 8) {
        double t[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) t[k] = c0 + 32 * k < nCTA ? pt[q * nCTA + c0 + 32 * k] : 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (c0 + 32 * k < nCTA) v += t[k];
      }
      v = warp_sum(v);
      if (lane == 0) red[q] = v;
    }
#endif
    __syncthreads();
  };
  auto lane_flush = [&](int q, double v) {
    v = warp_sum(v);
    if (lane == 0) s_acc[warp][q] += v;
  };

  int it = 0;
  bool first = true;
  double nb = 0.0, tgt = 0.0;
  int status = LC_NOT_CONVERGED;
  double relres = 0.0;
  for (;;) {
    // ------------------------------------------------ true residual -------
    clear(2);
    {
      double a0 = 0.0, a1 = 0.0;
      for (int64_t s = s_begin; s < A.nslices; s += s_step) {
        int64_t u = A.slice_row0[s] + lane;
        if (u >= nunits) continue;
        int64_t p0 = A.slice_ptr[s];
        int wd = A.stencil ? A.W : (int)((A.slice_ptr[s + 1] - p0) >> 5);
        double acc[BS];
#pragma unroll
        for (int a = 0; a < BS; ++a) acc[a] = 0.0;
        if (BS == 3 && A.cval) {
          block_row_dc(A, s, lane, wd, u, P.x, acc);
        } else if (BS == 3 && !A.stencil && A.vw == 5) {
          block_row_sell5(A, p0, lane, P.x, acc);
        } else
        for (int k = 0; k < wd; ++k) {
          int64_t c = sv_col(A, p0 + lane, k, u);
          if (BS == 1) {
            acc[0] = __fma_rn(sv_val(A, p0 + lane, k, u), P.x[c], acc[0]);
          } else {
            const double* vb = A.val + 9 * (p0 + 32ll * k) + lane;
            double y0 = P.x[3 * c], y1 = P.x[3 * c + 1], y2 = P.x[3 * c + 2];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              acc[a] = __fma_rn(vb[32 * (3 * a)], y0, acc[a]);
              acc[a] = __fma_rn(vb[32 * (3 * a + 1)], y1, acc[a]);
              acc[a] = __fma_rn(vb[32 * (3 * a + 2)], y2, acc[a]);
            }
          }
        }
        double rv[BS];
#pragma unroll
        for (int a = 0; a < BS; ++a) {
          double bi = P.b[BS * u + a];
          double ri = bi - acc[a];
          rv[a] = ri;
          a0 = __fma_rn(ri, ri, a0);
          a1 = __fma_rn(bi, bi, a1);
        }
        if (P.exact_cgs2) {
#pragma unroll
          for (int a = 0; a < BS; ++a) P.r[BS * u + a] = rv[a];
        } else {                                   // scaled basis: U_0 = r, t = M^-1 U_0 (cell-local)
          double tt[BS];
          block_apply<BS>(A.dinv + BS * BS * u, rv, tt);
#pragma unroll
          for (int a = 0; a < BS; ++a) { P.V[BS * u + a] = rv[a]; P.t[BS * u + a] = tt[a]; }
        }
      }
      lane_flush(0, a0);
      lane_flush(1, a1);
    }
    publish(2);
    grid_barrier(P.bar, bar_epoch);
    reduce(2);
    double beta = sqrt(red[0]);
    if (first) { nb = sqrt(red[1]); tgt = nb > 0 ? P.eps * nb : P.eps; }
    relres = nb > 0 ? beta / nb : beta;
    if (!isfinite(beta)) { status = LC_ERR_NONFINITE; break; }
    if (beta <= tgt) { status = LC_OK; break; }
    if (it >= P.max_iters) { status = LC_NOT_CONVERGED; break; }
    first = false;
    if (threadIdx.x <= m) { gv[threadIdx.x] = 0.0; sig[threadIdx.x] = 1.0; }
    __syncthreads();
    if (threadIdx.x == 0) { gv[0] = beta; if (!P.exact_cgs2) sig[0] = 1.0 / beta; }
    __syncthreads();
    double hnorm = beta;
    const double* src = P.r;
    int jend = 0;
    for (int j = 0; j < m; ++j) {
      TLG(tk);
      double* Vj = P.V + (size_t)j * n;
      // ---- 1a (exact-CGS2 mode): v_j = src / h, t = M^-1 v_j.  The scaled-basis (Gram) mode has t = M^-1 U_j
      // from the previous update pass (or the residual pass) and skips this pass and its barrier.
      if (P.exact_cgs2) {
      for (int64_t s = s_begin; s < A.nslices; s += s_step) {
        int64_t u = A.slice_row0[s] + lane;
        if (u >= nunits) continue;
        double v[BS], tt[BS];
#pragma unroll
        for (int a = 0; a < BS; ++a) { v[a] = src[BS * u + a] / hnorm; Vj[BS * u + a] = v[a]; }
        block_apply<BS>(A.dinv + BS * BS * u, v, tt);
#pragma unroll
        for (int a = 0; a < BS; ++a) P.t[BS * u + a] = tt[a];
      }
      grid_barrier(P.bar, bar_epoch);
      }
      TLG(tk);
      TLG(tk);
      // ---- 1b: w = A t, h_i = V_i . w.  A warp owns 1-2 slices per chunk: their w values stay in registers
      // and the (j+1) dots are formed i by i (no per-thread accumulator array in local memory).
      clear(j + 1);
      // (CC slices per chunk: kCC, or 1 when no warp has a second slice -- a small subsystem -- so that no
      // warp issues the clamped loads of an absent slice)
      auto dots_pass = [&](auto cc_tag) {
      constexpr int CC = decltype(cc_tag)::value;
      for (int64_t s0 = s_begin; s0 < A.nslices; s0 += CC * s_step) {
        double wv[CC][BS];
        int64_t ea[CC];                 // this lane's first element (a row past the end reads element 0, times w = 0)
        bool ok[CC];
#pragma unroll
        for (int cc = 0; cc < CC; ++cc) {
          const int64_t s = s0 + cc * s_step;
          const int64_t u = s < A.nslices ? A.slice_row0[s] + lane : nunits;
          ok[cc] = u < nunits;
          ea[cc] = ok[cc] ? BS * u : 0;
#pragma unroll
          for (int a = 0; a < BS; ++a) wv[cc][a] = 0.0;
          if (ok[cc]) {
            const int64_t p0 = A.slice_ptr[s];
            const int wd = A.stencil ? A.W : (int)((A.slice_ptr[s + 1] - p0) >> 5);
            if (BS == 3 && A.cval) {
              block_row_dc(A, s, lane, wd, u, P.t, wv[cc]);
            } else if (BS == 3 && !A.stencil && A.vw == 5) {
              block_row_sell5(A, p0, lane, P.t, wv[cc]);
            } else
#pragma unroll 5
            for (int k = 0; k < wd; ++k) {
              const int64_t c = sv_col(A, p0 + lane, k, u);
              if (BS == 1) {
                wv[cc][0] = __fma_rn(sv_val(A, p0 + lane, k, u), P.t[c], wv[cc][0]);
              } else {
                const double* vb = A.val + 9 * (p0 + 32ll * k) + lane;
                const double y0 = P.t[3 * c], y1 = P.t[3 * c + 1], y2 = P.t[3 * c + 2];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                  wv[cc][a] = __fma_rn(vb[32 * (3 * a)], y0, wv[cc][a]);
                  wv[cc][a] = __fma_rn(vb[32 * (3 * a + 1)], y1, wv[cc][a]);
                  wv[cc][a] = __fma_rn(vb[32 * (3 * a + 2)], y2, wv[cc][a]);
                }
              }
            }
#pragma unroll
            for (int a = 0; a < BS; ++a) P.w[BS * u + a] = wv[cc][a];
          }
        }
        const double* Vj = P.V + (size_t)j * n;
        double vj[CC][BS];
#pragma unroll
        for (int cc = 0; cc < CC; ++cc)
#pragma unroll
          for (int a = 0; a < BS; ++a) vj[cc][a] = (ok[cc] && !P.exact_cgs2) ? Vj[ea[cc] + a] : 0.0;
        // i in blocks of IB (the loop is left to ptxas' own unrolling: #pragma unroll 1 / 2 / 4 measured 52.7 / 49.1 /
        // 51.7 us per config 4 step against 49.2, and 1.59 / 1.43 / 1.40 ms against 1.36 ms for its local solve).
        // Every load of the block issues before its first use: the addresses are clamped
        // (vector min(i, j), element 0 for a row past the end) instead of guarded, so no branch separates the
        // loads -- guarded, ptxas issued one vector's loads, waited, multiplied, and only then loaded the next
        // (18.5% of the kernel's stall samples sat on the first multiply, profiles/r02_p).  The block's 2 IB
        // sums are combined over the lanes by one merged butterfly (warp_sum_multi).
        for (int i0 = 0; i0 <= j; i0 += IB) {
          double vi[IB][CC][BS];
#pragma unroll
          for (int ii = 0; ii < IB; ++ii) {
            const double* Vi = P.V + (size_t)(i0 + ii <= j ? i0 + ii : j) * n;
#pragma unroll
            for (int cc = 0; cc < CC; ++cc)
#pragma unroll
              for (int a = 0; a < BS; ++a) vi[ii][cc][a] = ld_last(Vi + ea[cc] + a);
          }
          double dq[kNP];                 // d[0..IB), then gq[0..IB), zero padding up to a power of two
#pragma unroll
          for (int q = 0; q < kNP; ++q) dq[q] = 0.0;
#pragma unroll
          for (int ii = 0; ii < IB; ++ii)
#pragma unroll
            for (int cc = 0; cc < CC; ++cc)
#pragma unroll
              for (int a = 0; a < BS; ++a) {
                dq[ii] = __fma_rn(vi[ii][cc][a], wv[cc][a], dq[ii]);
                dq[IB + ii] = __fma_rn(vi[ii][cc][a], vj[cc][a], dq[IB + ii]);
              }
          const double tot = warp_sum_multi<kNP>(dq, lane);     // lane l: the sum of dq[l % kNP]
          const int q = lane & (kNP - 1);
          if (lane < kNP && q < 2 * IB) {
            const int ii = q < IB ? q : q - IB;
            if (i0 + ii <= j && (q < IB || !P.exact_cgs2)) s_acc[warp][(q < IB ? 0 : j + 1) + i0 + ii] += tot;
          }
        }
      }
      };
      if (A.nslices > s_step) dots_pass(std::integral_constant<int, kCC>{});
      else dots_pass(std::integral_constant<int, 1>{});
      if (!P.exact_cgs2) {
        // ---- low-sync CGS2 (R39): G = V^T V gains column j in the same pass; the second projection
        // h2 = V^T (w - V h) = h - G h comes from scalars, and both updates merge into one pass.
        publish(2 * (j + 1));
        TLG(tk);
        grid_barrier(P.bar, bar_epoch);
        reduce(2 * (j + 1));
        TLG(tk);
        if (threadIdx.x <= j) {                     // dots of the stored U_i: V_i = sig_i U_i, w = sig_j A t
          const double sc = sig[threadIdx.x] * sig[j];
          const double gij = sc * red[j + 1 + threadIdx.x];
          Gm[threadIdx.x * (kMaxM + 1) + j] = gij;
          Gm[j * (kMaxM + 1) + threadIdx.x] = gij;
          H[threadIdx.x * m + j] = sc * red[threadIdx.x];
        }
        __syncthreads();
        __shared__ double hh[kMaxM + 1];
        if (threadIdx.x <= j) {
          const int i = threadIdx.x;
          double gh = 0.0;
          for (int k = 0; k <= j; ++k) gh = __fma_rn(Gm[i * (kMaxM + 1) + k], H[k * m + j], gh);
          hh[i] = H[i * m + j] + (H[i * m + j] - gh);        // h + h2, h2 = h - G h
        }
        __syncthreads();
        if (threadIdx.x <= j) {
          H[threadIdx.x * m + j] = hh[threadIdx.x];
          hh[threadIdx.x] *= sig[threadIdx.x];                // coefficient of the stored U_i
        }
        __syncthreads();
        const double sj = sig[j];
        clear(1);
        {
          double a0 = 0.0;
          for (int64_t sr = s_begin; sr < A.nslices; sr += s_step) {
            const int64_t s = kGRev ? A.nslices - 1 - sr : sr;
            const int64_t u = A.slice_row0[s] + lane;
            if (u >= nunits) continue;
            double ww[BS];
#pragma unroll
            for (int a = 0; a < BS; ++a) ww[a] = sj * P.w[BS * u + a];
            // blocks of IB basis vectors, from V_j down (LC_GMRES_VREV); clamped vector index with a zero
            // coefficient instead of a guard, so the block's loads all issue together
            for (int ib = 0; ib <= j / IB; ++ib) {
              const int i0 = LC_GMRES_VREV ? (j / IB - ib) * IB : ib * IB;
              double vv[IB][BS];
#pragma unroll
              for (int ii = 0; ii < IB; ++ii)
#pragma unroll
                for (int a = 0; a < BS; ++a)
                  vv[ii][a] = ld_last(P.V + (size_t)(i0 + ii <= j ? i0 + ii : j) * n + BS * u + a);
#pragma unroll
              for (int i2 = 0; i2 < IB; ++i2) {          // descending inside the block too: the same chain for any IB
                const int ii = LC_GMRES_VREV ? IB - 1 - i2 : i2;
                if (i0 + ii > j) continue;
                const double hi = hh[i0 + ii];
#pragma unroll
                for (int a = 0; a < BS; ++a) ww[a] = __fma_rn(-hi, vv[ii][a], ww[a]);
              }
            }
            // U_{j+1} = w (normalised lazily through sig_{j+1}) and t = M^-1 U_{j+1} for the next step
            double tt[BS];
            block_apply<BS>(A.dinv + BS * BS * u, ww, tt);
            double* Un = P.V + (size_t)(j + 1) * n;
#pragma unroll
            for (int a = 0; a < BS; ++a) {
              Un[BS * u + a] = ww[a];
              P.t[BS * u + a] = tt[a];
              a0 = __fma_rn(ww[a], ww[a], a0);
            }
          }
          lane_flush(0, a0);
        }
        publish(1);
        TLG(tk);
        grid_barrier(P.bar, bar_epoch);
        reduce(1);
        TLG(tk);
      } else {
      publish(j + 1);
      TLG(tk);
      grid_barrier(P.bar, bar_epoch);
      reduce(j + 1);
      TLG(tk);
      // keep h in smem column j of H (pass-1 part)
      if (threadIdx.x <= j) H[threadIdx.x * m + j] = red[threadIdx.x];
      __syncthreads();
      // ---- 2: w -= V h, h2_i = V_i . w (same register chunking)
      clear(j + 1);
      for (int64_t s0 = s_begin; s0 < A.nslices; s0 += 2 * s_step) {
        double wv[2][BS];
        int64_t uu[2];
        bool ok[2];
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int64_t s = s0 + cc * s_step;
          uu[cc] = s < A.nslices ? A.slice_row0[s] + lane : nunits;
          ok[cc] = uu[cc] < nunits;
#pragma unroll
          for (int a = 0; a < BS; ++a) wv[cc][a] = 0.0;
          if (ok[cc]) {
            const int64_t u = uu[cc];
#pragma unroll
            for (int a = 0; a < BS; ++a) wv[cc][a] = P.w[BS * u + a];
            for (int i = 0; i <= j; ++i) {
              const double* Vi = P.V + (size_t)i * n;
              const double hi = H[i * m + j];
#pragma unroll
              for (int a = 0; a < BS; ++a) wv[cc][a] = __fma_rn(-hi, Vi[BS * u + a], wv[cc][a]);
            }
#pragma unroll
            for (int a = 0; a < BS; ++a) P.w[BS * u + a] = wv[cc][a];
          }
        }
        for (int i = 0; i <= j; ++i) {
          const double* Vi = P.V + (size_t)i * n;
          double d = 0.0;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc)
            if (ok[cc]) {
#pragma unroll
              for (int a = 0; a < BS; ++a) d = __fma_rn(Vi[BS * uu[cc] + a], wv[cc][a], d);
            }
          lane_flush(i, d);
        }
      }
      publish(j + 1);
      TLG(tk);
      grid_barrier(P.bar, bar_epoch);
      reduce(j + 1);
      TLG(tk);
      // ---- 3: w -= V h2, ||w||^2
      clear(1);
      {
        double a0 = 0.0;
        for (int64_t s = s_begin; s < A.nslices; s += s_step) {
          int64_t u = A.slice_row0[s] + lane;
          if (u >= nunits) continue;
          double ww[BS];
#pragma unroll
          for (int a = 0; a < BS; ++a) ww[a] = P.w[BS * u + a];
          for (int i = 0; i <= j; ++i) {
            const double* Vi = P.V + (size_t)i * n;
            double h2 = red[i];
#pragma unroll
            for (int a = 0; a < BS; ++a) ww[a] = __fma_rn(-h2, Vi[BS * u + a], ww[a]);
          }
#pragma unroll
          for (int a = 0; a < BS; ++a) { P.w[BS * u + a] = ww[a]; a0 = __fma_rn(ww[a], ww[a], a0); }
        }
        // red[] still holds h2: add it to H before it is overwritten
        __syncthreads();
        if (threadIdx.x <= j) H[threadIdx.x * m + j] += red[threadIdx.x];
        lane_flush(0, a0);
      }
      publish(1);
      TLG(tk);
      grid_barrier(P.bar, bar_epoch);
      reduce(1);
      TLG(tk);
      }
      if (threadIdx.x == 0) {
        double hn = sqrt(red[0]);
        H[(j + 1) * m + j] = hn;
        for (int i = 0; i < j; ++i) {
          double t0 = H[i * m + j], t1 = H[(i + 1) * m + j];
          H[i * m + j] = cs[i] * t0 + sn[i] * t1;
          H[(i + 1) * m + j] = -sn[i] * t0 + cs[i] * t1;
        }
        double hd = H[j * m + j], hs = H[(j + 1) * m + j];
        double den = sqrt(hd * hd + hs * hs);
        if (den == 0.0) { cs[j] = 1.0; sn[j] = 0.0; } else { cs[j] = hd / den; sn[j] = hs / den; }
        H[j * m + j] = cs[j] * hd + sn[j] * hs;
        H[(j + 1) * m + j] = 0.0;
        gv[j + 1] = -sn[j] * gv[j];
        gv[j] = cs[j] * gv[j];
        red[kMaxQ - 1] = hn;
        if (!P.exact_cgs2 && j + 1 <= m) sig[j + 1] = 1.0 / hn;
      }
      __syncthreads();
      hnorm = red[kMaxQ - 1];
      ++it;
      jend = j + 1;
      src = P.w;
      double gj = gv[j + 1];
      if (!isfinite(gj)) { status = LC_ERR_NONFINITE; break; }
      if (fabs(gj) <= tgt || hnorm == 0.0 || it >= P.max_iters) break;
    }
    if (status == LC_ERR_NONFINITE) break;
    // ---- y = H^-1 g (upper triangular), x += M^-1 (V y)
    if (threadIdx.x == 0) {
      for (int i = jend - 1; i >= 0; --i) {
        double s = gv[i];
        for (int k = i + 1; k < jend; ++k) s -= H[i * m + k] * yv[k];
        yv[i] = s / H[i * m + i];
      }
    }
    __syncthreads();
    for (int64_t s = s_begin; s < A.nslices; s += s_step) {
      int64_t u = A.slice_row0[s] + lane;
      if (u >= nunits) continue;
      double acc[BS], tt[BS];
#pragma unroll
      for (int a = 0; a < BS; ++a) acc[a] = 0.0;
      for (int i = 0; i < jend; ++i) {
        const double* Vi = P.V + (size_t)i * n;
        double yi = yv[i] * sig[i];
#pragma unroll
        for (int a = 0; a < BS; ++a) acc[a] = __fma_rn(yi, Vi[BS * u + a], acc[a]);
      }
      block_apply<BS>(A.dinv + BS * BS * u, acc, tt);
#pragma unroll
      for (int a = 0; a < BS; ++a) P.x[BS * u + a] += tt[a];
    }
    grid_barrier(P.bar, bar_epoch);
  }
  if (bid == 0 && threadIdx.x == 0) { P.out[0] = it; P.out[1] = status; *P.out_relres = relres; }
  if (P.scatter_idx) {
    for (int64_t s = s_begin; s < A.nslices; s += s_step) {
      int64_t u = A.slice_row0[s] + lane;
      if (u >= nunits) continue;
      int64_t gidx = P.scatter_idx[u];
#pragma unroll
      for (int a = 0; a < BS; ++a) P.x_full[BS * gidx + a] = P.x[BS * u + a];
    }
  }
}

lc_status run_gmres(const Sell& M, const double* b, double* x, const int32_t* scatter_idx, double* x_full,
                    const double* x_init, const lc_solver_params* p, cudaStream_t s, lc_solve_info* info,
                    Pending* defer) {
  if (M.nseg != 1) { set_error("GMRES: batched (block-diagonal) systems are not supported"); return LC_ERR_DIMENSION; }
  const int BS = M.block;
  const int m = p->restart;
  const int64_t n = M.nunits * BS;
  // basis blocking kIB for every kernel (the 3T kernel is instantiated once whatever the couplings' storage)
  void* fn = BS == 1 ? (void*)k_gmres<1, kIB> : (void*)k_gmres<3, kIB>;
  int64_t max_ctas = 0;
  const size_t dsmem = 0;
  lc_status st = max_coresident(fn, kGT, dsmem, &max_ctas);
  if (st) return st;
  max_ctas = std::min<int64_t>(max_ctas, (int64_t)kGMinB * num_sms());
  int64_t nCTA = std::min<int64_t>(max_ctas, (M.nslices + kGW - 1) / kGW);
  if (nCTA < 1) nCTA = 1;
  size_t vbytes = ((sizeof(double) * (size_t)n) + 255) & ~(size_t)255;
  size_t bytes = vbytes * (3 + (m + 1) + (scatter_idx ? 1 : 0)) + sizeof(double) * 2 * kMaxQ * nCTA + sizeof(GridBar) + 384;
  void* ws = nullptr;
  st = dalloc(&ws, bytes, s);
  if (st) return st;
  char* w = (char*)ws;
  GmresArgs a;
  a.A = view(M);
  a.b = b;
  a.r = (double*)w; w += vbytes;
  a.w = (double*)w; w += vbytes;
  a.t = (double*)w; w += vbytes;
  a.V = (double*)w; w += vbytes * (m + 1);
  if (scatter_idx) {
    a.x = (double*)w; w += vbytes;
    cudaError_t e = cudaMemcpyAsync(a.x, x_init, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) { dfree(ws, s); return cuda_fail(e, "cudaMemcpyAsync"); }
  } else {
    a.x = x;
  }
  a.part = (double*)w; w += sizeof(double) * 2 * kMaxQ * nCTA;
  w = (char*)((((uintptr_t)w) + 127) & ~(uintptr_t)127);
  a.bar = (GridBar*)w; w += sizeof(GridBar);
  a.out = (int*)w;
  a.out_relres = (double*)(w + 16);
  a.scatter_idx = scatter_idx;
  a.x_full = x_full;
  a.n = n;
  a.eps = p->rel_tol;
  a.m = m;
  a.max_iters = p->max_iters;
  a.exact_cgs2 = tuning().gmres_exact_cgs2;
  SolveClock clk(defer);
  cudaError_t e = cudaMemsetAsync(a.bar, 0, sizeof(GridBar), s);
  cudaEventRecord(clk.e0, s);
  void* args[] = {&a};
  if (e == cudaSuccess) e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)nCTA), dim3(kGT), args, dsmem, s);
  count_launch();
  cudaEventRecord(clk.e1, s);
  struct FreeAfter { void* p; cudaStream_t s; ~FreeAfter() { dfree(p, s); } } fa{ws, s};
  return solve_finish(e, clk, defer, 1, a.out, a.out + 1, a.out_relres, LC_KERNEL_GMRES, 1, s, info, "GMRES kernel");
}

}  // namespace lc

#ifdef LC_DEBUG_TIMELINE
extern "C" int lc_debug_timeline_gmres(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, lc::g_tlg, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -1;
}
#endif
