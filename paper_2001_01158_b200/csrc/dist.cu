// dist.cu -- NEXT-4: the row-partitioned multi-GPU form of the path (Sec. 2.4, Alg. 4/5).
//
// Rank l owns the row slab I_l of A, b, x.  Per rank the operator is the stencil layout of its
// slab with offsets relative to the slab, so a column c = u + off[k] outside [0, n_l) is a halo row of the
// lower (c < 0) or upper (c >= n_l) neighbour.  B200 form of the paper's communication steps:
//   - "communicate all adjacency components of x from other processors" (Alg. 4 l.4, Alg. 5 l.4, l.17) and
//     the per-iteration halo of the Krylov solve are NOT separate exchanges: the warps of a slab-boundary
//     slice load the neighbour's entries straight from its peer-visible workspace (NVLink P2P loads in a
//     multi-GPU run; ld.global.cv so no stale line is reused), inside the same pass that consumes them;
//   - every global reduction (||b||, max c, K, the admission counts, the Krylov dots) is a fixed-order
//     exchange: after the rank's grid barrier its CTA 0 combines the per-CTA partials, stores the rank's
//     4-vector into slot [seq & 1][rank] of EVERY rank's exchange block and raises flag[rank] = seq there
//     (st.release.sys); every CTA of every rank waits for all flags >= seq and combines
//     the p slots in rank order, so all ranks hold bitwise identical scalars and take identical decisions.
//     Slots are double-buffered by seq parity: a rank can publish seq + 2 only after every rank published
//     seq + 1, which each did after all of its CTAs had read seq.
// One rank per GPU launches the kernel over its own CTAs; with fewer GPUs the p ranks are emulated by ONE
// cooperative launch whose CTAs are split into p groups (blockIdx / nCTA = rank slot), so every wait is
// between co-resident CTAs (B200_PROFILING: never separate launches that wait on each other).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lc_internal.cuh"

namespace lc {

constexpr int kDT = 256;          // threads per CTA
constexpr int kDW = kDT / 32;
constexpr int kMaxRanks = LC_DIST_MAX_RANKS;
constexpr uint8_t kOutD = 255;

struct DXch {                     // one rank's exchange block (peer-visible)
  double slot[2][kMaxRanks][4];
  unsigned long long flag[kMaxRanks];
};

struct DPeer {                    // a neighbour slab's peer-visible vectors (n = 0: no neighbour)
  const double *x0, *x, *z, *p0, *p1;
  const uint8_t* om;
  int64_t n;
};

struct DArgs {
  SellView A;                     // the slab (stencil layout, slab-relative offsets)
  int64_t n, nglob;
  int rank, nranks, minoff, maxoff;
  const double* b;                // rhs of this launch (b, or b_sub for the masked solve)
  double *x0, *x, *z, *p0, *p1;   // own peer-visible vectors
  uint8_t* om;                    // own domain flags (peer-visible)
  double *r, *q, *bs;             // own local vectors
  DPeer lo, hi;
  double* part;                   // [nCTA][4]
  GridBar* bar;
  DXch* xch;                      // own exchange block
  DXch* xpeer[kMaxRanks];         // every rank's exchange block (own included)
  unsigned long long seq0;        // last sequence number used before this launch
  unsigned long long* seq_out;
  // solve
  int masked, max_iters;
  int lazyx;                      // x updated every second iteration (as k_pcg's lazy x, depth 2)
  double eps;
  double* x_user;                 // exit: x_user[u] = x[u] (all rows, or Omega rows when masked)
  // domain
  int crit, thr, rounds, hops;
  double param;
  // results (rank-local copies): i[0] iterations / K-part, i[1] status, i[2] rounds; d[0] relres / tau,
  // d[1] global K
  int* out_i;
  double* out_d;
};

// every rank slot's arguments travel in the launch's parameter space (constant bank: loop-invariant fields
// stay in registers, no aliasing with the stores of the passes)
struct DPack {
  DArgs a[kMaxRanks];
};

// ---------------------------------------------------------------- memory ops ----
__device__ __forceinline__ unsigned long long ld_acq_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint8_t ldcv_u8(const uint8_t* p) {
  unsigned short v;
  asm volatile("ld.global.cv.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return (uint8_t)v;
}

// barrier over the nb CTAs of one rank: the counter form of grid_barrier (lc_internal.cuh) on the rank's own
// GridBar; `epoch` counts this CTA's rank barriers
__device__ __forceinline__ void rank_barrier(GridBar* gb, unsigned nb, unsigned long long& epoch) {
  __syncthreads();
  epoch += nb;
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

// ---------------------------------------------------------------- reductions ----
// op 0: four sums; op 1: (double-double pair, max, sum)
__device__ __forceinline__ void comb(int op, double* a, const double* b) {
  if (op == 0) {
    a[0] += b[0]; a[1] += b[1]; a[2] += b[2]; a[3] += b[3];
  } else {
    dd_add(a[0], a[1], b[0], b[1]);
    a[2] = fmax(a[2], b[2]);
    a[3] += b[3];
  }
}
__device__ __forceinline__ void warp_comb(int op, double* a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) t[j] = __shfl_xor_sync(0xffffffffu, a[j], o);
    comb(op, a, t);
  }
}

// Global (all ranks) combination of the threads' 4-vectors `a`; result in s_out[4] for every thread.
__device__ void xreduce(const DArgs& P, unsigned bid, unsigned nCTA, int op, double* a, double (*s_w)[4],
                        double* s_out, unsigned long long seq, unsigned long long& bep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_comb(op, a);
  if (lane == 0)
    for (int j = 0; j < 4; ++j) s_w[warp][j] = a[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    double c[4] = {s_w[0][0], s_w[0][1], s_w[0][2], s_w[0][3]};
    for (int w = 1; w < kDW; ++w) comb(op, c, s_w[w]);
    for (int j = 0; j < 4; ++j) P.part[4 * bid + j] = c[j];
  }
  rank_barrier(P.bar, nCTA, bep);
  const int par = (int)(seq & 1);
  if (bid == 0) {
    double c[4] = {0.0, 0.0, 0.0, 0.0};
    for (unsigned i = threadIdx.x; i < nCTA; i += kDT) comb(op, c, P.part + 4 * i);
    warp_comb(op, c);
    __syncthreads();
    if (lane == 0)
      for (int j = 0; j < 4; ++j) s_w[warp][j] = c[j];
    __syncthreads();
    if (threadIdx.x == 0) {
      double t[4] = {s_w[0][0], s_w[0][1], s_w[0][2], s_w[0][3]};
      for (int w = 1; w < kDW; ++w) comb(op, t, s_w[w]);
      for (int j = 0; j < 4; ++j) s_out[j] = t[j];
    }
    __syncthreads();
    // thread q publishes the rank's value to rank q (in parallel over the ranks)
    if (threadIdx.x < (unsigned)P.nranks) {
      DXch* X = P.xpeer[threadIdx.x];
      for (int j = 0; j < 4; ++j) X->slot[par][P.rank][j] = s_out[j];
      st_rel_sys(&X->flag[P.rank], seq);          // release at system scope: the slot and (cumulatively)
                                                  // the rank's pass writes observed through its barrier
    }
  }
  // thread q waits for rank q's value; thread 0 then combines the ranks in order
  __shared__ double s_v[kMaxRanks][4];
  if (threadIdx.x < (unsigned)P.nranks) {
    const int q = threadIdx.x;
    while (ld_acq_sys(&P.xch->flag[q]) < seq) {
    }
    for (int j = 0; j < 4; ++j) s_v[q][j] = __ldcv(&P.xch->slot[par][q][j]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t[4] = {s_v[0][0], s_v[0][1], s_v[0][2], s_v[0][3]};
    for (int q = 1; q < P.nranks; ++q) comb(op, t, s_v[q]);
    for (int j = 0; j < 4; ++j) s_out[j] = t[j];
  }
  __syncthreads();
}

// ---------------------------------------------------------------- operands ----
// W: 0 x, 1 z, 2 p = z + beta p_old, 3 x0, 4 x with its pending lazy update (beta = its alpha, pold / par =
// its direction): the CONFIRM pass of a lazy-x solve
template <int OP>
__device__ __forceinline__ double opl(const DArgs& P, int c, double beta, const double* pold) {
  if (OP == 0) return P.x[c];
  if (OP == 1) return P.z[c];
  if (OP == 2) return __fma_rn(beta, pold[c], P.z[c]);
  if (OP == 4) return __fma_rn(beta, pold[c], P.x[c]);
  return P.x0[c];
}
template <int OP>
__device__ __forceinline__ double opp(const DPeer& Q, int i, double beta, int par) {
  if (OP == 0) return __ldcv(Q.x + i);
  if (OP == 1) return __ldcv(Q.z + i);
  if (OP == 2) return __fma_rn(beta, __ldcv((par ? Q.p1 : Q.p0) + i), __ldcv(Q.z + i));
  if (OP == 4) return __fma_rn(beta, __ldcv((par ? Q.p1 : Q.p0) + i), __ldcv(Q.x + i));
  return __ldcv(Q.x0 + i);
}
// operand at slab-relative column c (edge slices may leave [0, n): the neighbours' rows; outside the
// global matrix only zero holes point, and they read 0)
template <int OP>
__device__ __forceinline__ double opnd(const DArgs& P, int c, bool edge, double beta, const double* pold, int par) {
  if (edge) {
    if (c < 0) return P.lo.n ? opp<OP>(P.lo, c + (int)P.lo.n, beta, par) : 0.0;
    if (c >= (int)P.n) return P.hi.n ? opp<OP>(P.hi, c - (int)P.n, beta, par) : 0.0;
  }
  return opl<OP>(P, c, beta, pold);
}
__device__ __forceinline__ uint8_t flag_at(const DArgs& P, int c, bool edge) {
  if (edge) {
    if (c < 0) return P.lo.n ? ldcv_u8(P.lo.om + c + P.lo.n) : kOutD;
    if (c >= (int)P.n) return P.hi.n ? ldcv_u8(P.hi.om + c - P.n) : kOutD;
  }
  return P.om[c];
}
__device__ __forceinline__ bool slice_edge(const DArgs& P, int64_t s) {
  return 32 * s + P.minoff < 0 || 32 * s + 31 + P.maxoff >= P.n;
}

// ---------------------------------------------------------------- PCG ----
enum DMode : int { D_INIT = 0, D_RESET, D_FIRST, D_NORMAL, D_UPDATE, D_CONFIRM, D_DONE };

// one slice of pass A.  EDGE: the slice reaches a neighbour slab (operands of rows outside [0, n) are
// peer loads); else every column is clamped into [0, n) (only zero holes at the global boundary clamp).
template <int WM, int OP, bool EDGE>
__device__ __forceinline__ void dslice_body(const DArgs& P, int64_t s, int lane, bool init, double beta, int par,
                                       const double* __restrict__ pold, double* __restrict__ pnew, double* a) {
  const SellView& A = P.A;
  const int n = (int)P.n;
  const int u = (int)(32 * s) + lane;
  if (u >= n) return;
  const double* vp = A.val + 32ll * A.vw * s + lane;
  double v[WM], y[WM];
#pragma unroll
  for (int k = 0; k < WM; ++k) {
    const bool use = WM != 8 || k < A.W;     // WM 5 / 7: exactly that width
    v[k] = use ? __ldg(vp + 32 * k) : 0.0;
    int c = u + A.off[k];
    if (!EDGE) c = c < 0 ? 0 : (c >= n ? n - 1 : c);
    y[k] = use ? opnd<OP>(P, c, EDGE, beta, pold, par) : 0.0;
  }
  double acc = 0.0, own = 0.0;
#pragma unroll
  for (int k = 0; k < WM; ++k) {
    acc = __fma_rn(v[k], y[k], acc);
    if (A.off[k] == 0 && (WM != 8 || k < A.W)) own = y[k];
  }
  if (P.masked && P.om[u] == kOutD) return;
  if (OP == 0 || OP == 4) {
    const double bi = P.b[u];
    const double ri = bi - acc;
    P.r[u] = ri;
    a[0] = __fma_rn(ri, ri, a[0]);
    if (init) a[1] = __fma_rn(bi, bi, a[1]);
  } else {
    pnew[u] = own;
    P.q[u] = acc;
    a[0] = __fma_rn(own, acc, a[0]);
  }
}

template <int WM, int OP, bool EDGE>
__device__ __forceinline__ void dslice(const DArgs& P, int64_t s, int lane, bool init, double beta, int par,
                                       const double* __restrict__ pold, double* __restrict__ pnew, double* a) {
  dslice_body<WM, OP, EDGE>(P, s, lane, init, beta, par, pold, pnew, a);
}
// the few slab-edge slices: out of line, so their peer-load code does not raise the hot loop's registers
template <int WM, int OP>
__device__ __noinline__ void dslice_edge(const DArgs& P, int64_t s, int lane, bool init, double beta, int par,
                                         const double* pold, double* pnew, double* a) {
  dslice_body<WM, OP, true>(P, s, lane, init, beta, par, pold, pnew, a);
}

// pass A over the rank's slices: OP 0: r = b - A x (+ r^T r, b^T b); OP 1/2: q = A p with p = z (+ beta p_old)
// written for own rows (+ p^T q).  Interior slices [sa, sb) first (no halo code), then the few edge slices.
// Masked solves skip rows outside Omega (their vectors stay 0).
template <int WM, int OP>
__device__ __forceinline__ void dpass_a(const DArgs& P, int64_t sa, int64_t sb, int64_t w0, int64_t wst, int lane,
                                        bool init, double beta, int par, double* a) {
  const double* pold = par ? P.p1 : P.p0;        // (OP 4: the pending direction)
  double* pnew = par ? P.p0 : P.p1;
#pragma unroll 1
  for (int64_t s = sa + w0; s < sb; s += wst) dslice<WM, OP, false>(P, s, lane, init, beta, par, pold, pnew, a);
  const int64_t ne = sa + (P.A.nslices - sb);
#pragma unroll 1
  for (int64_t j = w0; j < ne; j += wst)
    dslice_edge<WM, OP>(P, j < sa ? j : sb + (j - sa), lane, init, beta, par, pold, pnew, a);
}

// pass A with the interior value stream staged by TMA (as k_pcg's pass_a_tma): CTA b owns the chunks
// c = b + t nCTA of 8 consecutive slices, thread 0 keeps kDStages chunks in flight (cp.async.bulk +
// mbarrier complete_tx) and each warp reads its slice's values from shared memory; a slab-edge slice takes
// the out-of-line path (values from L2, operands from the neighbour slab).
constexpr int kDStages = 2;
template <int WM, int OP>
__device__ __forceinline__ void dpass_a_tma(const DArgs& P, double* stg, uint64_t* bars, unsigned bid, unsigned nCTA,
                                            int warp, int lane, bool init, double beta, int par, double* a) {
  const SellView& A = P.A;
  const double* pold = par ? P.p1 : P.p0;
  double* pnew = par ? P.p0 : P.p1;
  const int64_t ns = A.nslices, nch = (ns + kDW - 1) / kDW;
  const int64_t chd = (int64_t)kDW * 32 * WM;
  const int n = (int)P.n, nu1 = n - 1;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kDStages; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int64_t t) {
    const int64_t c = bid + t * nCTA;
    if (c >= nch) return;
    const int st = (int)(t % kDStages);
    const int64_t j0c = (int64_t)kDW * c;
    const int nsl = (int)((ns - j0c) < kDW ? (ns - j0c) : kDW);
    const unsigned bytes = (unsigned)(32 * WM * 8) * nsl;
    mbar_expect_tx(&bars[st], bytes);
    tma_bulk_g2s(stg + st * chd, A.val + j0c * 32 * WM, bytes, &bars[st]);
  };
  if (threadIdx.x == 0)
    for (int t = 0; t < kDStages; ++t) issue(t);
#pragma unroll 1
  for (int64_t t = 0;; ++t) {
    const int64_t c = bid + t * nCTA;
    if (c >= nch) break;
    const int st = (int)(t % kDStages);
    mbar_wait(&bars[st], (unsigned)((t / kDStages) & 1));
    const int64_t s = (int64_t)kDW * c + warp;
    const int u = (int)(32 * s) + lane;
    if (s < ns && u < n) {
      const bool edge = (P.lo.n && 32 * s + P.minoff < 0) || (P.hi.n && 32 * s + 31 + P.maxoff >= P.n);
      if (edge) {
        dslice_edge<WM, OP>(P, s, lane, init, beta, par, pold, pnew, a);
      } else {
        const double* sp = stg + st * chd + (int64_t)warp * 32 * WM + lane;
        double v[WM], y[WM];
#pragma unroll
        for (int k = 0; k < WM; ++k) {
          int cc = u + A.off[k];
          cc = cc < 0 ? 0 : (cc > nu1 ? nu1 : cc);
          v[k] = sp[32 * k];
          y[k] = opl<OP>(P, cc, beta, pold);
        }
        double acc = 0.0, own = 0.0;
#pragma unroll
        for (int k = 0; k < WM; ++k) {
          acc = __fma_rn(v[k], y[k], acc);
          if (A.off[k] == 0) own = y[k];
        }
        if (!P.masked || P.om[u] != kOutD) {
          if (OP == 0 || OP == 4) {
            const double bi = P.b[u];
            const double ri = bi - acc;
            P.r[u] = ri;
            a[0] = __fma_rn(ri, ri, a[0]);
            if (init) a[1] = __fma_rn(bi, bi, a[1]);
          } else {
            pnew[u] = own;
            P.q[u] = acc;
            a[0] = __fma_rn(own, acc, a[0]);
          }
        }
      }
    }
    __syncthreads();                               // every warp is done with stage st
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();
      issue(t + kDStages);
    }
  }
}

template <int WM>
__global__ void __launch_bounds__(kDT, 4) k_dpcg(const __grid_constant__ DPack pk, int nCTA, int tma) {
  __shared__ double s_w[kDW][4], s_out[4];
  extern __shared__ __align__(128) double dsm[];   // TMA stages: kDStages x 8 slices x 32 x WM values
  __shared__ __align__(8) uint64_t s_bars[kDStages];
  __shared__ int s_mode, s_par, s_it, s_final, s_exit, s_pend, s_pbuf;
  __shared__ double s_rho, s_alpha, s_beta, s_tgt, s_nb, s_palpha;
  const unsigned slot = blockIdx.x / nCTA, bid = blockIdx.x % nCTA;
  if (threadIdx.x == 0) {
    s_mode = D_INIT; s_par = 0; s_it = 0; s_final = 0; s_exit = 0; s_pend = 0; s_pbuf = 0;
    s_rho = s_alpha = s_beta = 0.0; s_tgt = s_nb = 0.0; s_palpha = 0.0;
  }
  __syncthreads();
  const DArgs& P = pk.a[slot];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w0 = (int64_t)bid * kDW + warp, wst = (int64_t)nCTA * kDW;
  unsigned long long seq = P.seq0, bep = 0;
  // interior slices: every column of every row inside the slab (or a zero hole at the global boundary)
  const int64_t nsl = P.A.nslices;
  int64_t sa = P.lo.n ? (-P.minoff + 31) / 32 : 0;
  int64_t sb = P.hi.n ? (P.n - 32 - P.maxoff >= 0 ? (P.n - 32 - P.maxoff) / 32 + 1 : 0) : nsl;
  sa = sa < nsl ? sa : nsl;
  sb = sb > sa ? sb : sa;
  auto finish = [&](int status, double rn) {
    s_mode = D_DONE;
    if (bid == 0) {
      P.out_i[0] = s_it;
      P.out_i[1] = status;
      P.out_d[0] = s_nb > 0 ? rn / s_nb : rn;
    }
  };
  for (;;) {
    // ---- pass A
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    const int mode = s_mode;
    if (mode == D_CONFIRM && s_pend) {            // lazy x: true residual at x + the pending alpha p
      if (WM != 8 && tma) dpass_a_tma<WM, 4>(P, dsm, s_bars, bid, nCTA, warp, lane, false, s_palpha, s_pbuf, a);
      else dpass_a<WM, 4>(P, sa, sb, w0, wst, lane, false, s_palpha, s_pbuf, a);
    } else if (WM != 8 && tma) {
      if (mode == D_INIT || mode == D_CONFIRM)
        dpass_a_tma<WM, 0>(P, dsm, s_bars, bid, nCTA, warp, lane, mode == D_INIT, 0.0, s_par, a);
      else if (mode == D_FIRST) dpass_a_tma<WM, 1>(P, dsm, s_bars, bid, nCTA, warp, lane, false, 0.0, s_par, a);
      else if (mode == D_NORMAL) dpass_a_tma<WM, 2>(P, dsm, s_bars, bid, nCTA, warp, lane, false, s_beta, s_par, a);
    } else if (mode == D_INIT || mode == D_CONFIRM) {
      dpass_a<WM, 0>(P, sa, sb, w0, wst, lane, mode == D_INIT, 0.0, s_par, a);
    } else if (mode == D_FIRST) {
      dpass_a<WM, 1>(P, sa, sb, w0, wst, lane, false, 0.0, s_par, a);
    } else if (mode == D_NORMAL) {
      dpass_a<WM, 2>(P, sa, sb, w0, wst, lane, false, s_beta, s_par, a);
    }
    xreduce(P, bid, nCTA, 0, a, s_w, s_out, ++seq, bep);
    if (threadIdx.x == 0) {
      const double s0 = s_out[0], s1 = s_out[1];
      if (mode == D_INIT) {
        s_nb = sqrt(s1);
        s_tgt = s_nb > 0 ? P.eps * s_nb : P.eps;
        const double rn = sqrt(s0);
        if (!isfinite(rn)) finish(LC_ERR_NONFINITE, rn);
        else if (rn <= s_tgt) finish(LC_OK, rn);
        else if (P.max_iters == 0) finish(LC_NOT_CONVERGED, rn);       // Eq. 6 check only
        else s_mode = D_RESET;
      } else if (mode == D_FIRST || mode == D_NORMAL) {
        if (!(s0 > 0)) finish(isfinite(s0) ? LC_ERR_BREAKDOWN : LC_ERR_NONFINITE, NAN);
        else { s_alpha = s_rho / s0; s_mode = D_UPDATE; s_par ^= 1; }
      } else if (mode == D_CONFIRM) {
        const double rn = sqrt(s0);
        if (!isfinite(rn)) finish(LC_ERR_NONFINITE, rn);
        else if (rn <= s_tgt) finish(LC_OK, rn);
        else if (s_final) finish(LC_NOT_CONVERGED, rn);
        else s_mode = D_RESET;
      }
    }
    __syncthreads();
    // ---- pass B (own rows only)
    const int modeb = s_mode;
    a[0] = a[1] = a[2] = a[3] = 0.0;
    if (modeb == D_UPDATE || modeb == D_RESET) {
      // own rows as 16-byte pairs (the slab vectors are 256-byte aligned); rows outside Omega of a masked
      // solve hold p = q = r = 0 and stay 0
      const double alpha = s_alpha;
      const double2* pp = reinterpret_cast<const double2*>(s_par ? P.p1 : P.p0);
      double2* x2 = reinterpret_cast<double2*>(P.x);
      double2* r2 = reinterpret_cast<double2*>(P.r);
      double2* z2 = reinterpret_cast<double2*>(P.z);
      const double2* q2 = reinterpret_cast<const double2*>(P.q);
      const double2* d2 = reinterpret_cast<const double2*>(P.A.dinv);
      const int64_t npair = P.n >> 1, gt = (int64_t)bid * kDT + threadIdx.x, gs = (int64_t)nCTA * kDT;
      // lazy x (as k_pcg): every second UPDATE leaves x alone, the next applies both updates in order
      const int pend = s_pend;
      const double pa = s_palpha;
      const double2* po2 = reinterpret_cast<const double2*>(s_pbuf ? P.p1 : P.p0);
      if (modeb == D_UPDATE && P.lazyx && !pend) {
#pragma unroll 2
        for (int64_t i = gt; i < npair; i += gs) {
          double2 rv = r2[i], qv = q2[i], dv = d2[i];
          rv.x = __fma_rn(-alpha, qv.x, rv.x); rv.y = __fma_rn(-alpha, qv.y, rv.y);
          const double2 zv = make_double2(rv.x * dv.x, rv.y * dv.y);
          r2[i] = rv; z2[i] = zv;
          a[0] = __fma_rn(rv.x, zv.x, a[0]); a[0] = __fma_rn(rv.y, zv.y, a[0]);
          a[1] = __fma_rn(rv.x, rv.x, a[1]); a[1] = __fma_rn(rv.y, rv.y, a[1]);
        }
      } else if (modeb == D_UPDATE && pend) {
#pragma unroll 2
        for (int64_t i = gt; i < npair; i += gs) {
          double2 xv = x2[i], ov = po2[i], pv = pp[i], rv = r2[i], qv = q2[i], dv = d2[i];
          xv.x = __fma_rn(alpha, pv.x, __fma_rn(pa, ov.x, xv.x)); xv.y = __fma_rn(alpha, pv.y, __fma_rn(pa, ov.y, xv.y));
          rv.x = __fma_rn(-alpha, qv.x, rv.x); rv.y = __fma_rn(-alpha, qv.y, rv.y);
          const double2 zv = make_double2(rv.x * dv.x, rv.y * dv.y);
          x2[i] = xv; r2[i] = rv; z2[i] = zv;
          a[0] = __fma_rn(rv.x, zv.x, a[0]); a[0] = __fma_rn(rv.y, zv.y, a[0]);
          a[1] = __fma_rn(rv.x, rv.x, a[1]); a[1] = __fma_rn(rv.y, rv.y, a[1]);
        }
      } else if (modeb == D_UPDATE) {
#pragma unroll 2
        for (int64_t i = gt; i < npair; i += gs) {
          double2 xv = x2[i], pv = pp[i], rv = r2[i], qv = q2[i], dv = d2[i];
          xv.x = __fma_rn(alpha, pv.x, xv.x); xv.y = __fma_rn(alpha, pv.y, xv.y);
          rv.x = __fma_rn(-alpha, qv.x, rv.x); rv.y = __fma_rn(-alpha, qv.y, rv.y);
          const double2 zv = make_double2(rv.x * dv.x, rv.y * dv.y);
          x2[i] = xv; r2[i] = rv; z2[i] = zv;
          a[0] = __fma_rn(rv.x, zv.x, a[0]); a[0] = __fma_rn(rv.y, zv.y, a[0]);
          a[1] = __fma_rn(rv.x, rv.x, a[1]); a[1] = __fma_rn(rv.y, rv.y, a[1]);
        }
      } else {
#pragma unroll 2
        for (int64_t i = gt; i < npair; i += gs) {
          const double2 rv = r2[i], dv = d2[i];
          const double2 zv = make_double2(rv.x * dv.x, rv.y * dv.y);
          z2[i] = zv;
          a[0] = __fma_rn(rv.x, zv.x, a[0]); a[0] = __fma_rn(rv.y, zv.y, a[0]);
          if (pend) {                               // RESET: apply the pending update
            double2 xv = x2[i];
            const double2 ov = po2[i];
            xv.x = __fma_rn(pa, ov.x, xv.x); xv.y = __fma_rn(pa, ov.y, xv.y);
            x2[i] = xv;
          }
        }
      }
      if ((P.n & 1) && gt == 0) {
        const int64_t u = P.n - 1;
        const double* p1 = s_par ? P.p1 : P.p0;
        const double* po = s_pbuf ? P.p1 : P.p0;
        const double di = P.A.dinv[u];
        if (modeb == D_UPDATE) {
          const double ri = __fma_rn(-alpha, P.q[u], P.r[u]);
          const double zi = ri * di;
          if (!P.lazyx) P.x[u] = __fma_rn(alpha, p1[u], P.x[u]);
          else if (pend) P.x[u] = __fma_rn(alpha, p1[u], __fma_rn(pa, po[u], P.x[u]));
          P.r[u] = ri; P.z[u] = zi;
          a[0] = __fma_rn(ri, zi, a[0]);
          a[1] = __fma_rn(ri, ri, a[1]);
        } else {
          const double ri = P.r[u];
          const double zi = ri * di;
          P.z[u] = zi;
          a[0] = __fma_rn(ri, zi, a[0]);
          if (pend) P.x[u] = __fma_rn(pa, po[u], P.x[u]);
        }
      }
    }
    xreduce(P, bid, nCTA, 0, a, s_w, s_out, ++seq, bep);
    if (threadIdx.x == 0) {
      const double s0 = s_out[0], s1 = s_out[1];
      if (modeb == D_UPDATE) {
        s_it += 1;
        if (P.lazyx) {
          if (s_pend) s_pend = 0;
          else { s_pend = 1; s_pbuf = s_par; s_palpha = s_alpha; }
        }
        if (!isfinite(s1) || sqrt(s1) <= s_tgt || s_it >= P.max_iters) {
          s_mode = D_CONFIRM;
          s_final = (s_it >= P.max_iters) || !isfinite(s1);
        } else {
          s_beta = s0 / s_rho;
          s_rho = s0;
          s_mode = D_NORMAL;
        }
      } else if (modeb == D_RESET) {
        s_rho = s0;
        s_mode = D_FIRST;
        s_pend = 0;
      }
      s_exit = s_mode == D_DONE;
    }
    __syncthreads();
    if (s_exit) break;
  }
  // a8 (Eq. 4) / the global solve's result: back into the caller's slab (with a still pending lazy update)
  const double* po = s_pbuf ? P.p1 : P.p0;
  for (int64_t u = (int64_t)bid * kDT + threadIdx.x; u < P.n; u += (int64_t)nCTA * kDT)
    if (!P.masked || P.om[u] != kOutD) P.x_user[u] = s_pend ? __fma_rn(s_palpha, po[u], P.x[u]) : P.x[u];
  if (bid == 0 && threadIdx.x == 0) *P.seq_out = seq;
}

// ---------------------------------------------------------------- domain ----
// Alg. 4 / Alg. 5 on the partition, then the masked extraction (Eq. 3) and the masked-solve start state.
template <int WM>
__global__ void __launch_bounds__(kDT, 2) k_ddomain(const __grid_constant__ DPack pk, int nCTA, int) {
  __shared__ double s_w[kDW][4], s_out[4];
  const unsigned slot = blockIdx.x / nCTA, bid = blockIdx.x % nCTA;
  const DArgs& P = pk.a[slot];
  const SellView& A = P.A;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w0 = (int64_t)bid * kDW + warp, wst = (int64_t)nCTA * kDW;
  const int n = (int)P.n;
  unsigned long long seq = P.seq0, bep = 0;
  double* crit = P.q;
  // ---- criterion (Alg. 5 l.3-5 residual / Alg. 4 l.3-8 gradient) + ||b||^2 (double-double) + max c
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t s = w0; s < A.nslices; s += wst) {
    const int u = (int)(32 * s) + lane;
    if (u >= n) continue;
    const bool edge = slice_edge(P, s);
    const double* vp = A.val + 32ll * A.vw * s + lane;
    double c;
    if (P.crit == LC_CRIT_RESIDUAL) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < WM; ++k) {
        if (k >= A.W) break;
        int cc = u + A.off[k];
        if (!edge) cc = cc < 0 ? 0 : (cc >= n ? n - 1 : cc);
        acc = __fma_rn(__ldg(vp + 32 * k), opnd<3>(P, cc, edge, 0.0, nullptr, 0), acc);
      }
      const double bi = P.b[u];
      const double ri = bi - acc;
      P.r[u] = ri;
      c = fabs(ri);
      dd_add_sq(a[0], a[1], bi);
    } else {
      const double xi = P.x0[u];
      double acc = 0.0;
      const unsigned m = A.mask[u];
      for (int k = 0; k < A.W; ++k) {
        if (!((m >> k) & 1) || A.off[k] == 0) continue;
        acc = acc + fabs(xi - opnd<3>(P, u + A.off[k], true, 0.0, nullptr, 0));
      }
      c = acc;
    }
    crit[u] = c;
    a[2] = fmax(a[2], c);
  }
  xreduce(P, bid, nCTA, 1, a, s_w, s_out, ++seq, bep);
  double tau, tc;
  if (P.thr == LC_THR_PERCENTILE) {
    // nearest-rank p-quantile of c over ALL ranks (R14): radix select on the f64 bit patterns (c >= 0, so the
    // patterns order like the values), 2 bits per pass -- the four digit counts of the keys that still match
    // the prefix are one exchange (exact integers in doubles), every CTA of every rank takes the same digit
    long long k = (long long)ceil(P.param * (double)P.nglob) - 1;
    if (k < 0) k = 0;
    if (k > P.nglob - 1) k = P.nglob - 1;
    unsigned long long prefix = 0ull, mask = 0ull;
    for (int shift = 62; shift >= 0; shift -= 2) {
      a[0] = a[1] = a[2] = a[3] = 0.0;
      for (int64_t u = (int64_t)bid * kDT + threadIdx.x; u < n; u += (int64_t)nCTA * kDT) {
        const unsigned long long key = (unsigned long long)__double_as_longlong(crit[u]);
        if ((key & mask) != prefix) continue;
        const int d = (int)((key >> shift) & 3ull);
        a[0] += d == 0 ? 1.0 : 0.0; a[1] += d == 1 ? 1.0 : 0.0; a[2] += d == 2 ? 1.0 : 0.0; a[3] += d == 3 ? 1.0 : 0.0;
      }
      xreduce(P, bid, nCTA, 0, a, s_w, s_out, ++seq, bep);
      long long cum = 0;
      int d = 0;
      for (; d < 3; ++d) {
        const long long cnt = (long long)s_out[d];
        if (k < cum + cnt) break;
        cum += cnt;
      }
      k -= cum;
      prefix |= (unsigned long long)d << shift;
      mask |= 3ull << shift;
      __syncthreads();                                                       // s_out is rewritten by the next pass
    }
    tau = __longlong_as_double((long long)prefix);
    tc = tau;
  } else if (P.thr == LC_THR_PAPER) {
    const double nb = sqrt(s_out[0] + s_out[1]);
    tau = P.param * nb / sqrt((double)P.nglob);                              // Eq. 7 with the global N
    tc = tau;
  } else {
    tau = P.param * s_out[2];                                                // Alg. 4 l.12, global g_max
    tc = P.param == 0.0 ? -1.0 : tau;                                        // alpha = 0 => Omega (R11)
  }
  // ---- mark (strict, R10) and K
  a[0] = a[1] = a[2] = a[3] = 0.0;
  for (int64_t u = (int64_t)bid * kDT + threadIdx.x; u < n; u += (int64_t)nCTA * kDT) {
    const bool in = crit[u] > tc;
    P.om[u] = in ? 0 : kOutD;
    a[0] += in ? 1.0 : 0.0;
  }
  xreduce(P, bid, nCTA, 0, a, s_w, s_out, ++seq, bep);                           // also: flags visible to peers
  int stage = 1, rounds = 0;
  // ---- Alg. 5 l.15-34: expansion rounds; stop when the GLOBAL admission count is 0 (R40)
  for (int rd = 0; rd < P.rounds; ++rd, ++stage) {
    a[0] = a[1] = a[2] = a[3] = 0.0;
    for (int64_t s = w0; s < A.nslices; s += wst) {
      const int u = (int)(32 * s) + lane;
      if (u >= n) continue;
      if (P.om[u] < stage) continue;
      const bool edge = slice_edge(P, s);
      const double* vp = A.val + 32ll * A.vw * s + lane;
      const unsigned m = A.mask[u];
      bool nbr = false;
      double sum = 0.0;
      for (int k = 0; k < A.W; ++k) {
        if (!((m >> k) & 1) || A.off[k] == 0) continue;
        const int cc = u + A.off[k];
        if (flag_at(P, cc, edge) < stage) {
          nbr = true;
          sum = sum + fabs(__ldg(vp + 32 * k) * opnd<3>(P, cc, true, 0.0, nullptr, 0));
        }
      }
      if (nbr && fabs(P.r[u]) + sum > tc) {                                  // Eq. 8
        P.om[u] = (uint8_t)stage;
        a[0] += 1.0;
      }
    }
    xreduce(P, bid, nCTA, 0, a, s_w, s_out, ++seq, bep);
    ++rounds;
    if (s_out[0] == 0.0) { stage = 1 + P.rounds; break; }
  }
  stage = 1 + P.rounds;
  // ---- unconditional dilation hops (R15)
  for (int h = 0; h < P.hops; ++h, ++stage) {
    a[0] = a[1] = a[2] = a[3] = 0.0;
    for (int64_t s = w0; s < A.nslices; s += wst) {
      const int u = (int)(32 * s) + lane;
      if (u >= n) continue;
      if (P.om[u] < stage) continue;
      const bool edge = slice_edge(P, s);
      const unsigned m = A.mask[u];
      for (int k = 0; k < A.W; ++k) {
        if (!((m >> k) & 1) || A.off[k] == 0) continue;
        if (flag_at(P, u + A.off[k], edge) < stage) { P.om[u] = (uint8_t)stage; break; }
      }
    }
    xreduce(P, bid, nCTA, 0, a, s_w, s_out, ++seq, bep);
  }
  // ---- Eq. 3 on Omega rows: b_sub = b - (fma chain over stored columns outside Omega, ascending);
  //      masked-solve start: x = x0 on Omega, 0 elsewhere; r, z, q, p0, p1 = 0
  a[0] = a[1] = a[2] = a[3] = 0.0;
  for (int64_t s = w0; s < A.nslices; s += wst) {
    const int u = (int)(32 * s) + lane;
    if (u >= n) continue;
    const bool edge = slice_edge(P, s);
    const bool in = P.om[u] != kOutD;
    double bsu = 0.0, xu = 0.0;
    if (in) {
      const double* vp = A.val + 32ll * A.vw * s + lane;
      const unsigned m = A.mask[u];
      double acc = 0.0;
      for (int k = 0; k < A.W; ++k) {
        if (!((m >> k) & 1)) continue;
        const int cc = u + A.off[k];
        if (flag_at(P, cc, edge) == kOutD) acc = __fma_rn(__ldg(vp + 32 * k), opnd<3>(P, cc, true, 0.0, nullptr, 0), acc);
      }
      bsu = P.b[u] - acc;
      xu = P.x0[u];
      a[0] += 1.0;
    }
    P.bs[u] = bsu;
    P.x[u] = xu;
    P.r[u] = 0.0; P.z[u] = 0.0; P.q[u] = 0.0; P.p0[u] = 0.0; P.p1[u] = 0.0;
  }
  xreduce(P, bid, nCTA, 0, a, s_w, s_out, ++seq, bep);
  if (bid == 0 && threadIdx.x == 0) {
    P.out_d[0] = tau;
    P.out_d[1] = s_out[0];
    P.out_i[2] = rounds;
    *P.seq_out = seq;
  }
}

}  // namespace lc

using namespace lc;

// ---------------------------------------------------------------- handle ----
struct lc_dist_s {
  int64_t nglob = 0, row0 = 0, n = 0;
  int rank = 0, nranks = 1;
  Sell A;
  int minoff = 0, maxoff = 0;
  void* pv = nullptr;                 // peer-visible block (cudaMalloc)
  double *x0 = nullptr, *x = nullptr, *z = nullptr, *p0 = nullptr, *p1 = nullptr;
  uint8_t* om = nullptr;
  DXch* xch = nullptr;
  void* loc = nullptr;                // local block
  double *r = nullptr, *q = nullptr, *bs = nullptr, *part = nullptr, *out_d = nullptr;
  GridBar* bar = nullptr;
  int* out_i = nullptr;
  unsigned long long* seq_dev = nullptr;
  unsigned long long seq = 0;
  DPeer lo{}, hi{};
  DXch* xpeer[kMaxRanks] = {nullptr};
  std::vector<void*> opened;          // IPC mappings to close
  int connected = 0, have_domain = 0;
  double tau = 0.0;
  int64_t K = 0;
};

namespace {

struct PvLayout { size_t x0, x, z, p0, p1, om, xch, bytes; };
PvLayout pv_layout(int64_t n) {
  PvLayout L;
  size_t o = 0;
  const size_t vb = ((sizeof(double) * (size_t)n) + 255) & ~(size_t)255;
  L.x0 = o; o += vb; L.x = o; o += vb; L.z = o; o += vb; L.p0 = o; o += vb; L.p1 = o; o += vb;
  L.om = o; o += ((size_t)n + 255) & ~(size_t)255;
  L.xch = o; o += (sizeof(DXch) + 255) & ~(size_t)255;
  L.bytes = o;
  return L;
}
DPeer peer_of(char* base, int64_t n) {
  PvLayout L = pv_layout(n);
  DPeer q;
  q.x0 = (const double*)(base + L.x0); q.x = (const double*)(base + L.x); q.z = (const double*)(base + L.z);
  q.p0 = (const double*)(base + L.p0); q.p1 = (const double*)(base + L.p1); q.om = (const uint8_t*)(base + L.om);
  q.n = n;
  return q;
}

void* kernel_of(int which, int W) {
  const int wi = W == 5 ? 0 : W == 7 ? 1 : 2;      // 5- / 7-point stencils, else the generic width
  void* const f[6] = {(void*)k_dpcg<5>, (void*)k_dpcg<7>, (void*)k_dpcg<8>,
                      (void*)k_ddomain<5>, (void*)k_ddomain<7>, (void*)k_ddomain<8>};
  return f[which * 3 + wi];
}

lc_status check_ranks(lc_dist* R, int nr, const char* who) {
  if (!R || nr < 1 || nr > kMaxRanks) { set_error(std::string(who) + ": need 1..8 rank handles"); return LC_ERR_INVALID_ARG; }
  for (int i = 0; i < nr; ++i) {
    if (!R[i]) { set_error(std::string(who) + ": NULL rank handle"); return LC_ERR_INVALID_ARG; }
    if (!R[i]->connected) { set_error(std::string(who) + ": rank not connected (lc_dist_connect*)"); return LC_ERR_INVALID_ARG; }
    if (nr > 1 && (R[i]->rank != i || R[i]->nranks != nr)) {
      set_error(std::string(who) + ": emulation needs all nranks handles in rank order");
      return LC_ERR_INVALID_ARG;
    }
  }
  return LC_OK;
}

DArgs base_args(lc_dist D) {
  DArgs a;
  memset(&a, 0, sizeof(a));
  a.A = view(D->A);
  a.n = D->n; a.nglob = D->nglob; a.rank = D->rank; a.nranks = D->nranks;
  a.minoff = D->minoff; a.maxoff = D->maxoff;
  a.x0 = D->x0; a.x = D->x; a.z = D->z; a.p0 = D->p0; a.p1 = D->p1; a.om = D->om;
  a.r = D->r; a.q = D->q; a.bs = D->bs;
  a.lo = D->lo; a.hi = D->hi;
  a.part = D->part; a.bar = D->bar; a.xch = D->xch;
  for (int q = 0; q < kMaxRanks; ++q) a.xpeer[q] = D->xpeer[q];
  a.seq0 = D->seq; a.seq_out = D->seq_dev;
  a.out_i = D->out_i; a.out_d = D->out_d;
  return a;
}

// one cooperative launch over the nr ranks driven by this call (nCTA CTAs each); syncs, reads back seq
lc_status launch(lc_dist* R, int nr, int which, std::vector<DArgs>& args, cudaStream_t s, float* ms) {
  int W = R[0]->A.maxw;
  for (int i = 1; i < nr; ++i)
    if (R[i]->A.maxw != W) W = 8;                      // mixed widths: the generic variant
  void* fn = kernel_of(which, W);
  int tma = (which == 0 && (W == 5 || W == 7) && tuning().pcg_tma) ? 1 : 0;
  const size_t dsmem = tma ? (size_t)kDStages * kDW * 32 * W * sizeof(double) : 0;
  int64_t dmax = 0;
  lc_status st = max_coresident(fn, kDT, dsmem, &dmax);
  if (st) return st;
  int64_t ns = 1;
  for (int i = 0; i < nr; ++i) ns = std::max<int64_t>(ns, R[i]->A.nslices);
  int nCTA = (int)std::min<int64_t>(dmax / nr, (ns + kDW - 1) / kDW);
  if (nCTA < 1) nCTA = 1;
  DPack pk;
  memset(&pk, 0, sizeof(pk));
  for (int i = 0; i < nr; ++i) pk.a[i] = args[i];
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < nr && e == cudaSuccess; ++i) e = cudaMemsetAsync(R[i]->bar, 0, sizeof(GridBar), s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  void* kargs[] = {(void*)&pk, (void*)&nCTA, (void*)&tma};
  if (e == cudaSuccess) e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)(nr * nCTA)), dim3(kDT), kargs, dsmem, s);
  if (e == cudaSuccess) count_launch();
  cudaEventRecord(e1, s);
  std::vector<unsigned long long> sq(nr, 0);
  for (int i = 0; i < nr && e == cudaSuccess; ++i)
    e = cudaMemcpyAsync(&sq[i], R[i]->seq_dev, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && ms) cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  if (e != cudaSuccess) return cuda_fail(e, "dist kernel");
  for (int i = 0; i < nr; ++i) R[i]->seq = sq[i];
  return LC_OK;
}

lc_status run_dpcg(lc_dist* R, int nr, const double* const* b, double* const* xu, int masked,
                   const lc_solver_params* p, cudaStream_t s, lc_solve_info* info) {
  std::vector<DArgs> args(nr);
  for (int i = 0; i < nr; ++i) {
    DArgs a = base_args(R[i]);
    a.b = masked ? R[i]->bs : b[i];
    a.masked = masked;
    a.x_user = xu[i];
    a.eps = p->rel_tol;
    a.max_iters = p->max_iters;
    a.lazyx = tuning().lazy_x_depth > 1 ? 1 : 0;
    args[i] = a;
    if (!masked) LC_CUDA(cudaMemcpyAsync(R[i]->x, xu[i], sizeof(double) * R[i]->n, cudaMemcpyDeviceToDevice, s));
  }
  float ms = 0.f;
  lc_status st = launch(R, nr, 0, args, s, &ms);
  if (st) return st;
  int oi[2] = {0, 0};
  double od = 0.0;
  LC_CUDA(cudaMemcpyAsync(oi, R[0]->out_i, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  LC_CUDA(cudaMemcpyAsync(&od, R[0]->out_d, sizeof(double), cudaMemcpyDeviceToHost, s));
  LC_CUDA(cudaStreamSynchronize(s));
  if (info) {
    info->iterations = oi[0];
    info->status = oi[1];
    info->rel_residual = od;
    info->seconds = ms * 1e-3;
  }
  return oi[1] < 0 ? (lc_status)oi[1] : (oi[1] == LC_NOT_CONVERGED ? LC_NOT_CONVERGED : LC_OK);
}

}  // namespace

extern "C" lc_status lc_dist_create(int64_t n_global, int64_t row0, int64_t n_local, int32_t rank, int32_t nranks,
                                    const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                                    int32_t inputs_on_device, void* stream, lc_dist* out) {
  if (!out) { set_error("lc_dist_create: out is NULL"); return LC_ERR_INVALID_ARG; }
  *out = nullptr;
  if (!row_ptr || !col_idx || !values) { set_error("lc_dist_create: null array"); return LC_ERR_INVALID_ARG; }
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || n_local < 1 || row0 < 0 ||
      row0 + n_local > n_global || n_global > (int64_t)INT32_MAX - 64) {
    set_error("lc_dist_create: need 1 <= nranks <= 8, 0 <= rank < nranks, n_local >= 1, row0 + n_local <= n_global < 2^31");
    return LC_ERR_DIMENSION;
  }
  cudaStream_t s = (cudaStream_t)stream;
  lc_dist_s* D = new lc_dist_s();
  D->nglob = n_global; D->row0 = row0; D->n = n_local; D->rank = rank; D->nranks = nranks;
  int64_t nnz = 0;
  lc_status st = build_slab(n_global, row0, n_local, row_ptr, col_idx, values, inputs_on_device, s, D->A, &nnz);
  if (st) { delete D; return st; }
  D->minoff = 0; D->maxoff = 0;
  for (int k = 0; k < D->A.maxw; ++k) { D->minoff = std::min(D->minoff, D->A.off[k]); D->maxoff = std::max(D->maxoff, D->A.off[k]); }
  const PvLayout L = pv_layout(n_local);
  const size_t vb = ((sizeof(double) * (size_t)n_local) + 255) & ~(size_t)255;
  const int maxcta = (2048 / kDT) * num_sms();     // upper bound of co-resident CTAs
  const size_t lbytes = 3 * vb + (sizeof(double) * 4 * maxcta + 255) + sizeof(GridBar) + 1024;
  cudaError_t e = cudaMalloc(&D->pv, L.bytes);
  if (e == cudaSuccess) e = cudaMemsetAsync(D->pv, 0, L.bytes, s);
  if (e != cudaSuccess) { D->A.release(s); delete D; return cuda_fail(e, "lc_dist_create: workspace"); }
  char* b = (char*)D->pv;
  D->x0 = (double*)(b + L.x0); D->x = (double*)(b + L.x); D->z = (double*)(b + L.z);
  D->p0 = (double*)(b + L.p0); D->p1 = (double*)(b + L.p1); D->om = (uint8_t*)(b + L.om); D->xch = (DXch*)(b + L.xch);
  st = dalloc(&D->loc, lbytes, s);
  if (st) { cudaFree(D->pv); D->A.release(s); delete D; return st; }
  char* w = (char*)D->loc;
  D->r = (double*)w; w += vb;
  D->q = (double*)w; w += vb;
  D->bs = (double*)w; w += vb;
  D->part = (double*)w; w += (sizeof(double) * 4 * maxcta + 255) & ~(size_t)255;
  D->bar = (GridBar*)w; w += (sizeof(GridBar) + 255) & ~(size_t)255;
  D->out_i = (int*)w; w += 64;
  D->out_d = (double*)w; w += 64;
  D->seq_dev = (unsigned long long*)w;
  e = cudaMemsetAsync(D->loc, 0, lbytes, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { lc_dist_destroy(D); return cuda_fail(e, "lc_dist_create"); }
  *out = D;
  return LC_OK;
}

extern "C" lc_status lc_dist_export_handle(lc_dist D, void* handle) {
  if (!D || !handle) { set_error("lc_dist_export_handle: null argument"); return LC_ERR_INVALID_ARG; }
  static_assert(sizeof(cudaIpcMemHandle_t) <= LC_DIST_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  LC_CUDA(cudaIpcGetMemHandle(&h, D->pv));
  memset(handle, 0, LC_DIST_HANDLE_BYTES);
  memcpy(handle, &h, sizeof(h));
  return LC_OK;
}

static lc_status check_halo(lc_dist D, const int64_t* nl) {
  if (D->rank > 0 && nl[D->rank - 1] < -D->minoff) {
    set_error("lc_dist_connect: the lower neighbour slab is shorter than the stencil reach into it");
    return LC_ERR_DIMENSION;
  }
  if (D->rank + 1 < D->nranks && nl[D->rank + 1] < D->maxoff) {
    set_error("lc_dist_connect: the upper neighbour slab is shorter than the stencil reach into it");
    return LC_ERR_DIMENSION;
  }
  return LC_OK;
}

extern "C" lc_status lc_dist_connect(lc_dist D, const void* handles, const int64_t* n_local_all) {
  if (!D || !handles || !n_local_all) { set_error("lc_dist_connect: null argument"); return LC_ERR_INVALID_ARG; }
  lc_status st = check_halo(D, n_local_all);
  if (st) return st;
  for (int q = 0; q < D->nranks; ++q) {
    char* base;
    if (q == D->rank) {
      base = (char*)D->pv;
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, (const char*)handles + (size_t)q * LC_DIST_HANDLE_BYTES, sizeof(h));
      void* p = nullptr;
      LC_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      D->opened.push_back(p);
      base = (char*)p;
    }
    D->xpeer[q] = (DXch*)(base + pv_layout(n_local_all[q]).xch);
    if (q == D->rank - 1) D->lo = peer_of(base, n_local_all[q]);
    if (q == D->rank + 1) D->hi = peer_of(base, n_local_all[q]);
  }
  D->connected = 1;
  return LC_OK;
}

extern "C" lc_status lc_dist_connect_local(lc_dist* R, int32_t nr) {
  if (!R || nr < 1 || nr > kMaxRanks) { set_error("lc_dist_connect_local: need 1..8 handles"); return LC_ERR_INVALID_ARG; }
  std::vector<int64_t> nl(nr);
  for (int i = 0; i < nr; ++i) {
    if (!R[i] || R[i]->rank != i || R[i]->nranks != nr) {
      set_error("lc_dist_connect_local: handles must be ranks 0..nranks-1 of one partition, in order");
      return LC_ERR_INVALID_ARG;
    }
    if (i > 0 && R[i]->row0 != R[i - 1]->row0 + R[i - 1]->n) {
      set_error("lc_dist_connect_local: slabs must be contiguous and ascending");
      return LC_ERR_DIMENSION;
    }
    nl[i] = R[i]->n;
  }
  if (R[0]->row0 != 0 || R[nr - 1]->row0 + R[nr - 1]->n != R[0]->nglob) {
    set_error("lc_dist_connect_local: slabs must cover [0, n_global)");
    return LC_ERR_DIMENSION;
  }
  for (int i = 0; i < nr; ++i) {
    lc_status st = check_halo(R[i], nl.data());
    if (st) return st;
  }
  for (int i = 0; i < nr; ++i) {
    for (int q = 0; q < nr; ++q) R[i]->xpeer[q] = R[q]->xch;
    R[i]->lo = i > 0 ? peer_of((char*)R[i - 1]->pv, R[i - 1]->n) : DPeer{};
    R[i]->hi = i + 1 < nr ? peer_of((char*)R[i + 1]->pv, R[i + 1]->n) : DPeer{};
    R[i]->connected = 1;
  }
  return LC_OK;
}

extern "C" lc_status lc_dist_select_domain(lc_dist* R, int32_t nr, const double* const* b, const double* const* x0,
                                           const lc_domain_params* p, void* stream, int64_t* K_global) {
  lc_status st = check_ranks(R, nr, "lc_dist_select_domain");
  if (st) return st;
  if (!b || !x0 || !p) { set_error("lc_dist_select_domain: null argument"); return LC_ERR_INVALID_ARG; }
  if (p->criterion != LC_CRIT_RESIDUAL && p->criterion != LC_CRIT_GRADIENT) {
    set_error("lc_dist_select_domain: bad criterion"); return LC_ERR_INVALID_ARG;
  }
  if (p->threshold == LC_THR_PAPER ? !(p->param > 0)
      : p->threshold == LC_THR_REL_MAX ? !(p->param >= 0 && p->param <= 1)
      : p->threshold == LC_THR_PERCENTILE ? !(p->param > 0 && p->param < 1) : true) {
    set_error("lc_dist_select_domain: bad threshold / param (eps > 0, theta in [0,1], p in (0,1))");
    return LC_ERR_INVALID_ARG;
  }
  if (p->expand_rounds < 0 || p->expand_rounds > 64 || p->dilate_hops < 0 || p->dilate_hops > 64 ||
      (p->expand_rounds > 0 && p->criterion != LC_CRIT_RESIDUAL)) {
    set_error("lc_dist_select_domain: expand_rounds in [0,64] (residual criterion only), dilate_hops in [0,64]");
    return LC_ERR_INVALID_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<DArgs> args(nr);
  for (int i = 0; i < nr; ++i) {
    if (!b[i] || !x0[i]) { set_error("lc_dist_select_domain: null slab pointer"); return LC_ERR_INVALID_ARG; }
    LC_CUDA(cudaMemcpyAsync(R[i]->x0, x0[i], sizeof(double) * R[i]->n, cudaMemcpyDeviceToDevice, s));
    DArgs a = base_args(R[i]);
    a.b = b[i];
    a.crit = p->criterion; a.thr = p->threshold; a.rounds = p->expand_rounds; a.hops = p->dilate_hops;
    a.param = p->param;
    args[i] = a;
  }
  st = launch(R, nr, 1, args, s, nullptr);
  if (st) return st;
  double od[2] = {0.0, 0.0};
  for (int i = 0; i < nr; ++i) {
    LC_CUDA(cudaMemcpyAsync(od, R[i]->out_d, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    R[i]->tau = od[0];
    R[i]->K = (int64_t)od[1];
    R[i]->have_domain = 1;
  }
  if (K_global) *K_global = (int64_t)od[1];
  return LC_OK;
}

extern "C" lc_status lc_dist_domain_export(lc_dist D, uint8_t* flag_dev, double* tau_host, void* stream) {
  if (!D) { set_error("lc_dist_domain_export: NULL handle"); return LC_ERR_INVALID_ARG; }
  if (!D->have_domain) { set_error("lc_dist_domain_export: no domain selected"); return LC_ERR_INVALID_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  if (flag_dev) LC_CUDA(cudaMemcpyAsync(flag_dev, D->om, D->n, cudaMemcpyDeviceToDevice, s));
  if (tau_host) *tau_host = D->tau;
  LC_CUDA(cudaStreamSynchronize(s));
  return LC_OK;
}

static lc_status check_solver(const lc_solver_params* p, const char* who) {
  if (!p || p->method != LC_PCG || !(p->rel_tol > 0) || p->max_iters < 0) {
    set_error(std::string(who) + ": needs LC_PCG, rel_tol > 0, max_iters >= 0");
    return LC_ERR_INVALID_ARG;
  }
  return LC_OK;
}

extern "C" lc_status lc_dist_solve_local(lc_dist* R, int32_t nr, const lc_solver_params* p, double* const* x,
                                         void* stream, lc_solve_info* info) {
  lc_status st = check_ranks(R, nr, "lc_dist_solve_local");
  if (st) return st;
  if ((st = check_solver(p, "lc_dist_solve_local"))) return st;
  if (!x) { set_error("lc_dist_solve_local: null x"); return LC_ERR_INVALID_ARG; }
  for (int i = 0; i < nr; ++i)
    if (R[i]->have_domain != 1) {
      set_error("lc_dist_solve_local: needs the state of a preceding lc_dist_select_domain (consumed by a solve)");
      return LC_ERR_INVALID_ARG;
    }
  for (int i = 0; i < nr; ++i) R[i]->have_domain = 2;
  if (R[0]->K == 0) {
    if (info) { info->iterations = 0; info->status = LC_OK; info->rel_residual = 0.0; info->seconds = 0.0; }
    return LC_OK;
  }
  return run_dpcg(R, nr, nullptr, x, 1, p, (cudaStream_t)stream, info);
}

extern "C" lc_status lc_dist_solve_global(lc_dist* R, int32_t nr, const double* const* b, double* const* x,
                                          const lc_solver_params* p, void* stream, lc_solve_info* info) {
  lc_status st = check_ranks(R, nr, "lc_dist_solve_global");
  if (st) return st;
  if ((st = check_solver(p, "lc_dist_solve_global"))) return st;
  if (!b || !x) { set_error("lc_dist_solve_global: null b / x"); return LC_ERR_INVALID_ARG; }
  for (int i = 0; i < nr; ++i)
    if (R[i]->have_domain == 1) R[i]->have_domain = 2;      // the iterate vectors are reused
  return run_dpcg(R, nr, b, x, 0, p, (cudaStream_t)stream, info);
}

extern "C" void lc_dist_destroy(lc_dist D) {
  if (!D) return;
  for (void* p : D->opened) cudaIpcCloseMemHandle(p);
  D->A.release(0);
  dfree(D->loc, 0);
  cudaStreamSynchronize(0);
  if (D->pv) cudaFree(D->pv);
  delete D;
}
