// pcg.cu -- Jacobi-preconditioned CG as ONE persistent cooperative kernel
// (SURVEY 8(a) a7 local solve, a8 assembly, a9 global solve, a10 method0).
//
// The Krylov loop never returns to the host.  Two grid-wide barriers separate
// the two fused passes of an iteration:
//
//   pass A  q = A p with the p-update p = z + beta p_old applied on the fly to
//           every operand (own row written to the other p buffer), fused with
//           the p^T q partials;                    [or r = b - A x for INIT/CONFIRM]
//   pass B  x += alpha p, r -= alpha q, z = D^-1 r, fused with r^T z and r^T r.
//
// Step order and the true-residual confirmation follow the oracle (or_pcg):
// tolerance eps ||b||_2 (Eq. 6), recursive test then the true
// residual (R19); iterations = SpMVs with p (R30).
//
// Work distribution: the slices (all of them, or an active-slice list) are
// interleaved over every warp of the grid, so the grid sweeps one contiguous
// window of rows (plane neighbours of a 7-point stencil stay L2 hits) and a
// batched block-diagonal system (config 3) keeps every SM busy until its last
// group converges.  Every CTA holds the scalar state of ALL segments and
// updates it identically from fixed-order reductions (G = 1: each CTA sums the
// per-CTA partials; G > 1: CTA g reduces segment g, one extra grid barrier),
// so control flow is grid-uniform and results are bitwise deterministic.
//
// Masked local solves (stencil layout): B = A[Omega, Omega] is applied as the
// stencil SpMV restricted to rows in Omega on vectors that are zero outside
// Omega, over the slices that contain Omega rows.  The dropped couplings
// multiply exact zeros, so each row's fma chain equals B's chain (R22).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "lc_internal.cuh"

namespace cg = cooperative_groups;

namespace lc {

#ifndef LC_PCG_PT
#define LC_PCG_PT 256
#endif
constexpr int kPT = LC_PCG_PT;        // threads per CTA
constexpr int kPW = kPT / 32;        // warps per CTA
constexpr int kMaxSeg = 64;

enum Mode : int { M_INIT = 0, M_RESET, M_FIRST, M_NORMAL, M_UPDATE, M_CONFIRM, M_DONE };

struct PcgArgs {
  SellView A;
  const double* b;
  double* x;
  double* r;
  double* z;
  double* q;
  double* p0;
  double* p1;
  double* p2;                   // third search-direction buffer (np3: lazy x of depth 3)
  int np3;                      // 1: p rotates over p0, p1, p2; 0: over p0, p1
  double* part;                 // [nCTA][G][2]
  double* red;                  // [G][2]  (G > 1)
  double* subred;               // [2][kBarSub][G][2]  (G > 1: per-sub-group sums, double-buffered)
  GridBar* bar;                 // zeroed at launch
  int* out_iters;               // [G]
  int* out_status;
  double* out_relres;
  const int32_t* slist;         // optional active slices (ascending)
  const int64_t* nlist;         // device count of slist
  const uint8_t* omega;         // optional: unit u is a row of the subsystem iff omega[u] != 255
  const int64_t* seg_j0;        // [G+1] start of each segment's run in the slice space (list or slices)
  const int32_t* scatter_idx;   // explicit local solve: x_full[scatter_idx[l]] = x[l] at exit
  double* x_full;
  double* x_user;               // masked local solve: x_user[u] = x[u] for u in Omega at exit
  double eps;
  int max_iters;
  int G;
  int reg_units;                // > 0: equal segments of reg_units units, spg slices each (arithmetic maps)
  int spg;
  int vec2;                     // flat double2 update pass (G = 1, no list, aligned)
  int tma;                      // pass A values staged by TMA (G = 1, no list, stencil layout)
  int lazyx;                    // (vec2 solves) x is updated every lazyx-th iteration (0: every one): pass B
  int cluster;                  // launched as ONE thread-block cluster (small G = 1 systems): cluster
                                // barriers and DSMEM partial exchange instead of the global grid barrier
  int clus;                     // (G > 1, lock step) launched in thread-block clusters: cluster_reduce_barrier
  int teams;                    // > 0 (G > 1): the CTAs form `teams` contiguous teams; team t solves segments
                                // t, t + teams, ... one after another as G = 1 systems with its own barrier
  unsigned long long* tctr;     // [teams][16] team barrier counters (zeroed at launch)
  int stream_vals;              // the matrix stream loads with the L2 evict_first policy (stream_policy_wanted)
  long long l2_bytes;           // dynamic teams: the policy follows the active groups' working set
};

struct SegState {
  int mode, par, it, final_;
  double rho, alpha, beta, tgt, nb;
  int pend, pbuf, pbuf2;        // lazy x (P.lazyx): x lacks palpha p[pbuf] (pend >= 1), then palpha2 p[pbuf2]
  int npass;                    // dynamic teams: passes done on the segment (parity of its chunk partials)
  double palpha, palpha2;       // (pend = 2), p[i] = p0 / p1 / p2
};

__device__ __forceinline__ void slice_map(const PcgArgs& P, int64_t s, int& g, int64_t& row0, int64_t& end) {
  if (P.G == 1) {                    // one segment: slice s holds units 32 s .. (no table loads on the path)
    g = 0; row0 = 32 * s; end = P.A.nunits;
    return;
  }
  if (P.reg_units > 0) {
    if (P.G == 1) {
      g = 0; row0 = 32 * s; end = P.reg_units;
    } else {
      g = (int)(s / P.spg);
      row0 = (int64_t)g * P.reg_units + 32 * (s - (int64_t)g * P.spg);
      end = (int64_t)(g + 1) * P.reg_units;
    }
  } else {
    g = P.A.slice_seg[s];
    row0 = P.A.slice_row0[s];
    end = P.A.seg_unit0[g + 1];
  }
}

// search-direction buffer i and its successor in the rotation
__device__ __forceinline__ double* pvec(const PcgArgs& P, int i) { return i == 0 ? P.p0 : (i == 1 ? P.p1 : P.p2); }
__device__ __forceinline__ int pnext(const PcgArgs& P, int i) { return P.np3 ? (i == 2 ? 0 : i + 1) : (i ^ 1); }

// slice_map for a slice whose segment g is already known (the batched loops know it from the active-run
// table): no 64-bit division by the slices per segment on the path to the slice's loads
__device__ __forceinline__ void slice_map_g(const PcgArgs& P, int64_t s, int g, int64_t& row0, int64_t& end) {
  if (P.reg_units > 0) {
    row0 = (int64_t)g * P.reg_units + 32 * (s - (int64_t)g * P.spg);
    end = (int64_t)(g + 1) * P.reg_units;
  } else {
    row0 = P.A.slice_row0[s];
    end = P.A.seg_unit0[g + 1];
  }
}

// One row of a slice times an operand y(c).  WM > 0: slice width bound known at compile time; the
// loop is fully unrolled so all value loads and gathers issue together (stencil: columns are
// u + off[k], no column loads at all).  Returns the fma chain; *own = y at the diagonal slot when
// ST (the own p value comes from the diagonal gather).
// symmetric stencil storage: value of slot k of row u (ST == 2).  Upper slots (k >= kd) are stored with the
// row; a lower slot is the mirror a_vu of row v = u + off[k], read from v's upper slot mir[k] (an L2 hit:
// that row's values were streamed by a neighbouring warp moments earlier).
__device__ __forceinline__ double sym_val(const SellView& A, const double* __restrict__ vp, int k, int ui) {
  if (k >= A.kd) return __ldg(vp + 32 * (k - A.kd));
  const int v = ui + A.off[k];
  if (v < 0) return 0.0;
  int sv, lv;
  if (A.ru >= A.nunits) { sv = v >> 5; lv = v & 31; }
  else { const int g = v / A.ru, r = v - g * A.ru; sv = g * A.spg + (r >> 5); lv = r & 31; }
  return __ldg(A.val + 32ll * A.vw * sv + 32 * A.mir[k] + lv);
}

template <int WM, int ST, class Ld>
__device__ __forceinline__ double row_dot(const SellView& A, int64_t pl, int w, int64_t u, Ld ld, double* own,
                                          unsigned long long pol) {
  double acc = 0.0;
  const double* vp = A.val + pl;
  if (WM > 0) {
    constexpr int WA = WM > 0 ? WM : 1;
    double v[WA], y[WA];
    const int nu1 = (int)A.nunits - 1;   // n < 2^31 (checked in lc_create_csr): 32-bit index math
    const int ui = (int)u;
#pragma unroll
    for (int k = 0; k < WM; ++k) {
      int c;
      if (ST) {
        c = ui + A.off[k];
        c = c < 0 ? 0 : (c > nu1 ? nu1 : c);
      } else {
        c = (k < w) ? __ldg(A.col + pl + 32 * k) : 0;
      }
      v[k] = ST == 2 ? sym_val(A, vp, k, ui) : (ST || k < w) ? ldg_pol(vp + 32 * k, pol) : 0.0;
      y[k] = (ST || k < w) ? ld(c) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < WM; ++k)
      if (ST || k < w) acc = __fma_rn(v[k], y[k], acc);
    if (ST) {
#pragma unroll
      for (int k = 0; k < WM; ++k)
        if (A.off[k] == 0) *own = y[k];
    }
  } else {
    for (int k = 0; k < w; ++k) {
      int c = (int)sv_col(A, pl, k, u);
      double yk = ld(c);
      if (ST && c == u) *own = yk;
      acc = __fma_rn(ST == 2 ? sym_val(A, vp, k, (int)u) : __ldg(vp + 32 * k), yk, acc);
    }
  }
  return acc;
}

// Pass A slice loop for one mode (single segment: the mode is grid-uniform, so it is hoisted out of
// the loop and each mode gets a small loop body).  MODE 0: r = b - A x (INIT/CONFIRM, init adds b^T b);
// 1: FIRST (p = z); 2: NORMAL (p = z + beta p_old on the fly).
template <int WM, int ST, int MODE>
__device__ __forceinline__ void pass_a_loop(const PcgArgs& P, int64_t j0, int64_t jlim, int64_t jstep, int lane,
                                            bool init, double beta, const double* __restrict__ pold,
                                            double* __restrict__ pnew, double& a0, double& a1, int gk = -1,
                                            const double* __restrict__ xp = nullptr, double xa = 0.0,
                                            const double* __restrict__ xp2 = nullptr, double xa2 = 0.0) {
  const SellView& A = P.A;
  const unsigned long long strm = l2_stream_policy(P.stream_vals != 0);
  // (gk >= 0: every slice belongs to segment gk)
  // the slice list entry and the row's Omega flag are loaded one slice ahead (masked solves walk a list of
  // slices; without the prefetch every slice starts with two dependent load latencies)
  int64_t s_next = j0 < jlim ? (P.slist ? (int64_t)P.slist[j0] : j0) : 0;
  uint8_t om_next = 0;
  auto om_of = [&](int64_t s_) -> uint8_t {
    int g_;
    int64_t r0_, e_;
    if (gk >= 0) slice_map_g(P, s_, gk, r0_, e_);
    else slice_map(P, s_, g_, r0_, e_);
    return r0_ + lane < e_ ? P.omega[r0_ + lane] : (uint8_t)0;
  };
  if (P.omega && j0 < jlim) om_next = om_of(s_next);
  // SELL: the slice's first slot and width are loaded one slice ahead too (column loads then follow directly)
  int64_t sp_next = 0, se_next = 0;
  if (!ST && j0 < jlim) { sp_next = A.slice_ptr[s_next]; se_next = A.slice_ptr[s_next + 1]; }
#pragma unroll 1
  for (int64_t j = j0; j < jlim; j += jstep) {
    const int64_t s = s_next;
    const uint8_t om_cur = om_next;
    const int64_t sp_cur = sp_next, se_cur = se_next;
    if (j + jstep < jlim) {
      s_next = P.slist ? (int64_t)P.slist[j + jstep] : j + jstep;
      if (P.omega) om_next = om_of(s_next);
      if (!ST) { sp_next = A.slice_ptr[s_next]; se_next = A.slice_ptr[s_next + 1]; }
    }
    int g;
    int64_t row0, end;
    if (gk >= 0) slice_map_g(P, s, gk, row0, end);
    else slice_map(P, s, g, row0, end);
    const int64_t u = row0 + lane;
    if (u >= end) continue;
    const int64_t pl = (ST ? 32ll * A.vw * s : sp_cur) + lane;
    const int w = ST ? A.W : (int)((se_cur - sp_cur) >> 5);
    double own = 0.0;
    const bool in = !P.omega || om_cur != 255;
    if (MODE == 0) {
      const double* xx = P.x;
      double acc = xp ? row_dot<WM, ST>(A, pl, w, u, [&](int c) {
                          const double t = __fma_rn(xa, xp[c], xx[c]);
                          return xp2 ? __fma_rn(xa2, xp2[c], t) : t; }, &own, strm)
                      : row_dot<WM, ST>(A, pl, w, u, [&](int c) { return xx[c]; }, &own, strm);
      if (in) {
        double bi = P.b[u];
        double ri = bi - acc;
        P.r[u] = ri;
        a0 = __fma_rn(ri, ri, a0);
        if (init) a1 = __fma_rn(bi, bi, a1);
      }
    } else {
      const double* zz = P.z;
      double acc;
      if (MODE == 1) acc = row_dot<WM, ST>(A, pl, w, u, [&](int c) { return zz[c]; }, &own, strm);
      else acc = row_dot<WM, ST>(A, pl, w, u, [&](int c) { return __fma_rn(beta, pold[c], zz[c]); }, &own, strm);
      if (in) {
        double pi = ST ? own : (MODE == 1 ? zz[u] : __fma_rn(beta, pold[u], zz[u]));
        pnew[u] = pi;
        P.q[u] = acc;
        a0 = __fma_rn(pi, acc, a0);
      }
    }
  }
}

#ifdef LC_DEBUG_TIMELINE
__device__ unsigned long long g_tl[8192];
__device__ __forceinline__ void tl_mark(int& k) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && k < 8192) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tl[k] = t;
  }
  ++k;
}
#define TL(k) tl_mark(k)
// per-CTA pass timeline: [pass - g_cta_pass0][bid][0: pass start, 1: pass end, 2: reduction/barrier out]
__device__ unsigned long long g_cta[64][1024][3];
__device__ int g_cta_pass0;
__device__ __forceinline__ void cta_mark(int pc, int slot) {
  const int k = pc - g_cta_pass0;
  if (threadIdx.x == 0 && k >= 0 && k < 64 && blockIdx.x < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_cta[k][blockIdx.x][slot] = t;
  }
}
#define CT(pc, slot) cta_mark(pc, slot)
#else
#define TL(k) (void)0
#define CT(pc, slot) (void)0
#endif
#ifndef LCV_MINB
#define LCV_MINB (1024 / LC_PCG_PT)
#endif
#ifndef LCV_MINB_SELL
#define LCV_MINB_SELL LCV_MINB
#endif
// Pass A with the value stream staged by TMA (single segment, stencil layouts, no slice list): CTA b owns
// the chunks c = b + t nCTA of 8 consecutive slices (exactly the slices its 8 warps take in the
// interleaved order); thread 0 keeps kStages chunks in flight with cp.async.bulk into a shared-memory
// ring (mbarrier complete_tx), the warps read their slice's values from shared memory, so the DRAM
// stream no longer waits on each warp's gather latency.  Gathers and the symmetric mirrors stay loads.
#ifndef LC_PCG_STAGES
#define LC_PCG_STAGES 2
#endif
constexpr int kStages = LC_PCG_STAGES;
template <int WM, int ST, int MODE>
__device__ __forceinline__ void pass_a_tma(const PcgArgs& P, double* stg, uint64_t* bars, int64_t bid, int64_t nCTA,
                                           int warp, int lane, bool init, double beta,
                                           const double* __restrict__ pold, double* __restrict__ pnew, double& a0,
                                           double& a1, const double* __restrict__ xp = nullptr, double xa = 0.0,
                                           const double* __restrict__ xp2 = nullptr, double xa2 = 0.0) {
  const SellView& A = P.A;
  constexpr int W = WM > 0 ? WM : 1;
  const int vw = A.vw;
  const int64_t njs = P.slist ? *P.nlist : A.nslices;          // index space: listed or all slices
  const int64_t nch = (njs + kPW - 1) / kPW;
  const int64_t chd = (int64_t)kPW * 32 * vw;                    // doubles per chunk
  // uniform-width SELL (ST == 0, the explicit subsystems): the chunk's int32 columns are staged after the values
  int32_t* const scol = reinterpret_cast<int32_t*>(stg + kStages * chd);
  const int n = (int)A.nunits, nu1 = n - 1;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kStages; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const unsigned long long pol = l2_stream_policy(P.stream_vals != 0);
  auto issue = [&](int64_t t) {
    const int64_t c = bid + t * nCTA;
    if (c >= nch) return;
    const int st = (int)(t % kStages);
    const int64_t j0c = (int64_t)kPW * c;
    const int nsl = (int)((njs - j0c) < kPW ? (njs - j0c) : kPW);
    const unsigned sbytes = (unsigned)(32 * vw * 8);
    if (!P.slist) {                                              // 8 consecutive slices: one copy
      mbar_expect_tx(&bars[st], sbytes * nsl * (ST == 0 ? 3 : 2) / 2);
      tma_bulk_g2s_pol(stg + st * chd, A.val + j0c * 32 * vw, sbytes * nsl, &bars[st], pol);
      if (ST == 0) tma_bulk_g2s_pol(scol + st * chd, A.col + j0c * 32 * vw, sbytes * nsl / 2, &bars[st], pol);
    } else {                                                     // listed slices: one copy each
      mbar_expect_tx(&bars[st], sbytes * nsl);
      for (int w = 0; w < nsl; ++w)
        tma_bulk_g2s(stg + st * chd + (int64_t)w * 32 * vw, A.val + (int64_t)P.slist[j0c + w] * 32 * vw, sbytes,
                     &bars[st]);
    }
  };
  if (threadIdx.x == 0)
    for (int t = 0; t < kStages; ++t) issue(t);
  // masked solves: the Omega flag of the row is loaded one chunk ahead, so no row waits on its flag load
  auto om_at = [&](int64_t c) -> uint8_t {
    const int64_t js = (int64_t)kPW * c + warp;
    const int64_t u = 32 * (P.slist ? (js < njs ? (int64_t)P.slist[js] : 0) : js) + lane;
    return (c < nch && js < njs && u < n) ? P.omega[u] : (uint8_t)0;
  };
  uint8_t om_next = P.omega ? om_at(bid) : (uint8_t)0;
#pragma unroll 1
  for (int64_t t = 0;; ++t) {
    const int64_t c = bid + t * nCTA;
    if (c >= nch) break;
    const uint8_t om_cur = om_next;
    if (P.omega) om_next = om_at(c + nCTA);
    const int st = (int)(t % kStages);
    mbar_wait(&bars[st], (unsigned)((t / kStages) & 1));
    const int64_t js = (int64_t)kPW * c + warp;
    const int64_t s = js < njs ? (P.slist ? (int64_t)P.slist[js] : js) : 0;
    const int u = (int)(32 * s) + lane;
    if (js < njs && u < n) {
      const bool in = !P.omega || om_cur != 255;
      const double* sp = stg + st * chd + (int64_t)warp * 32 * vw + lane;
      const int32_t* scp = scol + st * chd + (int64_t)warp * 32 * vw + lane;
      double v[W], y[W];
#pragma unroll
      for (int k = 0; k < W; ++k) {
        int cc;
        if (ST == 0) cc = scp[32 * k];
        else {
          cc = u + A.off[k];
          cc = cc < 0 ? 0 : (cc > nu1 ? nu1 : cc);
        }
        if (ST == 2) {
          if (k >= A.kd) v[k] = sp[32 * (k - A.kd)];
          else {
            const int vr = u + A.off[k];
            v[k] = vr < 0 ? 0.0 : __ldg(A.val + 32ll * vw * (vr >> 5) + 32 * A.mir[k] + (vr & 31));
          }
        } else {
          v[k] = sp[32 * k];
        }
        if (MODE == 0) {                                            // (x with its pending updates)
          y[k] = P.x[cc];
          if (xp) y[k] = __fma_rn(xa, xp[cc], y[k]);
          if (xp2) y[k] = __fma_rn(xa2, xp2[cc], y[k]);
        }
        else if (MODE == 1) y[k] = P.z[cc];
        else y[k] = __fma_rn(beta, pold[cc], P.z[cc]);
      }
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < W; ++k) acc = __fma_rn(v[k], y[k], acc);
      if (MODE == 0) {
        if (in) {
          const double bi = P.b[u];
          const double ri = bi - acc;
          P.r[u] = ri;
          a0 = __fma_rn(ri, ri, a0);
          if (init) a1 = __fma_rn(bi, bi, a1);
        }
      } else if (in) {
        double pi = 0.0;
        if (ST == 0) pi = MODE == 1 ? P.z[u] : __fma_rn(beta, pold[u], P.z[u]);
        else {
#pragma unroll
          for (int k = 0; k < W; ++k)
            if (A.off[k] == 0) pi = y[k];
        }
        pnew[u] = pi;
        P.q[u] = acc;
        a0 = __fma_rn(pi, acc, a0);
      }
    }
    __syncthreads();                               // every warp is done with stage st
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();                    // generic reads of st before the async-proxy refill
      issue(t + kStages);
    }
  }
}

// KIND: 0 = one segment (G = 1), 1 = batched lock step (G > 1), 2 = batched teams (each team a G = 1 solve)
template <int WM, int ST, int KIND>
__global__ void __launch_bounds__(kPT, ST == 0 ? LCV_MINB_SELL : LCV_MINB) k_pcg(PcgArgs P) {
  unsigned long long bar_epoch = 0;
  const unsigned long long strm = l2_stream_policy(P.stream_vals != 0);   // the matrix stream's L2 policy word
  unsigned tree_gen = 0;                        // tree barriers passed (G > 1)
  __shared__ SegState S[kMaxSeg];
  __shared__ double s_acc[kPW][kMaxSeg][2];
  __shared__ double s_red[kPW][2];
  __shared__ double s_sum[kMaxSeg][2];
  __shared__ long long s_segj0[kMaxSeg + 1];   // segment runs in slice space
  __shared__ int s_act[kMaxSeg + 1];           // active segments of the current pass (+ sentinel)
  __shared__ long long s_actj[kMaxSeg + 1];    // their runs concatenated
  __shared__ double s_cpart[2][2];             // cluster mode: this CTA's partials, double-buffered by pass
  // batched solves launched in clusters (P.clus): the CTA's partials for the cluster reduction, and its scratch
  __shared__ double s_mine[KIND == 1 ? 2 * kMaxSeg : 1];
  __shared__ double s_chunk[KIND == 1 ? kPT : 1];
  unsigned long long ctr_target = 0;
  int cpar = 0;
  extern __shared__ __align__(128) double dsm[];   // TMA stages (P.tma): kStages x 8 slices x 32 x vw values
  __shared__ __align__(8) uint64_t s_bars[kStages];
  const SellView& A = P.A;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nCTA = gridDim.x, bid = blockIdx.x;
  // team mode: CTAs [tb0, tb1) form team `team`; every pass below runs over the team's current segment only
  constexpr bool TEAM = KIND == 2;
  const int TM = TEAM ? P.teams : 0;           // compile-time 0 in the single-grid kernels
  int team = 0;
  const int TD = TM > 0 ? TM : 1;
  if (TM)
    while (team < TM - 1 && bid >= (int64_t)(team + 1) * nCTA / TD) ++team;
  const int64_t tb0 = TM ? (int64_t)team * nCTA / TD : 0;
  const int64_t tn = TM ? (int64_t)(team + 1) * nCTA / TD - tb0 : nCTA;
  const int G = KIND == 1 ? P.G : 1;            // compile-time 1 except in the lock-step kernels
  int gseg = TM ? team : 0;                     // segment being solved (team mode)
  int64_t j0 = (bid - tb0) * kPW + warp;
  const int64_t jstep = tn * kPW;
  int64_t jlim = P.slist ? *P.nlist : A.nslices;
  for (int g = threadIdx.x; g <= P.G; g += kPT) s_segj0[g] = P.seg_j0[g];
  if (threadIdx.x < kMaxSeg) {
    S[threadIdx.x].mode = M_INIT; S[threadIdx.x].par = 0; S[threadIdx.x].it = 0; S[threadIdx.x].final_ = 0;
    S[threadIdx.x].beta = 0.0; S[threadIdx.x].alpha = 0.0; S[threadIdx.x].rho = 0.0;
    S[threadIdx.x].pend = 0; S[threadIdx.x].pbuf = 0; S[threadIdx.x].palpha = 0.0; S[threadIdx.x].npass = 0;
    S[threadIdx.x].pbuf2 = 0; S[threadIdx.x].palpha2 = 0.0;
  }
  __syncthreads();

  auto clear_acc = [&]() {
    for (int t = threadIdx.x; t < kPW * G * 2; t += kPT) {
      int w = t / (G * 2), rest = t % (G * 2);
      s_acc[w][rest >> 1][rest & 1] = 0.0;
    }
    __syncthreads();
  };
  auto flush = [&](int g, double a0, double a1) {
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    if (lane == 0) { s_acc[warp][g][0] += a0; s_acc[warp][g][1] += a1; }
  };
  // per-CTA partials -> part[bid][g][j]; then every CTA obtains s_sum[g][j] for all g (fixed order)
  auto reduce_all = [&]() {
    __syncthreads();
    if (KIND == 0 && P.cluster) {
      // one cluster (G = 1): partials stay in shared memory and are read across the cluster (DSMEM)
      cg::cluster_group cl = cg::this_cluster();
      if (threadIdx.x < 2) {
        double v = 0.0;
        for (int w = 0; w < kPW; ++w) v += s_acc[w][0][threadIdx.x];
        s_cpart[cpar][threadIdx.x] = v;
      }
      cl.sync();
      if (threadIdx.x < 2) {
        double o = 0.0;
        for (int r = 0; r < (int)nCTA; ++r) o += cl.map_shared_rank(&s_cpart[cpar][0], r)[threadIdx.x];
        s_sum[0][threadIdx.x] = o;
      }
      cpar ^= 1;
      __syncthreads();
      return;
    }
    // G = 1: the partials are double-buffered by pass, since a CTA that leaves the barrier early may finish its
    // next pass and store its next partial before a slower CTA has read this one (short passes)
    double* const pt = P.part + (G == 1 ? (size_t)cpar * 2 * nCTA : 0);
    if (KIND == 1 && P.clus) {
      // batched, launched in clusters: the CTA's partials stay in shared memory for the cluster reduction
      for (int t = threadIdx.x; t < G * 2; t += kPT) {
        double v = 0.0;
        for (int w = 0; w < kPW; ++w) v += s_acc[w][t >> 1][t & 1];
        s_mine[t] = v;
      }
      cluster_reduce_barrier<kPT, 2 * kMaxSeg>(P.bar, P.part, s_mine, &s_sum[0][0], 2 * G, s_chunk, ctr_target,
                                               tree_gen);
      return;
    }
    for (int t = threadIdx.x; t < G * 2; t += kPT) {
      double v = 0.0;
      for (int w = 0; w < kPW; ++w) v += s_acc[w][t >> 1][t & 1];
      pt[(bid * G) * 2 + t] = v;
    }
    if (G == 1) {
      cpar ^= 1;
      if (TM) team_barrier(P.tctr + 16 * team, bar_epoch, (unsigned)tn);
      else grid_barrier(P.bar, bar_epoch);
      double a0 = 0.0, a1 = 0.0;
      for (int64_t c = tb0 + threadIdx.x; c < tb0 + tn; c += kPT) { a0 += pt[2 * c]; a1 += pt[2 * c + 1]; }
      a0 = warp_sum(a0); a1 = warp_sum(a1);
      if (lane == 0) { s_red[warp][0] = a0; s_red[warp][1] = a1; }
      __syncthreads();
#if LCV_RED_ALL
      {
        double o0 = 0.0, o1 = 0.0;
        for (int w = 0; w < kPW; ++w) { o0 += s_red[w][0]; o1 += s_red[w][1]; }
        if (threadIdx.x == 0) { s_sum[0][0] = o0; s_sum[0][1] = o1; }
      }
#else
      if (threadIdx.x < 2) {
        double o = 0.0;
        for (int w = 0; w < kPW; ++w) o += s_red[w][threadIdx.x];
        s_sum[0][threadIdx.x] = o;
      }
#endif
    } else {
      tree_reduce_barrier<kPW, 2 * kMaxSeg>(P.bar, P.part, P.subred, &s_sum[0][0], 2 * G,
                                            reinterpret_cast<double (*)[2 * kMaxSeg]>(&s_acc[0][0][0]), tree_gen);
    }
    __syncthreads();
  };
  auto finish = [&](int g, int status, double rn) {
    SegState& T = S[g];
    T.mode = M_DONE;
    const int go = TM ? gseg : g;
    if (bid == (TM ? tb0 : g % nCTA)) {
      P.out_iters[go] = T.it;
      P.out_status[go] = status;
      P.out_relres[go] = T.nb > 0 ? rn / T.nb : rn;
    }
  };
  auto in_omega = [&](int64_t u) -> bool { return !P.omega || P.omega[u] != 255; };
  // G > 1: the slice space of a pass = the runs of the segments active in that pass, concatenated, so all
  // warps share the remaining groups' work once others have converged.  Returns the total length.
  auto build_active = [&](int pass) -> int64_t {
    if (threadIdx.x == 0) {
      long long J = 0;
      int na = 0;
      for (int g = 0; g < G; ++g) {
        int md = S[g].mode;
        bool act = pass == 0 ? (md == M_INIT || md == M_CONFIRM || md == M_FIRST || md == M_NORMAL)
                             : (md == M_UPDATE || md == M_RESET);
        if (act) { s_act[na] = g; s_actj[na] = J; J += s_segj0[g + 1] - s_segj0[g]; ++na; }
      }
      s_actj[na] = J;
      s_act[na] = G;
    }
    __syncthreads();
    int na = 0;
    while (s_act[na] != G) ++na;
    return s_actj[na];
  };

#ifdef LC_DEBUG_TIMELINE
  int tlk = 0;
#endif
  int pc = 0;                                   // pass counter (debug timeline)
  (void)pc;
  for (; gseg < (TM ? P.G : 1); gseg += (TM ? TM : 1)) {
  if (TM) {                                     // next segment of this team: a fresh G = 1 solve on its run
    __syncthreads();
    j0 = s_segj0[gseg] + (bid - tb0) * kPW + warp;
    jlim = s_segj0[gseg + 1];
    if (threadIdx.x == 0) {
      S[0].mode = M_INIT; S[0].par = 0; S[0].it = 0; S[0].final_ = 0;
      S[0].beta = 0.0; S[0].alpha = 0.0; S[0].rho = 0.0;
      S[0].pend = 0; S[0].pbuf = 0; S[0].palpha = 0.0; S[0].pbuf2 = 0; S[0].palpha2 = 0.0;
    }
    __syncthreads();
  }
  for (;;) {
    // ------------------------------------------------------------ pass A ----
    TL(tlk);
    CT(pc, 0);
    clear_acc();
    if (G == 1) {
      const int mode = S[0].mode;
      double a0 = 0.0, a1 = 0.0;
      const double beta = S[0].beta;
      const double* pold = pvec(P, S[0].par);
      double* pnew = pvec(P, pnext(P, S[0].par));
      // lazy x: a CONFIRM pass gathers x with its pending updates (x itself is completed by the next pass B)
      const double* xp = (KIND == 0 && S[0].pend >= 1) ? pvec(P, S[0].pbuf) : nullptr;
      const double* xp2 = (KIND == 0 && S[0].pend >= 2) ? pvec(P, S[0].pbuf2) : nullptr;
      const double xa = S[0].palpha, xa2 = S[0].palpha2;
      if (KIND == 0 && WM > 0 && P.tma) {
        if (mode == M_INIT || mode == M_CONFIRM)
          pass_a_tma<WM, ST, 0>(P, dsm, s_bars, bid, nCTA, warp, lane, mode == M_INIT, beta, pold, pnew, a0, a1, xp,
                                xa, xp2, xa2);
        else if (mode == M_FIRST)
          pass_a_tma<WM, ST, 1>(P, dsm, s_bars, bid, nCTA, warp, lane, false, beta, pold, pnew, a0, a1);
        else if (mode == M_NORMAL)
          pass_a_tma<WM, ST, 2>(P, dsm, s_bars, bid, nCTA, warp, lane, false, beta, pold, pnew, a0, a1);
      } else if (mode == M_INIT || mode == M_CONFIRM)
        pass_a_loop<WM, ST, 0>(P, j0, jlim, jstep, lane, mode == M_INIT, beta, pold, pnew, a0, a1, TEAM ? gseg : -1,
                               xp, xa, xp2, xa2);
      else if (mode == M_FIRST)
        pass_a_loop<WM, ST, 1>(P, j0, jlim, jstep, lane, false, beta, pold, pnew, a0, a1, TEAM ? gseg : -1);
      else if (mode == M_NORMAL)
        pass_a_loop<WM, ST, 2>(P, j0, jlim, jstep, lane, false, beta, pold, pnew, a0, a1, TEAM ? gseg : -1);
      flush(0, a0, a1);
    } else {
      const int64_t J = build_active(0);
      int gcur = -1, mode = M_DONE, ka = 0;
      double a0 = 0.0, a1 = 0.0, beta = 0.0;
      const double* pold = nullptr;
      double* pnew = nullptr;
      for (int64_t j = j0; j < J; j += jstep) {
        while (s_actj[ka + 1] <= j) ++ka;
        const int g = s_act[ka];
        const int64_t jj = s_segj0[g] + (j - s_actj[ka]);
        const int64_t s = P.slist ? (int64_t)P.slist[jj] : jj;
        int64_t row0, end;
        slice_map_g(P, s, g, row0, end);
        if (g != gcur) {
          if (gcur >= 0) flush(gcur, a0, a1);
          a0 = a1 = 0.0;
          gcur = g;
          mode = S[g].mode;
          beta = S[g].beta;
          pold = S[g].par ? P.p1 : P.p0;
          pnew = S[g].par ? P.p0 : P.p1;
        }
        if (mode == M_DONE || mode == M_RESET) continue;
        const int64_t u = row0 + lane;
        if (u >= end) continue;
        const int64_t pl = (ST ? 32ll * A.vw * s : A.slice_ptr[s]) + lane;
        const int w = ST ? A.W : (int)((A.slice_ptr[s + 1] - (pl - lane)) >> 5);
        double own = 0.0;
        if (mode == M_INIT || mode == M_CONFIRM) {
          const double* xx = P.x;
          double acc = row_dot<WM, ST>(A, pl, w, u, [&](int c) { return xx[c]; }, &own, strm);
          if (in_omega(u)) {
            double bi = P.b[u];
            double ri = bi - acc;
            P.r[u] = ri;
            a0 = __fma_rn(ri, ri, a0);
            if (mode == M_INIT) a1 = __fma_rn(bi, bi, a1);
          }
        } else {
          const double* zz = P.z;
          double acc;
          if (mode == M_FIRST) acc = row_dot<WM, ST>(A, pl, w, u, [&](int c) { return zz[c]; }, &own, strm);
          else acc = row_dot<WM, ST>(A, pl, w, u, [&](int c) { return __fma_rn(beta, pold[c], zz[c]); }, &own, strm);
          if (in_omega(u)) {
            double pi = ST ? own : (mode == M_FIRST ? zz[u] : __fma_rn(beta, pold[u], zz[u]));
            pnew[u] = pi;
            P.q[u] = acc;
            a0 = __fma_rn(pi, acc, a0);
          }
        }
      }
      if (gcur >= 0) flush(gcur, a0, a1);
    }
    TL(tlk);
    CT(pc, 1);
    reduce_all();
    CT(pc, 2);
    ++pc;
    TL(tlk);
    // ---------------------------------------------------- pass A scalars ----
    // segments are independent: thread g updates segment g's state
    for (int g = threadIdx.x; g < G; g += kPT) {
      SegState& T = S[g];
      double s0 = s_sum[g][0], s1 = s_sum[g][1];
      if (T.mode == M_INIT) {
        T.nb = sqrt(s1);
        T.tgt = T.nb > 0 ? P.eps * T.nb : P.eps;
        double rn = sqrt(s0);
        if (!isfinite(rn)) finish(g, LC_ERR_NONFINITE, rn);
        else if (rn <= T.tgt) finish(g, LC_OK, rn);
        else if (P.max_iters == 0) finish(g, LC_NOT_CONVERGED, rn);   // Eq. 6 check only
        else T.mode = M_RESET;
      } else if (T.mode == M_FIRST || T.mode == M_NORMAL) {
        double pq = s0;
        if (!(pq > 0)) finish(g, isfinite(pq) ? LC_ERR_BREAKDOWN : LC_ERR_NONFINITE, NAN);
        else { T.alpha = T.rho / pq; T.mode = M_UPDATE; T.par = pnext(P, T.par); }
      } else if (T.mode == M_CONFIRM) {
        double rn = sqrt(s0);
        if (!isfinite(rn)) finish(g, LC_ERR_NONFINITE, rn);
        else if (rn <= T.tgt) finish(g, LC_OK, rn);
        else if (T.final_) finish(g, LC_NOT_CONVERGED, rn);
        else T.mode = M_RESET;
      }
    }
    __syncthreads();
    // ------------------------------------------------------------ pass B ----
    TL(tlk);
    CT(pc, 0);
    clear_acc();
    if (KIND == 0 && P.vec2) {
      // single segment over all rows: flat grid-stride over row pairs with 16-byte loads/stores
      const int mode = S[0].mode;
      double a0 = 0.0, a1 = 0.0;
      if (mode == M_UPDATE || mode == M_RESET) {
        const double alpha = S[0].alpha;
        const double2* pp = reinterpret_cast<const double2*>(pvec(P, S[0].par));
        double2* x2 = reinterpret_cast<double2*>(P.x);
        double2* r2 = reinterpret_cast<double2*>(P.r);
        double2* z2 = reinterpret_cast<double2*>(P.z);
        const double2* q2 = reinterpret_cast<const double2*>(P.q);
        const double2* d2 = reinterpret_cast<const double2*>(A.dinv);
        const int64_t n = A.nunits, npair = n >> 1;
        const int64_t gt = bid * kPT + threadIdx.x, gs = nCTA * kPT;
        // lazy x (depth L = P.lazyx): L - 1 UPDATE passes leave x alone (r, z only: 40 instead of 64 B per row;
        // x lacks the pending alpha_i p_i), the L-th applies them all in order, x = fma(alpha_k, p_k, fma(...,
        // fma(alpha_k-L+1, p_k-L+1, x))): the same roundings as updating every pass.  p_k-L+1 .. p_k survive until
        // then (L = 3 rotates p over three buffers).  A RESET applies the pending updates, and so does the exit.
        const int pend = S[0].pend;
        const double pa = S[0].palpha, pa2 = S[0].palpha2;
        const double2* t1 = reinterpret_cast<const double2*>(pvec(P, S[0].pbuf));
        const double2* t2 = reinterpret_cast<const double2*>(pvec(P, S[0].pbuf2));
        if (mode == M_UPDATE && P.lazyx && pend < P.lazyx - 1) {
#pragma unroll 2
          for (int64_t i = gt; i < npair; i += gs) {
            double2 rv = r2[i], qv = q2[i], dv = d2[i];
            rv.x = __fma_rn(-alpha, qv.x, rv.x); rv.y = __fma_rn(-alpha, qv.y, rv.y);
            double2 zv = make_double2(rv.x * dv.x, rv.y * dv.y);
            r2[i] = rv; z2[i] = zv;
            a0 = __fma_rn(rv.x, zv.x, a0); a0 = __fma_rn(rv.y, zv.y, a0);
            a1 = __fma_rn(rv.x, rv.x, a1); a1 = __fma_rn(rv.y, rv.y, a1);
          }
          if ((n & 1) && gt == 0) {
            int64_t u = n - 1;
            double ri = __fma_rn(-alpha, P.q[u], P.r[u]);
            double zi = ri * A.dinv[u];
            P.r[u] = ri; P.z[u] = zi;
            a0 = __fma_rn(ri, zi, a0); a1 = __fma_rn(ri, ri, a1);
          }
        } else if (mode == M_UPDATE && pend == 2) {
#pragma unroll 2
          for (int64_t i = gt; i < npair; i += gs) {
            double2 xv = x2[i], ov = t1[i], ov2 = t2[i], pv = pp[i], rv = r2[i], qv = q2[i], dv = d2[i];
            xv.x = __fma_rn(alpha, pv.x, __fma_rn(pa2, ov2.x, __fma_rn(pa, ov.x, xv.x)));
            xv.y = __fma_rn(alpha, pv.y, __fma_rn(pa2, ov2.y, __fma_rn(pa, ov.y, xv.y)));
            rv.x = __fma_rn(-alpha, qv.x, rv.x); rv.y = __fma_rn(-alpha, qv.y, rv.y);
            double2 zv = make_double2(rv.x * dv.x, rv.y * dv.y);
            x2[i] = xv; r2[i] = rv; z2[i] = zv;
            a0 = __fma_rn(rv.x, zv.x, a0); a0 = __fma_rn(rv.y, zv.y, a0);
            a1 = __fma_rn(rv.x, rv.x, a1); a1 = __fma_rn(rv.y, rv.y, a1);
          }
          if ((n & 1) && gt == 0) {
            int64_t u = n - 1;
            double xi = __fma_rn(alpha, pvec(P, S[0].par)[u],
                                 __fma_rn(pa2, pvec(P, S[0].pbuf2)[u], __fma_rn(pa, pvec(P, S[0].pbuf)[u], P.x[u])));
            double ri = __fma_rn(-alpha, P.q[u], P.r[u]);
            double zi = ri * A.dinv[u];
            P.x[u] = xi; P.r[u] = ri; P.z[u] = zi;
            a0 = __fma_rn(ri, zi, a0); a1 = __fma_rn(ri, ri, a1);
          }
        } else if (mode == M_UPDATE && pend == 1) {
#pragma unroll 2
          for (int64_t i = gt; i < npair; i += gs) {
            double2 xv = x2[i], ov = t1[i], pv = pp[i], rv = r2[i], qv = q2[i], dv = d2[i];
            xv.x = __fma_rn(alpha, pv.x, __fma_rn(pa, ov.x, xv.x)); xv.y = __fma_rn(alpha, pv.y, __fma_rn(pa, ov.y, xv.y));
            rv.x = __fma_rn(-alpha, qv.x, rv.x); rv.y = __fma_rn(-alpha, qv.y, rv.y);
            double2 zv = make_double2(rv.x * dv.x, rv.y * dv.y);
            x2[i] = xv; r2[i] = rv; z2[i] = zv;
            a0 = __fma_rn(rv.x, zv.x, a0); a0 = __fma_rn(rv.y, zv.y, a0);
            a1 = __fma_rn(rv.x, rv.x, a1); a1 = __fma_rn(rv.y, rv.y, a1);
          }
          if ((n & 1) && gt == 0) {
            int64_t u = n - 1;
            double xi = __fma_rn(alpha, pvec(P, S[0].par)[u], __fma_rn(pa, pvec(P, S[0].pbuf)[u], P.x[u]));
            double ri = __fma_rn(-alpha, P.q[u], P.r[u]);
            double zi = ri * A.dinv[u];
            P.x[u] = xi; P.r[u] = ri; P.z[u] = zi;
            a0 = __fma_rn(ri, zi, a0); a1 = __fma_rn(ri, ri, a1);
          }
        } else if (mode == M_UPDATE) {
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
            int64_t u = n - 1;
            double xi = __fma_rn(alpha, pvec(P, S[0].par)[u], P.x[u]);
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
            if (pend) {
              double2 xv = x2[i], ov = t1[i];
              xv.x = __fma_rn(pa, ov.x, xv.x); xv.y = __fma_rn(pa, ov.y, xv.y);
              if (pend == 2) {
                const double2 ov2 = t2[i];
                xv.x = __fma_rn(pa2, ov2.x, xv.x); xv.y = __fma_rn(pa2, ov2.y, xv.y);
              }
              x2[i] = xv;
            }
          }
          if ((n & 1) && gt == 0) {
            int64_t u = n - 1;
            double zi = P.r[u] * A.dinv[u];
            P.z[u] = zi;
            a0 = __fma_rn(P.r[u], zi, a0);
            if (pend) {
              double xi = __fma_rn(pa, pvec(P, S[0].pbuf)[u], P.x[u]);
              if (pend == 2) xi = __fma_rn(pa2, pvec(P, S[0].pbuf2)[u], xi);
              P.x[u] = xi;
            }
          }
        }
      }
      flush(0, a0, a1);
    } else {
      const int64_t J = G == 1 ? jlim : build_active(1);
      int gcur = -1, mode = M_DONE, ka = 0;
      double a0 = 0.0, a1 = 0.0, alpha = 0.0;
      const double* pp = nullptr;
      for (int64_t j = j0; j < J; j += jstep) {
        int64_t s;
        int g;
        int64_t row0, end;
        if (G == 1) {
          s = P.slist ? (int64_t)P.slist[j] : j;
          if (TEAM) slice_map_g(P, s, gseg, row0, end);
          else slice_map(P, s, g, row0, end);
          g = 0;                                  // (a team's current segment lives in S[0])
        } else {
          while (s_actj[ka + 1] <= j) ++ka;
          g = s_act[ka];
          const int64_t jj = s_segj0[g] + (j - s_actj[ka]);
          s = P.slist ? (int64_t)P.slist[jj] : jj;
          slice_map_g(P, s, g, row0, end);
        }
        if (g != gcur) {
          if (gcur >= 0) flush(gcur, a0, a1);
          a0 = a1 = 0.0;
          gcur = g;
          mode = S[g].mode;
          alpha = S[g].alpha;
          pp = S[g].par ? P.p1 : P.p0;
        }
        if (mode != M_UPDATE && mode != M_RESET) continue;
        const int64_t u = row0 + lane;
        if (u >= end) continue;
        // rows outside Omega (masked solves) hold p = q = r = 0, so the update leaves them 0
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
      if (gcur >= 0) flush(gcur, a0, a1);
    }
    TL(tlk);
    CT(pc, 1);
    reduce_all();
    CT(pc, 2);
    ++pc;
    TL(tlk);
    // ---------------------------------------------------- pass B scalars ----
    int active = 0;
    for (int g = threadIdx.x; g < G; g += kPT) {
      SegState& T = S[g];
      double s0 = s_sum[g][0], s1 = s_sum[g][1];
      if (T.mode == M_UPDATE) {
        T.it += 1;
        if (KIND == 0 && P.lazyx) {               // the update just done left alpha p pending / applied both
          if (T.pend == P.lazyx - 1) T.pend = 0;
          else if (T.pend == 0) { T.pend = 1; T.pbuf = T.par; T.palpha = T.alpha; }
          else { T.pend = 2; T.pbuf2 = T.par; T.palpha2 = T.alpha; }
        }
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
        T.pend = 0;                               // (the RESET pass applied a pending x update)
      }
      active += (T.mode != M_DONE);
    }
    if (!__syncthreads_or(active)) break;
  }
  if (KIND == 0 && S[0].pend) {
    // lazy x: the last update is still pending (the solve ended after a CONFIRM or a breakdown); apply it and
    // do a8 in the same loop (every row is completed and scattered by the same thread)
    const double* po = pvec(P, S[0].pbuf);
    const double* po2 = pvec(P, S[0].pbuf2);
    const double pa = S[0].palpha, pa2 = S[0].palpha2;
    const bool two = S[0].pend == 2;
    for (int64_t u = bid * kPT + threadIdx.x; u < A.nunits; u += nCTA * kPT) {
      double xi = __fma_rn(pa, po[u], P.x[u]);
      if (two) xi = __fma_rn(pa2, po2[u], xi);
      P.x[u] = xi;
      if (P.scatter_idx) P.x_full[P.scatter_idx[u]] = xi;
      else if (P.x_user && in_omega(u)) P.x_user[u] = xi;
    }
  } else
  // a8: x~[Omega] = xbar_B (Eq. 4), fused into the local solve's exit
  if (P.scatter_idx || P.x_user) {
    for (int64_t j = j0; j < jlim; j += jstep) {
      const int64_t s = P.slist ? (int64_t)P.slist[j] : j;
      int g;
      int64_t row0, end;
      slice_map(P, s, g, row0, end);
      const int64_t u = row0 + lane;
      if (u >= end) continue;
      if (P.scatter_idx) P.x_full[P.scatter_idx[u]] = P.x[u];
      else if (in_omega(u)) P.x_user[u] = P.x[u];
    }
  }
  }                                             // segments of the team
  if (KIND == 1 && P.clus) cg::this_cluster().sync();   // no CTA exits while its rank 0 may read its partials
}

// ------------------------------------------------ batched: dynamic teams ----
// Batched global solves (G > 1 equal segments, no slice list): the CTAs form one TEAM per active group -- team t of
// A active groups = CTAs [t nCTA / A, (t + 1) nCTA / A) -- and each team iterates its group's PCG with its own
// counter barrier, so teams never wait for each other's passes.  When a group converges its team raises the
// re-team request; every other team sees it at its next pass end (an OR over its CTAs' observations, so the whole
// team decides alike), stores its group's state and joins one grid barrier, after which the CTAs are split over the
// groups still active.  The slowest groups end up with the whole GPU, and no pass waits for the slowest of all
// CTAs of the grid (config 3 lock step: 7-11 us from a CTA's pass end to the end of its reducing barrier).
// Reductions do not depend on the team: the rows are cut into fixed chunks of kDynR slices, a warp adds a chunk's
// rows in a fixed order into one chunk partial, and every CTA of the team adds the group's chunk partials in a
// fixed order -- the results are bitwise the same whatever team sizes the timing of the re-team events produced.
#ifndef LC_DYN_R
#define LC_DYN_R 4
#endif
constexpr int kDynR = LC_DYN_R;          // slices per chunk (config 3 global: 4: 35.0 ms; 2: 35.8; 1: 39.8; 8: 37.7;
                                         // loading the update pass's operands of all 4 slices before the first
                                         // update spilled: 43.3 ms -- profiles/r02_t)
struct DynGroup {                        // a group's solver state between teams (global memory)
  int mode, par, it, final_, npass;
  unsigned gone;                         // 0, or the first phase without the group (its team finished it in phase
                                         // gone - 1): read for the active list, which must not depend on when a CTA
                                         // reads it -- a fast team may finish its group while a slow CTA still reads
  double rho, alpha, beta, tgt, nb, pad1;
  unsigned long long cbase;              // arrivals so far on the group's team counter
};
struct DynArgs {
  PcgArgs P;
  DynGroup* gst;                         // [G]
  double* cpart;                         // [2][G][nchk][2] chunk partials, double-buffered by the group's pass parity
  unsigned* fobs;                        // [2][nCTA] re-team request seen by the CTA before its team barrier
  unsigned long long* gctr;              // [G][16] team barrier counters (monotonic)
  unsigned* req;                         // re-team requests: phase k ends once *req > k
  int nchk;                              // chunks per group (the largest group's), the stride of cpart
};

template <int WM, int ST>
__global__ void __launch_bounds__(kPT, LCV_MINB) k_pcg_dyn(DynArgs D) {
  const PcgArgs& P = D.P;
  const SellView& A = P.A;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nCTA = gridDim.x, bid = blockIdx.x;
  const int G = P.G;
  __shared__ SegState S;
  __shared__ int s_act[kMaxSeg + 1];
  __shared__ int s_na, s_rt;
  __shared__ double s_w[kPW][2];
  __shared__ double s_sum[2];
  unsigned long long gepoch = 0;         // grid barriers (re-team phases) * nCTA
  unsigned phase = 0;
#ifdef LC_DEBUG_TIMELINE
  int tlk = 0;                           // CTA 0: per pass (start, chunks done, reduced) + the team size
#endif
  for (;;) {
    grid_barrier(P.bar, gepoch);         // phase boundary: every group's state is in D.gst
    if (threadIdx.x == 0) {
      int na = 0;
      for (int g = 0; g < G; ++g) {
        const unsigned gone = __ldcg(&D.gst[g].gone);
        if (gone == 0 || gone > phase) s_act[na++] = g;
      }
      s_na = na;
    }
    __syncthreads();
    const int na = s_na;
    if (na == 0) break;
    int t = (int)((bid * na) / nCTA);
    while (t > 0 && bid < (int64_t)t * nCTA / na) --t;
    while (t < na - 1 && bid >= (int64_t)(t + 1) * nCTA / na) ++t;
    const int64_t tb0 = (int64_t)t * nCTA / na, tn = (int64_t)(t + 1) * nCTA / na - tb0;
    const int g = s_act[t];
    if (threadIdx.x == 0) {
      const DynGroup& q = D.gst[g];
      S.mode = __ldcg(&q.mode); S.par = __ldcg(&q.par); S.it = __ldcg(&q.it); S.final_ = __ldcg(&q.final_);
      S.npass = __ldcg(&q.npass);
      S.rho = __ldcg(&q.rho); S.alpha = __ldcg(&q.alpha); S.beta = __ldcg(&q.beta); S.tgt = __ldcg(&q.tgt);
      S.nb = __ldcg(&q.nb);
    }
    unsigned long long* ctr = D.gctr + 16 * g;
    // the counter's arrivals so far come from the group's state (not from the counter itself: a fast member of
    // the new team may already have arrived for its first pass)
    unsigned long long target = 0;
    if (threadIdx.x == 0) target = __ldcg(&D.gst[g].cbase);
    __syncthreads();
    __shared__ long long s_g0, s_g1;
    if (threadIdx.x == 0) { s_g0 = P.A.seg_slice0[g]; s_g1 = P.A.seg_slice0[g + 1]; }
    __syncthreads();
    const int64_t s0g = s_g0, s1g = s_g1;
    const int64_t nchg = (s1g - s0g + kDynR - 1) / kDynR;   // this group's chunks
    // matrix-stream policy of this phase: evict_first while the active groups' working sets (values + 7 vectors)
    // exceed 3/4 of L2 together (the head of the solve); plain loads once they fit (the tail)
    const unsigned long long strm = l2_stream_policy(
        P.stream_vals >= 0 ? P.stream_vals != 0 : 4ll * na * (s1g - s0g) * 32 * (8 * A.W + 56) > 3 * P.l2_bytes);
    const int64_t kw = (bid - tb0) * kPW + warp, TW = tn * kPW;
    bool leave = false;
    while (!leave) {
      TL(tlk);
      const int mode = S.mode;
      const int par = S.npass & 1;
      double* cp = D.cpart + ((size_t)par * G + g) * (size_t)D.nchk * 2;
      // ---- the pass over this team's chunks
      const bool passA = mode == M_INIT || mode == M_CONFIRM || mode == M_FIRST || mode == M_NORMAL;
      const double beta = S.beta, alpha = S.alpha;
      const double* pold = S.par ? P.p1 : P.p0;
      double* pnew = S.par ? P.p0 : P.p1;
      for (int64_t c = kw; c < nchg; c += TW) {
        double a0 = 0.0, a1 = 0.0;
        for (int i = 0; i < kDynR; ++i) {
          const int64_t s = s0g + (int64_t)kDynR * c + i;
          if (s >= s1g) break;
          int64_t row0, end;
          slice_map_g(P, s, g, row0, end);
          const int64_t u = row0 + lane;
          if (u >= end) continue;
          if (passA) {
            const int64_t pl = (ST ? 32ll * A.vw * s : A.slice_ptr[s]) + lane;
            const int w = ST ? A.W : (int)((A.slice_ptr[s + 1] - (pl - lane)) >> 5);
            double own = 0.0;
            if (mode == M_INIT || mode == M_CONFIRM) {
              const double* xx = P.x;
              const double acc = row_dot<WM, ST>(A, pl, w, u, [&](int cc) { return xx[cc]; }, &own, strm);
              const double bi = P.b[u];
              const double ri = bi - acc;
              P.r[u] = ri;
              a0 = __fma_rn(ri, ri, a0);
              if (mode == M_INIT) a1 = __fma_rn(bi, bi, a1);
            } else {
              const double* zz = P.z;
              double acc;
              if (mode == M_FIRST) acc = row_dot<WM, ST>(A, pl, w, u, [&](int cc) { return zz[cc]; }, &own, strm);
              else acc = row_dot<WM, ST>(A, pl, w, u, [&](int cc) { return __fma_rn(beta, pold[cc], zz[cc]); }, &own, strm);
              const double pi = ST ? own : (mode == M_FIRST ? zz[u] : __fma_rn(beta, pold[u], zz[u]));
              pnew[u] = pi;
              P.q[u] = acc;
              a0 = __fma_rn(pi, acc, a0);
            }
          } else {
            const double di = A.dinv[u];
            if (mode == M_UPDATE) {
              const double* pp = S.par ? P.p1 : P.p0;
              const double xi = __fma_rn(alpha, pp[u], P.x[u]);
              const double ri = __fma_rn(-alpha, P.q[u], P.r[u]);
              const double zi = ri * di;
              P.x[u] = xi; P.r[u] = ri; P.z[u] = zi;
              a0 = __fma_rn(ri, zi, a0);
              a1 = __fma_rn(ri, ri, a1);
            } else {                                           // M_RESET
              const double ri = P.r[u];
              const double zi = ri * di;
              P.z[u] = zi;
              a0 = __fma_rn(ri, zi, a0);
            }
          }
        }
        a0 = warp_sum(a0);
        a1 = warp_sum(a1);
        if (lane == 0) { cp[2 * c] = a0; cp[2 * c + 1] = a1; }
      }
      TL(tlk);
      // ---- re-team request seen by this CTA (raises the group's flag word; ordered before the arrival by the
      // barrier's release), then the team barrier
      if (threadIdx.x == 0) {
        unsigned rq;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(rq) : "l"(D.req) : "memory");
        D.fobs[(size_t)par * nCTA + bid] = rq > phase ? 1u : 0u;
      }
      team_barrier(ctr, target, (unsigned)tn);
      // ---- the group's sums over its chunks (fixed order) and the team's decision
      {
        // thread i adds chunks i, i + kPT, ... in order, 8 loads in flight (one L2 round trip for 2048 chunks)
        double a0 = 0.0, a1 = 0.0;
        const double2* cp2 = reinterpret_cast<const double2*>(cp);
        for (int64_t c0 = threadIdx.x; c0 < nchg; c0 += 8 * kPT) {
          double2 v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = c0 + q * kPT < nchg ? __ldcg(cp2 + c0 + q * kPT) : make_double2(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < 8; ++q) { a0 += v[q].x; a1 += v[q].y; }
        }
        a0 = warp_sum(a0);
        a1 = warp_sum(a1);
        if (lane == 0) { s_w[warp][0] = a0; s_w[warp][1] = a1; }
        unsigned f = 0;                        // some member saw the request before this pass's barrier
        for (int64_t m = threadIdx.x; m < tn; m += kPT) f |= __ldcg(D.fobs + (size_t)par * nCTA + tb0 + m);
        f = __syncthreads_or(f);
        if (threadIdx.x == 0) {
          double o0 = 0.0, o1 = 0.0;
          for (int ww = 0; ww < kPW; ++ww) { o0 += s_w[ww][0]; o1 += s_w[ww][1]; }
          s_sum[0] = o0; s_sum[1] = o1;
          s_rt = (int)f;
        }
        __syncthreads();
      }
      TL(tlk);
#ifdef LC_DEBUG_TIMELINE
      if (bid == 0 && threadIdx.x == 0 && tlk < 8192) g_tl[tlk] = (unsigned long long)tn;
      ++tlk;
#endif
      // ---- scalars (thread 0; every CTA of the team computes the same)
      if (threadIdx.x == 0) {
        SegState& T = S;
        const double s0 = s_sum[0], s1 = s_sum[1];
        T.npass += 1;
        int fin = -100;
        double frn = 0.0;
        if (T.mode == M_INIT) {
          T.nb = sqrt(s1);
          T.tgt = T.nb > 0 ? P.eps * T.nb : P.eps;
          const double rn = sqrt(s0);
          if (!isfinite(rn)) { fin = LC_ERR_NONFINITE; frn = rn; }
          else if (rn <= T.tgt) { fin = LC_OK; frn = rn; }
          else if (P.max_iters == 0) { fin = LC_NOT_CONVERGED; frn = rn; }
          else T.mode = M_RESET;
        } else if (T.mode == M_FIRST || T.mode == M_NORMAL) {
          const double pq = s0;
          if (!(pq > 0)) { fin = isfinite(pq) ? LC_ERR_BREAKDOWN : LC_ERR_NONFINITE; frn = NAN; }
          else { T.alpha = T.rho / pq; T.mode = M_UPDATE; T.par ^= 1; }
        } else if (T.mode == M_CONFIRM) {
          const double rn = sqrt(s0);
          if (!isfinite(rn)) { fin = LC_ERR_NONFINITE; frn = rn; }
          else if (rn <= T.tgt) { fin = LC_OK; frn = rn; }
          else if (T.final_) { fin = LC_NOT_CONVERGED; frn = rn; }
          else T.mode = M_RESET;
        } else if (T.mode == M_UPDATE) {
          T.it += 1;
          const double rz = s0, rr = s1;
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
        if (fin != -100) {
          T.mode = M_DONE;
          if (bid == tb0) {
            P.out_iters[g] = T.it;
            P.out_status[g] = fin;
            P.out_relres[g] = T.nb > 0 ? frn / T.nb : frn;
          }
        }
      }
      __syncthreads();
      if (S.mode == M_DONE || s_rt) {
        // store the group's state (first CTA of the team), request the re-team (a finished group), leave
        if (bid == tb0 && threadIdx.x == 0) {
          DynGroup& q = D.gst[g];
          q.mode = S.mode; q.par = S.par; q.it = S.it; q.final_ = S.final_; q.npass = S.npass;
          q.rho = S.rho; q.alpha = S.alpha; q.beta = S.beta; q.tgt = S.tgt; q.nb = S.nb;
          q.cbase = target;
          if (S.mode == M_DONE) {
            q.gone = phase + 1;
            atomicMax(D.req, phase + 1);
          }
        }
        leave = true;
      }
    }
    ++phase;
  }
  // a8: x~[Omega] = xbar_B (Eq. 4) for explicit local subsystems, after every group converged
  if (P.scatter_idx)
    for (int64_t u = bid * kPT + threadIdx.x; u < A.nunits; u += nCTA * kPT) P.x_full[P.scatter_idx[u]] = P.x[u];
}

// ---------------------------------------------------------------- host ----
lc_status run_pcg(const PcgJob& job, const lc_solver_params* p, cudaStream_t s, lc_solve_info* info) {
  const Sell& M = *job.M;
  const int G = M.nseg;
  if (G > kMaxSeg) { set_error("PCG: at most 64 segments"); return LC_ERR_DIMENSION; }
  if (M.block != 1) { set_error("PCG: needs block = 1 (use LC_GMRES for block systems)"); return LC_ERR_INVALID_ARG; }
  if (pcg_dsmem_eligible(job)) return run_pcg_dsmem(job, p, s, info);     // fits one cluster's shared memory
  // compile-time width: SELL rows guard k < w, so W = 5 / 7 serve rows up to that width; stencil slices hold
  // exactly maxw slots, so they take W = 5 / 7 only when maxw is exactly that (else the generic loop)
  const int wi = (M.stencil ? (M.maxw == 5 ? 0 : M.maxw == 7 ? 1 : 2) : (M.maxw <= 5 ? 0 : M.maxw <= 7 ? 1 : 2)) +
                 (M.sym ? 6 : M.stencil ? 3 : 0);
#define LC_PCG_FNS(K) (void*)k_pcg<5, 0, K>, (void*)k_pcg<7, 0, K>, (void*)k_pcg<0, 0, K>, \
                      (void*)k_pcg<5, 1, K>, (void*)k_pcg<7, 1, K>, (void*)k_pcg<0, 1, K>, \
                      (void*)k_pcg<5, 2, K>, (void*)k_pcg<7, 2, K>, (void*)k_pcg<0, 2, K>
  void* const fns[27] = {LC_PCG_FNS(0), LC_PCG_FNS(1), LC_PCG_FNS(2)};
#undef LC_PCG_FNS
  // batched systems (G > 1), two schedules:
  //  - lock step: the whole grid sweeps the runs of all segments still active, pass by pass (every SM keeps
  //    streaming until the last segment converges);
  //  - teams: the CTAs form min(G, nCTA) contiguous teams, team t solves segments t, t + teams, ... one after
  //    another as G = 1 systems with its own counter barrier (no arrival-tree reduction over all segments).
  // A team's warps walk their slices one after another, so teams pay once each warp has only a few slices:
  // chosen when the rows worked on are <= 4 slices per warp of the grid (config 3: the masked local solves,
  // eta ~ 9%, 9.2 -> 4.9 ms; the global solves stay in lock step, 55 vs 80 ms with teams).  lc_tuning.batched_schedule forces either.
  const lc_tuning& tune = tuning();
  const int64_t rows_work = job.rows_hint >= 0 ? job.rows_hint : M.nunits;
  bool team_k = G > 1;
  lc_status st;
  // dynamic teams (k_pcg_dyn): batched global solves over equal segments (no slice list, no mask)
  const bool dyn_ok = G > 1 && !job.slist && !job.omega;
  if (team_k) {
    if (tune.batched_schedule >= 0) team_k = tune.batched_schedule == 1;
    else {
      // the team kernels' occupancy equals the lock-step kernels' (same launch bounds, 64 registers)
      int64_t lock_ctas = 0;
      st = max_coresident(fns[9 + wi], kPT, 0, &lock_ctas);
      if (st) return st;
      team_k = rows_work <= (int64_t)4 * 32 * kPW * lock_ctas;
    }
  }
  // (larger batched solves: lock step; two task-flow schedules measured slower, profiles/r01_aj)
  int kind = G == 1 ? 0 : team_k ? 2 : 1;
  void* fn = fns[wi + 9 * kind];
  // lock-step candidates without a slice list run as dynamic teams (lc_tuning.batched_schedule -1; 2 forces them
  // for the static-team candidates too: config 3's explicit local subsystems 4.70 ms with static teams, 5.60 with
  // dynamic ones -- their groups are small and converge alike, so the re-team stops cost more than they balance)
  if (kind >= 1 && dyn_ok && ((tune.batched_schedule == -1 && kind == 1) || tune.batched_schedule == 2)) {
    void* const dfns[9] = {(void*)k_pcg_dyn<5, 0>, (void*)k_pcg_dyn<7, 0>, (void*)k_pcg_dyn<0, 0>,
                           (void*)k_pcg_dyn<5, 1>, (void*)k_pcg_dyn<7, 1>, (void*)k_pcg_dyn<0, 1>,
                           (void*)k_pcg_dyn<5, 2>, (void*)k_pcg_dyn<7, 2>, (void*)k_pcg_dyn<0, 2>};
    int64_t dctas = 0;
    st = max_coresident(dfns[wi], kPT, 0, &dctas);
    if (st) return st;
    if (dctas >= G) { kind = 3; fn = dfns[wi]; }
  }
  // TMA staging for contiguous slice ranges (global solves); slice-list (masked) solves keep plain loads: the
  // per-slice bulk copies were 4% slower there in the bench (profiles/r01_h_tma_ab.txt)
  // (the explicit subsystems' uniform-width SELL slices stream their columns through the same ring)
  const bool tma = (M.stencil || M.uniform) && (M.maxw == 5 || M.maxw == 7) && G == 1 && !job.slist && tune.pcg_tma;
  const size_t dsmem = tma ? (size_t)kStages * kPW * 32 * (M.sym ? M.vw : M.maxw) * (M.stencil ? 8 : 12) : 0;
  int64_t max_ctas = 0;
  st = max_coresident(fn, kPT, dsmem, &max_ctas);
  if (st) return st;
  const int64_t n = M.nunits;
  const int64_t work = job.slist ? job.nlist_max : M.nslices;
  // small single-segment solves: one cluster of <= 16 CTAs (<= 512 slices = 4 per warp)
  const bool clus = G == 1 && work <= 16 * kPW * 4 && tune.pcg_cluster;
  int64_t nCTA = std::min<int64_t>(max_ctas, (std::max<int64_t>(work, 1) + kPW - 1) / kPW);
  if (tune.pcg_max_ctas > 0) nCTA = std::max<int64_t>(1, std::min<int64_t>(nCTA, tune.pcg_max_ctas));
  if (nCTA < 1) nCTA = 1;
  if (kind == 3) nCTA = max_ctas;          // every co-resident CTA: the teams split the grid among the groups
  // batched lock step: launched in clusters of CL CTAs (cluster_reduce_barrier: one level of global latency per
  // reduction instead of two), as many whole clusters as are co-resident
  int CL = (kind == 1 && tune.batched_cluster > 1) ? tune.batched_cluster : 0;
  if (CL) {
    int64_t maxcl = 0;
    if (max_clusters(fn, kPT, dsmem, CL, &maxcl) != LC_OK || maxcl < 1) { cudaGetLastError(); CL = 0; }
    else nCTA = std::max<int64_t>(1, std::min<int64_t>(maxcl, (nCTA + CL - 1) / CL)) * CL;
  }
  void* ws = nullptr;
  void* dws = nullptr;                            // dynamic teams' extra workspace
  const size_t vec = sizeof(double) * (size_t)n;
  const size_t vbytes = (vec + 255) & ~(size_t)255;
  const bool own_x = job.x_init != nullptr;
  const int teams = team_k ? (int)std::min<int64_t>(G, nCTA) : 0;
  const int npv = G == 1 ? 3 : 2;                 // search-direction buffers (3: lazy x of depth 3 possible)
  const size_t bytes = vbytes * (own_x ? 4 + npv : 3 + npv) + sizeof(double) * 2 * G * (2 * nCTA + 1 + 2 * kBarSub) + 16 * G +
                       sizeof(GridBar) + 640 + 128 * (size_t)kMaxSeg;
  st = dalloc(&ws, bytes, s);
  if (st) return st;
  char* w = (char*)ws;
  PcgArgs a;
  a.A = view(M);
  a.b = job.b;
  a.r = (double*)w; w += vbytes;
  a.z = (double*)w; w += vbytes;
  a.q = (double*)w; w += vbytes;
  a.p0 = (double*)w; w += vbytes;
  a.p1 = (double*)w; w += vbytes;
  a.p2 = nullptr;
  if (npv == 3) { a.p2 = (double*)w; w += vbytes; }
  cudaError_t e = cudaSuccess;
  if (own_x) {
    a.x = (double*)w; w += vbytes;
    e = cudaMemcpyAsync(a.x, job.x_init, vec, cudaMemcpyDeviceToDevice, s);
  } else {
    a.x = job.x;
  }
  if (job.omega && e == cudaSuccess) e = cudaMemsetAsync(a.r, 0, vbytes * (3 + npv), s);   // zero outside Omega
  // batched (G > 1): a boundary row's stencil holes gather z / p of the neighbouring segment (times an exact 0),
  // which may not have been written yet (its team has not started it, or it converged at INIT): start them at 0
  if (G > 1 && !job.omega && e == cudaSuccess) e = cudaMemsetAsync(a.z, 0, vbytes, s);
  if (G > 1 && !job.omega && e == cudaSuccess) e = cudaMemsetAsync(a.p0, 0, vbytes * 2, s);
  a.part = (double*)w; w += sizeof(double) * 2 * G * 2 * nCTA;   // G = 1: two buffers (by pass)
  a.red = (double*)w; w += sizeof(double) * 2 * G;
  a.subred = (double*)w; w += sizeof(double) * 2 * G * 2 * kBarSub;
  w = (char*)((((uintptr_t)w) + 127) & ~(uintptr_t)127);
  a.bar = (GridBar*)w; w += sizeof(GridBar);
  a.out_iters = (int*)w; w += 4 * G;
  a.out_status = (int*)w; w += 4 * G;
  a.out_relres = (double*)((((uintptr_t)w) + 7) & ~(uintptr_t)7);
  a.tctr = (unsigned long long*)((((uintptr_t)(a.out_relres + G)) + 127) & ~(uintptr_t)127);
  a.teams = teams;
  a.clus = CL ? 1 : 0;
  a.slist = job.slist;
  a.nlist = job.nlist_dev;
  a.omega = job.omega;
  a.seg_j0 = job.slist ? job.lseg : M.seg_slice0;
  a.scatter_idx = job.scatter_idx;
  a.x_full = job.x_full;
  a.x_user = job.x_user;
  a.eps = p->rel_tol;
  a.max_iters = p->max_iters;
  a.G = G;
  a.reg_units = job.reg_units;
  a.spg = job.spg;
  a.tma = tma && !clus ? 1 : 0;
  a.cluster = clus ? 1 : 0;
  // (masked solves qualify too: rows outside Omega hold p = q = r = z = 0 and x = 0, the update keeps them 0)
  a.vec2 = (G == 1 && !job.slist &&
            ((((uintptr_t)a.x) | ((uintptr_t)a.r) | ((uintptr_t)a.z) | ((uintptr_t)a.q) | ((uintptr_t)a.p0) |
              ((uintptr_t)a.p1) | ((uintptr_t)a.p2) | ((uintptr_t)M.dinv)) & 15) == 0) ? 1 : 0;
  // lazy x of depth 3 (tuning.lazy_x_depth: 2 or 3; 0 / 1: x updated every pass)
  a.lazyx = (kind == 0 && a.vec2 && tune.lazy_x_depth > 1) ? tune.lazy_x_depth : 0;
  a.np3 = a.lazyx == 3 ? 1 : 0;
  {
    // L2 policy of the matrix stream (lc_internal.cuh): bytes an iteration streams once, and the vectors it re-reads
    // (r, z, q, the search directions, x, 1/a_ii) over the rows worked on; dynamic teams decide per phase
    const int64_t mbytes = rows_work * (int64_t)M.maxw * (M.stencil ? 8 : 12);
    const int64_t wbytes = rows_work * 8 * (int64_t)(5 + npv);
    a.l2_bytes = l2_bytes();
    a.stream_vals = kind == 3 ? tune.l2_stream_hint : (stream_policy_wanted(mbytes, wbytes) ? 1 : 0);
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(a.bar, 0, sizeof(GridBar), s);
  if (e == cudaSuccess && teams) e = cudaMemsetAsync(a.tctr, 0, 128 * (size_t)teams, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.out_iters, 0, 8 * G, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.out_relres, 0, 8 * G, s);
  SolveClock clk(job.defer);
  cudaEventRecord(clk.e0, s);
  void* args[] = {&a};
  if (clus) {
    if (func_attr(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != LC_OK) cudaGetLastError();
    unsigned csz = (unsigned)std::min<int64_t>(16, std::max<int64_t>(1, (work + 4 * kPW - 1) / (4 * kPW)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csz);
    cfg.blockDim = dim3(kPT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csz;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (e == cudaSuccess) e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess && csz > 8) {           // non-portable size refused: fall back to 8
      cudaGetLastError();
      csz = 8;
      cfg.gridDim = dim3(csz);
      attr[0].val.clusterDim.x = csz;
      e = cudaLaunchKernelExC(&cfg, fn, args);
    }
  } else if (e == cudaSuccess && kind == 3) {
    // dynamic teams: per-group state, chunk partials, per-CTA request flags, team counters, request word
    int64_t spg_max = 0;                          // the largest segment's slices
    for (int g = 0; g < G; ++g) spg_max = std::max<int64_t>(spg_max, M.h_seg_slice0[g + 1] - M.h_seg_slice0[g]);
    const int nchk = (int)((spg_max + kDynR - 1) / kDynR);
    const size_t b_gst = ((sizeof(DynGroup) * G + 255) & ~(size_t)255);
    const size_t b_cp = ((sizeof(double) * 2 * 2 * (size_t)G * nchk + 255) & ~(size_t)255);
    const size_t b_fo = ((sizeof(unsigned) * 2 * (size_t)nCTA + 255) & ~(size_t)255);
    const size_t b_ct = (size_t)128 * G + 256;
    if (st = dalloc(&dws, b_gst + b_cp + b_fo + b_ct, s); st) { dfree(ws, s); return st; }
    DynArgs da;
    da.P = a;
    char* dw = (char*)dws;
    da.gst = (DynGroup*)dw; dw += b_gst;
    da.cpart = (double*)dw; dw += b_cp;
    da.fobs = (unsigned*)dw; dw += b_fo;
    da.gctr = (unsigned long long*)dw;
    da.req = (unsigned*)(dw + 128 * G);
    da.nchk = nchk;
    e = cudaMemsetAsync(da.gst, 0, b_gst, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(da.fobs, 0, b_fo, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(da.gctr, 0, b_ct, s);
    void* dargs[] = {&da};
    if (e == cudaSuccess) e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)nCTA), dim3(kPT), dargs, 0, s);
  } else if (e == cudaSuccess && CL) {
    // cooperative (co-residency is checked by the driver) and clustered
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nCTA);
    cfg.blockDim = dim3(kPT);
    cfg.dynamicSmemBytes = dsmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)CL; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    e = cudaLaunchKernelExC(&cfg, fn, args);
  } else if (e == cudaSuccess) {
    e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)nCTA), dim3(kPT), args, dsmem, s);
  }
  count_launch();
  cudaEventRecord(clk.e1, s);
  const int kernel = kind == 1 ? LC_KERNEL_PCG_LOCKSTEP : kind == 2 ? LC_KERNEL_PCG_TEAMS
                     : kind == 3 ? LC_KERNEL_PCG_DYNTEAMS : clus ? LC_KERNEL_PCG_CLUSTER : LC_KERNEL_PCG_GRID;
  // (the copies of solve_finish are enqueued before the stream-ordered free of the workspace they read)
  struct FreeAfter { void* p; cudaStream_t s; ~FreeAfter() { dfree(p, s); } } fa{ws, s}, fd{dws, s};
  return solve_finish(e, clk, job.defer, G, a.out_iters, a.out_status, a.out_relres, kernel,
                      a.lazyx > 1 ? a.lazyx : 1, s, info, "PCG kernel");
}

}  // namespace lc

#ifdef LC_DEBUG_TIMELINE
extern "C" int lc_debug_timeline(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, lc::g_tl, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -1;
}
extern "C" int lc_debug_cta_window(int pass0) {
  return cudaMemcpyToSymbol(lc::g_cta_pass0, &pass0, sizeof(int)) == cudaSuccess ? 0 : -1;
}
extern "C" int lc_debug_cta(unsigned long long* out) {   // [64][1024][3]
  return cudaMemcpyFromSymbol(out, lc::g_cta, sizeof(unsigned long long) * 64 * 1024 * 3) == cudaSuccess ? 0 : -1;
}
#endif
