// pcg_dsmem.cu -- Jacobi-PCG for small single-segment stencil systems held entirely on chip
// ("small systems: one thread-block cluster of <= 16 CTAs holds the Krylov vectors in
// DSMEM, and the matrix too where it fits").
//
// One thread-block cluster of nq <= 16 CTAs; CTA q owns the rows [q R, min(n, (q+1) R)) and keeps their
// stencil values, 1/a_ii, b and every Krylov vector (x, r, z, q, p, p_old) in its shared memory for the
// whole solve.  A gathered neighbour row owned by another CTA of the cluster is read from that CTA's shared
// memory (distributed shared memory, ld.shared::cluster through map_shared_rank).  One cluster barrier per
// pass (two per iteration); the per-CTA partial dots are double-buffered by pass and read across the cluster
// in rank order (fixed-order, bitwise deterministic).  The step order and the recursive/true residual
// protocol are those of k_pcg (pcg.cu, or_pcg): INIT/CONFIRM r = b - A x, FIRST/NORMAL q = A p with
// p = z + beta p_old formed on the fly, UPDATE x, r, z.  Device memory is touched only to load the system
// and to write x back, so an iteration costs shared-memory latencies instead of L2 round trips.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "lc_internal.cuh"

namespace cg = cooperative_groups;

namespace lc {

constexpr int kST = 512;                 // threads per CTA
constexpr int kSW = kST / 32;
constexpr int kMaxCluster = 16;
constexpr size_t kSmemBudget = 200 * 1024;   // dynamic shared memory per CTA

struct DsArgs {
  SellView A;                    // stencil layout (values + dinv read once)
  const double* b;
  const double* x_in;            // initial guess
  double* x_out;                 // result: all rows (global solve) or the Omega rows (masked local solve)
  const uint8_t* omega;          // masked solve: row u is in the subsystem iff omega[u] != 255
  int n, R;                      // rows, rows per CTA
  double eps;
  int max_iters;
  int* out_iters;
  int* out_status;
  double* out_relres;
};

enum DsMode : int { S_INIT = 0, S_RESET, S_FIRST, S_NORMAL, S_UPDATE, S_CONFIRM, S_DONE };

template <int W>
__global__ void __launch_bounds__(kST, 1) k_pcg_ds(DsArgs P) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double s_part[2][2], s_w[kSW][2], s_sum[2];
  __shared__ int s_mode, s_par, s_it, s_final, s_exit;
  __shared__ double s_rho, s_alpha, s_beta, s_tgt, s_nb;
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank(), nq = (int)cl.num_blocks();
  const int R = P.R, n = P.n;
  const int r0 = q * R, nr = max(0, min(n, r0 + R) - r0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const SellView& A = P.A;
  double* val = sm;                       // [W][R]
  double* x = val + (size_t)W * R;
  double* r = x + R;
  double* z = r + R;
  double* qv = z + R;
  double* p0 = qv + R;
  double* p1 = p0 + R;
  double* dv = p1 + R;
  double* bv = dv + R;
  uint8_t* om = reinterpret_cast<uint8_t*>(bv + R);
  // ---- load the CTA's rows
  for (int i = threadIdx.x; i < nr; i += kST) {
    const int u = r0 + i;
    const int64_t pl = 32ll * W * (u >> 5) + (u & 31);
#pragma unroll
    for (int k = 0; k < W; ++k) val[(size_t)k * R + i] = A.val[pl + 32 * k];
    x[i] = P.x_in[u];
    bv[i] = P.b[u];
    dv[i] = A.dinv[u];
    om[i] = P.omega ? P.omega[u] : 0;
    r[i] = 0.0; z[i] = 0.0; qv[i] = 0.0; p0[i] = 0.0; p1[i] = 0.0;
  }
  if (threadIdx.x == 0) {
    s_mode = S_INIT; s_par = 0; s_it = 0; s_final = 0; s_exit = 0;
    s_rho = s_alpha = s_beta = s_tgt = s_nb = 0.0;
  }
  cl.sync();
  // value of vector v (an array of this CTA's layout) at global row c, from the owning CTA
  auto at = [&](double* v, int c) -> double {
    const int owner = c / R;
    const int li = c - owner * R;
    if (owner == q) return v[li];
    return cl.map_shared_rank(v, owner)[li];
  };
  int ppar = 0;                           // partial buffer parity
  auto reduce = [&](double a0, double a1) {
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    if (lane == 0) { s_w[warp][0] = a0; s_w[warp][1] = a1; }
    __syncthreads();
    if (threadIdx.x < 2) {
      double t = 0.0;
      for (int w = 0; w < kSW; ++w) t += s_w[w][threadIdx.x];
      s_part[ppar][threadIdx.x] = t;
    }
    cl.sync();
    if (threadIdx.x < 2) {
      double t = 0.0;
      for (int o = 0; o < nq; ++o) t += cl.map_shared_rank(&s_part[ppar][0], o)[threadIdx.x];
      s_sum[threadIdx.x] = t;
    }
    ppar ^= 1;
    __syncthreads();
  };
  auto finish = [&](int status, double rn) {
    s_mode = S_DONE;
    if (q == 0) {
      *P.out_iters = s_it;
      *P.out_status = status;
      *P.out_relres = s_nb > 0 ? rn / s_nb : rn;
    }
  };
  const int nu1 = n - 1;
  for (;;) {
    // ---------------------------------------------------------------- pass A
    const int mode = s_mode;
    double a0 = 0.0, a1 = 0.0;
    if (mode == S_INIT || mode == S_CONFIRM || mode == S_FIRST || mode == S_NORMAL) {
      const double beta = s_beta;
      double* pold = s_par ? p1 : p0;
      double* pnew = s_par ? p0 : p1;
      for (int i = threadIdx.x; i < nr; i += kST) {
        const int u = r0 + i;
        double acc = 0.0, own = 0.0;
#pragma unroll
        for (int k = 0; k < W; ++k) {
          int c = u + A.off[k];
          c = c < 0 ? 0 : (c > nu1 ? nu1 : c);
          double y;
          if (mode == S_INIT || mode == S_CONFIRM) y = at(x, c);
          else if (mode == S_FIRST) y = at(z, c);
          else y = __fma_rn(beta, at(pold, c), at(z, c));
          acc = __fma_rn(val[(size_t)k * R + i], y, acc);
          if (A.off[k] == 0) own = y;
        }
        if (om[i] == 255) continue;                // masked solve: rows outside Omega stay 0
        if (mode == S_INIT || mode == S_CONFIRM) {
          const double bi = bv[i];
          const double ri = bi - acc;
          r[i] = ri;
          a0 = __fma_rn(ri, ri, a0);
          if (mode == S_INIT) a1 = __fma_rn(bi, bi, a1);
        } else {
          pnew[i] = own;
          qv[i] = acc;
          a0 = __fma_rn(own, acc, a0);
        }
      }
    }
    reduce(a0, a1);
    if (threadIdx.x == 0) {
      const double s0 = s_sum[0], s1 = s_sum[1];
      if (mode == S_INIT) {
        s_nb = sqrt(s1);
        s_tgt = s_nb > 0 ? P.eps * s_nb : P.eps;
        const double rn = sqrt(s0);
        if (!isfinite(rn)) finish(LC_ERR_NONFINITE, rn);
        else if (rn <= s_tgt) finish(LC_OK, rn);
        else if (P.max_iters == 0) finish(LC_NOT_CONVERGED, rn);       // Eq. 6 check only
        else s_mode = S_RESET;
      } else if (mode == S_FIRST || mode == S_NORMAL) {
        if (!(s0 > 0)) finish(isfinite(s0) ? LC_ERR_BREAKDOWN : LC_ERR_NONFINITE, NAN);
        else { s_alpha = s_rho / s0; s_mode = S_UPDATE; s_par ^= 1; }
      } else if (mode == S_CONFIRM) {
        const double rn = sqrt(s0);
        if (!isfinite(rn)) finish(LC_ERR_NONFINITE, rn);
        else if (rn <= s_tgt) finish(LC_OK, rn);
        else if (s_final) finish(LC_NOT_CONVERGED, rn);
        else s_mode = S_RESET;
      }
    }
    __syncthreads();
    // ---------------------------------------------------------------- pass B (own rows only)
    const int modeb = s_mode;
    a0 = a1 = 0.0;
    if (modeb == S_UPDATE || modeb == S_RESET) {
      const double alpha = s_alpha;
      const double* pp = s_par ? p1 : p0;
      for (int i = threadIdx.x; i < nr; i += kST) {
        if (modeb == S_UPDATE) {
          const double xi = __fma_rn(alpha, pp[i], x[i]);
          const double ri = __fma_rn(-alpha, qv[i], r[i]);
          const double zi = ri * dv[i];
          x[i] = xi; r[i] = ri; z[i] = zi;
          a0 = __fma_rn(ri, zi, a0);
          a1 = __fma_rn(ri, ri, a1);
        } else {
          const double zi = r[i] * dv[i];
          z[i] = zi;
          a0 = __fma_rn(r[i], zi, a0);
        }
      }
    }
    reduce(a0, a1);
    if (threadIdx.x == 0) {
      const double s0 = s_sum[0], s1 = s_sum[1];
      if (modeb == S_UPDATE) {
        s_it += 1;
        if (!isfinite(s1) || sqrt(s1) <= s_tgt || s_it >= P.max_iters) {
          s_mode = S_CONFIRM;
          s_final = (s_it >= P.max_iters) || !isfinite(s1);
        } else {
          s_beta = s0 / s_rho;
          s_rho = s0;
          s_mode = S_NORMAL;
        }
      } else if (modeb == S_RESET) {
        s_rho = s0;
        s_mode = S_FIRST;
      }
      s_exit = s_mode == S_DONE;
    }
    __syncthreads();
    if (s_exit) break;
  }
  // a8 (Eq. 4) / the global solve's result back to device memory
  for (int i = threadIdx.x; i < nr; i += kST)
    if (om[i] != 255) P.x_out[r0 + i] = x[i];
  cl.sync();                                       // no CTA leaves while others may still read its memory
}

// ---- single-reduction form (Chronopoulos-Gear recurrences): ONE cluster barrier per iteration -----------------
// The textbook iteration above synchronises twice (p^T A p for alpha, then r^T z for beta): ~1.1 us each on a
// 16-CTA cluster, of a 3 us iteration.  Here u = M^-1 r, w = A u and the recurrences p = u + beta p,
// s = w + beta s (= A p), x += alpha p, r -= alpha s give the same iterates in exact arithmetic with
// gamma = r^T u, delta = w^T u reduced together: beta' = gamma'/gamma, alpha' = gamma'/(delta' - beta' gamma'/alpha).
// One pass per iteration: a row updates p, s, x, r and then needs u_new = M^-1 r_new of its NEIGHBOURS for
// w_new = A u_new; instead of a second barrier every neighbour's u_new is recomputed from its old r, w, s and
// 1/a_cc (the same expression as its owner evaluates, so bitwise the same value) -- four shared-memory / DSMEM
// reads per neighbour instead of two; r, w, s are double-buffered by iteration.  Stopping test, true-residual
// confirmation and restart (R19) as above; iteration count = x updates (R30).
enum Ds1Mode : int { T_INIT = 0, T_START, T_LOOP, T_CONFIRM, T_DONE };

template <int W>
__global__ void __launch_bounds__(kST, 1) k_pcg_ds1(DsArgs P) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double s_part[2][3], s_w[kSW][3], s_sum[3];
  __shared__ int s_mode, s_par, s_it, s_final, s_exit;
  __shared__ double s_gamma, s_alpha, s_beta, s_tgt, s_nb;
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank(), nq = (int)cl.num_blocks();
  const int R = P.R, n = P.n;
  const int r0 = q * R, nr = max(0, min(n, r0 + R) - r0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const SellView& A = P.A;
  double* val = sm;                       // [W][R]
  double* x = val + (size_t)W * R;
  // r, w, s double-buffered by iteration: buffer b of r at x + (1 + b) R, of w at x + (3 + b) R, of s at x + (5 + b) R
  double* pv = x + 7 * R;
  double* dv = x + 8 * R;
  double* bv = x + 9 * R;
  uint8_t* om = reinterpret_cast<uint8_t*>(x + 10 * R);
  for (int i = threadIdx.x; i < nr; i += kST) {
    const int u = r0 + i;
    const int64_t pl = 32ll * W * (u >> 5) + (u & 31);
#pragma unroll
    for (int k = 0; k < W; ++k) val[(size_t)k * R + i] = A.val[pl + 32 * k];
    x[i] = P.x_in[u];
    bv[i] = P.b[u];
    dv[i] = A.dinv[u];
    om[i] = P.omega ? P.omega[u] : 0;
#pragma unroll
    for (int v = 1; v <= 7; ++v) x[(size_t)v * R + i] = 0.0;
  }
  if (threadIdx.x == 0) {
    s_mode = T_INIT; s_par = 0; s_it = 0; s_final = 0; s_exit = 0;
    s_gamma = s_alpha = s_beta = s_tgt = s_nb = 0.0;
  }
  cl.sync();
  int ppar = 0;
  auto reduce = [&](double a0, double a1, double a2) {
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    if (lane == 0) { s_w[warp][0] = a0; s_w[warp][1] = a1; s_w[warp][2] = a2; }
    __syncthreads();
    if (threadIdx.x < 3) {
      double t = 0.0;
      for (int w = 0; w < kSW; ++w) t += s_w[w][threadIdx.x];
      s_part[ppar][threadIdx.x] = t;
    }
    cl.sync();
    if (threadIdx.x < 3) {
      double t = 0.0;
      for (int o = 0; o < nq; ++o) t += cl.map_shared_rank(&s_part[ppar][0], o)[threadIdx.x];
      s_sum[threadIdx.x] = t;
    }
    ppar ^= 1;
    __syncthreads();
  };
  auto finish = [&](int status, double rn) {
    s_mode = T_DONE;
    if (q == 0) {
      *P.out_iters = s_it;
      *P.out_status = status;
      *P.out_relres = s_nb > 0 ? rn / s_nb : rn;
    }
  };
  const int nu1 = n - 1;
  for (;;) {
    const int mode = s_mode;
    const int cur = s_par;
    double* rc = x + (size_t)(1 + cur) * R;
    double* wc = x + (size_t)(3 + cur) * R;
    double* sc = x + (size_t)(5 + cur) * R;
    double* rn_ = x + (size_t)(2 - cur) * R;
    double* wn_ = x + (size_t)(4 - cur) * R;
    double* sn_ = x + (size_t)(6 - cur) * R;
    const double alpha = s_alpha, beta = s_beta;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int i = threadIdx.x; i < nr; i += kST) {
      if (om[i] == 255) continue;                  // masked solve: rows outside Omega stay 0
      const int u = r0 + i;
      if (mode == T_INIT || mode == T_CONFIRM) {   // r = b - A x
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < W; ++k) {
          int c = u + A.off[k];
          c = c < 0 ? 0 : (c > nu1 ? nu1 : c);
          const int owner = c / R, li = c - owner * R;
          const double y = owner == q ? x[li] : cl.map_shared_rank(x, owner)[li];
          acc = __fma_rn(val[(size_t)k * R + i], y, acc);
        }
        const double bi = bv[i];
        const double ri = bi - acc;
        rc[i] = ri;
        a0 = __fma_rn(ri, ri, a0);
        if (mode == T_INIT) a1 = __fma_rn(bi, bi, a1);
      } else if (mode == T_START) {                // w = A u, u = M^-1 r; gamma = r^T u, delta = w^T u
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < W; ++k) {
          int c = u + A.off[k];
          c = c < 0 ? 0 : (c > nu1 ? nu1 : c);
          const int owner = c / R, li = c - owner * R;
          const double* rr = owner == q ? rc : cl.map_shared_rank(rc, owner);
          const double* dd = owner == q ? dv : cl.map_shared_rank(dv, owner);
          acc = __fma_rn(val[(size_t)k * R + i], dd[li] * rr[li], acc);
        }
        const double ui = dv[i] * rc[i];
        wc[i] = acc;
        a0 = __fma_rn(rc[i], ui, a0);
        a1 = __fma_rn(acc, ui, a1);
      } else {                                     // T_LOOP
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < W; ++k) {
          int c = u + A.off[k];
          c = c < 0 ? 0 : (c > nu1 ? nu1 : c);
          const int owner = c / R, li = c - owner * R;
          const double* rr = owner == q ? rc : cl.map_shared_rank(rc, owner);
          const double* ww = owner == q ? wc : cl.map_shared_rank(wc, owner);
          const double* ss = owner == q ? sc : cl.map_shared_rank(sc, owner);
          const double* dd = owner == q ? dv : cl.map_shared_rank(dv, owner);
          const double s_c = __fma_rn(beta, ss[li], ww[li]);
          const double r_c = __fma_rn(-alpha, s_c, rr[li]);
          acc = __fma_rn(val[(size_t)k * R + i], dd[li] * r_c, acc);
        }
        const double ui = dv[i] * rc[i];
        const double pi = __fma_rn(beta, pv[i], ui);
        const double si = __fma_rn(beta, sc[i], wc[i]);
        const double rni = __fma_rn(-alpha, si, rc[i]);
        const double uni = dv[i] * rni;
        pv[i] = pi;
        x[i] = __fma_rn(alpha, pi, x[i]);
        sn_[i] = si; rn_[i] = rni; wn_[i] = acc;
        a0 = __fma_rn(rni, uni, a0);
        a1 = __fma_rn(acc, uni, a1);
        a2 = __fma_rn(rni, rni, a2);
      }
    }
    reduce(a0, a1, a2);
    if (threadIdx.x == 0) {
      const double s0 = s_sum[0], s1 = s_sum[1], s2 = s_sum[2];
      if (mode == T_INIT) {
        s_nb = sqrt(s1);
        s_tgt = s_nb > 0 ? P.eps * s_nb : P.eps;
        const double rn = sqrt(s0);
        if (!isfinite(rn)) finish(LC_ERR_NONFINITE, rn);
        else if (rn <= s_tgt) finish(LC_OK, rn);
        else if (P.max_iters == 0) finish(LC_NOT_CONVERGED, rn);       // Eq. 6 check only
        else s_mode = T_START;
      } else if (mode == T_CONFIRM) {
        const double rn = sqrt(s0);
        if (!isfinite(rn)) finish(LC_ERR_NONFINITE, rn);
        else if (rn <= s_tgt) finish(LC_OK, rn);
        else if (s_final) finish(LC_NOT_CONVERGED, rn);
        else s_mode = T_START;
      } else if (mode == T_START) {
        if (!(s1 > 0)) finish(isfinite(s1) ? LC_ERR_BREAKDOWN : LC_ERR_NONFINITE, NAN);
        else { s_gamma = s0; s_alpha = s0 / s1; s_beta = 0.0; s_mode = T_LOOP; }
      } else {                                     // T_LOOP: one x update done
        s_it += 1;
        s_par ^= 1;
        if (!isfinite(s2) || sqrt(s2) <= s_tgt || s_it >= P.max_iters) {
          s_mode = T_CONFIRM;
          s_final = (s_it >= P.max_iters) || !isfinite(s2);
        } else {
          const double b2 = s0 / s_gamma;
          const double den = s1 - b2 * s0 / s_alpha;
          if (!(den > 0)) finish(isfinite(den) ? LC_ERR_BREAKDOWN : LC_ERR_NONFINITE, NAN);
          else { s_beta = b2; s_alpha = s0 / den; s_gamma = s0; }
        }
      }
      s_exit = s_mode == T_DONE;
    }
    __syncthreads();
    if (s_exit) break;
    // (the pass of the next iteration reads other CTAs' rows of THIS pass: ordered by the cluster barrier inside
    // reduce(); their next writes go to the other buffers, and the buffers they then overwrite were last read
    // before the barrier of this iteration)
  }
  for (int i = threadIdx.x; i < nr; i += kST)
    if (om[i] != 255) P.x_out[r0 + i] = x[i];
  cl.sync();                                       // no CTA leaves while others may still read its memory
}

static size_t ds_row_bytes(int W) {             // values + 8 (textbook) / 10 (single-reduction) vectors + flag
  return (size_t)8 * W + 8 * (tuning().pcg_cluster_resident == 2 ? 10 : 8) + 1;
}

// true: the system fits the cluster-resident kernel (single segment, 5- or 7-point stencil, <= 16 CTAs)
bool pcg_dsmem_eligible(const PcgJob& job) {
  const Sell& M = *job.M;
  if (M.nseg != 1 || !M.stencil || M.sym || M.block != 1 || (M.maxw != 5 && M.maxw != 7)) return false;
  if (job.scatter_idx || !tuning().pcg_cluster_resident) return false;
  const int64_t rmax = (int64_t)((kSmemBudget - 64) / ds_row_bytes(M.maxw));
  return M.nunits <= rmax * kMaxCluster;
}

lc_status run_pcg_dsmem(const PcgJob& job, const lc_solver_params* p, cudaStream_t s, lc_solve_info* info) {
  const Sell& M = *job.M;
  const int W = M.maxw;
  const int n = (int)M.nunits;
  const bool single = tuning().pcg_cluster_resident == 2;
  void* fn = single ? (W == 5 ? (void*)k_pcg_ds1<5> : (void*)k_pcg_ds1<7>)
                    : (W == 5 ? (void*)k_pcg_ds<5> : (void*)k_pcg_ds<7>);
  lc_status st = func_attr(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget);
  if (st) return st;
  st = func_attr(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (st) return st;
  DevBuf ws(s);
  st = ws.alloc(64);
  if (st) return st;
  DsArgs a;
  a.A = view(M);
  a.b = job.b;
  a.x_in = job.x_init ? job.x_init : job.x;
  a.x_out = job.x_user ? job.x_user : job.x;
  a.omega = job.omega;
  a.n = n;
  a.eps = p->rel_tol;
  a.max_iters = p->max_iters;
  a.out_iters = (int*)ws.p;
  a.out_status = (int*)ws.p + 1;
  a.out_relres = (double*)((char*)ws.p + 8);
  SolveClock clk(job.defer);
  cudaError_t e = cudaMemsetAsync(ws.p, 0, 64, s);
  cudaEventRecord(clk.e0, s);
  // the largest cluster the device accepts (16 non-portable, else 8), rows split evenly
  for (int nq : {kMaxCluster, 8}) {
    a.R = (n + nq - 1) / nq;
    const size_t dsm = (size_t)a.R * ds_row_bytes(W) + 16;
    if (dsm > kSmemBudget) { e = cudaErrorInvalidValue; continue; }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nq);
    cfg.blockDim = dim3(kST);
    cfg.dynamicSmemBytes = dsm;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = nq;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {&a};
    e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e == cudaSuccess) break;
    cudaGetLastError();
  }
  if (e == cudaSuccess) count_launch();
  cudaEventRecord(clk.e1, s);
  return solve_finish(e, clk, job.defer, 1, a.out_iters, a.out_status, a.out_relres, LC_KERNEL_PCG_RESIDENT, 1, s,
                      info, "PCG (cluster-resident) kernel");
}

}  // namespace lc
