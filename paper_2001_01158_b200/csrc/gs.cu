// gs.cu -- lc_smooth_gs: forward Gauss-Seidel sweeps in natural row order (Alg. 1 l.7, P:381-382;
// one sweep in the paper's runs), bit-exact with the sequential oracle.
//
// Natural-order GS is a sparse triangular sweep: row i needs the NEW values of its lower neighbours
// (j < i) and the OLD values of its upper neighbours.  The sweep runs sync-free:
//   - warps claim 32-row slices in increasing order from an atomic counter (dynamic ids => a warp
//     only ever waits on slices claimed before it, which are running: forward progress);
//   - lower neighbours in earlier slices are waited for on per-slice flags (ld.acquire / st.release);
//   - upper neighbours are read before the slice writes anything (a structurally symmetric pattern
//     guarantees that any later row coupled to this slice waits for its flag, so they are still old);
//   - dependencies inside the slice are resolved by stepping through the 32 lanes in order, the new
//     values passed through shared memory.
// Each row evaluates exactly the oracle's expression: acc = fma chain over stored j != i ascending,
// x_i = (b_i - acc) / a_ii.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "lc_internal.cuh"

namespace lc {

constexpr int kGST = 256;
constexpr int kGSW = kGST / 32;
constexpr int kGSMaxW = 16;   // slots gathered per row in registers (wider rows take the generic path)

template <int ST>
__global__ void __launch_bounds__(kGST) k_gs_sweep(SellView A, int reg_units, int spg, const double* __restrict__ b,
                                                   double* x, unsigned* flags, unsigned sweep, unsigned* counter,
                                                   unsigned* err) {
  __shared__ double xs[kGSW][32];
  __shared__ unsigned s_claim[kGSW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nu1 = A.nunits - 1;
  for (;;) {
    if (lane == 0) s_claim[warp] = atomicAdd(counter, 1u);
    __syncwarp();
    const int64_t s = s_claim[warp];
    __syncwarp();
    if (s >= A.nslices) break;
    const int64_t g = s / spg;
    const int64_t row0 = g * reg_units + 32 * (s - g * spg), end = (g + 1) * reg_units;
    const int64_t u = row0 + lane;
    const bool valid = u < end;
    const int64_t pl = (ST ? 32ll * A.vw * s : A.slice_ptr[s]) + lane;
    const int w = ST ? A.W : (int)((A.slice_ptr[s + 1] - (pl - lane)) >> 5);
    double av[kGSMaxW], yv[kGSMaxW];
    int64_t cv[kGSMaxW];
    double d = 0.0;
    // ---- phase 1: gather operands (wait for lower slices; read upper values before any write)
    if (valid) {
      for (int k = 0; k < w && k < kGSMaxW; ++k) {
        bool real = sv_real(A, k, u);
        int64_t c = real ? sv_col(A, pl, k, u) : u;
        cv[k] = real ? c : -1;
        av[k] = sv_val(A, pl, k, u);
        yv[k] = 0.0;
        if (!real) continue;
        if (c == u) { d = av[k]; continue; }
        if (c < row0) {                                   // lower neighbour in an earlier slice: wait
          const int64_t sc = (c - g * reg_units) / 32 + g * spg;
          unsigned spins = 0;
          while (ld_acquire_u32(&flags[sc]) != sweep) {
            if (++spins > (1u << 22)) { atomicOr(err, 1u); break; }
          }
          yv[k] = __ldcg(x + c);                          // L2 (coherent), not a possibly stale L1 line
        } else if (c > u) {
          yv[k] = x[c];                                   // upper neighbour: old value
        }
      }
    }
    __syncwarp();
    // ---- phase 2: lanes in order; intra-slice lower neighbours come from xs (this sweep's values)
    for (int t = 0; t < 32; ++t) {
      if (lane == t && valid) {
        double acc = 0.0;
        for (int k = 0; k < w && k < kGSMaxW; ++k) {
          const int64_t c = cv[k];
          if (c < 0 || c == u) continue;
          double y = (c >= row0 && c < u) ? xs[warp][c - row0] : yv[k];
          acc = __fma_rn(av[k], y, acc);
        }
        double xn = (b[u] - acc) / d;
        xs[warp][lane] = xn;
        x[u] = xn;
      }
      __syncwarp();
    }
    if (lane == 0) {
      __threadfence();
      st_release_u32(&flags[s], sweep);
    }
    __syncwarp();
    (void)nu1;
  }
}

// Level-scheduled sweep for regular-grid stencils (offsets {-nx ny, -nx, -1, 0, 1, nx, nx ny} or the 2-D
// subset): in natural order row (ix, iy, iz) depends only on rows with smaller ix + iy + iz, so the rows
// of one level L = ix + iy + iz are independent and the levels run in order, separated by a grid
// barrier (or __syncthreads for a single CTA).  Same per-row arithmetic as above (bit-exact).  x is read
// through L2 (__ldcg): values written by other CTAs in earlier levels must not come from a stale L1 line.
struct Grid3 { int nx, ny, nz; };
__global__ void __launch_bounds__(kGST) k_gs_levels(SellView A, int reg_units, int spg, Grid3 gr, int G,
                                                    const double* __restrict__ b, double* x, int sweeps,
                                                    GridBar* bar) {
  unsigned long long bar_epoch = 0;
  const int64_t plane = (int64_t)gr.nx * gr.ny;
  const int64_t pairs = (int64_t)gr.ny * gr.nz;         // (iy, iz) candidates per level and segment
  const int nlev = gr.nx + gr.ny + gr.nz - 2;
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
  for (int sw = 0; sw < sweeps; ++sw)
    for (int L = 0; L < nlev; ++L) {
      for (int64_t t = gt; t < pairs * G; t += gs) {
        const int g = (int)(t / pairs);
        const int64_t pr = t - (int64_t)g * pairs;
        const int iz = (int)(pr / gr.ny), iy = (int)(pr - (int64_t)iz * gr.ny);
        const int ix = L - iy - iz;
        if (ix < 0 || ix >= gr.nx) continue;
        const int64_t lu = ix + (int64_t)gr.nx * iy + plane * iz;
        const int64_t u = (int64_t)g * reg_units + lu;
        const int64_t s = (int64_t)g * spg + (lu >> 5);
        const int64_t pl = 32ll * A.vw * s + (lu & 31);
        double acc = 0.0, d = 0.0;
        for (int k = 0; k < A.W; ++k) {
          if (!((A.mask[u] >> k) & 1)) continue;
          const double a = sv_val(A, pl, k, u);
          const int64_t c = u + A.off[k];
          if (c == u) { d = a; continue; }
          acc = __fma_rn(a, __ldcg(x + c), acc);
        }
        x[u] = (b[u] - acc) / d;
      }
      if (gridDim.x == 1) __syncthreads();
      else grid_barrier(bar, bar_epoch);
    }
}

// Line-pipelined sweep for 2-D five-point grids (offsets {-nx, -1, 0, 1, nx}; the paper's heat model):
// lane l of warp w of CTA c owns grid line L = c kLB + 32 w + l (iy of segment g = L / ny) and walks it in
// natural order, skewed one step behind line L - 1: at warp step tau it updates ix = tau - l, whose NEW
// lower neighbour x(ix, iy - 1) line L - 1 produced one step earlier (a register shuffle inside the warp;
// across warps a shared-memory ring with progress counters; across CTAs global memory behind a progress
// word published with release semantics), whose NEW left neighbour is the lane's own previous value, and
// whose right / upper neighbours are still OLD.  The critical path is the nx + ny - 1 wavefront of
// natural-order GS; no block-wide barrier sits on it (a barrier per step would also wait for the
// prefetches).  Matrix values, b and the old neighbours are prefetched kPF steps ahead into registers.  Per
// row the oracle's expression in the slot (ascending column) order, so the sweep is bit-exact.
constexpr int kLB = 128;        // lines per CTA (4 warps)
constexpr int kLW = kLB / 32;
constexpr int kPF = 8;          // prefetch depth (steps)
constexpr int kPub = 16;        // cross-CTA progress publication period (steps), a multiple of kPF
constexpr int kRing = 256;      // cross-warp ring of boundary values (per warp)
__global__ void __launch_bounds__(kLB) k_gs_lines(SellView A, int reg_units, int spg, int nx, int ny, int G,
                                                  const double* __restrict__ b, double* x, unsigned* prog) {
  // warp w's lane-31 outputs, slot ix % kRing = (value, ix) written and read as one 16-byte shared access,
  // so the consumer validates the slot by its tag without a fence on the producer's critical path
  __shared__ __align__(16) double2 s_ring[kLW][kRing];
  __shared__ volatile int s_cons[kLW];         // warp w: its lane 0 has consumed ix < s_cons[w]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, c = blockIdx.x;
  if (lane == 0) s_cons[w] = 0;
  for (int i = threadIdx.x; i < kLW * kRing; i += kLB) (&s_ring[0][0])[i] = make_double2(0.0, __longlong_as_double(-1ll));
  __syncthreads();
  const int64_t L = (int64_t)c * kLB + threadIdx.x;
  const bool line_ok = L < (int64_t)ny * G;
  const int g = line_ok ? (int)(L / ny) : 0;
  const int iy = line_ok ? (int)(L - (int64_t)g * ny) : 0;
  const int64_t base = (int64_t)g * reg_units + (int64_t)nx * iy;      // row of (0, iy) in segment g
  double pa[kPF][5], pb[kPF], p3[kPF], p4[kPF];
  unsigned pm[kPF];
  const int64_t nu1 = (int64_t)reg_units * G - 1;
  // loads independent of each other and of the mask (holes hold 0, neighbour indices clamped), so nothing
  // in a step waits on a prefetch issued for a later step (in-order issue would stall at the first use)
  auto load = [&](int q, int ix) {                       // branch-free: out-of-range steps load row base
    const int ixc = (line_ok && ix >= 0 && ix < nx) ? ix : 0;
    const int64_t lu = (int64_t)nx * iy + ixc, u = base + ixc;
    const int64_t sl = (int64_t)g * spg + (lu >> 5);
    const int64_t pl = 32ll * A.vw * sl + (lu & 31);
    pm[q] = A.mask[u];
#pragma unroll
    for (int k = 0; k < 5; ++k) pa[q][k] = __ldg(A.val + pl + 32 * k);
    pb[q] = b[u];
    p3[q] = __ldcg(x + (u + 1 <= nu1 ? u + 1 : nu1));       // old right neighbour
    p4[q] = __ldcg(x + (u + nx <= nu1 ? u + nx : nu1));     // old upper neighbour (not updated yet)
  };
#pragma unroll
  for (int q = 0; q < kPF; ++q) load(q, q - lane);
  // warp 0 of CTA c > 0: the previous CTA's last line, fetched 32 values at a time once published
  double bv = 0.0;
  int bnd_lo = 0, bnd_hi = 0;                              // x(ix, iy0 - 1) for ix in [bnd_lo, bnd_hi) held by lane ix - bnd_lo
  const int64_t prev_row0 = __shfl_sync(0xffffffffu, base, 0) - nx;   // lane 0's lower line (if any)
  double xl = 0.0, last = 0.0;                              // own new value at ix - 1; output of the step
  const int nsteps = nx + 31;
  for (int tau0 = 0; tau0 < nsteps; tau0 += kPF) {
#pragma unroll
    for (int q = 0; q < kPF; ++q) {
      const int tau = tau0 + q;
      const int ix = tau - lane;
      const bool act = line_ok && ix >= 0 && ix < nx;
      double y0 = __shfl_up_sync(0xffffffffu, last, 1);   // line L - 1 at ix (lanes 1..31)
      if (w == 0) {                                        // previous CTA's last line (same segment)
        const bool need = __shfl_sync(0xffffffffu, act && (pm[q] & 1u) && ix >= bnd_hi, 0);
        if (need) {                                        // warp-uniform refill of the boundary window
          int pr = 0;
          if (lane == 0) {                                 // relaxed polling, one acquire fence after it
            while ((pr = (int)*(volatile unsigned*)(prog + c - 1)) <= tau) {
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
          }
          pr = __shfl_sync(0xffffffffu, pr, 0);
          bnd_lo = tau;
          bnd_hi = min(tau + 32, pr);
          bv = tau + lane < bnd_hi ? __ldcg(x + prev_row0 + tau + lane) : 0.0;
        }
        const double bw = __shfl_sync(0xffffffffu, bv, (tau - bnd_lo) & 31);
        if (lane == 0 && act && (pm[q] & 1u)) y0 = bw;
      } else if (lane == 0 && act && (pm[q] & 1u)) {       // previous warp's lane 31
        const unsigned a = (unsigned)__cvta_generic_to_shared(&s_ring[w - 1][ix % kRing]);
        long long vb, tg;
        do {
          asm volatile("ld.volatile.shared.v2.b64 {%0, %1}, [%2];" : "=l"(vb), "=l"(tg) : "r"(a));
        } while (tg != ix);
        y0 = __longlong_as_double(vb);
      }
      // the row update with selects instead of branches (the warp stays converged for the shuffles)
      const unsigned m = act ? pm[q] : 0u;
      double acc = 0.0;
      acc = (m & 1u) ? __fma_rn(pa[q][0], y0, acc) : acc;
      acc = (m & 2u) ? __fma_rn(pa[q][1], xl, acc) : acc;
      acc = (m & 8u) ? __fma_rn(pa[q][3], p3[q], acc) : acc;
      acc = (m & 16u) ? __fma_rn(pa[q][4], p4[q], acc) : acc;
      const double xn = act ? (pb[q] - acc) / pa[q][2] : 0.0;
      if (act) x[base + ix] = xn;
      xl = act ? xn : xl;
      if (lane == 31 && w < kLW - 1 && act) {              // hand the value to the next warp's lane 0
        while (ix - s_cons[w + 1] >= kRing) {
        }
        const unsigned a = (unsigned)__cvta_generic_to_shared(&s_ring[w][ix % kRing]);
        asm volatile("st.volatile.shared.v2.b64 [%0], {%1, %2};" ::"r"(a), "l"(__double_as_longlong(xn)),
                     "l"((long long)ix) : "memory");
      }
      last = xn;
      if (lane == 0) s_cons[w] = tau + 1;                  // (every step: a line that needs no values never blocks)
      load(q, tau + kPF - lane);                           // ring slot q now serves step tau + kPF
      __syncwarp();
    }
    // the CTA's last line publishes its progress for the next CTA's first line
    if (w == kLW - 1 && lane == 31 && ((tau0 / kPF) % (kPub / kPF) == kPub / kPF - 1 || tau0 + kPF >= nsteps)) {
      int done = tau0 + kPF - 31;                          // ix < done are written
      done = done < 0 ? 0 : (done > nx ? nx : done);
      __threadfence();
      st_release_u32(prog + c, (unsigned)done);
    }
  }
}

// every stored coupling of a stencil row must be a true grid neighbour (else the level schedule is invalid)
__global__ void k_check_grid(SellView A, int reg_units, Grid3 gr, int64_t n, unsigned* bad) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t lu = u % reg_units, plane = (int64_t)gr.nx * gr.ny;
  const int ix = (int)(lu % gr.nx), iy = (int)((lu / gr.nx) % gr.ny), iz = (int)(lu / plane);
  for (int k = 0; k < A.W; ++k) {
    if (!((A.mask[u] >> k) & 1)) continue;
    const int o = A.off[k];
    bool ok = o == 0 || (o == -1 && ix > 0) || (o == 1 && ix < gr.nx - 1) ||
              (o == -gr.nx && iy > 0) || (o == gr.nx && iy < gr.ny - 1) ||
              (gr.nz > 1 && o == -plane && iz > 0) || (gr.nz > 1 && o == plane && iz < gr.nz - 1);
    if (!ok) { atomicOr(bad, 1u); return; }
  }
}

// structural symmetry of a general (explicit-column) SELL pattern: every stored (u, v), v != u, has (v, u)
// stored.  The sync-free sweep relies on it (a later row coupled to this slice must wait for its flag).
__global__ void k_check_pattern_sym(SellView A, int64_t n, int reg_units, int spg, unsigned* bad) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  auto slot0 = [&](int64_t v) {
    const int64_t g = v / reg_units, lv = v - g * reg_units;
    return A.slice_ptr[g * spg + (lv >> 5)] + (lv & 31);
  };
  const int64_t pu = slot0(u);
  const int lu = A.rowlen[u];
  for (int k = 0; k < lu; ++k) {
    const int64_t v = A.col[pu + 32ll * k];
    if (v == u) continue;
    const int64_t pv = slot0(v);
    const int lv = A.rowlen[v];
    bool found = false;
    for (int q = 0; q < lv; ++q) found |= (A.col[pv + 32ll * q] == u);
    if (!found) { atomicOr(bad, 1u); return; }
  }
}

}  // namespace lc

using namespace lc;

extern "C" lc_status lc_smooth_gs(lc_matrix M, const double* b, double* x, int32_t sweeps, void* stream) {
  if (!M || !b || !x || sweeps < 0) { set_error("lc_smooth_gs: null argument or sweeps < 0"); return LC_ERR_INVALID_ARG; }
  if (M->block != 1) { set_error("lc_smooth_gs: needs block = 1"); return LC_ERR_INVALID_ARG; }
  if (lc_status cs = check_matrix(M, "lc_smooth_gs")) return cs;
  Touch tA(M->use, (cudaStream_t)stream);
  if (M->A.maxw > kGSMaxW) { set_error("lc_smooth_gs: rows longer than 16 entries are not supported"); return LC_ERR_PATTERN; }
  if (M->A.stencil) {   // structural symmetry of the stencil: the offset set must be symmetric
    for (int k = 0; k < M->A.maxw; ++k) {
      bool found = false;
      for (int l = 0; l < M->A.maxw; ++l) found |= (M->A.off[l] == -M->A.off[k]);
      if (!found) { set_error("lc_smooth_gs: pattern must be structurally symmetric"); return LC_ERR_PATTERN; }
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (!M->A.stencil && M->pattern_sym < 0) {     // general layout: check the pattern once per matrix
    DevBuf ws(s);
    lc_status st = ws.alloc(64);
    if (st) return st;
    LC_CUDA(cudaMemsetAsync(ws.p, 0, 64, s));
    k_check_pattern_sym<<<(unsigned)((M->n + 255) / 256), 256, 0, s>>>(view(M->A), M->n, M->seg_units,
                                                                          (M->seg_units + 31) / 32, (unsigned*)ws.p);
    LC_LAUNCHED();
    unsigned bad = 0;
    LC_CUDA(cudaMemcpyAsync(&bad, ws.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    M->pattern_sym = bad ? 0 : 1;
  }
  if (!M->A.stencil && M->pattern_sym == 0) {
    set_error("lc_smooth_gs: pattern must be structurally symmetric");
    return LC_ERR_PATTERN;
  }
  if (sweeps == 0) return LC_OK;
  const Sell& A = M->A;
  // ---- regular-grid stencil?  offsets {-(nx ny), -nx, -1, 0, 1, nx, nx ny} (3-D) or {-nx, -1, 0, 1, nx}
  Grid3 gr{0, 0, 0};
  if (A.stencil) {
    const int W = A.maxw;
    const int64_t su = M->seg_units;
    if (W == 5 && A.off[0] < -1 && A.off[1] == -1 && A.off[2] == 0 && A.off[3] == 1 && A.off[4] == -A.off[0]) {
      int nx = -A.off[0];
      if (su % nx == 0) gr = Grid3{nx, (int)(su / nx), 1};
    } else if (W == 7 && A.off[2] == -1 && A.off[3] == 0 && A.off[4] == 1 && A.off[5] == -A.off[1] &&
               A.off[6] == -A.off[0] && A.off[1] < -1 && A.off[0] < A.off[1] && (-A.off[0]) % (-A.off[1]) == 0) {
      int nx = -A.off[1], ny = (-A.off[0]) / nx;
      if (su % ((int64_t)nx * ny) == 0) gr = Grid3{nx, ny, (int)(su / ((int64_t)nx * ny))};
    }
  }
  if (gr.nx > 0) {
    DevBuf ws(s);
    lc_status st = ws.alloc(64);
    if (st) return st;
    LC_CUDA(cudaMemsetAsync(ws.p, 0, 64, s));
    unsigned bad = 0;
    k_check_grid<<<(unsigned)((M->n + 255) / 256), 256, 0, s>>>(view(A), M->seg_units, gr, M->n, (unsigned*)ws.p);
    count_launch();
    LC_CUDA(cudaMemcpyAsync(&bad, ws.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    if (bad) gr.nx = 0;
  }
  // 2-D five-point grid: line-pipelined sweep (lines of 128 per CTA, all CTAs co-resident)
  const int64_t glines = (int64_t)gr.ny * M->batch;
  int lines_ok = 0;
  if (gr.nx > 0 && gr.nz == 1 && tuning().gs_lines) {
    int64_t mc = 0;
    lc_status st = max_coresident((const void*)k_gs_lines, kLB, 0, &mc);
    if (st) return st;
    lines_ok = (glines + kLB - 1) / kLB <= mc;
  }
  if (lines_ok) {
    const int nCTA = (int)((glines + kLB - 1) / kLB);
    DevBuf wsb(s);
    lc_status st = wsb.alloc(sizeof(unsigned) * (size_t)nCTA * sweeps + 64);
    if (st) return st;
    void* ws = wsb.p;
    LC_CUDA(cudaMemsetAsync(ws, 0, sizeof(unsigned) * (size_t)nCTA * sweeps + 64, s));
    SellView V = view(A);
    const int spg = (M->seg_units + 31) / 32;
    int ru = M->seg_units, G = M->batch, nx = gr.nx, ny = gr.ny;
    for (int sw = 0; sw < sweeps; ++sw) {
      unsigned* prog = (unsigned*)ws + (size_t)nCTA * sw;
      void* args[] = {&V, &ru, (void*)&spg, &nx, &ny, &G, (void*)&b, &x, &prog};
      // cooperative: CTA c spins on CTA c - 1's progress, so all CTAs must be co-resident
      LC_CUDA(cudaLaunchCooperativeKernel((void*)k_gs_lines, dim3((unsigned)nCTA), dim3(kLB), args, 0, s));
      count_launch();
    }
    LC_CUDA(cudaStreamSynchronize(s));
    return LC_OK;
  }
  if (gr.nx > 0) {
    DevBuf wsb(s);
    lc_status st = wsb.alloc(sizeof(GridBar));
    if (st) return st;
    void* ws = wsb.p;
    LC_CUDA(cudaMemsetAsync(ws, 0, sizeof(GridBar), s));
    const int64_t work = (int64_t)gr.ny * gr.nz * M->batch;
    int per_sm = 0;
    LC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gs_levels, kGST, 0));
    int64_t nCTA = std::min<int64_t>((int64_t)std::max(per_sm, 1) * num_sms(), (work + kGST - 1) / kGST);
    if (nCTA < 1) nCTA = 1;
    SellView V = view(A);
    const int spg = (M->seg_units + 31) / 32;
    int ru = M->seg_units, G = M->batch;
    GridBar* bar = (GridBar*)ws;
    void* args[] = {&V, &ru, (void*)&spg, &gr, &G, (void*)&b, &x, &sweeps, &bar};
    LC_CUDA(cudaLaunchCooperativeKernel((void*)k_gs_levels, dim3((unsigned)nCTA), dim3(kGST), args, 0, s));
    count_launch();
    LC_CUDA(cudaStreamSynchronize(s));
    return LC_OK;
  }
  DevBuf wsb(s);
  const size_t fbytes = sizeof(unsigned) * (size_t)(A.nslices + 1);
  lc_status st = wsb.alloc(fbytes + 64 * (sweeps + 1));
  if (st) return st;
  void* ws = wsb.p;
  unsigned* flags = (unsigned*)ws;
  unsigned* counters = (unsigned*)((char*)ws + ((fbytes + 63) & ~(size_t)63));
  unsigned* err = counters + 16 * sweeps;
  LC_CUDA(cudaMemsetAsync(ws, 0, fbytes + 64 * (sweeps + 1), s));
  const int spg = (M->seg_units + 31) / 32;
  int per_sm = 0;
  void* fn = A.stencil ? (void*)k_gs_sweep<1> : (void*)k_gs_sweep<0>;
  LC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGST, 0));
  int64_t nCTA = std::min<int64_t>((int64_t)std::max(per_sm, 1) * num_sms(), (A.nslices + kGSW - 1) / kGSW);
  if (nCTA < 1) nCTA = 1;
  SellView V = view(A);
  for (int sw = 1; sw <= sweeps; ++sw) {
    if (A.stencil)
      k_gs_sweep<1><<<(unsigned)nCTA, kGST, 0, s>>>(V, M->seg_units, spg, b, x, flags, (unsigned)sw,
                                                    counters + 16 * (sw - 1), err);
    else
      k_gs_sweep<0><<<(unsigned)nCTA, kGST, 0, s>>>(V, M->seg_units, spg, b, x, flags, (unsigned)sw,
                                                    counters + 16 * (sw - 1), err);
    LC_LAUNCHED();
  }
  unsigned h_err = 0;
  LC_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  LC_CUDA(cudaStreamSynchronize(s));
  if (h_err) { set_error("lc_smooth_gs: dependency wait timed out"); return LC_ERR_CUDA; }
  return LC_OK;
}
