// heat.cu -- NEXT-2: the paper's own model workload end to end on the device:
//   lc_heat_assemble  backward-Euler / five-point Picard system of the 2-D nonlinear heat equation
//                     (kappa = T^3.5, T_l = 1, T_r = 1e-4, Neumann in y) at a Picard iterate;
//   lc_heat_run       Alg. 6: time steps x Picard iterations, each linear system solved by method0,
//                     method1 (Alg. 2) or method2 (Alg. 3) through the C-ABI, x0 = previous iterate,
//                     stop when ||T^{n+1,s+1} - T^{n+1,s}||_2 < picard_tol.
// Node placement and face rule as the oracle (or_heat_assemble): interior nodes x_p = (p+1) h,
// h = 1/(nx+1), Dirichlet ghost nodes at x = 0, 1, arithmetic-mean faces (R26), kappa(T) evaluated as
// T^k sqrt(T) (R38) -- the same IEEE operations in the same order, so the CSR is bit-identical.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <vector>

#include "lc_internal.cuh"

namespace lc {

__device__ __forceinline__ double kappa_pow(double t, int k) {
  double v = 1.0;
  for (int i = 0; i < k; ++i) v = v * t;
  return v * sqrt(t);
}

__global__ void k_heat_assemble(int nx, int ny, double dt, int khalf, double Tl, double Tr,
                                const double* __restrict__ Ts, const double* __restrict__ Told,
                                int64_t* __restrict__ rp, int32_t* __restrict__ ci, double* __restrict__ a,
                                double* __restrict__ b) {
  const int64_t n = (int64_t)nx * ny;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p = (int)(i % nx), q = (int)(i / nx);
  const double h = 1.0 / (nx + 1), lam = dt / (h * h);
  const double ki = kappa_pow(Ts[i], khalf);
  // closed-form row start: full y-rows before q, then nodes before p in row q
  const int wq = 5 - (q == 0) - (q == ny - 1);
  int64_t z = (int64_t)q * (5 * nx - 2) - (q > 0 ? nx : 0) + (int64_t)p * wq - (p > 0 ? 1 : 0);
  rp[i] = z;
  double diag = 0.0, rhs = Told[i];
  if (q > 0) { double kf = 0.5 * (ki + kappa_pow(Ts[i - nx], khalf)); ci[z] = (int32_t)(i - nx); a[z++] = -lam * kf; diag += kf; }
  if (p > 0) { double kf = 0.5 * (ki + kappa_pow(Ts[i - 1], khalf)); ci[z] = (int32_t)(i - 1); a[z++] = -lam * kf; diag += kf; }
  else { double kf = 0.5 * (ki + kappa_pow(Tl, khalf)); diag += kf; rhs += lam * kf * Tl; }
  const int64_t zd = z++;
  if (p < nx - 1) { double kf = 0.5 * (ki + kappa_pow(Ts[i + 1], khalf)); ci[z] = (int32_t)(i + 1); a[z++] = -lam * kf; diag += kf; }
  else { double kf = 0.5 * (ki + kappa_pow(Tr, khalf)); diag += kf; rhs += lam * kf * Tr; }
  if (q < ny - 1) { double kf = 0.5 * (ki + kappa_pow(Ts[i + nx], khalf)); ci[z] = (int32_t)(i + nx); a[z++] = -lam * kf; diag += kf; }
  ci[zd] = (int32_t)i;
  a[zd] = 1.0 + lam * diag;
  b[i] = rhs;
  if (i == n - 1) rp[n] = z;
}

// ||u - v||_2^2 partials (fixed-order two-level reduction)
constexpr int kNT = 256, kNB = 256;
__global__ void k_diff2_part(const double* __restrict__ u, const double* __restrict__ v, int64_t n,
                             double* __restrict__ part) {
  double a = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)kNT * gridDim.x) {
    double d = u[i] - v[i];
    a = __fma_rn(d, d, a);
  }
  a = warp_sum(a);
  __shared__ double sw[kNT / 32];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kNT / 32; ++w) t += sw[w];
    part[blockIdx.x] = t;
  }
}
__global__ void k_diff2_final(const double* __restrict__ part, int nb, double* out) {
  double a = 0.0;
  for (int i = threadIdx.x; i < nb; i += 32) a += part[i];
  a = warp_sum(a);
  if (threadIdx.x == 0) *out = a;
}

}  // namespace lc

using namespace lc;

extern "C" lc_status lc_heat_assemble(int32_t nx, int32_t ny, double dt, int32_t khalf, double t_left,
                                      double t_right, const double* Ts, const double* Told, int64_t* row_ptr,
                                      int32_t* col_idx, double* values, double* b, void* stream) {
  if (nx < 2 || ny < 2 || (int64_t)nx * ny > INT32_MAX / 8 || !(dt > 0) || khalf < 0 || !Ts || !Told || !row_ptr ||
      !col_idx || !values || !b || !(t_left > 0) || !(t_right > 0)) {
    set_error("lc_heat_assemble: need nx, ny >= 2, dt > 0, khalf >= 0, positive boundary values, non-null arrays");
    return LC_ERR_INVALID_ARG;
  }
  const int64_t n = (int64_t)nx * ny;
  k_heat_assemble<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(nx, ny, dt, khalf, t_left, t_right, Ts,
                                                                                Told, row_ptr, col_idx, values, b);
  LC_LAUNCHED();
  return LC_OK;
}

extern "C" lc_status lc_heat_run(const lc_heat_params* hp, double* T, int32_t* picard_per_step, double* eta_per_step,
                                 void* stream, lc_heat_report* rep) {
  if (!hp || !T) { set_error("lc_heat_run: null argument"); return LC_ERR_INVALID_ARG; }
  if (hp->method < 0 || hp->method > 2 || hp->steps < 0 || hp->picard_max < 1 || !(hp->picard_tol > 0)) {
    set_error("lc_heat_run: method in {0,1,2}, steps >= 0, picard_max >= 1, picard_tol > 0");
    return LC_ERR_INVALID_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int nx = hp->nx, ny = hp->ny;
  const int64_t n = (int64_t)nx * ny, nnz = 5 * n;
  lc_heat_report R;
  memset(&R, 0, sizeof(R));
  auto t0 = std::chrono::steady_clock::now();
  void* ws = nullptr;
  const size_t vb = ((sizeof(double) * n) + 255) & ~(size_t)255;
  const size_t bytes = sizeof(int64_t) * (n + 1) + 256 + sizeof(int32_t) * nnz + 256 + sizeof(double) * nnz + 256 +
                       4 * vb + sizeof(double) * (kNB + 1) + 256;
  lc_status st = dalloc(&ws, bytes, s);
  if (st) return st;
  char* w = (char*)ws;
  auto take = [&](size_t nb) { char* p = w; w += (nb + 255) & ~(size_t)255; return p; };
  int64_t* rp = (int64_t*)take(sizeof(int64_t) * (n + 1));
  int32_t* ci = (int32_t*)take(sizeof(int32_t) * nnz);
  double* val = (double*)take(sizeof(double) * nnz);
  double* b = (double*)take(sizeof(double) * n);
  double* Ts = (double*)take(sizeof(double) * n);
  double* Tn = (double*)take(sizeof(double) * n);
  double* part = (double*)take(sizeof(double) * (kNB + 1));
  lc_solver_params sp{LC_PCG, LC_JACOBI, 30, hp->rel_tol, 20000};
  lc_domain_params dp{};
  if (hp->method == 1) dp = lc_domain_params{LC_CRIT_GRADIENT, LC_THR_REL_MAX, hp->alpha, 0, 0};
  if (hp->method == 2) dp = lc_domain_params{LC_CRIT_RESIDUAL, LC_THR_PAPER, hp->rel_tol, hp->e_max, 0};
  const unsigned nbr = (unsigned)std::min<int64_t>(kNB, (n + kNT - 1) / kNT);
  lc_matrix A = nullptr;
#define CKH(x) do { st = (x); if (st < 0) goto done; } while (0)
#define CKHC(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { st = cuda_fail(_e, #x); goto done; } } while (0)
  for (int step = 0; step < hp->steps; ++step) {
    CKHC(cudaMemcpyAsync(Ts, T, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));      // T^{n+1,0} = T^n
    int sit = 0;
    double eta_step = 0.0;
    bool conv = false;
    while (sit < hp->picard_max && !conv) {
      CKH(lc_heat_assemble(nx, ny, hp->dt, hp->khalf, hp->t_left, hp->t_right, Ts, T, rp, ci, val, b, s));
      if (!A) CKH(lc_create_csr(n, 1, 1, rp, ci, val, 1, LC_FMT_SELL32, s, &A));   // pattern fixed for the run
      else CKH(lc_update_values(A, rp, ci, val, 1, s));
      CKHC(cudaMemcpyAsync(Tn, Ts, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));  // x0 = previous iterate
      lc_solve_info info;
      if (hp->method > 0) {                                                           // Alg. 1 l.2-7
        lc_domain D = nullptr;
        int64_t K = 0;
        st = lc_select_domain(A, b, Tn, &dp, s, &D, &K);
        if (st < 0) goto done;
        eta_step += (double)K / n;
        R.eta_sum += (double)K / n;
        if (K > 0) {
          lc_sub S = nullptr;
          st = lc_extract_sub(A, D, b, Tn, s, &S);
          if (st >= 0) st = lc_solve_local(S, &sp, Tn, s, &info);
          if (st >= 0) R.it_local += info.iterations;
          if (st == LC_NOT_CONVERGED) R.local_not_converged += 1;      // non-fatal (R18)
          lc_destroy_sub(S);
        }
        lc_destroy_domain(D);
        if (st < 0) goto done;
        if (hp->gs_sweeps > 0) {
          st = lc_smooth_gs(A, b, Tn, hp->gs_sweeps, s);
          if (st < 0) goto done;
        }
      }
      st = lc_solve_global(A, b, Tn, &sp, s, &info);                                 // Alg. 1 l.8-11
      if (st < 0) goto done;
      if (st == LC_NOT_CONVERGED) R.global_not_converged += 1;
      R.it_global += info.iterations;
      // Picard test ||T^{n+1,s+1} - T^{n+1,s}||_2 < tol
      k_diff2_part<<<nbr, kNT, 0, s>>>(Tn, Ts, n, part);
      count_launch();
      k_diff2_final<<<1, 32, 0, s>>>(part, (int)nbr, part + kNB);
      count_launch();
      double d2 = 0.0;
      CKHC(cudaMemcpyAsync(&d2, part + kNB, sizeof(double), cudaMemcpyDeviceToHost, s));
      CKHC(cudaStreamSynchronize(s));
      std::swap(Ts, Tn);
      ++sit;
      R.picard_total += 1;
      conv = sqrt(d2) < hp->picard_tol;
    }
    if (!conv) R.picard_max_hit += 1;
    if (picard_per_step) picard_per_step[step] = sit;
    if (eta_per_step) eta_per_step[step] = sit ? eta_step / sit : 0.0;
    CKHC(cudaMemcpyAsync(T, Ts, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    R.steps = step + 1;
  }
  st = LC_OK;
done:
  lc_destroy_matrix(A);
  dfree(ws, s);
  cudaStreamSynchronize(s);
  R.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (rep) *rep = R;
  return st < 0 ? st : (R.global_not_converged ? LC_NOT_CONVERGED : LC_OK);
#undef CKH
#undef CKHC
}
