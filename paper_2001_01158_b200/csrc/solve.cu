// solve.cu -- lc_solve_local / lc_solve_global: dispatch to the persistent
// Krylov kernels (pcg.cu, gmres.cu).
#include <algorithm>

#include "lc_internal.cuh"

namespace lc {
lc_status run_pcg(const PcgJob& job, const lc_solver_params* p, cudaStream_t s, lc_solve_info* info);
lc_status run_gmres(const Sell& M, const double* b, double* x, const int32_t* scatter_idx, double* x_full,
                    const double* x_init, const lc_solver_params* p, cudaStream_t s, lc_solve_info* info,
                    Pending* defer);

lc_status check_solver_params(const lc_solver_params* p) {
  if (!p) { set_error("solver params NULL"); return LC_ERR_INVALID_ARG; }
  if (!(p->rel_tol > 0) || p->max_iters < 0) { set_error("solver: need rel_tol > 0, max_iters >= 0"); return LC_ERR_INVALID_ARG; }
  if (p->method == LC_PCG) {
    if (p->precond != LC_JACOBI) { set_error("PCG uses LC_JACOBI"); return LC_ERR_INVALID_ARG; }
  } else if (p->method == LC_GMRES) {
    if (p->precond != LC_BLOCK_JACOBI && p->precond != LC_JACOBI) { set_error("GMRES: bad precond"); return LC_ERR_INVALID_ARG; }
    if (p->restart < 1 || p->restart > 40) { set_error("GMRES: restart in [1, 40]"); return LC_ERR_INVALID_ARG; }
  } else {
    set_error("solver: method must be LC_PCG or LC_GMRES");
    return LC_ERR_INVALID_ARG;
  }
  return LC_OK;
}

static lc_status run(const Sell& M, const double* b, double* x, const int32_t* scatter_idx, double* x_full,
                     const double* x_init, const lc_solver_params* p, cudaStream_t s, lc_solve_info* info,
                     int reg_units, int spg, Pending* defer) {
  if (p->method == LC_PCG) {
    PcgJob job;
    job.M = &M; job.b = b; job.x = x; job.x_init = x_init; job.scatter_idx = scatter_idx; job.x_full = x_full;
    job.reg_units = reg_units; job.spg = spg; job.defer = defer;
    return run_pcg(job, p, s, info);
  }
  return run_gmres(M, b, x, scatter_idx, x_full, x_init, p, s, info, defer);
}

// Alg. 1 l.5-6 (lc_solve_local; lc_local_method passes a Pending record and skips the checks it already made)
lc_status solve_local_impl(lc_sub S, const lc_solver_params* p, double* x, cudaStream_t stream, lc_solve_info* info,
                           Pending* defer) {
  if (S->K_units == 0) {   // empty Omega: x~ = x0 (R12)
    if (info)
      for (int g = 0; g < S->nseg; ++g) info[g] = lc_solve_info{0, LC_OK, 0.0, 0.0, LC_KERNEL_NONE, 1};
    return LC_OK;
  }
  Touch tS(S->use, (cudaStream_t)stream);
  if (S->masked) {
    if (lc_status cs = check_matrix(S->A, "lc_solve_local")) return cs;
    Touch tA(S->A->use, (cudaStream_t)stream);
    if (p->method != LC_PCG) {
      set_error("lc_solve_local: GMRES on a masked (stencil, block = 1) subsystem is not supported");
      return LC_ERR_INVALID_ARG;
    }
    const lc_matrix_s* A = S->A;
    PcgJob job;
    job.M = &A->A; job.b = S->bs; job.x_init = S->xm0; job.slist = S->slist; job.nlist_dev = S->nlist; job.lseg = S->lseg;
    // near-full domains: sweep all slices with the Omega mask instead of the list (contiguous, TMA-staged)
    if (A->batch == 1 && S->K_units * 10 >= A->n * 8) job.slist = nullptr;
    job.nlist_max = std::min<int64_t>(A->A.nslices, S->K_units);
    job.omega = S->omega; job.x_user = x;
    job.reg_units = A->seg_units; job.spg = (A->seg_units + 31) / 32;
    job.rows_hint = S->K_units;
    job.defer = defer;
    return run_pcg(job, p, (cudaStream_t)stream, info);
  }
  return run(S->B, S->bsub, nullptr, S->idx, x, S->xB0, p, (cudaStream_t)stream, info, 0, 0, defer);
}

// Alg. 1 l.8-11 / method0 (lc_solve_global)
lc_status solve_global_impl(lc_matrix A, const double* b, double* x, const lc_solver_params* p, cudaStream_t stream,
                            lc_solve_info* info, Pending* defer) {
  Touch tA(A->use, stream);
  return run(A->A, b, x, nullptr, nullptr, nullptr, p, stream, info, A->seg_units, (A->seg_units + 31) / 32, defer);
}
}  // namespace lc

using namespace lc;

extern "C" lc_status lc_solve_local(lc_sub S, const lc_solver_params* p, double* x, void* stream,
                                    lc_solve_info* info) {
  if (!S || !x) { set_error("lc_solve_local: null argument"); return LC_ERR_INVALID_ARG; }
  lc_status st = check_solver_params(p);
  if (st) return st;
  return solve_local_impl(S, p, x, (cudaStream_t)stream, info, nullptr);
}

extern "C" lc_status lc_solve_global(lc_matrix A, const double* b, double* x, const lc_solver_params* p, void* stream,
                                     lc_solve_info* info) {
  if (!A || !b || !x) { set_error("lc_solve_global: null argument"); return LC_ERR_INVALID_ARG; }
  lc_status st = check_solver_params(p);
  if (st) return st;
  if (lc_status cs = check_matrix(A, "lc_solve_global")) return cs;
  return solve_global_impl(A, b, x, p, (cudaStream_t)stream, info, nullptr);
}
