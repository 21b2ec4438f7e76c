// method.cu -- lc_local_method: Alg. 1 in one call.
//
// The same steps as the C-ABI sequence lc_select_domain -> lc_extract_sub -> lc_solve_local -> lc_smooth_gs ->
// lc_solve_global (and the same kernels), with the intermediate handles kept inside the library and the solve
// reports deferred: the Krylov launches copy their per-segment outputs into pinned host records behind
// themselves, so the host runs ahead of the device from the domain's K to the end and synchronises once there.
#include <map>
#include <new>
#include <vector>

#include "lc_internal.cuh"

namespace lc {
lc_status check_solver_params(const lc_solver_params* p);
lc_status solve_local_impl(lc_sub S, const lc_solver_params* p, double* x, cudaStream_t s, lc_solve_info* info,
                           Pending* defer);
lc_status solve_global_impl(lc_matrix A, const double* b, double* x, const lc_solver_params* p, cudaStream_t s,
                            lc_solve_info* info, Pending* defer);
lc_status domain_rows_out(const lc_domain_s* D, int32_t* idx_dev, cudaStream_t s);

namespace {
// per (host thread, device): two pinned solve records (local, global) and the phase events.  A call returns only
// after its final synchronisation, so one set per thread and device is never in use twice.  (Kept for the life of
// the process: a few hundred bytes of pinned memory and 10 events per host thread and device.)
struct MethodArena {
  Pending* pend = nullptr;        // pinned [2]
  cudaEvent_t ph[6] = {};
  bool ok = false;
};
thread_local std::map<int, MethodArena> t_arena;

lc_status arena(MethodArena** out) {
  int dev = 0;
  LC_CUDA(cudaGetDevice(&dev));
  MethodArena& a = t_arena[dev];
  if (!a.ok) {
    void* p = nullptr;
    LC_CUDA(cudaHostAlloc(&p, sizeof(Pending) * 2, cudaHostAllocPortable));
    a.pend = static_cast<Pending*>(p);
    for (int k = 0; k < 2; ++k) {
      new (&a.pend[k]) Pending();
      LC_CUDA(cudaEventCreate(&a.pend[k].e0));
      LC_CUDA(cudaEventCreate(&a.pend[k].e1));
    }
    for (auto& e : a.ph) LC_CUDA(cudaEventCreate(&e));
    a.ok = true;
  }
  *out = &a;
  return LC_OK;
}

// free a handle made inside the call: every use was on `s`, so its frees are ordered on `s` directly
void drop(lc_domain_s* D, cudaStream_t s) {
  if (!D) return;
  if (D->use.ev) cudaEventDestroy(D->use.ev);
  D->use.ev = nullptr;
  D->release(s);
  delete D;
}
void drop(lc_sub_s* S, cudaStream_t s) {
  if (!S) return;
  if (S->use.ev) cudaEventDestroy(S->use.ev);
  S->use.ev = nullptr;
  S->release(s);
  delete S;
}
}  // namespace
}  // namespace lc

using namespace lc;

extern "C" lc_status lc_local_method(lc_matrix A, const double* b, const double* x0, const lc_domain_params* dp,
                                     const lc_solver_params* sp, int32_t gs_sweeps, double* x, double* xt_dev,
                                     int32_t* idx_dev, void* stream, int64_t* K_host, lc_solve_info* local_info,
                                     lc_solve_info* global_info, lc_method_times* times) {
  if (!A || !b || !x0 || !x) { set_error("lc_local_method: null argument"); return LC_ERR_INVALID_ARG; }
  if (x == x0 || x == b) { set_error("lc_local_method: x may not alias b or x0"); return LC_ERR_INVALID_ARG; }
  if (gs_sweeps < 0) { set_error("lc_local_method: gs_sweeps < 0"); return LC_ERR_INVALID_ARG; }
  lc_status st = check_solver_params(sp);
  if (st) return st;
  if ((st = check_matrix(A, "lc_local_method"))) return st;
  const int G = A->batch;
  if (G > kMaxSegs) { set_error("lc_local_method: at most 64 segments"); return LC_ERR_DIMENSION; }
  MethodArena* ar = nullptr;
  if ((st = arena(&ar))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  Touch tA(A->use, s);
  Pending* pl = &ar->pend[0];
  Pending* pg = &ar->pend[1];
  pl->armed = pg->armed = 0;
  const int64_t len = A->n * A->block;
  cudaEventRecord(ar->ph[0], s);
  LC_CUDA(cudaMemcpyAsync(x, x0, sizeof(double) * len, cudaMemcpyDeviceToDevice, s));
  std::vector<int64_t> K(G, 0);
  lc_domain D = nullptr;
  lc_sub S = nullptr;
  bool local_ran = false;
  if (dp) {
    // l.2 (one synchronisation: K fixes the subsystem's representation, size and kernel)
    if ((st = lc_select_domain(A, b, x0, dp, stream, &D, K.data()))) return st;
    cudaEventRecord(ar->ph[1], s);
    if (idx_dev && (st = domain_rows_out(D, idx_dev, s))) { drop(D, s); return st; }
    if (D->K_units > 0) {
      // l.3-4
      if ((st = lc_extract_sub(A, D, b, x0, stream, &S))) { drop(D, s); return st; }
      cudaEventRecord(ar->ph[2], s);
      // l.5-6: xbar_B and x~ (Eq. 4) into x, report deferred
      st = solve_local_impl(S, sp, x, s, local_info, pl);
      if (st < 0) { drop(S, s); drop(D, s); return st; }
      local_ran = true;
    } else {
      cudaEventRecord(ar->ph[2], s);
    }
    cudaEventRecord(ar->ph[3], s);
    if (xt_dev) {
      cudaError_t e = cudaMemcpyAsync(xt_dev, x, sizeof(double) * len, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) { drop(S, s); drop(D, s); return cuda_fail(e, "lc_local_method: x~ copy"); }
    }
    // l.7
    if (gs_sweeps > 0 && (st = lc_smooth_gs(A, b, x, gs_sweeps, stream))) { drop(S, s); drop(D, s); return st; }
    cudaEventRecord(ar->ph[4], s);
    // the subsystem and the domain are done with: stream-ordered frees behind the local solve
    drop(S, s);
    drop(D, s);
  } else {
    for (int k = 1; k <= 4; ++k) cudaEventRecord(ar->ph[k], s);
    if (xt_dev) LC_CUDA(cudaMemcpyAsync(xt_dev, x0, sizeof(double) * len, cudaMemcpyDeviceToDevice, s));
  }
  // l.8-11 (Eq. 6 check at x~, else the global solve from x~); report deferred
  st = solve_global_impl(A, b, x, sp, s, global_info, pg);
  if (st < 0) {
    cudaStreamSynchronize(s);
    return st;
  }
  cudaEventRecord(ar->ph[5], s);
  LC_CUDA(cudaStreamSynchronize(s));   // the one synchronisation of the solves
  if (K_host)
    for (int g = 0; g < G; ++g) K_host[g] = K[g];
  lc_status st_local = LC_OK;
  if (local_ran) st_local = pending_info(*pl, local_info);
  else if (local_info)
    for (int g = 0; g < G; ++g) local_info[g] = lc_solve_info{0, LC_OK, 0.0, 0.0, LC_KERNEL_NONE, 1};
  const lc_status st_global = pending_info(*pg, global_info);
  if (times) {
    float ms[5] = {0, 0, 0, 0, 0};
    for (int k = 0; k < 5; ++k) cudaEventElapsedTime(&ms[k], ar->ph[k], ar->ph[k + 1]);
    times->select = ms[0]; times->extract = ms[1]; times->local = ms[2]; times->gs = ms[3]; times->global = ms[4];
  }
  if (st_local < 0) {
    set_error("lc_local_method: the local solve broke down (see local_info.status)");
    return st_local;
  }
  return st_global;
}
