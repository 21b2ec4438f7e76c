/*
 * lc.h -- C-ABI of liblc.so: the B200 (sm_100a) hot path of the local
 * character-based method for sequences of sparse solves A x = b
 * (Ye, An, Xu, arXiv 2001.01158; "P:a-b" = /root/reference/PAPER.md lines).
 *
 * The method (Alg. 1), input (A, x0, b) -> output x:
 *   lc_create_csr     A (Eq. 1) into the library's device layout
 *   lc_select_domain  Omega_local (Alg. 2 P:480-500 / Alg. 3)      Alg. 1 l.2
 *   lc_extract_sub    B, b_B - E x_C^(0) (Eq. 2-3)                 Alg. 1 l.3-4
 *   lc_solve_local    xbar_B, then x~ = Q (xbar_B; x_C^(0)) (Eq. 4) Alg. 1 l.5-6
 *   lc_solve_global   Eq. 6 check at x~, else the global solve from x~         Alg. 1 l.8-11
 *   (method0 of P:987 = lc_solve_global from x0.)
 *
 * Conventions (all entry points):
 *   - Plain pointers and sizes only.  "device" = a CUDA device pointer on the
 *     current device; "host" = ordinary host memory.  `stream` is a cudaStream_t
 *     passed as void* (NULL = legacy default stream); all device work of a call is
 *     enqueued on it.
 *   - Vectors b, x0, x are caller-owned DEVICE arrays of length n*block (f64).
 *     They are read (b, x0) or read and written (x) on `stream`; the library never
 *     frees them.  Inputs are never modified except `x`.
 *   - Handles (lc_matrix, lc_domain, lc_sub) own their device buffers until the
 *     matching lc_destroy_*; destroying NULL is a no-op.
 *   - Every call returns lc_status; no exception crosses the ABI.  On error the
 *     output handle is set to NULL and lc_last_error() returns a thread-local
 *     message describing the failure.
 *   - Synchronisation: a call returns once its host-visible outputs (K, tau,
 *     solve info) are ready; these are the only host<->device syncs of the path.
 *   - Indices are 0-based.  Column indices within a row must be strictly
 *     ascending (the canonical per-row order of all row sums, R22).
 *   - The library has no CPU fallback: without a usable sm_100 device every
 *     call fails with LC_ERR_CUDA.
 */
#ifndef LC_H
#define LC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LC_OK = 0,
  LC_NOT_CONVERGED = 1,      /* non-fatal: x holds the best iterate; see lc_solve_info */
  LC_ERR_INVALID_ARG = -1,   /* null pointer, bad enum, eps <= 0, alpha/theta not in [0,1], p not in (0,1) ... */
  LC_ERR_DIMENSION = -2,     /* n, block, batch inconsistent (n % batch, n/batch > 2^31 ...) */
  LC_ERR_PATTERN = -3,       /* columns unsorted / duplicated / out of range, or diagonal not stored */
  LC_ERR_ZERO_DIAGONAL = -4, /* Jacobi / block-Jacobi needs a_ii != 0 (an invertible 3x3 cell block) */
  LC_ERR_BREAKDOWN = -5,     /* PCG: p^T A p <= 0 (A not SPD) */
  LC_ERR_NONFINITE = -6,     /* NaN / Inf in a reduction */
  LC_ERR_CUDA = -7,          /* CUDA runtime error (message in lc_last_error) */
  LC_ERR_OOM = -8            /* device allocation failed */
} lc_status;

/* internal storage format of lc_create_csr */
enum { LC_FMT_SELL32 = 0 /* SELL-C-sigma, C = 32, sigma = 1 (row order kept) */ };
/* local-domain criterion (lc_domain_params.criterion) */
enum { LC_CRIT_RESIDUAL = 0 /* |r_i|, r = b - A x0 (Alg. 3 l.4) */,
       LC_CRIT_GRADIENT = 1 /* g_i of Eq. 5 on x0 */ };
/* threshold rule (lc_domain_params.threshold) */
enum { LC_THR_PAPER = 0      /* tau = eps ||b||_2 / sqrt(N) (Eq. 7), param = eps */,
       LC_THR_REL_MAX = 1    /* tau = theta * max_i c_i (Alg. 2 l.10), param = theta (= alpha) */,
       LC_THR_PERCENTILE = 2 /* tau = nearest-rank p-quantile of c (R14), param = p */ };
/* solver (lc_solver_params.method / precond) */
enum { LC_PCG = 0, LC_GMRES = 1 };
enum { LC_JACOBI = 0, LC_BLOCK_JACOBI = 1 };

typedef struct lc_matrix_s* lc_matrix;
typedef struct lc_domain_s* lc_domain;
typedef struct lc_sub_s* lc_sub;

/*
 * A (Eq. 1).  block = 1: n scalar rows, CSR row_ptr[n+1] (int64), col_idx[nnz]
 * (int32), values[nnz] (f64).  block = 3: n = number of cells (block rows),
 * row_ptr/col_idx are block-level and values holds 9 f64 per block, row-major;
 * unknowns are interleaved per cell.  batch = G >= 1: A is
 * block-diagonal with G equal independent segments of n/G rows (the G group
 * systems of multi-group diffusion, solved together); b and x stack the
 * segments.  inputs_on_device != 0: the three arrays are device pointers,
 * else host pointers.  The arrays are COPIED (the caller keeps ownership).
 * The pattern is validated on the device (sorted, unique, in range, diagonal
 * stored) -> LC_ERR_PATTERN; a zero diagonal (singular cell block) ->
 * LC_ERR_ZERO_DIAGONAL.  fmt must be LC_FMT_SELL32.
 */
lc_status lc_create_csr(int64_t n, int32_t block, int32_t batch, const int64_t* row_ptr, const int32_t* col_idx,
                        const double* values, int32_t inputs_on_device, int32_t fmt, void* stream, lc_matrix* A);

/*
 * New values for the SAME pattern A was created with (the systems of a time-step / Picard sequence share
 * their mesh): row_ptr / col_idx must equal the creation arrays (not re-validated), values
 * are copied into A's layout in place (host or device inputs as in lc_create_csr).  A zero diagonal ->
 * LC_ERR_ZERO_DIAGONAL; values that are no longer symmetric under the symmetric stencil layout ->
 * LC_ERR_PATTERN (recreate the matrix).  Syncs `stream`.
 */
lc_status lc_update_values(lc_matrix A, const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                           int32_t inputs_on_device, void* stream);

typedef struct {
  int32_t criterion;     /* LC_CRIT_* */
  int32_t threshold;     /* LC_THR_* */
  double param;          /* eps (> 0) | theta in [0,1] (0 => Omega) | p in (0,1) */
  int32_t expand_rounds; /* Alg. 3 E_max, residual criterion only; 0 = none; <= 64 */
  int32_t dilate_hops;   /* unconditional dilation by graph hops of A's pattern (R15); 0 = none */
} lc_domain_params;

/*
 * Omega_local (Alg. 1 l.2).  Per segment g: criterion c_u, threshold tau_g,
 * Omega_g = {u : c_u > tau_g} (strict, R10), then E_max expansion rounds of
 * Alg. 3 (admit neighbour j iff |r_j| + sum_{l in Omega} |a_jl x0_l| > tau, all
 * admissions of a round simultaneous, stop early when a round admits nothing)
 * and dilate_hops unconditional neighbour unions.  For block = 3 the unit is the
 * cell (R16): c = max of the three |r| components, cells enter whole; the
 * gradient criterion needs block = 1.  b, x0: device [n*block].
 * K_host (host, [batch]): number of scalar unknowns in Omega_g.  Syncs `stream`.
 */
lc_status lc_select_domain(lc_matrix A, const double* b, const double* x0, const lc_domain_params* p, void* stream,
                           lc_domain* dom, int64_t* K_host);

/*
 * Copy out Omega_local.  idx_dev (device, optional, [sum K]): the ascending
 * global scalar-row indices of Omega (segment by segment).  tau_host (host,
 * optional, [batch]).  crit_dev (device, optional, [n]): the per-unit criterion
 * c_u (|r| max over the cell, or g).  adm_dev (device, optional, [n]): per unit,
 * the Eq. 8 admission value of the last expansion round in which the unit was a
 * neighbour of Omega, NaN if never.  Syncs `stream`.
 */
lc_status lc_domain_export(lc_domain dom, int32_t* idx_dev, double* tau_host, double* crit_dev, double* adm_dev,
                           void* stream);

/*
 * B = A[Omega, Omega] in local numbering (Eq. 2; F and C are never formed),
 * b_sub = b_B - E x_C^(0) (Eq. 3; per row the fma chain over stored columns
 * outside Omega, ascending, then one subtraction), x_B0 = x0[Omega] and the
 * (block-)Jacobi inverse diagonal of B.  K = 0 gives an empty handle.
 * Representation (no effect on results): B is either materialised (SELL-32 over
 * the Omega rows) or, for stencil matrices, applied as A's stencil restricted to
 * Omega on vectors that vanish outside it ("masked"); K <= n/2 with K >= 65536
 * gets the materialised form, near-full and small domains the masked one
 * (DESIGN.md s5).  A masked handle refers to A's device
 * layout: destroy the sub handle before A.  Errors: LC_ERR_INVALID_ARG (null
 * handle / vectors), LC_ERR_OOM, LC_ERR_CUDA.
 */
lc_status lc_extract_sub(lc_matrix A, lc_domain dom, const double* b, const double* x0, void* stream, lc_sub* sub);

/*
 * Copy out what lc_extract_sub computed (Eq. 3), whatever the representation: bsub_dev, xB0_dev (device,
 * each optional, [sum K * block]) receive b_sub = b_B - E x_C^(0) and x_B0 = x0[Omega] in the order of
 * Omega (ascending global rows, segment by segment; the cell's 3 unknowns together for block = 3).  For
 * parity checks against the oracle's extraction.  Syncs `stream`.
 */
lc_status lc_sub_export(lc_sub sub, double* bsub_dev, double* xB0_dev, void* stream);

typedef struct {
  int32_t method;    /* LC_PCG (Jacobi-preconditioned CG, SPD systems) | LC_GMRES (right-preconditioned
                        block-Jacobi GMRES(restart) with CGS2, nonsymmetric block = 3 systems) */
  int32_t precond;   /* LC_JACOBI for LC_PCG; LC_BLOCK_JACOBI (3x3 cell blocks) for LC_GMRES */
  int32_t restart;   /* GMRES restart length (30); ignored by PCG; <= 40 */
  double rel_tol;    /* eps of Eq. 6: stop when ||b - A x||_2 <= eps ||b||_2 (absolute if b = 0) */
  int32_t max_iters; /* PCG: SpMVs with p; GMRES: Arnoldi steps.  Exceeding -> LC_NOT_CONVERGED */
} lc_solver_params;

typedef struct {
  int32_t iterations;       /* PCG SpMVs with p / cumulative GMRES Arnoldi steps (R30) */
  int32_t status;           /* LC_OK | LC_NOT_CONVERGED | LC_ERR_BREAKDOWN | LC_ERR_NONFINITE */
  double rel_residual;      /* ||b - A x||_2 / ||b||_2 of the returned x (true residual) */
  double seconds;           /* device time of the solve (CUDA events) */
  int32_t kernel;           /* which Krylov kernel ran (LC_KERNEL_*) */
  int32_t lazy_x_depth;     /* PCG: x updated every lazy_x_depth-th iteration (1 = every iteration) */
} lc_solve_info;

/* lc_solve_info.kernel */
enum { LC_KERNEL_NONE = 0      /* no launch (empty subsystem) */,
       LC_KERNEL_PCG_GRID = 1  /* cooperative persistent grid, one segment */,
       LC_KERNEL_PCG_CLUSTER = 2 /* one thread-block cluster (<= 512 slices) */,
       LC_KERNEL_PCG_RESIDENT = 3 /* cluster with the system resident in shared memory (<= ~30k rows) */,
       LC_KERNEL_PCG_LOCKSTEP = 4 /* batched, all active segments swept in lock step */,
       LC_KERNEL_PCG_TEAMS = 5    /* batched, one team of CTAs per segment */,
       LC_KERNEL_GMRES = 6,
       LC_KERNEL_PCG_DYNTEAMS = 7 /* batched, one team per active segment, re-teamed as segments converge */ };

/*
 * Alg. 1 l.5-6: solve B xbar_B = b_sub from x_B0 to ||b_sub - B xbar|| <= eps ||b_sub||
 * (R17), then x~: x[Omega] = xbar_B, the complement untouched (Eq. 4).
 * x: device [n*block], in = x0, out = x~.  info: host [batch] (per segment).
 * Returns the worst per-segment status (LC_NOT_CONVERGED is non-fatal, R18).
 */
lc_status lc_solve_local(lc_sub sub, const lc_solver_params* p, double* x, void* stream, lc_solve_info* info);

/*
 * Alg. 1 l.8-11 (and method0): r = b - A x; if Eq. 6 holds, 0 iterations; else
 * the Krylov solve of the whole system warm-started from x.  x: device, in/out.
 */
lc_status lc_solve_global(lc_matrix A, const double* b, double* x, const lc_solver_params* p, void* stream,
                          lc_solve_info* info);

/* device-stream time of each phase of lc_local_method (ms, CUDA events on `stream`; launches included) */
typedef struct {
  double select;    /* Alg. 1 l.2   (lc_select_domain) */
  double extract;   /* Alg. 1 l.3-4 (lc_extract_sub) */
  double local;     /* Alg. 1 l.5-6 (lc_solve_local: xbar_B and the assembly of x~) */
  double gs;        /* Alg. 1 l.7   (lc_smooth_gs) */
  double global;    /* Alg. 1 l.8-11 (lc_solve_global from x~) */
} lc_method_times;

/*
 * Alg. 1 in ONE call: input (A, b, x0), output x.  Same operations, kernels and results as the
 * sequence lc_select_domain -> lc_extract_sub -> lc_solve_local -> gs_sweeps x lc_smooth_gs (l.7, 0 = none,
 * R8) -> lc_solve_global, but the intermediate handles stay inside the library and the host synchronises twice
 * (after the domain, whose K fixes the subsystem's size and kernel; at the end, for the solve reports) instead
 * of after every step; lc_smooth_gs keeps its own syncs.  dp = NULL runs method0 (the global solve from
 * x0).  b, x0: device [n*block], read only.  x: device [n*block], out (may not alias b or x0).
 * Optional outputs (NULL = not wanted):
 *   xt_dev      device [n*block]: x~ of Eq. 4 before the GS sweeps and the global solve
 *   idx_dev     device [n*block]: Omega's ascending scalar rows (sum K entries, as lc_domain_export)
 *   K_host      host [batch]: |Omega| per segment (scalar unknowns; 0 for method0)
 *   local_info  host [batch]: the local solve per segment (iterations 0, kernel LC_KERNEL_NONE if K = 0)
 *   global_info host [batch]: the global solve per segment
 *   times       host: device time of each phase
 * Returns the global solve's status (LC_NOT_CONVERGED non-fatal), or the first error of any phase; a local
 * solve that stops at its cap is non-fatal (R18: it continues with the best iterate), see local_info.
 */
lc_status lc_local_method(lc_matrix A, const double* b, const double* x0, const lc_domain_params* dp,
                          const lc_solver_params* sp, int32_t gs_sweeps, double* x, double* xt_dev, int32_t* idx_dev,
                          void* stream, int64_t* K_host, lc_solve_info* local_info, lc_solve_info* global_info,
                          lc_method_times* times);

/*
 * y = A x (the operator of Eq. 1; the product inside the residual of Alg. 3 l.4, and inside every
 * Krylov iteration).  x, y: device [n*block], must not alias.  Per row the canonical chain (R22): stored
 * entries in ascending column order with explicit fma, so y equals the oracle's or_spmv bitwise.
 * Enqueued on `stream`, no sync.
 */
lc_status lc_spmv(lc_matrix A, const double* x, double* y, void* stream);

/*
 * y = A x straight from CSR device arrays (n rows, row_ptr [n+1] int64, col_idx / values [nnz]): the
 * row-slab CSR kernel (each warp's 32-row slab copied into shared memory with coalesced loads).
 * The handles keep the SELL / stencil layouts instead (faster on every config, profiles/
 * r01_ac); this entry point serves CSR data that is never converted.  Bit-exact with or_spmv (R22).
 * Enqueued on `stream`, no sync.
 */
lc_status lc_spmv_csr(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                      const double* x, double* y, void* stream);

/* storage layout chosen by lc_create_csr */
enum { LC_LAYOUT_SELL = 0     /* SELL-32 with explicit int32 column per slot (12 B per slot) */,
       LC_LAYOUT_STENCIL = 1  /* every row's column offsets lie in one sorted set of <= 16 offsets: values only,
                                 slot k = column row + off[k] (zero "holes" where a row lacks it), 8 B per slot */,
       LC_LAYOUT_SYMSTENCIL = 2 /* stencil layout of a bitwise-symmetric matrix (block 1): only the diagonal and
                                   upper-offset slots are stored; a_uv (v < u) is read as a_vu */ };
/*
 * Alg. 1 l.7 (one sweep in the paper's runs): `sweeps` forward Gauss-Seidel sweeps
 * in natural row order on A x = b, in place on x (device [n]): x_i <- (b_i - sum_{j != i} a_ij x_j) / a_ii
 * with the sum over stored j != i in ascending order (R22), j < i already updated.  Bit-exact with
 * the sequential definition.  Needs block = 1, rows of at most 16 entries and a structurally
 * symmetric pattern (LC_ERR_PATTERN otherwise).  Syncs `stream`.
 */
lc_status lc_smooth_gs(lc_matrix A, const double* b, double* x, int32_t sweeps, void* stream);

/* ---- NEXT-2: the paper's own model workload, the 2-D nonlinear heat equation ---- */

/*
 * Backward-Euler / five-point Picard system at the iterate Ts (Eq. picard-equs) on nx x ny
 * interior nodes x_p = (p+1)/(nx+1) (row i = p + nx q): kappa(T) = T^(khalf + 1/2) (paper: khalf = 3,
 * evaluated as T^khalf sqrt(T), R38), face kappa the arithmetic mean (R26), Dirichlet t_left
 * at x = 0 and t_right at x = 1, no flux at y = 0, 1:
 *   (1 + lam sum_f kf) T_i - lam sum_{interior f} kf T_nb = Told_i + lam sum_{boundary f} kf T_bnd,
 * lam = dt (nx+1)^2.  Device arrays: Ts, Told [nx ny]; outputs row_ptr [nx ny + 1], col_idx and values
 * [5 nx ny - 2 nx - 2 ny] (ascending columns), b [nx ny].  Enqueued on `stream`, no sync.
 */
lc_status lc_heat_assemble(int32_t nx, int32_t ny, double dt, int32_t khalf, double t_left, double t_right,
                           const double* Ts, const double* Told, int64_t* row_ptr, int32_t* col_idx, double* values,
                           double* b, void* stream);

typedef struct {
  int32_t nx, ny;        /* interior nodes (paper: 99 x 99) */
  double dt;             /* time step (paper: 1e-2) */
  int32_t khalf;         /* kappa = T^(khalf + 1/2) (paper: 3) */
  double t_left, t_right;/* Dirichlet values (paper: 1, 1e-4) */
  int32_t steps;         /* time steps (paper: 100) */
  double picard_tol;     /* ||T^{n+1,s+1} - T^{n+1,s}||_2 < picard_tol (paper: 1e-8) */
  int32_t picard_max;    /* Picard cap per step */
  int32_t method;        /* 0 = method0 (global PCG), 1 = method1 (Alg. 2), 2 = method2 (Alg. 3) */
  double alpha;          /* method1 alpha (paper: 1e-4) */
  int32_t e_max;         /* method2 E_max (paper: 1) */
  int32_t gs_sweeps;     /* Alg. 1 l.7 sweeps (paper: 1) */
  double rel_tol;        /* linear tolerance eps (paper: 1e-10); also eps of method2's tau */
} lc_heat_params;

typedef struct {
  int32_t steps, picard_total, picard_max_hit;
  int64_t it_local, it_global;   /* summed Krylov iterations */
  double eta_sum;                /* sum over linear solves of K / N */
  double seconds;                /* host wall time of the run */
  int32_t local_not_converged;   /* local solves that hit max_iters (non-fatal, R18) */
  int32_t global_not_converged;  /* global solves that hit max_iters: lc_heat_run then returns LC_NOT_CONVERGED */
} lc_heat_report;

/*
 * Alg. 6 on the device: T (device [nx ny]) in = T^0, out = T^steps.  Every Picard linear
 * system is assembled by lc_heat_assemble and solved by the selected method with x0 = the previous
 * Picard iterate.  picard_per_step / eta_per_step (host, optional, [steps]) receive the
 * Picard count and the mean eta of each step.  Syncs `stream` once per Picard iteration.  Returns
 * LC_NOT_CONVERGED (non-fatal, T still advanced) when any global linear solve hit its iteration cap.
 */
lc_status lc_heat_run(const lc_heat_params* p, double* T, int32_t* picard_per_step, double* eta_per_step,
                      void* stream, lc_heat_report* rep);

/* ---- NEXT-4: the row-partitioned multi-GPU form (Sec. 2.4, Alg. 4/5) ----
 *
 * A, b, x are partitioned by rows over p ranks: rank l owns the contiguous slab
 * I_l = [row0_l, row0_l + n_l), slabs ascending by rank and covering [0, N).  One lc_dist handle = one
 * rank's slab (its rows of A in the stencil layout, offsets relative to the slab) plus a workspace whose
 * iterate vectors and exchange block are PEER-VISIBLE (plain cudaMalloc, exportable by CUDA IPC).
 * The kernels read the neighbour slabs' halo rows directly from peer memory ("communicate all adjacency
 * components", Alg. 4 l.4 / Alg. 5 l.4, l.17) and perform every global reduction (Alg. 4 l.9, l.15,
 * Alg. 5 l.11, l.27, the Krylov dot products) as a fixed-order exchange through each rank's exchange block:
 * no NCCL call and no host round trip inside a phase; every rank obtains bitwise identical scalars.
 *
 * Two ways to run p ranks:
 *   - one process per GPU: each process creates its rank's handle, exports it (lc_dist_export_handle),
 *     the caller all-gathers the handles (e.g. torch.distributed) and calls lc_dist_connect; every compute
 *     call then takes ranks = &own handle, nr = 1, and all p processes must make the same calls in the same
 *     order (each rank's kernel waits for its peers' contributions);
 *   - emulation (p ranks on ONE device, one process): lc_dist_connect_local wires the handles together and
 *     every compute call takes all p handles (nr = p): ONE cooperative launch runs all ranks' CTAs, so the
 *     ranks' mutual waits are between co-resident CTAs (never separate launches waiting on each other).
 * Restrictions: block = 1, a constant-offset stencil (<= 8 offsets) in every slab (LC_ERR_PATTERN
 * otherwise), p <= 8, each slab at least as long as the stencil reach into it (checked at connect),
 * Jacobi-PCG solves, residual or gradient criterion with the paper / rel-max thresholds.
 */
typedef struct lc_dist_s* lc_dist;
enum { LC_DIST_MAX_RANKS = 8, LC_DIST_HANDLE_BYTES = 64 };

/*
 * Rank `rank` of `nranks`: rows [row0, row0 + n_local) of the n_global-row matrix A.  row_ptr [n_local + 1]
 * (int64, row_ptr[0] = 0), col_idx (int32, GLOBAL column numbers, strictly ascending per row, diagonal
 * stored) and values (f64); host arrays, or device arrays if inputs_on_device.  Copied.  Allocates the
 * rank's workspace (about 6 vectors of n_local f64 + n_local bytes).  Syncs `stream`.
 */
lc_status lc_dist_create(int64_t n_global, int64_t row0, int64_t n_local, int32_t rank, int32_t nranks,
                         const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                         int32_t inputs_on_device, void* stream, lc_dist* D);

/* CUDA IPC handle (LC_DIST_HANDLE_BYTES bytes, host) of the rank's peer-visible workspace */
lc_status lc_dist_export_handle(lc_dist D, void* handle);

/*
 * One process per rank: open every peer's workspace.  handles: host, nranks x LC_DIST_HANDLE_BYTES in rank
 * order (the own entry is ignored); n_local_all: host [nranks] slab lengths.  LC_ERR_DIMENSION when a
 * neighbour slab is shorter than the stencil reach into it.
 */
lc_status lc_dist_connect(lc_dist D, const void* handles, const int64_t* n_local_all);

/* Emulation: all nranks handles of this process (rank order, one device) see each other directly. */
lc_status lc_dist_connect_local(lc_dist* ranks, int32_t nranks);

/*
 * Alg. 4 (gradient) / Alg. 5 (residual) on the partition, followed by the masked
 * extraction of Eq. 3 (b_sub on Omega rows, x_B0 = x0 on Omega) for lc_dist_solve_local.  ranks: the nr
 * handles this call drives (see above); b, x0: host arrays of nr device pointers to each rank's slab
 * [n_local].  The threshold uses the GLOBAL ||b||_2 (double-double, R23) and N, or the global max of the
 * criterion; an expansion round stops when the GLOBAL admission count is 0 (R40), so Omega equals
 * the one lc_select_domain finds on the whole matrix.  Dilation hops as in lc_select_domain.  The percentile
 * threshold (R14) is the nearest-rank quantile over ALL ranks' rows: a radix select whose digit counts are
 * exchanged like the other reductions, so every rank holds bitwise lc_select_domain's tau.  K_global (host, optional): |Omega| over all ranks.  Syncs `stream`.
 */
lc_status lc_dist_select_domain(lc_dist* ranks, int32_t nr, const double* const* b, const double* const* x0,
                                const lc_domain_params* p, void* stream, int64_t* K_global);

/* The rank's domain flags: flag_dev (device, optional, [n_local]) = stage at which row row0 + i entered
   Omega (0 = criterion, 1.. = expansion / dilation round) or 255 = outside; tau_host (host, optional). */
lc_status lc_dist_domain_export(lc_dist D, uint8_t* flag_dev, double* tau_host, void* stream);

/*
 * Alg. 1 l.5-6 on the partition: Jacobi-PCG on B xbar = b_sub from x_B0 (the state lc_dist_select_domain
 * left in the handles), tolerance eps ||b_sub||_2 (global), then x~[Omega] = xbar (Eq. 4).  x: host array of
 * nr device pointers (in = x0 slab, out = x~ slab).  info (host, optional): the global iteration count,
 * status and relative residual (identical on every rank).  K = 0: no-op with 0 iterations.  Syncs `stream`.
 */
lc_status lc_dist_solve_local(lc_dist* ranks, int32_t nr, const lc_solver_params* p, double* const* x, void* stream,
                              lc_solve_info* info);

/* Alg. 1 l.8-11 / method0 on the partition: Jacobi-PCG on A x = b from x (b, x: host arrays of nr device
   pointers to the slabs; x in/out).  p->method must be LC_PCG.  Syncs `stream`. */
lc_status lc_dist_solve_global(lc_dist* ranks, int32_t nr, const double* const* b, double* const* x,
                               const lc_solver_params* p, void* stream, lc_solve_info* info);

void lc_dist_destroy(lc_dist D);

/* ---- tuning: kernel / layout choices that never change results beyond the parity bars ----
 *
 * Every field selects between implementations of the SAME operation (all of them parity-tested against the
 * oracle); the defaults are what the library picks on its own.  The setting belongs to the CALLING HOST
 * THREAD (thread-local; a new thread starts with the defaults) and is read when a call is made: layout
 * choices when the matrix / subsystem is created, kernel choices when a solve is launched.  No environment
 * variable is consulted anywhere in the library.
 */
typedef struct {
  int32_t stencil_layout;       /* 1 (default): constant-offset stencils are stored without column indices
                                   (LC_LAYOUT_STENCIL); 0: always SELL-32 with explicit columns */
  int32_t symmetric_layout;     /* 0 (default); 1: bitwise-symmetric stencils store diagonal + upper slots */
  int32_t pcg_cluster_resident; /* stencil systems of <= ~27k rows run a PCG whose matrix and vectors stay in the
                                   shared memory of one thread-block cluster.  2 (default): the single-reduction
                                   form (Chronopoulos-Gear recurrences, one cluster barrier per iteration; the same
                                   iterates in exact arithmetic, the parity bars hold); 1: the textbook two-reduction
                                   order (bitwise the grid kernels' arithmetic, <= ~30k rows); 0: never */
  int32_t pcg_cluster;          /* 1 (default): single-segment solves of <= 512 slices launch as ONE cluster with
                                   hardware cluster barriers; 0: always the cooperative grid */
  int32_t pcg_tma;              /* 1 (default): TMA bulk-copy ring for the value stream of contiguous solves */
  int32_t lazy_x_depth;         /* 3 (default) or 2: x updated every 3rd / 2nd PCG iteration (same roundings,
                                   DESIGN.md s6); 0 or 1: every iteration */
  int32_t batched_schedule;     /* -1 (default) automatic, 0 lock step, 1 static teams, 2 dynamic teams (batched
                                   PCG, G > 1; dynamic teams need equal segments without a slice list) */
  int32_t pcg_max_ctas;         /* 0 (default): occupancy x SMs; > 0 caps the grid of the PCG kernels */
  int32_t sub_repr;             /* -1 (default) automatic, 0 explicit SELL B, 1 masked on A's stencil layout */
  int32_t gmres_exact_cgs2;     /* 0 (default): Gram-form CGS2 (R39); 1: the textbook two passes */
  int32_t gs_lines;             /* 1 (default): 2-D five-point grids take the line-pipelined GS sweep; 0: the
                                   level schedule */
  int32_t spmv_csr_tma;         /* 1 (default): lc_spmv_csr stages its row chunks by TMA when the three CSR arrays
                                   are 16-byte aligned; 0: the warp row-slab kernel */
  int32_t spmv_tma;             /* 1 (default): lc_spmv stages the SELL-32 slice stream by TMA (block 1); 2: the
                                   stencil layouts (5 / 7 slots) too (slower there); 0: plain loads */
  int32_t batched_cluster;      /* 0 (default): batched lock-step PCG reduces through the two-level reducing
                                   barrier; 2..16: launched in clusters of that many CTAs, reductions through
                                   distributed shared memory + one counter level (measured no faster in situ,
                                   profiles/r02_e_batched_reduce.md) */
  int32_t block_dcoup;          /* 1 (default): block 3 stencil matrices whose off-diagonal blocks are diagonal (the
                                   3T couplings) keep a compact copy without those blocks' explicit zeros for the
                                   GMRES SpMVs (21 instead of 45 values per cell, bitwise the same chains); 0: no */
  int32_t l2_stream_hint;       /* -1 (default): the PCG kernels load the matrix stream (values, columns) with the L2
                                   evict_first policy when the solve's working set exceeds L2 while its vectors
                                   are at most twice L2 (they then stay cached between passes); 0: never; 1: always.
                                   Cache policy only: results are bitwise the same */
} lc_tuning;

/* the defaults listed above (host output) */
void lc_tuning_defaults(lc_tuning* t);
/* set the calling thread's tuning (NULL = defaults); LC_ERR_INVALID_ARG for out-of-range fields */
lc_status lc_set_tuning(const lc_tuning* t);
/* the calling thread's tuning (host output) */
lc_status lc_get_tuning(lc_tuning* t);

/* introspection (host outputs, each optional): unknowns n*block, stored scalars, batch, SELL slices, max row
   length (slots), layout (LC_LAYOUT_*), bytes one SpMV streams for the matrix (values + columns + metadata; for
   block 3 stencil matrices with diagonal coupling blocks, the compact copy the GMRES SpMVs read) */
lc_status lc_matrix_info(lc_matrix A, int64_t* n_unknowns, int64_t* nnz, int32_t* batch, int64_t* nslices,
                         int32_t* max_row, int32_t* layout, int64_t* matrix_bytes);

void lc_destroy_matrix(lc_matrix A);
void lc_destroy_domain(lc_domain dom);
void lc_destroy_sub(lc_sub sub);

/* thread-local message of the last failing call on this thread ("" if none) */
const char* lc_last_error(void);

/* number of CUDA kernels this library has launched in the process (for the bench's gpu_launches) */
int64_t lc_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* LC_H */
