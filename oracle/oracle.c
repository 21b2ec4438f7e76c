/*
 * oracle.c -- plain, slow, single-threaded CPU oracle of the local
 * character-based method (Ye, An, Xu, arXiv 2001.01158).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.  The
 * product path (paper_2001_01158_b200/) never imports, links or calls it, and
 * this file shares no code, header, helper or constant with the CUDA path.
 *
 * Compiled with  -O2 -ffp-contract=off  (no fast-math, no implicit
 * contraction): every fused multiply-add below is an explicit fma() call.
 *
 * Citations: "P:a-b" = /root/reference/PAPER.md lines; equation numbers as in
 * SURVEY.md s0 (Eq.1 A x = b P:193-200, Eq.2 partition P:267-288, Eq.3
 * subsystem P:349-353, Eq.4 assembly P:355-366, Eq.5 gradient P:440-445,
 * Eq.6 criterion P:521-526, Eq.7 bad points P:562-571, Eq.8 bound P:625-630).
 * "Rxx" = the reading of an ambiguous passage listed in DESIGN.md s3.
 *
 * Matrices are CSR with scalar rows: row_ptr int64[n+1], col int32[nnz]
 * (ascending, unique, diagonal stored), val f64[nnz].  Block (3x3 BSR)
 * systems are handed to the oracle expanded to scalar CSR (or_bsr_to_csr),
 * whose ascending scalar-column order is the canonical per-row order (R22).
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (paper values of Example 1 / Table 1, closed forms, brute force, dense LU,
 * invariants).  No function is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define OR_OK 0
#define OR_NOT_CONVERGED 1
#define OR_ERR_INVALID_ARG (-1)
#define OR_ERR_ZERO_DIAGONAL (-4)
#define OR_ERR_BREAKDOWN (-5)
#define OR_ERR_NONFINITE (-6)
#define OR_ERR_OOM (-8)

/* ------------------------------------------------------------------------ */
/* Sparse primitives                                                        */
/* ------------------------------------------------------------------------ */

/* y = A x, per-row fma chain over stored entries in ascending column order (R22). */
void or_spmv(int64_t n, const int64_t* rp, const int32_t* ci, const double* a, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) acc = fma(a[k], x[ci[k]], acc);
    y[i] = acc;
  }
}

/* r = b - A x: "Compute the initial residual r_i = b_i - sum_j a_ij x_j" (Alg. 3 l.4);
   acc is the R22 fma chain, then one subtraction. */
void or_residual(int64_t n, const int64_t* rp, const int32_t* ci, const double* a, const double* b,
                 const double* x, double* r) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) acc = fma(a[k], x[ci[k]], acc);
    r[i] = b[i] - acc;
  }
}

/* ||v||_2 with sum v_i^2 accumulated in double-double (TwoProd via fma, TwoSum),
   rounded to f64, then sqrt (R23).  Used for ||b||_2 in tau = eps ||b||_2 / sqrt(N) (Eq. 7). */
double or_norm2(int64_t n, const double* v) {
  double hi = 0.0, lo = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double p = v[i] * v[i];
    double pe = fma(v[i], v[i], -p);          /* TwoProd error */
    double s = hi + p;                        /* TwoSum(hi, p) */
    double bp = s - hi;
    double se = (hi - (s - bp)) + (p - bp);
    hi = s;
    lo = lo + (se + pe);
  }
  double s = hi + lo;
  return sqrt(s);
}

/* plain sequential dot product (Krylov dots, R24) */
static double dot(int64_t n, const double* x, const double* y) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s = fma(x[i], y[i], s);
  return s;
}

/* Eq. 5: g_i = sum_{j : a_ij stored} |x_i - x_j|, ascending j, plain adds;
   the j = i term is |x_i - x_i| = 0 and is skipped. */
void or_gradient(int64_t n, const int64_t* rp, const int32_t* ci, const double* x, double* g) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      int64_t j = ci[k];
      if (j == i) continue;
      acc = acc + fabs(x[i] - x[j]);
    }
    g[i] = acc;
  }
}

/* Expand a 3x3-block BSR matrix (block row ptr, block cols, 9 f64 per block row-major)
   to scalar CSR.  Scalar row 3c+alpha lists blocks ascending, beta ascending. */
void or_bsr_to_csr(int64_t nb, const int64_t* brp, const int32_t* bci, const double* bval, int64_t* rp,
                   int32_t* ci, double* a) {
  int64_t k = 0;
  for (int64_t c = 0; c < nb; ++c)
    for (int al = 0; al < 3; ++al) {
      rp[3 * c + al] = k;
      for (int64_t t = brp[c]; t < brp[c + 1]; ++t)
        for (int be = 0; be < 3; ++be) {
          ci[k] = 3 * bci[t] + be;
          a[k] = bval[9 * t + 3 * al + be];
          ++k;
        }
    }
  rp[3 * nb] = k;
}

/* ------------------------------------------------------------------------ */
/* Local-domain construction (Alg. 2, Alg. 3, Eq. 7, Eq. 8)                  */
/* ------------------------------------------------------------------------ */

typedef struct {
  int32_t criterion;     /* 0 = residual (Alg. 3), 1 = gradient (Alg. 2) */
  int32_t threshold;     /* 0 = paper tau = eps ||b||/sqrt(N) (Eq. 7); 1 = rel-max theta * max c (Alg. 2);
                            2 = nearest-rank percentile (R14) */
  double param;          /* eps | theta (= alpha) | p */
  int32_t expand_rounds; /* Alg. 3 E_max */
  int32_t dilate_hops;   /* unconditional neighbour dilation (R15) */
  int32_t cell;          /* unknowns per cell: 1, or 3 for cell-granular 3T domains (R16) */
} or_domain_params;

typedef struct {
  int32_t rounds;        /* expansion rounds executed (including the one that admitted nothing) */
  int64_t front[64];     /* |N| per round (Alg. 3 l.11) */
  int64_t admitted[64];  /* K_0 per round (Alg. 3 l.13-18) */
  int64_t K_after[64];   /* K after the round */
  int64_t K_base;        /* K after the bad-point / threshold step */
} or_trace;

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* cell u is adjacent to a marked cell: exists stored (row of u, l), cell(l) in Omega, cell(l) != u */
static int touches(int64_t u, int cell, const int64_t* rp, const int32_t* ci, const uint8_t* inO) {
  for (int al = 0; al < cell; ++al) {
    int64_t i = u * cell + al;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      int64_t v = ci[k] / cell;
      if (v != u && inO[v]) return 1;
    }
  }
  return 0;
}

/*
 * Omega_local selection.  Outputs:
 *   flag[n]  (per scalar row, 1 = in Omega_local); K = number of scalar rows in Omega;
 *   crit[m]  per unit (m = n / cell): the base criterion c_u (|r| max over the cell, or g);
 *   adm[m]   the admission value |r_j| + sum_l |a_jl x0_l| of the LAST expansion round in which
 *            unit u was a neighbour (NaN if never);
 *   tau      the threshold.
 */
int or_select_domain(int64_t n, const int64_t* rp, const int32_t* ci, const double* a, const double* b,
                     const double* x0, const or_domain_params* p, uint8_t* flag, double* crit, double* adm,
                     double* tau_out, int64_t* K_out, or_trace* tr) {
  int cell = p->cell;
  if (cell != 1 && cell != 3) return OR_ERR_INVALID_ARG;
  if (n % cell) return OR_ERR_INVALID_ARG;
  if (p->criterion == 1 && cell != 1) return OR_ERR_INVALID_ARG;
  if (p->expand_rounds < 0 || p->expand_rounds > 64 || p->dilate_hops < 0) return OR_ERR_INVALID_ARG;
  if (p->threshold == 0 && !(p->param > 0)) return OR_ERR_INVALID_ARG;
  if (p->threshold == 1 && !(p->param >= 0 && p->param <= 1)) return OR_ERR_INVALID_ARG;
  if (p->threshold == 2 && !(p->param > 0 && p->param < 1)) return OR_ERR_INVALID_ARG;
  if (p->expand_rounds > 0 && p->criterion != 0) return OR_ERR_INVALID_ARG; /* Alg. 3 only */
  int64_t m = n / cell;
  double* r = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  uint8_t* inO = (uint8_t*)calloc((size_t)(m ? m : 1), 1);
  uint8_t* add = (uint8_t*)calloc((size_t)(m ? m : 1), 1);
  if (!r || !inO || !add) { free(r); free(inO); free(add); return OR_ERR_OOM; }
  memset(tr, 0, sizeof(*tr));

  /* ---- criterion c_u ---- */
  if (p->criterion == 0) {
    or_residual(n, rp, ci, a, b, x0, r);                         /* Alg. 3 l.4 */
    for (int64_t u = 0; u < m; ++u) {
      double c = 0.0;
      for (int al = 0; al < cell; ++al) { double v = fabs(r[u * cell + al]); if (v > c) c = v; }
      crit[u] = c;                                                /* |r_i| (max over a cell, R16) */
    }
  } else {
    or_gradient(n, rp, ci, x0, crit);                             /* Alg. 2 l.4, Eq. 5 */
  }
  for (int64_t u = 0; u < m; ++u) adm[u] = NAN;

  /* ---- threshold ---- */
  double tau; int full = 0;
  if (p->threshold == 0) {
    /* Eq. 7: tau = eps ||b||_2 / sqrt(N), N = number of scalar unknowns */
    tau = p->param * or_norm2(n, b) / sqrt((double)n);
  } else if (p->threshold == 1) {
    /* Alg. 2 l.5-8 and l.10: tau = alpha * g_max; alpha = 0 => Omega (R11) */
    double cmax = 0.0;
    for (int64_t u = 0; u < m; ++u) if (crit[u] > cmax) cmax = crit[u];
    tau = p->param * cmax;
    if (p->param == 0.0) full = 1;
  } else {
    /* R14: nearest-rank percentile, tau = sorted(c)[ceil(p m) - 1] */
    double* s = (double*)malloc(sizeof(double) * (size_t)(m ? m : 1));
    memcpy(s, crit, sizeof(double) * (size_t)m);
    qsort(s, (size_t)m, sizeof(double), cmp_double);
    int64_t k = (int64_t)ceil(p->param * (double)m) - 1;
    if (k < 0) k = 0;
    if (k >= m) k = m - 1;
    tau = m ? s[k] : 0.0;
    free(s);
  }

  /* ---- bad points / gradient marking: c_u > tau, strict (R10) ---- */
  for (int64_t u = 0; u < m; ++u) inO[u] = full ? 1 : (crit[u] > tau);
  int64_t Kc = 0;
  for (int64_t u = 0; u < m; ++u) Kc += inO[u];
  tr->K_base = Kc * cell;

  /* ---- Alg. 3 l.10-24: expansion rounds (admissions simultaneous; r never recomputed) ---- */
  for (int rd = 0; rd < p->expand_rounds; ++rd) {
    int64_t nf = 0, na = 0;
    for (int64_t u = 0; u < m; ++u) {
      add[u] = 0;
      if (inO[u] || !touches(u, cell, rp, ci, inO)) continue;   /* u in N (l.11) */
      ++nf;
      double best = 0.0;
      for (int al = 0; al < cell; ++al) {
        int64_t j = u * cell + al;
        double s = 0.0;                                          /* sum_{l in Omega} |a_jl x0_l| */
        for (int64_t k = rp[j]; k < rp[j + 1]; ++k) {
          int64_t l = ci[k];
          if (inO[l / cell]) s = s + fabs(a[k] * x0[l]);
        }
        double v = fabs(r[j]) + s;                               /* Eq. 8 left side */
        if (al == 0 || v > best) best = v;
      }
      adm[u] = best;
      if (best > tau) { add[u] = 1; ++na; }                      /* l.14 */
    }
    tr->front[rd] = nf * cell; tr->admitted[rd] = na * cell;
    tr->rounds = rd + 1;
    if (na == 0) { tr->K_after[rd] = Kc * cell; break; }         /* l.22 break */
    for (int64_t u = 0; u < m; ++u) if (add[u]) inO[u] = 1;
    Kc += na;
    tr->K_after[rd] = Kc * cell;
  }

  /* ---- R15: unconditional dilation by d graph hops ---- */
  for (int hop = 0; hop < p->dilate_hops; ++hop) {
    for (int64_t u = 0; u < m; ++u) add[u] = (!inO[u] && touches(u, cell, rp, ci, inO));
    for (int64_t u = 0; u < m; ++u) if (add[u]) { inO[u] = 1; ++Kc; }
  }

  for (int64_t u = 0; u < m; ++u)
    for (int al = 0; al < cell; ++al) flag[u * cell + al] = inO[u];
  *K_out = Kc * cell;
  *tau_out = tau;
  free(r); free(inO); free(add);
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Extraction (Eq. 2, Eq. 3) and assembly (Eq. 4)                            */
/* ------------------------------------------------------------------------ */

/*
 * Given flag[n] (Omega_local), build:
 *   idx[K]     = i_1 < ... < i_K (Q as an index map, R7),
 *   B          = A[Omega, Omega] in local numbering, CSR (Brp[K+1], Bci, Ba; capacity nnz(A)),
 *   bsub[K]    = b_B - E x_C^(0): b_i - (fma chain over stored j not in Omega, ascending) (Eq. 3),
 *   xB0[K]     = x0[Omega].
 */
int or_extract(int64_t n, const int64_t* rp, const int32_t* ci, const double* a, const double* b,
               const double* x0, const uint8_t* flag, int64_t* idx, int64_t* Brp, int32_t* Bci, double* Ba,
               double* bsub, double* xB0, int64_t* K_out, int64_t* Bnnz_out) {
  int64_t* inv = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  if (!inv) return OR_ERR_OOM;
  int64_t K = 0;
  for (int64_t i = 0; i < n; ++i) inv[i] = flag[i] ? K++ : -1;
  int64_t z = 0;
  for (int64_t i = 0, l = 0; i < n; ++i) {
    if (!flag[i]) continue;
    idx[l] = i;
    Brp[l] = z;
    double acc = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      int64_t j = ci[k];
      if (inv[j] >= 0) { Bci[z] = (int32_t)inv[j]; Ba[z] = a[k]; ++z; }   /* B block */
      else acc = fma(a[k], x0[j], acc);                                    /* E x_C^(0) */
    }
    bsub[l] = b[i] - acc;
    xB0[l] = x0[i];
    ++l;
  }
  Brp[K] = z;
  *K_out = K; *Bnnz_out = z;
  free(inv);
  return OR_OK;
}

/* Eq. 4: x~ = Q (xbar_B ; x_C^(0)) -- overwrite the Omega entries of x (= x0 on entry). */
void or_assemble(int64_t K, const int64_t* idx, const double* xB, double* x) {
  for (int64_t l = 0; l < K; ++l) x[idx[l]] = xB[l];
}

/* ------------------------------------------------------------------------ */
/* Krylov solvers (Eq. 6 stopping test)                                      */
/* ------------------------------------------------------------------------ */

/*
 * Jacobi-preconditioned CG, textbook step order (BASELINE.json "CG for the SPD
 * systems ... Jacobi").  Stopping test Eq. 6: ||b - A x||_2 <= eps ||b||_2 (absolute eps if b = 0),
 * tested on the recursive residual and confirmed with the true residual (R19).
 * iterations = number of SpMVs with p (R30).
 */
int or_pcg(int64_t n, const int64_t* rp, const int32_t* ci, const double* a, const double* b, double* x,
           double eps, int max_iters, int* iters, double* relres) {
  *iters = 0;
  double nb = or_norm2(n, b);
  double tgt = nb > 0 ? eps * nb : eps;
  if (n == 0) { *relres = 0; return OR_OK; }
  double* dinv = (double*)malloc(sizeof(double) * n);
  double* r = (double*)malloc(sizeof(double) * n);
  double* z = (double*)malloc(sizeof(double) * n);
  double* pp = (double*)malloc(sizeof(double) * n);
  double* q = (double*)malloc(sizeof(double) * n);
  if (!dinv || !r || !z || !pp || !q) { free(dinv); free(r); free(z); free(pp); free(q); return OR_ERR_OOM; }
  int st = OR_NOT_CONVERGED;
  for (int64_t i = 0; i < n; ++i) {
    double d = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) if (ci[k] == i) d = a[k];
    if (d == 0.0) { st = OR_ERR_ZERO_DIAGONAL; goto done; }
    dinv[i] = 1.0 / d;
  }
  or_residual(n, rp, ci, a, b, x, r);                         /* 1. r = b - A x */
  double rn = sqrt(dot(n, r, r));
  if (rn <= tgt) { *relres = nb > 0 ? rn / nb : rn; st = OR_OK; goto done; }
  if (max_iters <= 0) { *relres = nb > 0 ? rn / nb : rn; goto done; }   /* cap 0: the Eq. 6 check only (R34) */
  for (;;) {
    for (int64_t i = 0; i < n; ++i) { z[i] = r[i] * dinv[i]; pp[i] = z[i]; }   /* 2. z = D^-1 r, p = z */
    double rho = dot(n, r, z);
    for (;;) {
      or_spmv(n, rp, ci, a, pp, q);                            /* 3. q = A p */
      double pi = dot(n, pp, q);
      if (!(pi > 0)) { st = isfinite(pi) ? OR_ERR_BREAKDOWN : OR_ERR_NONFINITE; goto done; }
      double alpha = rho / pi;
      for (int64_t i = 0; i < n; ++i) {
        x[i] = fma(alpha, pp[i], x[i]);
        r[i] = fma(-alpha, q[i], r[i]);
        z[i] = r[i] * dinv[i];
      }
      double rho1 = dot(n, r, z), sigma = dot(n, r, r);
      ++*iters;
      if (!isfinite(sigma)) { st = OR_ERR_NONFINITE; goto done; }
      if (sqrt(sigma) <= tgt) {                                /* 4. recursive test, then R19 confirm */
        or_residual(n, rp, ci, a, b, x, r);
        rn = sqrt(dot(n, r, r));
        if (rn <= tgt) { *relres = nb > 0 ? rn / nb : rn; st = OR_OK; goto done; }
        if (*iters >= max_iters) { *relres = nb > 0 ? rn / nb : rn; goto done; }
        break;                                                 /* restart from the true residual */
      }
      if (*iters >= max_iters) {
        or_residual(n, rp, ci, a, b, x, q);
        rn = sqrt(dot(n, q, q)); *relres = nb > 0 ? rn / nb : rn; goto done;
      }
      double beta = rho1 / rho;                                /* 5. p = z + beta p */
      rho = rho1;
      for (int64_t i = 0; i < n; ++i) pp[i] = fma(beta, pp[i], z[i]);
    }
  }
done:
  free(dinv); free(r); free(z); free(pp); free(q);
  return st;
}

/* invert a bs x bs block (bs <= 3) by LU without pivoting (diagonally dominant blocks) */
static int inv_block(int bs, const double* A, double* Ainv) {
  double L[9] = {0}, U[9] = {0};
  for (int i = 0; i < bs; ++i)
    for (int j = 0; j < bs; ++j) U[i * bs + j] = A[i * bs + j];
  for (int i = 0; i < bs; ++i) L[i * bs + i] = 1.0;
  for (int k = 0; k < bs; ++k) {
    if (U[k * bs + k] == 0.0) return -1;
    for (int i = k + 1; i < bs; ++i) {
      double f = U[i * bs + k] / U[k * bs + k];
      L[i * bs + k] = f;
      for (int j = k; j < bs; ++j) U[i * bs + j] -= f * U[k * bs + j];
    }
  }
  for (int c = 0; c < bs; ++c) {               /* solve L U x = e_c */
    double y[3];
    for (int i = 0; i < bs; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int j = 0; j < i; ++j) s -= L[i * bs + j] * y[j];
      y[i] = s;
    }
    for (int i = bs - 1; i >= 0; --i) {
      double s = y[i];
      for (int j = i + 1; j < bs; ++j) s -= U[i * bs + j] * Ainv[j * bs + c];
      Ainv[i * bs + c] = s / U[i * bs + i];
    }
  }
  return 0;
}

static void apply_bj(int64_t n, int bs, const double* Minv, const double* v, double* t) {
  for (int64_t c = 0; c < n / bs; ++c)
    for (int i = 0; i < bs; ++i) {
      double s = 0.0;
      for (int j = 0; j < bs; ++j) s = fma(Minv[c * bs * bs + i * bs + j], v[c * bs + j], s);
      t[c * bs + i] = s;
    }
}

/*
 * Restarted GMRES(m), RIGHT-preconditioned with block-Jacobi M = blockdiag(bs x bs cell blocks)
 * (R20, R33), classical Gram-Schmidt with one re-orthogonalisation (CGS2, R21), Givens rotations.
 * Stopping: |g_{j+1}| <= tgt (the Arnoldi residual estimate of Eq. 6), confirmed by the true
 * residual at the end of the cycle (R19).  iterations = cumulative Arnoldi steps (R30).
 */
int or_gmres_bj(int64_t n, const int64_t* rp, const int32_t* ci, const double* a, int bs, const double* b,
                double* x, double eps, int restart, int max_iters, int* iters, double* relres) {
  *iters = 0;
  if (bs < 1 || bs > 3 || n % bs || restart < 1) return OR_ERR_INVALID_ARG;
  double nb = or_norm2(n, b);
  double tgt = nb > 0 ? eps * nb : eps;
  if (n == 0) { *relres = 0; return OR_OK; }
  int m = restart;
  int64_t nc = n / bs;
  double* Minv = (double*)malloc(sizeof(double) * nc * bs * bs);
  double* V = (double*)malloc(sizeof(double) * (size_t)n * (m + 1));
  double* w = (double*)malloc(sizeof(double) * n);
  double* t = (double*)malloc(sizeof(double) * n);
  double* r = (double*)malloc(sizeof(double) * n);
  double* H = (double*)calloc((size_t)(m + 1) * m, sizeof(double));
  double *cs = (double*)malloc(sizeof(double) * m), *sn = (double*)malloc(sizeof(double) * m);
  double *g = (double*)malloc(sizeof(double) * (m + 1)), *y = (double*)malloc(sizeof(double) * m);
  double *h = (double*)malloc(sizeof(double) * (m + 1)), *h2 = (double*)malloc(sizeof(double) * (m + 1));
  int st = OR_NOT_CONVERGED;
  if (!Minv || !V || !w || !t || !r || !H || !cs || !sn || !g || !y || !h || !h2) { st = OR_ERR_OOM; goto done; }
  for (int64_t c = 0; c < nc; ++c) {              /* diagonal blocks of A */
    double D[9] = {0};
    for (int i = 0; i < bs; ++i) {
      int64_t row = c * bs + i;
      for (int64_t k = rp[row]; k < rp[row + 1]; ++k) {
        int64_t j = ci[k];
        if (j / bs == c) D[i * bs + (j % bs)] = a[k];
      }
    }
    if (inv_block(bs, D, Minv + c * bs * bs)) { st = OR_ERR_ZERO_DIAGONAL; goto done; }
  }
  or_residual(n, rp, ci, a, b, x, r);
  double beta = sqrt(dot(n, r, r));
  if (beta <= tgt) { *relres = nb > 0 ? beta / nb : beta; st = OR_OK; goto done; }
  for (;;) {
    for (int64_t i = 0; i < n; ++i) V[i] = r[i] / beta;            /* v_0 = r / beta */
    for (int i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = beta;
    int jend = 0;
    for (int j = 0; j < m; ++j) {
      double* vj = V + (size_t)j * n;
      apply_bj(n, bs, Minv, vj, t);                                  /* t = M^-1 v_j */
      or_spmv(n, rp, ci, a, t, w);                                   /* w = A t */
      for (int i = 0; i <= j; ++i) h[i] = dot(n, V + (size_t)i * n, w);   /* CGS pass 1 */
      for (int i = 0; i <= j; ++i) { const double* vi = V + (size_t)i * n;
        for (int64_t e = 0; e < n; ++e) w[e] = fma(-h[i], vi[e], w[e]); }
      for (int i = 0; i <= j; ++i) h2[i] = dot(n, V + (size_t)i * n, w);  /* CGS pass 2 */
      for (int i = 0; i <= j; ++i) { const double* vi = V + (size_t)i * n;
        for (int64_t e = 0; e < n; ++e) w[e] = fma(-h2[i], vi[e], w[e]); }
      for (int i = 0; i <= j; ++i) H[i * m + j] = h[i] + h2[i];
      double hn = sqrt(dot(n, w, w));
      H[(j + 1) * m + j] = hn;
      if (hn != 0.0) { double* vn = V + (size_t)(j + 1) * n; for (int64_t e = 0; e < n; ++e) vn[e] = w[e] / hn; }
      for (int i = 0; i < j; ++i) {                                  /* previous rotations */
        double t0 = H[i * m + j], t1 = H[(i + 1) * m + j];
        H[i * m + j] = cs[i] * t0 + sn[i] * t1;
        H[(i + 1) * m + j] = -sn[i] * t0 + cs[i] * t1;
      }
      double hd = H[j * m + j], hs = H[(j + 1) * m + j];
      double den = sqrt(hd * hd + hs * hs);
      if (den == 0.0) { cs[j] = 1.0; sn[j] = 0.0; } else { cs[j] = hd / den; sn[j] = hs / den; }
      H[j * m + j] = cs[j] * hd + sn[j] * hs;
      H[(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++*iters;
      jend = j + 1;
      if (!isfinite(g[j + 1])) { st = OR_ERR_NONFINITE; goto done; }
      if (fabs(g[j + 1]) <= tgt || hn == 0.0 || *iters >= max_iters) break;
    }
    for (int i = jend - 1; i >= 0; --i) {                            /* H y = g (upper triangular) */
      double s = g[i];
      for (int k = i + 1; k < jend; ++k) s -= H[i * m + k] * y[k];
      y[i] = s / H[i * m + i];
    }
    for (int64_t e = 0; e < n; ++e) w[e] = 0.0;                      /* x += M^-1 (V y) */
    for (int i = 0; i < jend; ++i) { const double* vi = V + (size_t)i * n;
      for (int64_t e = 0; e < n; ++e) w[e] = fma(y[i], vi[e], w[e]); }
    apply_bj(n, bs, Minv, w, t);
    for (int64_t e = 0; e < n; ++e) x[e] += t[e];
    or_residual(n, rp, ci, a, b, x, r);                              /* true residual (R19) */
    beta = sqrt(dot(n, r, r));
    *relres = nb > 0 ? beta / nb : beta;
    if (beta <= tgt) { st = OR_OK; goto done; }
    if (*iters >= max_iters) goto done;
    if (!isfinite(beta)) { st = OR_ERR_NONFINITE; goto done; }
  }
done:
  free(Minv); free(V); free(w); free(t); free(r); free(H); free(cs); free(sn); free(g); free(y); free(h); free(h2);
  return st;
}

/* ------------------------------------------------------------------------ */
/* Alg. 1 l.7: Gauss-Seidel smoothing of x~ (NEXT-1)       */
/* ------------------------------------------------------------------------ */

/* `sweeps` forward Gauss-Seidel sweeps in natural row order, in place:
   x_i <- (b_i - sum_{j != i} a_ij x_j) / a_ii, the sum the R22 fma chain over stored j != i ascending
   (j < i already updated in this sweep, j > i from the previous one).  SPEC S:145-153. */
int or_gauss_seidel(int64_t n, const int64_t* rp, const int32_t* ci, const double* a, const double* b, double* x,
                    int sweeps) {
  for (int sw = 0; sw < sweeps; ++sw)
    for (int64_t i = 0; i < n; ++i) {
      double acc = 0.0, d = 0.0;
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
        if (ci[k] == i) { d = a[k]; continue; }
        acc = fma(a[k], x[ci[k]], acc);
      }
      if (d == 0.0) return OR_ERR_ZERO_DIAGONAL;
      x[i] = (b[i] - acc) / d;
    }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Alg. 1 end to end (lines 2-11; line 7 = gs_sweeps Gauss-Seidel sweeps, R8) */
/* ------------------------------------------------------------------------ */

typedef struct {
  int32_t method;     /* 0 = Jacobi-PCG, 1 = block-Jacobi GMRES */
  int32_t bs;         /* block size of the GMRES preconditioner */
  int32_t restart;    /* GMRES(m) */
  double eps;         /* Eq. 6 tolerance */
  int32_t max_iters;
  int32_t gs_sweeps;  /* Alg. 1 l.7 smoothing sweeps before the convergence check (0 on the parity path) */
} or_solver_params;

typedef struct {
  int64_t K;
  double tau;
  int32_t it_local, it_global;
  int32_t st_local, st_global;
  double relres_local, relres_global;
  double t_select, t_extract, t_local, t_global;   /* seconds, steady clock */
} or_report;

static double now_s(void) {
  struct timespec ts; clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

static int solve(int64_t n, const int64_t* rp, const int32_t* ci, const double* a, const double* b, double* x,
                 const or_solver_params* s, int* it, double* rr) {
  if (s->method == 0) return or_pcg(n, rp, ci, a, b, x, s->eps, s->max_iters, it, rr);
  return or_gmres_bj(n, rp, ci, a, s->bs, b, x, s->eps, s->restart, s->max_iters, it, rr);
}

/* method0 when dp == NULL: the global solve from x0.  Otherwise Alg. 1.
   x: in = x0, out = solution.  flag_out (optional, [n]) receives Omega_local; xt_out (optional, [n]) receives
   x~ = Q (xbar_B; x_C^(0)) of Eq. 4 after l.6, before the l.7 sweeps (a copy; no effect on the arithmetic). */
int or_local_method(int64_t n, const int64_t* rp, const int32_t* ci, const double* a, const double* b, double* x,
                    const or_domain_params* dp, const or_solver_params* sp, uint8_t* flag_out, or_report* rep,
                    double* xt_out) {
  memset(rep, 0, sizeof(*rep));
  int st;
  if (dp) {
    double t0 = now_s();
    uint8_t* flag = (uint8_t*)malloc(n ? n : 1);
    double* crit = (double*)malloc(sizeof(double) * (n ? n : 1));
    double* adm = (double*)malloc(sizeof(double) * (n ? n : 1));
    or_trace tr;
    st = or_select_domain(n, rp, ci, a, b, x, dp, flag, crit, adm, &rep->tau, &rep->K, &tr);   /* l.2 */
    free(crit); free(adm);
    if (st != OR_OK) { free(flag); return st; }
    if (flag_out) memcpy(flag_out, flag, n);
    double t1 = now_s();
    rep->t_select = t1 - t0;
    if (rep->K > 0) {
      int64_t nnz = rp[n], K, Bn;
      int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * rep->K);
      int64_t* Brp = (int64_t*)malloc(sizeof(int64_t) * (rep->K + 1));
      int32_t* Bci = (int32_t*)malloc(sizeof(int32_t) * nnz);
      double* Ba = (double*)malloc(sizeof(double) * nnz);
      double* bsub = (double*)malloc(sizeof(double) * rep->K);
      double* xB = (double*)malloc(sizeof(double) * rep->K);
      or_extract(n, rp, ci, a, b, x, flag, idx, Brp, Bci, Ba, bsub, xB, &K, &Bn);  /* l.3-4 */
      double t2 = now_s();
      rep->t_extract = t2 - t1;
      rep->st_local = solve(K, Brp, Bci, Ba, bsub, xB, sp, &rep->it_local, &rep->relres_local);  /* l.5 */
      or_assemble(K, idx, xB, x);                                                            /* l.6 */
      rep->t_local = now_s() - t2;
      free(idx); free(Brp); free(Bci); free(Ba); free(bsub); free(xB);
    }
    free(flag);
    if (xt_out) memcpy(xt_out, x, sizeof(double) * n);                                        /* x~ (Eq. 4) */
    if (sp->gs_sweeps > 0) {                                                                 /* l.7 */
      st = or_gauss_seidel(n, rp, ci, a, b, x, sp->gs_sweeps);
      if (st != OR_OK) return st;
    }
  }
  double t3 = now_s();
  st = solve(n, rp, ci, a, b, x, sp, &rep->it_global, &rep->relres_global);                  /* l.8-11 */
  rep->st_global = st;
  rep->t_global = now_s() - t3;
  return st;
}

/* ------------------------------------------------------------------------ */
/* NEXT-2: the paper's 2-D nonlinear heat model and Alg. 6     */
/* ------------------------------------------------------------------------ */

/* kappa(T) = T^(k + 1/2) evaluated as T^k * sqrt(T) (R38: IEEE-exact operations, so the CPU and GPU
   assemblies are bitwise identical; the paper's T^3.5 is k = 3) */
static double kappa_pow(double t, int k) {
  double v = 1.0;
  for (int i = 0; i < k; ++i) v = v * t;
  return v * sqrt(t);
}

/* Backward Euler + five-point FV on nx x ny interior nodes x_p = (p+1) h, h = 1/(nx+1) (SPEC heat-model),
   Dirichlet T_l at x = 0 and T_r at x = 1 (ghost nodes at distance h), homogeneous Neumann at y = 0, 1
   (no flux), face conductivity the arithmetic mean (R26), kappa frozen at the Picard iterate Ts (Eq.
   picard-equs).  Row i = p + nx q, columns ascending:
     (1 + lam sum_f kf) T_i - lam sum_{f interior} kf T_nb = T_old_i + lam sum_{f boundary} kf T_bnd,
   lam = dt / h^2.  rp[nx ny + 1], ci, a (5 nx ny - 2 nx - 2 ny), b[nx ny]. */
void or_heat_assemble(int nx, int ny, double dt, int khalf, double Tl, double Tr, const double* Ts,
                      const double* Told, int64_t* rp, int32_t* ci, double* a, double* b) {
  double h = 1.0 / (nx + 1), lam = dt / (h * h);
  double kl = kappa_pow(Tl, khalf), kr = kappa_pow(Tr, khalf);
  int64_t z = 0;
  for (int q = 0; q < ny; ++q)
    for (int p = 0; p < nx; ++p) {
      int64_t i = p + (int64_t)nx * q;
      double ki = kappa_pow(Ts[i], khalf);
      double diag = 0.0, rhs = Told[i];
      rp[i] = z;
      if (q > 0) { double kf = 0.5 * (ki + kappa_pow(Ts[i - nx], khalf)); ci[z] = (int32_t)(i - nx); a[z++] = -lam * kf; diag += kf; }
      if (p > 0) { double kf = 0.5 * (ki + kappa_pow(Ts[i - 1], khalf)); ci[z] = (int32_t)(i - 1); a[z++] = -lam * kf; diag += kf; }
      else { double kf = 0.5 * (ki + kl); diag += kf; rhs += lam * kf * Tl; }
      int64_t zd = z++;
      if (p < nx - 1) { double kf = 0.5 * (ki + kappa_pow(Ts[i + 1], khalf)); ci[z] = (int32_t)(i + 1); a[z++] = -lam * kf; diag += kf; }
      else { double kf = 0.5 * (ki + kr); diag += kf; rhs += lam * kf * Tr; }
      if (q < ny - 1) { double kf = 0.5 * (ki + kappa_pow(Ts[i + nx], khalf)); ci[z] = (int32_t)(i + nx); a[z++] = -lam * kf; diag += kf; }
      ci[zd] = (int32_t)i;
      a[zd] = 1.0 + lam * diag;
      b[i] = rhs;
    }
  rp[(int64_t)nx * ny] = z;
}

typedef struct {
  int32_t steps, picard_total, picard_max_hit;
  int64_t it_local, it_global;
  double eta_sum;          /* sum over linear solves of K/N */
  double seconds;
} or_heat_report;

/* Alg. 6: for n: T^{n+1,0} = T^n; for s: assemble at T^{n+1,s}, solve with x0 = T^{n+1,s}
   (method0 if dp == NULL, else Alg. 1 with dp, sp), stop when ||T^{n+1,s+1} - T^{n+1,s}||_2 < picard_tol.
   T: in = T^0, out = T^steps.  picard_per_step (optional, [steps]) receives the Picard counts. */
int or_heat_run(int nx, int ny, double dt, int khalf, double Tl, double Tr, int steps, double picard_tol,
                int picard_max, const or_domain_params* dp, const or_solver_params* sp, double* T,
                int32_t* picard_per_step, or_heat_report* rep) {
  int64_t n = (int64_t)nx * ny, nnz = 5 * n;
  int64_t* rp = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  int32_t* ci = (int32_t*)malloc(sizeof(int32_t) * nnz);
  double* a = (double*)malloc(sizeof(double) * nnz);
  double* b = (double*)malloc(sizeof(double) * n);
  double* Ts = (double*)malloc(sizeof(double) * n);
  double* Tn = (double*)malloc(sizeof(double) * n);
  memset(rep, 0, sizeof(*rep));
  double t0 = now_s();
  int st = OR_OK;
  for (int step = 0; step < steps; ++step) {
    memcpy(Ts, T, sizeof(double) * n);                         /* T^{n+1,0} = T^n */
    int s;
    for (s = 0; s < picard_max; ++s) {
      or_heat_assemble(nx, ny, dt, khalf, Tl, Tr, Ts, T, rp, ci, a, b);
      memcpy(Tn, Ts, sizeof(double) * n);                      /* x0 = previous Picard iterate */
      or_report r;
      st = or_local_method(n, rp, ci, a, b, Tn, dp, sp, NULL, &r, NULL);
      if (st < 0) goto done;
      rep->it_local += r.it_local; rep->it_global += r.it_global; rep->eta_sum += (double)r.K / n;
      rep->picard_total += 1;
      double d2 = 0.0;
      for (int64_t i = 0; i < n; ++i) { double d = Tn[i] - Ts[i]; d2 = fma(d, d, d2); }
      memcpy(Ts, Tn, sizeof(double) * n);
      if (sqrt(d2) < picard_tol) { ++s; break; }
    }
    if (s >= picard_max) rep->picard_max_hit += 1;
    if (picard_per_step) picard_per_step[step] = s;
    memcpy(T, Ts, sizeof(double) * n);
    rep->steps = step + 1;
  }
done:
  rep->seconds = now_s() - t0;
  free(rp); free(ci); free(a); free(b); free(Ts); free(Tn);
  return st < 0 ? st : OR_OK;
}
