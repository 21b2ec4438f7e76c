/*
 * synth.c -- seeded synthetic input generator for the five BASELINE.json configs.
 *
 * This module is shared by the oracle tests and the CUDA path.  It holds NONE
 * of the local character-based method's arithmetic: it only builds the
 * problems A_s, b_s = A_s x*_s and x0_s = x*_{s-1} ("lock-step inputs",
 * SURVEY.md R28/R29) the method is later applied to.  Everything here is
 * evaluated once on the host, so both sides consume identical bits.
 *
 * Recipe:
 *   - cell-centred unit grid, h = 1/n, index i = ix + nx*(iy + ny*iz);
 *   - A = D + lambda0 * L(k): L is the finite-volume operator with face
 *     coefficient k_f = (k_p + k_q)/2, Dirichlet x-faces (the boundary face adds
 *     2 k_p to the diagonal), Neumann elsewhere;
 *   - columns stored ascending, the diagonal always stored;
 *   - b = A x* is formed with the ascending fma chain so that b - A x* == 0;
 *   - RNG: SplitMix64, u = (z >> 11) * 2^-53, seed_c = 20010115 + c.
 *
 * Compiled with OpenMP (cell loops are independent, so the output is identical
 * for any thread count).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SEED_BASE 20010115ULL

static uint64_t sm64_next(uint64_t* st) {
  uint64_t z = (*st += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static double sm64_u01(uint64_t* st) { return (double)(sm64_next(st) >> 11) * 0x1.0p-53; }
/* counter-based draw: value number `idx` of stream `seed` */
static double hash_u01(uint64_t seed, uint64_t idx) {
  uint64_t st = seed ^ (idx * 0xD1B54A32D192ED03ULL);
  return sm64_u01(&st);
}

/* ---- smooth background T_bg = lo + (hi-lo)*(1/2 + 1/2*sum c_m sin(...)/sum c_m) ---- */
typedef struct { int a[4], b[4], e[4]; double c[4], phi[4], csum, lo, hi; } bg_t;

static void bg_init(bg_t* g, uint64_t seed, double lo, double hi) {
  uint64_t st = seed;
  g->csum = 0.0;
  for (int m = 0; m < 4; ++m) {
    g->a[m] = 1 + (int)(sm64_u01(&st) * 3.0);
    g->b[m] = 1 + (int)(sm64_u01(&st) * 3.0);
    g->e[m] = 1 + (int)(sm64_u01(&st) * 3.0);
    g->c[m] = 0.5 + 0.5 * sm64_u01(&st);
    g->phi[m] = 2.0 * M_PI * sm64_u01(&st);
    g->csum += g->c[m];
  }
  g->lo = lo; g->hi = hi;
}
static double bg_eval(const bg_t* g, double x, double y, double z, int dim3) {
  double s = 0.0;
  for (int m = 0; m < 4; ++m) {
    double arg = 2.0 * M_PI * (g->a[m] * x + g->b[m] * y + (dim3 ? g->e[m] * z : 0.0)) + g->phi[m];
    s += g->c[m] * sin(arg);
  }
  return g->lo + (g->hi - g->lo) * (0.5 + 0.5 * s / g->csum);
}

/* ---- scalar stencil assembly: A = diag_add + lambda0 * L(kc) ---- */
static int64_t row_len(int64_t ix, int64_t iy, int64_t iz, int64_t nx, int64_t ny, int64_t nz) {
  int64_t l = 1 + (ix > 0) + (ix < nx - 1) + (iy > 0) + (iy < ny - 1);
  if (nz > 1) l += (iz > 0) + (iz < nz - 1);
  return l;
}

static void build_rowptr(int64_t nx, int64_t ny, int64_t nz, int64_t off_rows, int64_t off_nnz, int64_t* rp) {
  int64_t N = nx * ny * nz, acc = off_nnz;
  for (int64_t i = 0; i < N; ++i) {
    int64_t ix = i % nx, iy = (i / nx) % ny, iz = i / (nx * ny);
    rp[off_rows + i] = acc;
    acc += row_len(ix, iy, iz, nx, ny, nz);
  }
  rp[off_rows + N] = acc;
}

/* fills rows [0,N) of one segment whose rowptr is rp (already offset), column offset coff */
static void assemble_scalar(int64_t nx, int64_t ny, int64_t nz, double lambda0, const double* kc,
                            const double* diag_add, const int64_t* rp, int64_t coff, int32_t* ci, double* val) {
  int64_t N = nx * ny * nz, pl = nx * ny;
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < N; ++p) {
    int64_t ix = p % nx, iy = (p / nx) % ny, iz = p / pl;
    int64_t nb[6]; int nn = 0;           /* ascending neighbour list excluding self */
    int64_t lo[3], hi[3]; int nlo = 0, nhi = 0;
    if (nz > 1 && iz > 0) lo[nlo++] = p - pl;
    if (iy > 0) lo[nlo++] = p - nx;
    if (ix > 0) lo[nlo++] = p - 1;
    if (ix < nx - 1) hi[nhi++] = p + 1;
    if (iy < ny - 1) hi[nhi++] = p + nx;
    if (nz > 1 && iz < nz - 1) hi[nhi++] = p + pl;
    (void)nb; (void)nn;
    double d = diag_add[p];
    int64_t k = rp[p];
    for (int t = 0; t < nlo; ++t) {
      double kf = 0.5 * (kc[p] + kc[lo[t]]);
      ci[k] = (int32_t)(coff + lo[t]); val[k] = -lambda0 * kf; d += lambda0 * kf; ++k;
    }
    int64_t kd = k++;
    for (int t = 0; t < nhi; ++t) {
      double kf = 0.5 * (kc[p] + kc[hi[t]]);
      ci[k] = (int32_t)(coff + hi[t]); val[k] = -lambda0 * kf; d += lambda0 * kf; ++k;
    }
    if (ix == 0) d += lambda0 * 2.0 * kc[p];
    if (ix == nx - 1) d += lambda0 * 2.0 * kc[p];
    ci[kd] = (int32_t)(coff + p); val[kd] = d;
  }
}

/* b = A x with the ascending fma chain (CSR, scalar rows) */
static void csr_apply(int64_t nrows, const int64_t* rp, const int32_t* ci, const double* val, const double* x,
                      double* b) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nrows; ++i) {
    double acc = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) acc = fma(val[k], x[ci[k]], acc);
    b[i] = acc;
  }
}

/* ---- public API ---------------------------------------------------------- */

/* Default grid sizes of BASELINE.json configs[0..4] */
int synth_default_n(int config) {
  switch (config) { case 1: return 64; case 2: return 1024; case 3: return 512; case 4: return 512; case 5: return 256; }
  return -1;
}
int synth_default_systems(int config) {
  switch (config) { case 1: return 10; case 2: return 50; case 3: return 20; case 4: return 30; case 5: return 20; }
  return -1;
}

/* dims: nrows = scalar rows (block rows for config 4), nnz = stored scalars (blocks for config 4) */
int synth_dims(int config, int n, int G, int64_t* nrows, int64_t* nnz, int* block) {
  if (n < 2) return -1;
  int64_t nn = n;
  *block = 1;
  switch (config) {
    case 1: case 2:
      *nrows = nn * nn; *nnz = 5 * nn * nn - 4 * nn; return 0;
    case 3:
      if (G < 1) return -1;
      *nrows = (int64_t)G * nn * nn; *nnz = (int64_t)G * (5 * nn * nn - 4 * nn); return 0;
    case 4:
      *block = 3; *nrows = nn * nn; *nnz = 5 * nn * nn - 4 * nn; return 0;
    case 5:
      *nrows = nn * nn * nn; *nnz = 7 * nn * nn * nn - 6 * nn * nn; return 0;
  }
  return -1;
}

static void cfg1_field(int n, const bg_t* bg, double c0x, double c0y, int s, double* T) {
  double h = 1.0 / n;
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < (int64_t)n * n; ++p) {
    int ix = (int)(p % n), iy = (int)(p / n);
    double cx = c0x + s, cy = c0y;
    double rho2 = (ix - cx) * (ix - cx) + (iy - cy) * (iy - cy);
    T[p] = bg_eval(bg, (ix + 0.5) * h, (iy + 0.5) * h, 0.0, 0) + 10.0 * exp(-rho2 / (2.0 * 16.0));
  }
}

static void cfg2_field(int n, const bg_t* bg, double cx, double cy, int s, double* T) {
  double h = 1.0 / n, R = (100.0 + 2.0 * s) * n / 1024.0;
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < (int64_t)n * n; ++p) {
    int ix = (int)(p % n), iy = (int)(p / n);
    double rho = sqrt((ix - cx) * (ix - cx) + (iy - cy) * (iy - cy));
    T[p] = bg_eval(bg, (ix + 0.5) * h, (iy + 0.5) * h, 0.0, 0) + 0.8 * 0.5 * (1.0 - tanh((rho - R) / 2.0));
  }
}

/* config 3 temperature T_k (k may be -1) */
static double cfg3_T(double x, double tbg, double xf, double h, int k) {
  double Tinf = 0.1 + 0.9 * 0.5 * (1.0 - tanh((x - xf) / (2.0 * h))) + tbg;
  double w = 4.0 * h;
  return Tinf + pow(0.5, k + 1) * 0.2 * exp(-(x - xf) * (x - xf) / (2.0 * w * w));
}

static void cfg5_field(int n, const bg_t* bg, const double c[3], int s, double* T) {
  double h = 1.0 / n, R = (64.0 + s) * n / 256.0;
  int64_t N = (int64_t)n * n * n;
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < N; ++p) {
    int ix = (int)(p % n), iy = (int)((p / n) % n), iz = (int)(p / ((int64_t)n * n));
    double rho = sqrt((ix - c[0]) * (ix - c[0]) + (iy - c[1]) * (iy - c[1]) + (iz - c[2]) * (iz - c[2]));
    T[p] = bg_eval(bg, (ix + 0.5) * h, (iy + 0.5) * h, (iz + 0.5) * h, 1) + 0.9 * 0.5 * (1.0 - tanh(rho - R));
  }
}

static double pow25(double t) { return pow(t, 2.5); }

/*
 * Generate system s of config `config` at grid size n (G groups for config 3).
 * Outputs (caller-allocated, sizes from synth_dims):
 *   rp[nrows+1], ci[nnz], val[nnz*block*block], b[nrows*block], x0[nrows*block], xs[nrows*block]
 * seed_offset is added to the per-config seed (0 = the canonical inputs).
 */
int synth_system(int config, int n, int G, int s, uint64_t seed_offset, int64_t* rp, int32_t* ci, double* val,
                 double* b, double* x0, double* xs) {
  int64_t nrows, nnz; int block;
  if (synth_dims(config, n, G, &nrows, &nnz, &block) != 0) return -1;
  uint64_t seed = SEED_BASE + (uint64_t)config + seed_offset * 1000003ULL;
  uint64_t st = seed;
  double h = 1.0 / n;
  int64_t nn = n;

  if (config == 1) {
    bg_t bg; bg_init(&bg, seed ^ 0x1111ULL, 0.1, 1.0);
    double c0x = 3.0 * n / 8.0 + sm64_u01(&st) * n / 4.0;
    double c0y = 3.0 * n / 8.0 + sm64_u01(&st) * n / 4.0;
    double lambda0 = 1e-2 * (double)n * (double)n;
    int64_t N = nn * nn;
    double* kc = (double*)malloc(sizeof(double) * N);
    double* da = (double*)malloc(sizeof(double) * N);
    cfg1_field(n, &bg, c0x, c0y, s, xs);
    cfg1_field(n, &bg, c0x, c0y, s - 1, x0);
    for (int64_t p = 0; p < N; ++p) { kc[p] = pow25(x0[p]); da[p] = 1.0; }
    build_rowptr(nn, nn, 1, 0, 0, rp);
    assemble_scalar(nn, nn, 1, lambda0, kc, da, rp, 0, ci, val);
    csr_apply(N, rp, ci, val, xs, b);
    free(kc); free(da);
    return 0;
  }
  if (config == 2) {
    bg_t bg; bg_init(&bg, seed ^ 0x2222ULL, 0.1, 0.2);
    double sx[4], sy[4]; int perm[4] = {0, 1, 2, 3};
    for (int r = 0; r < 4; ++r) { sx[r] = sm64_u01(&st); sy[r] = sm64_u01(&st); }
    for (int r = 3; r > 0; --r) { int j = (int)(sm64_u01(&st) * (r + 1)); int t = perm[r]; perm[r] = perm[j]; perm[j] = t; }
    double cx = n / 2.0 + (2.0 * sm64_u01(&st) - 1.0) * 32.0 * n / 1024.0;
    double cy = n / 2.0 + (2.0 * sm64_u01(&st) - 1.0) * 32.0 * n / 1024.0;
    int64_t N = nn * nn;
    double* kc = (double*)malloc(sizeof(double) * N);
    double* da = (double*)malloc(sizeof(double) * N);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < N; ++p) {
      double px = ((p % n) + 0.5) * h, py = ((p / n) + 0.5) * h;
      int best = 0; double bd = 1e300;
      for (int r = 0; r < 4; ++r) {
        double d = (px - sx[r]) * (px - sx[r]) + (py - sy[r]) * (py - sy[r]);
        if (d < bd) { bd = d; best = r; }
      }
      kc[p] = 1e-2 * pow(10.0, 4.0 * perm[best] / 3.0);
      da[p] = 1.0;
    }
    cfg2_field(n, &bg, cx, cy, s, xs);
    cfg2_field(n, &bg, cx, cy, s - 1, x0);
    build_rowptr(nn, nn, 1, 0, 0, rp);
    assemble_scalar(nn, nn, 1, 10.0, kc, da, rp, 0, ci, val);
    csr_apply(N, rp, ci, val, xs, b);
    free(kc); free(da);
    return 0;
  }
  if (config == 3) {
    bg_t bg; bg_init(&bg, seed ^ 0x3333ULL, 0.0, 0.05);
    double xf = 0.3 + 0.4 * sm64_u01(&st);
    int64_t Ng = nn * nn;
    double lambda0 = 100.0, lambda_a = 100.0 / ((double)n * (double)n);
    double* Tk = (double*)malloc(sizeof(double) * Ng);
    double* Tkm = (double*)malloc(sizeof(double) * Ng);
    double* kc = (double*)malloc(sizeof(double) * Ng);
    double* da = (double*)malloc(sizeof(double) * Ng);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < Ng; ++p) {
      double px = ((p % n) + 0.5) * h, py = ((p / n) + 0.5) * h;
      double tbg = bg_eval(&bg, px, py, 0.0, 0);
      Tk[p] = cfg3_T(px, tbg, xf, h, s);
      Tkm[p] = cfg3_T(px, tbg, xf, h, s - 1);
    }
    int64_t seg_nnz = 5 * nn * nn - 4 * nn;
    for (int g = 0; g < G; ++g) {
      double expo = (G > 1) ? (double)g / (double)(G - 1) : 0.0;
      double sigma0 = pow(10.0, -2.0 + 4.0 * expo);
      double scale = pow(10.0, -4.0 * expo);
      int64_t ro = (int64_t)g * Ng;
#pragma omp parallel for schedule(static)
      for (int64_t p = 0; p < Ng; ++p) {
        double t = Tkm[p];
        double sig = sigma0 / (t * t * t);
        kc[p] = 1.0 / (3.0 * sig);
        da[p] = 1.0 + lambda_a * sig;
        double t4 = Tk[p] * Tk[p]; t4 *= t4;
        double tm4 = t * t; tm4 *= tm4;
        xs[ro + p] = scale * t4;
        x0[ro + p] = scale * tm4;
      }
      build_rowptr(nn, nn, 1, ro, (int64_t)g * seg_nnz, rp);
      assemble_scalar(nn, nn, 1, lambda0, kc, da, rp + ro, ro, ci, val);
    }
    csr_apply(nrows, rp, ci, val, xs, b);
    free(Tk); free(Tkm); free(kc); free(da);
    return 0;
  }
  if (config == 4) {
    /* 3T: BSR 3x3, unknowns interleaved (e,i,r) per cell */
    bg_t bg[3];
    for (int a = 0; a < 3; ++a) bg_init(&bg[a], seed ^ (0x4444ULL + (uint64_t)a), 0.3, 1.0);
    double cx = n / 4.0 + sm64_u01(&st) * n / 2.0, cy = n / 4.0 + sm64_u01(&st) * n / 2.0;
    const double H[3] = {1.0, 0.5, 0.8}, kap[3] = {1.0, 0.1, 1.0};
    const double dt = 1e-2, lambda0 = 10.0;
    int64_t N = nn * nn;
    double* K = (double*)malloc(sizeof(double) * 3 * N);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < N; ++p) {
      int ix = (int)(p % n), iy = (int)(p / n);
      double rho2 = (ix - cx) * (ix - cx) + (iy - cy) * (iy - cy);
      double gau = exp(-rho2 / (2.0 * 64.0));
      for (int a = 0; a < 3; ++a) {
        double tb = bg_eval(&bg[a], (ix + 0.5) * h, (iy + 0.5) * h, 0.0, 0);
        xs[3 * p + a] = tb + H[a] * (1.0 - pow(0.5, s + 1)) * gau;
        x0[3 * p + a] = tb + H[a] * (1.0 - pow(0.5, s)) * gau;
        K[3 * p + a] = kap[a] * pow25(x0[3 * p + a]);
      }
    }
    build_rowptr(nn, nn, 1, 0, 0, rp);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < N; ++p) {
      int64_t ix = p % n, iy = p / n;
      double C[3], wei, wer;
      for (int a = 0; a < 3; ++a) C[a] = 0.5 + 1.5 * hash_u01(seed ^ 0xC0FFEEULL, (uint64_t)p * 8 + a);
      wei = pow(10.0, -2.0 + 5.0 * hash_u01(seed ^ 0xC0FFEEULL, (uint64_t)p * 8 + 3));
      wer = pow(10.0, -2.0 + 5.0 * hash_u01(seed ^ 0xC0FFEEULL, (uint64_t)p * 8 + 4));
      double W[3][3] = {{wei + wer, -wei, -wer}, {-wei, wei, 0.0}, {-wer, 0.0, wer}};
      int64_t nbr[4]; int nb = 0, self_pos;
      if (iy > 0) nbr[nb++] = p - n;
      if (ix > 0) nbr[nb++] = p - 1;
      self_pos = nb;
      if (ix < n - 1) nbr[nb++] = p + 1;
      if (iy < n - 1) nbr[nb++] = p + n;
      double dsum[3] = {0, 0, 0};
      int64_t k = rp[p];
      for (int t = 0; t <= nb; ++t) {
        int64_t blk;
        if (t == self_pos) { blk = k + self_pos; ci[blk] = (int32_t)p; continue; }
        int tt = t > self_pos ? t - 1 : t;
        int64_t q = nbr[tt];
        blk = k + t;
        ci[blk] = (int32_t)q;
        for (int a = 0; a < 3; ++a)
          for (int bb = 0; bb < 3; ++bb) val[blk * 9 + 3 * a + bb] = 0.0;
        for (int a = 0; a < 3; ++a) {
          double kf = 0.5 * (K[3 * p + a] + K[3 * q + a]);
          val[blk * 9 + 4 * a] = -lambda0 * kf / C[a];
          dsum[a] += kf;
        }
      }
      for (int a = 0; a < 3; ++a) {
        if (ix == 0) dsum[a] += 2.0 * K[3 * p + a];
        if (ix == n - 1) dsum[a] += 2.0 * K[3 * p + a];
      }
      int64_t blk = k + self_pos;
      for (int a = 0; a < 3; ++a)
        for (int bb = 0; bb < 3; ++bb)
          val[blk * 9 + 3 * a + bb] = (a == bb ? 1.0 + lambda0 * dsum[a] / C[a] : 0.0) + dt * W[a][bb] / C[a];
    }
    /* b = A x* with the scalar ascending fma chain: blocks ascending, beta ascending */
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < N; ++p)
      for (int a = 0; a < 3; ++a) {
        double acc = 0.0;
        for (int64_t k = rp[p]; k < rp[p + 1]; ++k)
          for (int bb = 0; bb < 3; ++bb) acc = fma(val[k * 9 + 3 * a + bb], xs[3 * (int64_t)ci[k] + bb], acc);
        b[3 * p + a] = acc;
      }
    free(K);
    return 0;
  }
  if (config == 5) {
    bg_t bg; bg_init(&bg, seed ^ 0x5555ULL, 0.1, 0.15);
    double c[3];
    for (int a = 0; a < 3; ++a) c[a] = n / 2.0 + (2.0 * sm64_u01(&st) - 1.0) * n / 32.0;
    int64_t N = nn * nn * nn;
    double* kc = (double*)malloc(sizeof(double) * N);
    double* da = (double*)malloc(sizeof(double) * N);
    cfg5_field(n, &bg, c, s, xs);
    cfg5_field(n, &bg, c, s - 1, x0);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < N; ++p) { kc[p] = pow25(x0[p]); da[p] = 1.0; }
    build_rowptr(nn, nn, nn, 0, 0, rp);
    assemble_scalar(nn, nn, nn, 10.0, kc, da, rp, 0, ci, val);
    csr_apply(N, rp, ci, val, xs, b);
    free(kc); free(da);
    return 0;
  }
  return -1;
}

/* Tiny random systems for oracle self-tests: n x n, bandwidth bw, row-diagonally
   dominant (margin 1) with seeded values; structurally symmetric; optional SPD. */
int64_t synth_random_nnz(int n, int bw) {
  int64_t z = 0;
  for (int i = 0; i < n; ++i) for (int j = i - bw; j <= i + bw; ++j) if (j >= 0 && j < n) ++z;
  return z;
}
int synth_random(int n, int bw, int spd, uint64_t seed, int64_t* rp, int32_t* ci, double* val, double* b,
                 double* x0, double* xs) {
  int64_t k = 0;
  /* symmetric off-diagonal values a_ij = a_ji from a counter hash of (min,max) */
  for (int i = 0; i < n; ++i) {
    rp[i] = k;
    double rowsum = 0.0; int64_t kd = -1;
    for (int j = i - bw; j <= i + bw; ++j) {
      if (j < 0 || j >= n) continue;
      ci[k] = j;
      if (j == i) { kd = k; val[k] = 0.0; }
      else {
        int lo = i < j ? i : j, hi = i < j ? j : i;
        uint64_t key = (uint64_t)lo * 65537ULL + (uint64_t)hi + (spd ? 0 : (uint64_t)(i > j) * 7919ULL);
        double v = -hash_u01(seed, key);
        val[k] = v; rowsum += fabs(v);
      }
      ++k;
    }
    val[kd] = rowsum + 1.0;
  }
  rp[n] = k;
  for (int i = 0; i < n; ++i) { xs[i] = 2.0 * hash_u01(seed ^ 0xABCDULL, (uint64_t)i) - 1.0;
                                x0[i] = xs[i] + 0.1 * (2.0 * hash_u01(seed ^ 0x1234ULL, (uint64_t)i) - 1.0); }
  csr_apply(n, rp, ci, val, xs, b);
  return 0;
}
