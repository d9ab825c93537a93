/*
 * psi_oracle.c — CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker for the CUDA path in
 * paper_0904_0939_b200/csrc; only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * never routes through it.
 *
 * Each function restates one numba kernel of psibox
 * (/root/reference/pkg/src/psibox/kernels.py) with the same per-site
 * evaluation order.  Compiled with -ffp-contract=off (no FMA), as numba
 * compiles the reference (fastmath off), so the stencil and coefficient
 * arithmetic is bit-identical to the reference; plane sums accumulate
 * sequentially in (j asc, k asc) order exactly like the reference loops.
 * Parity is pinned against fixtures generated from the reference itself
 * (tests/golden/make_golden.py).
 *
 * Arrays are (planes, ext, ext) fp64 C-order, ext = N+2; plane ranges are
 * inclusive local indices x_lo..x_hi.  OpenMP parallelises over planes only,
 * which leaves every per-plane result independent of the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define AT(arr, i, j, k) (arr)[((int64_t)(i) * ext + (j)) * ext + (k)]

int oracle_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

/* kernels.stencil_update, kernels.py:22-37 */
void oracle_stencil_update(const double* psi, const double* ca, const double* cc, double* out,
                           int64_t planes, int64_t ext, int64_t x_lo, int64_t x_hi) {
  (void)planes;
  const int64_t n1 = ext - 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = x_lo; i <= x_hi; ++i)
    for (int64_t j = 1; j < n1; ++j)
      for (int64_t k = 1; k < n1; ++k) {
        double s = AT(psi, i - 1, j, k) + AT(psi, i + 1, j, k);
        s = s + AT(psi, i, j - 1, k);
        s = s + AT(psi, i, j + 1, k);
        s = s + AT(psi, i, j, k - 1);
        s = s + AT(psi, i, j, k + 1);
        s = s - 6.0 * AT(psi, i, j, k);
        AT(out, i, j, k) = AT(ca, i, j, k) * AT(psi, i, j, k) + AT(cc, i, j, k) * s;
      }
}

/* stencil_update with A and C formed from V in the order of
 * potential._coefficients (potential.py:102-115):
 *   denom = 1 + h V, A = (1 - h V)/denom, B = 1/denom, C = B*c0,
 * h = 0.5*dtau, c0 = dtau/(((2m)a)a).  Bit-identical to passing the
 * numpy-built coef arrays. */
void oracle_stencil_update_v(const double* psi, const double* v, double h, double c0, double* out,
                             int64_t planes, int64_t ext, int64_t x_lo, int64_t x_hi) {
  (void)planes;
  const int64_t n1 = ext - 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = x_lo; i <= x_hi; ++i)
    for (int64_t j = 1; j < n1; ++j)
      for (int64_t k = 1; k < n1; ++k) {
        const double hv = h * AT(v, i, j, k);
        const double denom = 1.0 + hv;
        const double A = (1.0 - hv) / denom;
        const double B = 1.0 / denom;
        const double C = B * c0;
        double s = AT(psi, i - 1, j, k) + AT(psi, i + 1, j, k);
        s = s + AT(psi, i, j - 1, k);
        s = s + AT(psi, i, j + 1, k);
        s = s + AT(psi, i, j, k - 1);
        s = s + AT(psi, i, j, k + 1);
        s = s - 6.0 * AT(psi, i, j, k);
        AT(out, i, j, k) = A * AT(psi, i, j, k) + C * s;
      }
}

/* kernels.norm_plane_sums, kernels.py:40-49 */
void oracle_norm_plane_sums(const double* psi, int64_t planes, int64_t ext, int64_t x_lo,
                            int64_t x_hi, double* out) {
  (void)planes;
  const int64_t n1 = ext - 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = x_lo; i <= x_hi; ++i) {
    double acc = 0.0;
    for (int64_t j = 1; j < n1; ++j)
      for (int64_t k = 1; k < n1; ++k) acc += AT(psi, i, j, k) * AT(psi, i, j, k);
    out[i - x_lo] = acc;
  }
}

/* kernels.energy_plane_sums, kernels.py:52-74 */
void oracle_energy_plane_sums(const double* psi, const double* v, double kin, int64_t planes,
                              int64_t ext, int64_t x_lo, int64_t x_hi, double* num_out,
                              double* den_out) {
  (void)planes;
  const int64_t n1 = ext - 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = x_lo; i <= x_hi; ++i) {
    double num = 0.0, den = 0.0;
    for (int64_t j = 1; j < n1; ++j)
      for (int64_t k = 1; k < n1; ++k) {
        double s = AT(psi, i - 1, j, k) + AT(psi, i + 1, j, k);
        s = s + AT(psi, i, j - 1, k);
        s = s + AT(psi, i, j + 1, k);
        s = s + AT(psi, i, j, k - 1);
        s = s + AT(psi, i, j, k + 1);
        s = s - 6.0 * AT(psi, i, j, k);
        const double p = AT(psi, i, j, k);
        const double h = AT(v, i, j, k) * p - kin * s;
        num += p * h;
        den += p * p;
      }
    num_out[i - x_lo] = num;
    den_out[i - x_lo] = den;
  }
}

/* kernels.radius2_plane_sums, kernels.py:77-100 */
void oracle_radius2_plane_sums(const double* psi, int64_t x_global0, double center, double a,
                               int64_t planes, int64_t ext, int64_t x_lo, int64_t x_hi,
                               double* r2_out, double* den_out) {
  (void)planes;
  const int64_t n1 = ext - 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = x_lo; i <= x_hi; ++i) {
    const double dx = ((double)(x_global0 + (i - x_lo)) - center) * a;
    const double dx2 = dx * dx;
    double r2acc = 0.0, den = 0.0;
    for (int64_t j = 1; j < n1; ++j) {
      const double dy = ((double)j - center) * a;
      const double dy2 = dy * dy;
      for (int64_t k = 1; k < n1; ++k) {
        const double dz = ((double)k - center) * a;
        const double r2 = dx2 + dy2 + dz * dz;
        const double w = AT(psi, i, j, k) * AT(psi, i, j, k);
        r2acc += w * r2;
        den += w;
      }
    }
    r2_out[i - x_lo] = r2acc;
    den_out[i - x_lo] = den;
  }
}

/* kernels.dot_plane_sums, kernels.py:103-112 */
void oracle_dot_plane_sums(const double* psi1, const double* psi2, int64_t planes, int64_t ext,
                           int64_t x_lo, int64_t x_hi, double* out) {
  (void)planes;
  const int64_t n1 = ext - 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = x_lo; i <= x_hi; ++i) {
    double acc = 0.0;
    for (int64_t j = 1; j < n1; ++j)
      for (int64_t k = 1; k < n1; ++k) acc += AT(psi1, i, j, k) * AT(psi2, i, j, k);
    out[i - x_lo] = acc;
  }
}

/* numpy DOUBLE_pairwise_sum (numpy/_core/src/umath/loops_utils.h.src), as used
 * by np.sum in observables.combine_plane_sums (observables.py:32-34);
 * np.sum(a) == 0.0 + pairwise(a, n) (checked in tests/test_oracle.py). */
static double pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int q = 0; q < 8; ++q) r[q] = a[q];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int q = 0; q < 8; ++q) r[q] += a[i + q];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise(a, n2) + pairwise(a + n2, n - n2);
  }
}

double oracle_np_sum(const double* a, int64_t n) { return 0.0 + pairwise(a, n); }

/* psi *= f over count doubles (evolve.py:180, parallel.py:479) */
void oracle_scale(double* psi, int64_t count, double f) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) psi[i] *= f;
}

/* potential._coefficients (potential.py:102-115) over count doubles */
void oracle_coefficients(const double* v, int64_t count, double dtau, double m, double a,
                         double* A, double* B, double* C) {
  const double h = 0.5 * dtau;
  const double c0 = dtau / (((2.0 * m) * a) * a);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    const double denom = 1.0 + h * v[i];
    A[i] = (1.0 - h * v[i]) / denom;
    B[i] = 1.0 / denom;
    C[i] = B[i] * c0;
  }
}
