/*
 * ORACLE — test infrastructure only (never linked into the product).
 *
 * Plain-C restatement of the reference's numba kernels, evaluated in the
 * same operation order with FP contraction disabled (-ffp-contract=off), so
 * that results are bit-identical to numba's non-fastmath LLVM code:
 *
 *   or_signed_svd   <- _signed_svd_batch + _jacobi_eigh3
 *                      (/root/reference/pkg/src/schurpd/material.py:69-221)
 *   or_uvt          <- _uvt_batch        (material.py:224-233)
 *   or_udvt         <- _u_diag_vt_batch  (material.py:236-245), with the clamp of
 *                      biphasic_projections (material.py:287) applied first
 *   or_lsolve       <- _lsolve           (linalg.py:203-213)
 *   or_ltsolve      <- _ltsolve          (linalg.py:216-223)
 *
 * Built by oracle/Makefile into oracle/_build/liboracle.so (ctypes).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

/* Worker count for the element loops (OR_THREADS env, default 1); the
 * per-element math is independent, so splitting ranges keeps results
 * identical for any thread count. */
static int or_threads(void) {
  const char *s = getenv("OR_THREADS");
  int t = s ? atoi(s) : 1;
  return t < 1 ? 1 : (t > 256 ? 256 : t);
}

typedef struct {
  int64_t lo, hi;
  const double *F;
  double *U, *S, *V;
} svd_job;

static void jacobi_eigh3(double A[3][3], double V[3][3]) {
  /* material.py:69-113 */
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.0 : 0.0;
  double scale = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double a = fabs(A[i][j]);
      if (a > scale) scale = a; /* max(scale, a) */
    }
  if (scale == 0.0) return;
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = fabs(A[0][1]) + fabs(A[0][2]) + fabs(A[1][2]);
    if (off <= 1e-30 * scale) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double apq = A[p][q];
        if (apq == 0.0) continue;
        double tau = (A[q][q] - A[p][p]) / (2.0 * apq);
        double t;
        if (tau >= 0.0)
          t = 1.0 / (tau + sqrt(1.0 + tau * tau));
        else
          t = -1.0 / (-tau + sqrt(1.0 + tau * tau));
        double c = 1.0 / sqrt(1.0 + t * t);
        double s = t * c;
        for (int k = 0; k < 3; ++k) {
          double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = c * vkp - s * vkq;
          V[k][q] = s * vkp + c * vkq;
        }
      }
  }
}

static void signed_svd1(const double *f /*3x3 row-major*/, double *u, double *S, double *v) {
  /* material.py:116-221 for one matrix */
  double A[3][3], Ve[3][3];
#define F_(i, j) f[(i)*3 + (j)]
#define U_(i, j) u[(i)*3 + (j)]
#define V_(i, j) v[(i)*3 + (j)]
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += F_(k, i) * F_(k, j);
      A[i][j] = acc;
    }
  jacobi_eigh3(A, Ve);
  double d0 = A[0][0], d1 = A[1][1], d2 = A[2][2], tmp;
  int i0 = 0, i1 = 1, i2 = 2, ti;
  if (d1 > d0) { tmp = d0; d0 = d1; d1 = tmp; ti = i0; i0 = i1; i1 = ti; }
  if (d2 > d0) { tmp = d0; d0 = d2; d2 = tmp; ti = i0; i0 = i2; i2 = ti; }
  if (d2 > d1) { tmp = d1; d1 = d2; d2 = tmp; ti = i1; i1 = i2; i2 = ti; }
  (void)d0; (void)d1; (void)d2;
  for (int r = 0; r < 3; ++r) {
    V_(r, 0) = Ve[r][i0];
    V_(r, 1) = Ve[r][i1];
    V_(r, 2) = Ve[r][i2];
  }
  double detv = V_(0, 0) * (V_(1, 1) * V_(2, 2) - V_(1, 2) * V_(2, 1)) -
                V_(0, 1) * (V_(1, 0) * V_(2, 2) - V_(1, 2) * V_(2, 0)) +
                V_(0, 2) * (V_(1, 0) * V_(2, 1) - V_(1, 1) * V_(2, 0));
  if (detv < 0.0)
    for (int r = 0; r < 3; ++r) V_(r, 2) = -V_(r, 2);
  double w0x = F_(0, 0) * V_(0, 0) + F_(0, 1) * V_(1, 0) + F_(0, 2) * V_(2, 0);
  double w0y = F_(1, 0) * V_(0, 0) + F_(1, 1) * V_(1, 0) + F_(1, 2) * V_(2, 0);
  double w0z = F_(2, 0) * V_(0, 0) + F_(2, 1) * V_(1, 0) + F_(2, 2) * V_(2, 0);
  double s0 = sqrt(w0x * w0x + w0y * w0y + w0z * w0z);
  if (s0 <= 1e-300) {
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        U_(r, c) = (r == c) ? 1.0 : 0.0;
        V_(r, c) = (r == c) ? 1.0 : 0.0;
      }
    S[0] = S[1] = S[2] = 0.0;
    return;
  }
  U_(0, 0) = w0x / s0;
  U_(1, 0) = w0y / s0;
  U_(2, 0) = w0z / s0;
  double w1x = F_(0, 0) * V_(0, 1) + F_(0, 1) * V_(1, 1) + F_(0, 2) * V_(2, 1);
  double w1y = F_(1, 0) * V_(0, 1) + F_(1, 1) * V_(1, 1) + F_(1, 2) * V_(2, 1);
  double w1z = F_(2, 0) * V_(0, 1) + F_(2, 1) * V_(1, 1) + F_(2, 2) * V_(2, 1);
  double dot01 = U_(0, 0) * w1x + U_(1, 0) * w1y + U_(2, 0) * w1z;
  w1x -= dot01 * U_(0, 0);
  w1y -= dot01 * U_(1, 0);
  w1z -= dot01 * U_(2, 0);
  double n1 = sqrt(w1x * w1x + w1y * w1y + w1z * w1z);
  double s1;
  if (n1 > 1e-12 * s0) {
    U_(0, 1) = w1x / n1;
    U_(1, 1) = w1y / n1;
    U_(2, 1) = w1z / n1;
    s1 = n1;
  } else {
    double ax = fabs(U_(0, 0)), ay = fabs(U_(1, 0)), az = fabs(U_(2, 0));
    double tx, ty, tz;
    if (ax <= ay && ax <= az) { tx = 1.0; ty = 0.0; tz = 0.0; }
    else if (ay <= az) { tx = 0.0; ty = 1.0; tz = 0.0; }
    else { tx = 0.0; ty = 0.0; tz = 1.0; }
    double dt = U_(0, 0) * tx + U_(1, 0) * ty + U_(2, 0) * tz;
    tx -= dt * U_(0, 0);
    ty -= dt * U_(1, 0);
    tz -= dt * U_(2, 0);
    double nt = sqrt(tx * tx + ty * ty + tz * tz);
    U_(0, 1) = tx / nt;
    U_(1, 1) = ty / nt;
    U_(2, 1) = tz / nt;
    s1 = 0.0;
  }
  U_(0, 2) = U_(1, 0) * U_(2, 1) - U_(2, 0) * U_(1, 1);
  U_(1, 2) = U_(2, 0) * U_(0, 1) - U_(0, 0) * U_(2, 1);
  U_(2, 2) = U_(0, 0) * U_(1, 1) - U_(1, 0) * U_(0, 1);
  S[0] = s0;
  S[1] = s1;
  double w2x = F_(0, 0) * V_(0, 2) + F_(0, 1) * V_(1, 2) + F_(0, 2) * V_(2, 2);
  double w2y = F_(1, 0) * V_(0, 2) + F_(1, 1) * V_(1, 2) + F_(1, 2) * V_(2, 2);
  double w2z = F_(2, 0) * V_(0, 2) + F_(2, 1) * V_(1, 2) + F_(2, 2) * V_(2, 2);
  S[2] = U_(0, 2) * w2x + U_(1, 2) * w2y + U_(2, 2) * w2z;
#undef F_
#undef U_
#undef V_
}

static void *svd_worker(void *arg) {
  svd_job *j = (svd_job *)arg;
  for (int64_t e = j->lo; e < j->hi; ++e) signed_svd1(j->F + 9 * e, j->U + 9 * e, j->S + 3 * e, j->V + 9 * e);
  return NULL;
}

void or_signed_svd(int64_t n, const double *F, double *U, double *S, double *V) {
  int T = or_threads();
  if (T == 1 || n < 4096) {
    svd_job j = {0, n, F, U, S, V};
    svd_worker(&j);
    return;
  }
  pthread_t th[256];
  svd_job jobs[256];
  for (int t = 0; t < T; ++t) {
    jobs[t].lo = n * t / T;
    jobs[t].hi = n * (t + 1) / T;
    jobs[t].F = F; jobs[t].U = U; jobs[t].S = S; jobs[t].V = V;
    pthread_create(&th[t], NULL, svd_worker, &jobs[t]);
  }
  for (int t = 0; t < T; ++t) pthread_join(th[t], NULL);
}

void or_uvt(int64_t n, const double *U, const double *V, double *out) {
  for (int64_t e = 0; e < n; ++e)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += U[9 * e + 3 * r + k] * V[9 * e + 3 * c + k];
        out[9 * e + 3 * r + c] = acc;
      }
}

void or_udvt(int64_t n, const double *U, const double *S, const double *V, double *out) {
  for (int64_t e = 0; e < n; ++e)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += U[9 * e + 3 * r + k] * S[3 * e + k] * V[9 * e + 3 * c + k];
        out[9 * e + 3 * r + c] = acc;
      }
}

/* x <- L^-1 x, column-oriented CSC with the diagonal first in each column. */
void or_lsolve(int64_t n, const int64_t *Lp, const int64_t *Li, const double *Lx, double *x) {
  for (int64_t j = 0; j < n; ++j) {
    double xj = x[j];
    if (xj != 0.0) {
      xj /= Lx[Lp[j]];
      x[j] = xj;
      for (int64_t p = Lp[j] + 1; p < Lp[j + 1]; ++p) x[Li[p]] -= Lx[p] * xj;
    }
  }
}

/* x <- L^-T x */
void or_ltsolve(int64_t n, const int64_t *Lp, const int64_t *Li, const double *Lx, double *x) {
  for (int64_t j = n - 1; j >= 0; --j) {
    double xj = x[j];
    for (int64_t p = Lp[j] + 1; p < Lp[j + 1]; ++p) xj -= Lx[p] * x[Li[p]];
    x[j] = xj / Lx[Lp[j]];
  }
}

/* Three RHS columns in one sweep over L (same arithmetic per column). */
void or_lsolve3(int64_t n, const int64_t *Lp, const int64_t *Li, const double *Lx, double *x /*(n,3) row-major*/) {
  for (int c = 0; c < 3; ++c)
    for (int64_t j = 0; j < n; ++j) {
      double xj = x[3 * j + c];
      if (xj != 0.0) {
        xj /= Lx[Lp[j]];
        x[3 * j + c] = xj;
        for (int64_t p = Lp[j] + 1; p < Lp[j + 1]; ++p) x[3 * Li[p] + c] -= Lx[p] * xj;
      }
    }
}

void or_ltsolve3(int64_t n, const int64_t *Lp, const int64_t *Li, const double *Lx, double *x) {
  for (int c = 0; c < 3; ++c)
    for (int64_t j = n - 1; j >= 0; --j) {
      double xj = x[3 * j + c];
      for (int64_t p = Lp[j] + 1; p < Lp[j + 1]; ++p) xj -= Lx[p] * x[3 * Li[p] + c];
      x[3 * j + c] = xj / Lx[Lp[j]];
    }
}
