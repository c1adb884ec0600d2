/*
 * ORACLE -- test infrastructure only, never a product path.
 *
 * Plain-C restatement of the two column loops of the LU-with-incremental-pivoting
 * oracle (oracle/tiles_lu_qr.py getrf_inc / tstrf), i.e. of PLASMA's
 * core_dgetrf_incpiv panel (partial pivoting inside the panel rows) and
 * core_dtstrf panel (pairwise pivoting of [U; A], swap-behind into dL).  The
 * reference DAG kinds they stand for: /root/reference/pkg/src/hetsim/kernels.py:28-33,
 * access lists kernels.py:152-167.
 *
 * Same operations in the same order as the NumPy oracle -- x *= (1 / pivot),
 * then a -= x * u (two roundings; built with -ffp-contract=off, no FMA), first
 * maximal |.| wins -- so the results are bit-identical to it
 * (tests/test_oracle_numeric.py::test_c_panels_match_numpy).  It exists because
 * the NumPy column loop costs ~0.6 s per nb=1024 TSTRF, and the 496 TSTRFs of an
 * N=32768 LU form a serial chain (each RWs the diagonal tile).
 *
 * Tiles are column-major with leading dimension ld.  Build: oracle/Makefile
 * (or __graft_entry__.build()) -> oracle/liboracle.so.
 */
#include <math.h>
#include <stdint.h>

/* core_dgetrf_incpiv panel on columns [ii, ii+sb) of the m x n tile a (rows [ii, m) take part).
 * ipiv[j] = absolute row swapped with row j.  Returns 1 if an exactly zero pivot was met. */
int ora_getrf_panel(double* a, int lda, int m, int ii, int sb, int64_t* ipiv) {
  int singular = 0;
  for (int j = ii; j < ii + sb; ++j) {
    double* cj = a + (int64_t)j * lda;
    int p = j;
    double best = fabs(cj[j]);
    for (int r = j + 1; r < m; ++r) {
      const double v = fabs(cj[r]);
      if (v > best) {
        best = v;
        p = r;
      }
    }
    ipiv[j] = p;
    if (p != j) {
      for (int c = ii; c < ii + sb; ++c) {
        double* col = a + (int64_t)c * lda;
        const double t = col[j];
        col[j] = col[p];
        col[p] = t;
      }
    }
    if (cj[j] == 0.0) {
      singular = 1;
      continue;
    }
    const double inv = 1.0 / cj[j];
    for (int r = j + 1; r < m; ++r) cj[r] *= inv;
    for (int c = j + 1; c < ii + sb; ++c) {
      double* col = a + (int64_t)c * lda;
      const double u = col[j];
      for (int r = j + 1; r < m; ++r) {
        const double prod = cj[r] * u;
        col[r] -= prod;
      }
    }
  }
  return singular;
}

/* core_dtstrf panel on columns [ii, ii+sb) of (u: n x n upper tile, a: m x n tile).
 * ipiv[j] = row of a swapped with u row j, or unchanged (-1 preset by the caller);
 * dl (ib x n, leading dimension lddl) row j-ii gets a's earlier panel multipliers of the
 * row that moved up.  Returns 1 if an exactly zero pivot was met. */
int ora_tstrf_panel(double* u, int ldu, double* a, int lda, int m, int ii, int sb, int64_t* ipiv, double* dl,
                    int lddl) {
  int singular = 0;
  for (int j = ii; j < ii + sb; ++j) {
    double* aj = a + (int64_t)j * lda;
    int r = 0;
    double best = fabs(aj[0]);
    for (int q = 1; q < m; ++q) {
      const double v = fabs(aj[q]);
      if (v > best) {
        best = v;
        r = q;
      }
    }
    if (fabs(aj[r]) > fabs(u[j + (int64_t)j * ldu])) {
      for (int c = j; c < ii + sb; ++c) {
        double* uc = u + (int64_t)c * ldu;
        double* ac = a + (int64_t)c * lda;
        const double t = uc[j];
        uc[j] = ac[r];
        ac[r] = t;
      }
      for (int c = ii; c < j; ++c) {
        double* ac = a + (int64_t)c * lda;
        dl[(j - ii) + (int64_t)c * lddl] = ac[r];
        ac[r] = 0.0;
      }
      ipiv[j] = r;
    }
    const double piv = u[j + (int64_t)j * ldu];
    if (piv == 0.0) {
      singular = 1;
      continue;
    }
    const double inv = 1.0 / piv;
    for (int q = 0; q < m; ++q) aj[q] *= inv;
    for (int c = j + 1; c < ii + sb; ++c) {
      double* ac = a + (int64_t)c * lda;
      const double uv = u[j + (int64_t)c * ldu];
      for (int q = 0; q < m; ++q) {
        const double prod = aj[q] * uv;
        ac[q] -= prod;
      }
    }
  }
  return singular;
}
