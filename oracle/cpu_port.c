/* CPU oracle, TEST INFRASTRUCTURE ONLY: the reference's sparse products
 * (reference pkg/src/svdrec/linalg.py:141-158, ``sparse_dense_mul``: scipy
 * ``A @ X`` / ``A.T @ X``) as a threaded CSR x dense kernel, so the oracle
 * port of the whole Alg. 5 pipeline runs on all host cores (bench.py's
 * cpu_baseline / --impl reference legs time it; tests check it against
 * scipy).  The product never loads this library.
 *
 * Y[r, :] = sum_t data[t] * X[indices[t], :] for t in row r, summed in
 * index order -- the order scipy's csr_matvecs uses, so the result equals
 * scipy's bit for bit.  A.T @ X is the same call on the CSR of A.T
 * (scipy's csc_matvecs scatters in row order, which for a fixed output
 * element is again ascending source-row order).  Rows are handed out in
 * dynamic blocks of 256 over POSIX threads.
 */
#include <pthread.h>
#include <stdint.h>
#include <string.h>

typedef struct {
  int64_t m, b;
  const int64_t* indptr;
  const int32_t* indices;
  const double* data;
  const double* X;
  double* Y;
  int64_t next;
} SpJob;

__attribute__((target_clones("avx512f", "avx2", "default"))) static void row(const SpJob* J, int64_t r) {
  const int64_t b = J->b;
  double* y = J->Y + r * b;
  memset(y, 0, (size_t)b * sizeof(double));
  for (int64_t t = J->indptr[r]; t < J->indptr[r + 1]; ++t) {
    const double v = J->data[t];
    const double* x = J->X + (int64_t)J->indices[t] * b;
    for (int64_t c = 0; c < b; ++c) y[c] += v * x[c];
  }
}

static void* sp_worker(void* arg) {
  SpJob* J = (SpJob*)arg;
  for (;;) {
    const int64_t r0 = __atomic_fetch_add(&J->next, 256, __ATOMIC_RELAXED);
    if (r0 >= J->m) break;
    const int64_t r1 = r0 + 256 < J->m ? r0 + 256 : J->m;
    for (int64_t r = r0; r < r1; ++r) row(J, r);
  }
  return 0;
}

/* X: rows x b row-major (rows = column count of the CSR); Y: m x b. */
int svdrec_oracle_spmm(int64_t m, const int64_t* indptr, const int32_t* indices, const double* data,
                       const double* X, int64_t b, double* Y, int nthreads) {
  SpJob J = {m, b, indptr, indices, data, X, Y, 0};
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  int started = 0;
  for (int i = 1; i < nthreads; ++i)
    if (pthread_create(&th[started], 0, sp_worker, &J) == 0) ++started;
  sp_worker(&J);
  for (int i = 0; i < started; ++i) pthread_join(th[i], 0);
  return 0;
}
