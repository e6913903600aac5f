/* CPU oracle, TEST INFRASTRUCTURE ONLY: the reference's per-sample Alg. 4
 * scoring loop (reference pkg/src/svdrec/cf.py:108-143, ``_predict``) in
 * plain C, samples spread over POSIX threads (dynamic blocks of 64).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs load this (through oracle/svdrec_oracle.py); the
 * product never does.  Same arithmetic as the reference per sample: for
 * every rated item l of the user with a nonzero factor norm, the cosine
 * sim_l = (T_l . T_j) / (|T_l| |T_j|); weight = sum sim_l; raw = (sum sim_l
 * r_l) / weight, clamped to [lo, hi]; the user's mean rating (or the global
 * mean for a user without ratings) when the item or every rated item has a
 * zero norm, or |weight| < 1e-9 (cf.py:23).  Sums run in rating order
 * (numpy's pairwise sums may round differently in the last bits).
 *
 * Built by __graft_entry__.build() / oracle/Makefile into
 * oracle/libsvdrec_oracle.so (no -march: the dot product is cloned for
 * AVX-512 / AVX2 / baseline x86-64 and picked at load time).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>

#define WEIGHT_FLOOR 1e-9

typedef double v4d __attribute__((vector_size(32)));

/* dot product in 8 interleaved partial sums (two 4-wide vectors), combined
 * at the end; the row of the next rated item is prefetched meanwhile */
__attribute__((target_clones("avx512f", "avx2", "default"))) static double dot(const double* a, const double* b,
                                                                                 int64_t k) {
  v4d s0 = {0, 0, 0, 0}, s1 = {0, 0, 0, 0};
  int64_t i = 0;
  for (; i + 8 <= k; i += 8) {
    v4d a0, a1, b0, b1;
    __builtin_memcpy(&a0, a + i, 32);
    __builtin_memcpy(&a1, a + i + 4, 32);
    __builtin_memcpy(&b0, b + i, 32);
    __builtin_memcpy(&b1, b + i + 4, 32);
    s0 += a0 * b0;
    s1 += a1 * b1;
  }
  double t = 0.0;
  for (; i < k; ++i) t += a[i] * b[i];
  const v4d s = s0 + s1;
  return ((s[0] + s[1]) + (s[2] + s[3])) + t;
}

static double clamp(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

typedef struct {
  int64_t ns;
  const int64_t *users, *items, *indptr;
  const int32_t* indices;
  const double *data, *Tt, *norms;
  int64_t k;
  double lo, hi, gmean;
  double *value, *raw;
  uint8_t* fallback;
  int64_t next; /* next block of samples (atomic) */
} Job;

static void score(const Job* J, int64_t s) {
  const int64_t u = J->users[s], j = J->items[s];
  const int64_t a = J->indptr[u], e = J->indptr[u + 1];
  const int64_t k = J->k;
  const double nj = J->norms[j];
  int fb = 1;
  double r = 0.0;
  if (nj != 0.0 && e > a) {
    const double* tj = J->Tt + j * k;
    double w = 0.0, num = 0.0;
    int known = 0;
    for (int64_t t = a; t < e; ++t) {
      const int64_t l = J->indices[t];
      if (t + 2 < e) {
        const char* nx = (const char*)(J->Tt + (int64_t)J->indices[t + 2] * k);
        for (int64_t o = 0; o < k * 8; o += 64) __builtin_prefetch(nx + o);
      }
      const double nl = J->norms[l];
      if (nl > 0.0) {
        const double sim = dot(J->Tt + l * k, tj, k) / (nl * nj);
        w += sim;
        num += sim * J->data[t];
        known = 1;
      }
    }
    if (known && fabs(w) >= WEIGHT_FLOOR) {
      r = num / w;
      fb = 0;
    }
  }
  if (fb) {
    if (e > a) {
      double m = 0.0;
      for (int64_t t = a; t < e; ++t) m += J->data[t];
      r = m / (double)(e - a);
    } else {
      r = J->gmean;
    }
  }
  J->raw[s] = r;
  J->value[s] = clamp(r, J->lo, J->hi);
  J->fallback[s] = (uint8_t)fb;
}

static void* worker(void* arg) {
  Job* J = (Job*)arg;
  for (;;) {
    const int64_t s0 = __atomic_fetch_add(&J->next, 64, __ATOMIC_RELAXED);
    if (s0 >= J->ns) break;
    const int64_t s1 = s0 + 64 < J->ns ? s0 + 64 : J->ns;
    for (int64_t s = s0; s < s1; ++s) score(J, s);
  }
  return 0;
}

/* Tt: n x k row-major (row l = column l of T); norms[l] = |T_l|. */
int svdrec_oracle_predict(int64_t ns, const int64_t* users, const int64_t* items, const int64_t* indptr,
                          const int32_t* indices, const double* data, const double* Tt, int64_t k,
                          const double* norms, double lo, double hi, double gmean, double* value, double* raw,
                          uint8_t* fallback, int nthreads) {
  Job J = {ns, users, items, indptr, indices, data, Tt, norms, k, lo, hi, gmean, value, raw, fallback, 0};
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  int started = 0;
  for (int i = 1; i < nthreads; ++i)
    if (pthread_create(&th[started], 0, worker, &J) == 0) ++started;
  worker(&J);
  for (int i = 0; i < started; ++i) pthread_join(th[i], 0);
  return 0;
}
