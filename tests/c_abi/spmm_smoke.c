/* A plain-C consumer of libsvdrec_b200.so (no Python, no torch): the
 * binding a C / cgo / JNI host would write.  Builds a random CSR, runs
 * svdrec_spmm with (a) the trivial plan -- one segment per row, no warp
 * schedule -- and (b) a contiguous warp schedule with the chunk plan the
 * library builds from it (svdrec_chunk_plan / svdrec_warp_chunks: the
 * pipelined TMA path), and checks both against a host loop; then checks
 * the error contract.
 * Exit code 0 = pass.  Build: see tests/test_gpu_c_abi.py. */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "svdrec_b200.h"

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 2;                                                            \
    }                                                                      \
  } while (0)

static uint64_t rng = 88172645463325252ull;
static double urand(void) {
  rng ^= rng << 13, rng ^= rng >> 7, rng ^= rng << 17;
  return (double)(rng >> 11) / 9007199254740992.0;
}

static void* dev_copy(const void* h, size_t n) {
  void* d = NULL;
  if (cudaMalloc(&d, n ? n : 16) != cudaSuccess) return NULL;
  if (n) cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
  return d;
}

int main(void) {
  if (svdrec_abi_version() != 1) return 3;
  const int64_t m = 5000, n = 700;
  const int b = 20;
  int64_t* indptr = malloc((m + 1) * sizeof(int64_t));
  indptr[0] = 0;
  for (int64_t i = 0; i < m; ++i) indptr[i + 1] = indptr[i] + 1 + (int64_t)(urand() * (i % 97 == 0 ? 2500 : 30));
  const int64_t nnz = indptr[m];
  int32_t* ind = malloc(nnz * sizeof(int32_t));
  double* val = malloc(nnz * sizeof(double));
  for (int64_t i = 0; i < m; ++i) {  /* increasing columns per row */
    int64_t len = indptr[i + 1] - indptr[i];
    int32_t c = (int32_t)(urand() * 3);
    for (int64_t t = 0; t < len; ++t) {
      ind[indptr[i] + t] = c % (int32_t)n;
      val[indptr[i] + t] = 0.5 * (1 + (int)(urand() * 10));
      c += 1 + (int32_t)(urand() * 2);
    }
  }
  double* X = malloc(n * b * sizeof(double));
  for (int64_t t = 0; t < n * b; ++t) X[t] = urand() - 0.5;
  double* ref = calloc(m * b, sizeof(double));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t t = indptr[i]; t < indptr[i + 1]; ++t)
      for (int j = 0; j < b; ++j) ref[i * b + j] += val[t] * X[(int64_t)ind[t] * b + j];

  /* trivial plan: one segment per row, direct stores, no split rows */
  int32_t* seg_row = malloc(m * sizeof(int32_t));
  int32_t* seg_slot = malloc(m * sizeof(int32_t));
  for (int64_t i = 0; i < m; ++i) seg_row[i] = (int32_t)i, seg_slot[i] = -1;
  int32_t* d_seg_row = dev_copy(seg_row, m * 4);
  int64_t* d_seg_begin = dev_copy(indptr, m * 8);
  int64_t* d_seg_end = dev_copy(indptr + 1, m * 8);
  int32_t* d_seg_slot = dev_copy(seg_slot, m * 4);
  int32_t* d_ind = dev_copy(ind, nnz * 4);
  double* d_val = dev_copy(val, nnz * 8);
  double* d_X = dev_copy(X, n * b * 8);
  double *d_Y = NULL, *d_part = NULL;
  CK(cudaMalloc((void**)&d_Y, m * b * 8));
  CK(cudaMalloc((void**)&d_part, 16 * b * 8));
  double* Y = malloc(m * b * sizeof(double));
  int fails = 0;
  for (int pass = 0; pass < 2; ++pass) {
    int64_t nwarp = 0;
    int32_t *d_ws = NULL, *d_wc = NULL;
    int64_t* d_cbase = NULL;
    void* d_recs = NULL;
    if (pass == 1) { /* contiguous warp ranges of about equal nonzeros */
      nwarp = (int64_t)svdrec_device_sm_count() * svdrec_spmm_warps_per_sm(b);
      if (nwarp > m) nwarp = m;
      int32_t* ws = malloc((nwarp + 1) * sizeof(int32_t));
      int64_t r = 0;
      for (int64_t w = 0; w <= nwarp; ++w) {
        const int64_t target = nnz * w / nwarp;
        while (r < m && indptr[r] < target) ++r;
        ws[w] = (int32_t)(w == nwarp ? m : r);
        if (w && ws[w] < ws[w - 1]) ws[w] = ws[w - 1];
      }
      d_ws = dev_copy(ws, (nwarp + 1) * 4);
      free(ws);
      CK(cudaMalloc((void**)&d_cbase, (m + 1) * 8));
      CK(cudaMalloc(&d_recs, (nnz / 32 + 2 * m) * 16));
      CK(cudaMalloc((void**)&d_wc, (nwarp + 1) * 4));
      int prc = svdrec_chunk_plan(m, d_seg_row, d_seg_begin, d_seg_end, d_seg_slot, NULL, NULL, d_cbase, d_recs, NULL);
      if (!prc) prc = svdrec_warp_chunks(nwarp, d_ws, m, d_cbase, d_wc, NULL);
      if (prc) {
        fprintf(stderr, "chunk plan: %s\n", svdrec_last_error());
        return 4;
      }
    }
    CK(cudaMemset(d_Y, 0, m * b * 8));
    int rc = svdrec_spmm(m, d_seg_row, d_seg_begin, d_seg_end, d_seg_slot, d_ind, d_val, d_X, b, n, d_Y, b, b, 0,
                         NULL, NULL, NULL, nwarp, d_ws, d_wc, d_recs, NULL, NULL, d_part, NULL);
    if (rc) {
      fprintf(stderr, "svdrec_spmm: %s\n", svdrec_last_error());
      return 4;
    }
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(Y, d_Y, m * b * 8, cudaMemcpyDeviceToHost));
    double worst = 0.0;
    for (int64_t t = 0; t < m * b; ++t) {
      const double d = fabs(Y[t] - ref[t]) / (1.0 + fabs(ref[t]));
      if (d > worst) worst = d;
    }
    printf("pass %d (nwarp %lld): max rel err %.3e\n", pass, (long long)nwarp, worst);
    if (!(worst <= 1e-12)) ++fails;
    if (d_ws) cudaFree(d_ws);
    if (d_wc) cudaFree(d_wc);
    if (d_cbase) cudaFree(d_cbase);
    if (d_recs) cudaFree(d_recs);
  }
  /* error contract: bad arguments -> nonzero status and a message */
  int rc = svdrec_spmm(m, d_seg_row, d_seg_begin, d_seg_end, d_seg_slot, d_ind, d_val, d_X, 1, n, d_Y, b, b, 0, NULL,
                       NULL, NULL, 0, NULL, NULL, NULL, NULL, NULL, d_part, NULL);
  if (rc == 0 || svdrec_last_error()[0] == 0) ++fails;
  printf("bad ldx -> rc %d: %s\n", rc, svdrec_last_error());
  printf("%s\n", fails ? "FAIL" : "PASS");
  return fails ? 1 : 0;
}
