// Probe: TMA tile::gather4 on a row-major float64 matrix (n x b, ld).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/g4 tools/probe_gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k_g4(const __grid_constant__ CUtensorMap tm, const int* rows, int nrows, int b, double* out) {
  __shared__ __align__(128) double sm[32 * 32];
  __shared__ __align__(8) uint64_t bar;
  const unsigned sbar = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::);
  }
  __syncthreads();
  const int ng = (nrows + 3) / 4;
  if (threadIdx.x == 0) {
    const unsigned bytes = ng * 4 * b * 8;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(bytes));
  }
  __syncwarp();
  if (threadIdx.x < ng) {
    const int t = threadIdx.x;
    int r[4];
    for (int i = 0; i < 4; ++i) r[i] = 4 * t + i < nrows ? rows[4 * t + i] : -1;
    const unsigned dst = (unsigned)__cvta_generic_to_shared(sm + 4 * t * b);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(sbar)
        : "memory");
  }
  // wait phase 0
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(sbar), "r"(0));
  }
  for (int i = threadIdx.x; i < ng * 4 * b; i += blockDim.x) out[i] = sm[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 1000, b = 20, ld = 22;
  std::vector<double> h(n * ld);
  for (int i = 0; i < n * ld; ++i) h[i] = i;
  double *dX, *dout;
  int* drows;
  cudaMalloc(&dX, h.size() * 8);
  cudaMalloc(&dout, 32 * 32 * 8);
  cudaMalloc(&drows, 32 * 4);
  cudaMemcpy(dX, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  int rows[32];
  for (int i = 0; i < 32; ++i) rows[i] = (i * 37 + 5) % n;
  cudaMemcpy(drows, rows, sizeof(rows), cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no encode fn\n"); return 1; }
  for (int boxh : {1, 4}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)b, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    cuuint32_t box[2] = {(cuuint32_t)b, (cuuint32_t)boxh};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dX, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("boxh %d encode %d\n", boxh, (int)r);
    if (r) continue;
    for (int nr : {32, 30}) {
      cudaMemset(dout, 0xff, 32 * 32 * 8);
      k_g4<<<1, 32>>>(tm, drows, nr, b, dout);
      cudaError_t e = cudaDeviceSynchronize();
      printf("  nrows %d: %s\n", nr, cudaGetErrorString(e));
      if (e) return 2;
      std::vector<double> o(32 * 32);
      cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int i = 0; i < 32; ++i)
        for (int c = 0; c < b; ++c) {
          double want = i < nr ? h[rows[i] * ld + c] : 0.0;
          if (o[i * b + c] != want) ++bad;
        }
      printf("  mismatches %d (row0 %g %g, row31 %g)\n", bad, o[0], o[1], o[31 * b]);
    }
  }
  return 0;
}
