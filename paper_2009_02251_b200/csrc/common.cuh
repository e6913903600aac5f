// Shared helpers for the svdrec_b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "../../include/svdrec_b200.h"

namespace svdrec {

void set_error(const char* fmt, ...);
void note_launches(int n);

// Check the last launch(es) and count ``n`` kernel launches issued by this
// library (svdrec_launch_count).
inline int check_launch(const char* what, int n = 1) {
  note_launches(n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

#define SVDREC_ARG(cond, ...)          \
  do {                                 \
    if (!(cond)) {                     \
      ::svdrec::set_error(__VA_ARGS__); \
      return SVDREC_E_ARG;             \
    }                                  \
  } while (0)

#define SVDREC_CUDA(call)                                                     \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      ::svdrec::set_error("%s:%d %s", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return (int)e_;                                                         \
    }                                                                         \
  } while (0)

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

int sm_count();

// occupancy (resident CTAs per SM) cached per (kernel, device, block, smem)
cudaError_t blocks_per_sm(const void* kernel, int threads, size_t smem, int* out);
template <class K>
cudaError_t blocks_per_sm(K* kernel, int threads, size_t smem, int* out) {
  return blocks_per_sm(reinterpret_cast<const void*>(kernel), threads, smem, out);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute is per device, so a process driving several GPUs sets it on
// each of them (lib.cu keeps the set of (kernel, device) pairs done).
bool smem_attr_done(const void* kernel, int dev);
void smem_attr_mark(const void* kernel, int dev);
template <class K>
cudaError_t smem_attr_once(K* kernel, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const void* key = reinterpret_cast<const void*>(kernel);
  if (smem_attr_done(key, dev)) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) smem_attr_mark(key, dev);
  return e;
}

// skinny.cu: tall-skinny GEMMs for q <= 32 (see the file header)
int64_t tn_skinny_slabs(int64_t r, int64_t p);
int launch_nn_skinny(int64_t r, int64_t p, int q, double alpha, const double* X, int64_t ldx, const double* C,
                     int64_t ldc, double beta, double* Y, int64_t ldy, cudaStream_t s);
bool launch_nn_wide(int64_t r, int64_t p, int64_t q, double alpha, const double* X, int64_t ldx, const double* C,
                    int64_t ldc, double beta, double* Y, int64_t ldy, cudaStream_t s, int* rc);
bool tn_tma_able(int64_t r, int64_t p, int64_t q, const double* X, int64_t ldx, const double* Y, int64_t ldy);
int launch_tn_skinny(int64_t r, int64_t p, int64_t q, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                     double* part, int64_t nslab, cudaStream_t s);

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic sum of p[k * stride] for k < n by one warp: lane l takes
// k = l, l+32, ... in order, then a fixed butterfly (valid in every lane).
// Replaces one-thread loops over split partials, which serialise n L2 round
// trips per output.
__device__ __forceinline__ double warp_strided_sum(const double* __restrict__ p, int64_t n, int64_t stride) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int64_t k = lane; k < n; k += 32) s += p[k * stride];
  return warp_sum(s);
}

// Fixed-order block sum (result valid in every thread). ``scratch`` holds
// blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < nw ? scratch[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) scratch[0] = t;
  }
  __syncthreads();
  t = scratch[0];
  __syncthreads();
  return t;
}

}  // namespace svdrec
