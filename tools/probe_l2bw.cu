// Probe: L2-resident read bandwidth on B200 for the access shapes of the hot
// path (streaming, random row gathers through LDG, random rows through TMA
// bulk copies).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_l2bw tools/probe_l2bw.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void k_stream(const double2* __restrict__ a, int64_t n2, int reps, double* out) {
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < reps; ++r)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
      double2 v = __ldg(a + i);
      acc.x += v.x;
      acc.y += v.y;
    }
  if (acc.x == 12345.0) out[0] = acc.y;
}

// each warp gathers rows of ROWB bytes at random row indices; lanes cover the row with 16-B loads
template <int ROWD>
__global__ void k_gather(const double* __restrict__ a, int64_t nrows, const int* __restrict__ idx, int64_t nidx,
                         double* out) {
  constexpr int V = ROWD / 2;  // double2 per row
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0;
  for (int64_t b = w * 8; b < nidx; b += nw * 8) {
    double2 v[8][(V + 31) / 32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = idx[b + q];
#pragma unroll
      for (int t = 0; t < (V + 31) / 32; ++t) {
        const int c = lane + 32 * t;
        v[q][t] = c < V ? __ldg(reinterpret_cast<const double2*>(a + (int64_t)r * ROWD) + c) : make_double2(0, 0);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int t = 0; t < (V + 31) / 32; ++t) acc += v[q][t].x + v[q][t].y;
  }
  if (acc == 12345.0) out[0] = acc;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

// one warp per CTA slice: lane 0 issues bulk copies of whole rows into a ring of stages
template <int ROWD>
__global__ void k_bulk(const double* __restrict__ a, const int* __restrict__ idx, int64_t nidx, double* out) {
  constexpr int RPS = 8;  // rows per stage
  constexpr int S = 4;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[8 * S];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* ring = sm + (size_t)wib * S * RPS * ROWD;
  uint64_t* bar = bars + wib * S;
  if (lane < S) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(bar + lane)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t nst = 0;
  for (int64_t b = w * RPS; b < nidx; b += nw * RPS) ++nst;
  double acc = 0;
  auto issue = [&](int64_t st) {
    const int slot = (int)(st % S);
    const int64_t b = (w + st * nw) * RPS;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar + slot)),
                   "r"(RPS * ROWD * 8) : "memory");
    __syncwarp();
    if (lane < RPS) bulk_g2s(ring + (slot * RPS + lane) * ROWD, a + (int64_t)idx[b + lane] * ROWD, ROWD * 8, bar + slot);
  };
  for (int64_t st = 0; st < S - 1 && st < nst; ++st) issue(st);
  for (int64_t st = 0; st < nst; ++st) {
    if (st + S - 1 < nst) issue(st + S - 1);
    const int slot = (int)(st % S);
    unsigned done = 0, par = (unsigned)((st / S) & 1);
    do {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"((unsigned)__cvta_generic_to_shared(bar + slot)), "r"(par) : "memory");
    } while (!done);
    const double* rs = ring + slot * RPS * ROWD;
    for (int e = lane; e < RPS * ROWD; e += 32) acc += rs[e];
    __syncwarp();
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t bytes = 48ll << 20;  // L2-resident
  double* a;
  double* out;
  cudaMalloc(&a, bytes);
  cudaMalloc(&out, 64);
  cudaMemset(a, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // streaming
  for (int g : {sms * 2, sms * 4, sms * 8}) {
    k_stream<<<g, 512>>>((double2*)a, bytes / 16, 1, out);
    cudaEventRecord(e0);
    k_stream<<<g, 512>>>((double2*)a, bytes / 16, 10, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("stream grid %d: %.1f GB/s\n", g, 10.0 * bytes / ms / 1e6);
  }
  // random gathers
  const int64_t nidx = 1 << 22;
  int* idx;
  cudaMalloc(&idx, nidx * 4);
  int* h = (int*)malloc(nidx * 4);
  uint64_t s = 88172645463325252ull;
  auto run_gather = [&](auto kern, int rowd, int tpb, int blocks_per_sm) {
    const int64_t nrows = bytes / (rowd * 8);
    for (int64_t i = 0; i < nidx; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (int)(s % nrows);
    }
    cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice);
    kern<<<sms * blocks_per_sm, tpb>>>(a, nrows, idx, nidx, out);
    cudaEventRecord(e0);
    kern<<<sms * blocks_per_sm, tpb>>>(a, nrows, idx, nidx, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("gather row %d B, %d x %d thr/SM: %.1f GB/s (%s)\n", rowd * 8, blocks_per_sm, tpb,
           (double)nidx * rowd * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run_gather(k_gather<20>, 20, 256, 4);
  run_gather(k_gather<20>, 20, 256, 8);
  run_gather(k_gather<24>, 24, 256, 8);
  run_gather(k_gather<32>, 32, 256, 8);
  run_gather(k_gather<16>, 16, 256, 8);
  run_gather(k_gather<64>, 64, 256, 8);
  run_gather(k_gather<240>, 240, 256, 2);
  run_gather(k_gather<240>, 240, 256, 4);
  // bulk copies
  auto run_bulk = [&](auto kern, int rowd, int warps) {
    const int64_t nrows = bytes / (rowd * 8);
    for (int64_t i = 0; i < nidx; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (int)(s % nrows);
    }
    cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice);
    const size_t smem = (size_t)warps * 4 * 8 * rowd * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<sms, warps * 32, smem>>>(a, idx, nidx, out);
    cudaEventRecord(e0);
    kern<<<sms, warps * 32, smem>>>(a, idx, nidx, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("bulk row %d B, %d warps/SM smem %zu: %.1f GB/s (%s)\n", rowd * 8, warps, smem,
           (double)nidx * rowd * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run_bulk(k_bulk<20>, 20, 8);
  run_bulk(k_bulk<240>, 240, 2);
  run_bulk(k_bulk<240>, 240, 3);
  return 0;
}
