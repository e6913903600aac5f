// Probe: FP64 tensor (mma.sync m8n8k4 f64) vs FP64 FMA throughput on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_dmma tools/probe_dmma.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_dmma(int iters, double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

__global__ void k_dfma(int iters, double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(a, b, c[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int wpb : {4, 8, 16}) {
    const int iters = 20000;
    k_dmma<<<sms * 2, wpb * 32>>>(100, out);
    cudaEventRecord(e0);
    k_dmma<<<sms * 2, wpb * 32>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * sms * 2 * wpb;
    printf("dmma m8n8k4 %d warps/CTA x2: %.1f TFLOP/s (%s)\n", wpb, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    k_dfma<<<sms * 2, wpb * 32>>>(100, out);
    cudaEventRecord(e0);
    k_dfma<<<sms * 2, wpb * 32>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * 32 * (double)iters * sms * 2 * wpb;
    printf("dfma %d warps/CTA x2: %.1f TFLOP/s\n", wpb, flops / ms / 1e9);
  }
  return 0;
}
