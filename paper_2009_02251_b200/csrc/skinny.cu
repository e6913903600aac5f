// Tall-skinny float64 GEMMs for the QB deflations (q = block width <= 32).
//
//   nn:  Y (r x q) = alpha X (r x p) C (p x q) + beta Y      (Q @ C, B.T @ C)
//   tn:  part[s]   = X[slab s].T @ Y[slab s]  (p x q)        (Q.T @ Y, B @ X)
//
// Reference: the products Q @ (B @ X), Q @ (Q.T @ X), B.T @ (Q.T @ X) of
// rsvd.py:135-142, 179-194.  X (Q or B.T, r x k with k up to the rank cap)
// is the only large operand, so both kernels are built to stream it: 32-deep
// stages double-buffered through cp.async (LDGSTS) so the next tile is in
// flight while the current one is multiplied, and 4 x ceil(q/8) outputs per
// thread so every shared-memory read feeds several FMAs.  r x q operands
// (Y, C) are tiny.  The tn reduction over r is split into row slabs whose
// partials the caller sums in a fixed order (deterministic).
#include "common.cuh"

namespace svdrec {
namespace {

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;  // src-size 0: zero-fill, nothing read
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

constexpr int kT = 256;  // threads: 32 row (or p) groups x 8 q groups
constexpr int RT = 128;  // nn: rows per CTA (4 per thread)
constexpr int KP = 32;   // nn: p per stage
constexpr int PT = 128;  // tn: p per CTA (4 per thread)
constexpr int RB = 32;   // tn: rows per stage

struct NnSmem {
  double x[2][RT][KP + 1];
  double c[2][KP][33];
};
struct TnSmem {
  double x[2][RB][PT + 1];
  double y[2][RB][33];
};

template <int QPT>
__global__ void __launch_bounds__(kT) k_nn_skinny(int64_t r, int64_t p, int q, double alpha,
                                                  const double* __restrict__ X, int64_t ldx,
                                                  const double* __restrict__ C, int64_t ldc, double beta,
                                                  double* __restrict__ Y, int64_t ldy) {
  extern __shared__ __align__(16) unsigned char smraw[];
  NnSmem& sm = *reinterpret_cast<NnSmem*>(smraw);
  const int qg = threadIdx.x & 7, rg = threadIdx.x >> 3;
  const int64_t r0 = (int64_t)blockIdx.x * RT;
  const int nst = (int)((p + KP - 1) / KP);
  auto issue = [&](int st, int buf) {
    const int64_t k0 = (int64_t)st * KP;
    for (int e = threadIdx.x; e < RT * KP; e += kT) {
      const int rr = e / KP, kk = e % KP;
      const int64_t gr = r0 + rr, gk = k0 + kk;
      const bool ok = gr < r && gk < p;
      cp_async8(&sm.x[buf][rr][kk], ok ? X + gr * ldx + gk : X, ok);
    }
    for (int e = threadIdx.x; e < KP * 32; e += kT) {
      const int kk = e / 32, qq = e % 32;
      const int64_t gk = k0 + kk;
      const bool ok = gk < p && qq < q;
      cp_async8(&sm.c[buf][kk][qq], ok ? C + gk * ldc + qq : C, ok);
    }
    cp_commit();
  };
  double acc[4][QPT];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < QPT; ++j) acc[i][j] = 0.0;
  issue(0, 0);
  for (int st = 0; st < nst; ++st) {
    const int buf = st & 1;
    if (st + 1 < nst) {
      issue(st + 1, buf ^ 1);
      cp_wait1();
    } else {
      cp_wait0();
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < KP; ++kk) {
      double xv[4], cv[QPT];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = sm.x[buf][rg * 4 + i][kk];
#pragma unroll
      for (int j = 0; j < QPT; ++j) cv[j] = sm.c[buf][kk][qg * QPT + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < QPT; ++j) acc[i][j] = fma(xv[i], cv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gr = r0 + rg * 4 + i;
    if (gr >= r) continue;
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
      const int qq = qg * QPT + j;
      if (qq >= q) continue;
      double* y = Y + gr * ldy + qq;
      *y = beta == 0.0 ? alpha * acc[i][j] : fma(alpha, acc[i][j], beta * *y);
    }
  }
}

template <int QPT>
__global__ void __launch_bounds__(kT) k_tn_skinny(int64_t r, int64_t p, int q, const double* __restrict__ X,
                                                  int64_t ldx, const double* __restrict__ Y, int64_t ldy,
                                                  double* __restrict__ part, int64_t rows_per) {
  extern __shared__ __align__(16) unsigned char smraw[];
  TnSmem& sm = *reinterpret_cast<TnSmem*>(smraw);
  const int qg = threadIdx.x & 7, pg = threadIdx.x >> 3;
  const int64_t p0 = (int64_t)blockIdx.y * PT;
  const int64_t rs = (int64_t)blockIdx.x * rows_per, re = min64(r, rs + rows_per);
  const int nst = (int)((re - rs + RB - 1) / RB);
  auto issue = [&](int st, int buf) {
    const int64_t b0 = rs + (int64_t)st * RB;
    for (int e = threadIdx.x; e < RB * PT; e += kT) {
      const int rr = e / PT, pp = e % PT;
      const int64_t gr = b0 + rr, gp = p0 + pp;
      const bool ok = gr < re && gp < p;
      cp_async8(&sm.x[buf][rr][pp], ok ? X + gr * ldx + gp : X, ok);
    }
    for (int e = threadIdx.x; e < RB * 32; e += kT) {
      const int rr = e / 32, qq = e % 32;
      const int64_t gr = b0 + rr;
      const bool ok = gr < re && qq < q;
      cp_async8(&sm.y[buf][rr][qq], ok ? Y + gr * ldy + qq : Y, ok);
    }
    cp_commit();
  };
  double acc[4][QPT];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < QPT; ++j) acc[i][j] = 0.0;
  if (nst > 0) issue(0, 0);
  for (int st = 0; st < nst; ++st) {
    const int buf = st & 1;
    if (st + 1 < nst) {
      issue(st + 1, buf ^ 1);
      cp_wait1();
    } else {
      cp_wait0();
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < RB; ++rr) {
      double xv[4], yv[QPT];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = sm.x[buf][rr][pg * 4 + i];
#pragma unroll
      for (int j = 0; j < QPT; ++j) yv[j] = sm.y[buf][rr][qg * QPT + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < QPT; ++j) acc[i][j] = fma(xv[i], yv[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* dst = part + (int64_t)blockIdx.x * p * q;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gp = p0 + pg * 4 + i;
    if (gp >= p) continue;
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
      const int qq = qg * QPT + j;
      if (qq < q) dst[gp * q + qq] = acc[i][j];
    }
  }
}

template <int QPT>
int nn_launch(int64_t r, int64_t p, int q, double alpha, const double* X, int64_t ldx, const double* C, int64_t ldc,
              double beta, double* Y, int64_t ldy, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    SVDREC_CUDA(cudaFuncSetAttribute(k_nn_skinny<QPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(NnSmem)));
    attr = true;
  }
  k_nn_skinny<QPT><<<(unsigned)((r + RT - 1) / RT), kT, sizeof(NnSmem), s>>>(r, p, q, alpha, X, ldx, C, ldc, beta,
                                                                            Y, ldy);
  return check_launch("gemm_nn_skinny");
}

template <int QPT>
int tn_launch(int64_t r, int64_t p, int q, const double* X, int64_t ldx, const double* Y, int64_t ldy, double* part,
              int64_t nslab, int64_t rows_per, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    SVDREC_CUDA(cudaFuncSetAttribute(k_tn_skinny<QPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(TnSmem)));
    attr = true;
  }
  dim3 grid((unsigned)nslab, (unsigned)((p + PT - 1) / PT));
  k_tn_skinny<QPT><<<grid, kT, sizeof(TnSmem), s>>>(r, p, q, X, ldx, Y, ldy, part, rows_per);
  return check_launch("gemm_tn_skinny");
}

}  // namespace

int64_t tn_skinny_slabs(int64_t r, int64_t p) {
  const int64_t gy = (p + PT - 1) / PT;
  int64_t s = (3 * (int64_t)sm_count() + gy - 1) / gy;
  const int64_t max_s = (r + 4 * RB - 1) / (4 * RB);  // >= 4 stages per slab
  if (s > max_s) s = max_s;
  return s < 1 ? 1 : s;
}

int launch_nn_skinny(int64_t r, int64_t p, int q, double alpha, const double* X, int64_t ldx, const double* C,
                     int64_t ldc, double beta, double* Y, int64_t ldy, cudaStream_t s) {
  const int qpt = (q + 7) / 8;
  switch (qpt) {
    case 1: return nn_launch<1>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
    case 2: return nn_launch<2>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
    case 3: return nn_launch<3>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
    default: return nn_launch<4>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
  }
}

int launch_tn_skinny(int64_t r, int64_t p, int q, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                     double* part, int64_t nslab, cudaStream_t s) {
  const int64_t rows_per = (r + nslab - 1) / nslab;
  const int qpt = (q + 7) / 8;
  switch (qpt) {
    case 1: return tn_launch<1>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s);
    case 2: return tn_launch<2>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s);
    case 3: return tn_launch<3>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s);
    default: return tn_launch<4>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s);
  }
}

}  // namespace svdrec
