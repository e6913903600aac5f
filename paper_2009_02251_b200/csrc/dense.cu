// Dense tall-skinny contractions and fixed-order reductions (float64).
//
// The QB loop's deflation products (reference rsvd.py:135-142, 179-194):
//   Q @ (B @ X)    -> gemm_tn(Bt, X) then gemm_nn(Q, ., alpha=-1, beta=1)
//   Q @ (Q.T @ X)  -> gemm_tn(Q, X)  then gemm_nn(Q, ., -1, 1)
//   B.T @ (Q.T @ q)-> gemm_tn(Q, q)  then gemm_nn(Bt, ., -1, 1)
// plus the Gram of eig_svd (linalg.py:127, B @ B.T = Bt.T @ Bt) and the
// Frobenius / row-energy reductions of the error indicator (rsvd.py:146,
// 197, 209).  Q (m x K) and Bt = B.T (n x K) are row-major with a fixed
// leading dimension so a new block is appended by writing K..K+b columns.
//
// All reductions over the tall dimension are split across CTAs into a
// partial buffer and summed in a fixed order, so results are bitwise
// reproducible.  Round-1 tiles are classic smem-tiled FMA (fp64 has no
// tensor-core advantage on B200: DMMA and DFMA peak at the same rate);
// both kernels are bound by streaming the tall operand from HBM.
#include "common.cuh"

namespace svdrec {
namespace {

constexpr int TP = 64;   // output rows per CTA tile (the p / r direction)
constexpr int TK = 16;   // reduction step

// ---- gemm_tn: partial[s] = X[rs:re].T @ Y[rs:re] ---------------------------
// thread (tx, ty) in 16 x 16 computes outputs p = p0 + ty*4 + i, q = q0 + tx*QT + j
template <int QT>
__global__ void __launch_bounds__(256) k_gemm_tn(int64_t r, int64_t p, int64_t q, const double* __restrict__ X,
                                                 int64_t ldx, const double* __restrict__ Y, int64_t ldy,
                                                 double* __restrict__ part, int64_t rows_per_split) {
  constexpr int TQ = 16 * QT;
  __shared__ double Xs[TK][TP + 1];
  __shared__ double Ys[TK][TQ + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t p0 = (int64_t)blockIdx.x * TP, q0 = (int64_t)blockIdx.y * TQ;
  const int64_t rs = (int64_t)blockIdx.z * rows_per_split;
  const int64_t re = min(r, rs + rows_per_split);
  double acc[4][QT];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < QT; ++j) acc[i][j] = 0.0;
  for (int64_t r0 = rs; r0 < re; r0 += TK) {
    for (int e = threadIdx.x; e < TK * TP; e += 256) {
      const int rr = e / TP, pp = e % TP;
      const int64_t gr = r0 + rr, gp = p0 + pp;
      Xs[rr][pp] = (gr < re && gp < p) ? X[gr * ldx + gp] : 0.0;
    }
    for (int e = threadIdx.x; e < TK * TQ; e += 256) {
      const int rr = e / TQ, qq = e % TQ;
      const int64_t gr = r0 + rr, gq = q0 + qq;
      Ys[rr][qq] = (gr < re && gq < q) ? Y[gr * ldy + gq] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < TK; ++rr) {
      double xv[4], yv[QT];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = Xs[rr][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < QT; ++j) yv[j] = Ys[rr][tx * QT + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < QT; ++j) acc[i][j] = fma(xv[i], yv[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* dst = part + (int64_t)blockIdx.z * p * q;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gp = p0 + ty * 4 + i;
    if (gp >= p) continue;
#pragma unroll
    for (int j = 0; j < QT; ++j) {
      const int64_t gq = q0 + tx * QT + j;
      if (gq < q) dst[gp * q + gq] = acc[i][j];
    }
  }
}

// one warp per output element: the split partials are summed by the lanes
// (fixed strided subsets + butterfly), not serially by one thread
__global__ void k_tn_reduce(int64_t p, int64_t q, int64_t nsplit, const double* __restrict__ part, double alpha,
                            double beta, double* __restrict__ C, int64_t ldc) {
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= p * q) return;
  const double s = warp_strided_sum(part + t, nsplit, p * q);
  if ((threadIdx.x & 31) == 0) {
    const int64_t i = t / q, j = t - i * q;
    double* c = C + i * ldc + j;
    *c = beta == 0.0 ? alpha * s : fma(alpha, s, beta * *c);
  }
}

// ---- gemm_nn: Y = alpha X @ C + beta Y -------------------------------------
template <int QT>
__global__ void __launch_bounds__(256) k_gemm_nn(int64_t r, int64_t p, int64_t q, double alpha,
                                                 const double* __restrict__ X, int64_t ldx,
                                                 const double* __restrict__ C, int64_t ldc, double beta,
                                                 double* __restrict__ Y, int64_t ldy) {
  constexpr int TQ = 16 * QT;
  __shared__ double Xs[TP][TK + 1];
  __shared__ double Cs[TK][TQ + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = (int64_t)blockIdx.x * TP, q0 = (int64_t)blockIdx.y * TQ;
  double acc[4][QT];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < QT; ++j) acc[i][j] = 0.0;
  for (int64_t k0 = 0; k0 < p; k0 += TK) {
    for (int e = threadIdx.x; e < TP * TK; e += 256) {
      const int rr = e / TK, kk = e % TK;
      const int64_t gr = r0 + rr, gk = k0 + kk;
      Xs[rr][kk] = (gr < r && gk < p) ? X[gr * ldx + gk] : 0.0;
    }
    for (int e = threadIdx.x; e < TK * TQ; e += 256) {
      const int kk = e / TQ, qq = e % TQ;
      const int64_t gk = k0 + kk, gq = q0 + qq;
      Cs[kk][qq] = (gk < p && gq < q) ? C[gk * ldc + gq] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      double xv[4], cv[QT];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = Xs[ty * 4 + i][kk];
#pragma unroll
      for (int j = 0; j < QT; ++j) cv[j] = Cs[kk][tx * QT + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < QT; ++j) acc[i][j] = fma(xv[i], cv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gr = r0 + ty * 4 + i;
    if (gr >= r) continue;
#pragma unroll
    for (int j = 0; j < QT; ++j) {
      const int64_t gq = q0 + tx * QT + j;
      if (gq >= q) continue;
      double* y = Y + gr * ldy + gq;
      *y = beta == 0.0 ? alpha * acc[i][j] : fma(alpha, acc[i][j], beta * *y);
    }
  }
}

// ---- per-column sum of squares ---------------------------------------------
__global__ void __launch_bounds__(256) k_sumsq_part(int64_t r, int64_t q, const double* __restrict__ X,
                                                    int64_t ldx, int64_t rows_per, double* __restrict__ part) {
  __shared__ double red[256];
  const int64_t rs = (int64_t)blockIdx.x * rows_per, re = min(r, rs + rows_per);
  const int qc = (int)min64(q, 256);
  const int lanes_r = 256 / qc;
  const int c_in = threadIdx.x % qc, r_in = threadIdx.x / qc;
  for (int64_t c0 = 0; c0 < q; c0 += qc) {
    double acc = 0.0;
    const int64_t c = c0 + c_in;
    if (r_in < lanes_r && c < q)
      for (int64_t i = rs + r_in; i < re; i += lanes_r) {
        const double v = X[i * ldx + c];
        acc = fma(v, v, acc);
      }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < qc && c0 + threadIdx.x < q) {
      double s = 0.0;
      for (int k = 0; k < lanes_r; ++k) s += red[k * qc + threadIdx.x];
      part[(int64_t)blockIdx.x * q + c0 + threadIdx.x] = s;
    }
    __syncthreads();
  }
}

__global__ void k_sumsq_final(int64_t q, int64_t nblk, const double* __restrict__ part, double* colsq,
                              double* total) {
  __shared__ double red[256];
  double mine = 0.0;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t c = warp; c < q; c += nw) {
    const double s = warp_strided_sum(part + c, nblk, q);
    if ((threadIdx.x & 31) == 0) {
      if (colsq) colsq[c] = s;
      mine += s;
    }
  }
  const double t = block_sum(mine, red);
  if (threadIdx.x == 0 && total) *total = t;
}

// ---- prediction error sums: |p - t| and (p - t)^2 ---------------------------
__global__ void __launch_bounds__(256) k_err_part(int64_t n, const double* __restrict__ pred,
                                                  const double* __restrict__ truth, int64_t per,
                                                  double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t s = (int64_t)blockIdx.x * per, e = min(n, s + per);
  double a = 0.0, q = 0.0;
  for (int64_t i = s + threadIdx.x; i < e; i += blockDim.x) {
    const double d = pred[i] - truth[i];
    a += fabs(d);
    q = fma(d, d, q);
  }
  a = block_sum(a, red);
  q = block_sum(q, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = q;
  }
}

__global__ void k_err_final(int64_t nblk, const double* __restrict__ part, double* out2) {
  const double a = warp_strided_sum(part, nblk, 2);
  const double q = warp_strided_sum(part + 1, nblk, 2);
  if (threadIdx.x == 0) {
    out2[0] = a;
    out2[1] = q;
  }
}

int64_t tn_splits(int64_t r, int64_t tiles) {
  const int64_t want = (int64_t)sm_count() * 2;
  int64_t s = (want + tiles - 1) / tiles;
  const int64_t max_s = (r + 255) / 256;  // keep >= 256 rows per split
  if (s > max_s) s = max_s;
  return s < 1 ? 1 : s;
}

int64_t sumsq_blocks(int64_t r) {
  // short per-thread chains (<= ~128 rows per CTA): the partial sums are
  // latency-bound, not bandwidth-bound, at the QB engine's n x b blocks
  int64_t nb = (r + 127) / 128;
  const int64_t cap = (int64_t)sm_count() * 4;
  return nb > cap ? cap : (nb < 1 ? 1 : nb);
}

}  // namespace
}  // namespace svdrec

using namespace svdrec;

extern "C" size_t svdrec_gemm_tn_workspace_bytes(int64_t r, int64_t p, int64_t q) {
  // fewest possible tiles -> most splits: an upper bound for any call
  const int64_t tiles = ((p + TP - 1) / TP) * ((q + 63) / 64);
  size_t b = (size_t)tn_splits(r, tiles) * (size_t)p * (size_t)q * 8;
  {
    const size_t bs = (size_t)tn_skinny_slabs(r, p) * (size_t)p * (size_t)q * 8;
    if (bs > b) b = bs;
  }
  return align_up(b + 256) + 4096;
}

extern "C" int svdrec_gemm_tn(int64_t r, int64_t p, int64_t q, double alpha, const double* d_X, int64_t ldx,
                              const double* d_Y, int64_t ldy, double beta, double* d_C, int64_t ldc,
                              void* d_work, size_t work_bytes, void* stream) {
  SVDREC_ARG(r >= 0 && p >= 0 && q >= 0 && ldx >= p && ldy >= q && ldc >= q, "gemm_tn: bad arguments");
  if (p == 0 || q == 0) return 0;
  cudaStream_t s = as_stream(stream);
  if (r > 0 && (q <= 32 || tn_tma_able(r, p, q, d_X, ldx, d_Y, ldy))) {  // DMMA path, slab partials
    const int64_t ns = tn_skinny_slabs(r, p);
    const size_t need = (size_t)ns * (size_t)p * (size_t)q * 8;
    if (need > work_bytes) {
      set_error("gemm_tn: workspace %zu < %zu", work_bytes, need);
      return SVDREC_E_WORKSPACE;
    }
    double* part = static_cast<double*>(d_work);
    int rc = launch_tn_skinny(r, p, q, d_X, ldx, d_Y, ldy, part, ns, s);
    if (rc) return rc;
    const int64_t tot = p * q;
    k_tn_reduce<<<(unsigned)((tot * 32 + 255) / 256), 256, 0, s>>>(p, q, ns, part, alpha, beta, d_C, ldc);
    return check_launch("gemm_tn_reduce");
  }
  const bool narrow = q <= 32;
  const int64_t TQ = narrow ? 32 : 64;
  const int64_t gp = (p + TP - 1) / TP, gq = (q + TQ - 1) / TQ;
  int64_t ns = r > 0 ? tn_splits(r, gp * gq) : 1;
  const size_t need = (size_t)ns * (size_t)p * (size_t)q * 8;
  if (need > work_bytes) {
    set_error("gemm_tn: workspace %zu < %zu", work_bytes, need);
    return SVDREC_E_WORKSPACE;
  }
  double* part = static_cast<double*>(d_work);
  const int64_t rps = r > 0 ? (r + ns - 1) / ns : 1;
  dim3 grid((unsigned)gp, (unsigned)gq, (unsigned)ns);
  if (narrow)
    k_gemm_tn<2><<<grid, 256, 0, s>>>(r, p, q, d_X, ldx, d_Y, ldy, part, rps);
  else
    k_gemm_tn<4><<<grid, 256, 0, s>>>(r, p, q, d_X, ldx, d_Y, ldy, part, rps);
  int rc = check_launch("gemm_tn");
  if (rc) return rc;
  const int64_t tot = p * q;
  k_tn_reduce<<<(unsigned)((tot * 32 + 255) / 256), 256, 0, s>>>(p, q, ns, part, alpha, beta, d_C, ldc);
  return check_launch("gemm_tn_reduce");
}

extern "C" int svdrec_gemm_nn(int64_t r, int64_t p, int64_t q, double alpha, const double* d_X, int64_t ldx,
                              const double* d_C, int64_t ldc, double beta, double* d_Y, int64_t ldy,
                              void* stream) {
  SVDREC_ARG(r >= 0 && p >= 0 && q >= 0 && ldx >= p && ldc >= q && ldy >= q, "gemm_nn: bad arguments");
  if (r == 0 || q == 0) return 0;
  cudaStream_t s = as_stream(stream);
  if (p > 0 && r > 0) {
    int rc = 0;
    if (launch_nn_wide(r, p, q, alpha, d_X, ldx, d_C, ldc, beta, d_Y, ldy, s, &rc)) return rc;
  }
  if (q <= 32 && p > 0) return launch_nn_skinny(r, p, (int)q, alpha, d_X, ldx, d_C, ldc, beta, d_Y, ldy, s);
  const bool narrow = q <= 32;
  const int64_t TQ = narrow ? 32 : 64;
  dim3 grid((unsigned)((r + TP - 1) / TP), (unsigned)((q + TQ - 1) / TQ));
  if (narrow)
    k_gemm_nn<2><<<grid, 256, 0, s>>>(r, p, q, alpha, d_X, ldx, d_C, ldc, beta, d_Y, ldy);
  else
    k_gemm_nn<4><<<grid, 256, 0, s>>>(r, p, q, alpha, d_X, ldx, d_C, ldc, beta, d_Y, ldy);
  return check_launch("gemm_nn");
}

extern "C" size_t svdrec_sumsq_workspace_bytes(int64_t r, int64_t q) {
  return align_up((size_t)sumsq_blocks(r) * (size_t)(q > 0 ? q : 1) * 8);
}

extern "C" int svdrec_sumsq(int64_t r, int64_t q, const double* d_X, int64_t ldx, double* d_colsq,
                            double* d_total, void* d_work, size_t work_bytes, void* stream) {
  SVDREC_ARG(r >= 0 && q >= 1 && ldx >= q, "sumsq: bad arguments");
  cudaStream_t s = as_stream(stream);
  const int64_t nb = sumsq_blocks(r);
  if ((size_t)nb * q * 8 > work_bytes) {
    set_error("sumsq: workspace too small");
    return SVDREC_E_WORKSPACE;
  }
  double* part = static_cast<double*>(d_work);
  const int64_t per = r > 0 ? (r + nb - 1) / nb : 1;
  k_sumsq_part<<<(unsigned)nb, 256, 0, s>>>(r, q, d_X, ldx, per, part);
  int rc = check_launch("sumsq_part");
  if (rc) return rc;
  k_sumsq_final<<<1, 256, 0, s>>>(q, nb, part, d_colsq, d_total);
  return check_launch("sumsq_final");
}

extern "C" size_t svdrec_err_sum_workspace_bytes(int64_t nsamp) {
  return align_up((size_t)sumsq_blocks(nsamp) * 16);
}

extern "C" int svdrec_err_sum(int64_t nsamp, const double* d_pred, const double* d_truth, double* d_out2,
                              void* d_work, size_t work_bytes, void* stream) {
  SVDREC_ARG(nsamp >= 0, "err_sum: bad arguments");
  cudaStream_t s = as_stream(stream);
  const int64_t nb = sumsq_blocks(nsamp);
  if ((size_t)nb * 16 > work_bytes) {
    set_error("err_sum: workspace too small");
    return SVDREC_E_WORKSPACE;
  }
  double* part = static_cast<double*>(d_work);
  const int64_t per = nsamp > 0 ? (nsamp + nb - 1) / nb : 1;
  k_err_part<<<(unsigned)nb, 256, 0, s>>>(nsamp, d_pred, d_truth, per, part);
  int rc = check_launch("err_part");
  if (rc) return rc;
  k_err_final<<<1, 32, 0, s>>>(nb, part, d_out2);
  return check_launch("err_final");
}

namespace svdrec {
namespace {
__global__ void __launch_bounds__(256) k_vsum_part(int64_t n, const double* __restrict__ x, int64_t per,
                                                   double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t s = (int64_t)blockIdx.x * per, e = min64(n, s + per);
  double a = 0.0;
  for (int64_t i = s + threadIdx.x; i < e; i += blockDim.x) a += x[i];
  a = block_sum(a, red);
  if (threadIdx.x == 0) part[blockIdx.x] = a;
}
__global__ void k_vsum_final(int64_t nblk, const double* __restrict__ part, double* out) {
  const double a = warp_strided_sum(part, nblk, 1);
  if (threadIdx.x == 0) *out = a;
}
}  // namespace
}  // namespace svdrec

extern "C" size_t svdrec_vec_sum_workspace_bytes(int64_t n) { return align_up((size_t)sumsq_blocks(n) * 8); }

extern "C" int svdrec_vec_sum(int64_t n, const double* d_x, double* d_out, void* d_work, size_t work_bytes,
                              void* stream) {
  SVDREC_ARG(n >= 0, "vec_sum: bad arguments");
  cudaStream_t s = as_stream(stream);
  const int64_t nb = sumsq_blocks(n);
  if ((size_t)nb * 8 > work_bytes) {
    set_error("vec_sum: workspace too small");
    return SVDREC_E_WORKSPACE;
  }
  double* part = static_cast<double*>(d_work);
  const int64_t per = n > 0 ? (n + nb - 1) / nb : 1;
  k_vsum_part<<<(unsigned)nb, 256, 0, s>>>(n, d_x, per, part);
  int rc = check_launch("vec_sum_part");
  if (rc) return rc;
  k_vsum_final<<<1, 32, 0, s>>>(nb, part, d_out);
  return check_launch("vec_sum_final");
}
