// Tall-skinny float64 GEMMs for the QB deflations (q = block width <= 32),
// on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64: 256 FMAs per warp
// instruction; measured 37.2 TFLOP/s on B200 vs 34.0 for DFMA, and at a
// fraction of the issue slots).
//
//   nn:  Y (r x q) = alpha X (r x p) C (p x q) + beta Y      (Q @ C, B.T @ C)
//   tn:  part[s]   = X[slab s].T @ Y[slab s]  (p x q)        (Q.T @ Y, B @ X)
//
// Reference: the products Q @ (B @ X), Q @ (Q.T @ X), B.T @ (Q.T @ X) of
// rsvd.py:135-142, 179-194 and the Gram of CholeskyQR.  X (Q or B.T, r x k
// with k up to the rank cap) is the only large operand, so both kernels
// stream it straight from HBM into the A fragments (a lane's fragment
// element is one double; the 32 lanes of a load cover 8 rows x 32 B, whole
// sectors) with a D-deep register prefetch; the small operand's fragments
// come through L1.  The tn reduction over r is split into row slabs whose
// partials are summed in a fixed order (deterministic).
#include "tma.cuh"

namespace svdrec {
namespace {

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// NN.  A warp owns T consecutive row tiles of 8*MT rows (T chosen so that
// every warp gets the same count) and walks the flattened (tile, k-step)
// sequence with D k-steps of A fragments in flight.  Fragment layout
// (m8n8k4): A[g][t], B[t][g], C[g][2t..2t+1] with g = lane/4, t = lane%4.
template <int MT, int NT, int D>
__global__ void __launch_bounds__(128) k_nn_mma(int64_t r, int64_t p, int q, double alpha,
                                                const double* __restrict__ X, int64_t ldx,
                                                const double* __restrict__ C, int64_t ldc, double beta,
                                                double* __restrict__ Y, int64_t ldy, int64_t ntiles, int tpw) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t t0 = w * tpw;
  if (t0 >= ntiles) return;
  const int nt = (int)min64(tpw, ntiles - t0);
  const int nk = (int)((p + 3) / 4);
  // flattened (tile, step) sequence; the prefetch cursor (pt, ps) runs D
  // steps ahead of the compute cursor (ct, cs) -- no divisions in the loop
  int pt = 0, ps = 0;
  auto ld = [&](double (&av)[MT], double (&bv)[NT]) {
    const bool live = pt < nt;
    const int64_t k = 4 * (int64_t)ps + tq;
    const int64_t rbase = (t0 + pt) * (8 * MT) + g;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int64_t row = rbase + 8 * i;
      av[i] = (live && row < r && k < p) ? __ldcs(X + row * ldx + k) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int col = 8 * j + g;
      bv[j] = (live && k < p && col < q) ? __ldg(C + k * ldc + col) : 0.0;
    }
    if (++ps == nk) {
      ps = 0;
      ++pt;
    }
  };
  double a[D][MT], b[D][NT];
#pragma unroll
  for (int d = 0; d < D; ++d) ld(a[d], b[d]);
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int ct = 0, cs = 0;
  while (ct < nt) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (ct < nt) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(acc[i][j], a[d][i], b[d][j]);
        ld(a[d], b[d]);
        if (++cs == nk) {  // tile complete: epilogue, reset
          const int64_t rbase = (t0 + ct) * (8 * MT) + g;
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            const int64_t row = rbase + 8 * i;
            if (row < r) {
              double* yr = Y + row * ldy;
#pragma unroll
              for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const int col = 8 * j + 2 * tq + e;
                  if (col < q) yr[col] = beta == 0.0 ? alpha * acc[i][j][e] : fma(alpha, acc[i][j][e], beta * yr[col]);
                }
            }
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
          }
          cs = 0;
          ++ct;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// TN.  CTA = 8 warps on one 8*MT-column block of X (blockIdx.y) and one row
// slab (blockIdx.x); warp w takes the w-th eighth of the slab in 4-row
// k-steps, D steps of A (X.T) and B (Y) fragments in flight.  The 8 warp
// partials are added in warp order through shared memory, then one partial
// per CTA goes to ``part`` for the fixed-order slab reduction.
constexpr int kTnWarps = 8;

template <int MT, int NT, int D>
__global__ void __launch_bounds__(kTnWarps * 32, 2) k_tn_mma(int64_t r, int64_t p, int q,
                                                             const double* __restrict__ X, int64_t ldx,
                                                             const double* __restrict__ Y, int64_t ldy,
                                                             double* __restrict__ part, int64_t rows_per) {
  __shared__ double red[MT][NT][2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t p0 = (int64_t)blockIdx.y * (8 * MT);
  const int64_t rs = (int64_t)blockIdx.x * rows_per, re = min64(r, rs + rows_per);
  const int64_t wr = ((rows_per + kTnWarps - 1) / kTnWarps + 3) / 4 * 4;  // rows per warp, whole k-steps
  const int64_t ws = rs + warp * wr, we = min64(re, ws + wr);
  const int nk = we > ws ? (int)((we - ws + 3) / 4) : 0;
  auto ld = [&](int s, double (&av)[MT], double (&bv)[NT]) {
    const int64_t row = ws + 4 * (int64_t)s + tq;
    const bool ok = s < nk && row < we;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int64_t col = p0 + 8 * i + g;
      av[i] = (ok && col < p) ? __ldcs(X + row * ldx + col) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int col = 8 * j + g;
      bv[j] = (ok && col < q) ? __ldg(Y + row * ldy + col) : 0.0;
    }
  };
  double a[D][MT], b[D][NT];
#pragma unroll
  for (int d = 0; d < D; ++d) ld(d, a[d], b[d]);
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int s0 = 0; s0 < nk; s0 += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (s0 + d < nk) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(acc[i][j], a[d][i], b[d][j]);
        ld(s0 + d + D, a[d], b[d]);
      }
    }
  }
  for (int w = 0; w < kTnWarps; ++w) {
    if (warp == w) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) red[i][j][e][lane] = (w == 0 ? 0.0 : red[i][j][e][lane]) + acc[i][j][e];
    }
    __syncthreads();
  }
  double* dst = part + (int64_t)blockIdx.x * p * q;
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t pr = p0 + 8 * i + g;
          const int col = 8 * j + 2 * tq + e;
          if (pr < p && col < q) dst[pr * q + col] = red[i][j][e][lane];
        }
  }
}

// ---------------------------------------------------------------------------
// TMA-staged variants (16-B aligned operands, even pitches): the X tiles are
// brought in by the tensor-memory accelerator into a 4-deep shared-memory
// ring (bytes in flight without registers: the register-prefetch kernels
// above stall on HBM latency at ~50% DMMA issue), fragments read with
// conflict-free LDS.64 (20- / 40-double row pitch puts the 8 (resp. 4) rows
// of a fragment load in distinct bank quarters (halves)).
constexpr int kNnRT = 128, kNnKP = 20, kNnS = 4;  // rows per tile, k per stage, stages

// kNnW warps per CTA, each on kNnRT / kNnW rows of the 128-row tile
#ifndef SVDREC_NN_WARPS
#define SVDREC_NN_WARPS 8
#endif
constexpr int kNnW = SVDREC_NN_WARPS;

template <int NT>
__global__ void __launch_bounds__(kNnW * 32) k_nn_tma(const __grid_constant__ CUtensorMap tmX,
                                                const __grid_constant__ CUtensorMap tmC, int64_t r, int64_t p, int q,
                                                double alpha, double beta, double* __restrict__ Y, int64_t ldy,
                                                int64_t ntiles, int tpc, int qb) {
  constexpr int MT = kNnRT / (8 * kNnW);  // 8 * MT rows per warp
  const int col0 = 32 * blockIdx.y;  // column block (q > 32: several, C box qb = 32 wide)
  const bool vec2 = (ldy % 2 == 0) && (reinterpret_cast<uintptr_t>(Y) % 16 == 0);
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[kNnS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int xstage = kNnRT * kNnKP, cstage = kNnKP * qb;
  const int stage = xstage + ((cstage + 15) & ~15);  // keep every TMA destination 128-B aligned
  const int64_t t0 = (int64_t)blockIdx.x * tpc;
  const int nt = (int)min64(tpc, ntiles - t0);
  const int nks = (int)((p + kNnKP - 1) / kNnKP);
  const int64_t total = (int64_t)nt * nks;
  if (threadIdx.x < kNnS) mbar_init(bar + threadIdx.x, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  int pt = 0, ps = 0;  // producer cursor (thread 0 only)
  auto issue = [&](int64_t n) {
    const int slot = (int)(n % kNnS);
    double* xs = sm + slot * stage;
    mbar_expect_tx(bar + slot, (unsigned)((xstage + cstage) * 8));
    tma_load_2d(xs, &tmX, ps * kNnKP, (int)((t0 + pt) * kNnRT), bar + slot);
    tma_load_2d(xs + xstage, &tmC, col0, ps * kNnKP, bar + slot);
    if (++ps == nks) {
      ps = 0;
      ++pt;
    }
  };
  if (threadIdx.x == 0)
    for (int64_t n = 0; n < kNnS - 1 && n < total; ++n) issue(n);
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int ct = 0, cs = 0;
  for (int64_t n = 0; n < total; ++n) {
    const int slot = (int)(n % kNnS);
    mbar_wait(bar + slot, (unsigned)((n / kNnS) & 1));
    const double* xs = sm + slot * stage + (8 * MT * warp + g) * kNnKP + tq;
    const double* cs_ = sm + slot * stage + xstage + tq * qb + g;
#pragma unroll
    for (int kk = 0; kk < kNnKP / 4; ++kk) {
      double a[MT], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) a[i] = xs[8 * i * kNnKP + 4 * kk];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = (8 * j + g < qb && col0 + 8 * j + g < q) ? cs_[4 * kk * qb + 8 * j] : 0.0;
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j], a[i], b[j]);
    }
    if (++cs == nks) {
      const int64_t rbase = (t0 + ct) * kNnRT + 8 * MT * warp + g;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int64_t row = rbase + 8 * i;
        if (row < r) {
          double* yr = Y + row * ldy;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const int lc = 8 * j + 2 * tq, col = col0 + lc;
            if (vec2 && col + 1 < q && lc + 1 < qb) {  // whole-sector 16-B store
              double2* p2 = reinterpret_cast<double2*>(yr + col);
              double2 v = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
              if (beta != 0.0) {
                const double2 o = *p2;
                v = make_double2(fma(alpha, acc[i][j][0], beta * o.x), fma(alpha, acc[i][j][1], beta * o.y));
              }
              *p2 = v;
              continue;
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              if (col + e < q && lc + e < qb)
                yr[col + e] = beta == 0.0 ? alpha * acc[i][j][e] : fma(alpha, acc[i][j][e], beta * yr[col + e]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      }
      cs = 0;
      ++ct;
    }
    __syncthreads();  // every warp is done with slot (n - 1) % S ... and n
    if (threadIdx.x == 0 && n + kNnS - 1 < total) issue(n + kNnS - 1);
  }
}

constexpr int kTnRB = 32, kTnS2 = 4;  // rows per stage, stages

// CTA = 4 warps on one 8*MT-column block of X and one row slab; warp w
// takes k-steps w, w+4 of every 32-row stage.  Warp partials are added in
// warp order through shared memory; one partial per CTA.
template <int MT, int NT>
__global__ void __launch_bounds__(128) k_tn_tma(const __grid_constant__ CUtensorMap tmX,
                                                const __grid_constant__ CUtensorMap tmY, int64_t r, int64_t p, int q,
                                                double* __restrict__ part, int64_t rows_per, int qb) {
  constexpr int PB = 8 * MT;
  const int col0 = 32 * blockIdx.z;  // column block of Y (q > 32: box qb = 32 wide)
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[kTnS2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int xstage = kTnRB * PB, ystage = kTnRB * qb;
  const int stage = ((xstage + 15) & ~15) + ((ystage + 15) & ~15);
  const int yoff = (xstage + 15) & ~15;
  const int64_t p0 = (int64_t)blockIdx.y * PB;
  const int64_t rs = (int64_t)blockIdx.x * rows_per, re = min64(r, rs + rows_per);
  const int nst = re > rs ? (int)((re - rs + kTnRB - 1) / kTnRB) : 0;
  if (threadIdx.x < kTnS2) mbar_init(bar + threadIdx.x, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  auto issue = [&](int n) {
    const int slot = n % kTnS2;
    double* xs = sm + slot * stage;
    mbar_expect_tx(bar + slot, (unsigned)((xstage + ystage) * 8));
    const int row = (int)(rs + (int64_t)n * kTnRB);
    tma_load_2d(xs, &tmX, (int)p0, row, bar + slot);
    tma_load_2d(xs + yoff, &tmY, col0, row, bar + slot);
  };
  if (threadIdx.x == 0)
    for (int n = 0; n < kTnS2 - 1 && n < nst; ++n) issue(n);
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int n = 0; n < nst; ++n) {
    const int slot = n % kTnS2;
    mbar_wait(bar + slot, (unsigned)((n / kTnS2) & 1));
    const int64_t row0 = rs + (int64_t)n * kTnRB;
    const double* xs = sm + slot * stage;
    const double* ys = xs + yoff;
#pragma unroll
    for (int h = 0; h < kTnRB / 16; ++h) {
      const int kr = 16 * h + 4 * warp + tq;  // this lane's row within the stage
      // rows past the slab end belong to the next slab: mask them (TMA only
      // zero-fills past the matrix end)
      const bool rok = row0 + kr < re;
      double a[MT], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) a[i] = rok ? xs[kr * PB + 8 * i + g] : 0.0;
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = (rok && 8 * j + g < qb) ? ys[kr * qb + 8 * j + g] : 0.0;
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
    if (threadIdx.x == 0 && n + kTnS2 - 1 < nst) issue(n + kTnS2 - 1);
  }
  // warp-ordered sum through shared memory (the ring is free now)
  double* red = sm;
  for (int w = 0; w < 4; ++w) {
    if (warp == w) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double* c = red + ((i * NT + j) * 2 + e) * 32 + lane;
            *c = (w == 0 ? 0.0 : *c) + acc[i][j][e];
          }
    }
    __syncthreads();
  }
  double* dst = part + (int64_t)blockIdx.x * p * q;
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t pr = p0 + 8 * i + g;
          const int col = col0 + 8 * j + 2 * tq + e;
          if (pr < p && col < q && 8 * j + 2 * tq + e < qb) dst[pr * q + col] = red[((i * NT + j) * 2 + e) * 32 + lane];
        }
  }
}

template <int NT>
int nn_tma_launch(int64_t r, int64_t p, int64_t q, double alpha, const double* X, int64_t ldx, const double* C,
                  int64_t ldc, double beta, double* Y, int64_t ldy, cudaStream_t s) {
  const int qb = q > 32 ? 32 : (int)q;
  CUtensorMap tx, tc;
  int rc = make_map_2d(&tx, X, r, p, ldx, kNnKP, kNnRT);
  if (!rc) rc = make_map_2d(&tc, C, p, q, ldc, qb, kNnKP);
  if (rc) return rc;
  const int stage = kNnRT * kNnKP + ((kNnKP * qb + 15) & ~15);
  const size_t smem = (size_t)kNnS * stage * 8;
  SVDREC_CUDA(smem_attr_once(k_nn_tma<NT>, 100 * 1024));
  const int64_t ntiles = (r + kNnRT - 1) / kNnRT;
  const int64_t gy = (q + 31) / 32;
  int per_sm = 0;  // smem depends on qb
  SVDREC_CUDA(blocks_per_sm(k_nn_tma<NT>, kNnW * 32, smem, &per_sm));
  const int64_t slots = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1);
  const int64_t per_col = (slots + gy - 1) / gy;  // CTAs per column block
  const int tpc = (int)((ntiles + per_col - 1) / per_col);
  const int64_t grid = (ntiles + tpc - 1) / tpc;
  k_nn_tma<NT><<<dim3((unsigned)grid, (unsigned)gy), kNnW * 32, smem, s>>>(tx, tc, r, p, (int)q, alpha, beta, Y, ldy,
                                                                     ntiles, tpc, qb);
  return check_launch("gemm_nn_tma");
}

template <int MT, int NT>
int tn_tma_launch(int64_t r, int64_t p, int64_t q, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                  double* part, int64_t nslab, int64_t rows_per, cudaStream_t s) {
  const int qb = q > 32 ? 32 : (int)q;
  CUtensorMap tx, ty;
  int rc = make_map_2d(&tx, X, r, p, ldx, 8 * MT, kTnRB);
  if (!rc) rc = make_map_2d(&ty, Y, r, q, ldy, qb, kTnRB);
  if (rc) return rc;
  const int stage = ((kTnRB * 8 * MT + 15) & ~15) + ((kTnRB * qb + 15) & ~15);
  size_t smem = (size_t)kTnS2 * stage * 8;
  const size_t red = (size_t)MT * NT * 2 * 32 * 8;
  if (smem < red) smem = red;
  SVDREC_CUDA(smem_attr_once(k_tn_tma<MT, NT>, 100 * 1024));
  dim3 grid((unsigned)nslab, (unsigned)((p + 8 * MT - 1) / (8 * MT)), (unsigned)((q + 31) / 32));
  k_tn_tma<MT, NT><<<grid, 128, smem, s>>>(tx, ty, r, p, (int)q, part, rows_per, qb);
  return check_launch("gemm_tn_tma");
}

template <int MT, int NT>
int nn_launch(int64_t r, int64_t p, int q, double alpha, const double* X, int64_t ldx, const double* C, int64_t ldc,
              double beta, double* Y, int64_t ldy, cudaStream_t s) {
  const int64_t ntiles = (r + 8 * MT - 1) / (8 * MT);
  int per_sm = 0;  // resident 4-warp CTAs per SM (register bound)
  SVDREC_CUDA(blocks_per_sm(k_nn_mma<MT, NT, 4>, 128, 0, &per_sm));
  if (per_sm < 1) per_sm = 1;
  const int64_t max_warps = (int64_t)sm_count() * per_sm * 4;
  const int tpw = (int)((ntiles + max_warps - 1) / max_warps);
  const int64_t warps = (ntiles + tpw - 1) / tpw;
  k_nn_mma<MT, NT, 4><<<(unsigned)((warps + 3) / 4), 128, 0, s>>>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy,
                                                                  ntiles, tpw);
  return check_launch("gemm_nn_mma");
}

template <int MT, int NT>
int tn_launch(int64_t r, int64_t p, int q, const double* X, int64_t ldx, const double* Y, int64_t ldy, double* part,
              int64_t nslab, int64_t rows_per, cudaStream_t s) {
  dim3 grid((unsigned)nslab, (unsigned)((p + 8 * MT - 1) / (8 * MT)));
  k_tn_mma<MT, NT, 4><<<grid, kTnWarps * 32, 0, s>>>(r, p, q, X, ldx, Y, ldy, part, rows_per);
  return check_launch("gemm_tn_mma");
}

}  // namespace

// p-block width of the tn kernel: 8 * MT columns, MT = 4 (or fewer for a
// narrow X, e.g. the 20-column Gram)
static int tn_mt(int64_t p) { return p <= 8 ? 1 : p <= 16 ? 2 : p <= 24 ? 3 : 4; }
// TMA path: 40-column blocks for wide X (row pitch 320 B: the 4 rows of an
// A fragment fall in 2 bank halves), the narrow cases as above
static int tn_tma_mt(int64_t p) { return p <= 8 ? 1 : p <= 16 ? 2 : p <= 24 ? 3 : 5; }

int64_t tn_skinny_slabs(int64_t r, int64_t p) {
  const int64_t gy = (p + 8 * tn_mt(p) - 1) / (8 * tn_mt(p));
  int64_t s = (2 * (int64_t)sm_count() + gy - 1) / gy;
  const int64_t max_s = (r + 255) / 256;  // >= 256 rows per slab (32 per warp)
  if (s > max_s) s = max_s;
  return s < 1 ? 1 : s;
}

int launch_nn_skinny(int64_t r, int64_t p, int q, double alpha, const double* X, int64_t ldx, const double* C,
                     int64_t ldc, double beta, double* Y, int64_t ldy, cudaStream_t s) {
  if (q % 2 == 0 && tma_ok(X, ldx) && tma_ok(C, ldc) && r < (1ll << 31) && p < (1ll << 31)) {
    switch (q > 32 ? 4 : (q + 7) / 8) {
      case 1: return nn_tma_launch<1>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
      case 2: return nn_tma_launch<2>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
      case 3: return nn_tma_launch<3>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
      default: return nn_tma_launch<4>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
    }
  }
  switch ((q + 7) / 8) {
    case 1: return nn_launch<2, 1>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
    case 2: return nn_launch<2, 2>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
    case 3: return nn_launch<2, 3>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
    default: return nn_launch<2, 4>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
  }
}

// any q: the DMMA/TMA kernel over 32-column blocks of C (false: operands
// not TMA-able, caller falls back)
bool launch_nn_wide(int64_t r, int64_t p, int64_t q, double alpha, const double* X, int64_t ldx, const double* C,
                    int64_t ldc, double beta, double* Y, int64_t ldy, cudaStream_t s, int* rc) {
  if (!(q % 2 == 0 && tma_ok(X, ldx) && tma_ok(C, ldc) && r < (1ll << 31) && p < (1ll << 31))) return false;
  *rc = q > 32 ? nn_tma_launch<4>(r, p, q, alpha, X, ldx, C, ldc, beta, Y, ldy, s)
               : launch_nn_skinny(r, p, (int)q, alpha, X, ldx, C, ldc, beta, Y, ldy, s);
  return true;
}

bool tn_tma_able(int64_t r, int64_t p, int64_t q, const double* X, int64_t ldx, const double* Y, int64_t ldy) {
  return q % 2 == 0 && tma_ok(X, ldx) && tma_ok(Y, ldy) && r < (1ll << 31) && p < (1ll << 31);
}

int launch_tn_skinny(int64_t r, int64_t p, int64_t q, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                     double* part, int64_t nslab, cudaStream_t s) {
  const int64_t rows_per = (r + nslab - 1) / nslab;
  const int nt = q > 32 ? 4 : (q + 7) / 8;
  if (q % 2 == 0 && tma_ok(X, ldx) && tma_ok(Y, ldy) && r < (1ll << 31) && p < (1ll << 31)) {
#define SVDREC_TNT(M)                                                                        \
  switch (nt) {                                                                             \
    case 1: return tn_tma_launch<M, 1>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s);  \
    case 2: return tn_tma_launch<M, 2>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s);  \
    case 3: return tn_tma_launch<M, 3>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s);  \
    default: return tn_tma_launch<M, 4>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s); \
  }
    switch (tn_tma_mt(p)) {
      case 1: SVDREC_TNT(1)
      case 2: SVDREC_TNT(2)
      case 3: SVDREC_TNT(3)
      default: SVDREC_TNT(5)
    }
#undef SVDREC_TNT
  }
#define SVDREC_TN(M)                                                                     \
  switch (nt) {                                                                          \
    case 1: return tn_launch<M, 1>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s);   \
    case 2: return tn_launch<M, 2>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s);   \
    case 3: return tn_launch<M, 3>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s);   \
    default: return tn_launch<M, 4>(r, p, q, X, ldx, Y, ldy, part, nslab, rows_per, s);  \
  }
  switch (tn_mt(p)) {
    case 1: SVDREC_TN(1)
    case 2: SVDREC_TN(2)
    case 3: SVDREC_TN(3)
    default: SVDREC_TN(4)
  }
#undef SVDREC_TN
}

}  // namespace svdrec
