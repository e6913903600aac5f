// Inverse square root of the small SPD Gram G = B B.T by coupled
// Newton-Schulz iteration, in one cooperative kernel.
//
// Why: Alg. 5 scores every block (reference cf.py:227-240) through
// latent_from_qb's eig_svd(B.T) (cf.py:77-92), but the CF prediction of
// Alg. 4 (cf.py:108-143) only ever uses cosines between item columns of
// T = S^(1/2) U.T, and T.T T = B.T (B B.T)^(-1/2) B.  So per block we need
// Z = G^(-1/2), not an eigendecomposition: with x_l = B[:, l] and
// y_l = Z x_l, cos(T_l, T_j) = x_j.y_l / (|x_l|_Z |x_j|_Z).  The iteration
// (A = G / ||G||_F, Y0 = A, Z0 = I)
//     T = (3 I - Z Y) / 2,   Y <- Y T,   Z <- T Z
// converges quadratically to Y = A^(1/2), Z = A^(-1/2); every step is
// k x k GEMM work spread over the whole GPU, with two grid barriers per
// iteration instead of Jacobi's thousands of dependent rotation rounds.
// The eigendecomposition itself (syev) runs once, for the returned factors.
#include <cooperative_groups.h>

#include "tma.cuh"

namespace cg = cooperative_groups;

namespace svdrec {
namespace {

constexpr int NT = 32;    // output tile (k=240 -> 64 tiles per GEMM phase)
constexpr int KC = 192;   // reduction columns staged per pass
constexpr int kNsThreads = 128;  // 4 warps: warp w owns tile rows 8w..8w+7, all 32 columns
constexpr int kLdA = KC + 4;     // A panel pitch: 8 fragment rows land in distinct 32-B bank quarters
constexpr int kLdB = NT + 8;     // B panel pitch (320 B): the 4 fragment rows in 2 bank halves
constexpr size_t kNsSmem = ((size_t)NT * kLdA + (size_t)KC * kLdB) * sizeof(double);

__device__ __forceinline__ void cp_async8_zf(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0) : "memory");
}

__device__ __forceinline__ void dmma_ns(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// C[tile] = alpha * (A @ B)[tile] + diag * I[tile] on the FP64 tensor cores
// (DMMA m8n8k4); returns the tile's sum of (C - I)^2 when ``resid`` (all
// matrices k x k, ld = k).  The 32 x k row panel of A and k x 32 column
// panel of B are staged in shared memory in KC-wide passes.
__device__ double tile_gemm(double* sm, double* red, int k, const double* __restrict__ A,
                            const double* __restrict__ B, double* __restrict__ C, int ti, int tj, double alpha,
                            double diag, bool resid) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int r0 = ti * NT, c0 = tj * NT;
  double* sa = sm;             // [NT][kLdA]
  double* sb = sm + NT * kLdA; // [KC][kLdB]
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
  for (int k0 = 0; k0 < k; k0 += KC) {
    const int kc = min(KC, k - k0);
    const int kc4 = (kc + 3) & ~3;
    __syncthreads();  // previous pass / tile done with the panels
    // coalesced panel loads as cp.async (all in flight at once; a plain
    // load -> st.shared loop serialises on each load's L2 latency), zero
    // fill outside the matrix
    for (int rr = warp; rr < NT; rr += kNsThreads / 32) {
      const int gr = r0 + rr;
      const double* src = A + (int64_t)(gr < k ? gr : 0) * k + k0;
      for (int kk = lane; kk < kc4; kk += 32) cp_async8_zf(sa + rr * kLdA + kk, src + (kk < kc ? kk : 0), gr < k && kk < kc);
    }
    for (int kk = warp; kk < kc4; kk += kNsThreads / 32) {
      const int gc = c0 + lane;
      cp_async8_zf(sb + kk * kLdB + lane, B + (int64_t)(k0 + (kk < kc ? kk : 0)) * k + (gc < k ? gc : 0),
                   gc < k && kk < kc);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    const double* ap = sa + (8 * warp + g) * kLdA + tq;
    const double* bp = sb + tq * kLdB + g;
#pragma unroll 4
    for (int s = 0; s < kc4 / 4; ++s) {
      const double a = ap[4 * s];
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_ns(acc[j], a, bp[4 * s * kLdB + 8 * j]);
    }
  }
  double rs = 0.0;
  const int gr = r0 + 8 * warp + g;
  if (gr < k) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gc = c0 + 8 * j + 2 * tq + e;
        if (gc < k) {
          const double v = alpha * acc[j][e] + (gr == gc ? diag : 0.0);
          C[(int64_t)gr * k + gc] = v;
          if (resid) {
            const double d = v - (gr == gc ? 1.0 : 0.0);
            rs = fma(d, d, rs);
          }
        }
      }
  }
  if (resid) rs = block_sum(rs, red);
  return rs;
}

// TMA variant of tile_gemm (k even): each operand panel is ONE tensor-map
// copy into shared memory (A: 32 rows x kKcT columns, pitch 244 doubles =
// 1952 B = 32 mod 128, so the 8 rows of an A fragment fall in distinct
// bank quarters; B: kKcT rows x 40 columns, pitch 320 B = 2 bank halves),
// zero fill past k.  The per-element cp.async loop it replaces spent ~10 us
// per tile issuing 15 k copies through 128 threads.
constexpr int kKcT = 244, kBwT = 40;
constexpr size_t kNsSmemT = ((size_t)NT * kKcT + (size_t)kKcT * kBwT) * sizeof(double);

struct NsMaps {
  CUtensorMap a[5];  // A-operand boxes {kKcT cols, 32 rows} of Y0, Y1, Z0, Z1, T
  CUtensorMap b[5];  // B-operand boxes {40 cols, kKcT rows}
};

__device__ double tile_gemm_tma(double* sm, uint64_t* bar, unsigned& phase, double* red, int k, const NsMaps& maps,
                                int ia, int ib, double* __restrict__ C, int ti, int tj, double alpha, double diag,
                                bool resid) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int r0 = ti * NT, c0 = tj * NT;
  double* sa = sm;                // [NT][kKcT]
  double* sb = sm + NT * kKcT;    // [kKcT][kBwT]
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
  for (int k0 = 0; k0 < k; k0 += kKcT) {
    __syncthreads();  // previous pass / tile done with the panels
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, (unsigned)((NT * kKcT + kKcT * kBwT) * 8));
      tma_load_2d(sa, &maps.a[ia], k0, r0, bar);
      tma_load_2d(sb, &maps.b[ib], c0, k0, bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    const int ks = (min(kKcT, k - k0) + 3) >> 2;
    const double* ap = sa + (8 * warp + g) * kKcT + tq;
    const double* bp = sb + tq * kBwT + g;
#pragma unroll 4
    for (int s = 0; s < ks; ++s) {
      const double a = ap[4 * s];
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_ns(acc[j], a, bp[4 * s * kBwT + 8 * j]);
    }
  }
  double rs = 0.0;
  const int gr = r0 + 8 * warp + g;
  if (gr < k) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gc = c0 + 8 * j + 2 * tq + e;
        if (gc < k) {
          const double v = alpha * acc[j][e] + (gr == gc ? diag : 0.0);
          C[(int64_t)gr * k + gc] = v;
          if (resid) {
            const double d = v - (gr == gc ? 1.0 : 0.0);
            rs = fma(d, d, rs);
          }
        }
      }
  }
  if (resid) rs = block_sum(rs, red);
  return rs;
}

// work: Y0, Y1, Z0, Z1, T (k x k each), part (ntiles), misc
__global__ void __launch_bounds__(kNsThreads) k_ns(int k, const double* __restrict__ G, int64_t ldg,
                                                   double* __restrict__ out, int64_t ldo, double* __restrict__ Y0,
                                                   double* __restrict__ Y1, double* __restrict__ Z0,
                                                   double* __restrict__ Z1, double* __restrict__ T,
                                                   double* __restrict__ part, int maxit, uint32_t* d_status,
                                                   int* d_iters, const __grid_constant__ NsMaps maps, int use_tma) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) double ns_sm[];
  __shared__ double red[32];
  __shared__ __align__(8) uint64_t tbar;
  unsigned tphase = 0;
  if (threadIdx.x == 0) mbar_init(&tbar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  // buffer ids of Y, Yn, Z, Zn for the tensor maps (0 Y0, 1 Y1, 2 Z0, 3 Z1, 4 T)
  int iy = 0, iyn = 1, iz = 2, izn = 3;
  const int nt = (k + NT - 1) / NT;
  const int ntiles = nt * nt;
  // scale: A = G / ||G||_F has spectrum in (0, 1] and a larger smallest
  // eigenvalue than G / trace(G) (fewer iterations); trace kept for the
  // reference's singularity floor
  const int64_t kk = (int64_t)k * k;
  {
    double fs = 0.0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < kk; t += (int64_t)gridDim.x * blockDim.x) {
      const double g = G[(t / k) * ldg + t % k];
      fs = fma(g, g, fs);
    }
    fs = block_sum(fs, red);
    if (threadIdx.x == 0) part[blockIdx.x] = fs;
  }
  grid.sync();
  // block-parallel loads, fixed-order block sums: every block gets the
  // same values (no serial chain of dependent L2 reads)
  double fro2 = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) fro2 += part[b];
  fro2 = block_sum(fro2, red);
  double tr = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) tr += G[(int64_t)i * ldg + i];
  tr = block_sum(tr, red);
  const double c_scale = sqrt(fro2);
  const double inv_c = c_scale > 0.0 ? 1.0 / c_scale : 0.0;
  grid.sync();  // part[] is reused below
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < kk; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / k, j = t % k;
    Y0[t] = G[i * ldg + j] * inv_c;
    Z0[t] = (i == j) ? 1.0 : 0.0;
  }
  grid.sync();
  double* Y = Y0;
  double* Yn = Y1;
  double* Z = Z0;
  double* Zn = Z1;
  double prev = 1e300;
  int it = 0;
  bool done = false;
  for (; it < maxit; ++it) {
    // phase A: T = 1.5 I - 0.5 Z Y, residual ||T - I||_F^2 per tile
    for (int w = blockIdx.x; w < ntiles; w += gridDim.x) {
      const double rs = use_tma ? tile_gemm_tma(ns_sm, &tbar, tphase, red, k, maps, iz, iy, T, w / nt, w % nt, -0.5,
                                                1.5, true)
                                : tile_gemm(ns_sm, red, k, Z, Y, T, w / nt, w % nt, -0.5, 1.5, true);
      if (threadIdx.x == 0) part[w] = rs;
    }
    grid.sync();
    double r = 0.0;
    for (int w = threadIdx.x; w < ntiles; w += blockDim.x) r += part[w];
    r = sqrt(block_sum(r, red));  // same fixed order in every block
    // quadratic convergence down to rounding, or stagnation at rounding level
    if (r <= 8.0 * 2.220446049250313e-16 * sqrt((double)k) || (r < 1e-9 && r > 0.5 * prev)) {
      done = true;
      break;
    }
    prev = r;
    // phase B: Y <- Y T, Z <- T Z
    for (int w = blockIdx.x; w < 2 * ntiles; w += gridDim.x) {
      const int q = w % ntiles;
      if (use_tma) {
        if (w < ntiles)
          tile_gemm_tma(ns_sm, &tbar, tphase, red, k, maps, iy, 4, Yn, q / nt, q % nt, 1.0, 0.0, false);
        else
          tile_gemm_tma(ns_sm, &tbar, tphase, red, k, maps, 4, iz, Zn, q / nt, q % nt, 1.0, 0.0, false);
      } else if (w < ntiles) {
        tile_gemm(ns_sm, red, k, Y, T, Yn, q / nt, q % nt, 1.0, 0.0, false);
      } else {
        tile_gemm(ns_sm, red, k, T, Z, Zn, q / nt, q % nt, 1.0, 0.0, false);
      }
    }
    grid.sync();
    double* t1 = Y;
    Y = Yn;
    Yn = t1;
    double* t2 = Z;
    Z = Zn;
    Zn = t2;
    const int u1 = iy;
    iy = iyn;
    iyn = u1;
    const int u2 = iz;
    iz = izn;
    izn = u2;
  }
  grid.sync();  // every block is done reading part[] before it is reused
  // G^(-1/2) = A^(-1/2) / sqrt(||G||_F); ||A^(-1/2)||_F^2 = sum 1/mu_i bounds
  // the smallest scaled eigenvalue from below (inconclusive -> flag)
  const double s = sqrt(inv_c);
  double fz = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < kk; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / k, j = t % k;
    out[i * ldo + j] = Z[t] * s;
    fz = fma(Z[t], Z[t], fz);
  }
  fz = block_sum(fz, red);
  if (threadIdx.x == 0) part[blockIdx.x] = fz;
  grid.sync();
  if (blockIdx.x != 0) return;
  double f = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) f += part[b];
  f = block_sum(f, red);
  if (threadIdx.x == 0) {
    if (d_iters) *d_iters = it;
    // the reference raises when lambda_min < 1e-14 trace(G); with
    // mu = lambda / ||G||_F and mu_min >= 1 / ||A^(-1/2)||_F^2 = 1 / f that is
    // impossible when f * 1e-14 * trace / ||G||_F <= 1; otherwise ask the
    // host for the exact check
    if (d_status && (!done || !(f * 1e-14 * tr * inv_c <= 1.0) || !(tr > 0.0)))
      atomicOr(d_status, SVDREC_STATUS_NS_CHECK);
  }
}

}  // namespace
}  // namespace svdrec

using namespace svdrec;

extern "C" size_t svdrec_inv_sqrt_workspace_bytes(int32_t k) {
  const int nt = (k + NT - 1) / NT;
  return 5 * align_up((size_t)k * k * 8) + align_up((size_t)(nt * nt + 4096) * 8) + 256;
}

extern "C" int svdrec_inv_sqrt(int32_t k, const double* d_G, int64_t ldg, double* d_Z, int64_t ldz, void* d_work,
                               size_t work_bytes, uint32_t* d_status, int32_t* d_iters, void* stream) {
  SVDREC_ARG(k >= 1 && ldg >= k && ldz >= k, "inv_sqrt: bad arguments");
  if (work_bytes < svdrec_inv_sqrt_workspace_bytes(k)) {
    set_error("inv_sqrt: workspace too small");
    return SVDREC_E_WORKSPACE;
  }
  const int use_tma = (k % 2 == 0) && k >= 2;
  const size_t smem = use_tma ? kNsSmemT : kNsSmem;
  SVDREC_CUDA(smem_attr_once(k_ns, (int)kNsSmemT));
  int per_sm = 0;
  SVDREC_CUDA(blocks_per_sm(k_ns, kNsThreads, smem, &per_sm));
  int max_blocks = per_sm * sm_count();
  if (max_blocks > 4 * sm_count()) max_blocks = 4 * sm_count();
  if (max_blocks > 4096) max_blocks = 4096;
  if (max_blocks < 1) max_blocks = 1;
  const int nt = (k + NT - 1) / NT;
  int nblk = 2 * nt * nt;
  if (nblk > max_blocks) nblk = max_blocks;
  char* w = static_cast<char*>(d_work);
  const size_t m = align_up((size_t)k * k * 8);
  double* Y0 = reinterpret_cast<double*>(w);
  double* Y1 = reinterpret_cast<double*>(w + m);
  double* Z0 = reinterpret_cast<double*>(w + 2 * m);
  double* Z1 = reinterpret_cast<double*>(w + 3 * m);
  double* T = reinterpret_cast<double*>(w + 4 * m);
  double* part = reinterpret_cast<double*>(w + 5 * m);
  NsMaps maps;
  if (use_tma) {
    double* bufs[5] = {Y0, Y1, Z0, Z1, T};
    for (int i = 0; i < 5; ++i) {
      int rc = make_map_2d(&maps.a[i], bufs[i], k, k, k, kKcT, NT);
      if (!rc) rc = make_map_2d(&maps.b[i], bufs[i], k, k, k, kBwT, kKcT);
      if (rc) return rc;
    }
  } else {
    memset(&maps, 0, sizeof(maps));
  }
  int kk = k, maxit = 100, ut = use_tma;
  void* args[] = {&kk, &d_G, &ldg, &d_Z, &ldz, &Y0, &Y1, &Z0, &Z1, &T, &part, &maxit, &d_status, &d_iters, &maps, &ut};
  SVDREC_CUDA(cudaLaunchCooperativeKernel((void*)k_ns, dim3(nblk), dim3(kNsThreads), args, smem, as_stream(stream)));
  note_launches(1);
  return 0;
}
