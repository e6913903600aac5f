// Symmetric PSD eigendecomposition of the k x k Gram for eig_svd.
//
// Replaces scipy.linalg.eigh(gram) in eig_svd (reference
// pkg/src/svdrec/linalg.py:108-138), used by adaptive_pca's final SVD
// (rsvd.py:385) and by latent_from_qb every block of Alg. 5 (cf.py:88).
// Parallel one-sided (Hestenes) Jacobi: columns of W = G V are rotated in
// round-robin pair order (k/2 disjoint pairs per round, one warp per pair,
// one grid barrier per round) until all pairs are orthogonal; then
// w_i = ||W[:, i]|| and V holds the eigenvectors.  The output is sorted
// ascending like LAPACK's, and the eigenvalue floor of the reference
// (w[0] <= 0 or w[0] < 1e-14 * trace) is reported as a status flag.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace svdrec {
namespace {

constexpr int kJThreads = 256;
constexpr int kMaxSweeps = 40;

__device__ __forceinline__ void pair_of(int n, int round, int p, int& i, int& j) {
  // circle method over n (even) players
  if (p == 0) {
    i = n - 1;
    j = round;
  } else {
    i = (round + p) % (n - 1);
    j = (round - p + (n - 1)) % (n - 1);
  }
}

// W column-major rows x k (column c at W + c*rows), V column-major k x k.
__global__ void __launch_bounds__(kJThreads) k_jacobi(int64_t rows, int k, double* __restrict__ W,
                                                      double* __restrict__ V, int* __restrict__ flags, double tol, const double* __restrict__ gnorm_p, uint32_t* d_status) {
  const double gabs = gnorm_p ? 8.0 * 2.220446049250313e-16 * (*gnorm_p) : 0.0;
  cg::grid_group grid = cg::this_grid();
  const int n = (k + 1) & ~1;
  const int npairs = n / 2;
  const int lane = threadIdx.x & 31;
  const int warp = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  int sweep = 0;
  for (; sweep < kMaxSweeps; ++sweep) {
    // three flag words: the one reset here was last read two sweeps ago,
    // with a full sweep of grid barriers in between
    if (blockIdx.x == 0 && threadIdx.x == 0) flags[(sweep + 1) % 3] = 0;
    for (int round = 0; round < n - 1; ++round) {
      for (int pp = warp; pp < npairs; pp += nwarps) {
        int i, j;
        pair_of(n, round, pp, i, j);
        if (i >= k || j >= k) continue;
        if (i > j) {
          const int t = i;
          i = j;
          j = t;
        }
        double* wi = W + (int64_t)i * rows;
        double* wj = W + (int64_t)j * rows;
        double a = 0.0, bq = 0.0, g = 0.0;
        for (int64_t e = lane; e < rows; e += 32) {
          const double x = wi[e], y = wj[e];
          a = fma(x, x, a);
          bq = fma(y, y, bq);
          g = fma(x, y, g);
        }
        a = warp_sum(a);
        bq = warp_sum(bq);
        g = warp_sum(g);
        if (g == 0.0 || fabs(g) <= tol * sqrt(a * bq) || fabs(g) <= gabs * (sqrt(a) + sqrt(bq))) continue;
        const double zeta = (bq - a) / (2.0 * g);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double c = 1.0 / sqrt(fma(t, t, 1.0));
        const double s = c * t;
        for (int64_t e = lane; e < rows; e += 32) {
          const double x = wi[e], y = wj[e];
          wi[e] = c * x - s * y;
          wj[e] = s * x + c * y;
        }
        double* vi = V + (int64_t)i * k;
        double* vj = V + (int64_t)j * k;
        for (int e = lane; e < k; e += 32) {
          const double x = vi[e], y = vj[e];
          vi[e] = c * x - s * y;
          vj[e] = s * x + c * y;
        }
        if (lane == 0) flags[sweep % 3] = 1;
      }
      grid.sync();
    }
    if (*(volatile int*)&flags[sweep % 3] == 0) break;
  }
  if (sweep == kMaxSweeps && blockIdx.x == 0 && threadIdx.x == 0 && d_status)
    atomicOr(d_status, SVDREC_STATUS_NO_CONVERGE);
}

// eigenvalue_i = ||W[:, i]||; sort ascending (rank by comparison, ties by
// index) and scatter V columns into the row-major output.
__global__ void k_norms(int64_t rows, const double* __restrict__ W, double* __restrict__ lam) {
  const int i = blockIdx.x;
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < rows; e += blockDim.x)
    s = fma(W[(int64_t)i * rows + e], W[(int64_t)i * rows + e], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) lam[i] = sqrt(s);
}

__global__ void k_sort_out(int k, const double* __restrict__ lam, const double* __restrict__ Vc, double* __restrict__ w,
                           double* __restrict__ Vout, int64_t ldv, const double* __restrict__ G, int64_t ldg,
                           uint32_t* d_status, int descending, int64_t rows, const double* __restrict__ Wc,
                           double* __restrict__ Uout, int64_t ldu) {
  const int i = blockIdx.x;
  const double li = lam[i];
  __shared__ int rank_s;
  if (threadIdx.x == 0) rank_s = 0;
  __syncthreads();
  int cnt = 0;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const double lj = lam[j];
    cnt += descending ? ((lj > li) || (lj == li && j < i)) : ((lj < li) || (lj == li && j < i));
  }
  atomicAdd(&rank_s, cnt);
  __syncthreads();
  const int rk = rank_s;
  if (threadIdx.x == 0) w[rk] = li;
  for (int e = threadIdx.x; e < k; e += blockDim.x) Vout[(int64_t)e * ldv + rk] = Vc[(int64_t)i * k + e];
  if (Uout) {
    const double inv = li > 0.0 ? 1.0 / li : 0.0;
    for (int64_t e = threadIdx.x; e < rows; e += blockDim.x) Uout[e * ldu + rk] = Wc[(int64_t)i * rows + e] * inv;
  }
  if (G && rk == 0 && threadIdx.x == 0 && d_status) {
    double tr = 0.0;
    for (int e = 0; e < k; ++e) tr += G[(int64_t)e * ldg + e];
    if (li <= 0.0 || li < 1e-14 * tr) atomicOr(d_status, SVDREC_STATUS_NEAR_SINGULAR);
  }
}

// W (column-major rows x k) <- A (row-major, lda); V <- I_k
__global__ void k_init(int64_t rows, int k, const double* __restrict__ A, int64_t lda, double* __restrict__ W,
                       double* __restrict__ V) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < rows * k) {
    const int64_t c = t / rows, e = t % rows;
    W[t] = A[e * lda + c];
  }
  if (t < (int64_t)k * k) V[t] = (t / k == t % k) ? 1.0 : 0.0;
}

// Warm start: V <- V0 (row-major k x k, columns = start basis),
// W <- G V0 (column-major).  The previous block's eigenvectors padded with
// the identity make the new Gram nearly diagonal, so few sweeps remain.
__global__ void k_init_warm(int k, const double* __restrict__ G, int64_t ldg, const double* __restrict__ V0,
                            int64_t ldv0, double* __restrict__ W, double* __restrict__ V) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)k * k) return;
  const int c = (int)(t / k), e = (int)(t % k);
  double acc = 0.0;
  for (int q = 0; q < k; ++q) acc = fma(G[(int64_t)e * ldg + q], V0[(int64_t)q * ldv0 + c], acc);
  W[t] = acc;
  V[t] = V0[(int64_t)e * ldv0 + c];
}

// ---- blocked one-sided Jacobi --------------------------------------------
// Columns are grouped in blocks of kBW; each outer round pairs blocks
// (circle method over the blocks), one CTA per block pair loads the pair's
// 2*kBW columns of W into shared memory, runs one full inner one-sided
// sweep over those columns (kBW warps, one column pair each per inner
// round, __syncthreads between inner rounds), writes them back and applies
// the accumulated 2kBW x 2kBW rotation to the same columns of V.  One grid
// barrier per outer round: (nblocks - 1) per sweep instead of (k - 1).
constexpr int kBW = 16;
constexpr int kBT = kBW * 32;  // threads per CTA: one warp per inner pair

__device__ __forceinline__ void circle(int n, int round, int p, int& i, int& j) {
  if (p == 0) {
    i = n - 1;
    j = round;
  } else {
    i = (round + p) % (n - 1);
    j = (round - p + (n - 1)) % (n - 1);
  }
}

__global__ void __launch_bounds__(kBT) k_bjacobi(int rows, int k, double* __restrict__ W, double* __restrict__ V,
                                                 int* __restrict__ flags, double tol, const double* __restrict__ gnorm_p,
                                                 uint32_t* d_status) {
  cg::grid_group grid = cg::this_grid();
  const double gabs = gnorm_p ? 8.0 * 2.220446049250313e-16 * (*gnorm_p) : 0.0;
  extern __shared__ double sw[];                 // [2*kBW][ldw]
  __shared__ double Jm[2 * kBW][2 * kBW + 1];    // accumulated rotation (column-major: Jm[col][row])
  __shared__ int cols[2 * kBW];
  const int ldw = rows | 1;
  const int nb = (k + kBW - 1) / kBW;
  const int nbp = (nb + 1) & ~1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    if (blockIdx.x == 0 && threadIdx.x == 0) flags[(sweep + 1) % 3] = 0;
    for (int round = 0; round < (nbp > 1 ? nbp - 1 : 1); ++round) {
      for (int g = blockIdx.x; g < (nbp > 1 ? nbp / 2 : 1); g += gridDim.x) {
        int bi, bj;
        if (nbp > 1) {
          circle(nbp, round, g, bi, bj);
        } else {
          bi = 0;
          bj = 1;  // single block: the second half is empty
        }
        if (threadIdx.x < 2 * kBW) {
          const int l = threadIdx.x;
          const int c = (l < kBW) ? bi * kBW + l : bj * kBW + (l - kBW);
          cols[l] = (c < k && (l < kBW ? bi : bj) < nb) ? c : -1;
        }
        for (int t = threadIdx.x; t < 2 * kBW * 2 * kBW; t += kBT) Jm[t / (2 * kBW)][t % (2 * kBW)] = 0.0;
        __syncthreads();
        if (threadIdx.x < 2 * kBW) Jm[threadIdx.x][threadIdx.x] = 1.0;
        for (int t = threadIdx.x; t < 2 * kBW * rows; t += kBT) {
          const int l = t / rows, e = t - l * rows;
          sw[l * ldw + e] = cols[l] >= 0 ? W[(int64_t)cols[l] * rows + e] : 0.0;
        }
        __syncthreads();
        bool rotated = false;
        for (int ir = 0; ir < 2 * kBW - 1; ++ir) {
          int a, b;
          circle(2 * kBW, ir, warp, a, b);
          if (cols[a] >= 0 && cols[b] >= 0) {
            double* wa = sw + a * ldw;
            double* wb = sw + b * ldw;
            double al = 0.0, be = 0.0, ga = 0.0;
            for (int e = lane; e < rows; e += 32) {
              const double x = wa[e], y = wb[e];
              al = fma(x, x, al);
              be = fma(y, y, be);
              ga = fma(x, y, ga);
            }
            al = warp_sum(al);
            be = warp_sum(be);
            ga = warp_sum(ga);
            if (ga != 0.0 && fabs(ga) > tol * sqrt(al * be) && fabs(ga) > gabs * (sqrt(al) + sqrt(be))) {
              const double zeta = (be - al) / (2.0 * ga);
              const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
              const double c = 1.0 / sqrt(fma(t, t, 1.0));
              const double s = c * t;
              for (int e = lane; e < rows; e += 32) {
                const double x = wa[e], y = wb[e];
                wa[e] = c * x - s * y;
                wb[e] = s * x + c * y;
              }
              const double x = Jm[a][lane], y = Jm[b][lane];
              Jm[a][lane] = c * x - s * y;
              Jm[b][lane] = s * x + c * y;
              rotated = true;
            }
          }
          __syncthreads();
        }
        if (rotated && lane == 0) flags[sweep % 3] = 1;
        for (int t = threadIdx.x; t < 2 * kBW * rows; t += kBT) {
          const int l = t / rows, e = t - l * rows;
          if (cols[l] >= 0) W[(int64_t)cols[l] * rows + e] = sw[l * ldw + e];
        }
        __syncthreads();
        // V[:, cols] <- V[:, cols] @ Jm, rows of V in chunks staged in sw
        for (int e0 = 0; e0 < k; e0 += (rows > 64 ? 64 : rows)) {
          const int ch = min(rows > 64 ? 64 : rows, k - e0);
          for (int t = threadIdx.x; t < 2 * kBW * ch; t += kBT) {
            const int l = t / ch, e = t - l * ch;
            sw[l * ldw + e] = cols[l] >= 0 ? V[(int64_t)cols[l] * k + e0 + e] : 0.0;
          }
          __syncthreads();
          for (int t = threadIdx.x; t < 2 * kBW * ch; t += kBT) {
            const int l = t / ch, e = t - l * ch;
            if (cols[l] < 0) continue;
            double acc = 0.0;
#pragma unroll 8
            for (int q = 0; q < 2 * kBW; ++q) acc = fma(sw[q * ldw + e], Jm[l][q], acc);
            V[(int64_t)cols[l] * k + e0 + e] = acc;
          }
          __syncthreads();
        }
      }
      grid.sync();
    }
    if (*(volatile int*)&flags[sweep % 3] == 0) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) flags[3] = sweep;  // diagnostics: sweeps used
  if (sweep == 60 && blockIdx.x == 0 && threadIdx.x == 0 && d_status) atomicOr(d_status, SVDREC_STATUS_NO_CONVERGE);
}

constexpr int kBRowsMax = 760;  // 2*kBW*ldw*8 <= 200 KB

// Frobenius norm of n contiguous doubles; applied to W right after the
// (warm) init, where ||G V0||_F = ||G||_F.
__global__ void k_fro(int64_t n, const double* __restrict__ G, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(G[i], G[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = sqrt(s);
}

// shared driver: one-sided Jacobi on the rows x k block A
int run_jacobi(int64_t rows, int k, const double* A, int64_t lda, double* W, double* V, double* lam, int* flags,
               uint32_t* d_status, cudaStream_t s, const double* V0 = nullptr, int64_t ldv0 = 0, bool absolute = false) {
  const int64_t tot = rows * k > (int64_t)k * k ? rows * k : (int64_t)k * k;
  if (V0 && rows == k)
    k_init_warm<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(k, A, lda, V0, ldv0, W, V);
  else
    k_init<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(rows, k, A, lda, W, V);
  int rc = check_launch("jacobi_init");
  if (rc) return rc;
  // symmetric input: stop rotating once |w_i.w_j| is at the eps*||G|| level of
  // the columns themselves (their absolute error), as LAPACK eigh guarantees
  const double* gnp = nullptr;
  if (absolute) {
    k_fro<<<1, 256, 0, s>>>(rows * k, W, lam);
    rc = check_launch("jacobi_fro");
    if (rc) return rc;
    gnp = lam;
  }
  const double tol_b = fmin(1e-10, 2.220446049250313e-16 * (double)(rows > 4 ? rows : 4));
  if (k > 1 && rows <= kBRowsMax) {
    const size_t smem = (size_t)2 * kBW * (kBRowsMax | 1) * 8;
    SVDREC_CUDA(smem_attr_once(k_bjacobi, (int)smem));
    int per_sm = 0;
    SVDREC_CUDA(blocks_per_sm(k_bjacobi, kBT, smem, &per_sm));
    int max_blocks_b = per_sm * sm_count();
    if (max_blocks_b < 1) max_blocks_b = 1;
    const int nb = (k + kBW - 1) / kBW;
    const int npairs = nb > 1 ? ((nb + 1) & ~1) / 2 : 1;
    int nblk = npairs < max_blocks_b ? npairs : max_blocks_b;
    int r32 = (int)rows, kk32 = k;
    double tol = tol_b;
    void* args[] = {&r32, &kk32, &W, &V, &flags, &tol, &gnp, &d_status};
    SVDREC_CUDA(cudaMemsetAsync(flags, 0, 3 * sizeof(int), s));
    SVDREC_CUDA(cudaLaunchCooperativeKernel((void*)k_bjacobi, dim3(nblk), dim3(kBT), args, smem, s));
    note_launches(1);
  } else if (k > 1) {
    int per_sm = 0;
    SVDREC_CUDA(blocks_per_sm(k_jacobi, kJThreads, 0, &per_sm));
    int max_blocks = per_sm * sm_count();
    if (max_blocks < 1) max_blocks = 1;
    const int npairs = ((k + 1) & ~1) / 2;
    int nblk = (npairs * 32 + kJThreads - 1) / kJThreads;
    if (nblk > max_blocks) nblk = max_blocks;
    // convergence floor of the computed cosine: ~rows ulps of the dot products
    const int64_t lenf = rows > 4 ? rows : 4;
    double tol = 2.220446049250313e-16 * (double)lenf;
    if (tol > 1e-10) tol = 1e-10;
    int64_t rr = rows;
    int kk32 = k;
    void* args[] = {&rr, &kk32, &W, &V, &flags, &tol, &gnp, &d_status};
    SVDREC_CUDA(cudaMemsetAsync(flags, 0, 3 * sizeof(int), s));
    SVDREC_CUDA(cudaLaunchCooperativeKernel((void*)k_jacobi, dim3(nblk), dim3(kJThreads), args, 0, s));
    note_launches(1);
  }
  k_norms<<<k, 128, 0, s>>>(rows, W, lam);
  return check_launch("jacobi_norms");
}

}  // namespace
}  // namespace svdrec

using namespace svdrec;

extern "C" size_t svdrec_syev_workspace_bytes(int32_t k) {
  return 2 * align_up((size_t)k * k * 8) + align_up((size_t)k * 8) + 256;
}

extern "C" int svdrec_syev(int32_t k, const double* d_G, int64_t ldg, const double* d_V0, int64_t ldv0, double* d_w,
                           double* d_V, int64_t ldv, void* d_work, size_t work_bytes, uint32_t* d_status,
                           void* stream) {
  SVDREC_ARG(k >= 1 && ldg >= k && ldv >= k, "syev: bad arguments");
  if (work_bytes < svdrec_syev_workspace_bytes(k)) {
    set_error("syev: workspace too small");
    return SVDREC_E_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  char* w = static_cast<char*>(d_work);
  double* W = reinterpret_cast<double*>(w);
  double* V = reinterpret_cast<double*>(w + align_up((size_t)k * k * 8));
  double* lam = reinterpret_cast<double*>(w + 2 * align_up((size_t)k * k * 8));
  int* flags = reinterpret_cast<int*>(w + 2 * align_up((size_t)k * k * 8) + align_up((size_t)k * 8));
  SVDREC_ARG(!d_V0 || ldv0 >= k, "syev: bad ldv0");
  int rc = run_jacobi(k, k, d_G, ldg, W, V, lam, flags, d_status, s, d_V0, ldv0, true);
  if (rc) return rc;
  k_sort_out<<<k, 128, 0, s>>>(k, lam, V, d_w, d_V, ldv, d_G, ldg, d_status, 0, 0, nullptr, nullptr, 0);
  return check_launch("syev_sort");
}

extern "C" size_t svdrec_gesvj_workspace_bytes(int64_t rows, int32_t k) {
  return align_up((size_t)rows * k * 8) + align_up((size_t)k * k * 8) + align_up((size_t)k * 8) + 256;
}

extern "C" int svdrec_gesvj(int64_t rows, int32_t k, const double* d_A, int64_t lda, double* d_s, double* d_U,
                            int64_t ldu, double* d_V, int64_t ldv, void* d_work, size_t work_bytes,
                            uint32_t* d_status, void* stream) {
  SVDREC_ARG(k >= 1 && rows >= k && lda >= k && ldu >= k && ldv >= k, "gesvj: needs rows >= k >= 1");
  if (work_bytes < svdrec_gesvj_workspace_bytes(rows, k)) {
    set_error("gesvj: workspace too small");
    return SVDREC_E_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  char* w = static_cast<char*>(d_work);
  double* W = reinterpret_cast<double*>(w);
  double* V = reinterpret_cast<double*>(w + align_up((size_t)rows * k * 8));
  double* lam = reinterpret_cast<double*>(w + align_up((size_t)rows * k * 8) + align_up((size_t)k * k * 8));
  int* flags = reinterpret_cast<int*>(w + align_up((size_t)rows * k * 8) + align_up((size_t)k * k * 8) +
                                      align_up((size_t)k * 8));
  int rc = run_jacobi(rows, k, d_A, lda, W, V, lam, flags, d_status, s);
  if (rc) return rc;
  k_sort_out<<<k, 128, 0, s>>>(k, lam, V, d_s, d_V, ldv, nullptr, 0, d_status, 1, rows, W, d_U, ldu);
  return check_launch("gesvj_sort");
}
