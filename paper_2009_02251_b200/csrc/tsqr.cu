// Tall-skinny Householder QR (TSQR) -> explicit orthonormal Q.
//
// Replaces orthonormal_basis (reference pkg/src/svdrec/linalg.py:54-81,
// scipy.linalg.qr economic = LAPACK dgeqrf + dorgqr), called 2-4 times per
// block by the QB engines (rsvd.py:136-142, 186-193).  A flat Householder
// QR is b sequential column steps over all m rows; here the rows are cut
// into chunks that fit one CTA's shared memory, each CTA factors its chunk
// with Householder reflections entirely on-chip, the b x b R factors are
// stacked and factored again (a reduction tree, 2-4 levels for m <= 10^7),
// and the explicit Q is rebuilt top-down by applying each chunk's
// reflectors to its b x b block of the coarser Q.  Every matrix element is
// read once and written once per direction, there are no grid-wide
// barriers, and the result is orthonormal to working precision even for
// rank-deficient input (the reference's check_rank=False contract).
// Q is unique up to column signs; all consumers downstream are sign
// invariant (B = Q.T A rows flip, B.T B, Q B and row energies do not).
#include <vector>

#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

extern "C" size_t svdrec_gemm_tn_workspace_bytes(int64_t r, int64_t p, int64_t q);
extern "C" int svdrec_gemm_tn(int64_t r, int64_t p, int64_t q, double alpha, const double* d_X, int64_t ldx,
                              const double* d_Y, int64_t ldy, double beta, double* d_C, int64_t ldc, void* d_work,
                              size_t work_bytes, void* stream);
extern "C" int svdrec_gemm_nn(int64_t r, int64_t p, int64_t q, double alpha, const double* d_X, int64_t ldx,
                              const double* d_C, int64_t ldc, double beta, double* d_Y, int64_t ldy, void* stream);

namespace svdrec {
namespace {

constexpr int kThreads = 256;
constexpr size_t kChunkBytes = 96 * 1024;  // one chunk's panel in smem

// Rows per chunk: small panels (~32 KB) so several CTAs share an SM and hide
// each other's barrier latency, but >= 2b so every tree level halves the
// rows, and <= the 2-matrix shared-memory budget of the Q builder.
inline int rc_max_for(int b) {
  int rc = (int)(32768 / (8 * (size_t)b));
  if (rc < 2 * b) rc = 2 * b;
  const int cap = (int)(kChunkBytes / (8 * (size_t)b));
  return rc < cap ? rc : cap;
}

struct Level {
  int64_t rows, nc;
  size_t off_v, off_tau, off_next, off_q;
};

struct Plan {
  int b;
  int rcmax;
  std::vector<Level> lv;
  size_t total;
};

Plan make_plan(int64_t r, int b) {
  Plan p;
  p.b = b;
  p.rcmax = rc_max_for(b);
  size_t o = 0;
  int64_t rows = r;
  while (true) {
    Level L{};
    L.rows = rows;
    L.nc = (rows + p.rcmax - 1) / p.rcmax;
    L.off_v = o;
    o = align_up(o + (size_t)rows * b * 8);
    L.off_tau = o;
    o = align_up(o + (size_t)L.nc * b * 8);
    L.off_next = o;
    o = align_up(o + (size_t)L.nc * b * b * 8);
    L.off_q = o;
    o = align_up(o + (p.lv.empty() ? 0 : (size_t)rows * b * 8));
    p.lv.push_back(L);
    if (L.nc == 1) break;
    rows = L.nc * b;
  }
  p.total = o;
  return p;
}

__device__ __forceinline__ void chunk_range(int64_t rows, int64_t nc, int64_t c, int64_t& a, int64_t& e) {
  a = (c * rows) / nc;
  e = ((c + 1) * rows) / nc;
}

// Householder QR of one chunk.  M is column-major in smem: M[col*ldm + row].
__device__ void factor_chunk(int64_t c, int64_t rows, int64_t nc, int b, const double* __restrict__ in,
                             int64_t ldin, double* __restrict__ vout, double* __restrict__ tau,
                             double* __restrict__ rout) {
  extern __shared__ double sm[];
  __shared__ double dots[128];
  __shared__ double wv[128];
  __shared__ double coef[3];  // tau, beta, scale
  int64_t a, e;
  chunk_range(rows, nc, c, a, e);
  const int rc = (int)(e - a);
  const int ldm = rc | 1;
  double* M = sm;
  for (int t = threadIdx.x; t < rc * b; t += kThreads) {
    const int i = t / b, col = t - i * b;
    M[col * ldm + i] = in[(a + i) * ldin + col];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int jmax = min(b, rc);
  for (int j = 0; j < jmax; ++j) {
    const double* xj = M + j * ldm;
    for (int col = j + warp; col < b; col += kThreads / 32) {
      const double* mc = M + col * ldm;
      double s = 0.0;
      for (int i = j + 1 + lane; i < rc; i += 32) s = fma(xj[i], mc[i], s);
      s = warp_sum(s);
      if (lane == 0) dots[col] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const double alpha = xj[j], sigma = dots[j];
      double t = 0.0, beta = alpha, scale = 0.0;
      if (sigma != 0.0) {
        const double nrm = sqrt(fma(alpha, alpha, sigma));
        beta = alpha >= 0.0 ? -nrm : nrm;
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      coef[0] = t;
      coef[1] = beta;
      coef[2] = scale;
    }
    __syncthreads();
    const double t = coef[0], scale = coef[2];
    for (int col = j + 1 + threadIdx.x; col < b; col += kThreads) wv[col] = t * fma(scale, dots[col], M[col * ldm + j]);
    // v into column j (v_j = 1 implicit)
    for (int i = j + 1 + threadIdx.x; i < rc; i += kThreads) M[j * ldm + i] *= scale;
    __syncthreads();
    const int ncol = b - j - 1, nrow = rc - j;
    for (int q = threadIdx.x; q < ncol * nrow; q += kThreads) {
      const int cc = j + 1 + q / nrow, i = j + q % nrow;
      const double vi = (i == j) ? 1.0 : M[j * ldm + i];
      M[cc * ldm + i] -= wv[cc] * vi;
    }
    if (threadIdx.x == 0) {
      tau[c * b + j] = t;
      M[j * ldm + j] = coef[1];  // R_jj
    }
    __syncthreads();
  }
  for (int j = jmax; j < b; ++j)
    if (threadIdx.x == 0) tau[c * b + j] = 0.0;
  // R (b x b row-major, upper) -> rout rows c*b .. c*b+b-1
  for (int t = threadIdx.x; t < b * b; t += kThreads) {
    const int i = t / b, col = t - i * b;
    rout[(c * b + i) * (int64_t)b + col] = (col >= i && i < rc) ? M[col * ldm + i] : 0.0;
  }
  // reflectors (strict lower part) -> vout rows a..e-1 (row-major, ld b)
  for (int t = threadIdx.x; t < rc * b; t += kThreads) {
    const int i = t / b, col = t - i * b;
    vout[(a + i) * (int64_t)b + col] = i > col ? M[col * ldm + i] : 0.0;
  }
}

// Apply one chunk's reflectors to E = [Qc ; 0] (Qc = rows c*b.. of the
// coarser explicit Q, or the identity at the top) and store the chunk's
// rows of this level's explicit Q.
__device__ void buildq_chunk(int64_t c, int64_t rows, int64_t nc, int b, const double* __restrict__ vin,
                             const double* __restrict__ tau, const double* __restrict__ qcoarse,
                             double* __restrict__ qout, int64_t ldq) {
  extern __shared__ double sm[];
  __shared__ double wv[128];
  int64_t a, e;
  chunk_range(rows, nc, c, a, e);
  const int rc = (int)(e - a);
  const int ldm = rc | 1;
  double* V = sm;
  double* E = sm + (size_t)b * ldm;
  for (int t = threadIdx.x; t < rc * b; t += kThreads) {
    const int i = t / b, col = t - i * b;
    V[col * ldm + i] = vin[(a + i) * (int64_t)b + col];
    double ev = 0.0;
    if (i < b) ev = qcoarse ? qcoarse[(c * b + i) * (int64_t)b + col] : (i == col ? 1.0 : 0.0);
    E[col * ldm + i] = ev;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int jmax = min(b, rc);
  for (int j = jmax - 1; j >= 0; --j) {
    const double t = tau[c * b + j];
    if (t == 0.0) continue;  // uniform across the block
    const double* v = V + j * ldm;
    for (int col = warp; col < b; col += kThreads / 32) {
      const double* ec = E + col * ldm;
      double s = lane == 0 ? ec[j] : 0.0;
      for (int i = j + 1 + lane; i < rc; i += 32) s = fma(v[i], ec[i], s);
      s = warp_sum(s);
      if (lane == 0) wv[col] = t * s;
    }
    __syncthreads();
    const int nrow = rc - j;
    for (int q = threadIdx.x; q < b * nrow; q += kThreads) {
      const int col = q / nrow, i = j + q % nrow;
      const double vi = (i == j) ? 1.0 : v[i];
      E[col * ldm + i] -= wv[col] * vi;
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < rc * b; t += kThreads) {
    const int i = t / b, col = t - i * b;
    qout[(a + i) * ldq + col] = E[col * ldm + i];
  }
}

__global__ void __launch_bounds__(kThreads) k_factor(int64_t rows, int64_t nc, int b, const double* __restrict__ in,
                                                     int64_t ldin, double* __restrict__ vout,
                                                     double* __restrict__ tau, double* __restrict__ rout) {
  factor_chunk(blockIdx.x, rows, nc, b, in, ldin, vout, tau, rout);
}

__global__ void __launch_bounds__(kThreads) k_buildq(int64_t rows, int64_t nc, int b, const double* __restrict__ vin,
                                                     const double* __restrict__ tau,
                                                     const double* __restrict__ qcoarse, double* __restrict__ qout,
                                                     int64_t ldq) {
  buildq_chunk(blockIdx.x, rows, nc, b, vin, tau, qcoarse, qout, ldq);
}

// The whole TSQR (every factor level, then every Q level) as ONE cooperative
// launch, gated on a device flag: the CholeskyQR2 fallback costs a single
// launch that returns at once when the flag is clear (it was 2 x levels
// launches, ~20 us per orth call).
constexpr int kMaxLevels = 24;  // halving tree: rows up to ~2^23 x (chunk rows) at b = 64
struct CoopLevels {
  int nl;
  int64_t rows[kMaxLevels], nc[kMaxLevels];
  double* v[kMaxLevels];
  double* tau[kMaxLevels];
  double* next[kMaxLevels];
  double* q[kMaxLevels];
};

__global__ void __launch_bounds__(kThreads) k_tsqr_coop(const __grid_constant__ CoopLevels L, int b,
                                                        const double* __restrict__ A, int64_t lda,
                                                        double* __restrict__ Q, int64_t ldq, double* __restrict__ R,
                                                        const uint32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;  // uniform: CholeskyQR2 succeeded
  cg::grid_group grid = cg::this_grid();
  const double* in = A;
  int64_t ldin = lda;
  for (int l = 0; l < L.nl; ++l) {
    double* rout = (l == L.nl - 1) ? R : L.next[l];
    for (int64_t c = blockIdx.x; c < L.nc[l]; c += gridDim.x) {
      factor_chunk(c, L.rows[l], L.nc[l], b, in, ldin, L.v[l], L.tau[l], rout);
      __syncthreads();
    }
    grid.sync();
    in = rout;
    ldin = b;
  }
  const double* coarse = nullptr;
  for (int l = L.nl - 1; l >= 0; --l) {
    double* qo = l == 0 ? Q : L.q[l];
    const int64_t ldo = l == 0 ? ldq : b;
    for (int64_t c = blockIdx.x; c < L.nc[l]; c += gridDim.x) {
      buildq_chunk(c, L.rows[l], L.nc[l], b, L.v[l], L.tau[l], coarse, qo, ldo);
      __syncthreads();
    }
    grid.sync();
    coarse = qo;
  }
}

}  // namespace
}  // namespace svdrec

using namespace svdrec;

extern "C" size_t svdrec_tsqr_workspace_bytes(int64_t r, int32_t b) {
  if (b < 1 || b > 80 || r < b) return 256;
  return make_plan(r, b).total + 256;
}

namespace svdrec {
namespace {

// TSQR launch sequence; with ``gate`` non-null every kernel returns at once
// unless *gate != 0 (the CholeskyQR2 fast path flagged itself unreliable).
int run_tsqr(const Plan& p, int64_t r, int32_t b, const double* d_A, int64_t lda, double* d_Q, int64_t ldq,
             double* d_R, char* w, const uint32_t* gate, cudaStream_t s) {
  const size_t smem_f = (size_t)b * ((p.rcmax + 1) | 1) * 8;
  const size_t smem_q = 2 * smem_f;
  SVDREC_CUDA(smem_attr_once(k_factor, 2 * kChunkBytes + 4096));
  SVDREC_CUDA(smem_attr_once(k_buildq, 2 * kChunkBytes + 4096));
  const int nl = (int)p.lv.size();
  const double* in = d_A;
  int64_t ldin = lda;
  for (int l = 0; l < nl; ++l) {
    const Level& L = p.lv[l];
    double* rout = (l == nl - 1) ? d_R : reinterpret_cast<double*>(w + L.off_next);
    k_factor<<<(unsigned)L.nc, kThreads, smem_f, s>>>(L.rows, L.nc, b, in, ldin,
                                                      reinterpret_cast<double*>(w + L.off_v),
                                                      reinterpret_cast<double*>(w + L.off_tau), rout);
    int rc = check_launch("tsqr_factor");
    if (rc) return rc;
    in = rout;
    ldin = b;
  }
  const double* coarse = nullptr;
  for (int l = nl - 1; l >= 0; --l) {
    const Level& L = p.lv[l];
    double* qo = l == 0 ? d_Q : reinterpret_cast<double*>(w + L.off_q);
    const int64_t ldo = l == 0 ? ldq : b;
    k_buildq<<<(unsigned)L.nc, kThreads, smem_q, s>>>(L.rows, L.nc, b, reinterpret_cast<double*>(w + L.off_v),
                                                      reinterpret_cast<double*>(w + L.off_tau), coarse, qo, ldo);
    int rc = check_launch("tsqr_buildq");
    if (rc) return rc;
    coarse = qo;
  }
  return 0;
}

// Gated cooperative TSQR (see k_tsqr_coop).
int run_tsqr_gated(const Plan& p, int64_t r, int32_t b, const double* d_A, int64_t lda, double* d_Q, int64_t ldq,
                   double* d_R, char* w, const uint32_t* gate, cudaStream_t s) {
  const size_t smem_f = (size_t)b * ((p.rcmax + 1) | 1) * 8;
  const size_t smem_q = 2 * smem_f;
  const int nl = (int)p.lv.size();
  if (nl > kMaxLevels) {
    set_error("orth: TSQR tree deeper than %d levels", kMaxLevels);
    return SVDREC_E_UNSUPPORTED;
  }
  SVDREC_CUDA(smem_attr_once(k_tsqr_coop, 2 * kChunkBytes + 4096));
  CoopLevels L{};
  L.nl = nl;
  int64_t maxnc = 1;
  for (int l = 0; l < nl; ++l) {
    const Level& v = p.lv[l];
    L.rows[l] = v.rows;
    L.nc[l] = v.nc;
    L.v[l] = reinterpret_cast<double*>(w + v.off_v);
    L.tau[l] = reinterpret_cast<double*>(w + v.off_tau);
    L.next[l] = reinterpret_cast<double*>(w + v.off_next);
    L.q[l] = reinterpret_cast<double*>(w + v.off_q);
    if (v.nc > maxnc) maxnc = v.nc;
  }
  int per_sm = 0;
  SVDREC_CUDA(blocks_per_sm(k_tsqr_coop, kThreads, smem_q, &per_sm));
  int64_t grid = (int64_t)(per_sm > 0 ? per_sm : 1) * sm_count();
  if (grid > maxnc) grid = maxnc;
  int32_t bb = b;
  void* args[] = {&L, &bb, &d_A, &lda, &d_Q, &ldq, &d_R, &gate};
  SVDREC_CUDA(cudaLaunchCooperativeKernel((void*)k_tsqr_coop, dim3((unsigned)grid), dim3(kThreads), args, smem_q, s));
  note_launches(1);
  return 0;
}

// ---- CholeskyQR2 fast path -------------------------------------------------
// G = Y.T Y over a row range per CTA (upper triangle pairs), fixed-order sum.
constexpr int kGramRows = 64;

// Cholesky G = R.T R (upper R) of the reduced Gram pairs, then R^-1.
// flag |= 1 when a pivot is non-positive or (min R_jj / max R_jj)^2 < 1e-12
// (kappa(Y) > 1e6: CholeskyQR2 would not reach working-precision
// orthogonality), in which case the TSQR fallback runs.  R^-1 is built in
// the lower triangle of the same shared array (column c by thread c).
// Cholesky of the Gram held in G's upper triangle (b <= 64), then R^-1 into
// Rinv (b x b, row-major).  flag |= 1 when a pivot is non-positive or
// (min R_jj / max R_jj)^2 < 1e-12 (kappa(Y) > 1e6: CholeskyQR2 would not
// reach working-precision orthogonality), in which case the TSQR fallback
// runs.  R^-1 is built in the strict lower triangle of G (column c by
// thread c).  Whole CTA; G, dinv, bad in shared memory.
__device__ void chol_inv_smem(int b, double (*G)[65], double* dinv, int* bad, double* __restrict__ Rinv,
                              uint32_t* __restrict__ flag, uint32_t* __restrict__ zero_flag = nullptr) {
  if (threadIdx.x == 0) *bad = 0;
  __syncthreads();
  double dmax = 0.0, dmin = 1e300;
  for (int j = 0; j < b; ++j) {
    if (threadIdx.x == 0) {
      const double d = G[j][j];
      if (!(d > 0.0)) *bad = 1;
      G[j][j] = d > 0.0 ? sqrt(d) : 1.0;
      dinv[j] = 1.0 / G[j][j];
    }
    __syncthreads();
    const double rjj = G[j][j];
    for (int c = j + 1 + threadIdx.x; c < b; c += blockDim.x) G[j][c] /= rjj;
    __syncthreads();
    const int nt = b - j - 1;
    for (int t = threadIdx.x; t < nt * nt; t += blockDim.x) {
      const int c1 = j + 1 + t / nt, c2 = j + 1 + t % nt;
      if (c2 >= c1) G[c1][c2] -= G[j][c1] * G[j][c2];
    }
    __syncthreads();
    dmax = fmax(dmax, rjj);
    dmin = fmin(dmin, rjj);
  }
  if (threadIdx.x == 0 && (*bad || dmin * dmin < 1e-12 * dmax * dmax)) atomicOr(flag, 1u);
  if (threadIdx.x == 0 && zero_flag && *bad) atomicOr(zero_flag, 1u);
  const int c = threadIdx.x;
  if (c < b) {
    for (int i = c - 1; i >= 0; --i) {
      double x = G[i][c] * dinv[c];
      for (int t = i + 1; t < c; ++t) x = fma(G[i][t], G[c][t], x);
      G[c][i] = -x * dinv[i];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < b * b; t += blockDim.x) {
    const int i = t / b, cc = t - i * b;
    Rinv[t] = i == cc ? dinv[cc] : (i < cc ? G[cc][i] : 0.0);
  }
}

// ---------------------------------------------------------------------------
// DMMA CholeskyQR pass for b <= 32 (NT = ceil(b/8) fragment tiles).
//
// k_cqr_gram: G = Y.T Y on the FP64 tensor cores.  A k-step is 4 rows; the
// A fragment of m-tile i (A[8i+g][t] = Y[row t][8i+g]) and the B fragment of
// n-tile j (B[t][8j+g] = Y[row t][8j+g]) are the same loads, so one 8-B load
// per tile per lane feeds the NT(NT+1)/2 upper tiles.  Warp partials are
// added in warp order in shared memory, CTA partials go to ``part``; the
// CTA that finishes last (atomic ticket) sums them in CTA order, factors G
// and writes R^-1 -- one launch for Gram, reduction, Cholesky and inverse.
constexpr int kCqrThreads = 512, kCqrWarps = kCqrThreads / 32, kCqrKs = 8, kCqrGroup = 16;

__device__ __forceinline__ void dmma_cq(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Cholesky G = R.T R and R^-1 for b <= 32 by a whole CTA (>= 32 warps'
// worth of work is not needed; what matters is the dependent chain):
//  * factorisation: ONE barrier per column -- every thread reads the pivot
//    and forms 1/R_jj itself, the trailing update uses the unscaled row j
//    (G_c1c2 -= G_jc1 G_jc2 / G_jj) while row j is scaled in place;
//  * inverse: columns of R^-1 are independent -- warp w solves column c = w
//    (, w + nwarps) with lane t holding x_t and a warp sum per row: no
//    barriers at all.
// Same flag rule as chol_inv_smem.  G: upper triangle in, destroyed.
__device__ void chol_inv_cta(int b, double (*G)[65], double* dinv, double* __restrict__ Rinv,
                             uint32_t* __restrict__ flag, uint32_t* __restrict__ zero_flag = nullptr) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
  bool bad = false;
  double dmax = 0.0, dmin = 1e300;
  for (int j = 0; j < b; ++j) {
    const double d = G[j][j];
    const double dd = d > 0.0 ? d : 1.0;
    const double inv = rsqrt(dd), rjj = dd * inv, invd = inv * inv;  // one MUFU-seeded op on the chain
    bad |= !(d > 0.0);
    dmax = fmax(dmax, rjj);
    dmin = fmin(dmin, rjj);
    // trailing update from the unscaled row j: 2-D thread map (c2 = t % 32,
    // c1 = t / 32 + 16 k), no divisions
    for (int t = tid; t < 32 * 32; t += nth) {
      const int c1 = t >> 5, c2 = t & 31;
      if (c1 > j && c2 >= c1 && c2 < b) G[c1][c2] = fma(-G[j][c1] * invd, G[j][c2], G[c1][c2]);
    }
    __syncthreads();  // the update has read row j (unscaled)
    if (tid < 32) {
      const int c = tid;
      if (c == j) {
        G[j][j] = rjj;
        dinv[j] = inv;
      } else if (c > j && c < b) {
        G[j][c] *= inv;
      }
    }
    __syncthreads();
  }
  if (tid == 0 && (bad || dmin * dmin < 1e-12 * dmax * dmax)) atomicOr(flag, 1u);
  if (tid == 0 && zero_flag && bad) atomicOr(zero_flag, 1u);  // every thread saw the same pivots
  // X = R^-1, column c: x_c = 1/R_cc, x_i = -(sum_{t=i+1..c} R_it x_t) / R_ii
  for (int c = warp; c < b; c += nwarps) {
    double xl = lane == c ? dinv[c] : 0.0;  // x_lane
    for (int i = c - 1; i >= 0; --i) {
      double p = (lane > i && lane <= c) ? G[i][lane] * xl : 0.0;
      p = warp_sum(p);
      if (lane == i) xl = -p * dinv[i];
    }
    if (lane <= c) Rinv[lane * b + c] = xl;
    else if (lane < b) Rinv[lane * b + c] = 0.0;
  }
}

template <int NT>
__global__ void __launch_bounds__(kCqrThreads) k_cqr_gram(int64_t r, int b, const double* __restrict__ Y, int64_t ldy,
                                                          double* __restrict__ part, double* __restrict__ gpart,
                                                          unsigned* __restrict__ tickets, double* __restrict__ Rinv,
                                                          uint32_t* __restrict__ flag, double* __restrict__ Gout) {
  constexpr int BP = 8 * NT, E = BP * BP;  // padded width, entries per partial
  __shared__ double red[NT * NT * 2 * 32];
  __shared__ double G[64][65];
  __shared__ double dinv[64];
  __shared__ unsigned arrive;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  // 32 rows (8 k-steps of 4) per warp, all loaded at once: one DRAM round
  const int64_t ws = ((int64_t)blockIdx.x * kCqrWarps + warp) * (4 * kCqrKs);
  double y[kCqrKs][NT];
#pragma unroll
  for (int s = 0; s < kCqrKs; ++s) {
    const int64_t row = ws + 4 * s + tq;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int col = 8 * t + g;
      y[s][t] = (row < r && col < b) ? __ldcs(Y + row * ldy + col) : 0.0;
    }
  }
  double acc[NT][NT][2];
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < kCqrKs; ++s)
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
      for (int j = i; j < NT; ++j) dmma_cq(acc[i][j], y[s][i], y[s][j]);
  // warp-ordered CTA sum
  for (int w = 0; w < kCqrWarps; ++w) {
    if (warp == w) {
#pragma unroll
      for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int j = i; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double* c = red + ((i * NT + j) * 2 + e) * 32 + lane;
            *c = (w == 0 ? 0.0 : *c) + acc[i][j][e];
          }
    }
    __syncthreads();
  }
  // CTA partial (BP x BP, lower tiles zero)
  double* mine = part + (int64_t)blockIdx.x * E;
  for (int t = threadIdx.x; t < E; t += kCqrThreads) mine[t] = 0.0;
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
      for (int j = i; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) mine[(8 * i + g) * BP + 8 * j + 2 * tq + e] = red[((i * NT + j) * 2 + e) * 32 + lane];
  }
  // two-level fixed-order reduction: the last CTA of each group of
  // kCqrGroup sums the group's partials, the last group finisher sums the
  // group partials (tickets rest at 0 between calls)
  const unsigned ngroups = (gridDim.x + kCqrGroup - 1) / kCqrGroup;
  const unsigned grp = blockIdx.x / kCqrGroup;
  const unsigned g0 = grp * kCqrGroup, gn = min(gridDim.x, g0 + kCqrGroup) - g0;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) arrive = atomicAdd(tickets + 1 + grp, 1u);
  __syncthreads();
  if (arrive != gn - 1) return;
  __threadfence();
  for (int t = threadIdx.x; t < E; t += kCqrThreads) {
    double x[kCqrGroup];  // all loads in flight, then the fixed-order sum
#pragma unroll
    for (int c = 0; c < kCqrGroup; ++c) x[c] = c < (int)gn ? __ldcg(part + (int64_t)(g0 + c) * E + t) : 0.0;
    double v = 0.0;
#pragma unroll
    for (int c = 0; c < kCqrGroup; ++c) v += x[c];
    gpart[(int64_t)grp * E + t] = v;
  }
  if (threadIdx.x == 0) tickets[1 + grp] = 0u;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) arrive = atomicAdd(tickets, 1u);
  __syncthreads();
  if (arrive != ngroups - 1) return;
  __threadfence();
  for (int t = threadIdx.x; t < E; t += kCqrThreads) {
    const int m = t / BP, n = t - m * BP;
    double v = 0.0;
    for (unsigned c0 = 0; c0 < ngroups; c0 += kCqrGroup) {
      double x[kCqrGroup];
#pragma unroll
      for (int c = 0; c < kCqrGroup; ++c) x[c] = c0 + c < ngroups ? __ldcg(gpart + (int64_t)(c0 + c) * E + t) : 0.0;
#pragma unroll
      for (int c = 0; c < kCqrGroup; ++c) v += x[c];
    }
    if (m < b && n < b) G[m][n] = v;
  }
  if (threadIdx.x == 0) tickets[0] = 0u;
  __syncthreads();
  if (Gout) {  // Gram only (row-sharded CholeskyQR: the caller all-reduces it)
    for (int t = threadIdx.x; t < b * b; t += kCqrThreads) {
      const int i = t / b, j = t - i * b;
      Gout[t] = i <= j ? G[i][j] : G[j][i];
    }
    return;
  }
  chol_inv_cta(b, G, dinv, Rinv, flag);
}

template <int NT>
__global__ void __launch_bounds__(256) k_cqr_apply(int64_t r, int b, const double* __restrict__ Y, int64_t ldy,
                                                   const double* __restrict__ Rinv, double* __restrict__ out,
                                                   int64_t ldo, const uint32_t* __restrict__ flag, int only_if_clear) {
  constexpr int BP = 8 * NT, NK = 2 * NT, MT = 2;  // k-steps of 4 over the padded width; 16-row tiles
  __shared__ double Rs[BP][BP + 1];
  if (only_if_clear && *flag) return;
  const bool vec2 = (ldo % 2 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  for (int t = threadIdx.x; t < BP * BP; t += blockDim.x) {
    const int i = t / BP, j = t % BP;
    Rs[i][j] = (i < b && j < b) ? Rinv[i * b + j] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ntiles = (r + 8 * MT - 1) / (8 * MT);
  auto ld = [&](int64_t tile, double (&a)[NK][MT]) {
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int64_t row = tile * (8 * MT) + 8 * i + g;
#pragma unroll
      for (int s = 0; s < NK; ++s) {
        const int col = 4 * s + tq;
        a[s][i] = (tile < ntiles && row < r && col < b) ? __ldcs(Y + row * ldy + col) : 0.0;
      }
    }
  };
  int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double a[NK][MT];
  ld(tile, a);
  for (; tile < ntiles; tile += nw) {
    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int s = 0; s < NK; ++s) {
      double bf[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = Rs[4 * s + tq][8 * j + g];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma_cq(acc[i][j], a[s][i], bf[j]);
    }
    ld(tile + nw, a);
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int64_t row = tile * (8 * MT) + 8 * i + g;
      if (row < r) {
        double* o = out + row * ldo;
        // a lane's two fragment columns are adjacent: one 16-B store
        // (whole sectors; 8-B stores left half-written sectors that cost
        // ~10x the output bytes in DRAM writes)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int col = 8 * j + 2 * tq;
          if (vec2 && col + 1 < b) {
            *reinterpret_cast<double2*>(o + col) = make_double2(acc[i][j][0], acc[i][j][1]);
            continue;
          }
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (col + e < b) o[col + e] = acc[i][j][e];
          }
      }
    }
  }
}

struct OrthLayout {
  size_t off_flag, off_rinv, off_red, off_part, off_tmp, off_tsqr, off_cqr, off_tickets, off_g, off_gemm, off_tmp2,
      gemm_bytes, total;
  int nparts;
  int64_t rows_per;
};

int64_t cqr_ctas(int64_t r) { return (r + kCqrWarps * 4 * kCqrKs - 1) / (kCqrWarps * 4 * kCqrKs); }

OrthLayout orth_layout(int64_t r, int b) {
  OrthLayout L{};
  L.nparts = 2 * sm_count();
  L.rows_per = (r + L.nparts - 1) / L.nparts;
  if (L.rows_per < kGramRows) {
    L.rows_per = kGramRows;
    L.nparts = (int)((r + kGramRows - 1) / kGramRows);
  }
  size_t o = 0;
  L.off_flag = o;  // flag words (4), then the DMMA path's reduction tickets
  L.off_tickets = o + 16;
  o = align_up(o + 16 + (size_t)(2 + (cqr_ctas(r) + kCqrGroup - 1) / kCqrGroup) * 4);
  L.off_red = o;
  o = align_up(o + (size_t)b * (b + 1) / 2 * 8);
  L.off_rinv = o;
  o = align_up(o + (size_t)b * b * 8);
  L.off_part = o;
  o = align_up(o + (size_t)L.nparts * (b * (b + 1) / 2) * 8);
  L.off_tmp = o;
  o = align_up(o + (size_t)r * b * 8);
  L.off_tsqr = o;
  o = align_up(o + make_plan(r, b).total);
  L.off_cqr = o;  // DMMA path: CTA partials + group partials (BP x BP each, BP <= 32) + tickets
  o = align_up(o + (size_t)(cqr_ctas(r) + (cqr_ctas(r) + kCqrGroup - 1) / kCqrGroup) * 32 * 32 * 8);
  if (b > 32) {  // wide blocks: Gram / apply on the DMMA GEMMs, second pass into tmp2
    L.off_g = o;
    o = align_up(o + (size_t)b * b * 8);
    L.gemm_bytes = svdrec_gemm_tn_workspace_bytes(r, b, b);
    L.off_gemm = o;
    o = align_up(o + L.gemm_bytes);
    L.off_tmp2 = o;
    o = align_up(o + (size_t)r * b * 8);
  }
  L.total = o;
  return L;
}

template <int NT>
int cqr_pass_nt(int64_t r, int b, const double* Y, int64_t ldy, double* out, int64_t ldo, const OrthLayout& L,
                char* w, int only_if_clear, cudaStream_t s) {
  double* rinv = reinterpret_cast<double*>(w + L.off_rinv);
  uint32_t* flag = reinterpret_cast<uint32_t*>(w + L.off_flag);
  const int64_t nc = cqr_ctas(r);
  double* part = reinterpret_cast<double*>(w + L.off_cqr);
  double* gpart = part + nc * (8 * NT) * (8 * NT);
  unsigned* tickets = reinterpret_cast<unsigned*>(w + L.off_tickets);
  k_cqr_gram<NT><<<(unsigned)nc, kCqrThreads, 0, s>>>(r, b, Y, ldy, part, gpart, tickets, rinv, flag, nullptr);
  const int64_t tiles = (r + 15) / 16;
  int64_t grid = (tiles + 7) / 8;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (grid > cap) grid = cap;
  k_cqr_apply<NT><<<(unsigned)grid, 256, 0, s>>>(r, b, Y, ldy, rinv, out, ldo, flag, only_if_clear);
  return check_launch("cqr_pass", 2);
}

int cqr_pass(int64_t r, int b, const double* Y, int64_t ldy, double* out, int64_t ldo, const OrthLayout& L, char* w,
             int only_if_clear, cudaStream_t s) {
  switch ((b + 7) / 8) {
    case 1: return cqr_pass_nt<1>(r, b, Y, ldy, out, ldo, L, w, only_if_clear, s);
    case 2: return cqr_pass_nt<2>(r, b, Y, ldy, out, ldo, L, w, only_if_clear, s);
    case 3: return cqr_pass_nt<3>(r, b, Y, ldy, out, ldo, L, w, only_if_clear, s);
    default: return cqr_pass_nt<4>(r, b, Y, ldy, out, ldo, L, w, only_if_clear, s);
  }
}



// ---- Row-sharded CholeskyQR building blocks --------------------------------
// A rank holding rows [r0, r1) of a tall block Y computes its Gram partial
// (svdrec_gram), the caller all-reduces the b x b partials, and every rank
// factors the same G and applies R^-1 to its own rows (svdrec_chol_apply).

// R = chol(G + shift_rel * trace(G) * I) (upper), Rinv = R^-1; one CTA.
// flag |= 1 as in the CholeskyQR2 path (kappa > 1e6 or a bad pivot);
// zero_flag |= 1 on a non-positive pivot (the caller's status word).
__global__ void __launch_bounds__(kCqrThreads) k_chol_full(int b, const double* __restrict__ G, int64_t ldg,
                                                           double shift_rel, double* __restrict__ Rinv,
                                                           uint32_t* __restrict__ flag,
                                                           uint32_t* __restrict__ zero_flag) {
  __shared__ double Gs[64][65];
  __shared__ double dinv[64];
  __shared__ int bad;
  __shared__ double shift;
  if (threadIdx.x < 32) {
    double t = 0.0;
    for (int i = threadIdx.x; i < b; i += 32) t += G[i * ldg + i];
    t = warp_sum(t);
    if (threadIdx.x == 0) shift = shift_rel * t;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < b * b; t += blockDim.x) {
    const int i = t / b, j = t - i * b;
    if (i <= j) Gs[i][j] = G[i * ldg + j] + (i == j ? shift : 0.0);
  }
  __syncthreads();
  if (b <= 32)
    chol_inv_cta(b, Gs, dinv, Rinv, flag, zero_flag);
  else
    chol_inv_smem(b, Gs, dinv, &bad, Rinv, flag, zero_flag);
}

// One CholeskyQR pass for 32 < b <= 64 on the DMMA GEMMs (TMA-staged
// tall-skinny kernels of skinny.cu): G = Y.T Y, R = chol(G + shift tr(G) I),
// out = Y R^-1.  out must not alias Y.
int cholqr_pass_wide(int64_t r, int b, const double* Y, int64_t ldy, double* out, int64_t ldo, double* G,
                     void* gw, size_t gwb, double* rinv, uint32_t* flag, uint32_t* zero_flag, double shift_rel,
                     cudaStream_t s) {
  int rc = svdrec_gemm_tn(r, b, b, 1.0, Y, ldy, Y, ldy, 0.0, G, b, gw, gwb, s);
  if (rc) return rc;
  k_chol_full<<<1, kCqrThreads, 0, s>>>(b, G, b, shift_rel, rinv, flag, zero_flag);
  rc = check_launch("cholqr_wide");
  if (rc) return rc;
  return svdrec_gemm_nn(r, b, b, 1.0, Y, ldy, rinv, b, 0.0, out, ldo, s);
}

// dst = src (r x b) unless the flag is set (the TSQR fallback owns dst then)
__global__ void k_gated_copy(int64_t r, int b, const double* __restrict__ src, int64_t lds, double* __restrict__ dst,
                             int64_t ldd, const uint32_t* __restrict__ flag) {
  if (*flag) return;
  const int64_t n = r * b;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / b;
    const int j = (int)(t - i * b);
    dst[i * ldd + j] = src[i * lds + j];
  }
}

struct GramLayout {
  size_t off_tickets, off_part, off_pairs, total;
  int nparts;
  int64_t rows_per;
};

GramLayout gram_layout(int64_t r, int b) {
  GramLayout L{};
  size_t o = 0;
  L.off_tickets = o;
  o = align_up(o + (size_t)(2 + (cqr_ctas(r) + kCqrGroup - 1) / kCqrGroup) * 4);
  L.nparts = 2 * sm_count();
  L.rows_per = (r + L.nparts - 1) / L.nparts;
  if (L.rows_per < kGramRows) {
    L.rows_per = kGramRows;
    L.nparts = (int)((r + kGramRows - 1) / kGramRows);
  }
  L.off_part = o;
  const size_t dmma = (size_t)(cqr_ctas(r) + (cqr_ctas(r) + kCqrGroup - 1) / kCqrGroup) * 32 * 32 * 8;
  const size_t gemm = svdrec_gemm_tn_workspace_bytes(r, b, b);  // b > 32: the DMMA GEMM
  o = align_up(o + (b <= 32 ? dmma : gemm));
  L.off_pairs = o;
  o = align_up(o + (size_t)b * (b + 1) / 2 * 8);
  L.total = o;
  return L;
}

template <int NT>
void gram_nt(int64_t r, int b, const double* Y, int64_t ldy, double* G, const GramLayout& L, char* w, cudaStream_t s) {
  const int64_t nc = cqr_ctas(r);
  double* part = reinterpret_cast<double*>(w + L.off_part);
  double* gpart = part + nc * (8 * NT) * (8 * NT);
  unsigned* tickets = reinterpret_cast<unsigned*>(w + L.off_tickets);
  k_cqr_gram<NT><<<(unsigned)nc, kCqrThreads, 0, s>>>(r, b, Y, ldy, part, gpart, tickets, nullptr, nullptr, G);
}

template <int NT>
void cqr_apply_launch(int64_t r, int b, const double* Y, int64_t ldy, const double* rinv, double* out, int64_t ldo,
                      const uint32_t* flag, cudaStream_t s) {
  const int64_t tiles = (r + 15) / 16;
  int64_t grid = (tiles + 7) / 8;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (grid > cap) grid = cap;
  k_cqr_apply<NT><<<(unsigned)grid, 256, 0, s>>>(r, b, Y, ldy, rinv, out, ldo, flag, 0);
}

}  // namespace
}  // namespace svdrec

extern "C" int svdrec_tsqr(int64_t r, int32_t b, const double* d_A, int64_t lda, double* d_Q, int64_t ldq,
                           double* d_R, void* d_work, size_t work_bytes, void* stream) {
  SVDREC_ARG(b >= 1 && b <= 80, "tsqr: block width %d outside [1, 80]", b);
  SVDREC_ARG(r >= b, "tsqr: needs rows >= cols (%lld < %d)", (long long)r, b);
  SVDREC_ARG(lda >= b && ldq >= b, "tsqr: bad leading dimension");
  const Plan p = make_plan(r, b);
  if (work_bytes < p.total) {
    set_error("tsqr: workspace %zu < %zu", work_bytes, p.total);
    return SVDREC_E_WORKSPACE;
  }
  return run_tsqr(p, r, b, d_A, lda, d_Q, ldq, d_R, static_cast<char*>(d_work), nullptr, as_stream(stream));
}

extern "C" size_t svdrec_orth_workspace_bytes(int64_t r, int32_t b) {
  if (b < 1 || b > 80 || r < b) return 256;
  return orth_layout(r, b).total + 256;
}

extern "C" int svdrec_orth(int64_t r, int32_t b, const double* d_A, int64_t lda, double* d_Q, int64_t ldq,
                           void* d_work, size_t work_bytes, void* stream) {
  SVDREC_ARG(b >= 1 && b <= 80, "orth: block width %d outside [1, 80]", b);
  SVDREC_ARG(r >= b, "orth: needs rows >= cols (%lld < %d)", (long long)r, b);
  SVDREC_ARG(lda >= b && ldq >= b, "orth: bad leading dimension");
  const OrthLayout L = orth_layout(r, b);
  if (work_bytes < L.total) {
    set_error("orth: workspace %zu < %zu", work_bytes, L.total);
    return SVDREC_E_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  char* w = static_cast<char*>(d_work);
  uint32_t* flag = reinterpret_cast<uint32_t*>(w + L.off_flag);
  double* tmp = reinterpret_cast<double*>(w + L.off_tmp);
  if (b > 64)  // CholeskyQR2 tiles hold b <= 64: Householder directly
    return run_tsqr(make_plan(r, b), r, b, d_A, lda, d_Q, ldq, reinterpret_cast<double*>(w + L.off_rinv),
                    w + L.off_tsqr, nullptr, s);
  // flag and tickets (the scratch workspace is shared with other calls)
  SVDREC_CUDA(cudaMemsetAsync(flag, 0, L.off_tickets - L.off_flag + (2 + (cqr_ctas(r) + kCqrGroup - 1) / kCqrGroup) * 4,
                              s));
  int rc;
  if (b <= 32) {  // DMMA passes
    rc = cqr_pass(r, b, d_A, lda, tmp, b, L, w, 0, s);  // Q1 = A R1^-1
    if (rc) return rc;
    rc = cqr_pass(r, b, tmp, b, d_Q, ldq, L, w, 1, s);  // Q = Q1 R2^-1 (if both passes are sound)
  } else {  // 32 < b <= 64: DMMA GEMM passes; pass 2 into tmp2, copied to Q unless flagged
    double* G = reinterpret_cast<double*>(w + L.off_g);
    double* rinv = reinterpret_cast<double*>(w + L.off_rinv);
    double* tmp2 = reinterpret_cast<double*>(w + L.off_tmp2);
    rc = cholqr_pass_wide(r, b, d_A, lda, tmp, b, G, w + L.off_gemm, L.gemm_bytes, rinv, flag, nullptr, 0.0, s);
    if (rc) return rc;
    rc = cholqr_pass_wide(r, b, tmp, b, tmp2, b, G, w + L.off_gemm, L.gemm_bytes, rinv, flag, nullptr, 0.0, s);
    if (rc) return rc;
    const int64_t n = r * b;
    int64_t grid = (n + 255) / 256;
    if (grid > (int64_t)sm_count() * 16) grid = (int64_t)sm_count() * 16;
    k_gated_copy<<<(unsigned)grid, 256, 0, s>>>(r, b, tmp2, b, d_Q, ldq, flag);
    rc = check_launch("orth_copy");
  }
  if (rc) return rc;
  // fallback: Householder TSQR from the untouched input, only if flagged
  double* dummy_r = reinterpret_cast<double*>(w + L.off_rinv);
  return run_tsqr_gated(make_plan(r, b), r, b, d_A, lda, d_Q, ldq, dummy_r, w + L.off_tsqr, flag, s);
}

extern "C" size_t svdrec_gram_workspace_bytes(int64_t r, int32_t b) {
  if (b < 1 || b > 64 || r < 0) return 256;
  return svdrec::gram_layout(r, b).total + 256;
}

extern "C" int svdrec_gram(int64_t r, int32_t b, const double* d_Y, int64_t ldy, double* d_G, void* d_work,
                           size_t work_bytes, void* stream) {
  using namespace svdrec;
  SVDREC_ARG(b >= 1 && b <= 64, "gram: block width %d outside [1, 64]", b);
  SVDREC_ARG(r >= 0 && (r == 0 || ldy >= b), "gram: bad shape or leading dimension");
  cudaStream_t s = as_stream(stream);
  if (r == 0) {
    SVDREC_CUDA(cudaMemsetAsync(d_G, 0, (size_t)b * b * 8, s));
    return 0;
  }
  const GramLayout L = gram_layout(r, b);
  if (work_bytes < L.total) {
    set_error("gram: workspace %zu < %zu", work_bytes, L.total);
    return SVDREC_E_WORKSPACE;
  }
  char* w = static_cast<char*>(d_work);
  if (b <= 32) {
    SVDREC_CUDA(cudaMemsetAsync(w + L.off_tickets, 0, (size_t)(2 + (cqr_ctas(r) + kCqrGroup - 1) / kCqrGroup) * 4, s));
    switch ((b + 7) / 8) {
      case 1: gram_nt<1>(r, b, d_Y, ldy, d_G, L, w, s); break;
      case 2: gram_nt<2>(r, b, d_Y, ldy, d_G, L, w, s); break;
      case 3: gram_nt<3>(r, b, d_Y, ldy, d_G, L, w, s); break;
      default: gram_nt<4>(r, b, d_Y, ldy, d_G, L, w, s); break;
    }
    return check_launch("gram", 1);
  }
  return svdrec_gemm_tn(r, b, b, 1.0, d_Y, ldy, d_Y, ldy, 0.0, d_G, b, w + L.off_part,
                        L.off_pairs - L.off_part, s);
}

extern "C" size_t svdrec_chol_apply_workspace_bytes(int64_t r, int32_t b) {
  if (b < 1 || b > 64 || r < 0) return 256;
  // b > 32: the apply is a DMMA GEMM, through a temporary when Q aliases Y
  return svdrec::align_up(16) + svdrec::align_up((size_t)b * b * 8) +
         (b > 32 ? svdrec::align_up((size_t)r * b * 8) : 0) + 256;
}

extern "C" int svdrec_chol_apply(int64_t r, int32_t b, const double* d_G, int64_t ldg, double shift_rel,
                                 const double* d_Y, int64_t ldy, double* d_Q, int64_t ldq, uint32_t* d_status,
                                 void* d_work, size_t work_bytes, void* stream) {
  using namespace svdrec;
  SVDREC_ARG(b >= 1 && b <= 64, "chol_apply: block width %d outside [1, 64]", b);
  SVDREC_ARG(r >= 0 && ldg >= b && (r == 0 || (ldy >= b && ldq >= b)), "chol_apply: bad shape or leading dimension");
  SVDREC_ARG(shift_rel >= 0.0, "chol_apply: negative shift");
  const size_t need = align_up(16) + align_up((size_t)b * b * 8) + (b > 32 ? align_up((size_t)r * b * 8) : 0);
  if (work_bytes < need) {
    set_error("chol_apply: workspace %zu < %zu", work_bytes, need);
    return SVDREC_E_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  char* w = static_cast<char*>(d_work);
  uint32_t* flag = reinterpret_cast<uint32_t*>(w);
  double* rinv = reinterpret_cast<double*>(w + align_up(16));
  SVDREC_CUDA(cudaMemsetAsync(flag, 0, 16, s));
  k_chol_full<<<1, kCqrThreads, 0, s>>>(b, d_G, ldg, shift_rel, rinv, flag, d_status);
  if (r == 0) return check_launch("chol_apply", 1);
  switch ((b + 7) / 8) {
    case 1: cqr_apply_launch<1>(r, b, d_Y, ldy, rinv, d_Q, ldq, flag, s); break;
    case 2: cqr_apply_launch<2>(r, b, d_Y, ldy, rinv, d_Q, ldq, flag, s); break;
    case 3: cqr_apply_launch<3>(r, b, d_Y, ldy, rinv, d_Q, ldq, flag, s); break;
    case 4: cqr_apply_launch<4>(r, b, d_Y, ldy, rinv, d_Q, ldq, flag, s); break;
    default: {
      const bool alias = d_Q == d_Y;
      double* dst = alias ? reinterpret_cast<double*>(w + align_up(16) + align_up((size_t)b * b * 8)) : d_Q;
      const int64_t ldd = alias ? b : ldq;
      int rc = svdrec_gemm_nn(r, b, b, 1.0, d_Y, ldy, rinv, b, 0.0, dst, ldd, s);
      if (rc) return rc;
      if (alias) SVDREC_CUDA(cudaMemcpy2DAsync(d_Q, ldq * 8, dst, ldd * 8, (size_t)b * 8, r, cudaMemcpyDeviceToDevice, s));
      return check_launch("chol_apply", 1);
    }
  }
  return check_launch("chol_apply", 2);
}
