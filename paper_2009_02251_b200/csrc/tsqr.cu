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

#include "common.cuh"

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
__global__ void __launch_bounds__(kThreads) k_factor(int64_t rows, int64_t nc, int b, const double* __restrict__ in,
                                                     int64_t ldin, double* __restrict__ vout,
                                                     double* __restrict__ tau, double* __restrict__ rout,
                                                     const uint32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;  // CholeskyQR2 succeeded: fallback not needed
  extern __shared__ double sm[];
  __shared__ double dots[128];
  __shared__ double wv[128];
  __shared__ double coef[3];  // tau, beta, scale
  const int64_t c = blockIdx.x;
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
__global__ void __launch_bounds__(kThreads) k_buildq(int64_t rows, int64_t nc, int b, const double* __restrict__ vin,
                                                     const double* __restrict__ tau,
                                                     const double* __restrict__ qcoarse, double* __restrict__ qout,
                                                     int64_t ldq, const uint32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;
  extern __shared__ double sm[];
  __shared__ double wv[128];
  const int64_t c = blockIdx.x;
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
  static bool attr_set = false;
  const size_t smem_f = (size_t)b * ((p.rcmax + 1) | 1) * 8;
  const size_t smem_q = 2 * smem_f;
  if (!attr_set) {
    SVDREC_CUDA(cudaFuncSetAttribute(k_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kChunkBytes + 4096));
    SVDREC_CUDA(cudaFuncSetAttribute(k_buildq, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kChunkBytes + 4096));
    attr_set = true;
  }
  const int nl = (int)p.lv.size();
  const double* in = d_A;
  int64_t ldin = lda;
  for (int l = 0; l < nl; ++l) {
    const Level& L = p.lv[l];
    double* rout = (l == nl - 1) ? d_R : reinterpret_cast<double*>(w + L.off_next);
    k_factor<<<(unsigned)L.nc, kThreads, smem_f, s>>>(L.rows, L.nc, b, in, ldin,
                                                      reinterpret_cast<double*>(w + L.off_v),
                                                      reinterpret_cast<double*>(w + L.off_tau), rout, gate);
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
                                                      reinterpret_cast<double*>(w + L.off_tau), coarse, qo, ldo,
                                                      gate);
    int rc = check_launch("tsqr_buildq");
    if (rc) return rc;
    coarse = qo;
  }
  return 0;
}

// ---- CholeskyQR2 fast path -------------------------------------------------
// G = Y.T Y over a row range per CTA (upper triangle pairs), fixed-order sum.
constexpr int kGramRows = 64;
constexpr int kApplyRows = 128;

// G = Y.T Y partial per CTA row slab.  Rows are staged 64 at a time in
// shared memory; each thread owns up to 12 (i <= j) pairs whose indices are
// computed once, then accumulates over the slab.
__global__ void __launch_bounds__(256) k_gram_part(int64_t r, int b, const double* __restrict__ Y, int64_t ldy,
                                                   int64_t rows_per, double* __restrict__ part) {
  __shared__ double ys[kGramRows][65];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min64(r, r0 + rows_per);
  const int npairs = b * (b + 1) / 2;
  int pi[12], pj[12];
  double acc[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) {
    const int pidx = threadIdx.x + q * 256;
    acc[q] = 0.0;
    pi[q] = -1;
    pj[q] = 0;
    if (pidx < npairs) {
      int i = 0, off = 0;
      while (off + (b - i) <= pidx) {
        off += b - i;
        ++i;
      }
      pi[q] = i;
      pj[q] = i + (pidx - off);
    }
  }
  for (int64_t base = r0; base < r1; base += kGramRows) {
    for (int t = threadIdx.x; t < kGramRows * b; t += blockDim.x) {
      const int rr = t / b, c = t - rr * b;
      const int64_t gr = base + rr;
      ys[rr][c] = gr < r1 ? Y[gr * ldy + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 12; ++q) {
      if (pi[q] >= 0) {
        const int i = pi[q], j = pj[q];
        double a = acc[q];
#pragma unroll 8
        for (int rr = 0; rr < kGramRows; ++rr) a = fma(ys[rr][i], ys[rr][j], a);
        acc[q] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 12; ++q) {
    const int pidx = threadIdx.x + q * 256;
    if (pidx < npairs) part[(int64_t)blockIdx.x * npairs + pidx] = acc[q];
  }
}

// Fixed-order sum of the per-CTA Gram partials, one warp per pair.
__global__ void k_pairs_reduce(int npairs, int nparts, const double* __restrict__ part, double* __restrict__ out) {
  const int t = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (t >= npairs) return;
  const double s = warp_strided_sum(part + t, nparts, npairs);
  if ((threadIdx.x & 31) == 0) out[t] = s;
}

// Cholesky G = R.T R (upper R) of the reduced Gram pairs, then R^-1.
// flag |= 1 when a pivot is non-positive or (min R_jj / max R_jj)^2 < 1e-12
// (kappa(Y) > 1e6: CholeskyQR2 would not reach working-precision
// orthogonality), in which case the TSQR fallback runs.  R^-1 is built in
// the lower triangle of the same shared array (column c by thread c).
__global__ void __launch_bounds__(256) k_chol_inv(int b, const double* __restrict__ pairs, double* __restrict__ Rinv,
                                                  uint32_t* __restrict__ flag) {
  __shared__ double G[64][65];
  __shared__ double dinv[64];
  __shared__ int bad;
  const int npairs = b * (b + 1) / 2;
  if (threadIdx.x == 0) bad = 0;
  for (int pidx = threadIdx.x; pidx < npairs; pidx += blockDim.x) {
    int i = 0, off = 0;
    while (off + (b - i) <= pidx) {
      off += b - i;
      ++i;
    }
    const int j = i + (pidx - off);
    G[i][j] = pairs[pidx];
  }
  __syncthreads();
  double dmax = 0.0, dmin = 1e300;
  for (int j = 0; j < b; ++j) {
    if (threadIdx.x == 0) {
      const double d = G[j][j];
      if (!(d > 0.0)) bad = 1;
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
  if (threadIdx.x == 0 && (bad || dmin * dmin < 1e-12 * dmax * dmax)) atomicOr(flag, 1u);
  // column c of R^-1: x_c = 1/R_cc, x_i = -(sum_{t=i+1..c} R_it x_t) / R_ii,
  // stored at G[c][i] (strict lower triangle, row owned by thread c)
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

// out = Y @ Rinv (upper triangular), one thread per row over a 128-row
// tile staged (and written back) through shared memory for coalescing;
// with ``only_if_clear`` nothing is stored when the flag is set (the TSQR
// fallback owns the output then).
__global__ void __launch_bounds__(kApplyRows) k_trapply(int64_t r, int b, const double* __restrict__ Y, int64_t ldy,
                                                        const double* __restrict__ Rinv, double* __restrict__ out,
                                                        int64_t ldo, const uint32_t* __restrict__ flag,
                                                        int only_if_clear) {
  extern __shared__ double sm[];
  if (only_if_clear && *flag) return;
  const int ldp = b | 1;
  double* Ys = sm;
  double* Rs = sm + kApplyRows * ldp;
  for (int t = threadIdx.x; t < b * b; t += blockDim.x) Rs[t] = Rinv[t];
  const int64_t r0 = (int64_t)blockIdx.x * kApplyRows;
  const int nr = (int)min64(kApplyRows, r - r0);
  for (int t = threadIdx.x; t < nr * b; t += blockDim.x) {
    const int rr = t / b, c = t - rr * b;
    Ys[rr * ldp + c] = Y[(r0 + rr) * ldy + c];
  }
  __syncthreads();
  if (threadIdx.x < nr) {
    double* yr = Ys + threadIdx.x * ldp;
    for (int j = b - 1; j >= 0; --j) {  // descending: in-place overwrite is safe
      double a = 0.0;
      for (int q = 0; q <= j; ++q) a = fma(yr[q], Rs[q * b + j], a);
      yr[j] = a;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nr * b; t += blockDim.x) {
    const int rr = t / b, c = t - rr * b;
    out[(r0 + rr) * ldo + c] = Ys[rr * ldp + c];
  }
}

struct OrthLayout {
  size_t off_flag, off_rinv, off_red, off_part, off_tmp, off_tsqr, total;
  int nparts;
  int64_t rows_per;
};

OrthLayout orth_layout(int64_t r, int b) {
  OrthLayout L{};
  L.nparts = 2 * sm_count();
  L.rows_per = (r + L.nparts - 1) / L.nparts;
  if (L.rows_per < kGramRows) {
    L.rows_per = kGramRows;
    L.nparts = (int)((r + kGramRows - 1) / kGramRows);
  }
  size_t o = 0;
  L.off_flag = o;
  o = align_up(o + 16);
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
  L.total = o;
  return L;
}

int cholqr_pass(int64_t r, int b, const double* Y, int64_t ldy, double* out, int64_t ldo, const OrthLayout& L,
                char* w, int only_if_clear, cudaStream_t s) {
  double* part = reinterpret_cast<double*>(w + L.off_part);
  double* rinv = reinterpret_cast<double*>(w + L.off_rinv);
  uint32_t* flag = reinterpret_cast<uint32_t*>(w + L.off_flag);
  k_gram_part<<<(unsigned)L.nparts, 256, 0, s>>>(r, b, Y, ldy, L.rows_per, part);
  double* red = reinterpret_cast<double*>(w + L.off_red);
  const int npairs = b * (b + 1) / 2;
  k_pairs_reduce<<<(unsigned)((npairs * 32 + 255) / 256), 256, 0, s>>>(npairs, L.nparts, part, red);
  k_chol_inv<<<1, 256, 0, s>>>(b, red, rinv, flag);
  const size_t smem = ((size_t)kApplyRows * (b | 1) + (size_t)b * b) * 8;
  static bool attr = false;
  if (!attr) {
    SVDREC_CUDA(cudaFuncSetAttribute(k_trapply, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    attr = true;
  }
  k_trapply<<<(unsigned)((r + kApplyRows - 1) / kApplyRows), kApplyRows, smem, s>>>(r, b, Y, ldy, rinv, out, ldo,
                                                                                     flag, only_if_clear);
  return check_launch("cholqr_pass", 4);
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
  SVDREC_CUDA(cudaMemsetAsync(flag, 0, 16, s));
  int rc = cholqr_pass(r, b, d_A, lda, tmp, b, L, w, 0, s);  // Q1 = A R1^-1
  if (rc) return rc;
  rc = cholqr_pass(r, b, tmp, b, d_Q, ldq, L, w, 1, s);  // Q = Q1 R2^-1 (if both passes are sound)
  if (rc) return rc;
  // fallback: Householder TSQR from the untouched input, only if flagged
  double* dummy_r = reinterpret_cast<double*>(w + L.off_rinv);
  return run_tsqr(make_plan(r, b), r, b, d_A, lda, d_Q, ldq, dummy_r, w + L.off_tsqr, flag, s);
}
