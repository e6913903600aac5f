// Tall-skinny LU with partial pivoting -> P.L (lu_lower_basis).
//
// Replaces scipy.linalg.lu(M, permute_l=True) in lu_lower_basis (reference
// pkg/src/svdrec/linalg.py:84-97), the cheap range finder of Alg. 3
// (rsvd.py:180, 190).  Right-looking partial pivoting, exactly as LAPACK
// dgetf2 picks pivots (largest |value| among not-yet-pivoted rows; ties ->
// lowest row index), but rows are never swapped: the result is already in
// the original row order that permute_l=True returns.  One cooperative
// kernel: per column, each CTA reduces its rows' pivot candidate, one grid
// barrier publishes all candidates, every CTA picks the same winner and
// eliminates its own rows against the pivot row.  b grid barriers total.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace svdrec {
namespace {

constexpr int kLuThreads = 256;

struct Cand {
  double a;
  long long row;
};

__device__ __forceinline__ bool better(double a, long long ra, double b, long long rb) {
  return a > b || (a == b && ra < rb);
}

__global__ void __launch_bounds__(kLuThreads) k_lu(int64_t r, int b, double* __restrict__ A, int64_t lda,
                                                   double* __restrict__ udiag, int32_t* __restrict__ pivstep,
                                                   Cand* __restrict__ slots, uint32_t* d_status) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sa[kLuThreads / 32];
  __shared__ long long sr[kLuThreads / 32];
  __shared__ long long piv_row;
  __shared__ double piv_val;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  const int nblk = gridDim.x;
  for (int64_t i = gt; i < r; i += gs) pivstep[i] = -1;
  for (int j = 0; j < b; ++j) {
    // local candidate
    double best = -1.0;
    long long brow = -1;
    for (int64_t i = gt; i < r; i += gs) {
      if (pivstep[i] >= 0) continue;
      const double v = fabs(A[i * lda + j]);
      if (better(v, i, best, brow) || brow < 0) {
        best = v;
        brow = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const long long orow = __shfl_xor_sync(0xffffffffu, brow, o);
      if (orow >= 0 && (brow < 0 || better(ob, orow, best, brow))) {
        best = ob;
        brow = orow;
      }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
      sa[warp] = best;
      sr[warp] = brow;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bb = -1.0;
      long long br = -1;
      for (int w = 0; w < kLuThreads / 32; ++w)
        if (sr[w] >= 0 && (br < 0 || better(sa[w], sr[w], bb, br))) {
          bb = sa[w];
          br = sr[w];
        }
      slots[(size_t)(j & 1) * nblk + blockIdx.x] = Cand{bb, br};
    }
    grid.sync();
    {
      // every block reduces all candidates in parallel (same fixed result)
      double bb = -1.0;
      long long br = -1;
      const Cand* sl = slots + (size_t)(j & 1) * nblk;
      for (int k = threadIdx.x; k < nblk; k += blockDim.x) {
        const Cand cc = sl[k];
        if (cc.row >= 0 && (br < 0 || better(cc.a, cc.row, bb, br))) {
          bb = cc.a;
          br = cc.row;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, bb, o);
        const long long orow = __shfl_xor_sync(0xffffffffu, br, o);
        if (orow >= 0 && (br < 0 || better(ob, orow, bb, br))) {
          bb = ob;
          br = orow;
        }
      }
      if (lane == 0) {
        sa[warp] = bb;
        sr[warp] = br;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double b2 = -1.0;
        long long r2 = -1;
        for (int w = 0; w < kLuThreads / 32; ++w)
          if (sr[w] >= 0 && (r2 < 0 || better(sa[w], sr[w], b2, r2))) {
            b2 = sa[w];
            r2 = sr[w];
          }
        piv_row = r2;
        piv_val = r2 >= 0 ? A[r2 * lda + j] : 0.0;
      }
    }
    __syncthreads();
    const long long p = piv_row;
    const double pv = piv_val;
    if (gt == 0) {
      udiag[j] = pv;
      if (pv == 0.0 && d_status) atomicOr(d_status, SVDREC_STATUS_ZERO_PIVOT);
    }
    for (int64_t i = gt; i < r; i += gs) {
      if (i == p) {
        pivstep[i] = j;
        continue;
      }
      if (pivstep[i] >= 0 || pv == 0.0) continue;
      double* row = A + i * lda;
      const double l = row[j] / pv;
      row[j] = l;
      const double* prow = A + p * lda;
      for (int c = j + 1; c < b; ++c) row[c] = fma(-l, prow[c], row[c]);
    }
    // make this step's row updates (and the pivot row) visible before the
    // next step's candidate scan reads them from other CTAs' rows
    __threadfence();
  }
  grid.sync();
  for (int64_t i = gt; i < r; i += gs) {
    const int s = pivstep[i];
    if (s < 0) continue;
    double* row = A + i * lda;
    row[s] = 1.0;
    for (int c = s + 1; c < b; ++c) row[c] = 0.0;
  }
}

// Panel-resident variant: CTA c owns rows [c*rpc, (c+1)*rpc) and keeps them
// in shared memory for all b steps.  Each step every CTA publishes its best
// candidate together with that row's current values, so after the single
// grid barrier every CTA has the winning pivot row without another pass.
// cand layout per (parity, block): [|value|, row, values[0..b)].
__global__ void __launch_bounds__(kLuThreads) k_lu_smem(int64_t r, int b, double* __restrict__ A, int64_t lda,
                                                        double* __restrict__ udiag, int64_t rpc,
                                                        double* __restrict__ cand, uint32_t* d_status) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double P[];
  __shared__ double sa[kLuThreads / 32];
  __shared__ long long sr[kLuThreads / 32];
  __shared__ double prow[128];
  __shared__ long long piv_row;
  __shared__ double piv_val;
  __shared__ int piv_blk;
  const int ldp = b | 1;
  const int64_t r0 = (int64_t)blockIdx.x * rpc;
  const int nl = (int)(r0 < r ? min64(rpc, r - r0) : 0);
  int* pstep = reinterpret_cast<int*>(P + (size_t)rpc * ldp);
  const int nblk = gridDim.x;
  const int stride = b + 2;
  for (int t = threadIdx.x; t < nl * b; t += kLuThreads) {
    const int i = t / b, c = t - i * b;
    P[i * ldp + c] = A[(r0 + i) * lda + c];
  }
  for (int i = threadIdx.x; i < nl; i += kLuThreads) pstep[i] = -1;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = 0; j < b; ++j) {
    double best = -1.0;
    long long brow = -1;
    for (int i = threadIdx.x; i < nl; i += kLuThreads) {
      if (pstep[i] >= 0) continue;
      const double v = fabs(P[i * ldp + j]);
      if (brow < 0 || better(v, r0 + i, best, brow)) {
        best = v;
        brow = r0 + i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const long long orow = __shfl_xor_sync(0xffffffffu, brow, o);
      if (orow >= 0 && (brow < 0 || better(ob, orow, best, brow))) {
        best = ob;
        brow = orow;
      }
    }
    if (lane == 0) {
      sa[warp] = best;
      sr[warp] = brow;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bb = -1.0;
      long long br = -1;
      for (int w = 0; w < kLuThreads / 32; ++w)
        if (sr[w] >= 0 && (br < 0 || better(sa[w], sr[w], bb, br))) {
          bb = sa[w];
          br = sr[w];
        }
      piv_row = br;
    }
    __syncthreads();
    double* my = cand + ((size_t)(j & 1) * nblk + blockIdx.x) * stride;
    const long long lb = piv_row;
    if (threadIdx.x == 0) {
      my[0] = lb >= 0 ? fabs(P[(lb - r0) * ldp + j]) : -1.0;
      my[1] = (double)lb;
    }
    for (int c = threadIdx.x; c < b; c += kLuThreads) my[2 + c] = lb >= 0 ? P[(lb - r0) * ldp + c] : 0.0;
    grid.sync();
    {
      double bb = -1.0;
      long long br = -1;
      int bk = -1;
      const double* base = cand + (size_t)(j & 1) * nblk * stride;
      for (int k = threadIdx.x; k < nblk; k += kLuThreads) {
        const double a = base[(size_t)k * stride];
        const long long rw = (long long)base[(size_t)k * stride + 1];
        if (rw >= 0 && (br < 0 || better(a, rw, bb, br))) {
          bb = a;
          br = rw;
          bk = k;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, bb, o);
        const long long orow = __shfl_xor_sync(0xffffffffu, br, o);
        const int okk = __shfl_xor_sync(0xffffffffu, bk, o);
        if (orow >= 0 && (br < 0 || better(ob, orow, bb, br))) {
          bb = ob;
          br = orow;
          bk = okk;
        }
      }
      __syncthreads();
      if (lane == 0) {
        sa[warp] = bb;
        sr[warp] = br;
        reinterpret_cast<int*>(prow)[warp] = bk;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double b2 = -1.0;
        long long r2 = -1;
        int k2 = -1;
        for (int w = 0; w < kLuThreads / 32; ++w)
          if (sr[w] >= 0 && (r2 < 0 || better(sa[w], sr[w], b2, r2))) {
            b2 = sa[w];
            r2 = sr[w];
            k2 = reinterpret_cast<int*>(prow)[w];
          }
        piv_row = r2;
        piv_blk = k2;
      }
      __syncthreads();
      const double* win = base + (size_t)piv_blk * stride + 2;
      for (int c = threadIdx.x; c < b; c += kLuThreads) prow[c] = win[c];
      __syncthreads();
      if (threadIdx.x == 0) piv_val = prow[j];
      __syncthreads();
    }
    const long long p = piv_row;
    const double pv = piv_val;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      udiag[j] = pv;
      if (pv == 0.0 && d_status) atomicOr(d_status, SVDREC_STATUS_ZERO_PIVOT);
    }
    for (int i = threadIdx.x; i < nl; i += kLuThreads) {
      if (r0 + i == p) {
        pstep[i] = j;
        continue;
      }
      if (pstep[i] >= 0 || pv == 0.0) continue;
      double* row = P + i * ldp;
      const double l = row[j] / pv;
      row[j] = l;
      for (int c = j + 1; c < b; ++c) row[c] = fma(-l, prow[c], row[c]);
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < nl * b; t += kLuThreads) {
    const int i = t / b, c = t - i * b;
    const int s = pstep[i];
    double v = P[i * ldp + c];
    if (s >= 0 && c >= s) v = (c == s) ? 1.0 : 0.0;
    A[(r0 + i) * lda + c] = v;
  }
}

constexpr size_t kLuSmemMax = 100 * 1024;

}  // namespace
}  // namespace svdrec

using namespace svdrec;

extern "C" size_t svdrec_lu_workspace_bytes(int64_t r, int32_t b) {
  return align_up((size_t)r * 4) + align_up(2 * sizeof(Cand) * (size_t)sm_count() * 8) +
         align_up(2 * (size_t)sm_count() * 8 * (size_t)(b + 2) * 8) + 256;
}

namespace {
// Panel-resident LU if each of (2 per SM) CTAs can hold its rows on-chip.
int try_lu_smem(int64_t r, int32_t b, double* d_A, int64_t lda, double* d_udiag, char* w, uint32_t* d_status,
                cudaStream_t s, bool* used) {
  *used = false;
  if (b > 128) return 0;
  const int nblk = 2 * sm_count();
  const int64_t rpc = (r + nblk - 1) / nblk;
  const size_t smem = (size_t)rpc * (b | 1) * 8 + (size_t)rpc * 4 + 64;
  if (smem > kLuSmemMax) return 0;
  SVDREC_CUDA(smem_attr_once(k_lu_smem, (int)kLuSmemMax));
  int per_sm = 0;
  SVDREC_CUDA(blocks_per_sm(k_lu_smem, kLuThreads, smem, &per_sm));
  if (per_sm < 2) return 0;
  double* cand = reinterpret_cast<double*>(w + align_up((size_t)r * 4) + align_up(2 * sizeof(Cand) * (size_t)sm_count() * 8));
  int32_t bb = b;
  int64_t rr = r, rp = rpc;
  void* args[] = {&rr, &bb, &d_A, &lda, &d_udiag, &rp, &cand, &d_status};
  SVDREC_CUDA(cudaLaunchCooperativeKernel((void*)k_lu_smem, dim3(nblk), dim3(kLuThreads), args, smem, s));
  note_launches(1);
  *used = true;
  return 0;
}
}  // namespace

extern "C" int svdrec_lu_fast_path(int64_t r, int32_t b) {
  if (b < 1 || b > 128 || r < b) return 0;
  const int nblk = 2 * sm_count();
  const int64_t rpc = (r + nblk - 1) / nblk;
  return (size_t)rpc * (b | 1) * 8 + (size_t)rpc * 4 + 64 <= kLuSmemMax ? 1 : 0;
}

extern "C" int svdrec_lu_lower(int64_t r, int32_t b, double* d_A, int64_t lda, double* d_udiag, void* d_work,
                               size_t work_bytes, uint32_t* d_status, void* stream) {
  SVDREC_ARG(b >= 1 && r >= b && lda >= b, "lu_lower: needs rows >= cols >= 1");
  if (work_bytes < svdrec_lu_workspace_bytes(r, b)) {
    set_error("lu_lower: workspace too small");
    return SVDREC_E_WORKSPACE;
  }
  bool used = false;
  int rc = try_lu_smem(r, b, d_A, lda, d_udiag, static_cast<char*>(d_work), d_status, as_stream(stream), &used);
  if (rc || used) return rc;
  int per_sm = 0;
  SVDREC_CUDA(blocks_per_sm(k_lu, kLuThreads, 0, &per_sm));
  int max_blocks = per_sm * sm_count();
  // grid barrier cost grows with the block count: 2 CTAs per SM is plenty
  if (max_blocks > sm_count() * 2) max_blocks = sm_count() * 2;
  if (max_blocks < 1) max_blocks = 1;
  int64_t want = (r + kLuThreads - 1) / kLuThreads;
  int nblk = (int)(want < max_blocks ? want : max_blocks);
  if (nblk < 1) nblk = 1;
  char* w = static_cast<char*>(d_work);
  int32_t* pivstep = reinterpret_cast<int32_t*>(w);
  Cand* slots = reinterpret_cast<Cand*>(w + align_up((size_t)r * 4));
  int32_t bb = b;
  void* args[] = {&r, &bb, &d_A, &lda, &d_udiag, &pivstep, &slots, &d_status};
  SVDREC_CUDA(cudaLaunchCooperativeKernel((void*)k_lu, dim3(nblk), dim3(kLuThreads), args, 0, as_stream(stream)));
  note_launches(1);
  return 0;
}
