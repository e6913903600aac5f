// CSR sparse x tall-skinny dense product: Y = A @ X (X row-major n x b).
//
// Replaces sparse_dense_mul (reference pkg/src/svdrec/linalg.py:141-158),
// the only route by which the reference touches the rating matrix; every
// sketch / power / projection pass of Algs. 1-3 (rsvd.py:135-143,
// 179-194) is one call.  A.T @ X is the same kernel on the CSR of A.T.
//
// HBM design: the CSR stream (int32 column + float64 value = 12 B per
// nonzero) is read once with coalesced 32-wide loads; the dense rows of X
// (b doubles, 16-B vector loads) are gathered through L1/L2 (X is small
// next to A: n*b*8 bytes).  One warp owns one row segment; its 32 lanes are
// split into NPW groups of LPN = ceil(b/VEC) lanes, so NPW nonzeros are in
// flight per step (b = 20: 3 nonzeros x 10 lanes x double2).  Column/value
// pairs are fetched 32 at a time and broadcast with shuffles.  Rows longer
// than the plan's segment cap (power-law items) are split; their partial
// sums land in a scratch slot and a fix-up kernel adds them in slot order,
// so the result is bitwise deterministic.
#include "common.cuh"

namespace svdrec {
namespace {

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
  using T = double;
};
template <>
struct VecT<2> {
  using T = double2;
};

__device__ __forceinline__ void fma_v(double& acc, double v, double x) { acc = fma(v, x, acc); }
__device__ __forceinline__ void fma_v(double2& acc, double v, double2 x) {
  acc.x = fma(v, x.x, acc.x);
  acc.y = fma(v, x.y, acc.y);
}
__device__ __forceinline__ double shfl_v(double a, int src) { return __shfl_sync(0xffffffffu, a, src); }
__device__ __forceinline__ double2 shfl_v(double2 a, int src) {
  return make_double2(__shfl_sync(0xffffffffu, a.x, src), __shfl_sync(0xffffffffu, a.y, src));
}
__device__ __forceinline__ void add_v(double& a, double b) { a += b; }
__device__ __forceinline__ void add_v(double2& a, double2 b) {
  a.x += b.x;
  a.y += b.y;
}
__device__ __forceinline__ void zero_v(double& a) { a = 0.0; }
__device__ __forceinline__ void zero_v(double2& a) { a = make_double2(0.0, 0.0); }

template <int VEC>
__global__ void __launch_bounds__(256) k_spmm(int64_t nseg, const int32_t* __restrict__ seg_row,
                                              const int64_t* __restrict__ seg_begin,
                                              const int64_t* __restrict__ seg_end,
                                              const int32_t* __restrict__ seg_slot,
                                              const int32_t* __restrict__ indices,
                                              const double* __restrict__ values, const double* __restrict__ X,
                                              int64_t ldx, double* __restrict__ Y, int64_t ldy, int b,
                                              double* __restrict__ partial, int lpn, int npw) {
  using V = typename VecT<VEC>::T;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int slot = lane / lpn;
  const int cv = lane - slot * lpn;
  const bool active = slot < npw;
  const int ctile = lpn * VEC;  // columns covered per column tile
  for (int64_t s = warp; s < nseg; s += nwarps) {
    const int64_t beg = seg_begin[s], end = seg_end[s];
    const int32_t row = seg_row[s];
    const int32_t pslot = seg_slot[s];
    for (int c0 = 0; c0 < b; c0 += ctile) {
      const int col = c0 + cv * VEC;
      const bool colok = active && col < b;
      V acc;
      zero_v(acc);
      for (int64_t base = beg; base < end; base += 32) {
        const int64_t my = base + lane;
        int32_t ci = 0;
        double vi = 0.0;
        if (my < end) {
          ci = __ldg(indices + my);
          vi = __ldg(values + my);
        }
        const int nvalid = (int)min64(32, end - base);
        // four gathers in flight per lane, then the FMAs in nonzero order
        for (int j = 0; j < nvalid; j += 4 * npw) {
          V xs[4];
          double vs[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int src = j + q * npw + slot;
            const int32_t c = __shfl_sync(0xffffffffu, ci, src & 31);
            const double v = __shfl_sync(0xffffffffu, vi, src & 31);
            const bool ok = colok && src < nvalid;
            vs[q] = ok ? v : 0.0;
            if (ok)
              xs[q] = *reinterpret_cast<const V*>(X + (int64_t)c * ldx + col);
            else
              zero_v(xs[q]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) fma_v(acc, vs[q], xs[q]);
        }
      }
      // fold the npw slot groups onto slot 0 (fixed order)
      V tot = acc;
      for (int g = 1; g < npw; ++g) {
        const V o = shfl_v(acc, (lane + g * lpn) & 31);
        if (slot == 0) add_v(tot, o);
      }
      if (slot == 0 && col < b) {
        double* dst = pslot < 0 ? (Y + (int64_t)row * ldy + col) : (partial + (int64_t)pslot * b + col);
        *reinterpret_cast<V*>(dst) = tot;
      }
    }
  }
}

__global__ void k_fixup(int64_t nlong, const int32_t* __restrict__ long_row, const int32_t* __restrict__ s0,
                        const int32_t* __restrict__ s1, const double* __restrict__ partial, double* __restrict__ Y,
                        int64_t ldy, int b) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = t / b;
  const int c = (int)(t - r * b);
  if (r >= nlong) return;
  double acc = 0.0;
  for (int32_t s = s0[r]; s < s1[r]; ++s) acc += partial[(int64_t)s * b + c];
  Y[(int64_t)long_row[r] * ldy + c] = acc;
}

}  // namespace
}  // namespace svdrec

using namespace svdrec;

extern "C" int svdrec_spmm(int64_t nseg, const int32_t* d_seg_row, const int64_t* d_seg_begin,
                           const int64_t* d_seg_end, const int32_t* d_seg_slot, const int32_t* d_indices,
                           const double* d_values, const double* d_X, int64_t ldx, double* d_Y, int64_t ldy,
                           int32_t b, int64_t nlong, const int32_t* d_long_row, const int32_t* d_long_slot0,
                           const int32_t* d_long_slot1, double* d_partial, void* stream) {
  SVDREC_ARG(b >= 1 && ldx >= b && ldy >= b && nseg >= 0 && nlong >= 0, "spmm: bad arguments b=%d", b);
  if (nseg == 0) return 0;
  cudaStream_t s = as_stream(stream);
  const bool vec2 = (b % 2 == 0) && (ldx % 2 == 0) && (ldy % 2 == 0) &&
                    ((reinterpret_cast<uintptr_t>(d_X) | reinterpret_cast<uintptr_t>(d_Y) |
                      reinterpret_cast<uintptr_t>(d_partial)) %
                         16 ==
                     0);
  const int vec = vec2 ? 2 : 1;
  const int lanes_needed = (b + vec - 1) / vec;
  const int lpn = lanes_needed >= 32 ? 32 : lanes_needed;
  const int npw = 32 / lpn;
  const int tb = 256;
  const int64_t warps = nseg;
  int64_t grid = (warps * 32 + tb - 1) / tb;
  const int64_t cap = (int64_t)sm_count() * 8 * 64;
  if (grid > cap) grid = cap;
  if (vec2)
    k_spmm<2><<<(unsigned)grid, tb, 0, s>>>(nseg, d_seg_row, d_seg_begin, d_seg_end, d_seg_slot, d_indices,
                                             d_values, d_X, ldx, d_Y, ldy, b, d_partial, lpn, npw);
  else
    k_spmm<1><<<(unsigned)grid, tb, 0, s>>>(nseg, d_seg_row, d_seg_begin, d_seg_end, d_seg_slot, d_indices,
                                             d_values, d_X, ldx, d_Y, ldy, b, d_partial, lpn, npw);
  int rc = check_launch("spmm");
  if (rc) return rc;
  if (nlong > 0) {
    const int64_t tot = nlong * b;
    k_fixup<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(nlong, d_long_row, d_long_slot0, d_long_slot1,
                                                          d_partial, d_Y, ldy, b);
    rc = check_launch("spmm_fixup");
  }
  return rc;
}
