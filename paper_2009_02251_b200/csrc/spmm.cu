// CSR sparse x tall-skinny dense product: Y = A @ X (X row-major n x b).
//
// Replaces sparse_dense_mul (reference pkg/src/svdrec/linalg.py:141-158),
// the only route by which the reference touches the rating matrix; every
// sketch / power / projection pass of Algs. 1-3 (rsvd.py:135-143,
// 179-194) is one call.  A.T @ X is the same kernel on the CSR of A.T.
//
// Kernels (which one runs is decided in svdrec_spmm / by the host,
// kernels.py):
//   k_spmm_pipe  even b <= 32 (the headline's b = 20): chunk-record pipeline,
//                CSR chunks and records through cp.async rings, X rows by
//                TMA gather4 into per-warp row rings;
//   k_spmm_tma   32 < b <= 64 (b % 4 == 0): the segment-metadata TMA pipeline;
//   k_spmm_hc    A @ X of a rating matrix at even b <= 32 where it measured
//                faster: packed hot-first CSR, the most rated items' rows of
//                X in shared memory, cold rows gathered into registers;
//   k_spmm_hot   A @ X at b = 64: the register-gather hot-set kernel;
//   k_spmm       any b / unaligned operands: one warp per row segment, 32
//                (column, value) pairs at a time broadcast by shuffles.
// Rows longer than the plan's segment cap (power-law items) are split; their
// partial sums land in a scratch slot and a fix-up kernel adds them in slot
// order, so every result is bitwise deterministic.
#include <cstdlib>

#include "tma.cuh"

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

// ---------------------------------------------------------------------------
// TMA-pipelined variant on segment metadata (round 1; now the wide blocks'
// kernel: 32 < b <= 64, V = 4 doubles per lane).  Each warp
// owns a contiguous, nonzero-balanced range of segments (host plan
// ``warp_seg``; segment metadata read 32 at a time) and streams it in chunks
// of 32 nonzeros through a ring of S = 2 shared-memory stages: while chunk c
// is accumulated, the X rows of chunk c+1 are in flight and the CSR of chunk
// c+2 is loading (evict-first, so the 216-MB CSR stream does not push X out
// of L2).  Summation order per output is the same as k_spmm: lane group g
// of G = 32/P takes nonzeros g, g+G, ... of each 32-chunk, groups folded in
// order.  Measured on the c3 bench (ms per step, 48 calls): k_spmm 25.4,
// cp.async (LDGSTS) staging 20.1 (L1 data pipe 90% busy: the rows crossed
// it twice), this kernel 16.8.
// Rows are fetched with the sm_100 tensor-memory-accelerator gather
// (cp.async.bulk.tensor.2d ... tile::gather4: four X rows of b doubles per
// instruction, lanes 0..7 each issue one per chunk) completing on one
// mbarrier per stage, so the gathered bytes cross the L1 data pipe once
// (the consumer's LDS).  Padding rows use coordinate -1: TMA zero-fills
// out-of-bounds rows and still counts their bytes.
// TX: element type of X (double, or float for the fp32 variant).  G4 and
// ROWS count TX elements; STG (the stage size) and ROWSD count doubles.
template <int P, int V = 2, typename TX = double>
struct TmaGeom {
  static constexpr int ES = (int)sizeof(TX);
  static constexpr int B = V * P;  // columns: P lanes x V values
  static constexpr int G4 = (4 * B * ES + 127) / 128 * 128 / ES;  // elements per gather4 block (128-B aligned)
  static constexpr int ROWS = 8 * G4;                              // 32 rows
  static constexpr int ROWSD = ROWS * ES / 8;
  static constexpr int STG = ROWSD + 64;  // k_spmm_tma stage: + 32 values + 16 (meta, pad) + 16 (32 column ids)
};

// V doubles per lane (V = 2: b <= 32; V = 4: 32 < b <= 64, b % 4 == 0),
// held as V/2 double2.
template <int V>
struct Acc {
  double2 h[V / 2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < V / 2; ++i) h[i] = make_double2(0.0, 0.0);
  }
  __device__ __forceinline__ void load(const double* p) {
#pragma unroll
    for (int i = 0; i < V / 2; ++i) h[i] = reinterpret_cast<const double2*>(p)[i];
  }
  __device__ __forceinline__ void load(const float* p) {
#pragma unroll
    for (int i = 0; i < V / 2; ++i) {
      const float2 f = reinterpret_cast<const float2*>(p)[i];
      h[i] = make_double2((double)f.x, (double)f.y);
    }
  }
  __device__ __forceinline__ void fma(double v, const Acc& x) {
#pragma unroll
    for (int i = 0; i < V / 2; ++i) {
      h[i].x = ::fma(v, x.h[i].x, h[i].x);
      h[i].y = ::fma(v, x.h[i].y, h[i].y);
    }
  }
  __device__ __forceinline__ void add(const Acc& o) {
#pragma unroll
    for (int i = 0; i < V / 2; ++i) {
      h[i].x += o.h[i].x;
      h[i].y += o.h[i].y;
    }
  }
  __device__ __forceinline__ Acc shfl(int src) const {
    Acc r;
#pragma unroll
    for (int i = 0; i < V / 2; ++i) r.h[i] = shfl_v(h[i], src);
    return r;
  }
  __device__ __forceinline__ void store(double* p) const {
#pragma unroll
    for (int i = 0; i < V / 2; ++i) reinterpret_cast<double2*>(p)[i] = h[i];
  }
};

template <int P, int S, int W, int V, typename TX = double>
__global__ void __launch_bounds__(W * 32, (V == 2 ? 2 : 1)) k_spmm_tma(
    const __grid_constant__ CUtensorMap tmX, int64_t nwarp, const int32_t* __restrict__ warp_seg,
    const int32_t* __restrict__ seg_row, const int64_t* __restrict__ seg_begin, const int64_t* __restrict__ seg_end,
    const int32_t* __restrict__ seg_slot, const int32_t* __restrict__ indices, const double* __restrict__ values,
    double* __restrict__ Y, int64_t ldy, double* __restrict__ partial) {
  using Gm = TmaGeom<P, V, TX>;
  constexpr int B = Gm::B, G = 32 / P, G4 = Gm::G4, ROWS = Gm::ROWSD, STG = Gm::STG;
  extern __shared__ __align__(128) double smd[];
  __shared__ __align__(8) uint64_t bars[W * S];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double* ring = smd + (size_t)wib * S * STG;
  uint64_t* bar = bars + wib * S;
  if (lane < S) mbar_init(bar + lane, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  if (w >= nwarp) return;
  const int g = lane / P, pc = lane - (lane / P) * P;
  const bool active = g < G;

  const int32_t s_lo = warp_seg[w], s_hi = warp_seg[w + 1];
  int32_t sb = s_lo;
  int64_t mb = 0, me = 0;
  int32_t mrow = 0, mslot = -1;
  auto load_meta = [&]() {
    const int32_t sg = sb + lane;
    if (sg < s_hi) {
      mb = seg_begin[sg];
      me = seg_end[sg];
      mrow = seg_row[sg];
      mslot = seg_slot[sg];
    }
  };
  load_meta();
  int32_t cur = s_lo;
  int64_t cb = 0, ce = 0;
  int32_t crow = 0, cslot = -1;
  bool cfirst = true;
  auto enter = [&]() {
    if (cur - sb >= 32) {
      sb = cur;
      load_meta();
    }
    const int i = cur - sb;
    cb = __shfl_sync(0xffffffffu, mb, i);
    ce = __shfl_sync(0xffffffffu, me, i);
    crow = __shfl_sync(0xffffffffu, mrow, i);
    cslot = __shfl_sync(0xffffffffu, mslot, i);
    cfirst = true;
  };
  if (cur < s_hi) enter();

  bool have = false;
  int32_t kci = -1;
  double kvi = 0.0;
  int4 km;
  auto load_chunk = [&]() {
    have = cur < s_hi;
    if (!have) return;
    const int nv = (int)min64(32, ce - cb);
    kci = -1;
    kvi = 0.0;
    if (lane < nv) {
      kci = __ldcs(indices + cb + lane);
      kvi = __ldcs(values + cb + lane);
    }
    const bool last = cb + 32 >= ce;
    km = make_int4(crow, cslot, nv, (cfirst ? 1 : 0) | (last ? 2 : 0));
    cfirst = false;
    cb += 32;
    if (last) {
      ++cur;
      if (cur < s_hi) enter();
    }
  };
  auto issue = [&](int slot) {
    double* st = ring + slot * STG;
    st[ROWS + lane] = kvi;
    if (lane == 0) *reinterpret_cast<int4*>(st + ROWS + 32) = km;
    const int ng = (km.z + 3) >> 2;
    const int t = lane & 7;
    const int r0 = __shfl_sync(0xffffffffu, kci, 4 * t);
    const int r1 = __shfl_sync(0xffffffffu, kci, 4 * t + 1);
    const int r2 = __shfl_sync(0xffffffffu, kci, 4 * t + 2);
    const int r3 = __shfl_sync(0xffffffffu, kci, 4 * t + 3);
    if (ng > 0) {
      if (lane == 0) mbar_expect_tx(bar + slot, (unsigned)(ng * 4 * B * sizeof(TX)));
      __syncwarp();
      if (lane < ng)
        tma_gather4(reinterpret_cast<TX*>(st) + lane * G4, &tmX, 0, r0, r1, r2, r3, bar + slot);
    } else if (lane == 0) {
      mbar_expect_tx(bar + slot, 0);  // empty or all-hot chunk: complete the phase
    }
  };

  // two accumulator pairs (even / odd steps of a chunk) halve the
  // dependent DFMA chain; they are added at the end of each row
  Acc<V> acc, acc1;
  acc.zero();
  acc1.zero();
  int64_t issued = 0, consumed = 0;
  load_chunk();
#pragma unroll
  for (int t = 0; t < S - 1; ++t) {
    if (have) {
      issue((int)(issued % S));
      ++issued;
      load_chunk();
    }
  }
  while (consumed < issued) {
    if (have) {
      issue((int)(issued % S));
      ++issued;
      load_chunk();
    }
    const int slot = (int)(consumed % S);
    mbar_wait(bar + slot, (unsigned)((consumed / S) & 1));
    __syncwarp();
    const double* st = ring + slot * STG;
    const int4 m = *reinterpret_cast<const int4*>(st + ROWS + 32);
    if (m.w & 1) {
      acc.zero();
      acc1.zero();
    }
    if (active) {
      // fully unrolled over the chunk's NS steps: unconditional loads at
      // constant smem offsets from one per-lane base (all in flight at
      // once; rows past the chunk are stale but in-bounds), FMAs masked
      constexpr int NS = (32 + G - 1) / G;
      const TX* sx = reinterpret_cast<const TX*>(st);
      const TX* xr = sx + ((g >> 2) * G4 + (g & 3) * B) + V * pc;
      const double* vr = st + ROWS + g;
      Acc<V> xs[NS];
      double vs[NS];
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        const int j = q * G + g;
        const int jo = q * G;
        const int jc = j < 32 ? j : 31;
        const TX* src = G4 == 4 * B ? xr + jo * B : sx + (jc >> 2) * G4 + (jc & 3) * B + V * pc;
        xs[q].load(src);
        vs[q] = vr[jc - g];
      }
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        if (q * G + g < m.z) {
          if (q & 1)
            acc1.fma(vs[q], xs[q]);
          else
            acc.fma(vs[q], xs[q]);
        }
      }
    }
    if (m.w & 2) {
      acc.add(acc1);
      Acc<V> tot = acc;
#pragma unroll
      for (int h = 1; h < G; ++h) {
        const Acc<V> o = acc.shfl((lane + h * P) & 31);
        if (g == 0) tot.add(o);
      }
      if (g == 0) {
        double* dst = m.y < 0 ? (Y + (int64_t)m.x * ldy + V * pc) : (partial + (int64_t)m.y * B + V * pc);
        tot.store(dst);
      }
    }
    ++consumed;
    __syncwarp();
  }
}

template <int P, int S, int W, int V = 2, typename TX = double>
int tma_launch(int64_t xrows, int64_t nwarp, const int32_t* warp_seg, const int32_t* seg_row,
               const int64_t* seg_begin, const int64_t* seg_end, const int32_t* seg_slot, const int32_t* indices,
               const double* values, const TX* X, int64_t ldx, double* Y, int64_t ldy, double* partial,
               cudaStream_t s) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) {
    set_error("spmm: cuTensorMapEncodeTiled unavailable");
    return SVDREC_E_UNSUPPORTED;
  }
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)(V * P), (cuuint64_t)xrows};
  const cuuint64_t strides[1] = {(cuuint64_t)ldx * sizeof(TX)};
  const cuuint32_t box[2] = {(cuuint32_t)(V * P), 1};
  const cuuint32_t es[2] = {1, 1};
  const CUtensorMapDataType dt = sizeof(TX) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const CUresult r = enc(&tm, dt, 2, const_cast<TX*>(X), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("spmm: tensor map encode failed (%d)", (int)r);
    return SVDREC_E_UNSUPPORTED;
  }
  constexpr size_t ring = (size_t)W * S * TmaGeom<P, V, TX>::STG * sizeof(double);
  constexpr size_t kMaxSmem = 226 * 1024;  // + the static mbarriers within the 227 KB opt-in
  static_assert(ring <= kMaxSmem, "spmm: gather rings exceed shared memory");
  SVDREC_CUDA(smem_attr_once(k_spmm_tma<P, S, W, V, TX>, (int)kMaxSmem));
  const int64_t grid = (nwarp + W - 1) / W;
  k_spmm_tma<P, S, W, V, TX><<<(unsigned)grid, W * 32, ring, s>>>(tm, nwarp, warp_seg, seg_row, seg_begin, seg_end,
                                                                  seg_slot, indices, values, Y, ldy, partial);
  return check_launch("spmm_tma");
}

// Wide blocks (32 < b <= 64, b % 4 == 0): four doubles per lane, P = b / 4
// lanes per row, one CTA of w4_warps(P) warps per SM (the rings of 4-row
// gathers of b-wide rows are twice as large).
constexpr int w4_warps(int P) {
  // two stages of TmaGeom<P, 4> per warp within the 226 KB budget, <= 8 warps
  return (226 * 1024) / (2 * (8 * ((4 * 4 * P * 8 + 127) / 128 * 16) + 64) * 8) < 8
             ? (226 * 1024) / (2 * (8 * ((4 * 4 * P * 8 + 127) / 128 * 16) + 64) * 8)
             : 8;
}

int tma_dispatch4(int b, int64_t xrows, int64_t nwarp, const int32_t* warp_seg, const int32_t* seg_row,
                  const int64_t* seg_begin, const int64_t* seg_end, const int32_t* seg_slot, const int32_t* indices,
                  const double* values, const double* X, int64_t ldx, double* Y, int64_t ldy, double* partial,
                  cudaStream_t s) {
#define SVDREC_TMA4(PP)                                                                                          \
  case PP:                                                                                                       \
    return tma_launch<PP, 2, w4_warps(PP), 4>(xrows, nwarp, warp_seg, seg_row, seg_begin, seg_end,       \
                                                     seg_slot, indices, values, X, ldx, Y, ldy, partial, s);
  switch (b / 4) {
    SVDREC_TMA4(9)
    SVDREC_TMA4(10)
    SVDREC_TMA4(11)
    SVDREC_TMA4(12)
    SVDREC_TMA4(13)
    SVDREC_TMA4(14)
    SVDREC_TMA4(15)
    SVDREC_TMA4(16)
    default:
      return SVDREC_E_ARG;
  }
#undef SVDREC_TMA4
}

// fp32 X, 32 < b <= 64 (b % 4 == 0): four floats per lane; the rings are
// half as wide as the double ones, so twice the warps fit (<= 12 per SM).
constexpr int w4f_warps(int P) {
  return (226 * 1024) / (2 * (8 * ((4 * 4 * P * 4 + 127) / 128 * 128) + 512)) < 12
             ? (226 * 1024) / (2 * (8 * ((4 * 4 * P * 4 + 127) / 128 * 128) + 512))
             : 12;
}

int tma_dispatch4_f32(int b, int64_t xrows, int64_t nwarp, const int32_t* warp_seg, const int32_t* seg_row,
                      const int64_t* seg_begin, const int64_t* seg_end, const int32_t* seg_slot,
                      const int32_t* indices, const double* values, const float* X, int64_t ldx, double* Y,
                      int64_t ldy, double* partial, cudaStream_t s) {
#define SVDREC_TMA4F(PP)                                                                                         \
  case PP:                                                                                                       \
    return tma_launch<PP, 2, w4f_warps(PP), 4, float>(xrows, nwarp, warp_seg, seg_row, seg_begin,         \
                                                              seg_end, seg_slot, indices, values, X, ldx, Y, ldy, \
                                                              partial, s);
  switch (b / 4) {
    SVDREC_TMA4F(9)
    SVDREC_TMA4F(10)
    SVDREC_TMA4F(11)
    SVDREC_TMA4F(12)
    SVDREC_TMA4F(13)
    SVDREC_TMA4F(14)
    SVDREC_TMA4F(15)
    SVDREC_TMA4F(16)
    default:
      return SVDREC_E_ARG;
  }
#undef SVDREC_TMA4F
}

// ---------------------------------------------------------------------------
// Chunk-record pipeline (round 2): the same gather4 rings, driven by the
// precomputed 16-B chunk records of csrc/ingest.cu (svdrec_chunk_plan)
// instead of per-segment metadata, shuffles and 64-bit bounds arithmetic --
// k_spmm_tma above runs ~390 warp instructions per 32-entry chunk and is
// bound by that serial stream (16 warps per SM, ~2,250 cycles per chunk per
// warp whatever the ring depth).  Here a chunk costs ~120:
//   fetch   the chunk's 32 column ids and values go global -> shared memory
//           by cp.async (LDGSTS, zero-filled past the
//           chunk's end), D chunks deep, so no register waits on the CSR
//           stream's HBM latency;
//   gather  lanes 0..7 read four ids each with one LDS.128 and issue the
//           gather4 of those X rows into the S-deep row ring (mbarrier tx);
//   consume as k_spmm_tma: NS unrolled LDS.128 + LDS.64 + DFMA steps on two
//           accumulator chains, fixed-order group fold at a segment's end.
// Summation order per output element is the one of k_spmm / k_spmm_tma.
// (an L2 evict-first cache hint on these 4- / 8-byte copies raises "illegal
// instruction" on sm_100a: plain .ca copies)
__device__ __forceinline__ void cp_async4(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int kRecRing = 16;   // per-warp ring of chunk records in shared memory
constexpr int kRecAhead = 8;   // records are copied in this many chunks ahead of their fetch

template <int P, int S, int D, int V, typename TX>
struct PipeGeom {
  using Gm = TmaGeom<P, V, TX>;
  static constexpr int CSRB = 384;  // bytes per CSR slot: 32 values, 32 ids
  static constexpr int WARPB = S * Gm::ROWSD * 8 + (D * CSRB + kRecRing * 16 + 127) / 128 * 128;  // bytes per warp
};

// Split rows folded into the SpMM kernel: slot -> split-row index, the rows'
// slot ranges and destinations, and one zero-initialised ticket per split row
// (done == nullptr: the separate fix-up kernel adds the partials instead).
struct FixArgs {
  const int32_t* slot_long;
  const int32_t* row;
  const int32_t* s0;
  const int32_t* s1;
  int* done;
};

template <int P, int S, int D, int W, int V, typename TX = double>
__global__ void __launch_bounds__(W * 32, (V == 2 ? 2 : 1)) k_spmm_pipe(
    const __grid_constant__ CUtensorMap tmX, int64_t nwarp, const int32_t* __restrict__ warp_chunk,
    const int4* __restrict__ chunks, const int32_t* __restrict__ indices, const double* __restrict__ values,
    double* __restrict__ Y, int64_t ldy, double* __restrict__ partial, FixArgs fix) {
  static_assert(D >= S, "spmm: the CSR ring must be at least as deep as the row ring");
  static_assert(kRecAhead >= 2 * (D - S + 1) && kRecAhead + D <= kRecRing, "spmm: record ring too small");
  using Gm = TmaGeom<P, V, TX>;
  using Pg = PipeGeom<P, S, D, V, TX>;
  constexpr int B = Gm::B, G = 32 / P, G4 = Gm::G4, ROWS = Gm::ROWSD;
  extern __shared__ __align__(128) unsigned char smb[];
  __shared__ __align__(8) uint64_t bars[W * S];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned char* base = smb + (size_t)wib * Pg::WARPB;
  double* rows = reinterpret_cast<double*>(base);                   // S stages of ROWS doubles
  unsigned char* csr = base + (size_t)S * ROWS * 8;                 // D slots of CSRB bytes
  int4* rring = reinterpret_cast<int4*>(csr + D * Pg::CSRB);        // kRecRing chunk records
  uint64_t* bar = bars + wib * S;
  if (lane < S) mbar_init(bar + lane, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  if (w >= nwarp) return;
  const int g = lane / P, pc = lane - (lane / P) * P;
  const bool active = g < G;
  // where this lane's piece of row j = q G + g sits in a stage (elements of
  // TX).  When four rows fill a whole number of 128-B units the rows are
  // contiguous and the offset is a constant per step; otherwise (gather4
  // blocks padded to 128 B: 3-, 5-, 7-lane rows, float rows) the NS offsets
  // are computed once here instead of per chunk.
  constexpr int NS = (32 + G - 1) / G;
  constexpr bool kContig = G4 == 4 * B;
  int offs[kContig ? 1 : NS];
  if constexpr (!kContig) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      const int jc = q * G + g < 32 ? q * G + g : 31;
      offs[q] = (jc >> 2) * G4 + (jc & 3) * B + V * pc;
    }
  } else {
    offs[0] = 0;
  }

  const int32_t c_lo = warp_chunk[w], c_hi = warp_chunk[w + 1];
  const int n = c_hi - c_lo;
  if (n <= 0) return;
  // the chunk records travel through their own small ring: the first
  // kRecAhead are read here, record j + kRecAhead is copied in (cp.async,
  // lane 0) at step j, so no step waits on a record's global load
  if (lane < kRecAhead && lane < n) rring[lane] = __ldg(chunks + c_lo + lane);
  __syncwarp();
  // The main loop is unrolled by D, so every ring index below is a
  // compile-time constant of the unrolled step u (i = i0 + u, i0 % D == 0):
  // CSR slot i % D = u, row stage i % S = u % S, and -- D / S being even --
  // the stage's phase parity too.
  static_assert(D % S == 0 && (D / S) % 2 == 0 && kRecRing % D == 0, "spmm: ring sizes must nest");
  auto fetch = [&](int f, int fs, int rj) {  // CSR of chunk f into slot fs; request record rj
    if (f < n) {
      const int4 rec = rring[f & (kRecRing - 1)];
      const int64_t off = (int64_t)(((uint64_t)(uint32_t)rec.w << 32) | (uint32_t)rec.x);
      const bool in = lane < (rec.z & 63);
      const int64_t o = off + (in ? lane : 0);
      unsigned char* sl = csr + fs * Pg::CSRB;
      cp_async8(sl + 8 * lane, values + o, in ? 8u : 0u);
      cp_async4(sl + 256 + 4 * lane, indices + o, in ? 4u : 0u);
    }
    if (rj >= 0 && rj < n && lane == 0) cp_async16(rring + (rj & (kRecRing - 1)), chunks + c_lo + rj);
    cp_async_commit();
  };
  auto gather = [&](int j, int gs, int gr) {  // chunk j: CSR slot gs -> row stage gr
    cp_async_wait<D - S>();
    __syncwarp();
    const unsigned char* sl = csr + gs * Pg::CSRB;
    const int nvf = rring[j & (kRecRing - 1)].z;
    const int ng = ((nvf & 63) + 3) >> 2;
    if (lane == 0) mbar_expect_tx(bar + gr, (unsigned)(ng * 4 * B * sizeof(TX)));
    if (lane < ng) {
      const int4 r = *reinterpret_cast<const int4*>(sl + 256 + 16 * lane);
      tma_gather4(reinterpret_cast<TX*>(rows + gr * ROWS) + lane * G4, &tmX, 0, r.x, r.y, r.z, r.w, bar + gr);
    }
  };
  Acc<V> acc, acc1;
  acc.zero();
  acc1.zero();
  auto consume = [&](int j, int cs, int cr, unsigned cph) {  // chunk j from CSR slot cs / row stage cr (parity cph)
    const unsigned char* sl = csr + cs * Pg::CSRB;
    const int4 m = rring[j & (kRecRing - 1)];  // y: destination, z: entries | flags
    const int nv = m.z & 63;
    mbar_wait(bar + cr, cph);
    if (active) {
      const TX* sx = reinterpret_cast<const TX*>(rows + cr * ROWS);
      const TX* xr = sx + ((g >> 2) * G4 + (g & 3) * B) + V * pc;
      const double* vr = reinterpret_cast<const double*>(sl) + g;
      Acc<V> xs[NS];
      double vs[NS];
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        const int jj = q * G + g;
        const int jo = q * G;
        const int jc = jj < 32 ? jj : 31;
        const TX* src = kContig ? xr + jo * B : sx + offs[kContig ? 0 : q];
        xs[q].load(src);
        vs[q] = vr[jc - g];
      }
      if (nv == 32) {
        // a full chunk (most of them): no per-step bounds
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          if ((q + 1) * G <= 32 || q * G + g < 32) {
            if (q & 1)
              acc1.fma(vs[q], xs[q]);
            else
              acc.fma(vs[q], xs[q]);
          }
        }
      } else {
        const int left = nv - g;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          if (q * G < left) {
            if (q & 1)
              acc1.fma(vs[q], xs[q]);
            else
              acc.fma(vs[q], xs[q]);
          }
        }
      }
    }
    if (m.z & 512) {
      acc.add(acc1);
      Acc<V> tot = acc;
#pragma unroll
      for (int h = 1; h < G; ++h) {
        const Acc<V> o = acc.shfl((lane + h * P) & 31);
        if (g == 0) tot.add(o);
      }
      if (g == 0) {
        double* dst = m.y >= 0 ? (Y + (int64_t)m.y * ldy + V * pc) : (partial + (int64_t)(~m.y) * B + V * pc);
        tot.store(dst);
      }
      if (m.y < 0 && fix.done != nullptr) {
        // a split row's segment: the warp that completes the row's last
        // outstanding segment adds the row's partial sums in slot order (the
        // fix-up kernel's sum, bit for bit) -- no separate launch
        __threadfence();  // this segment's partial is visible before its ticket
        __syncwarp();
        const int L = __ldg(fix.slot_long + (~m.y));
        const int s0 = __ldg(fix.s0 + L), s1 = __ldg(fix.s1 + L);
        int prev = 0;
        if (lane == 0) prev = atomicAdd(fix.done + L, 1);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == s1 - s0 - 1) {
          __threadfence();
          if (g == 0) {
            Acc<V> sum;
            sum.zero();
            for (int sl2 = s0; sl2 < s1; ++sl2) {
              Acc<V> p;
#pragma unroll
              for (int h = 0; h < V / 2; ++h)
                p.h[h] = __ldcg(reinterpret_cast<const double2*>(partial + (int64_t)sl2 * B + V * pc) + h);
              sum.add(p);
            }
            sum.store(Y + (int64_t)__ldg(fix.row + L) * ldy + V * pc);
          }
          if (lane == 0) fix.done[L] = 0;  // ready for the next launch
        }
      }
      acc.zero();  // the next segment starts at zero (segments never span warps)
      acc1.zero();
    }
    __syncwarp();  // every lane is done with the stage and the CSR slot
  };

  constexpr int F = D - S + 1;  // chunks fetched ahead of the gather
#pragma unroll
  for (int t = 0; t < F; ++t) fetch(t, t, -1);
  const int total = n + S - 1;
  for (int i0 = 0; i0 < total; i0 += D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int i = i0 + u;
      if (i < total) {
        if (i < n) gather(i, u, u % S);
        // chunk j = i - (S - 1) = i0 + e, e = u - S + 1: slot (u + F) % D, stage (u + 1) % S, phase
        // parity (j / S) & 1 = (e / S) & 1 for e >= 0, else 1 (i0 / S is even)
        if (i >= S - 1) {
          const int e = u - S + 1;
          consume(i - (S - 1), (u + F) % D, (u + 1) % S, e >= 0 ? (unsigned)((e / S) & 1) : 1u);
        }
        fetch(i + F, (u + F) % D, i + kRecAhead);
      }
    }
  }
  cp_async_wait<0>();
}

template <int P, int S, int D, int W, int V = 2, typename TX = double>
int pipe_launch(int64_t xrows, int64_t nwarp, const int32_t* warp_chunk, const void* chunks, const int32_t* indices,
                const double* values, const TX* X, int64_t ldx, double* Y, int64_t ldy, double* partial, FixArgs fix,
                cudaStream_t s) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) {
    set_error("spmm: cuTensorMapEncodeTiled unavailable");
    return SVDREC_E_UNSUPPORTED;
  }
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)(V * P), (cuuint64_t)xrows};
  const cuuint64_t strides[1] = {(cuuint64_t)ldx * sizeof(TX)};
  const cuuint32_t box[2] = {(cuuint32_t)(V * P), 1};
  const cuuint32_t es[2] = {1, 1};
  const CUtensorMapDataType dt = sizeof(TX) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const CUresult r = enc(&tm, dt, 2, const_cast<TX*>(X), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("spmm: tensor map encode failed (%d)", (int)r);
    return SVDREC_E_UNSUPPORTED;
  }
  constexpr size_t ring = (size_t)W * PipeGeom<P, S, D, V, TX>::WARPB;
  constexpr size_t kMaxSmem = 226 * 1024;
  if constexpr (ring > kMaxSmem) {
    set_error("spmm: the gather rings of this build exceed shared memory (b=%d)", V * P);
    return SVDREC_E_UNSUPPORTED;
  } else {
    SVDREC_CUDA(smem_attr_once(k_spmm_pipe<P, S, D, W, V, TX>, (int)kMaxSmem));
    const int64_t grid = (nwarp + W - 1) / W;
    k_spmm_pipe<P, S, D, W, V, TX><<<(unsigned)grid, W * 32, ring, s>>>(
        tm, nwarp, warp_chunk, reinterpret_cast<const int4*>(chunks), indices, values, Y, ldy, partial, fix);
    return check_launch("spmm_pipe");
  }
}

#ifndef SVDREC_SPMM_S2
#define SVDREC_SPMM_S2 2  // row-ring stages per warp
#endif
#ifndef SVDREC_SPMM_D2
#define SVDREC_SPMM_D2 4  // CSR-ring slots per warp
#endif
#ifndef SVDREC_SPMM_W2
#define SVDREC_SPMM_W2 8  // warps per CTA of the 2-CTA-per-SM variant (b <= 32)
#endif
constexpr int kS2 = SVDREC_SPMM_S2, kD2 = SVDREC_SPMM_D2, kW2 = SVDREC_SPMM_W2;

#define SVDREC_PIPE_ARGS xrows, nwarp, warp_chunk, chunks, indices, values, X, ldx, Y, ldy, partial, fix, s

// even b <= 32: the chunk-record pipeline, two CTAs of kW2 warps per SM
int pipe_dispatch(int b, int64_t xrows, int64_t nwarp, const int32_t* warp_chunk, const void* chunks,
                  const int32_t* indices, const double* values, const double* X, int64_t ldx, double* Y, int64_t ldy,
                  double* partial, FixArgs fix, cudaStream_t s) {
#define SVDREC_PIPE(PP) \
  case PP:              \
    return pipe_launch<PP, kS2, kD2, kW2, 2, double>(SVDREC_PIPE_ARGS);
  switch (b / 2) {
    SVDREC_PIPE(1) SVDREC_PIPE(2) SVDREC_PIPE(3) SVDREC_PIPE(4) SVDREC_PIPE(5) SVDREC_PIPE(6) SVDREC_PIPE(7)
    SVDREC_PIPE(8) SVDREC_PIPE(9) SVDREC_PIPE(10) SVDREC_PIPE(11) SVDREC_PIPE(12) SVDREC_PIPE(13)
    SVDREC_PIPE(14) SVDREC_PIPE(15) SVDREC_PIPE(16)
    default: return SVDREC_E_ARG;
  }
#undef SVDREC_PIPE
}

// fp32 X (the fp32 variant), b % 4 == 0 <= 32: the same kernel with float
// rows (half the gathered bytes; every TMA row a multiple of 16 B)
int pipe_dispatch_f32(int b, int64_t xrows, int64_t nwarp, const int32_t* warp_chunk, const void* chunks,
                      const int32_t* indices, const double* values, const float* X, int64_t ldx, double* Y,
                      int64_t ldy, double* partial, FixArgs fix, cudaStream_t s) {
#define SVDREC_PIPEF(PP) \
  case PP:               \
    return pipe_launch<PP, kS2, kD2, 8, 2, float>(SVDREC_PIPE_ARGS);
  switch (b / 2) {
    SVDREC_PIPEF(2) SVDREC_PIPEF(4) SVDREC_PIPEF(6) SVDREC_PIPEF(8) SVDREC_PIPEF(10) SVDREC_PIPEF(12)
    SVDREC_PIPEF(14) SVDREC_PIPEF(16)
    default: return SVDREC_E_ARG;
  }
#undef SVDREC_PIPEF
}

// ---------------------------------------------------------------------------
// Hot-set variant for A @ X on the popularity-ranked CSR (b even, b <= 32).
// Each row's entries are stored hottest item first; an entry's index is
// -(rank + 1) for the nhot most rated items -- whose rows of X are staged
// once per CTA in shared memory -- and the item id otherwise.  A 32-entry
// batch therefore splits into a shared-memory prefix (LDS) and an
// L2-gathered suffix (LDG, U steps in flight per lane), so only the cold
// entries reach L2 (c3, b = 20: 1,280 hot rows hold ~66 % of the ratings).
// One persistent CTA per SM; lanes as in k_spmm_tma (G = 32 / P groups of
// P lanes x 2 doubles), nonzero-balanced warp ranges, fixed-order group
// fold, two accumulator chains; loads are unconditional (masked entries
// read a valid row and contribute 0 * x).
struct __align__(16) TabEnt {
  int32_t off;  // hot: rank * P (double2 units in shared memory); cold: item * ldx / 2
  int32_t pad;
  double v;
};
constexpr int kHotWarps = 16;
constexpr int kTabSlots = 32 + 32;  // a batch + the padding of G * U <= 32 steps

// V = 2: P = b / 2 lanes of one double2 per row; V = 4: P = b / 4 lanes
// holding doubles {2pc, 2pc + 1} and {b/2 + 2pc, b/2 + 2pc + 1}, so each
// LDS.128 / LDG.128 reads one contiguous half row per group (for b = 64: a
// 128-B phase per 8 lanes, no bank conflicts).
template <int P, int U, int V>
__global__ void __launch_bounds__(512, 1) k_spmm_hot(
    int64_t nwarp, const int32_t* __restrict__ warp_seg, const int32_t* __restrict__ seg_row,
    const int64_t* __restrict__ seg_begin, const int64_t* __restrict__ seg_end, const int32_t* __restrict__ seg_slot,
    const int32_t* __restrict__ hidx, const double* __restrict__ hval, const double* __restrict__ X, int64_t ldx,
    const int32_t* __restrict__ hot_items, int nhot, double* __restrict__ Y, int64_t ldy,
    double* __restrict__ partial) {
  constexpr int B = V * P, G = 32 / P, H = B / 4;  // H: double2 offset of the second half (V = 4)
  constexpr int RB = B / 2;                        // double2 per row
  static_assert(G * U <= 32, "spmm_hot: padding exceeds the table");
  __shared__ TabEnt tabs[kHotWarps * 2 * kTabSlots];
  extern __shared__ __align__(16) double hs[];  // nhot rows of B doubles
  for (int t = threadIdx.x; t < nhot * RB; t += blockDim.x) {
    const int r = t / RB, c = t - (t / RB) * RB;
    reinterpret_cast<double2*>(hs)[t] =
        *reinterpret_cast<const double2*>(X + (int64_t)hot_items[r] * ldx + 2 * c);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nwarp) return;
  const int g = lane / P, pc = lane - (lane / P) * P;
  const bool active = g < G;
  const double2* hrow = reinterpret_cast<const double2*>(hs) + pc;   // + rank * RB
  const double2* xrow = reinterpret_cast<const double2*>(X) + pc;    // + item * ldx / 2
  const int64_t ldx2 = ldx / 2;
  const int32_t s_lo = warp_seg[w], s_hi = warp_seg[w + 1];
  // segment metadata, 32 segments at a time (as k_spmm_tma)
  int32_t sb = s_lo;
  int64_t mb = 0, me = 0;
  int32_t mrow = 0, mslot = -1;
  auto load_meta = [&]() {
    const int32_t sg = sb + lane;
    if (sg < s_hi) {
      mb = seg_begin[sg];
      me = seg_end[sg];
      mrow = seg_row[sg];
      mslot = seg_slot[sg];
    }
  };
  load_meta();
  int32_t cur = s_lo;
  int64_t cb = 0, ce = 0;
  int32_t crow = 0, cslot = -1;
  auto enter = [&]() {
    if (cur - sb >= 32) {
      sb = cur;
      load_meta();
    }
    const int i = cur - sb;
    cb = __shfl_sync(0xffffffffu, mb, i);
    ce = __shfl_sync(0xffffffffu, me, i);
    crow = __shfl_sync(0xffffffffu, mrow, i);
    cslot = __shfl_sync(0xffffffffu, mslot, i);
  };
  if (cur < s_hi) enter();
  // the next 32-entry batch is loading while one is accumulated (two
  // statically named buffers: no register move waits on a pending load)
  struct Batch {
    int32_t ci, row, slot;
    double vi;
    int nv, flags;  // flags bit 0: first batch of its segment, bit 1: last
    bool ok;        // a batch (empty rows give batches with nv = 0)
  };
  bool cfirst = true;
  auto load_batch = [&](Batch& k) {
    k.ok = cur < s_hi;
    if (!k.ok) return;
    k.nv = (int)min64(32, ce - cb);
    k.ci = 0;
    k.vi = 0.0;
    if (lane < k.nv) {
      k.ci = __ldcs(hidx + cb + lane);
      k.vi = __ldcs(hval + cb + lane);
    }
    const bool last = cb + 32 >= ce;
    k.flags = (cfirst ? 1 : 0) | (last ? 2 : 0);
    k.row = crow;
    k.slot = cslot;
    cfirst = false;
    cb += 32;
    if (last) {
      ++cur;
      cfirst = true;
      if (cur < s_hi) enter();
    }
  };
  // per-warp batch tables (offset, value): the hot prefix and the cold
  // suffix of the current batch, each padded with G * U zero entries so
  // the unrolled steps need no masks (a pad reads row 0 times 0.0)
  TabEnt* ht = tabs + (size_t)(threadIdx.x >> 5) * 2 * kTabSlots;
  TabEnt* ct = ht + kTabSlots;
  // two accumulator chains (even / odd steps); V = 4 lanes hold two halves
  double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
  double2 c0 = make_double2(0.0, 0.0), c1 = make_double2(0.0, 0.0);
  auto process = [&](const Batch& k) {
    const int32_t ci = k.ci;
    const double vi = k.vi;
    const int nv = k.nv;
    if (k.flags & 1) {
      a0 = a1 = c0 = c1 = make_double2(0.0, 0.0);
    }
    // the batch's hot and cold entries, each in row order, go to their
    // tables (a row's entries are in item order: hot and cold interleave)
    const bool hot = lane < nv && ci < 0;
    const unsigned hm = __ballot_sync(0xffffffffu, hot);
    const int nh = __popc(hm);
    const int hpos = __popc(hm & ((1u << lane) - 1u));
    __syncwarp();  // the previous batch's tables are consumed
    if (lane < nv) {
      if (hot)
        ht[hpos] = TabEnt{(-ci - 1) * RB, 0, vi};
      else
        ct[lane - hpos] = TabEnt{ci * (int32_t)ldx2, 0, vi};
    }
    if (lane < G * U) {
      ht[nh + lane] = TabEnt{0, 0, 0.0};
      ct[nv - nh + lane] = TabEnt{0, 0, 0.0};
    }
    __syncwarp();
    if (active) {
      // hot entries: shared memory
      for (int j = 0; j < nh; j += G * U) {
        double2 x[U], y[U];
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const TabEnt e = ht[j + u * G + g];
          v[u] = e.v;
          x[u] = hrow[e.off];
          if (V == 4) y[u] = hrow[e.off + H];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          double2& acc = (u & 1) ? a1 : a0;
          acc.x = fma(v[u], x[u].x, acc.x);
          acc.y = fma(v[u], x[u].y, acc.y);
          if (V == 4) {
            double2& acd = (u & 1) ? c1 : c0;
            acd.x = fma(v[u], y[u].x, acd.x);
            acd.y = fma(v[u], y[u].y, acd.y);
          }
        }
      }
      // cold entries: gathered from L2 / HBM
      for (int j = 0; j < nv - nh; j += G * U) {
        double2 x[U], y[U];
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const TabEnt e = ct[j + u * G + g];
          v[u] = e.v;
          x[u] = __ldg(xrow + e.off);
          if (V == 4) y[u] = __ldg(xrow + e.off + H);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          double2& acc = (u & 1) ? a1 : a0;
          acc.x = fma(v[u], x[u].x, acc.x);
          acc.y = fma(v[u], x[u].y, acc.y);
          if (V == 4) {
            double2& acd = (u & 1) ? c1 : c0;
            acd.x = fma(v[u], y[u].x, acd.x);
            acd.y = fma(v[u], y[u].y, acd.y);
          }
        }
      }
    }
    if (k.flags & 2) {
      double2 t0 = make_double2(a0.x + a1.x, a0.y + a1.y);
      double2 t1 = make_double2(c0.x + c1.x, c0.y + c1.y);
      double2 tot = t0, tot1 = t1;
#pragma unroll
      for (int h = 1; h < G; ++h) {
        const double2 o = shfl_v(t0, (lane + h * P) & 31);
        const double2 o1 = V == 4 ? shfl_v(t1, (lane + h * P) & 31) : o;
        if (g == 0) {
          tot.x += o.x;
          tot.y += o.y;
          if (V == 4) {
            tot1.x += o1.x;
            tot1.y += o1.y;
          }
        }
      }
      if (g == 0) {
        double* dst = k.slot < 0 ? (Y + (int64_t)k.row * ldy) : (partial + (int64_t)k.slot * B);
        *reinterpret_cast<double2*>(dst + 2 * pc) = tot;
        if (V == 4) *reinterpret_cast<double2*>(dst + 2 * H + 2 * pc) = tot1;
      }
    }
  };
  Batch q0, q1;
  load_batch(q0);
  load_batch(q1);
  while (q0.ok) {
    process(q0);
    load_batch(q0);
    if (!q1.ok) break;
    process(q1);
    load_batch(q1);
  }
}

// ---------------------------------------------------------------------------
// Hot / cold chunk kernel for A @ X (even b <= 32; round 2): the rows of X
// of the nhot most rated items sit in every CTA's shared memory (1,216 rows
// at b = 20 hold 64 % of the ratings).  The CSR is the PACKED hot-first copy
// (k_hot_pack: 16-B entries {rank or item, value}, every row's hot entries
// first) and its chunk plan never lets a chunk straddle a row's hot / cold
// boundary (csrc/ingest.cu), so a chunk is either
//   HOT   32 rows read from the shared-memory table (LDS.128), or
//   COLD  32 rows gathered straight into registers (LDG.128, all NS steps
//         in flight at once),
// with no per-batch ballot / table building (k_spmm_hot) and no TMA issue
// loop (11 instructions per gather4 in k_spmm_pipe).  Entries reach shared
// memory by one 16-B cp.async per lane per chunk (L1 bypassed), D chunks
// ahead; records through the ring of k_spmm_pipe.  No row rings: ~2.3 KB of
// shared memory per warp, the rest is the hot table.
struct __align__(16) PackEnt {
  int32_t id;  // hot chunk: popularity rank (row of the table); cold: item id
  int32_t pad;
  double v;
};

template <int D>
struct HcGeom {
  static constexpr int WARPB = D * 512 + kRecRing * 16;  // D slots of 32 entries + the record ring
};

template <int P, int D, int W>
__global__ void __launch_bounds__(W * 32, 1) k_spmm_hc(
    int64_t nwarp, const int32_t* __restrict__ warp_chunk, const int4* __restrict__ chunks,
    const PackEnt* __restrict__ ents, const double* __restrict__ X, int64_t ldx,
    const int32_t* __restrict__ hot_items, int nhot, double* __restrict__ Y, int64_t ldy,
    double* __restrict__ partial) {
  static_assert(kRecAhead >= 2 * D && kRecAhead + 1 <= kRecRing && kRecRing % D == 0, "spmm_hc: record ring too small");
  constexpr int B = 2 * P, G = 32 / P, RB = P;
  extern __shared__ __align__(128) unsigned char smb[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double2* hot = reinterpret_cast<double2*>(smb + (size_t)W * HcGeom<D>::WARPB);  // nhot rows of RB double2
  for (int t = threadIdx.x; t < nhot * RB; t += blockDim.x) {
    const int r = t / RB, c = t - (t / RB) * RB;
    hot[t] = *reinterpret_cast<const double2*>(X + (int64_t)hot_items[r] * ldx + 2 * c);
  }
  __syncthreads();
  if (w >= nwarp) return;
  PackEnt* slots = reinterpret_cast<PackEnt*>(smb + (size_t)wib * HcGeom<D>::WARPB);  // D x 32 entries
  int4* rring = reinterpret_cast<int4*>(slots + D * 32);
  // lane -> (row group g, 16-B piece pc of the row).  For 8 < P < 16 (rows of
  // 144..240 B) the first eight pieces of each group's row take one whole
  // quarter-warp -- a 128-B contiguous, conflict-free shared-memory phase --
  // and the rows' tails share the last phase; otherwise groups are
  // contiguous runs of P lanes.
  constexpr bool kPhased = P > 8 && P < 16;
  constexpr int T = kPhased ? P - 8 : 0;  // tail pieces per row
  int g, pc;
  if (kPhased) {
    if (lane < 8 * G) {
      g = lane >> 3;
      pc = lane & 7;
    } else {
      const int t = lane - 8 * G;
      g = t / (T ? T : 1);
      pc = 8 + t - g * T;
    }
  } else {
    g = lane / P;
    pc = lane - g * P;
  }
  const bool active = g < G;
  auto lane_of = [&](int gg, int p) { return kPhased ? (p < 8 ? 8 * gg + p : 8 * G + gg * T + (p - 8)) : gg * P + p; };
  const double2* hrow = hot + pc;
  const double2* xrow = reinterpret_cast<const double2*>(X) + pc;
  const int ldx2 = (int)(ldx / 2);  // row pitch in double2 (the host checks rows x pitch < 2^31)

  const int32_t c_lo = warp_chunk[w], c_hi = warp_chunk[w + 1];
  const int n = c_hi - c_lo;
  if (n <= 0) return;
  if (lane < kRecAhead && lane < n) rring[lane] = __ldg(chunks + c_lo + lane);
  __syncwarp();
  // Entries of chunk f into slot fs.  Lanes past the chunk's end copy only
  // the ID of the chunk's first entry (4 of 16 bytes, the rest zero-filled):
  // a pad then reads a row its output already depends on, times 0.0 -- the
  // accumulation needs no bounds, and a non-finite X pollutes nothing the
  // reference would not.
  auto fetch = [&](int f, int fs, int rj) {
    if (f < n) {
      const int4 rec = rring[f & (kRecRing - 1)];
      const int64_t off = (int64_t)(((uint64_t)(uint32_t)rec.w << 32) | (uint32_t)rec.x);
      const int nv = rec.z & 63;
      const bool in = lane < nv;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(slots + fs * 32 + lane)),
                   "l"(ents + off + (in ? lane : 0)), "r"(in ? 16u : (nv ? 4u : 0u))
                   : "memory");
    }
    if (rj < n && lane == 0) cp_async16(rring + (rj & (kRecRing - 1)), chunks + c_lo + rj);
    cp_async_commit();
  };
  Acc<2> acc, acc1;
  acc.zero();
  acc1.zero();
  auto consume = [&](int i, int cs) {
    cp_async_wait<D - 1>();  // chunk i's entries (and the records requested >= D steps ago) have landed
    __syncwarp();
    const int4 m = rring[i & (kRecRing - 1)];  // y: destination, z: entries | flags
    if (active && (m.z & 63)) {
      constexpr int NS = (32 + G - 1) / G;
      const PackEnt* sl = slots + cs * 32 + g;
      Acc<2> xs[NS];
      double vs[NS];
      if (m.z & 1024) {
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          const PackEnt e = sl[q * G + g < 32 ? q * G : 31 - g];
          xs[q].h[0] = hrow[e.id * RB];
          vs[q] = e.v;
        }
      } else {
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          const PackEnt e = sl[q * G + g < 32 ? q * G : 31 - g];
          xs[q].h[0] = __ldg(xrow + (int64_t)e.id * ldx2);
          vs[q] = e.v;
        }
      }
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        if ((q + 1) * G <= 32 || q * G + g < 32) {
          if (q & 1)
            acc1.fma(vs[q], xs[q]);
          else
            acc.fma(vs[q], xs[q]);
        }
      }
    }
    if (m.z & 512) {  // the segment's last chunk: fold the groups, store, start the next segment at zero
      acc.add(acc1);
      Acc<2> tot = acc;
#pragma unroll
      for (int h = 1; h < G; ++h) {
        const Acc<2> o = acc.shfl(lane_of(h, pc) & 31);
        if (g == 0) tot.add(o);
      }
      if (g == 0) {
        double* dst = m.y >= 0 ? (Y + (int64_t)m.y * ldy + 2 * pc) : (partial + (int64_t)(~m.y) * B + 2 * pc);
        tot.store(dst);
      }
      acc.zero();
      acc1.zero();
    }
    __syncwarp();  // every lane is done with the slot
  };
#pragma unroll
  for (int t = 0; t < D; ++t) fetch(t, t, n);  // (records 0 .. kRecAhead - 1 are already here)
  // unrolled by D: chunk i = i0 + u sits in slot u, and chunk i + D refills it
  for (int i0 = 0; i0 < n; i0 += D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int i = i0 + u;
      if (i < n) {
        consume(i, u);
        fetch(i + D, u, i + kRecAhead);
      }
    }
  }
  cp_async_wait<0>();
}

#ifndef SVDREC_HC_D
#define SVDREC_HC_D 4
#endif
#ifndef SVDREC_HC_W
#define SVDREC_HC_W 16
#endif
constexpr int kHcD = SVDREC_HC_D, kHcW = SVDREC_HC_W;
constexpr int kHcSmem = 226 * 1024;
constexpr int kHcTable = kHcSmem - kHcW * HcGeom<kHcD>::WARPB;  // bytes left for the hot rows

// The packed hot-first copy: every row stably partitioned into the entries
// of the nhot most rated items (id = popularity rank) and the rest (id =
// item), 16 B per entry; hot_cnt[r] = the row's hot entries.  One warp per
// row, two passes (count, then place with ballot prefixes).
__global__ void k_hot_pack(int64_t m, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           const double* __restrict__ values, const int32_t* __restrict__ rank, int nhot,
                           PackEnt* __restrict__ out, int32_t* __restrict__ hot_cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t r = w0; r < m; r += nw) {
    const int64_t a = indptr[r], b = indptr[r + 1];
    int64_t nh = 0;
    for (int64_t t0 = a; t0 < b; t0 += 32) {
      const int64_t t = t0 + lane;
      const bool hot = nhot > 0 && t < b && rank[indices[t]] < nhot;
      nh += __popc(__ballot_sync(0xffffffffu, hot));
    }
    if (lane == 0) hot_cnt[r] = (int32_t)nh;
    int64_t hrun = 0, crun = 0;
    for (int64_t t0 = a; t0 < b; t0 += 32) {
      const int64_t t = t0 + lane;
      const bool valid = t < b;
      int32_t c = 0, rk = 0;
      double v = 0.0;
      if (valid) {
        c = indices[t];
        rk = nhot > 0 ? rank[c] : 0;
        v = __ldcs(values + t);
      }
      const bool hot = nhot > 0 && valid && rk < nhot;
      const unsigned hm = __ballot_sync(0xffffffffu, hot), vm = __ballot_sync(0xffffffffu, valid);
      if (valid) {
        const int64_t pos = hot ? a + hrun + __popc(hm & lt) : a + nh + crun + __popc(vm & ~hm & lt);
        out[pos] = PackEnt{hot ? rk : c, 0, v};
      }
      hrun += __popc(hm);
      crun += __popc(vm & ~hm);
    }
  }
}

// The hot-set kernel's copy of a CSR: every row stably partitioned into the
// entries of the nhot most rated items (rank[item] < nhot) first and the
// rest after, each part in the row's order; index -(rank + 1) for hot
// entries, the item id otherwise.  One warp per row, two passes (count,
// then place with ballot prefixes).  Batches are then (nearly) all hot or
// all cold -- what the kernel needs; a full rank order is no faster.
__global__ void k_hot_partition(int64_t m, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                const double* __restrict__ values, const int32_t* __restrict__ rank, int nhot,
                                int32_t* __restrict__ out_idx, double* __restrict__ out_val) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t r = w0; r < m; r += nw) {
    const int64_t a = indptr[r], b = indptr[r + 1];
    int64_t nh = 0;
    for (int64_t t0 = a; t0 < b; t0 += 32) {
      const int64_t t = t0 + lane;
      const bool hot = t < b && rank[indices[t]] < nhot;
      nh += __popc(__ballot_sync(0xffffffffu, hot));
    }
    int64_t hrun = 0, crun = 0;
    for (int64_t t0 = a; t0 < b; t0 += 32) {
      const int64_t t = t0 + lane;
      const bool valid = t < b;
      int32_t c = 0, rk = 0;
      double v = 0.0;
      if (valid) {
        c = indices[t];
        rk = rank[c];
        v = __ldcs(values + t);
      }
      const bool hot = valid && rk < nhot;
      const unsigned hm = __ballot_sync(0xffffffffu, hot), vm = __ballot_sync(0xffffffffu, valid);
      if (valid) {
        const int64_t pos = hot ? a + hrun + __popc(hm & lt) : a + nh + crun + __popc(vm & ~hm & lt);
        out_idx[pos] = hot ? -(rk + 1) : c;
        out_val[pos] = v;
      }
      hrun += __popc(hm);
      crun += __popc(vm & ~hm);
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

extern "C" int svdrec_spmm_warps_per_sm(int32_t b) {
  if (b >= 1 && b <= 32 && b % 2 == 0) return 2 * kW2;  // two CTAs of kW2 warps
  if (b > 32 && b <= 64 && b % 4 == 0) {
    switch (b / 4) {
      case 9: return w4_warps(9);
      case 10: return w4_warps(10);
      case 11: return w4_warps(11);
      case 12: return w4_warps(12);
      case 13: return w4_warps(13);
      case 14: return w4_warps(14);
      case 15: return w4_warps(15);
      default: return w4_warps(16);
    }
  }
  return 16;  // plain kernel: the schedule is not used
}

namespace {
int run_fixup(int64_t nlong, const int32_t* d_long_row, const int32_t* d_long_slot0, const int32_t* d_long_slot1,
              const double* d_partial, double* d_Y, int64_t ldy, int32_t b, cudaStream_t s) {
  if (nlong <= 0) return 0;
  const int64_t tot = nlong * b;
  k_fixup<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(nlong, d_long_row, d_long_slot0, d_long_slot1, d_partial, d_Y,
                                                        ldy, b);
  return check_launch("spmm_fixup");
}
}  // namespace

extern "C" int svdrec_spmm(int64_t nseg, const int32_t* d_seg_row, const int64_t* d_seg_begin,
                           const int64_t* d_seg_end, const int32_t* d_seg_slot, const int32_t* d_indices,
                           const double* d_values, const double* d_X, int64_t ldx, int64_t xrows, double* d_Y,
                           int64_t ldy, int32_t b, int64_t nlong, const int32_t* d_long_row,
                           const int32_t* d_long_slot0, const int32_t* d_long_slot1, int64_t nwarp,
                           const int32_t* d_warp_seg, const int32_t* d_warp_chunk, const void* d_chunks,
                           const int32_t* d_slot_long, int32_t* d_long_done, double* d_partial, void* stream) {
  SVDREC_ARG(b >= 1 && ldx >= b && ldy >= b && nseg >= 0 && nlong >= 0, "spmm: bad arguments b=%d", b);
  SVDREC_ARG(!d_long_done || d_slot_long, "spmm: the in-kernel fix-up needs the slot -> split-row map");
  if (nseg == 0) return 0;
  cudaStream_t s = as_stream(stream);
  const bool vec2 = (b % 2 == 0) && (ldx % 2 == 0) && (ldy % 2 == 0) &&
                    ((reinterpret_cast<uintptr_t>(d_X) | reinterpret_cast<uintptr_t>(d_Y) |
                      reinterpret_cast<uintptr_t>(d_partial)) %
                         16 ==
                     0);
  // SVDREC_SPMM_KIND=0 forces the plain kernel (A/B measurements)
  static const int kind = getenv("SVDREC_SPMM_KIND") ? atoi(getenv("SVDREC_SPMM_KIND")) : 1;
  const bool sched = vec2 && nwarp > 0 && kind != 0 && xrows < (1ll << 31);
  int rc = 0;
  if (sched && b <= 32 && d_warp_chunk && d_chunks) {
    const FixArgs fix{d_slot_long, d_long_row, d_long_slot0, d_long_slot1, nlong > 0 ? d_long_done : nullptr};
    rc = pipe_dispatch(b, xrows, nwarp, d_warp_chunk, d_chunks, d_indices, d_values, d_X, ldx, d_Y, ldy, d_partial,
                       fix, s);
    if (rc || fix.done) return rc;  // the split rows were added inside the kernel
  } else if (sched && b > 32 && b <= 64 && b % 4 == 0 && ldx % 4 == 0 && d_warp_seg) {
    rc = tma_dispatch4(b, xrows, nwarp, d_warp_seg, d_seg_row, d_seg_begin, d_seg_end, d_seg_slot, d_indices,
                       d_values, d_X, ldx, d_Y, ldy, d_partial, s);
  } else {
    const int vec = vec2 ? 2 : 1;
    const int lanes_needed = (b + vec - 1) / vec;
    const int lpn = lanes_needed >= 32 ? 32 : lanes_needed;
    const int npw = 32 / lpn;
    const int tb = 256;
    int64_t grid = (nseg * 32 + tb - 1) / tb;
    const int64_t cap = (int64_t)sm_count() * 8 * 64;
    if (grid > cap) grid = cap;
    if (vec2)
      k_spmm<2><<<(unsigned)grid, tb, 0, s>>>(nseg, d_seg_row, d_seg_begin, d_seg_end, d_seg_slot, d_indices,
                                               d_values, d_X, ldx, d_Y, ldy, b, d_partial, lpn, npw);
    else
      k_spmm<1><<<(unsigned)grid, tb, 0, s>>>(nseg, d_seg_row, d_seg_begin, d_seg_end, d_seg_slot, d_indices,
                                               d_values, d_X, ldx, d_Y, ldy, b, d_partial, lpn, npw);
    rc = check_launch("spmm");
  }
  if (rc) return rc;
  return run_fixup(nlong, d_long_row, d_long_slot0, d_long_slot1, d_partial, d_Y, ldy, b, s);
}

extern "C" int svdrec_spmm_hot_rows(int32_t b) {
  // widths the register-gather hot-set kernel serves: 32 < b <= 64 with
  // b % 4 == 0 (4 doubles per lane); even b <= 32 run k_spmm_hc
  if (b <= 32 || b > 64 || b % 4) return 0;
  // one 512-thread CTA per SM; the hot rows fill the 227 KB opt-in
  return (int)((226 * 1024 - kHotWarps * 2 * kTabSlots * (int)sizeof(TabEnt)) / (8 * b));
}

extern "C" int svdrec_spmm_hot_partition(int64_t m, const int64_t* d_indptr, const int32_t* d_indices,
                                         const double* d_values, const int32_t* d_rank, int32_t nhot,
                                         int32_t* d_out_indices, double* d_out_values, void* stream) {
  SVDREC_ARG(m >= 0 && nhot >= 0, "spmm_hot_partition: bad arguments");
  if (m == 0) return 0;
  const int64_t grid = min64((m + 7) / 8, (int64_t)sm_count() * 16);
  k_hot_partition<<<(unsigned)grid, 256, 0, as_stream(stream)>>>(m, d_indptr, d_indices, d_values, d_rank, nhot,
                                                                  d_out_indices, d_out_values);
  return check_launch("spmm_hot_partition");
}

extern "C" int svdrec_spmm_hc_warps_per_sm(void) { return kHcW; }

extern "C" int svdrec_spmm_hc_rows(int32_t b) {
  if (b < 2 || b > 32 || b % 2) return 0;
  return kHcTable / (8 * b);
}

extern "C" int svdrec_spmm_hot_pack(int64_t m, const int64_t* d_indptr, const int32_t* d_indices,
                                    const double* d_values, const int32_t* d_rank, int32_t nhot, void* d_out,
                                    int32_t* d_hot_cnt, void* stream) {
  SVDREC_ARG(m >= 0 && nhot >= 0 && d_hot_cnt && (nhot == 0 || d_rank), "spmm_hot_pack: bad arguments");
  if (m == 0) return 0;
  const int64_t grid = min64((m + 7) / 8, (int64_t)sm_count() * 16);
  k_hot_pack<<<(unsigned)grid, 256, 0, as_stream(stream)>>>(m, d_indptr, d_indices, d_values, d_rank, nhot,
                                                             reinterpret_cast<PackEnt*>(d_out), d_hot_cnt);
  return check_launch("spmm_hot_pack");
}

extern "C" int svdrec_spmm_hc(int64_t nseg, const void* d_entries, const double* d_X, int64_t ldx, int64_t x_rows,
                              const int32_t* d_hot_items, int32_t nhot, double* d_Y, int64_t ldy, int32_t b,
                              int64_t nlong, const int32_t* d_long_row, const int32_t* d_long_slot0,
                              const int32_t* d_long_slot1, int64_t nwarp, const int32_t* d_warp_chunk,
                              const void* d_chunks, double* d_partial, void* stream) {
  SVDREC_ARG(svdrec_spmm_hc_rows(b) > 0 && ldx % 2 == 0 && ldy % 2 == 0 && ldx >= b && ldy >= b,
             "spmm_hc: needs even b <= 32 and 16-B aligned rows (b=%d)", b);
  SVDREC_ARG(nhot >= 0 && nhot <= svdrec_spmm_hc_rows(b) && nhot <= x_rows,
             "spmm_hc: %d hot rows exceed shared memory", nhot);
  SVDREC_ARG(nwarp > 0 && d_warp_chunk && d_chunks, "spmm_hc: needs a chunk plan (svdrec_spmm_hc_warps_per_sm)");
  SVDREC_ARG(x_rows * (ldx / 2) < (1ll << 31), "spmm_hc: X too large for 32-bit row offsets");
  SVDREC_ARG(((reinterpret_cast<uintptr_t>(d_X) | reinterpret_cast<uintptr_t>(d_Y) |
               reinterpret_cast<uintptr_t>(d_partial) | reinterpret_cast<uintptr_t>(d_entries)) % 16) == 0,
             "spmm_hc: operands must be 16-B aligned");
  if (nseg == 0) return 0;
  cudaStream_t s = as_stream(stream);
  const size_t smem = (size_t)kHcW * HcGeom<kHcD>::WARPB + (size_t)nhot * b * sizeof(double);
  const int64_t grid = (nwarp + kHcW - 1) / kHcW;
  switch (b / 2) {
#define SVDREC_HC(PP)                                                                                          \
  case PP:                                                                                                     \
    SVDREC_CUDA(smem_attr_once(k_spmm_hc<PP, kHcD, kHcW>, kHcSmem));                                            \
    k_spmm_hc<PP, kHcD, kHcW><<<(unsigned)grid, kHcW * 32, smem, s>>>(                                          \
        nwarp, d_warp_chunk, reinterpret_cast<const int4*>(d_chunks), reinterpret_cast<const PackEnt*>(d_entries), \
        d_X, ldx, d_hot_items, nhot, d_Y, ldy, d_partial);                                                     \
    break;
    SVDREC_HC(1) SVDREC_HC(2) SVDREC_HC(3) SVDREC_HC(4) SVDREC_HC(5) SVDREC_HC(6) SVDREC_HC(7) SVDREC_HC(8)
    SVDREC_HC(9) SVDREC_HC(10) SVDREC_HC(11) SVDREC_HC(12) SVDREC_HC(13) SVDREC_HC(14) SVDREC_HC(15) SVDREC_HC(16)
#undef SVDREC_HC
    default: return SVDREC_E_ARG;
  }
  const int rc = check_launch("spmm_hc");
  if (rc) return rc;
  return run_fixup(nlong, d_long_row, d_long_slot0, d_long_slot1, d_partial, d_Y, ldy, b, s);
}

extern "C" int svdrec_spmm_hot(int64_t nseg, const int32_t* d_seg_row, const int64_t* d_seg_begin,
                               const int64_t* d_seg_end, const int32_t* d_seg_slot, const int32_t* d_hidx,
                               const double* d_hval, const double* d_X, int64_t ldx, int64_t x_rows,
                               const int32_t* d_hot_items,
                               int32_t nhot, double* d_Y, int64_t ldy, int32_t b, int64_t nlong,
                               const int32_t* d_long_row, const int32_t* d_long_slot0, const int32_t* d_long_slot1,
                               int64_t nwarp, const int32_t* d_warp_seg, double* d_partial, void* stream) {
  SVDREC_ARG(svdrec_spmm_hot_rows(b) > 0 && ldx % 2 == 0 && ldy % 2 == 0 && ldx >= b && ldy >= b,
             "spmm_hot: needs 32 < b <= 64, b %% 4 == 0, and 16-B aligned rows (b=%d)", b);
  SVDREC_ARG(nhot >= 0 && nhot <= svdrec_spmm_hot_rows(b), "spmm_hot: %d hot rows exceed shared memory", nhot);
  SVDREC_ARG(nwarp > 0 && d_warp_seg, "spmm_hot: needs a warp schedule (16 warps per SM)");
  SVDREC_ARG(x_rows * (ldx / 2) < (1ll << 31), "spmm_hot: X too large for 32-bit row offsets");
  SVDREC_ARG(((reinterpret_cast<uintptr_t>(d_X) | reinterpret_cast<uintptr_t>(d_Y) |
               reinterpret_cast<uintptr_t>(d_partial)) % 16) == 0, "spmm_hot: operands must be 16-B aligned");
  if (nseg == 0) return 0;
  cudaStream_t s = as_stream(stream);
  const size_t smem = (size_t)nhot * b * sizeof(double);
  const int64_t grid = (nwarp + 15) / 16;
#define SVDREC_HOT(PP, VV)                                                                                 \
  case PP:                                                                                                 \
    SVDREC_CUDA(smem_attr_once(k_spmm_hot<PP, (PP < 8 ? PP : 8), VV>,                                     \
                               226 * 1024 - kHotWarps * 2 * kTabSlots * (int)sizeof(TabEnt)));           \
    k_spmm_hot<PP, (PP < 8 ? PP : 8), VV><<<(unsigned)grid, 512, smem, s>>>(                               \
        nwarp, d_warp_seg, d_seg_row, d_seg_begin, d_seg_end, d_seg_slot, d_hidx, d_hval, d_X, ldx,        \
        d_hot_items, nhot, d_Y, ldy, d_partial);                                                           \
    break;
  {
    switch (b / 4) {
      SVDREC_HOT(9, 4)
      SVDREC_HOT(10, 4)
      SVDREC_HOT(11, 4)
      SVDREC_HOT(12, 4)
      SVDREC_HOT(13, 4)
      SVDREC_HOT(14, 4)
      SVDREC_HOT(15, 4)
      SVDREC_HOT(16, 4)
      default:
        return SVDREC_E_ARG;
    }
  }
#undef SVDREC_HOT
  int rc = check_launch("spmm_hot");
  if (rc) return rc;
  if (nlong > 0) {
    const int64_t tot = nlong * b;
    k_fixup<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(nlong, d_long_row, d_long_slot0, d_long_slot1, d_partial,
                                                          d_Y, ldy, b);
    rc = check_launch("spmm_fixup");
  }
  return rc;
}

extern "C" int svdrec_spmm_x32(int64_t nseg, const int32_t* d_seg_row, const int64_t* d_seg_begin,
                               const int64_t* d_seg_end, const int32_t* d_seg_slot, const int32_t* d_indices,
                               const double* d_values, const float* d_X, int64_t ldx, int64_t xrows, double* d_Y,
                               int64_t ldy, int32_t b, int64_t nlong, const int32_t* d_long_row,
                               const int32_t* d_long_slot0, const int32_t* d_long_slot1, int64_t nwarp,
                               const int32_t* d_warp_seg, const int32_t* d_warp_chunk, const void* d_chunks,
                               const int32_t* d_slot_long, int32_t* d_long_done, double* d_partial, void* stream) {
  SVDREC_ARG(b >= 4 && b <= 64 && b % 4 == 0 && ldx >= b && ldx % 4 == 0 && ldy >= b && ldy % 2 == 0 && nseg >= 0 &&
                 nlong >= 0 && (b <= 32 || ldy % 4 == 0),
             "spmm_x32: needs b in {4, 8, ..., 64} and 16-B aligned rows (b=%d)", b);
  SVDREC_ARG(nwarp > 0 && (b <= 32 ? (d_warp_chunk && d_chunks) : d_warp_seg != nullptr),
             "spmm_x32: needs a schedule (chunk plan for b <= 32, warp ranges above)");
  SVDREC_ARG(((reinterpret_cast<uintptr_t>(d_X) | reinterpret_cast<uintptr_t>(d_Y) |
               reinterpret_cast<uintptr_t>(d_partial)) % 16) == 0,
             "spmm_x32: operands must be 16-B aligned");
  if (nseg == 0) return 0;
  cudaStream_t s = as_stream(stream);
  const bool infix = b <= 32 && nlong > 0 && d_long_done && d_slot_long;
  const FixArgs fix{d_slot_long, d_long_row, d_long_slot0, d_long_slot1, infix ? d_long_done : nullptr};
  const int rc = b <= 32 ? pipe_dispatch_f32(b, xrows, nwarp, d_warp_chunk, d_chunks, d_indices, d_values, d_X, ldx,
                                             d_Y, ldy, d_partial, fix, s)
                         : tma_dispatch4_f32(b, xrows, nwarp, d_warp_seg, d_seg_row, d_seg_begin, d_seg_end,
                                             d_seg_slot, d_indices, d_values, d_X, ldx, d_Y, ldy, d_partial, s);
  if (rc || infix) return rc;
  return run_fixup(nlong, d_long_row, d_long_slot0, d_long_slot1, d_partial, d_Y, ldy, b, s);
}

extern "C" int svdrec_spmm_x32_warps_per_sm(int32_t b) {
  if (b > 32 && b <= 64 && b % 4 == 0) {
    switch (b / 4) {
      case 9: return w4f_warps(9);
      case 10: return w4f_warps(10);
      case 11: return w4f_warps(11);
      case 12: return w4f_warps(12);
      case 13: return w4f_warps(13);
      case 14: return w4f_warps(14);
      case 15: return w4f_warps(15);
      default: return w4f_warps(16);
    }
  }
  return 16;  // two CTAs of 8 warps
}
