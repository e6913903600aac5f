// Device-side ingest: stable counting-sort transpose of a CSR.
//
// Builds the two derived layouts the hot path needs from the uploaded CSR
// of A (reference sparse.py keeps only A; its ``A.T @ X`` is scipy's
// transposed product, linalg.py:141-158):
//   * the CSR of A.T (item rows, users ascending) for A.T @ X;
//   * the popularity-ranked CSR for the CF scoring kernel (user rows, items
//     relabelled by popularity rank and stored in rank order) -- the
//     transpose of A.T with its rows taken in rank order.
// Both are "transpose the rows of a CSR, taken in a given order": output
// row c lists, in processing order, every input row r holding column c.
//
// No sort.  k_tr_expand lays out, per processing position, the input row
// (in processing order) and the entry's index (one warp per row, coalesced
// writes).  Then, per range of at most kBins output rows (columns of the
// input):
//   k_tr_hist    one CTA per contiguous slice of the processing positions:
//                column histogram in shared memory -> hist[c][cta];
//   k_tr_offsets one thread per column: off[c][cta] = out_indptr[c] + the
//                column's count in the slices before cta (fixed order);
//   k_tr_scatter each CTA re-walks its slice with its offsets in shared
//                memory.  An input row's columns are distinct, so entries
//                of one input row never collide: each 1024-entry tile is
//                processed input row by input row (one CTA barrier per
//                row), which keeps the output stable (processing order)
//                and deterministic.  The next tile's loads are in flight
//                while a tile is scattered (two-deep register pipeline).
// Traffic: the entries are read twice and written once (scattered); the
// per-(column, slice) tables are n x slices int32 (transient).
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace svdrec {
namespace {

constexpr int kTrThreads = 1024;
constexpr int kBins = 50 * 1024;  // output rows per range (int32 bins, 200 KB of shared memory)

__device__ __forceinline__ void slice(int64_t total, int64_t& t0, int64_t& t1) {
  t0 = total * (int64_t)blockIdx.x / gridDim.x;
  t1 = total * ((int64_t)blockIdx.x + 1) / gridDim.x;
}

// row_p[p] = processing row of position p; src_e[p] = its entry index
__global__ void k_tr_expand(int64_t nrows, const int64_t* __restrict__ pptr, const int64_t* __restrict__ indptr,
                            const int32_t* __restrict__ perm, int32_t* __restrict__ row_p,
                            int32_t* __restrict__ src_e) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = w0; q < nrows; q += nw) {
    const int64_t a = pptr[q], b = pptr[q + 1];
    const int64_t e0 = indptr[perm ? (int64_t)perm[q] : q];
    for (int64_t p = a + lane; p < b; p += 32) {
      row_p[p] = (int32_t)q;
      src_e[p] = (int32_t)(e0 + (p - a));
    }
  }
}

__global__ void __launch_bounds__(kTrThreads) k_tr_hist(const int32_t* __restrict__ src_e,
                                                         const int32_t* __restrict__ indices, int64_t total,
                                                         int32_t c0, int32_t nb, int32_t* __restrict__ hist) {
  extern __shared__ int32_t bins[];
  for (int c = threadIdx.x; c < nb; c += blockDim.x) bins[c] = 0;
  __syncthreads();
  int64_t t0, t1;
  slice(total, t0, t1);
#pragma unroll 4
  for (int64_t p = t0 + threadIdx.x; p < t1; p += blockDim.x) {
    const int32_t c = indices[__ldcs(src_e + p)] - c0;
    if ((uint32_t)c < (uint32_t)nb) atomicAdd(&bins[c], 1);
  }
  __syncthreads();
  const int64_t g = gridDim.x;
  for (int c = threadIdx.x; c < nb; c += blockDim.x) hist[(int64_t)c * g + blockIdx.x] = bins[c];
}

// per column: running sum over the slices, from the column's output start
__global__ void k_tr_offsets(int32_t nb, int32_t g, const int64_t* __restrict__ out_indptr, int32_t c0,
                             int32_t* __restrict__ hist) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nb) return;
  int64_t run = out_indptr[c0 + c];
  int32_t* h = hist + c * g;
  for (int i = 0; i < g; ++i) {
    const int32_t n = h[i];
    h[i] = (int32_t)run;
    run += n;
  }
}

// column totals of the histogram (for the output row pointers)
__global__ void k_tr_totals(int32_t nb, int32_t g, const int32_t* __restrict__ hist, int64_t* __restrict__ counts) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nb) return;
  int64_t s = 0;
  for (int i = 0; i < g; ++i) s += hist[c * g + i];
  counts[c] = s;
}

// relabel: output column id = the input row's processing position (rank)
// instead of its index
template <bool RELABEL>
__global__ void __launch_bounds__(kTrThreads) k_tr_scatter(const int32_t* __restrict__ row_p,
                                                            const int32_t* __restrict__ src_e,
                                                            const int32_t* __restrict__ perm,
                                                            const int32_t* __restrict__ indices,
                                                            const double* __restrict__ values, int64_t total,
                                                            int32_t c0, int32_t nb, const int32_t* __restrict__ hist,
                                                            int32_t* __restrict__ out_idx,
                                                            double* __restrict__ out_val) {
  extern __shared__ int32_t off[];
  __shared__ int32_t s_rows[2][2];
  const int64_t g = gridDim.x;
  for (int c = threadIdx.x; c < nb; c += blockDim.x) off[c] = hist[(int64_t)c * g + blockIdx.x];
  int64_t t0, t1;
  slice(total, t0, t1);
  const int T = blockDim.x;
  // two-deep pipeline: (row, entry) of tile i+2 and (column, value) of
  // tile i+1 are loading while tile i is scattered
  auto load_re = [&](int64_t p0, int32_t& r, int32_t& e) {
    const int64_t p = p0 + threadIdx.x;
    r = -1;
    e = -1;
    if (p < t1) {
      r = __ldcs(row_p + p);
      e = __ldcs(src_e + p);
    }
  };
  auto load_cv = [&](int32_t e, int32_t& c, double& v) {
    c = -1;
    v = 0.0;
    if (e >= 0) {
      c = __ldcs(indices + e) - c0;
      v = __ldcs(values + e);
    }
  };
  int32_t r_cur, e_cur, r_nx, e_nx, c_cur;
  double v_cur;
  load_re(t0, r_cur, e_cur);
  load_re(t0 + T, r_nx, e_nx);
  load_cv(e_cur, c_cur, v_cur);
  __syncthreads();  // offsets staged
  int par = 0;
  for (int64_t p0 = t0; p0 < t1; p0 += T) {
    // the tile's first and last rows
    if (threadIdx.x == 0) s_rows[par][0] = r_cur;
    if (p0 + threadIdx.x == min64(p0 + T, t1) - 1) s_rows[par][1] = r_cur;
    int32_t c_nx;
    double v_nx;
    load_cv(e_nx, c_nx, v_nx);  // tile i+1's columns / values
    int32_t r_nx2, e_nx2;
    load_re(p0 + 2 * T, r_nx2, e_nx2);  // tile i+2's rows / entries
    __syncthreads();
    const int32_t q = s_rows[par][0], ql = s_rows[par][1];
    for (int32_t rr = q; rr <= ql; ++rr) {
      if (r_cur == rr && (uint32_t)c_cur < (uint32_t)nb) {
        const int32_t pos = off[c_cur];
        off[c_cur] = pos + 1;
        out_idx[pos] = RELABEL ? rr : (perm ? perm[rr] : rr);
        out_val[pos] = v_cur;
      }
      __syncthreads();
    }
    r_cur = r_nx;
    c_cur = c_nx;
    v_cur = v_nx;
    r_nx = r_nx2;
    e_nx = e_nx2;
    par ^= 1;
  }
}

// Ranked rows without a sort: every row's entries relabelled by the item
// rank table and reordered by rank.  Ranks are distinct within a row, so
// an entry's position in its row is the number of the row's ranks below
// its own: one warp per row marks the row's ranks in a shared-memory
// bitset over all n ranks, scans the words' popcounts, and reads each
// position off the bitset (O(n / 32 + deg) per row, coalesced row-local
// writes).  n <= kRankBits.
constexpr int kRankWarps = 8;
constexpr int kRankBits = 64 * 1024;
constexpr int kRankWords = kRankBits / 32;

__global__ void __launch_bounds__(kRankWarps * 32) k_rank_rows(int64_t m, int32_t n, const int64_t* __restrict__ indptr,
                                                                const int32_t* __restrict__ indices,
                                                                const double* __restrict__ values,
                                                                const int32_t* __restrict__ rank,
                                                                int32_t* __restrict__ out_idx,
                                                                double* __restrict__ out_val) {
  extern __shared__ uint32_t rs_mem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nwords = (n + 31) >> 5;
  uint32_t* bits = rs_mem + (size_t)wid * 2 * nwords;
  uint32_t* pref = bits + nwords;  // exclusive prefix popcount per word
  const int64_t gw = (int64_t)blockIdx.x * kRankWarps + wid;
  const int64_t nw = (int64_t)gridDim.x * kRankWarps;
  for (int i = lane; i < nwords; i += 32) bits[i] = 0u;
  __syncwarp();
  for (int64_t r = gw; r < m; r += nw) {
    const int64_t a = indptr[r], b = indptr[r + 1];
    // (the three passes over the row are unrolled so that a typical row's
    // index and rank loads are all in flight at once)
#pragma unroll 4
    for (int64_t t = a + lane; t < b; t += 32) {
      const int32_t k = rank[indices[t]];
      atomicOr(&bits[k >> 5], 1u << (k & 31));
    }
    __syncwarp();
    // prefix popcount over the words: each lane a contiguous stretch
    const int per = (nwords + 31) >> 5;
    const int w0 = lane * per, w1 = min(nwords, w0 + per);
    int sum = 0;
    for (int i = w0; i < w1; ++i) sum += __popc(bits[i]);
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int run = incl - sum;
    for (int i = w0; i < w1; ++i) {
      pref[i] = (uint32_t)run;
      run += __popc(bits[i]);
    }
    __syncwarp();
#pragma unroll 4
    for (int64_t t = a + lane; t < b; t += 32) {
      const int32_t k = rank[indices[t]];
      const int pos = (int)pref[k >> 5] + __popc(bits[k >> 5] & ((1u << (k & 31)) - 1u));
      out_idx[a + pos] = k;
      out_val[a + pos] = values[t];
    }
    __syncwarp();
#pragma unroll 4
    for (int64_t t = a + lane; t < b; t += 32) bits[rank[indices[t]] >> 5] = 0u;  // clear only what was set
    __syncwarp();
  }
}

// Exclusive scan of int64 (n values) in three launches: per-tile sums,
// one CTA scanning the tile sums, per-tile scan plus offset.  Optional
// total written at out[n].
constexpr int kScanT = 1024;
constexpr int kScanPer = 8;  // values per thread per tile

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* sh, int64_t* total) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  int64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) sh[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int nwarp = blockDim.x >> 5;
    int64_t x = lane < nwarp ? sh[lane] : 0;
    int64_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += u;
    }
    if (lane < nwarp) sh[lane] = xi - x;
    if (lane == nwarp - 1) sh[32] = xi;
  }
  __syncthreads();
  const int64_t r = sh[wid] + incl - v;
  if (total) *total = sh[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanT) k_scan_tiles(int64_t n, const int64_t* __restrict__ in,
                                                       int64_t* __restrict__ tile_sum) {
  __shared__ int64_t sh[33];
  const int64_t base = (int64_t)blockIdx.x * kScanT * kScanPer + (int64_t)threadIdx.x * kScanPer;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i)
    if (base + i < n) s += in[base + i];
  int64_t tot;
  block_excl_scan(s, sh, &tot);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanT) k_scan_sums(int64_t ntiles, int64_t* __restrict__ tile_sum,
                                                      int64_t* __restrict__ grand) {
  __shared__ int64_t sh[33];
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < ntiles; b0 += kScanT) {
    const int64_t i = b0 + threadIdx.x;
    const int64_t v = i < ntiles ? tile_sum[i] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan(v, sh, &tot);
    if (i < ntiles) tile_sum[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && grand) *grand = carry;
}

__global__ void __launch_bounds__(kScanT) k_scan_apply(int64_t n, const int64_t* __restrict__ in,
                                                       const int64_t* __restrict__ tile_off,
                                                       int64_t* __restrict__ out) {
  __shared__ int64_t sh[33];
  const int64_t base = (int64_t)blockIdx.x * kScanT * kScanPer + (int64_t)threadIdx.x * kScanPer;
  int64_t v[kScanPer];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    v[i] = base + i < n ? in[base + i] : 0;
    s += v[i];
  }
  int64_t run = tile_off[blockIdx.x] + block_excl_scan(s, sh, nullptr);
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
}

// SpMM row-segment plan (sparse.py segment_plan / warp_plan): rows cut
// into segments of <= seg_max entries; split rows own consecutive partial
// slots (numbered in row order) and a fix-up record; the warp schedule
// cuts the segments into nwarp contiguous ranges of about equal cost
// (entries + 16 per segment).
__global__ void k_seg_count(int64_t m, const int64_t* __restrict__ indptr, int seg_max, int64_t* __restrict__ nps,
                            int64_t* __restrict__ split_nps, int64_t* __restrict__ is_split) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const int64_t d = indptr[r + 1] - indptr[r];
  const int64_t n = d <= seg_max ? 1 : (d + seg_max - 1) / seg_max;
  nps[r] = n;
  split_nps[r] = n > 1 ? n : 0;
  is_split[r] = n > 1 ? 1 : 0;
}

__global__ void k_seg_emit(int64_t m, const int64_t* __restrict__ indptr, int seg_max,
                           const int64_t* __restrict__ first, const int64_t* __restrict__ sbase,
                           const int64_t* __restrict__ lidx, int32_t* __restrict__ seg_row,
                           int64_t* __restrict__ seg_begin, int64_t* __restrict__ seg_end,
                           int32_t* __restrict__ seg_slot, int32_t* __restrict__ long_row,
                           int32_t* __restrict__ long_s0, int32_t* __restrict__ long_s1) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const int64_t a = indptr[r], e = indptr[r + 1];
  const int64_t d = e - a;
  const int64_t n = d <= seg_max ? 1 : (d + seg_max - 1) / seg_max;
  const int64_t f = first[r];
  for (int64_t j = 0; j < n; ++j) {
    const int64_t b = a + j * seg_max;
    seg_row[f + j] = (int32_t)r;
    seg_begin[f + j] = b;
    seg_end[f + j] = min64(b + seg_max, e);
    seg_slot[f + j] = n > 1 ? (int32_t)(sbase[r] + j) : -1;
  }
  if (n > 1) {
    const int64_t l = lidx[r];
    long_row[l] = (int32_t)r;
    long_s0[l] = (int32_t)sbase[r];
    long_s1[l] = (int32_t)(sbase[r] + n);
  }
}

__global__ void k_seg_cost(int64_t nseg, const int64_t* __restrict__ seg_begin, const int64_t* __restrict__ seg_end,
                           int seg_cost, int64_t* __restrict__ cost) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nseg) return;
  const int64_t d = seg_end[j] - seg_begin[j];
  // seg_cost < 0: the chunk kernels' cost -- whole 32-entry chunks (at least
  // one) plus -seg_cost per segment (its fold and store)
  cost[j] = seg_cost >= 0 ? d + seg_cost : (d <= 32 ? 32 : ((d + 31) >> 5) << 5) - seg_cost;
}

// excl: exclusive scan of the segment costs, total = their sum; cut i (1 <=
// i < nwarp) = 1 + the first j whose inclusive cost >= i * (total / nwarp)
// (float64, numpy searchsorted 'left'), capped at nseg
__global__ void k_warp_cuts(int64_t nseg, int64_t nwarp, const int64_t* __restrict__ excl,
                            const int64_t* __restrict__ d_total, int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > nwarp) return;
  if (i == 0 || i == nwarp || nseg == 0) {
    out[i] = i == 0 ? 0 : (int32_t)nseg;
    return;
  }
  const int64_t total = *d_total;
  const double target = (double)i * ((double)total / (double)nwarp);
  int64_t lo = 0, hi = nseg;  // first j in [0, nseg) with incl[j] >= target, else nseg
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int64_t incl = mid + 1 < nseg ? excl[mid + 1] : total;
    if ((double)incl >= target)
      hi = mid;
    else
      lo = mid + 1;
  }
  out[i] = (int32_t)min64(lo + 1, nseg);
}

// Chunk records of the pipelined SpMMs (csrc/spmm.cu k_spmm_pipe /
// k_spmm_hc): every segment cut into chunks of <= 32 nonzeros (an empty row
// is one chunk with no entries), one 16-B record each: x / w = low / high
// word of the first entry's offset, y = the output row (>= 0) or ~slot of a
// split row's partial sum, z = entries | first chunk of its segment << 8 |
// last << 9 | hot << 10.  With hot_cnt (the hot-first copy of the CSR: row r
// holds its hot_cnt[r] shared-memory-resident entries first) no chunk
// straddles a row's hot / cold boundary and each carries its kind.
__device__ __forceinline__ int64_t chunks_of(int64_t d) { return (d + 31) >> 5; }

__device__ __forceinline__ int64_t hot_end(int64_t a, int64_t e, int32_t row, const int64_t* __restrict__ indptr,
                                           const int32_t* __restrict__ hot_cnt) {
  if (!hot_cnt) return a;
  const int64_t hb = indptr[row] + hot_cnt[row];
  return hb < a ? a : (hb > e ? e : hb);
}

__global__ void k_chunk_count(int64_t nseg, const int32_t* __restrict__ seg_row,
                              const int64_t* __restrict__ seg_begin, const int64_t* __restrict__ seg_end,
                              const int64_t* __restrict__ indptr, const int32_t* __restrict__ hot_cnt,
                              int64_t* __restrict__ cnt) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nseg) return;
  const int64_t a = seg_begin[j], e = seg_end[j];
  const int64_t h = hot_end(a, e, seg_row[j], indptr, hot_cnt);
  const int64_t n = chunks_of(h - a) + chunks_of(e - h);
  cnt[j] = n ? n : 1;
}

__global__ void k_chunk_emit(int64_t nseg, const int32_t* __restrict__ seg_row, const int64_t* __restrict__ seg_begin,
                             const int64_t* __restrict__ seg_end, const int32_t* __restrict__ seg_slot,
                             const int64_t* __restrict__ indptr, const int32_t* __restrict__ hot_cnt,
                             const int64_t* __restrict__ cbase, int4* __restrict__ recs) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nseg) return;
  const int64_t a = seg_begin[j], e = seg_end[j];
  const int64_t h = hot_end(a, e, seg_row[j], indptr, hot_cnt);
  const int64_t nh = chunks_of(h - a), nc = chunks_of(e - h);
  const int32_t slot = seg_slot[j];
  const int32_t dst = slot < 0 ? seg_row[j] : ~slot;
  int4* out = recs + cbase[j];
  if (nh + nc == 0) {  // an empty row: one chunk without entries
    out[0] = make_int4(0, dst, 256 | 512, 0);
    return;
  }
  for (int64_t c = 0; c < nh + nc; ++c) {
    const bool hot = c < nh;
    const int64_t o = hot ? a + 32 * c : h + 32 * (c - nh);
    const int nv = (int)min64(32, (hot ? h : e) - o);
    out[c] = make_int4((int)(uint32_t)(o & 0xffffffffll), dst,
                       nv | (c == 0 ? 256 : 0) | (c == nh + nc - 1 ? 512 : 0) | (hot ? 1024 : 0),
                       (int)(uint32_t)(o >> 32));
  }
}

// warp_chunk[w] = first chunk of warp w's segment range (w = nwarp: the total)
__global__ void k_warp_chunks(int64_t nwarp, const int32_t* __restrict__ warp_seg, int64_t nseg,
                              const int64_t* __restrict__ cbase, const int64_t* __restrict__ total,
                              int32_t* __restrict__ warp_chunk) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w > nwarp) return;
  const int64_t sgm = warp_seg[w];
  warp_chunk[w] = (int32_t)(sgm < nseg ? cbase[sgm] : *total);
}

}  // namespace
}  // namespace svdrec

using namespace svdrec;

namespace svdrec {
// exclusive scan of n int64 values (in may alias out); total -> *d_total
// (nullable).  Scratch for the tile sums: a small cached device buffer.
int scan_i64(int64_t n, const int64_t* d_in, int64_t* d_out, int64_t* d_total, cudaStream_t s, int* launches) {
  const int64_t per_tile = (int64_t)kScanT * kScanPer;
  const int64_t ntiles = (n + per_tile - 1) / per_tile;
  // tile sums: a grow-only buffer per (device, stream), allocated and freed
  // stream-ordered on that stream, so scans issued concurrently on two
  // streams (e.g. SpMM plans beside the scoring plan) never share scratch
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<int64_t*, int64_t>> bufs;
  int dev = 0;
  cudaGetDevice(&dev);
  int64_t* buf = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = bufs[{dev, s}];
    if (ntiles + 1 > slot.second) {
      if (slot.first) cudaFreeAsync(slot.first, s);
      const int64_t cap = ntiles + 1 > 4096 ? ntiles + 1 : 4096;
      cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&slot.first), (size_t)cap * sizeof(int64_t), s);
      if (e != cudaSuccess) {
        slot = {nullptr, 0};
        return (int)e;
      }
      slot.second = cap;
    }
    buf = slot.first;
  }
  if (n > 0) {
    k_scan_tiles<<<(unsigned)ntiles, kScanT, 0, s>>>(n, d_in, buf);
    k_scan_sums<<<1, kScanT, 0, s>>>(ntiles, buf, d_total);
    k_scan_apply<<<(unsigned)ntiles, kScanT, 0, s>>>(n, d_in, buf, d_out);
    *launches += 3;
  } else if (d_total) {
    cudaMemsetAsync(d_total, 0, sizeof(int64_t), s);
  }
  return (int)cudaGetLastError();
}
}  // namespace svdrec

extern "C" int svdrec_rank_rows(int64_t m, int32_t n, const int64_t* d_indptr, const int32_t* d_indices,
                                const double* d_values, const int32_t* d_rank, int32_t* d_out_indices,
                                double* d_out_values, void* stream) {
  SVDREC_ARG(m >= 0 && n >= 1 && n <= kRankBits, "rank_rows: needs 1 <= n <= %d (n=%d)", kRankBits, n);
  if (m == 0) return 0;
  const int nwords = (n + 31) / 32;
  const size_t smem = (size_t)kRankWarps * 2 * nwords * sizeof(uint32_t);
  SVDREC_CUDA(smem_attr_once(k_rank_rows, (int)((size_t)kRankWarps * 2 * kRankWords * sizeof(uint32_t))));
  int per_sm = 0;
  SVDREC_CUDA(blocks_per_sm(k_rank_rows, kRankWarps * 32, smem, &per_sm));
  if (per_sm < 1) per_sm = 1;
  const int64_t grid = min64((int64_t)sm_count() * per_sm, (m + kRankWarps - 1) / kRankWarps);
  k_rank_rows<<<(unsigned)grid, kRankWarps * 32, smem, as_stream(stream)>>>(m, n, d_indptr, d_indices, d_values,
                                                                             d_rank, d_out_indices, d_out_values);
  return check_launch("rank_rows");
}

extern "C" int svdrec_seg_plan_count(int64_t m, const int64_t* d_indptr, int32_t seg_max, int64_t* d_first,
                                     int64_t* d_sbase, int64_t* d_lidx, int64_t* d_totals, void* stream) {
  SVDREC_ARG(m >= 0 && seg_max >= 1, "seg_plan_count: bad arguments");
  cudaStream_t s = as_stream(stream);
  if (m == 0) {
    SVDREC_CUDA(cudaMemsetAsync(d_totals, 0, 3 * sizeof(int64_t), s));
    return 0;
  }
  const unsigned grid = (unsigned)((m + 255) / 256);
  k_seg_count<<<grid, 256, 0, s>>>(m, d_indptr, seg_max, d_first, d_sbase, d_lidx);
  int launches = 1;
  int rc = scan_i64(m, d_first, d_first, d_totals + 0, s, &launches);
  if (!rc) rc = scan_i64(m, d_sbase, d_sbase, d_totals + 1, s, &launches);
  if (!rc) rc = scan_i64(m, d_lidx, d_lidx, d_totals + 2, s, &launches);
  if (rc) {
    set_error("seg_plan_count: %s", cudaGetErrorString((cudaError_t)rc));
    return rc;
  }
  return check_launch("seg_plan_count", launches);
}

extern "C" int svdrec_seg_plan_emit(int64_t m, const int64_t* d_indptr, int32_t seg_max, const int64_t* d_first,
                                    const int64_t* d_sbase, const int64_t* d_lidx, int32_t* d_seg_row,
                                    int64_t* d_seg_begin, int64_t* d_seg_end, int32_t* d_seg_slot,
                                    int32_t* d_long_row, int32_t* d_long_s0, int32_t* d_long_s1, void* stream) {
  SVDREC_ARG(m >= 0 && seg_max >= 1, "seg_plan_emit: bad arguments");
  if (m == 0) return 0;
  k_seg_emit<<<(unsigned)((m + 255) / 256), 256, 0, as_stream(stream)>>>(
      m, d_indptr, seg_max, d_first, d_sbase, d_lidx, d_seg_row, d_seg_begin, d_seg_end, d_seg_slot, d_long_row,
      d_long_s0, d_long_s1);
  return check_launch("seg_plan_emit");
}

extern "C" int svdrec_warp_plan(int64_t nseg, const int64_t* d_seg_begin, const int64_t* d_seg_end, int64_t nwarp,
                                int32_t seg_cost, int64_t* d_scratch, int32_t* d_out, void* stream) {
  SVDREC_ARG(nseg >= 0 && nwarp >= 1, "warp_plan: bad arguments");
  cudaStream_t s = as_stream(stream);
  int launches = 0;
  int64_t* cost = d_scratch;          // nseg
  int64_t* total = d_scratch + nseg;  // 1
  if (nseg > 0) {
    k_seg_cost<<<(unsigned)((nseg + 255) / 256), 256, 0, s>>>(nseg, d_seg_begin, d_seg_end, seg_cost, cost);
    launches += 1;
    const int rc = scan_i64(nseg, cost, cost, total, s, &launches);
    if (rc) {
      set_error("warp_plan: %s", cudaGetErrorString((cudaError_t)rc));
      return rc;
    }
  }
  k_warp_cuts<<<(unsigned)((nwarp + 1 + 255) / 256), 256, 0, s>>>(nseg, nwarp, cost, total, d_out);
  launches += 1;
  return check_launch("warp_plan", launches);
}

// Chunk plan of the pipelined SpMMs.  d_cbase: nseg + 1 int64 (exclusive scan
// of the chunk counts; [nseg] = their total); d_recs: room for
// nnz / 32 + 2 nseg records (an upper bound known without a read-back).
// d_indptr / d_hot_cnt (both or neither): the hot-first copy's row starts
// and hot-entry counts.
extern "C" int svdrec_chunk_plan(int64_t nseg, const int32_t* d_seg_row, const int64_t* d_seg_begin,
                                 const int64_t* d_seg_end, const int32_t* d_seg_slot, const int64_t* d_indptr,
                                 const int32_t* d_hot_cnt, int64_t* d_cbase, void* d_recs, void* stream) {
  SVDREC_ARG(nseg >= 0 && (!d_hot_cnt || d_indptr), "chunk_plan: bad arguments");
  cudaStream_t s = as_stream(stream);
  if (nseg == 0) {
    SVDREC_CUDA(cudaMemsetAsync(d_cbase, 0, sizeof(int64_t), s));
    return 0;
  }
  const unsigned grid = (unsigned)((nseg + 255) / 256);
  k_chunk_count<<<grid, 256, 0, s>>>(nseg, d_seg_row, d_seg_begin, d_seg_end, d_indptr, d_hot_cnt, d_cbase);
  int launches = 1;
  const int rc = scan_i64(nseg, d_cbase, d_cbase, d_cbase + nseg, s, &launches);
  if (rc) {
    set_error("chunk_plan: %s", cudaGetErrorString((cudaError_t)rc));
    return rc;
  }
  k_chunk_emit<<<grid, 256, 0, s>>>(nseg, d_seg_row, d_seg_begin, d_seg_end, d_seg_slot, d_indptr, d_hot_cnt, d_cbase,
                                    reinterpret_cast<int4*>(d_recs));
  return check_launch("chunk_plan", launches + 1);
}

extern "C" int svdrec_warp_chunks(int64_t nwarp, const int32_t* d_warp_seg, int64_t nseg, const int64_t* d_cbase,
                                  int32_t* d_warp_chunk, void* stream) {
  SVDREC_ARG(nwarp >= 1 && nseg >= 0, "warp_chunks: bad arguments");
  k_warp_chunks<<<(unsigned)((nwarp + 1 + 255) / 256), 256, 0, as_stream(stream)>>>(nwarp, d_warp_seg, nseg, d_cbase,
                                                                                    d_cbase + nseg, d_warp_chunk);
  return check_launch("warp_chunks");
}

extern "C" int svdrec_scan_i64(int64_t n, const int64_t* d_in, int64_t* d_out, int64_t* d_total, void* stream) {
  SVDREC_ARG(n >= 0, "scan_i64: bad arguments");
  int launches = 0;
  const int rc = scan_i64(n, d_in, d_out, d_total, as_stream(stream), &launches);
  if (rc) {
    set_error("scan_i64: %s", cudaGetErrorString((cudaError_t)rc));
    return rc;
  }
  return check_launch("scan_i64", launches);
}

extern "C" int64_t svdrec_csr_transpose_scratch(int64_t n_out) {
  // hist tables (int32, n_out x slices) + column totals (int64); the
  // per-position row / entry arrays are allocated by the caller's scratch
  // too: see svdrec_csr_transpose (2 x entries x int32 after these)
  const int64_t nb = n_out < kBins ? n_out : kBins;
  return (int64_t)align_up((size_t)nb * sm_count() * sizeof(int32_t)) + (int64_t)align_up((size_t)(n_out + 1) * 8);
}

extern "C" int svdrec_csr_transpose(int64_t nrows, int64_t n_out, int64_t total, const int64_t* d_indptr,
                                    const int32_t* d_indices, const double* d_values, const int32_t* d_perm,
                                    const int64_t* d_pptr, int32_t relabel, int64_t* d_out_indptr, int32_t* d_out_indices,
                                    double* d_out_values, void* d_scratch, int64_t scratch_bytes, void* stream) {
  SVDREC_ARG(nrows >= 0 && n_out >= 0 && d_pptr && d_indptr && d_out_indptr, "csr_transpose: bad arguments");
  cudaStream_t s = as_stream(stream);
  SVDREC_ARG(total >= 0 && total < (1ll << 31), "csr_transpose: %lld entries exceed int32 positions", (long long)total);
  const int64_t base = svdrec_csr_transpose_scratch(n_out);
  SVDREC_ARG(scratch_bytes >= base + 2 * (int64_t)align_up((size_t)total * 4),
             "csr_transpose: scratch too small (%lld < %lld)", (long long)scratch_bytes,
             (long long)(base + 2 * (int64_t)align_up((size_t)total * 4)));
  const int g = sm_count();
  char* ws = reinterpret_cast<char*>(d_scratch);
  int32_t* hist = reinterpret_cast<int32_t*>(ws);
  const int64_t nbmax = n_out < kBins ? n_out : kBins;
  int64_t* counts = reinterpret_cast<int64_t*>(ws + align_up((size_t)nbmax * g * sizeof(int32_t)));
  int32_t* row_p = reinterpret_cast<int32_t*>(ws + base);
  int32_t* src_e = reinterpret_cast<int32_t*>(ws + base + align_up((size_t)total * 4));
  const size_t smem = (size_t)nbmax * sizeof(int32_t);
  SVDREC_CUDA(smem_attr_once(k_tr_hist, (int)(kBins * sizeof(int32_t))));
  SVDREC_CUDA(smem_attr_once(k_tr_scatter<true>, (int)(kBins * sizeof(int32_t))));
  SVDREC_CUDA(smem_attr_once(k_tr_scatter<false>, (int)(kBins * sizeof(int32_t))));
  int launches = 0;
  if (total > 0) {
    k_tr_expand<<<g * 8, 256, 0, s>>>(nrows, d_pptr, d_indptr, d_perm, row_p, src_e);
    launches += 1;
  }
  // pass 1: column totals -> output row pointers
  for (int64_t c0 = 0; c0 < n_out; c0 += kBins) {
    const int32_t nb = (int32_t)min64(kBins, n_out - c0);
    k_tr_hist<<<g, kTrThreads, smem, s>>>(src_e, d_indices, total, (int32_t)c0, nb, hist);
    k_tr_totals<<<(nb + 255) / 256, 256, 0, s>>>(nb, g, hist, counts + c0);
    launches += 2;
  }
  SVDREC_CUDA((cudaError_t)scan_i64(n_out, counts, d_out_indptr, d_out_indptr + n_out, s, &launches));
  // pass 2: per range, histogram (kept from pass 1 for a single range) ->
  // offsets -> stable scatter
  for (int64_t c0 = 0; c0 < n_out && total > 0; c0 += kBins) {
    const int32_t nb = (int32_t)min64(kBins, n_out - c0);
    if (n_out > kBins) {
      k_tr_hist<<<g, kTrThreads, smem, s>>>(src_e, d_indices, total, (int32_t)c0, nb, hist);
      launches += 1;
    }
    k_tr_offsets<<<(nb + 255) / 256, 256, 0, s>>>(nb, g, d_out_indptr, (int32_t)c0, hist);
    if (relabel)
      k_tr_scatter<true><<<g, kTrThreads, smem, s>>>(row_p, src_e, d_perm, d_indices, d_values, total, (int32_t)c0,
                                                      nb, hist, d_out_indices, d_out_values);
    else
      k_tr_scatter<false><<<g, kTrThreads, smem, s>>>(row_p, src_e, d_perm, d_indices, d_values, total,
                                                       (int32_t)c0, nb, hist, d_out_indices, d_out_values);
    launches += 2;
  }
  return check_launch("csr_transpose", launches);
}
