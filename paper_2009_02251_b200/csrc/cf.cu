// Item-latent-factor collaborative filtering kernels (Alg. 4 / Alg. 5).
//
// Reference: cf.py:77-143 (latent_from_qb, _predict), cf.py:178-190
// (evaluate_mae), cf.py:243-254 (_check_disjoint).
//
// The reference predicts rating (u, j) as the cosine-weighted average of
// u's stored ratings:  sum_l A(u,l) cos(T_l, T_j) / sum_l cos(T_l, T_j).
// With unit item columns Tn_l = T_l / |T_l| (zero for |T_l| = 0, which the
// reference skips) both sums are dot products of Tn_j with two per-user
// k-vectors,  P_u = sum_l A(u,l) Tn_l  and  S_u = sum_l Tn_l,  so the work
// per user is one pass over the user's row (deg(u) * k gathers of unit
// item rows) plus one k-dot pair per held-out sample, instead of
// deg(u) * k per sample.  One warp owns one user's group of samples and
// keeps P_u, S_u in registers (k <= 1024).
#include <cstdlib>

#include "common.cuh"

namespace svdrec {
namespace {

constexpr double kWeightFloor = 1e-9;  // cf.py:23

__global__ void k_normalize(int64_t n, int k, const double* __restrict__ Tt, int64_t ldt, double* __restrict__ Tn,
                            int64_t ldn, double* __restrict__ norm) {
  const int lane = threadIdx.x & 31;
  const int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (item >= n) return;
  const double* src = Tt + item * ldt;
  double s = 0.0;
  for (int e = lane; e < k; e += 32) s = fma(src[e], src[e], s);
  s = warp_sum(s);
  const double nr = sqrt(s);
  const double inv = nr > 0.0 ? 1.0 / nr : 0.0;
  double* dst = Tn + item * ldn;
  for (int e = lane; e < k; e += 32) dst[e] = src[e] * inv;
  if (lane == 0) norm[item] = nr;
}

// Metric pair: n_l = sqrt(x_l . y_l); Xn = X / n, Yn = Y / n (0 if n = 0).
__global__ void k_normalize_pair(int64_t n, int k, const double* __restrict__ X, int64_t ldx,
                                 const double* __restrict__ Y, int64_t ldy, double* __restrict__ Xn,
                                 double* __restrict__ Yn, int64_t ldn, double* __restrict__ norm) {
  const int lane = threadIdx.x & 31;
  const int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (item >= n) return;
  const double* xr = X + item * ldx;
  const double* yr = Y + item * ldy;
  double s = 0.0;
  for (int e = lane; e < k; e += 32) s = fma(xr[e], yr[e], s);
  s = warp_sum(s);
  const double nr = s > 0.0 ? sqrt(s) : 0.0;
  const double inv = nr > 0.0 ? 1.0 / nr : 0.0;
  for (int e = lane; e < k; e += 32) {
    Xn[item * ldn + e] = xr[e] * inv;
    Yn[item * ldn + e] = yr[e] * inv;
  }
  if (lane == 0) norm[item] = nr;
}

// Row storage of the scoring kernel: 16-B vector loads, VE elements each
// (double2 or float4), so a row of k values costs k / VE loads per lane
// group instead of k -- the gathers are bound by load requests, not bytes.
template <typename TY, int VE>
struct RowVec;
template <typename TY>
struct RowVec<TY, 1> {
  using T = TY;
  __device__ __forceinline__ static void get(const T& x, double (&o)[1]) { o[0] = (double)x; }
};
template <>
struct RowVec<double, 2> {
  using T = double2;
  __device__ __forceinline__ static void get(const T& x, double (&o)[2]) {
    o[0] = x.x;
    o[1] = x.y;
  }
};
template <>
struct RowVec<float, 2> {
  using T = float2;
  __device__ __forceinline__ static void get(const T& x, double (&o)[2]) {
    o[0] = x.x;
    o[1] = x.y;
  }
};
template <>
struct RowVec<float, 4> {
  using T = float4;
  __device__ __forceinline__ static void get(const T& x, double (&o)[4]) {
    o[0] = x.x;
    o[1] = x.y;
    o[2] = x.z;
    o[3] = x.w;
  }
};

// Threads per CTA of the scoring kernel (one persistent CTA per SM): the
// register file caps the per-lane accumulators (2 * NT * VE doubles plus U
// rows of loads in flight), so wide k trades warps for registers.
template <int NA>  // accumulators per lane (NT * VE)
struct PredictShape {
  static constexpr int kThreads = NA <= 8 ? (NA <= 4 ? 768 : 640) : 256;
};

// dynamic shared memory of the scoring kernel: the hottest items' unit rows
constexpr size_t kHotBytes = 208 * 1024;

// Ratings processed per step of the gather loops: every lane keeps U * NT
// vector loads in flight, so narrow rows (small k) take more of them.
template <int NT, int VE>
struct PredictUnroll {  // narrow rows in flight cost fewer registers: take more of them
#ifndef SVDREC_CF_U1
#define SVDREC_CF_U1 8  // rows in flight per lane for the narrow (NT = 1) rows
#endif
  static constexpr int U = NT <= 1 ? SVDREC_CF_U1 : ((VE == 4 && NT <= 2) ? 8 : (NT == 4 && VE == 2 ? 3 : 4));
};

// P += v * row, S += row for U rows (one per q), lane-strided in VE-wide
// vectors (element (t * 32 + lane) * VE + i); padding entries point at a
// zero row.  The accumulation order is rating by rating.
template <int NT, int U, bool SHARED, typename TY, int VE>
__device__ __forceinline__ void accum(double (&P)[NT * VE], double (&S)[NT * VE], const TY* const (&rows)[U],
                                      const double (&vv)[U], int lane, int kp) {
  using V = typename RowVec<TY, VE>::T;
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int base = (t * 32 + lane) * VE;
    if (base < kp) {
      V x[U];
#pragma unroll
      for (int q = 0; q < U; ++q)
        x[q] = SHARED ? *reinterpret_cast<const V*>(rows[q] + base) : __ldg(reinterpret_cast<const V*>(rows[q] + base));
#pragma unroll
      for (int q = 0; q < U; ++q) {
        double xe[VE];
        RowVec<TY, VE>::get(x[q], xe);
#pragma unroll
        for (int i = 0; i < VE; ++i) {
          P[t * VE + i] = fma(vv[q], xe[i], P[t * VE + i]);
          S[t * VE + i] += xe[i];
        }
      }
    }
  }
}

// Items are relabelled by popularity rank (0 = most rated) and every user's
// ratings are stored in ascending rank order, so a user's hot items come
// first: the unit rows of the ``nhot`` most popular items (Yr[0, nhot),
// rank order) are staged once per CTA in shared memory and a 32-rating
// batch splits into a shared-memory prefix (LDS, no long latency) and an
// L2-gathered suffix (LDG, U rows in flight per lane).
// TY: storage type of the gathered unit rows (double; float for the fp32
// variant); rows are padded to kp (a multiple of VE) with zeros, ldy % VE
// == 0; accumulation stays double.
template <int NT, typename TY, int VE>
__global__ void __launch_bounds__(PredictShape<NT * VE>::kThreads, 1)
    k_predict(int64_t nwork, const int64_t* __restrict__ wstart, const int4* __restrict__ wmeta,
              const int32_t* __restrict__ items, const int32_t* __restrict__ rindices,
              const double* __restrict__ rvalues, int k, const TY* __restrict__ Yr,
              const double* __restrict__ Xn, int64_t ldn, int64_t ldy, const double* __restrict__ norm, double gmean,
              double lo, double hi, int nhot, int zrow, int* __restrict__ done, double* __restrict__ part,
              int* __restrict__ counter,
              double* __restrict__ out_val, double* __restrict__ out_raw, uint8_t* __restrict__ out_fb) {
  constexpr int NA = NT * VE;
  const int kp = (k + VE - 1) / VE * VE;
  // row pitches as 32-bit values: row * pitch is then one IMAD.WIDE instead
  // of a 64 x 64-bit multiply per gathered row (the host checks they fit)
  const int ldy32 = (int)ldy, ldn32 = (int)ldn;
  extern __shared__ __align__(16) unsigned char hs_raw[];
  TY* hs = reinterpret_cast<TY*>(hs_raw);  // nhot rows + a zero row (padding target), stride kp
  for (int64_t t = threadIdx.x; t < (int64_t)(nhot + 1) * kp; t += blockDim.x) {
    const int64_t sl = t / kp, e = t - sl * kp;
    hs[t] = sl < nhot ? Yr[sl * ldy + e] : TY(0);
  }
  // per-warp batch tables: a 32-rating batch's row ids (hot: shared-memory
  // row or the zero row; cold: Yr row or the zero row) and values, read by
  // every lane with broadcast LDS instead of three shuffles, a compare and a
  // select per rating; U trailing slots are padding for the U-wide steps
  constexpr int U = PredictUnroll<NT, VE>::U;
  constexpr int NWARP = PredictShape<NA>::kThreads / 32, BS = 32 + U;
  __shared__ __align__(16) int32_t s_hot[NWARP][BS];
  __shared__ int32_t s_cold[NWARP][BS];
  __shared__ __align__(16) double s_val[NWARP][BS];
  // the static tables and the dynamic hot rows share the 227 KB opt-in
  static_assert((size_t)NWARP * BS * 16 + kHotBytes <= 232448, "cf_predict: shared memory over the opt-in limit");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane < U) {
    s_hot[wid][32 + lane] = nhot;
    s_cold[wid][32 + lane] = zrow;
    s_val[wid][32 + lane] = 0.0;
  }
  __syncthreads();
  // Work items are (group, chunk) pairs, heaviest users first.  Users with
  // more than ``chunk`` ratings are split across warps: each chunk leaves
  // (P, S, sum v) in its partial slot and the warp that completes the group
  // last adds the slots in order (deterministic) and scores the samples.
  // Each work item's description is precomputed (one 8-B + two 16-B
  // loads); the next item is claimed while this one is processed.
  int wi = 0;
  if (lane == 0) wi = atomicAdd(counter, 1);
  wi = __shfl_sync(0xffffffffu, wi, 0);
  while (wi < nwork) {
    const int64_t a = __ldg(wstart + wi);
    const int4 m0 = __ldg(wmeta + 2 * (int64_t)wi);      // len, deg, s0, s1
    const int4 m1 = __ldg(wmeta + 2 * (int64_t)wi + 1);  // nch, slot, done, chunk index
    int wn = 0;
    if (lane == 0) wn = atomicAdd(counter, 1);
    const int64_t e = a + m0.x;
    const int64_t deg = m0.y;
    const int64_t s0 = m0.z, s1 = m0.w;
    const int nch = m1.x;
    // the first 32 samples' item ids, loaded now and used after the rating
    // loop (one dependent load less at the end of the item)
    int32_t jl_first = 0;
    if (lane < s1 - s0) jl_first = __ldg(items + s0 + lane);
    double P[NA], S[NA];
#pragma unroll
    for (int t = 0; t < NA; ++t) P[t] = S[t] = 0.0;
    double vsum = 0.0;
    // the next 32-entry CSR batch is loaded while this one is processed;
    // the CSR is streamed once per call, so its loads are evict-first
    // (__ldcs) and do not push the gathered item rows out of L2
    int32_t ci_next = 0x7fffffff;
    double vi_next = 0.0;
    if (a + lane < e) {
      ci_next = __ldcs(rindices + a + lane);
      vi_next = __ldcs(rvalues + a + lane);
    }
    for (int64_t base = a; base < e; base += 32) {
      const int32_t ci = ci_next;
      const double vi = vi_next;
      const int64_t nx = base + 32 + lane;
      ci_next = 0x7fffffff;
      vi_next = 0.0;
      if (nx < e) {
        ci_next = __ldcs(rindices + nx);
        vi_next = __ldcs(rvalues + nx);
      }
      const int nv = (int)min64(32, e - base);
      vsum += vi;  // this lane's entry (0 past the end)
      const bool hot = ci < nhot;  // ascending ranks: the hot entries are a prefix
      const int nh = __popc(__ballot_sync(0xffffffffu, hot));
      __syncwarp();  // the previous batch's tables are read
      s_hot[wid][lane] = hot ? ci : nhot;
      s_cold[wid][lane] = (lane < nv && !hot) ? ci : zrow;
      s_val[wid][lane] = vi;
      __syncwarp();
      for (int j = 0; j < nh; j += U) {  // j % U == 0: 16-B table reads when U % 4 == 0
        const TY* rows[U];
        double vv[U];
        if constexpr (U % 4 == 0) {
#pragma unroll
          for (int q = 0; q < U; q += 4) {
            const int4 id = *reinterpret_cast<const int4*>(&s_hot[wid][j + q]);
            const double2 v0 = *reinterpret_cast<const double2*>(&s_val[wid][j + q]);
            const double2 v1 = *reinterpret_cast<const double2*>(&s_val[wid][j + q + 2]);
            rows[q] = hs + (int64_t)id.x * kp;
            rows[q + 1] = hs + (int64_t)id.y * kp;
            rows[q + 2] = hs + (int64_t)id.z * kp;
            rows[q + 3] = hs + (int64_t)id.w * kp;
            vv[q] = v0.x;
            vv[q + 1] = v0.y;
            vv[q + 2] = v1.x;
            vv[q + 3] = v1.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < U; ++q) {
            rows[q] = hs + (int64_t)s_hot[wid][j + q] * kp;
            vv[q] = s_val[wid][j + q];
          }
        }
        accum<NT, U, true, TY, VE>(P, S, rows, vv, lane, kp);
      }
      for (int j = nh; j < nv; j += U) {
        const TY* rows[U];
        double vv[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          rows[q] = Yr + (int64_t)s_cold[wid][j + q] * ldy32;
          vv[q] = s_val[wid][j + q];
        }
        accum<NT, U, false, TY, VE>(P, S, rows, vv, lane, kp);
      }
    }
    vsum = warp_sum(vsum);
    if (nch > 1) {
      const int64_t pw = 2 * (int64_t)k + 1;
      const int slot = m1.y, slot0 = slot - m1.w;
      double* mine = part + (int64_t)slot * pw;
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int i = 0; i < VE; ++i) {
          const int idx = (t * 32 + lane) * VE + i;
          if (idx < k) {
            mine[idx] = P[t * VE + i];
            mine[k + idx] = S[t * VE + i];
          }
        }
      if (lane == 0) mine[2 * k] = vsum;
      __threadfence();
      int prev = 0;
      if (lane == 0) prev = atomicAdd(done + m1.z, 1);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev != nch - 1) {  // not the last chunk of this user
        wi = __shfl_sync(0xffffffffu, wn, 0);
        continue;
      }
      __threadfence();
#pragma unroll
      for (int t = 0; t < NA; ++t) P[t] = S[t] = 0.0;
      vsum = 0.0;
      for (int q = 0; q < nch; ++q) {
        const double* ps = part + ((int64_t)slot0 + q) * pw;
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int i = 0; i < VE; ++i) {
            const int idx = (t * 32 + lane) * VE + i;
            if (idx < k) {
              P[t * VE + i] += __ldcg(ps + idx);
              S[t * VE + i] += __ldcg(ps + k + idx);
            }
          }
        vsum += __ldcg(ps + 2 * k);
      }
    }
    const double mean = deg > 0 ? vsum / (double)deg : gmean;
    const double fb_val = fmin(fmax(mean, lo), hi);
    // score the group's samples: ids and norms of up to 32 samples are
    // fetched by the lanes at once, then two samples' rows are in flight
    // per step (the per-sample id -> norm -> row chain was latency-bound)
    for (int64_t sb = s0; sb < s1; sb += 32) {
      const int ns = (int)min64(32, s1 - sb);
      int32_t jl = 0;
      double nl = 0.0;
      if (lane < ns) {
        jl = sb == s0 ? jl_first : items[sb + lane];
        nl = norm[jl];
      }
      for (int q = 0; q < ns; q += 2) {
        const int32_t j0 = __shfl_sync(0xffffffffu, jl, q);
        const int32_t j1 = __shfl_sync(0xffffffffu, jl, (q + 1) & 31);
        const double n0 = __shfl_sync(0xffffffffu, nl, q);
        const double n1 = q + 1 < ns ? __shfl_sync(0xffffffffu, nl, (q + 1) & 31) : 0.0;
        const bool ok0 = n0 != 0.0 && deg > 0, ok1 = n1 != 0.0 && deg > 0;
        const double* row0 = Xn + (int64_t)j0 * ldn32;
        const double* row1 = Xn + (int64_t)j1 * ldn32;
        double num0 = 0.0, den0 = 0.0, num1 = 0.0, den1 = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int i = 0; i < VE; ++i) {
            const int idx = (t * 32 + lane) * VE + i;
            if (idx < k) {
              const double x0 = ok0 ? __ldg(row0 + idx) : 0.0;
              const double x1 = ok1 ? __ldg(row1 + idx) : 0.0;
              num0 = fma(x0, P[t * VE + i], num0);
              den0 = fma(x0, S[t * VE + i], den0);
              num1 = fma(x1, P[t * VE + i], num1);
              den1 = fma(x1, S[t * VE + i], den1);
            }
          }
        num0 = warp_sum(num0);
        den0 = warp_sum(den0);
        num1 = warp_sum(num1);
        den1 = warp_sum(den1);
        if (lane == 0) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (q + h >= ns) break;
            const bool ok = h ? ok1 : ok0;
            const double num = h ? num1 : num0, den = h ? den1 : den0;
            const int64_t sidx = sb + q + h;
            const bool fb = !ok || fabs(den) < kWeightFloor;
            const double raw = fb ? mean : num / den;
            out_raw[sidx] = raw;
            out_val[sidx] = fb ? fb_val : fmin(fmax(raw, lo), hi);
            out_fb[sidx] = fb ? 1 : 0;
          }
        }
      }
    }
    wi = __shfl_sync(0xffffffffu, wn, 0);
  }  // dynamic loop over work items
}

// Wide factors (k > 1024, e.g. the factors of a fixed-precision QB at a
// few thousand columns): one CTA per user group, the k columns in tiles of
// kWideCols (4 per thread); per tile P_u, S_u are built in registers from
// the user's rated unit rows and every sample's tile dot products are
// block-reduced in a fixed order and accumulated in out_raw (numerator) and
// out_val (denominator), finalised after the last tile.  Same arithmetic
// and fallback rules as k_predict; deterministic.
constexpr int kWideThreads = 256, kWideCols = 4 * kWideThreads;

template <typename TY>
__global__ void __launch_bounds__(kWideThreads) k_predict_wide(
    int64_t ngroups, const int64_t* __restrict__ goff, const int64_t* __restrict__ guser,
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ items, const int32_t* __restrict__ rindices,
    const double* __restrict__ rvalues, int k, const TY* __restrict__ Yr, int64_t ldy, const double* __restrict__ Xn,
    int64_t ldn, const double* __restrict__ norm, double gmean, double lo, double hi, double* __restrict__ out_val,
    double* __restrict__ out_raw, uint8_t* __restrict__ out_fb) {
  __shared__ double red[2][kWideThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t gi = blockIdx.x; gi < ngroups; gi += gridDim.x) {
    const int64_t s0 = goff[gi], s1 = goff[gi + 1];
    const int64_t u = guser[gi];
    const int64_t r0 = indptr[u], deg = indptr[u + 1] - r0;
    for (int c0 = 0; c0 < k; c0 += kWideCols) {
      double P[4] = {0.0, 0.0, 0.0, 0.0}, S[4] = {0.0, 0.0, 0.0, 0.0};
      for (int64_t t = 0; t < deg; ++t) {
        const double v = rvalues[r0 + t];
        const TY* row = Yr + (int64_t)rindices[r0 + t] * ldy;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int c = c0 + threadIdx.x + i * kWideThreads;
          if (c < k) {
            const double x = (double)row[c];
            P[i] = fma(v, x, P[i]);
            S[i] += x;
          }
        }
      }
      for (int64_t sidx = s0; sidx < s1; ++sidx) {
        const double* xr = Xn + (int64_t)items[sidx] * ldn;
        double num = 0.0, den = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int c = c0 + threadIdx.x + i * kWideThreads;
          if (c < k) {
            num = fma(xr[c], P[i], num);
            den = fma(xr[c], S[i], den);
          }
        }
        num = warp_sum(num);
        den = warp_sum(den);
        if (lane == 0) {
          red[0][wid] = num;
          red[1][wid] = den;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          double tn = 0.0, td = 0.0;
          for (int w = 0; w < kWideThreads / 32; ++w) {
            tn += red[0][w];
            td += red[1][w];
          }
          out_raw[sidx] = c0 ? out_raw[sidx] + tn : tn;
          out_val[sidx] = c0 ? out_val[sidx] + td : td;
        }
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) {
      double vsum = 0.0;
      for (int64_t t = 0; t < deg; ++t) vsum += rvalues[r0 + t];
      const double mean = deg > 0 ? vsum / (double)deg : gmean;
      for (int64_t sidx = s0; sidx < s1; ++sidx) {
        const double num = out_raw[sidx], den = out_val[sidx];
        const bool fb = norm[items[sidx]] == 0.0 || deg == 0 || fabs(den) < kWeightFloor;
        const double raw = fb ? mean : num / den;
        out_raw[sidx] = raw;
        out_val[sidx] = fmin(fmax(raw, lo), hi);
        out_fb[sidx] = fb ? 1 : 0;
      }
    }
    __syncthreads();
  }
}

__global__ void k_overlap(int64_t ns, const int32_t* __restrict__ users, const int32_t* __restrict__ items,
                          const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int32_t* count) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ns) return;
  int64_t lo = indptr[users[t]], hi = indptr[users[t] + 1];
  const int32_t it = items[t];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (indices[mid] < it)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < indptr[users[t] + 1] && indices[lo] == it) atomicAdd(count, 1);
}

// Scoring work plan (the WorkPlan of cf.py): k_plan_map writes, per group,
// the values four exclusive scans turn into the plan's bases (partial
// slots and completion counters of split groups, first work item of each
// group in heaviest-first order, ratings streamed); k_plan_fin turns them
// into the int32 bases and the plan's sizes; k_plan_emit writes every
// item's start and 8-int meta record.  Same arrays as the torch
// restatement it replaces (tests/test_gpu_ingest.py).
__device__ __forceinline__ int64_t plan_nch(int64_t d, int chunk) {
  // 32-bit division (a 64-bit one is a long emulated sequence on the GPU)
  return d <= chunk ? 1 : (int64_t)(((uint32_t)d + (uint32_t)chunk - 1u) / (uint32_t)chunk);
}

__global__ void k_plan_map(int64_t ng, const int64_t* __restrict__ gd, const int64_t* __restrict__ order, int chunk,
                           int64_t* __restrict__ slots, int64_t* __restrict__ split, int64_t* __restrict__ items) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t n = plan_nch(gd[g], chunk);
  slots[g] = n > 1 ? n : 0;
  split[g] = n > 1 ? 1 : 0;
  items[g] = plan_nch(gd[order[g]], chunk);
}

__global__ void k_plan_fin(int64_t ng, const int64_t* __restrict__ gd, int chunk, const int64_t* __restrict__ slots,
                           const int64_t* __restrict__ split, int32_t* __restrict__ slot0,
                           int32_t* __restrict__ done_idx) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const bool sp = plan_nch(gd[g], chunk) > 1;
  slot0[g] = sp ? (int32_t)slots[g] : -1;
  done_idx[g] = sp ? (int32_t)split[g] : -1;
}

// j: position in heaviest-first order
__global__ void k_plan_emit(int64_t ng, const int64_t* __restrict__ gd, const int64_t* __restrict__ order,
                            const int64_t* __restrict__ first, const int32_t* __restrict__ slot0,
                            const int32_t* __restrict__ done_idx, const int64_t* __restrict__ gs,
                            const int64_t* __restrict__ row_start, int chunk, int64_t* __restrict__ start,
                            int4* __restrict__ meta) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ng) return;
  const int64_t g = order[j];
  const int64_t deg = gd[g];
  const int64_t nch = plan_nch(deg, chunk);
  const bool split = nch > 1;
  const int64_t w0 = first[j];
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t off = split ? c * chunk : 0;
    const int64_t len = split ? min64(chunk, deg - off) : deg;
    start[w0 + c] = row_start[g] + off;
    meta[2 * (w0 + c)] = make_int4((int)len, (int)deg, (int)gs[g], (int)gs[g + 1]);
    meta[2 * (w0 + c) + 1] = make_int4((int)nch, split ? slot0[g] + (int)c : -1, done_idx[g], (int)c);
  }
}

}  // namespace
}  // namespace svdrec

using namespace svdrec;

extern "C" int svdrec_cf_normalize(int64_t n, int32_t k, const double* d_Tt, int64_t ldt, double* d_Tn, int64_t ldn,
                                   double* d_norm, void* stream) {
  SVDREC_ARG(n >= 0 && k >= 1 && ldt >= k && ldn >= k, "cf_normalize: bad arguments");
  if (n == 0) return 0;
  const int64_t thr = n * 32;
  k_normalize<<<(unsigned)((thr + 255) / 256), 256, 0, as_stream(stream)>>>(n, k, d_Tt, ldt, d_Tn, ldn, d_norm);
  return check_launch("cf_normalize");
}

extern "C" int svdrec_cf_normalize_pair(int64_t n, int32_t k, const double* d_X, int64_t ldx, const double* d_Y,
                                        int64_t ldy, double* d_Xn, double* d_Yn, int64_t ldn, double* d_norm,
                                        void* stream) {
  SVDREC_ARG(n >= 0 && k >= 1 && ldx >= k && ldy >= k && ldn >= k, "cf_normalize_pair: bad arguments");
  if (n == 0) return 0;
  const int64_t thr = n * 32;
  k_normalize_pair<<<(unsigned)((thr + 255) / 256), 256, 0, as_stream(stream)>>>(n, k, d_X, ldx, d_Y, ldy, d_Xn,
                                                                                 d_Yn, ldn, d_norm);
  return check_launch("cf_normalize_pair");
}

namespace {
template <typename TY>
int cf_predict_impl(int64_t nwork, const int64_t* d_work_start, const int32_t* d_work_meta, const int32_t* d_items,
                    const int32_t* d_ranked_indices, const double* d_ranked_values, int32_t k, const TY* d_Yr,
                    int64_t ldy, const double* d_Xn, int64_t ldn, const double* d_norm, double global_mean,
                    double rating_min, double rating_max, int32_t n_items, int32_t* d_done, int64_t ndone,
                    double* d_partial, int32_t* d_counter, double* d_value, double* d_raw, uint8_t* d_fallback,
                    void* stream) {
  SVDREC_ARG(nwork >= 0 && k >= 1 && ldn >= k && ldy >= k && n_items >= 0, "cf_predict: bad arguments");
  if (k > 1024) {
    set_error("cf_predict: latent dimension %d > 1024: use svdrec_cf_predict_wide", k);
    return SVDREC_E_UNSUPPORTED;
  }
  if (nwork == 0) return 0;
  SVDREC_ARG(d_counter && d_work_start && d_work_meta, "cf_predict: work plan required");
  SVDREC_ARG(reinterpret_cast<uintptr_t>(d_work_meta) % 16 == 0, "cf_predict: work meta must be 16-B aligned");
  cudaStream_t s = as_stream(stream);
  SVDREC_CUDA(cudaMemsetAsync(d_counter, 0, sizeof(int32_t), s));
  if (ndone > 0) SVDREC_CUDA(cudaMemsetAsync(d_done, 0, (size_t)ndone * sizeof(int32_t), s));
  // elements per lane and load: 16-B vectors for wide rows, narrower ones
  // for short rows (more lanes busy per rating)
  constexpr int VMAX = (int)(16 / sizeof(TY));
  const int ve = k <= 32 ? 1 : (k <= 64 || VMAX == 2 ? 2 : 4);
  SVDREC_ARG(ldy % VMAX == 0 && reinterpret_cast<uintptr_t>(d_Yr) % 16 == 0,
             "cf_predict: Yr rows must be 16-B aligned (ldy %% %d == 0)", VMAX);
  SVDREC_ARG(ldy < (1ll << 31) && ldn < (1ll << 31), "cf_predict: row pitches must fit 32 bits");
  const int kp = (k + ve - 1) / ve * ve;
  const int nt = (kp / ve + 31) / 32;  // vector steps per lane
  // one persistent CTA per SM holding the hottest items' unit rows in
  // shared memory (as many as fit in kHotBytes, plus the zero row)
  int nhot = (int)(kHotBytes / ((size_t)kp * sizeof(TY))) - 1;
  if (nhot > n_items) nhot = n_items;
  if (nhot < 0) nhot = 0;
  const size_t smem = (size_t)(nhot + 1) * kp * sizeof(TY);
  const int64_t grid = sm_count();
#define SVDREC_PRED(NT, VE)                                                                                   \
  do {                                                                                                        \
    SVDREC_CUDA(smem_attr_once(k_predict<NT, TY, VE>, (int)kHotBytes));                                     \
    k_predict<NT, TY, VE><<<(unsigned)grid, PredictShape<NT * VE>::kThreads, smem, s>>>(                      \
        nwork, d_work_start, reinterpret_cast<const int4*>(d_work_meta), d_items, d_ranked_indices,           \
        d_ranked_values, k, d_Yr, d_Xn, ldn, ldy, d_norm, global_mean, rating_min, rating_max, nhot, n_items, \
        d_done, d_partial, d_counter, d_value, d_raw, d_fallback);                                            \
  } while (0)
  if (ve == 1)
    SVDREC_PRED(1, 1);
  else if (ve == 2 && nt <= 1)
    SVDREC_PRED(1, 2);
  else if (VMAX == 4) {
    if (nt <= 1)
      SVDREC_PRED(1, VMAX);
    else if (nt <= 2)
      SVDREC_PRED(2, VMAX);
    else if (nt <= 4)
      SVDREC_PRED(4, VMAX);
    else
      SVDREC_PRED(8, VMAX);
  } else {
    if (nt <= 2)
      SVDREC_PRED(2, VMAX);
    else if (nt <= 3)
      SVDREC_PRED(3, VMAX);
    else if (nt <= 4)
      SVDREC_PRED(4, VMAX);
    else if (nt <= 8)
      SVDREC_PRED(8, VMAX);
    else
      SVDREC_PRED(16, VMAX);
  }
#undef SVDREC_PRED
  return check_launch("cf_predict");
}
}  // namespace

extern "C" int svdrec_cf_predict(int64_t nwork, const int64_t* d_work_start, const int32_t* d_work_meta,
                                 const int32_t* d_items, const int32_t* d_ranked_indices,
                                 const double* d_ranked_values, int32_t k, const double* d_Yr, int64_t ldy,
                                 const double* d_Xn, int64_t ldn, const double* d_norm, double global_mean,
                                 double rating_min, double rating_max, int32_t n_items, int32_t* d_done,
                                 int64_t ndone, double* d_partial, int32_t* d_counter, double* d_value,
                                 double* d_raw, uint8_t* d_fallback, void* stream) {
  return cf_predict_impl<double>(nwork, d_work_start, d_work_meta, d_items, d_ranked_indices, d_ranked_values, k,
                                 d_Yr, ldy, d_Xn, ldn, d_norm, global_mean, rating_min, rating_max, n_items, d_done,
                                 ndone, d_partial, d_counter, d_value, d_raw, d_fallback, stream);
}

extern "C" int svdrec_cf_predict_f32(int64_t nwork, const int64_t* d_work_start, const int32_t* d_work_meta,
                                     const int32_t* d_items, const int32_t* d_ranked_indices,
                                     const double* d_ranked_values, int32_t k, const float* d_Yr, int64_t ldy,
                                     const double* d_Xn, int64_t ldn, const double* d_norm, double global_mean,
                                     double rating_min, double rating_max, int32_t n_items, int32_t* d_done,
                                     int64_t ndone, double* d_partial, int32_t* d_counter, double* d_value,
                                     double* d_raw, uint8_t* d_fallback, void* stream) {
  return cf_predict_impl<float>(nwork, d_work_start, d_work_meta, d_items, d_ranked_indices, d_ranked_values, k,
                                d_Yr, ldy, d_Xn, ldn, d_norm, global_mean, rating_min, rating_max, n_items, d_done,
                                ndone, d_partial, d_counter, d_value, d_raw, d_fallback, stream);
}

extern "C" int svdrec_cf_predict_wide(int64_t ngroups, const int64_t* d_group_offsets, const int64_t* d_group_users,
                                      const int64_t* d_indptr, const int32_t* d_items,
                                      const int32_t* d_ranked_indices, const double* d_ranked_values, int32_t k,
                                      const double* d_Yr, int64_t ldy, const double* d_Xn, int64_t ldn,
                                      const double* d_norm, double global_mean, double rating_min, double rating_max,
                                      double* d_value, double* d_raw, uint8_t* d_fallback, void* stream) {
  SVDREC_ARG(ngroups >= 0 && k >= 1 && ldn >= k && ldy >= k, "cf_predict_wide: bad arguments");
  if (ngroups == 0) return 0;
  const int64_t cap = (int64_t)sm_count() * 8;
  const unsigned grid = (unsigned)(ngroups < cap ? ngroups : cap);
  k_predict_wide<double><<<grid, kWideThreads, 0, as_stream(stream)>>>(
      ngroups, d_group_offsets, d_group_users, d_indptr, d_items, d_ranked_indices, d_ranked_values, k, d_Yr, ldy,
      d_Xn, ldn, d_norm, global_mean, rating_min, rating_max, d_value, d_raw, d_fallback);
  return check_launch("cf_predict_wide");
}

extern "C" int svdrec_count_overlap(int64_t nsamp, const int32_t* d_users, const int32_t* d_items,
                                    const int64_t* d_indptr, const int32_t* d_indices, int32_t* d_count,
                                    void* stream) {
  SVDREC_ARG(nsamp >= 0, "count_overlap: bad arguments");
  cudaStream_t s = as_stream(stream);
  SVDREC_CUDA(cudaMemsetAsync(d_count, 0, sizeof(int32_t), s));
  if (nsamp == 0) return 0;
  k_overlap<<<(unsigned)((nsamp + 255) / 256), 256, 0, s>>>(nsamp, d_users, d_items, d_indptr, d_indices, d_count);
  return check_launch("count_overlap");
}

namespace svdrec {
int scan_i64(int64_t n, const int64_t* d_in, int64_t* d_out, int64_t* d_total, cudaStream_t s, int* launches);
}

extern "C" int svdrec_cf_plan_scan(int64_t ngroups, const int64_t* d_group_deg, const int64_t* d_order,
                                   int32_t chunk, int64_t* d_first, int32_t* d_slot0, int32_t* d_done_idx,
                                   int64_t* d_stats, void* stream) {
  SVDREC_ARG(ngroups >= 0 && chunk >= 1, "cf_plan_scan: bad arguments");
  cudaStream_t s = as_stream(stream);
  SVDREC_CUDA(cudaMemsetAsync(d_stats, 0, 4 * sizeof(int64_t), s));
  if (ngroups == 0) return 0;
  int64_t* tmp = nullptr;  // slots, split flags, ratings (exclusive scans in place)
  SVDREC_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), (size_t)ngroups * 3 * sizeof(int64_t), s));
  int64_t *slots = tmp, *split = tmp + ngroups, *rated = tmp + 2 * ngroups;
  const unsigned grid = (unsigned)((ngroups + 255) / 256);
  int launches = 0;
  k_plan_map<<<grid, 256, 0, s>>>(ngroups, d_group_deg, d_order, chunk, slots, split, d_first);
  launches += 1;
  int rc = scan_i64(ngroups, d_first, d_first, d_stats + 0, s, &launches);      // first item per ordered group
  if (!rc) rc = scan_i64(ngroups, split, split, d_stats + 1, s, &launches);       // completion counters
  if (!rc) rc = scan_i64(ngroups, slots, slots, d_stats + 2, s, &launches);       // partial slots
  if (!rc) rc = scan_i64(ngroups, d_group_deg, rated, d_stats + 3, s, &launches); // ratings streamed
  if (!rc) {
    k_plan_fin<<<grid, 256, 0, s>>>(ngroups, d_group_deg, chunk, slots, split, d_slot0, d_done_idx);
    launches += 1;
  }
  cudaFreeAsync(tmp, s);
  if (rc) {
    set_error("cf_plan_scan: %s", cudaGetErrorString((cudaError_t)rc));
    return rc;
  }
  return check_launch("cf_plan_scan", launches);
}

extern "C" int svdrec_cf_plan_emit(int64_t ngroups, const int64_t* d_group_deg, const int64_t* d_order,
                                   const int64_t* d_first, const int32_t* d_slot0, const int32_t* d_done_idx,
                                   const int64_t* d_group_start, const int64_t* d_row_start, int32_t chunk,
                                   int64_t* d_work_start, int32_t* d_work_meta, void* stream) {
  SVDREC_ARG(ngroups >= 0 && chunk >= 1, "cf_plan_emit: bad arguments");
  SVDREC_ARG(reinterpret_cast<uintptr_t>(d_work_meta) % 16 == 0, "cf_plan_emit: work meta must be 16-B aligned");
  if (ngroups == 0) return 0;
  k_plan_emit<<<(unsigned)((ngroups + 255) / 256), 256, 0, as_stream(stream)>>>(
      ngroups, d_group_deg, d_order, d_first, d_slot0, d_done_idx, d_group_start, d_row_start, chunk, d_work_start,
      reinterpret_cast<int4*>(d_work_meta));
  return check_launch("cf_plan_emit");
}
