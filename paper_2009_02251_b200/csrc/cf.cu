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
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

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

template <int MAXR>
__global__ void __launch_bounds__(512, (MAXR <= 4 ? 2 : 1)) k_predict(int64_t ngroups,
                                                                      const int64_t* __restrict__ gstart,
                                                    const int32_t* __restrict__ users,
                                                    const int32_t* __restrict__ items,
                                                    const int64_t* __restrict__ indptr,
                                                    const int32_t* __restrict__ indices,
                                                    const double* __restrict__ values, int k,
                                                    const double* __restrict__ Yn, const double* __restrict__ Xn,
                                                    int64_t ldn, const double* __restrict__ norm, double gmean,
                                                    double lo, double hi, const int32_t* __restrict__ rank,
                                                    const int32_t* __restrict__ hot, int nhot,
                                                    int64_t nwork, const int32_t* __restrict__ work,
                                                    const int32_t* __restrict__ ginfo, int chunk,
                                                    int* __restrict__ done, double* __restrict__ part,
                                                    int* __restrict__ counter,
                                                    double* __restrict__ out_val, double* __restrict__ out_raw,
                                                    uint8_t* __restrict__ out_fb) {
  // hot items (highest training degree) keep their unit rows in shared
  // memory: under Zipf popularity they carry most of the gathers
  // With a thread-block cluster the hot set is spread over the cluster's
  // distributed shared memory: hot item h lives in CTA h % csize at slot
  // h / csize, so a cluster of 8 stages 8x the rows one SM could hold, and
  // remote rows are read over DSMEM (bandwidth additive to L2's).  ``nhot``
  // is the cluster-wide count.
  extern __shared__ double hs[];
  __shared__ const double* peer[16];
  cg::cluster_group cl = cg::this_cluster();
  const int csize = (int)cl.num_blocks();
  const int crank = (int)cl.block_rank();
  const int nloc = (nhot - crank + csize - 1) / csize;  // slots this CTA holds
  for (int64_t t = threadIdx.x; t < (int64_t)nloc * k; t += blockDim.x) {
    const int64_t sl = t / k, e = t - sl * k;
    hs[t] = Yn[(int64_t)hot[sl * csize + crank] * ldn + e];
  }
  if (threadIdx.x < csize) peer[threadIdx.x] = cl.map_shared_rank(hs, threadIdx.x);
  cl.sync();  // every CTA's slice is staged before anyone reads it
  const int lane = threadIdx.x & 31;
  // Work items are (group, chunk) pairs, heaviest users first.  Users with
  // more than ``chunk`` ratings are split across warps: each chunk leaves
  // (P, S, sum v) in its partial slot and the warp that completes the group
  // last adds the slots in order (deterministic) and scores the samples.
  while (true) {
  int wi = 0;
  if (lane == 0) wi = atomicAdd(counter, 1);
  wi = __shfl_sync(0xffffffffu, wi, 0);
  if (wi >= nwork) break;
  const int64_t g = work[2 * (int64_t)wi];
  const int c = work[2 * (int64_t)wi + 1];
  const int nch = ginfo[3 * g];
  const int64_t s0 = gstart[g], s1 = gstart[g + 1];
  const int32_t u = users[s0];
  const int64_t ra = indptr[u], re = indptr[u + 1];
  const int64_t a = nch > 1 ? ra + (int64_t)c * chunk : ra;
  const int64_t e = nch > 1 ? min64(re, a + chunk) : re;
  double P[MAXR], S[MAXR];
#pragma unroll
  for (int t = 0; t < MAXR; ++t) P[t] = S[t] = 0.0;
  double vsum = 0.0;
  for (int64_t base = a; base < e; base += 32) {
    const int64_t my = base + lane;
    int32_t ci = 0, rk = 0x7fffffff;
    double vi = 0.0;
    if (my < e) {
      ci = __ldg(indices + my);
      vi = __ldg(values + my);
      rk = rank ? __ldg(rank + ci) : 0x7fffffff;
    }
    const int nv = (int)min64(32, e - base);
    // four nonzeros per step, branch-free (generic pointers into shared or
    // global memory), so each lane keeps 4 * MAXR independent loads in
    // flight; the accumulation order is still nonzero by nonzero
    for (int j = 0; j < nv; j += 4) {
      const double* rows[4];
      double vv[4], mk[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int jj = (j + q) & 31;
        const int32_t c = __shfl_sync(0xffffffffu, ci, jj);
        const int32_t r = __shfl_sync(0xffffffffu, rk, jj);
        const double v = __shfl_sync(0xffffffffu, vi, jj);
        const bool ok = j + q < nv;
        rows[q] = r >= nhot ? Yn + (int64_t)c * ldn
                            : (csize == 1 ? hs + (int64_t)r * k : peer[r % csize] + (int64_t)(r / csize) * k);
        vv[q] = ok ? v : 0.0;
        mk[q] = ok ? 1.0 : 0.0;
      }
      vsum += vv[0];
      vsum += vv[1];
      vsum += vv[2];
      vsum += vv[3];
#pragma unroll
      for (int t = 0; t < MAXR; ++t) {
        const int idx = lane + 32 * t;
        if (idx < k) {
          const double x0 = rows[0][idx], x1 = rows[1][idx], x2 = rows[2][idx], x3 = rows[3][idx];
          P[t] = fma(vv[0], x0, P[t]);
          P[t] = fma(vv[1], x1, P[t]);
          P[t] = fma(vv[2], x2, P[t]);
          P[t] = fma(vv[3], x3, P[t]);
          S[t] = fma(mk[0], x0, S[t]);
          S[t] = fma(mk[1], x1, S[t]);
          S[t] = fma(mk[2], x2, S[t]);
          S[t] = fma(mk[3], x3, S[t]);
        }
      }
    }
  }
  if (nch > 1) {
    const int64_t slot0 = ginfo[3 * g + 1];
    const int64_t pw = 2 * (int64_t)k + 1;
    double* mine = part + (slot0 + c) * pw;
#pragma unroll
    for (int t = 0; t < MAXR; ++t) {
      const int idx = lane + 32 * t;
      if (idx < k) {
        mine[idx] = P[t];
        mine[k + idx] = S[t];
      }
    }
    if (lane == 0) mine[2 * k] = vsum;
    __threadfence();
    int prev = 0;
    if (lane == 0) prev = atomicAdd(done + ginfo[3 * g + 2], 1);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != nch - 1) continue;  // not the last chunk of this user
    __threadfence();
#pragma unroll
    for (int t = 0; t < MAXR; ++t) P[t] = S[t] = 0.0;
    vsum = 0.0;
    for (int q = 0; q < nch; ++q) {
      const double* ps = part + (slot0 + q) * pw;
#pragma unroll
      for (int t = 0; t < MAXR; ++t) {
        const int idx = lane + 32 * t;
        if (idx < k) {
          P[t] += __ldcg(ps + idx);
          S[t] += __ldcg(ps + k + idx);
        }
      }
      vsum += __ldcg(ps + 2 * k);
    }
  }
  const int64_t deg = re - ra;
  const double mean = deg > 0 ? vsum / (double)deg : gmean;
  const double fb_val = fmin(fmax(mean, lo), hi);
  for (int64_t sidx = s0; sidx < s1; ++sidx) {
    const int32_t j = items[sidx];
    const double nj = norm[j];
    double num = 0.0, den = 0.0;
    if (nj != 0.0 && deg > 0) {
      const double* row = Xn + (int64_t)j * ldn;
#pragma unroll
      for (int t = 0; t < MAXR; ++t) {
        const int idx = lane + 32 * t;
        if (idx < k) {
          const double x = __ldg(row + idx);
          num = fma(x, P[t], num);
          den = fma(x, S[t], den);
        }
      }
      num = warp_sum(num);
      den = warp_sum(den);
    }
    if (lane == 0) {
      const bool fb = !(nj != 0.0 && deg > 0) || fabs(den) < kWeightFloor;
      const double raw = fb ? mean : num / den;
      out_raw[sidx] = raw;
      out_val[sidx] = fb ? fb_val : fmin(fmax(raw, lo), hi);
      out_fb[sidx] = fb ? 1 : 0;
    }
  }
  }  // dynamic loop over user groups
  cl.sync();  // peers may still be reading this CTA's slice
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

__global__ void k_lowrank(int64_t ns, const int32_t* __restrict__ users, const int32_t* __restrict__ items, int k,
                          const double* __restrict__ U, int64_t ldu, const double* __restrict__ s,
                          const double* __restrict__ V, int64_t ldv, double mu, double* __restrict__ pred) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= ns) return;
  const double* ur = U + (int64_t)users[t] * ldu;
  const double* vr = V + (int64_t)items[t] * ldv;
  double acc = 0.0;
  for (int e = lane; e < k; e += 32) acc = fma(ur[e] * s[e], vr[e], acc);
  acc = warp_sum(acc);
  if (lane == 0) pred[t] = mu + acc;
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

extern "C" int svdrec_cf_predict(int64_t ngroups, const int64_t* d_group_start, const int32_t* d_users,
                                 const int32_t* d_items, const int64_t* d_indptr, const int32_t* d_indices,
                                 const double* d_values, int32_t k, const double* d_Yn, const double* d_Xn,
                                 int64_t ldn,
                                 const double* d_norm, double global_mean, double rating_min, double rating_max,
                                 const int32_t* d_item_rank, const int32_t* d_hot_items, int32_t nhot_avail,
                                 int64_t nwork, const int32_t* d_work, const int32_t* d_ginfo, int32_t chunk,
                                 int32_t* d_done, int64_t ndone, double* d_partial, int32_t* d_counter,
                                 double* d_value, double* d_raw, uint8_t* d_fallback, void* stream) {
  SVDREC_ARG(ngroups >= 0 && k >= 1 && ldn >= k, "cf_predict: bad arguments");
  if (k > 1024) {
    set_error("cf_predict: latent dimension %d > 1024 unsupported", k);
    return SVDREC_E_UNSUPPORTED;
  }
  if (ngroups == 0) return 0;
  SVDREC_ARG(d_counter && d_work && d_ginfo && nwork >= ngroups, "cf_predict: work plan required");
  SVDREC_CUDA(cudaMemsetAsync(d_counter, 0, sizeof(int32_t), as_stream(stream)));
  if (ndone > 0) SVDREC_CUDA(cudaMemsetAsync(d_done, 0, (size_t)ndone * sizeof(int32_t), as_stream(stream)));
  cudaStream_t s = as_stream(stream);
  const int r = (k + 31) / 32;
  // 16-warp CTAs, persistent: two per SM for k <= 128 (more gathers in
  // flight), else one; each stages the hottest item rows in its shared
  // memory.  SVDREC_CF_CLUSTER=c (2..8) spreads the hot set over a c-CTA
  // cluster's distributed shared memory instead -- measured slower on B200
  // (remote 8-byte reads cost more than the L2 hits they replace: cluster 1 /
  // 2 / 4 / 8 -> 33.7 / 35.1 / 42.7 / 52.7 ms per bench step), so off.
  static const int csize_env = getenv("SVDREC_CF_CLUSTER") ? atoi(getenv("SVDREC_CF_CLUSTER")) : 1;
  int csize = csize_env >= 1 && csize_env <= 8 ? csize_env : 1;
  const int per_sm = (csize == 1 && r <= 4) ? 2 : 1;
  const size_t kHotBytes = per_sm == 2 ? 100 * 1024 : 200 * 1024;
  int nhot = d_item_rank && d_hot_items ? (int)(kHotBytes / ((size_t)k * 8)) * csize : 0;
  if (nhot > nhot_avail) nhot = nhot_avail;
  if (nhot < 0) nhot = 0;
  const size_t smem = (size_t)((nhot + csize - 1) / csize) * k * 8;
  const int64_t want = (ngroups + 15) / 16;
  int64_t grid = (int64_t)(per_sm * sm_count() / csize) * csize;
  if (want < grid) grid = ((want + csize - 1) / csize) * csize;
  if (grid < csize) grid = csize;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#define SVDREC_PRED(R)                                                                                       \
  do {                                                                                                       \
    static bool attr_set = false;                                                                            \
    if (!attr_set) {                                                                                         \
      SVDREC_CUDA(cudaFuncSetAttribute(k_predict<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024)); \
      attr_set = true;                                                                                       \
    }                                                                                                        \
    SVDREC_CUDA(cudaLaunchKernelEx(&cfg, k_predict<R>, ngroups, d_group_start, d_users, d_items, d_indptr,   \
                                   d_indices, d_values, k, d_Yn, d_Xn, ldn, d_norm, global_mean, rating_min, \
                                   rating_max, d_item_rank, d_hot_items, nhot, nwork, d_work, d_ginfo, chunk, \
                                   d_done, d_partial, d_counter, d_value, d_raw, d_fallback));                \
  } while (0)
  if (r <= 1)
    SVDREC_PRED(1);
  else if (r <= 2)
    SVDREC_PRED(2);
  else if (r <= 4)
    SVDREC_PRED(4);
  else if (r <= 8)
    SVDREC_PRED(8);
  else if (r <= 16)
    SVDREC_PRED(16);
  else
    SVDREC_PRED(32);
#undef SVDREC_PRED
  return check_launch("cf_predict");
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

extern "C" int svdrec_lowrank_predict(int64_t nsamp, const int32_t* d_users, const int32_t* d_items, int32_t k,
                                      const double* d_U, int64_t ldu, const double* d_s, const double* d_V,
                                      int64_t ldv, double mu, double* d_pred, void* stream) {
  SVDREC_ARG(nsamp >= 0 && k >= 1 && ldu >= k && ldv >= k, "lowrank_predict: bad arguments");
  if (nsamp == 0) return 0;
  const int64_t thr = nsamp * 32;
  k_lowrank<<<(unsigned)((thr + 255) / 256), 256, 0, as_stream(stream)>>>(nsamp, d_users, d_items, k, d_U, ldu, d_s,
                                                                          d_V, ldv, mu, d_pred);
  return check_launch("lowrank_predict");
}
