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

template <int MAXR>
__global__ void __launch_bounds__(128) k_predict(int64_t ngroups, const int64_t* __restrict__ gstart,
                                                 const int32_t* __restrict__ users, const int32_t* __restrict__ items,
                                                 const int64_t* __restrict__ indptr,
                                                 const int32_t* __restrict__ indices,
                                                 const double* __restrict__ values, int k,
                                                 const double* __restrict__ Yn, const double* __restrict__ Xn,
                                                 int64_t ldn,
                                                 const double* __restrict__ norm, double gmean, double lo, double hi,
                                                 double* __restrict__ out_val, double* __restrict__ out_raw,
                                                 uint8_t* __restrict__ out_fb) {
  const int lane = threadIdx.x & 31;
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (g >= ngroups) return;
  const int64_t s0 = gstart[g], s1 = gstart[g + 1];
  const int32_t u = users[s0];
  const int64_t a = indptr[u], e = indptr[u + 1];
  double P[MAXR], S[MAXR];
#pragma unroll
  for (int t = 0; t < MAXR; ++t) P[t] = S[t] = 0.0;
  double vsum = 0.0;
  for (int64_t base = a; base < e; base += 32) {
    const int64_t my = base + lane;
    int32_t ci = 0;
    double vi = 0.0;
    if (my < e) {
      ci = __ldg(indices + my);
      vi = __ldg(values + my);
    }
    const int nv = (int)min64(32, e - base);
    for (int j = 0; j < nv; ++j) {
      const int32_t c = __shfl_sync(0xffffffffu, ci, j);
      const double v = __shfl_sync(0xffffffffu, vi, j);
      vsum += v;
      const double* row = Yn + (int64_t)c * ldn;
#pragma unroll
      for (int t = 0; t < MAXR; ++t) {
        const int idx = lane + 32 * t;
        if (idx < k) {
          const double x = __ldg(row + idx);
          P[t] = fma(v, x, P[t]);
          S[t] += x;
        }
      }
    }
  }
  const int64_t deg = e - a;
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
                                 double* d_value, double* d_raw, uint8_t* d_fallback, void* stream) {
  SVDREC_ARG(ngroups >= 0 && k >= 1 && ldn >= k, "cf_predict: bad arguments");
  if (k > 1024) {
    set_error("cf_predict: latent dimension %d > 1024 unsupported", k);
    return SVDREC_E_UNSUPPORTED;
  }
  if (ngroups == 0) return 0;
  const int64_t thr = ngroups * 32;
  const unsigned grid = (unsigned)((thr + 127) / 128);
  cudaStream_t s = as_stream(stream);
  const int r = (k + 31) / 32;
#define SVDREC_PRED(R)                                                                                         \
  k_predict<R><<<grid, 128, 0, s>>>(ngroups, d_group_start, d_users, d_items, d_indptr, d_indices, d_values, k, \
                                    d_Yn, d_Xn, ldn, d_norm, global_mean, rating_min, rating_max, d_value, d_raw, \
                                    d_fallback)
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
