// Bit-exact GPU replica of numpy's Generator(Philox(key)).standard_normal.
//
// Reference: GaussianStream (pkg/src/svdrec/linalg.py:28-51) draws every
// sketch Omega from numpy's Philox4x64-10 + 256-layer ziggurat.  To keep the
// GPU factorization sketch-aligned with the reference (same selected rank k)
// the device sampler reproduces that stream bit for bit.
//
// The ziggurat consumes a data-dependent number of 64-bit raw words per
// sample, so the stream is a sequential parse.  It is a finite-state
// transducer with three states -- S (start of a sample), T+ / T- (inside the
// exponential-tail loop, carrying the sample's sign) -- whose moves consume
// one or two raw words.  The parse is parallelised exactly:
//   A. each thread owns a chunk of 32 raw positions and tabulates, for each
//      of the 6 possible entry configurations (entry offset 0/1 x state),
//      the exit configuration and the number of samples emitted (the five
//      secondary entries stop as soon as they meet the primary walk's
//      trajectory, usually within one or two moves);
//   B. each CTA composes its 1024 chunk tables with an inclusive
//      Hillis-Steele scan (composition of finite maps is associative);
//   C. one thread threads the true entry configuration through the CTA
//      aggregates (tens of steps);
//   D. every chunk re-walks from its true entry and writes its samples.
// Philox is counter-based, so raw words are recomputed, never stored.
#include "common.cuh"
#include "ziggurat_tables.h"

namespace svdrec {
namespace {

constexpr int kChunk = 8;  // raw words per chunk (small: the walks read a precomputed raw buffer)
constexpr int kScan = 1024;
constexpr int kCfg = 6;
constexpr uint64_t kM0 = 0xD2E7470EE14C6C93ULL, kM1 = 0xCA5A826395121157ULL;
constexpr uint64_t kW0 = 0x9E3779B97F4A7C15ULL, kW1 = 0xBB67AE8584CAA73BULL;

__device__ __forceinline__ void philox4x64(uint64_t ctr, uint64_t k0, uint64_t k1, uint64_t& o0,
                                           uint64_t& o1, uint64_t& o2, uint64_t& o3) {
  uint64_t c0 = ctr, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = kM0 * c0, hi0 = __umul64hi(kM0, c0);
    const uint64_t lo1 = kM1 * c2, hi1 = __umul64hi(kM1, c2);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += kW0;
    k1 += kW1;
  }
  o0 = c0;
  o1 = c1;
  o2 = c2;
  o3 = c3;
}

__device__ __forceinline__ uint64_t pick(uint64_t a, uint64_t b, uint64_t c, uint64_t d, uint32_t i) {
  return i == 0 ? a : (i == 1 ? b : (i == 2 ? c : d));
}

// Raw word source with a two-block window (numpy: word g is lane g%4 of the
// block whose counter is g/4 + 1).
struct Raw {
  uint64_t k0, k1;
  uint64_t blk;  // block index held in w*
  uint64_t w0, w1, w2, w3;
  bool has_next;
  uint64_t n0, n1, n2, n3;

  __device__ void init(uint64_t a, uint64_t b) {
    k0 = a;
    k1 = b;
    blk = ~0ULL;
    has_next = false;
  }
  __device__ void fill(uint64_t bi, uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d) {
    philox4x64(bi + 1, k0, k1, a, b, c, d);
  }
  __device__ uint64_t at(uint64_t g) {
    const uint64_t bi = g >> 2;
    if (bi != blk) {
      if (has_next && bi == blk + 1) {
        w0 = n0; w1 = n1; w2 = n2; w3 = n3;
        has_next = false;
      } else {
        fill(bi, w0, w1, w2, w3);
        has_next = false;
      }
      blk = bi;
    }
    return pick(w0, w1, w2, w3, (uint32_t)(g & 3));
  }
  // word g+1 without disturbing the current block
  __device__ uint64_t ahead(uint64_t g) {
    const uint64_t h = g + 1, bi = h >> 2;
    if (bi == blk) return pick(w0, w1, w2, w3, (uint32_t)(h & 3));
    if (!has_next) {
      fill(bi, n0, n1, n2, n3);
      has_next = true;
    }
    return pick(n0, n1, n2, n3, (uint32_t)(h & 3));
  }
};

// Raw words precomputed by k_raw into a buffer covering [pos0, pos0 + n).
struct RawBuf {
  const uint64_t* buf;
  uint64_t pos0;
  __device__ uint64_t at(uint64_t g) const { return __ldg(buf + (g - pos0)); }
  __device__ uint64_t ahead(uint64_t g) const { return __ldg(buf + (g + 1 - pos0)); }
};

// A thread's kChunk + 2 raw words staged in shared memory, transposed
// (word i of thread t at [i][t]: conflict-free; the natural [t][i] layout
// put a warp's loads 16-way on the same bank).
constexpr int kGauThreads = 128;
constexpr int kStage = kChunk + 2;

struct RawSmem {
  const uint64_t* sw;  // &stage[0][threadIdx.x]
  uint64_t base;       // this thread's chunk start
  __device__ uint64_t at(uint64_t g) const { return sw[(g - base) * kGauThreads]; }
  __device__ uint64_t ahead(uint64_t g) const { return sw[(g + 1 - base) * kGauThreads]; }
};

__device__ __forceinline__ void stage_raw(uint64_t* sw, const uint64_t* __restrict__ rawbuf, uint64_t cta_off,
                                          int64_t nraw) {
#pragma unroll
  for (int i = 0; i < kStage; ++i) {
    const uint64_t j = cta_off + (uint64_t)threadIdx.x * kChunk + i;
    sw[i * kGauThreads + threadIdx.x] = j < (uint64_t)nraw ? __ldg(rawbuf + j) : 0ull;
  }
}

__device__ __forceinline__ double u01(uint64_t w) {
  return __dmul_rn((double)(w >> 11), 1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double dbits(uint64_t b) { return __longlong_as_double((long long)b); }

// One transducer move from state st at raw position p (word w0 = raw[p]).
// Returns words consumed; sets next state, emit flag and value.
// Ziggurat tables in shared memory: the 256-entry lookups are indexed by
// random bytes, which __constant__ memory serialises across a warp.
struct ZigSmem {
  uint64_t ki[256], wi[256], fi[256];
  __device__ void load() {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
      ki[i] = svdrec_zig::kKi[i];
      wi[i] = svdrec_zig::kWiBits[i];
      fi[i] = svdrec_zig::kFiBits[i];
    }
  }
};

template <class RawT>
__device__ __forceinline__ int move(int st, uint64_t p, RawT& raw, const ZigSmem& zt, int& nst, bool& emit,
                                    double& val) {
  const uint64_t w0 = raw.at(p);
  if (st == 0) {
    const uint32_t idx = (uint32_t)(w0 & 0xff);
    const uint64_t r = w0 >> 8;
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = __dmul_rn((double)rabs, dbits(zt.wi[idx]));
    if (r & 1) x = -x;
    if (rabs < zt.ki[idx]) {
      nst = 0;
      emit = true;
      val = x;
      return 1;
    }
    if (idx == 0) {
      nst = ((rabs >> 8) & 1) ? 2 : 1;
      emit = false;
      return 1;
    }
    const double fa = dbits(zt.fi[idx - 1]), fb = dbits(zt.fi[idx]);
    const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(fa, fb), u01(raw.ahead(p))), fb);
    nst = 0;
    emit = lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x));
    val = x;
    return 2;
  }
  const double R = dbits(svdrec_zig::kTailRBits), invR = dbits(svdrec_zig::kTailInvRBits);
  const double xx = __dmul_rn(-invR, log1p(-u01(w0)));
  const double yy = -log1p(-u01(raw.ahead(p)));
  if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
    nst = 0;
    emit = true;
    const double v = __dadd_rn(R, xx);
    val = (st == 2) ? -v : v;
  } else {
    nst = st;
    emit = false;
  }
  return 2;
}

__device__ __forceinline__ uint32_t compose(uint32_t a_e, const uint32_t* b) {
  const uint32_t bb = b[a_e & 7];
  return (((a_e >> 3) + (bb >> 3)) << 3) | (bb & 7);
}

// A0. the raw words of [pos0, pos0 + n): one thread per Philox block
__global__ void k_raw(uint64_t k0, uint64_t k1, const uint64_t* __restrict__ pos0p, int64_t n,
                      uint64_t* __restrict__ buf) {
  const uint64_t pos0 = *pos0p;
  const uint64_t b0 = pos0 >> 2;
  const uint64_t bi = b0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * bi >= pos0 + (uint64_t)n) return;
  uint64_t w[4];
  philox4x64(bi + 1, k0, k1, w[0], w[1], w[2], w[3]);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint64_t g = 4 * bi + j;
    if (g >= pos0 && g < pos0 + (uint64_t)n) buf[g - pos0] = w[j];
  }
}

__global__ void __launch_bounds__(kGauThreads) k_tables(const uint64_t* __restrict__ rawbuf,
                                                        const uint64_t* __restrict__ pos0p, int64_t nchunks,
                                                        int64_t nraw, uint32_t* __restrict__ tab) {
  __shared__ uint64_t sw[kStage * kGauThreads];
  __shared__ ZigSmem zt;
  const uint64_t cta_off = (uint64_t)blockIdx.x * kGauThreads * kChunk;
  stage_raw(sw, rawbuf, cta_off, nraw);
  zt.load();
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const uint64_t pos0 = *pos0p;
  const uint64_t base = pos0 + (uint64_t)c * kChunk, end = base + kChunk;
  RawSmem raw{sw + threadIdx.x, base};
  // primary walk from (offset 0, S); remember which (position, state) it
  // visits and how many samples it had emitted before each.
  uint8_t vis[kChunk + 1];
  uint8_t cum[kChunk + 1];
#pragma unroll
  for (int i = 0; i <= kChunk; ++i) vis[i] = 0xff;
  uint64_t p = base;
  int st = 0;
  uint32_t cnt = 0;
  while (p < end) {
    vis[p - base] = (uint8_t)st;
    cum[p - base] = (uint8_t)cnt;
    int nst;
    bool emit;
    double v;
    p += move(st, p, raw, zt, nst, emit, v);
    st = nst;
    cnt += emit;
  }
  const uint32_t p_exit = (uint32_t)((p - end) * 3 + st), p_cnt = cnt;
  tab[c * kCfg] = (p_cnt << 3) | p_exit;
  // the other five entries follow the primary as soon as they meet it
  for (int cfg = 1; cfg < kCfg; ++cfg) {
    uint64_t q = base + (cfg / 3);
    int s2 = cfg % 3;
    uint32_t c2 = 0;
    bool merged = false;
    while (q < end) {
      const uint32_t off = (uint32_t)(q - base);
      if (vis[off] == (uint8_t)s2) {
        c2 += p_cnt - cum[off];
        merged = true;
        break;
      }
      int nst;
      bool emit;
      double v;
      q += move(s2, q, raw, zt, nst, emit, v);
      s2 = nst;
      c2 += emit;
    }
    tab[c * kCfg + cfg] = merged ? ((c2 << 3) | p_exit) : ((c2 << 3) | (uint32_t)((q - end) * 3 + s2));
  }
}

__global__ void __launch_bounds__(kScan) k_scan(const uint32_t* __restrict__ tab, int64_t nchunks,
                                                uint32_t* __restrict__ incl, uint32_t* __restrict__ agg) {
  __shared__ uint32_t s[kScan][kCfg];
  const int t = threadIdx.x;
  const int64_t c = (int64_t)blockIdx.x * kScan + t;
  uint32_t cur[kCfg];
#pragma unroll
  for (int e = 0; e < kCfg; ++e) cur[e] = c < nchunks ? tab[c * kCfg + e] : (uint32_t)e;
#pragma unroll
  for (int e = 0; e < kCfg; ++e) s[t][e] = cur[e];
  __syncthreads();
  for (int d = 1; d < kScan; d <<= 1) {
    uint32_t nxt[kCfg];
    if (t >= d) {
#pragma unroll
      for (int e = 0; e < kCfg; ++e) nxt[e] = compose(s[t - d][e], cur);
    }
    __syncthreads();
    if (t >= d) {
#pragma unroll
      for (int e = 0; e < kCfg; ++e) {
        cur[e] = nxt[e];
        s[t][e] = nxt[e];
      }
    }
    __syncthreads();
  }
  if (c < nchunks) {
#pragma unroll
    for (int e = 0; e < kCfg; ++e) incl[c * kCfg + e] = cur[e];
  }
  if (t == kScan - 1) {
#pragma unroll
    for (int e = 0; e < kCfg; ++e) agg[(int64_t)blockIdx.x * kCfg + e] = cur[e];
  }
}

// C. thread the true entry configuration through the CTA aggregates: the
// aggregate tables are staged in shared memory by the whole CTA first, so
// the sequential walk is shared-memory latency, not L2 latency, per step.
constexpr int kChainMax = 1536;  // CTA aggregates staged in 36 KB (more: read from global)

__global__ void __launch_bounds__(1024) k_chain(const uint32_t* __restrict__ agg, int64_t nblocks, int64_t count,
                                                uint32_t* __restrict__ cta_cfg, int64_t* __restrict__ cta_off,
                                                uint32_t* d_status) {
  __shared__ uint32_t sa[kChainMax * kCfg];
  const int64_t ns = nblocks < kChainMax ? nblocks : kChainMax;
  for (int64_t i = threadIdx.x; i < ns * kCfg; i += blockDim.x) sa[i] = agg[i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t cfg = 0;
  int64_t off = 0;
  for (int64_t g = 0; g < nblocks; ++g) {
    cta_cfg[g] = cfg;
    cta_off[g] = off;
    const uint32_t a = g < ns ? sa[g * kCfg + cfg] : agg[g * kCfg + cfg];
    off += a >> 3;
    cfg = a & 7;
  }
  if (off < count && d_status) atomicOr(d_status, SVDREC_STATUS_STREAM_SHORT);
}

__global__ void k_read_pos(const int64_t* d_pos, uint64_t* dst) { *dst = (uint64_t)*d_pos; }

struct NormalPlan {
  int64_t nchunks, nblocks;
  size_t off_tab, off_incl, off_agg, off_cfg, off_off, off_pos, off_raw, total;
  int64_t nraw;
};

NormalPlan plan_for(int64_t count) {
  NormalPlan p{};
  const int64_t raw = count + count / 16 + 1024;
  p.nchunks = (raw + kChunk - 1) / kChunk;
  p.nblocks = (p.nchunks + kScan - 1) / kScan;
  size_t o = 0;
  p.off_tab = o;
  o = align_up(o + (size_t)p.nchunks * kCfg * 4);
  p.off_incl = o;
  o = align_up(o + (size_t)p.nchunks * kCfg * 4);
  p.off_agg = o;
  o = align_up(o + (size_t)p.nblocks * kCfg * 4);
  p.off_cfg = o;
  o = align_up(o + (size_t)p.nblocks * 4);
  p.off_off = o;
  o = align_up(o + (size_t)p.nblocks * 8);
  p.off_pos = o;
  o = align_up(o + 8);
  p.nraw = p.nchunks * kChunk + 4;  // + the look-ahead word of a chunk's last move
  p.off_raw = o;
  o = align_up(o + (size_t)p.nraw * 8);
  p.total = o;
  return p;
}

__global__ void __launch_bounds__(kGauThreads) k_emit_from(const uint64_t* __restrict__ rawbuf, int64_t nraw,
                                                           int64_t* __restrict__ d_pos, const uint64_t* pos0p,
                            int64_t nchunks, const uint32_t* __restrict__ incl,
                            const uint32_t* __restrict__ cta_cfg, const int64_t* __restrict__ cta_off_,
                            int64_t count, int64_t cols, const int32_t* __restrict__ perm,
                            double* __restrict__ out, int64_t ld) {
  __shared__ uint64_t sw[kStage * kGauThreads];
  __shared__ ZigSmem zt;
  const uint64_t cta_off = (uint64_t)blockIdx.x * kGauThreads * kChunk;
  stage_raw(sw, rawbuf, cta_off, nraw);
  zt.load();
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const uint64_t pos0 = *pos0p;
  const int64_t g = c / kScan;
  uint32_t cfg = cta_cfg[g];
  int64_t off = cta_off_[g];
  if (c % kScan) {
    const uint32_t a = incl[(c - 1) * kCfg + cfg];
    off += a >> 3;
    cfg = a & 7;
  }
  if (off >= count) return;
  const uint64_t base = pos0 + (uint64_t)c * kChunk, end = base + kChunk;
  uint64_t p = base + cfg / 3;
  int st = cfg % 3;
  int64_t row = off / cols, col = off - row * cols;  // one division; then carried
  RawSmem raw{sw + threadIdx.x, base};
  while (p < end && off < count) {
    int nst;
    bool emit;
    double v;
    const int used = move(st, p, raw, zt, nst, emit, v);
    if (emit) {
      out[(perm ? (int64_t)perm[row] : row) * ld + col] = v;
      if (off == count - 1) *d_pos = (int64_t)(p + used);
      ++off;
      if (++col == cols) {
        col = 0;
        ++row;
      }
    }
    p += used;
    st = nst;
  }
}

}  // namespace
}  // namespace svdrec

using namespace svdrec;

extern "C" size_t svdrec_normal_workspace_bytes(int64_t count) {
  return count <= 0 ? 256 : plan_for(count).total;
}

extern "C" int svdrec_normal_fill(uint64_t key_lo, uint64_t key_hi, int64_t* d_pos, int64_t count,
                                  int64_t cols, const int32_t* d_row_perm, double* d_out, int64_t ld,
                                  void* d_work, size_t work_bytes, uint32_t* d_status, void* stream) {
  SVDREC_ARG(count >= 0 && cols >= 1 && ld >= cols, "normal_fill: bad shape count=%lld cols=%lld ld=%lld",
             (long long)count, (long long)cols, (long long)ld);
  SVDREC_ARG(count % cols == 0, "normal_fill: count must be a multiple of cols");
  if (count == 0) return 0;
  const NormalPlan p = plan_for(count);
  if (work_bytes < p.total) {
    set_error("normal_fill: workspace %zu < %zu", work_bytes, p.total);
    return SVDREC_E_WORKSPACE;
  }
  char* w = static_cast<char*>(d_work);
  auto* tab = reinterpret_cast<uint32_t*>(w + p.off_tab);
  auto* incl = reinterpret_cast<uint32_t*>(w + p.off_incl);
  auto* agg = reinterpret_cast<uint32_t*>(w + p.off_agg);
  auto* ccfg = reinterpret_cast<uint32_t*>(w + p.off_cfg);
  auto* coff = reinterpret_cast<int64_t*>(w + p.off_off);
  auto* pos0 = reinterpret_cast<uint64_t*>(w + p.off_pos);
  cudaStream_t s = as_stream(stream);
  const int tb = kGauThreads;
  const unsigned grid = (unsigned)((p.nchunks + tb - 1) / tb);
  auto* rawbuf = reinterpret_cast<uint64_t*>(w + p.off_raw);
  k_read_pos<<<1, 1, 0, s>>>(d_pos, pos0);
  const int64_t nblk4 = p.nraw / 4 + 2;
  k_raw<<<(unsigned)((nblk4 + 255) / 256), 256, 0, s>>>(key_lo, key_hi, pos0, p.nraw, rawbuf);
  k_tables<<<grid, tb, 0, s>>>(rawbuf, pos0, p.nchunks, p.nraw, tab);
  k_scan<<<(unsigned)p.nblocks, kScan, 0, s>>>(tab, p.nchunks, incl, agg);
  k_chain<<<1, 1024, 0, s>>>(agg, p.nblocks, count, ccfg, coff, d_status);
  k_emit_from<<<grid, tb, 0, s>>>(rawbuf, p.nraw, d_pos, pos0, p.nchunks, incl, ccfg, coff, count, cols, d_row_perm,
                                   d_out, ld);
  return check_launch("normal_fill", 6);
}
