// Library plumbing: error reporting, device attributes, ABI version.
#include <cstdarg>
#include <atomic>
#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"

namespace svdrec {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static std::atomic<long long> g_launches{0};

void note_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int sm_count() {
  static int n = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  });
  return n;
}

static std::mutex g_attr_mu;
static std::set<std::pair<const void*, int>> g_attr_done;

bool smem_attr_done(const void* kernel, int dev) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  return g_attr_done.count({kernel, dev}) != 0;
}

void smem_attr_mark(const void* kernel, int dev) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  g_attr_done.insert({kernel, dev});
}

}  // namespace svdrec

extern "C" int svdrec_abi_version(void) { return 1; }
extern "C" const char* svdrec_last_error(void) { return svdrec::g_err; }
extern "C" int svdrec_device_sm_count(void) { return svdrec::sm_count(); }
extern "C" long long svdrec_launch_count(void) { return svdrec::g_launches.load(); }

extern "C" int64_t svdrec_l2_window(void* stream, const void* d_base, int64_t bytes) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaStreamAttrValue v = {};
  if (bytes <= 0 || d_base == nullptr) {
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaGetLastError();
    return 0;
  }
  int dev = 0, maxp = 0, maxw = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  if (maxp <= 0 || maxw <= 0) return 0;
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
  if (cur < (size_t)maxp && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  const size_t nb = (size_t)bytes < (size_t)maxw ? (size_t)bytes : (size_t)maxw;
  v.accessPolicyWindow.base_ptr = const_cast<void*>(d_base);
  v.accessPolicyWindow.num_bytes = nb;
  const double ratio = (double)maxp / (double)nb;
  v.accessPolicyWindow.hitRatio = (float)(ratio < 1.0 ? ratio : 1.0);
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  if (cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return (int64_t)nb;
}
