// Library plumbing: error reporting, device attributes, ABI version.
#include <cstdarg>
#include <atomic>
#include <mutex>
#include <map>
#include <set>
#include <tuple>
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

// SM count of the CURRENT device (a process may drive several GPUs)
int sm_count() {
  static std::mutex mu;
  static std::map<int, int> per_dev;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = per_dev.find(dev);
  if (it != per_dev.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  per_dev[dev] = n;
  return n;
}

// cudaOccupancyMaxActiveBlocksPerMultiprocessor cached per (kernel, device,
// block size, dynamic shared memory)
cudaError_t blocks_per_sm(const void* kernel, int threads, size_t smem, int* out) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, size_t>, int> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_tuple(kernel, dev, threads, smem);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return cudaSuccess;
    }
  }
  int n = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = n;
  *out = n;
  return cudaSuccess;
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
