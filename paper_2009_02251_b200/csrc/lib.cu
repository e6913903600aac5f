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
