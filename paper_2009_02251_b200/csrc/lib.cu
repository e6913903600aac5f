// Library plumbing: error reporting, device attributes, ABI version.
#include <cstdarg>
#include <atomic>
#include <mutex>

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

}  // namespace svdrec

extern "C" int svdrec_abi_version(void) { return 1; }
extern "C" const char* svdrec_last_error(void) { return svdrec::g_err; }
extern "C" int svdrec_device_sm_count(void) { return svdrec::sm_count(); }
extern "C" long long svdrec_launch_count(void) { return svdrec::g_launches.load(); }
