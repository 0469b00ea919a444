// Library-level C ABI: version and thread-local error reporting.
#include <stdarg.h>

#include <atomic>

#include "hc_common.cuh"

namespace hc {
namespace {
thread_local char g_err[1024] = "";
std::atomic<unsigned long long> g_launches{0};
}  // namespace
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace hc

extern "C" const char* hc_version(void) { return "hcb200 0.1.0 (sm_100a)"; }
extern "C" const char* hc_last_error(void) { return hc::g_err; }
extern "C" unsigned long long hc_launch_count(void) { return hc::g_launches.load(); }
