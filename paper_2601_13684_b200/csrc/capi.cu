// Library-level C ABI: version and thread-local error reporting.
#include <stdarg.h>

#include "hc_common.cuh"

namespace hc {
namespace {
thread_local char g_err[1024] = "";
}
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace hc

extern "C" const char* hc_version(void) { return "hcb200 0.1.0 (sm_100a)"; }
extern "C" const char* hc_last_error(void) { return hc::g_err; }
