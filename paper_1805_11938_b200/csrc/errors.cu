// Thread-local error message and ABI version (include/spmvb.h).
#include "common.cuh"

namespace spmvb {
std::atomic<unsigned long long> g_launches{0};
namespace {
thread_local std::string g_last_error;
}

void set_error_message(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}
}  // namespace spmvb

extern "C" const char* spmvb_last_error(void) { return spmvb::g_last_error.c_str(); }
extern "C" int spmvb_abi_version(void) { return SPMVB_ABI_VERSION; }
extern "C" unsigned long long spmvb_launch_count(void) { return spmvb::g_launches.load(); }
