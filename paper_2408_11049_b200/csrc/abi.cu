// abi.cu — library-wide ABI entry points: version, thread-local error string, device query.

#include "md_internal.h"

namespace md {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

void clear_error() { g_last_error.clear(); }


int device_sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
  return n;
}

}  // namespace md

extern "C" int md_abi_version(void) { return MD_ABI_VERSION; }

extern "C" const char* md_last_error(void) { return md::g_last_error.c_str(); }
