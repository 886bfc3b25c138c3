// Thread-local error message + ABI version (include/spaigraph_b200.h).
#include "common.cuh"

namespace sg {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return SG_ECUDA;
}

}  // namespace sg

extern "C" int sg_abi_version(void) { return 1; }

extern "C" const char* sg_last_error(void) { return sg::g_last_error.c_str(); }
