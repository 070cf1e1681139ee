// Status / version plumbing of the C ABI (include/slideconv_b200.h).
#include <string>

#include "common.cuh"

namespace sc {
namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return SC_ERR_CUDA;
}

}  // namespace sc

extern "C" int sc_version(void) { return 10000; }

extern "C" const char* sc_last_error(void) { return sc::g_last_error.c_str(); }
