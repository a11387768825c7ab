// Library-level entry points: version, thread-local error text, struct sizes.
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"

namespace isc {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return ISC_E_CUDA;
}

}  // namespace isc

extern "C" int isc_abi_version(void) { return ISC_ABI_VERSION; }

extern "C" const char* isc_last_error(void) { return isc::g_last_error.c_str(); }

extern "C" size_t isc_struct_size(int which) {
  switch (which) {
    case 0: return sizeof(isc_render_args);
    case 1: return sizeof(isc_source);
    case 2: return sizeof(isc_camera);
    case 3: return sizeof(isc_clip_plane);
    case 4: return sizeof(isc_chain_step);
    case 5: return sizeof(isc_swap_args);
    case 6: return sizeof(isc_toy_args);
    default: return 0;
  }
}

extern "C" int isc_device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}
