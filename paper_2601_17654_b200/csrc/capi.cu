// capi.cu — library-level C ABI: error convention, version, device facts.
#include "common.cuh"

namespace kpo {
static thread_local char g_last_error[1024] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}
}  // namespace kpo

extern "C" const char* kpo_last_error(void) { return kpo::g_last_error; }

extern "C" int kpo_version(void) { return 1; }

extern "C" int kpo_device_info(int device, int* num_sms, int* smem_optin_bytes, int* cc_major, int* cc_minor) {
  KPO_CHECK_ARG(num_sms && smem_optin_bytes && cc_major && cc_minor, "device_info: null output");
  KPO_CUDA(cudaDeviceGetAttribute(num_sms, cudaDevAttrMultiProcessorCount, device));
  KPO_CUDA(cudaDeviceGetAttribute(smem_optin_bytes, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  KPO_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device));
  KPO_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  return KPO_OK;
}
