// abi.cu — version, error plumbing and device checks of the C ABI (include/sphinx.h).
#include "common.cuh"

namespace sphinx {

static thread_local int32_t g_last_cuda_error = 0;

sphinx_status cuda_fail(cudaError_t e) {
  g_last_cuda_error = static_cast<int32_t>(e);
  return SPHINX_ERR_CUDA;
}

sphinx_status check_device(int* sm_count) {
  static thread_local int cached_dev = -1;
  static thread_local int cached_ok = 0;
  static thread_local int cached_sms = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  if (dev != cached_dev) {
    int major = 0, minor = 0, sms = 0;
    if ((e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev)) != cudaSuccess)
      return cuda_fail(e);
    if ((e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev)) != cudaSuccess)
      return cuda_fail(e);
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
      return cuda_fail(e);
    cached_dev = dev;
    cached_ok = (major == 10 && minor == 0);
    cached_sms = sms;
  }
  if (sm_count) *sm_count = cached_sms;
  return cached_ok ? SPHINX_OK : SPHINX_ERR_DEVICE;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SPHINX_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

}  // namespace sphinx

extern "C" int32_t sphinx_abi_version(void) { return SPHINX_ABI_VERSION; }
extern "C" int32_t sphinx_last_cuda_error(void) { return sphinx::g_last_cuda_error; }
