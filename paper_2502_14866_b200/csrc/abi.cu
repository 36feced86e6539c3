// C-ABI utilities: version, thread-local error text, device check.
#include <string>

#include "sk_common.cuh"

namespace sk {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace sk

extern "C" const char* sk_version(void) { return "sparsekv-b200 0.1.0 (sm_100a; tcgen05 prefill, mma.sync decode)"; }

extern "C" const char* sk_last_error(void) { return sk::g_last_error.c_str(); }

extern "C" int sk_device_supported(int dev) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return 0;
  return prop.major == 10 && prop.minor == 0 ? 1 : 0;
}

extern "C" int64_t sk_slot_bytes(int32_t head_dim, int32_t page_size, int32_t bits, int32_t dtype) {
  (void)dtype;
  return sk::slot_bytes_of(head_dim, page_size, bits);
}
