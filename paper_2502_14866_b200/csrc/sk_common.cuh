// Shared definitions for the sparsekv-b200 kernels: pool layout, dtype
// traits, error reporting.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/sparsekv_b200.h"

namespace sk {

void set_error(const std::string& msg);

#define SK_CHECK_ARG(cond, msg)  \
  do {                           \
    if (!(cond)) {               \
      ::sk::set_error(msg);      \
      return SK_EINVAL;          \
    }                            \
  } while (0)

#define SK_CHECK_LAUNCH(what)                                                        \
  do {                                                                               \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess) {                                                         \
      ::sk::set_error(std::string(what) + ": " + cudaGetErrorString(_e));            \
      return SK_ECUDA;                                                               \
    }                                                                                \
  } while (0)

// ---- dtype traits -----------------------------------------------------------
template <typename T>
struct DT;
template <>
struct DT<__half> {
  static __device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
  static __device__ __forceinline__ __half from_f(float x) { return __float2half_rn(x); }
  static __device__ __forceinline__ float2 to_f2(uint32_t w) {
    return __half22float2(*reinterpret_cast<__half2*>(&w));
  }
};
template <>
struct DT<__nv_bfloat16> {
  static __device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  static __device__ __forceinline__ __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
  static __device__ __forceinline__ float2 to_f2(uint32_t w) {
    return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w));
  }
};

// ---- pool layout --------------------------------------------------------------
__host__ __device__ inline int code_row_bytes(int head_dim, int bits) {
  return bits == 0 ? head_dim * 2 : (bits <= 4 ? head_dim / 2 : head_dim);
}
__host__ __device__ inline int64_t slot_bytes_of(int head_dim, int page, int bits) {
  int64_t b = 2ll * page * code_row_bytes(head_dim, bits) + (bits ? 8ll * head_dim : 0);
  return (b + 127) / 128 * 128;
}

// Plain-old-data copy of sk_pool passed by value to kernels.
struct PoolView {
  int dtype, D, P, L, bits, max_pages, sink, local;
  int64_t slot_bytes;
  uint8_t* arena;
  const int32_t* page_table;
  uint8_t* stats;
  uint8_t* staging;
  const uint8_t* kind;
  int row_bytes;  // code row bytes

  __device__ __forceinline__ uint8_t* slot_ptr(int stream, int page) const {
    int32_t slot = page_table[(int64_t)stream * max_pages + page];
    return arena + (int64_t)slot * slot_bytes;
  }
  __device__ __forceinline__ uint8_t* k_codes(uint8_t* slot) const { return slot; }
  __device__ __forceinline__ uint8_t* v_codes(uint8_t* slot) const { return slot + (int64_t)P * row_bytes; }
  // bounds: [4][D] of dtype (k_lo, k_hi, v_lo, v_hi)
  __device__ __forceinline__ uint8_t* bounds(uint8_t* slot) const { return slot + 2ll * P * row_bytes; }
  __device__ __forceinline__ uint8_t* stats_ptr(int stream, int logical) const {
    return stats + (((int64_t)stream * max_pages * (P / L) + logical) * 2 * D) * 2;
  }
  __device__ __forceinline__ uint8_t* staging_ptr(int stream, int which) const {
    return staging + (((int64_t)stream * 2 + which) * P * D) * 2;
  }
};

inline PoolView make_view(const sk_pool& p) {
  PoolView v;
  v.dtype = p.dtype;
  v.D = p.head_dim;
  v.P = p.page_size;
  v.L = p.logical_page;
  v.bits = p.bits;
  v.max_pages = p.max_pages;
  v.sink = p.sink;
  v.local = p.local;
  v.slot_bytes = p.slot_bytes;
  v.arena = static_cast<uint8_t*>(p.arena);
  v.page_table = p.page_table;
  v.stats = static_cast<uint8_t*>(p.stats);
  v.staging = static_cast<uint8_t*>(p.staging);
  v.kind = p.kind;
  v.row_bytes = code_row_bytes(p.head_dim, p.bits);
  return v;
}

inline int check_pool(const sk_pool* p) {
  SK_CHECK_ARG(p != nullptr, "pool is NULL");
  SK_CHECK_ARG(p->dtype == SK_F16 || p->dtype == SK_BF16, "pool dtype must be f16 or bf16");
  SK_CHECK_ARG(p->head_dim == 64 || p->head_dim == 128, "head_dim must be 64 or 128 (pad smaller dims)");
  SK_CHECK_ARG(p->page_size >= 1 && p->page_size <= 128, "page_size must be in [1, 128]");
  SK_CHECK_ARG(p->logical_page >= 1 && p->page_size % p->logical_page == 0,
               "logical page size must divide physical page size");
  SK_CHECK_ARG(p->bits == 0 || (p->bits >= 2 && p->bits <= 8), "bits must be 0 or in [2, 8]");
  SK_CHECK_ARG(p->slot_bytes >= slot_bytes_of(p->head_dim, p->page_size, p->bits), "slot_bytes too small");
  SK_CHECK_ARG(p->arena && p->page_table && p->staging && p->kind, "pool buffers must be non-NULL");
  return SK_OK;
}

// SM count of the current device (cached per device; host only).
inline int device_sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// streaming-window membership of page p among n pages (heads.py:107-125 at
// query tile n-1): sink_end = min(sink, n), local_start = max(n - local, 0).
__host__ __device__ inline bool in_lambda(int p, int n, int sink, int local) {
  int sink_end = sink < n ? sink : n;
  int local_start = n - local > 0 ? n - local : 0;
  return p < sink_end || p >= local_start;
}

}  // namespace sk
