// K1b -- pool gather: dequantise the resident pages of a pool back into a
// token-major K/V history [tokens, streams, D] in the pool dtype.
//
// This is the history read of a chunked (continued) prefill: K4 streams K/V
// tiles with TMA, which cannot dequantise, so the cached part of the context
// is expanded once per chunk and the chunk's own raw K/V are placed after it.
// The values are those of PhysicalPage.dequantize (reference cache.py:54-56,
// cache.py:97-102: code * scale + zero, scale = (hi - lo) / (2^b - 1), 1 where
// that is not > 0) cast to the attention dtype, i.e. exactly what the decode
// path feeds its MMAs (reference engine.py:250-262).  Evicted pages of
// streaming streams are not written (no schedule visits them).
// HBM-bound: reads codes + bounds once (16-byte loads staged in shared
// memory), writes 2 * P * D values per page as 16-byte stores.
#include "sk_common.cuh"
#include "sk_layout.cuh"

namespace sk {

namespace {

template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b);
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// One CTA per (page, stream): the slot's K and V code regions are staged in
// shared memory with 16-byte loads, then every thread emits 8 consecutive
// channels of one token (one 16-byte store) for K and for V.
template <typename T>
__global__ void __launch_bounds__(256) gather_kernel(PoolView pv, T* __restrict__ k_out, T* __restrict__ v_out,
                                                     int64_t oss, int64_t ots, int n_tok) {
  extern __shared__ __align__(16) uint8_t s_codes[];  // [K region | V region] = 2 * P * row_bytes
  __shared__ float s_sc[4][128];                      // k_scale, k_lo, v_scale, v_lo (natural channel order)
  const int s = blockIdx.y, p = blockIdx.x;
  const int D = pv.D, P = pv.P;
  const int n_pages = (n_tok + P - 1) / P;
  if (p >= n_pages) return;
  if (pv.kind[s] != SK_KIND_DENSE && !in_lambda(p, n_pages, pv.sink, pv.local)) return;
  const uint8_t* slot = pv.slot_ptr(s, p);
  const int t_end = min(P, n_tok - p * P);
  const int tid = threadIdx.x;
  const int region = P * pv.row_bytes;
  {
    const uint4* src = reinterpret_cast<const uint4*>(slot);
    uint4* dst = reinterpret_cast<uint4*>(s_codes);
    // V (<=4-bit) rows of different channel octets m all start on the same
    // bank; XOR the 16-byte chunk index with m % 8 so a warp's 16 octets
    // spread over the banks (the reader applies the same swizzle).
    const int vsw = pv.bits >= 1 && pv.bits <= 4 ? 1 : 0;
    for (int i = tid; i < 2 * region / 16; i += blockDim.x) {
      int c = i;
      if (vsw && i >= region / 16) {
        int cv = i - region / 16;
        c = region / 16 + (cv ^ ((cv / (P / 4)) & 7));
      }
      dst[c] = __ldg(src + i);
    }
  }
  if (pv.bits) {
    const T* b = reinterpret_cast<const T*>(slot + 2 * region);
    const float levels = (float)((1 << pv.bits) - 1);
    for (int d = tid; d < D; d += blockDim.x) {
      float klo = DT<T>::to_f(b[kbound_pos(d, D)]), khi = DT<T>::to_f(b[D + kbound_pos(d, D)]);
      float vlo = DT<T>::to_f(b[2 * D + vbound_pos(d, D)]), vhi = DT<T>::to_f(b[3 * D + vbound_pos(d, D)]);
      float ks = (khi - klo) / levels, vs = (vhi - vlo) / levels;
      s_sc[0][d] = ks > 0.f ? ks : 1.f;
      s_sc[1][d] = klo;
      s_sc[2][d] = vs > 0.f ? vs : 1.f;
      s_sc[3][d] = vlo;
    }
  }
  __syncthreads();
  const uint8_t* kc = s_codes;
  const uint8_t* vc = s_codes + region;
  T* ko = k_out + (int64_t)p * P * ots + s * oss;
  T* vo = v_out + (int64_t)p * P * ots + s * oss;
  const int groups = D / 8;
  for (int i = tid; i < t_end * groups; i += blockDim.x) {
    const int t = i / groups, d0 = (i % groups) * 8;
    uint32_t kw[4], vw[4];
    if (pv.bits == 0) {
      const T* kr = reinterpret_cast<const T*>(kc);
      const T* vr = reinterpret_cast<const T*>(vc);
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        T a = kr[kpos_raw(t, d0 + e, D)], b = kr[kpos_raw(t, d0 + e + 1, D)];
        T c = vr[vpos_raw(t, d0 + e, P)], d = vr[vpos_raw(t, d0 + e + 1, P)];
        kw[e / 2] = (uint32_t)(*reinterpret_cast<uint16_t*>(&a)) | ((uint32_t)(*reinterpret_cast<uint16_t*>(&b)) << 16);
        vw[e / 2] = (uint32_t)(*reinterpret_cast<uint16_t*>(&c)) | ((uint32_t)(*reinterpret_cast<uint16_t*>(&d)) << 16);
      }
    } else {
      float kx[8], vx[8];
      if (pv.bits <= 4) {
        // sk_layout.cuh word view: channels 8m+2j+e of token t sit in the
        // 32-bit word t*D/2 + j*D/8 + (m/4)*4 at bit 4*(m%4) + 16e; channel
        // 8m+i of token t in word (32m + 4i + (t%8)/2)*P/8 + (t/32)*4 at bit
        // 4*((t/8)%4) + 16*(t%2).
        const int m = d0 / 8;
        const uint8_t* kb = kc + t * (D / 2) + (m / 4) * 4;
        const int ksh = 4 * (m % 4);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t w = *reinterpret_cast<const uint32_t*>(kb + j * (D / 8));
          kx[2 * j] = (float)((w >> ksh) & 0xF);
          kx[2 * j + 1] = (float)((w >> (16 + ksh)) & 0xF);
        }
        const int vb = (32 * m + (t % 8) / 2) * (P / 8) + (t / 32) * 4;
        const int vsh = 4 * ((t / 8) % 4) + 16 * (t % 2);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int byte = (vb + 4 * i * (P / 8)) ^ ((m & 7) << 4);
          vx[i] = (float)((*reinterpret_cast<const uint32_t*>(vc + byte) >> vsh) & 0xF);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          kx[e] = (float)kc[kpos_byte(t, d0 + e, D)];
          vx[e] = (float)vc[vpos_byte(t, d0 + e, P)];
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        kx[e] = fmaf(kx[e], s_sc[0][d0 + e], s_sc[1][d0 + e]);
        vx[e] = fmaf(vx[e], s_sc[2][d0 + e], s_sc[3][d0 + e]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        kw[e] = pack2<T>(kx[2 * e], kx[2 * e + 1]);
        vw[e] = pack2<T>(vx[2 * e], vx[2 * e + 1]);
      }
    }
    *reinterpret_cast<uint4*>(ko + t * ots + d0) = make_uint4(kw[0], kw[1], kw[2], kw[3]);
    *reinterpret_cast<uint4*>(vo + t * ots + d0) = make_uint4(vw[0], vw[1], vw[2], vw[3]);
  }
}

}  // namespace

int gather_launch(const sk_pool* pool, int n_streams, int n_tokens, void* k_out, void* v_out, int64_t oss,
                  int64_t ots, cudaStream_t st) {
  int rc = check_pool(pool);
  if (rc) return rc;
  SK_CHECK_ARG(n_streams >= 1 && n_tokens >= 1, "gather: empty launch");
  SK_CHECK_ARG(k_out && v_out, "gather: NULL pointer");
  SK_CHECK_ARG(oss >= pool->head_dim && ots >= oss * n_streams, "gather: output strides overlap");
  SK_CHECK_ARG((int64_t)(n_tokens + pool->page_size - 1) / pool->page_size <= pool->max_pages,
               "gather: more tokens than the pool holds");
  SK_CHECK_ARG(oss % 8 == 0 && ots % 8 == 0 && ((uintptr_t)k_out | (uintptr_t)v_out) % 16 == 0,
               "gather: outputs must be 16-byte aligned with strides in multiples of 8 elements");
  PoolView pv = make_view(*pool);
  dim3 grid((n_tokens + pv.P - 1) / pv.P, n_streams);
  const int smem = 2 * pv.P * pv.row_bytes;
  if (pv.dtype == SK_F16) {
    cudaFuncSetAttribute(gather_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    gather_kernel<__half><<<grid, 256, smem, st>>>(pv, (__half*)k_out, (__half*)v_out, oss, ots, n_tokens);
  } else {
    cudaFuncSetAttribute(gather_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    gather_kernel<__nv_bfloat16><<<grid, 256, smem, st>>>(pv, (__nv_bfloat16*)k_out, (__nv_bfloat16*)v_out, oss,
                                                          ots, n_tokens);
  }
  SK_CHECK_LAUNCH("gather_kernel");
  return SK_OK;
}

}  // namespace sk

extern "C" int sk_gather_pages(const sk_pool* pool, int32_t n_streams, int32_t n_tokens, void* k_out, void* v_out,
                               int64_t out_stream_stride, int64_t out_token_stride, void* stream) {
  return sk::gather_launch(pool, n_streams, n_tokens, k_out, v_out, out_stream_stride, out_token_stride,
                           static_cast<cudaStream_t>(stream));
}
