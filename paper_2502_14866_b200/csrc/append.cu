// K1 -- paged-KV append: quantise + page bounds + logical-page key stats.
//
// Replaces HeadPages.append / _rebuild_open_page / quantize_page /
// PageStats.from_keys / _evict_outside_window (reference cache.py:189-261,
// cache.py:20-51, cache.py:59-73).  One CTA rebuilds one (stream, page):
// the page's raw tokens come from the open-page staging (tokens already in
// the page) and from the new tokens; lo/hi per channel, codes
// clip(rint((x-lo)/scale)) in fp64 (bit-exact with numpy's round-half-even),
// and the (k_min, k_max) of every logical page are recomputed from raw data,
// exactly like the reference re-quantises the open page on every append.
// HBM-bound: reads the raw page once, writes codes + bounds + stats.
#include "append_impl.cuh"

namespace sk {

namespace {

template <typename T>
__global__ void __launch_bounds__(256) append_kernel(PoolView pv, const T* __restrict__ k_src,
                                                     const T* __restrict__ v_src, int64_t src_ss, int64_t src_ts,
                                                     const int32_t* __restrict__ tokens, int m) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int s = blockIdx.y;
  const int n0 = tokens[s];
  const int n1 = n0 + m;
  const int p = n0 / pv.P + blockIdx.x;
  if (p > (n1 - 1) / pv.P) return;
  append_page<T>(pv, s, p, n0, n1, k_src + s * src_ss, v_src + s * src_ss, src_ts, smem);
}

// One new token per stream (decode): a cluster of kAppendParts CTAs per
// stream (append_one_part), or its first CTA alone for a fresh page / raw
// pool (append_page); the cluster barrier orders every part's read of the
// stream's token count before part 0 advances it.
template <typename T>
__global__ void __launch_bounds__(256) append_one_kernel(PoolView pv, const T* __restrict__ k_src,
                                                         const T* __restrict__ v_src, int64_t src_ss,
                                                         int32_t* __restrict__ tokens) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int part = blockIdx.x, s = blockIdx.y;
  const int n0 = tokens[s];
  const T* kn = k_src + s * src_ss;
  const T* vn = v_src + s * src_ss;
  if (n0 % pv.P == 0 || pv.bits == 0) {
    if (part == 0) append_page<T>(pv, s, n0 / pv.P, n0, n0 + 1, kn, vn, 0, smem);
  } else {
    append_one_part<T>(pv, s, part, n0, kn, vn, smem);
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (part == 0 && threadIdx.x == 0) tokens[s] = n0 + 1;
}

__global__ void advance_tokens_kernel(int32_t* tokens, int n, int m) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) tokens[i] += m;
}

}  // namespace

int append_launch(const sk_pool* pool, int n_streams, const void* k_src, const void* v_src, int64_t ss, int64_t ts,
                  int32_t* tokens, int m, int max_pages_touched, cudaStream_t st) {
  int rc = check_pool(pool);
  if (rc) return rc;
  SK_CHECK_ARG(n_streams >= 1 && m >= 1 && max_pages_touched >= 1, "append: empty launch");
  SK_CHECK_ARG(k_src && v_src && tokens, "append: NULL pointer");
  SK_CHECK_ARG(ss % 8 == 0 && (ts % 8 == 0 || m == 1), "append: source strides must be multiples of 8 elements");
  SK_CHECK_ARG(pool->page_size % (pool->bits >= 1 && pool->bits <= 4 ? 32 : 16) == 0,
               "append: page_size must be a multiple of 32 (<=4-bit codes) or 16");
  PoolView pv = make_view(*pool);
  if (m == 1) {
    size_t smem1 = append_smem_bytes(pv.D, pv.P);
    size_t smem2 = append_part_smem_bytes(pv.D, pv.P);
    size_t sm = smem1 > smem2 ? smem1 : smem2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kAppendParts, n_streams, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kAppendParts;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (pv.dtype == SK_F16) {
      cudaFuncSetAttribute(append_one_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      e = cudaLaunchKernelEx(&cfg, append_one_kernel<__half>, pv, (const __half*)k_src, (const __half*)v_src, ss,
                             tokens);
    } else {
      cudaFuncSetAttribute(append_one_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      e = cudaLaunchKernelEx(&cfg, append_one_kernel<__nv_bfloat16>, pv, (const __nv_bfloat16*)k_src,
                             (const __nv_bfloat16*)v_src, ss, tokens);
    }
    if (e != cudaSuccess) {
      set_error(std::string("append_one_kernel: ") + cudaGetErrorString(e));
      return SK_ECUDA;
    }
    SK_CHECK_LAUNCH("append_one_kernel");
    return SK_OK;
  }
  size_t smem = append_smem_bytes(pv.D, pv.P);
  dim3 grid(max_pages_touched, n_streams);
  if (pv.dtype == SK_F16) {
    cudaFuncSetAttribute(append_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    append_kernel<__half><<<grid, 256, smem, st>>>(pv, (const __half*)k_src, (const __half*)v_src, ss, ts,
                                                   tokens, m);
  } else {
    cudaFuncSetAttribute(append_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    append_kernel<__nv_bfloat16><<<grid, 256, smem, st>>>(pv, (const __nv_bfloat16*)k_src,
                                                          (const __nv_bfloat16*)v_src, ss, ts, tokens, m);
  }
  SK_CHECK_LAUNCH("append_kernel");
  advance_tokens_kernel<<<(n_streams + 255) / 256, 256, 0, st>>>(tokens, n_streams, m);
  SK_CHECK_LAUNCH("advance_tokens_kernel");
  return SK_OK;
}

}  // namespace sk

extern "C" int sk_append_pages(const sk_pool* pool, int32_t n_streams, const void* k_src, const void* v_src,
                               int64_t src_stream_stride, int64_t src_token_stride, int32_t* tokens,
                               int32_t m_tokens, int32_t max_pages_touched, void* stream) {
  return sk::append_launch(pool, n_streams, k_src, v_src, src_stream_stride, src_token_stride, tokens, m_tokens,
                           max_pages_touched, static_cast<cudaStream_t>(stream));
}
