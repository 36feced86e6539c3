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

// One new token per stream (decode), for up to kMaxAppendLayers pools of one
// geometry in one launch (a decode step's appends of several layers): grid
// (kAppendParts, streams, layers), a cluster of kAppendParts CTAs per
// (layer, stream) running append_one_part -- or its first CTA alone for a
// fresh page / raw pool (append_page); the cluster barrier orders every
// part's read of the stream's token count before part 0 advances it.
constexpr int kMaxAppendLayers = 32;
struct AppendLayers {
  PoolView pv[kMaxAppendLayers];
  int32_t* tokens[kMaxAppendLayers];
  const void* k;
  const void* v;
  int64_t layer_stride, stream_stride;
};

template <typename T>
__global__ void __launch_bounds__(256) append_one_kernel(const __grid_constant__ AppendLayers a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int part = blockIdx.x, s = blockIdx.y, l = blockIdx.z;
  const PoolView& pv = a.pv[l];
  int32_t* tokens = a.tokens[l];
  const int n0 = tokens[s];
  const T* kn = reinterpret_cast<const T*>(a.k) + l * a.layer_stride + s * a.stream_stride;
  const T* vn = reinterpret_cast<const T*>(a.v) + l * a.layer_stride + s * a.stream_stride;
  if (n0 % pv.P == 0 || pv.bits == 0 || gridDim.x == 1) {  // fresh page / raw pool / one CTA per stream
    if (part == 0) append_page<T>(pv, s, n0 / pv.P, n0, n0 + 1, kn, vn, 0, smem);
  } else {
    append_one_part<T>(pv, s, part, n0, kn, vn, smem);
  }
  if (gridDim.x > 1)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  if (part == 0 && threadIdx.x == 0) tokens[s] = n0 + 1;
}

// Parts per (layer, stream): a cluster of kAppendParts when the appends are
// few (latency), one CTA rebuilding the page (append_page) once they alone
// fill the GPU several times over (cfg4's 128 streams x 8 layers).
template <typename T>
int append_one_launch(const AppendLayers& a, int n_layers, int n_streams, size_t smem, cudaStream_t st) {
  const int parts = (int64_t)n_layers * n_streams > 2 * device_sm_count() ? 1 : kAppendParts;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(parts, n_streams, n_layers);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = parts;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = parts > 1 ? 1 : 0;
  cudaFuncSetAttribute(append_one_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaError_t e = cudaLaunchKernelEx(&cfg, append_one_kernel<T>, a);
  if (e != cudaSuccess) {
    set_error(std::string("append_one_kernel: ") + cudaGetErrorString(e));
    return SK_ECUDA;
  }
  SK_CHECK_LAUNCH("append_one_kernel");
  return SK_OK;
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
    AppendLayers a;
    a.pv[0] = pv;
    a.tokens[0] = tokens;
    a.k = k_src;
    a.v = v_src;
    a.layer_stride = 0;
    a.stream_stride = ss;
    size_t smem1 = append_smem_bytes(pv.D, pv.P), smem2 = append_part_smem_bytes(pv.D, pv.P);
    const size_t sm = smem1 > smem2 ? smem1 : smem2;
    return pv.dtype == SK_F16 ? append_one_launch<__half>(a, 1, n_streams, sm, st)
                              : append_one_launch<__nv_bfloat16>(a, 1, n_streams, sm, st);
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

extern "C" int sk_append_token_layers(const sk_pool* pools, int32_t n_layers, int32_t n_streams, const void* k_src,
                                      const void* v_src, int64_t src_layer_stride, int64_t src_stream_stride,
                                      int32_t* const* tokens, void* stream) {
  using namespace sk;
  SK_CHECK_ARG(pools != nullptr && tokens != nullptr && n_layers >= 1 && n_streams >= 1, "append: empty launch");
  SK_CHECK_ARG(k_src && v_src, "append: NULL pointer");
  SK_CHECK_ARG(src_stream_stride % 8 == 0 && src_layer_stride % 8 == 0,
               "append: source strides must be multiples of 8 elements");
  for (int l = 0; l < n_layers; ++l) {
    int rc = check_pool(&pools[l]);
    if (rc) return rc;
    SK_CHECK_ARG(tokens[l] != nullptr, "append: NULL token counter");
    SK_CHECK_ARG(pools[l].dtype == pools[0].dtype && pools[l].head_dim == pools[0].head_dim &&
                     pools[l].page_size == pools[0].page_size && pools[l].bits == pools[0].bits,
                 "append: the layers' pools must share dtype, head_dim, page_size and bits");
    SK_CHECK_ARG(pools[l].page_size % (pools[l].bits >= 1 && pools[l].bits <= 4 ? 32 : 16) == 0,
                 "append: page_size must be a multiple of 32 (<=4-bit codes) or 16");
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int D = pools[0].head_dim, P = pools[0].page_size;
  size_t smem1 = append_smem_bytes(D, P), smem2 = append_part_smem_bytes(D, P);
  const size_t sm = smem1 > smem2 ? smem1 : smem2;
  for (int l0 = 0; l0 < n_layers; l0 += kMaxAppendLayers) {
    const int nl = n_layers - l0 < kMaxAppendLayers ? n_layers - l0 : kMaxAppendLayers;
    AppendLayers a;
    for (int i = 0; i < nl; ++i) {
      a.pv[i] = make_view(pools[l0 + i]);
      a.tokens[i] = tokens[l0 + i];
    }
    const int64_t el = 2;  // fp16 / bf16 elements
    a.k = static_cast<const uint8_t*>(k_src) + l0 * src_layer_stride * el;
    a.v = static_cast<const uint8_t*>(v_src) + l0 * src_layer_stride * el;
    a.layer_stride = src_layer_stride;
    a.stream_stride = src_stream_stride;
    int rc = pools[0].dtype == SK_F16 ? append_one_launch<__half>(a, nl, n_streams, sm, st)
                                      : append_one_launch<__nv_bfloat16>(a, nl, n_streams, sm, st);
    if (rc) return rc;
  }
  return SK_OK;
}
