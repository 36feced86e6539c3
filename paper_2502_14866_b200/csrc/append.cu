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

#ifndef SK_APPEND_FAST  // 0: every page through the generic rebuild (A/B builds)
#define SK_APPEND_FAST 1
#endif
#ifndef SK_APPEND_SFIRST
#define SK_APPEND_SFIRST 1
#endif
#ifndef SK_APPEND_MINB  // resident CTAs per SM the bulk kernel is compiled for
#define SK_APPEND_MINB 3
#endif

namespace sk {

namespace {

// Code of x from the fp32 quotient t32 = (x - lo) * (1/scale), rounded to
// nearest-even by the 1.5 * 2^23 magic add (FMA pipe, no F2I / FRND).
// t32 is within |t| * 2^-22.4 <= 2^-18.4 of numpy's fp64 quotient for
// t <= 15 (bits <= 4), so rint(t32) is numpy's np.round unless t32 lies
// within 2^-16 of a .5 tie; those (about 1 in 2^15 values) take the exact
// fp64 path (quant_code), kept
// out of line so the compiler cannot if-convert (predicate) its fp64
// instructions into every value's fast path.
__device__ __noinline__ uint32_t qcode_exact(float x, double lo, double sc, double inv, int levels) {
  return quant_code((double)x, lo, sc, inv, levels);
}
// packed fp32x2 (FADD2 / FMUL2 / FFMA2 on sm_100)
__device__ __forceinline__ uint64_t f2p(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2u(uint64_t r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ uint64_t f2add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// Codes of the two values of a T pair (channels ci, ci + 1) as n0 | n1 << 16:
// t = (x - lo) * inv and the magic add as packed pairs, the two code bytes
// gathered by one PRMT (byte 1 of 1.5 * 2^23 + n is zero).  A near-tie takes
// qcode_exact.
template <typename T>
__device__ __forceinline__ uint32_t qpair(uint32_t raw, uint64_t nlo2, uint64_t inv2, const double* lo64,
                                         const double* sc64, const double* inv64, int ci, int levels) {
  const float2 x = DT<T>::to_f2(raw);
  const uint64_t t2 = f2mul(f2add(f2p(x.x, x.y), nlo2), inv2);
  const uint64_t r2 = f2add(t2, f2p(12582912.f, 12582912.f));
  const float2 d = f2u(f2fma(f2add(r2, f2p(-12582912.f, -12582912.f)), f2p(-1.f, -1.f), t2));
  const float2 r = f2u(r2);
  const bool tie0 = fabsf(fabsf(d.x) - 0.5f) < 0x1p-16f, tie1 = fabsf(fabsf(d.y) - 0.5f) < 0x1p-16f;
  if (tie0 || tie1) {
    const uint32_t c0 = tie0 ? qcode_exact(x.x, lo64[ci], sc64[ci], inv64[ci], levels) : __float_as_uint(r.x) & 0xFFu;
    const uint32_t c1 =
        tie1 ? qcode_exact(x.y, lo64[ci + 1], sc64[ci + 1], inv64[ci + 1], levels) : __float_as_uint(r.y) & 0xFFu;
    return c0 | (c1 << 16);
  }
  return __byte_perm(__float_as_uint(r.x), __float_as_uint(r.y), 0x1410);
}

// Full-page fast path of the bulk append: a KV4 (bits <= 4) page of 64 new
// tokens, D = 128, logical pages of 16.  The raw page never touches shared
// memory: warp wq = (w, j) = (wq / 4, wq % 4) and lane (m, e) = (lane % 16,
// lane / 16) hold tokens t_i = 32w + 8i + 2j + e (i < 4) at dims
// 32(m/4) + 2(m%4) + 8sl + {0, 1} (sl < 4) of K and V, so a thread owns every
// nibble of the K word (t_i, j = m%4, w = m/4) and, with its lane^16 partner,
// the V words (channel, j, w) of its eight channels (sk_layout.cuh).  Only the
// per-channel min / max reductions go through shared memory.
// 1. raw K / V pairs, 16 x 4 bytes each per thread (a warp instruction reads
//    eight 16-byte runs of two token rows; the sl instructions share sectors in L1)
template <typename T>
__device__ __forceinline__ void load_full_kv4(const T* __restrict__ src_k, const T* __restrict__ src_v, int64_t src_ts,
                                              int tok0, uint32_t (&kr)[4][4], uint32_t (&vr)[4][4]) {
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int w = wq >> 2, j = wq & 3, m = lane & 15, e = lane >> 4;
  const int dbase = 32 * (m >> 2) + 2 * (m & 3);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t off = (int64_t)(tok0 + 32 * w + 8 * i + 2 * j + e) * src_ts + dbase;
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) {
      kr[i][sl] = __ldg(reinterpret_cast<const uint32_t*>(src_k + off + 8 * sl));
      vr[i][sl] = __ldg(reinterpret_cast<const uint32_t*>(src_v + off + 8 * sl));
    }
  }
}

template <typename T>
__device__ void append_full_kv4(const PoolView& pv, int s, int p, const uint32_t (&kr)[4][4],
                                const uint32_t (&vr)[4][4], uint8_t* smem) {
  constexpr int D = 128;
  using H2 = typename std::conditional<std::is_same<T, __half>::value, __half2, __nv_bfloat162>::type;
  auto hmin = [](uint32_t a, uint32_t b) {
    H2 r = __hmin2(*reinterpret_cast<H2*>(&a), *reinterpret_cast<H2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  };
  auto hmax = [](uint32_t a, uint32_t b) {
    H2 r = __hmax2(*reinterpret_cast<H2*>(&a), *reinterpret_cast<H2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  };
  const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
  const int w = wq >> 2, j = wq & 3, m = lane & 15, e = lane >> 4;
  const int dbase = 32 * (m >> 2) + 2 * (m & 3);
  const bool streaming = pv.kind[s] == SK_KIND_STREAMING;
  const int levels = (1 << pv.bits) - 1;
  uint4* red_k = reinterpret_cast<uint4*>(smem);         // [w 2][j 4][h 2][mm 2][m 16]
  uint4* red_v = red_k + 2 * 4 * 2 * 2 * 16;             // [wq 8][mm 2][m 16]
  uint4* kb = red_v + 8 * 2 * 16;                        // [mm 2][m 16] K page bounds
  uint4* vb = kb + 2 * 16;                               // [mm 2][m 16] V page bounds
  float* lo32 = reinterpret_cast<float*>(vb + 2 * 16);  // [which 2][q 128], q = 8m + 2sl + x
  float* inv32 = lo32 + 256;
  double* lo64 = reinterpret_cast<double*>(inv32 + 256);
  double* sc64 = lo64 + 256;
  double* inv64 = sc64 + 256;

  uint8_t* slot = pv.slot_ptr(s, p);  // issued early: read after two barriers
  // 2. per-thread min / max: K per logical page h (tokens i = 2h, 2h+1), V over
  //    all four tokens; then across e (lane ^ 16)
  uint32_t kmn[2][4], kmx[2][4], vmn[4], vmx[4];
#pragma unroll
  for (int sl = 0; sl < 4; ++sl) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      kmn[h][sl] = hmin(kr[2 * h][sl], kr[2 * h + 1][sl]);
      kmx[h][sl] = hmax(kr[2 * h][sl], kr[2 * h + 1][sl]);
      kmn[h][sl] = hmin(kmn[h][sl], __shfl_xor_sync(0xffffffffu, kmn[h][sl], 16));
      kmx[h][sl] = hmax(kmx[h][sl], __shfl_xor_sync(0xffffffffu, kmx[h][sl], 16));
    }
    vmn[sl] = hmin(hmin(vr[0][sl], vr[1][sl]), hmin(vr[2][sl], vr[3][sl]));
    vmx[sl] = hmax(hmax(vr[0][sl], vr[1][sl]), hmax(vr[2][sl], vr[3][sl]));
    vmn[sl] = hmin(vmn[sl], __shfl_xor_sync(0xffffffffu, vmn[sl], 16));
    vmx[sl] = hmax(vmx[sl], __shfl_xor_sync(0xffffffffu, vmx[sl], 16));
  }
  // lane e = 0 publishes the minima, e = 1 the maxima
#pragma unroll
  for (int h = 0; h < 2; ++h)
    red_k[(((w * 4 + j) * 2 + h) * 2 + e) * 16 + m] =
        e ? make_uint4(kmx[h][0], kmx[h][1], kmx[h][2], kmx[h][3]) : make_uint4(kmn[h][0], kmn[h][1], kmn[h][2], kmn[h][3]);
  red_v[(wq * 2 + e) * 16 + m] = e ? make_uint4(vmx[0], vmx[1], vmx[2], vmx[3]) : make_uint4(vmn[0], vmn[1], vmn[2], vmn[3]);
  __syncthreads();
  // 3. threads 0..127: logical page lp = tid % 4 of (mm, m) = tid / 4 -> key
  //    stats, then the K bounds across the four lanes; threads 128..159: V bounds
  if (tid < 128) {
    const int lp = tid & 3, mm = (tid >> 2) >> 4, mq = (tid >> 2) & 15, ww = lp >> 1, h = lp & 1;
    uint4 a = red_k[(((ww * 4 + 0) * 2 + h) * 2 + mm) * 16 + mq];
#pragma unroll
    for (int jj = 1; jj < 4; ++jj) {
      const uint4 b = red_k[(((ww * 4 + jj) * 2 + h) * 2 + mm) * 16 + mq];
      a = mm ? make_uint4(hmax(a.x, b.x), hmax(a.y, b.y), hmax(a.z, b.z), hmax(a.w, b.w))
             : make_uint4(hmin(a.x, b.x), hmin(a.y, b.y), hmin(a.z, b.z), hmin(a.w, b.w));
    }
    if (!streaming && pv.stats != nullptr) {
      T* st = reinterpret_cast<T*>(pv.stats_ptr(s, p * 4 + lp)) + mm * D + 32 * (mq >> 2) + 2 * (mq & 3);
      *reinterpret_cast<uint32_t*>(st) = a.x;
      *reinterpret_cast<uint32_t*>(st + 8) = a.y;
      *reinterpret_cast<uint32_t*>(st + 16) = a.z;
      *reinterpret_cast<uint32_t*>(st + 24) = a.w;
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      const uint4 b = make_uint4(__shfl_xor_sync(0xffffffffu, a.x, off), __shfl_xor_sync(0xffffffffu, a.y, off),
                                 __shfl_xor_sync(0xffffffffu, a.z, off), __shfl_xor_sync(0xffffffffu, a.w, off));
      a = mm ? make_uint4(hmax(a.x, b.x), hmax(a.y, b.y), hmax(a.z, b.z), hmax(a.w, b.w))
             : make_uint4(hmin(a.x, b.x), hmin(a.y, b.y), hmin(a.z, b.z), hmin(a.w, b.w));
    }
    if (lp == 0) kb[mm * 16 + mq] = a;
  } else if (tid < 160) {
    const int mm = (tid - 128) >> 4, mq = tid & 15;
    uint4 a = red_v[mm * 16 + mq];
#pragma unroll
    for (int q = 1; q < 8; ++q) {
      const uint4 b = red_v[(q * 2 + mm) * 16 + mq];
      a = mm ? make_uint4(hmax(a.x, b.x), hmax(a.y, b.y), hmax(a.z, b.z), hmax(a.w, b.w))
             : make_uint4(hmin(a.x, b.x), hmin(a.y, b.y), hmin(a.z, b.z), hmin(a.w, b.w));
    }
    vb[mm * 16 + mq] = a;
  }
  __syncthreads();
  // 4. one thread per (which, q): bounds -> the page slot, quantiser tables
  {
    const int which = tid >> 7, q = tid & 127, mq = q >> 3, sl = (q & 7) >> 1, x = q & 1;
    const uint4* b = which ? vb : kb;
    const T* lo_h = reinterpret_cast<const T*>(&b[mq]);
    const T* hi_h = reinterpret_cast<const T*>(&b[16 + mq]);
    const T lo_t = lo_h[q & 7], hi_t = hi_h[q & 7];
    const int c = 32 * (mq >> 2) + 2 * (mq & 3) + 8 * sl + x;
    T* bnd = reinterpret_cast<T*>(pv.bounds(slot));
    const int pos = which ? vbound_pos(c, D) : kbound_pos(c, D);
    bnd[(2 * which) * D + pos] = lo_t;
    bnd[(2 * which + 1) * D + pos] = hi_t;
    const float lo = DT<T>::to_f(lo_t), hi = DT<T>::to_f(hi_t);
    double sc = ((double)hi - (double)lo) / levels;
    if (!(sc > 0.0)) sc = 1.0;
    lo32[tid] = lo;
    inv32[tid] = (float)(1.0 / sc);
    lo64[tid] = lo;
    sc64[tid] = sc;
    inv64[tid] = 1.0 / sc;
  }
  __syncthreads();
  // 5. codes (near-ties through the exact fp64 path, about 1 value in 2^15)
  uint32_t* kw = reinterpret_cast<uint32_t*>(pv.k_codes(slot));
  uint32_t* vw = reinterpret_cast<uint32_t*>(pv.v_codes(slot));
  uint32_t kword[4], pw[4][2];
  {
    uint64_t nl[4], iv[4];
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) {
      nl[sl] = f2p(-lo32[8 * m + 2 * sl], -lo32[8 * m + 2 * sl + 1]);
      iv[sl] = f2p(inv32[8 * m + 2 * sl], inv32[8 * m + 2 * sl + 1]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t word = 0;
#pragma unroll
      for (int sl = 0; sl < 4; ++sl)
        word |= qpair<T>(kr[i][sl], nl[sl], iv[sl], lo64, sc64, inv64, 8 * m + 2 * sl, levels) << (4 * sl);
      kword[i] = word;
    }
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) {
      nl[sl] = f2p(-lo32[128 + 8 * m + 2 * sl], -lo32[128 + 8 * m + 2 * sl + 1]);
      iv[sl] = f2p(inv32[128 + 8 * m + 2 * sl], inv32[128 + 8 * m + 2 * sl + 1]);
    }
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) {
      uint32_t a = 0;  // channel x = 0 in the low half, x = 1 in the high half, token i at 4i
#pragma unroll
      for (int i = 0; i < 4; ++i)
        a |= qpair<T>(vr[i][sl], nl[sl], iv[sl], lo64, sc64, inv64, 128 + 8 * m + 2 * sl, levels) << (4 * i);
      // this thread's token parity e: nibbles at 4i + 16e of each channel's word
      pw[sl][0] = (a & 0xFFFFu) << (16 * e);
      pw[sl][1] = (a >> 16) << (16 * e);
    }
  }
  // K word (t_i, j = m%4, w = m/4); V words: the lane^16 partner holds the other
  // token parity e, lane e stores channel dbase + 8 sl + e
#pragma unroll
  for (int i = 0; i < 4; ++i) kw[(32 * w + 8 * i + 2 * j + e) * 16 + (m & 3) * 4 + (m >> 2)] = kword[i];
#pragma unroll
  for (int sl = 0; sl < 4; ++sl) {
    const uint32_t a = pw[sl][0] | __shfl_xor_sync(0xffffffffu, pw[sl][0], 16);
    const uint32_t b = pw[sl][1] | __shfl_xor_sync(0xffffffffu, pw[sl][1], 16);
    const int c = dbase + 8 * sl + e;
    vw[((c >> 3) * 32 + 4 * (c & 7) + j) * 2 + w] = e ? b : a;
  }
}

template <typename T>
__global__ void __launch_bounds__(256, SK_APPEND_MINB) append_kernel(PoolView pv, const T* __restrict__ k_src,
                                                        const T* __restrict__ v_src, int64_t src_ss, int64_t src_ts,
                                                        const int32_t* __restrict__ tokens, int m, int sfirst) {
  extern __shared__ __align__(16) uint8_t smem[];
  // sfirst: streams fastest, so the CTAs that run together read the same token
  // rows of the [token][stream][D] source -- whole DRAM rows at a time
  const int s = sfirst ? blockIdx.x : blockIdx.y;
  const int pi = sfirst ? blockIdx.y : blockIdx.x;  // page of this launch
  const T* sk_ = k_src + s * src_ss;
  const T* sv_ = v_src + s * src_ss;
  const bool fast = SK_APPEND_FAST && pv.bits >= 1 && pv.bits <= 4 && pv.D == 128 && pv.P == 64 && pv.L == 16;
  if (fast && (pi + 1) * 64 <= m) {
    // a bulk append usually starts on a page boundary: load the page's raw
    // tokens assuming n0 % 64 == 0 while the token count is still in flight
    uint32_t kr[4][4], vr[4][4];
    load_full_kv4<T>(sk_, sv_, src_ts, pi * 64, kr, vr);
    const int n0 = tokens[s];
    if (n0 % 64 == 0) {
      const int n1 = n0 + m, p = n0 / 64 + pi;
      const int count = (n1 + 63) / 64;
      const bool evicted = pv.kind[s] == SK_KIND_STREAMING && p >= pv.sink && p < count - pv.local;
      // a partial last page's tail is written to staging by the open page's CTA
      if (pi == 0 && (n1 - 1) / 64 != p && (n1 % 64) != 0) write_tail_from_src<T>(pv, s, n0, n1, sk_, sv_, src_ts);
      if (!evicted) append_full_kv4<T>(pv, s, p, kr, vr, smem);
      return;
    }
  }
  const int n0 = tokens[s];
  const int n1 = n0 + m;
  const int p = n0 / pv.P + pi;
  if (p > (n1 - 1) / pv.P) return;
  const int t0 = p * pv.P;
  if (fast && t0 >= n0 && t0 + 64 <= n1) {  // a full page of new tokens after an unaligned start
    const int count = (n1 + 63) / 64;
    const bool evicted = pv.kind[s] == SK_KIND_STREAMING && p >= pv.sink && p < count - pv.local;
    const int p_open = n0 / 64, p_last = (n1 - 1) / 64;
    if (p == p_open && p_last != p_open && (n1 % 64) != 0) write_tail_from_src<T>(pv, s, n0, n1, sk_, sv_, src_ts);
    if (!evicted) {
      uint32_t kr[4][4], vr[4][4];
      load_full_kv4<T>(sk_, sv_, src_ts, t0 - n0, kr, vr);
      append_full_kv4<T>(pv, s, p, kr, vr, smem);
    }
    return;
  }
  append_page<T>(pv, s, p, n0, n1, sk_, sv_, src_ts, smem);
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
#ifdef SK_APPEND_ONE_NOOP  // timing builds only (tools/ab_variant.sh): the decode step without its appends
  return;
#endif
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
  const int sfirst = SK_APPEND_SFIRST && max_pages_touched <= 65535;
  dim3 grid = sfirst ? dim3(n_streams, max_pages_touched) : dim3(max_pages_touched, n_streams);
  if (pv.dtype == SK_F16) {
    cudaFuncSetAttribute(append_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    append_kernel<__half><<<grid, 256, smem, st>>>(pv, (const __half*)k_src, (const __half*)v_src, ss, ts,
                                                   tokens, m, sfirst);
  } else {
    cudaFuncSetAttribute(append_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    append_kernel<__nv_bfloat16><<<grid, 256, smem, st>>>(pv, (const __nv_bfloat16*)k_src,
                                                          (const __nv_bfloat16*)v_src, ss, ts, tokens, m, sfirst);
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
