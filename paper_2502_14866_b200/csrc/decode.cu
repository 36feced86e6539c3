// K3 -- split-KV decode attention over the selected pages (+ fused append).
//
// Replaces the per-head page loop of Engine.decode_step (reference
// engine.py:257-285), PhysicalPage.dequantize (cache.py:97-102) and
// merge_block (attn.py:191-229).
//
// One CTA = one (stream, split); 4 warps each walk whole pages of the
// stream's page union (the selection for retrieval rows + the sink/local
// window for streaming rows, each page carrying the mask of group rows that
// attend it).  Per page a warp runs m16n8k16 tensor-core MMAs directly on
// the stored codes, using the dequantisation algebra
//     q . khat_t = sum_d (q_d s_d) c_td + sum_d q_d lo_d
//     sum_t p_t vhat_tc = s_c sum_t p_t c_tc + lo_c sum_t p_t
// so codes are unpacked to exact fp16 integers with one LOP3 + one HSUB2 per
// two codes (fragment-native layout written by K1, sk_layout.cuh) and never
// materialised as floats.  Group rows sit in the MMA's M dimension (GQA
// rows share every page load).  Online softmax in fp32 (exp2 domain); warps
// merge in shared memory, splits merge in the last CTA of the stream
// (atomic ticket) together with the new token's raw K/V, then -- if asked --
// that CTA appends the new token to its page (K1's page rebuild).
#include "append_impl.cuh"

namespace sk {
int append_launch(const sk_pool* pool, int n_streams, const void* k_src, const void* v_src, int64_t ss, int64_t ts,
                  int32_t* tokens, int m, int max_pages_touched, cudaStream_t st);
}  // namespace sk
#include "sk_sm100.cuh"

namespace sk {
namespace {

constexpr int kDecThreads = 256;

// Debug timeline: %globaltimer stamps at phase boundaries for the first
// CTA(s) of stream 0 (build with -DSK_DECODE_TIMING; read via sk_debug_times).
#ifdef SK_DECODE_TIMING
__device__ unsigned long long g_dec_times[64][32];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SK_STAMP(i)                                                                        \
  do {                                                                                     \
    if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < 64) g_dec_times[blockIdx.x][(i) + 1] = gtimer(); \
  } while (0)
#else
#define SK_STAMP(i) \
  do {              \
  } while (0)
#endif
#ifdef SK_DECODE_TIMING
#define SK_WSTAMP(i)                                                                                   \
  do {                                                                                                 \
    if ((threadIdx.x & 31) == 0 && blockIdx.y == 0 && blockIdx.x < 64)                               \
      g_dec_times[blockIdx.x][(i) + (threadIdx.x >> 5)] = gtimer();                                    \
  } while (0)
#else
#define SK_WSTAMP(i) \
  do {               \
  } while (0)
#endif
constexpr int kWarps = kDecThreads / 32;
constexpr int kMaxRows = 8;
constexpr int kMaxExtra = 64;
constexpr int kMaxSel = 2048;  // selection entries staged in smem
constexpr int kMaxPps = 16;    // pages per split (CTA)

struct DecodeParams {
  PoolView pv;
  int G;
  const void* q;
  int64_t q_ss, q_rs;
  const void* k_new;
  const void* v_new;
  int64_t new_ss;
  const uint32_t* row_mask;
  const int32_t* sel;
  const int32_t* sel_count;
  int sel_stride;
  int32_t* tokens;
  float scale_log2;
  void* out;
  int64_t out_ss, out_rs;
  int out_dtype;
  int pps;
  int fuse_append;
  float* ws_part;
  uint32_t* ws_ticket;
  int max_splits;
};

// m16n8k16 MMA, fp32 accumulate.  MT = __half or __nv_bfloat16 operands.
template <typename MT>
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  if constexpr (std::is_same<MT, __half>::value) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
}

template <typename MT>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  if constexpr (std::is_same<MT, __half>::value) {
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}
template <typename MT>
__device__ __forceinline__ float2 unpack2(uint32_t w) {
  if constexpr (std::is_same<MT, __half>::value) return __half22float2(*reinterpret_cast<__half2*>(&w));
  else return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w));
}

// nibble word -> fp16x2 register `slot` (exact integers 0..15)
__device__ __forceinline__ uint32_t nib2h(uint32_t w, int slot) {
  uint32_t x = ((w >> (4 * slot)) & 0x000F000Fu) | 0x64006400u;
  __half2 h = __hsub2(*reinterpret_cast<__half2*>(&x), __halves2half2(__ushort_as_half(0x6400), __ushort_as_half(0x6400)));
  return *reinterpret_cast<uint32_t*>(&h);
}
// byte pair (r2 = 0: bytes 0,1; r2 = 1: bytes 2,3) -> fp16x2 exact integers 0..255
__device__ __forceinline__ uint32_t byte2h(uint32_t w, int r2) {
  uint32_t x = __byte_perm(w, 0x64u, r2 ? 0x4342 : 0x4140);  // {b, 0x64, b', 0x64}
  __half2 h = __hsub2(*reinterpret_cast<__half2*>(&x), __halves2half2(__ushort_as_half(0x6400), __ushort_as_half(0x6400)));
  return *reinterpret_cast<uint32_t*>(&h);
}

// Binary search in an ascending int list.
__device__ __forceinline__ bool contains(const int32_t* a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    int v = a[mid];
    if (v == x) return true;
    if (v < x) lo = mid + 1; else hi = mid;
  }
  return false;
}

// KIND: 0 raw pages (MMA in T), 1 nibble codes, 2 byte codes (MMA in fp16).
//
// Work decomposition.  A CTA (8 warps) owns `pps` consecutive units (pages)
// of one stream's union.  All of them are staged into shared memory with
// one CTA-wide cp.async sweep, then each page is cut into P/16 token tiles
// of 16 tokens and the (page, tile) items are dealt to the warps: a warp
// runs QK for its 16 tokens (2 n-tiles x D/16 k-steps) and one PV k-step
// over all D/8 channel tiles, keeping its own online-softmax state.  Short
// per-warp chains + many resident warps hide the MMA / shuffle latencies
// (one warp per page serialised ~3.5k dependent instructions).
template <typename T, int KIND, int D, int P>
#ifndef SK_DEC_MINB
#define SK_DEC_MINB 2
#endif
__global__ void __launch_bounds__(kDecThreads, SK_DEC_MINB) decode_kernel(DecodeParams prm) {
  using MT = typename std::conditional<KIND == 0, T, __half>::type;
  constexpr int NKS = D / 16;   // QK k-steps
  constexpr int NCN = D / 8;    // PV n-tiles (8 channels)
  constexpr int NTT = P / 16;   // 16-token tiles per page
  constexpr int QR = D / 4;     // q / o / bounds values per thread
  constexpr int RB = KIND == 0 ? 2 * D : (KIND == 1 ? D / 2 : D);  // code row bytes
  constexpr int SLOT_USED = 2 * P * RB + (KIND == 0 ? 0 : 8 * D);  // bytes of a slot the kernel reads
  extern __shared__ __align__(16) uint8_t smem[];
#ifdef SK_DECODE_TIMING
  if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < 64) g_dec_times[blockIdx.x][0] = gtimer();
#endif
  __shared__ int s_sel[kMaxSel];
  __shared__ int s_extra[kMaxExtra];
  __shared__ int s_page[kMaxPps];
  __shared__ uint32_t s_um[kMaxPps];
  __shared__ int s_nextra, s_nunits;
  __shared__ uint32_t s_last;

  const PoolView& pv = prm.pv;
  const int s = blockIdx.y, split = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 2, j = lane & 3;
  const int G = prm.G;
  const int pps = prm.pps;
  const int u_begin = split * pps;
  const int32_t* sel = prm.sel + (int64_t)s * prm.sel_stride;
  // ---- one parallel round of header loads (no dependent global chains) ----
  const int n_tok = prm.tokens[s];
  const uint32_t rm_raw = prm.row_mask[s];
  const int cnt_raw = prm.sel_count[s];
  const int sel_w = min(prm.sel_stride, kMaxSel);
  if (n_tok < 0) s_sel[0] = 0;  // keep n_tok live for the stamp below
  SK_STAMP(6);
  for (int i = tid; i < sel_w; i += kDecThreads) s_sel[i] = sel[i];
  SK_STAMP(7);
  const bool row_ok = r < G;
  uint32_t qw[QR / 2];  // the thread's q values, packed pairs in the input dtype (exact)
  {
    const T* qrow = reinterpret_cast<const T*>(prm.q) + s * prm.q_ss + (int64_t)(row_ok ? r : 0) * prm.q_rs;
#pragma unroll
    for (int ri = 0; ri < D / 8; ++ri) {
      int d = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j;
      qw[ri] = *reinterpret_cast<const uint32_t*>(qrow + d);
    }
  }
  const int n_pages = (n_tok + P - 1) / P;
  const uint32_t gmask = (G >= 32) ? 0xffffffffu : ((1u << G) - 1u);
  const uint32_t rmask = rm_raw & gmask;
  const uint32_t smask = gmask & ~rmask;
  const int nsel = rmask ? cnt_raw : 0;
  const int sink_end = min(pv.sink, n_pages), local_start = max(n_pages - pv.local, 0);
  __syncthreads();
  SK_STAMP(8);
  // ---- the stream's page union from smem: selection + sink/local extras ----
  // warp 0: each lane tests one sink/local candidate against the staged
  // selection (binary search in smem), ballots keep the ascending order.
  if (warp == 0) {
    int ne = 0;
    if (smask) {
      const int loc0 = max(local_start, sink_end);
      const int ncand = sink_end + (n_pages - loc0);
      for (int base = 0; base < ncand; base += 32) {
        const int ci = base + lane;
        const int p = ci < sink_end ? ci : loc0 + (ci - sink_end);
        const bool extra = ci < ncand && !contains(s_sel, nsel, p);
        const uint32_t bal = __ballot_sync(0xffffffffu, extra);
        const int pos = ne + __popc(bal & ((1u << lane) - 1u));
        if (extra && pos < kMaxExtra) s_extra[pos] = p;
        ne += __popc(bal);
      }
      ne = min(ne, kMaxExtra);
    }
    __syncwarp();
    const int U0 = nsel + ne;
    const int nu = max(0, min(U0, u_begin + pps) - u_begin);
    if (lane < nu) {
      const int u = u_begin + lane;
      int pg;
      uint32_t um;
      if (u < nsel) {
        pg = s_sel[u];
        um = rmask | ((smask && (pg < sink_end || pg >= local_start)) ? smask : 0u);
      } else {
        pg = s_extra[u - nsel];
        um = smask;
      }
      s_page[lane] = pg;
      s_um[lane] = um;
    }
    if (lane == 0) {
      s_nextra = ne;
      s_nunits = nu;
    }
  }
  __syncthreads();
  SK_STAMP(0);
  const int U = nsel + s_nextra;
  const int n_used = (U + pps - 1) / pps;
  const int n_units = s_nunits;

  // ---- stage the CTA's pages in smem (one cp.async sweep) -------------------
  for (int i = 0; i < n_units; ++i) {
    const uint8_t* src = pv.slot_ptr(s, s_page[i]);
    uint8_t* dst = smem + i * SLOT_USED;
    for (int c = tid; c < SLOT_USED / 16; c += kDecThreads) cp_async16(dst + 16 * c, src + 16 * c);
  }
  cp_async_commit();

  // ---- per-thread row state: row r (lane/4), dims/channels of j (lane%4) ----
  if (!row_ok) {
#pragma unroll
    for (int ri = 0; ri < D / 8; ++ri) qw[ri] = 0u;
  }
  float o[QR];
#pragma unroll
  for (int i = 0; i < QR; ++i) o[i] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;
  const float sl2 = prm.scale_log2;
  const float inv_levels = KIND == 0 ? 1.f : 1.f / float((1 << pv.bits) - 1);
  cp_async_wait<0>();
  __syncthreads();
  SK_STAMP(1);
  // ---- per-page dequantisation tables, once per page (warp w -> page w) ----
  // tab[0:D)  = s_k / smax  (K bounds order)   tab[D:2D)  = lo_k
  // tab[2D:3D) = s_v         (V bounds order)   tab[3D:4D) = lo_v   tab[4D] = smax
  constexpr int TAB = 4 * D + 4;
  float* tabs = reinterpret_cast<float*>(smem + ((prm.pps * SLOT_USED + 15) & ~15));
  if constexpr (KIND != 0) {
    for (int i = warp; i < n_units; i += kWarps) {
      const T* bnd = reinterpret_cast<const T*>(smem + i * SLOT_USED + 2 * P * RB);
      float* tab = tabs + i * TAB;
      float mx = 0.f;
      float skv[D / 32];
#pragma unroll
      for (int q = 0; q < D / 32; ++q) {
        const int x = lane + 32 * q;
        const float lo = DT<T>::to_f(bnd[x]), hi = DT<T>::to_f(bnd[D + x]);
        const float sv = (hi - lo) * inv_levels;
        skv[q] = sv > 0.f ? sv : 1.f;
        mx = fmaxf(mx, skv[q]);
        tab[D + x] = lo;
        const float vlo = DT<T>::to_f(bnd[2 * D + x]), vhi = DT<T>::to_f(bnd[3 * D + x]);
        const float vs = (vhi - vlo) * inv_levels;
        tab[2 * D + x] = vs > 0.f ? vs : 1.f;
        tab[3 * D + x] = vlo;
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float inv = 1.f / mx;
#pragma unroll
      for (int q = 0; q < D / 32; ++q) tab[lane + 32 * q] = skv[q] * inv;
      if (lane == 0) tab[4 * D] = mx;
    }
    __syncthreads();
  }
  SK_STAMP(9);

  for (int item = warp; item < n_units * NTT; item += kWarps) {
    const int ui = item / NTT, tt = item % NTT;
    const int p = s_page[ui];
    const uint32_t um = s_um[ui];
    const bool attend = row_ok && ((um >> r) & 1u);
    const uint8_t* pg = smem + ui * SLOT_USED;
    const int tok_in_page = min(P, n_tok - p * P);
    if (16 * tt >= tok_in_page) continue;  // tile past the open page's tokens
#if defined(SK_DBG) && SK_DBG == 4
    continue;
#endif
    const uint8_t* kc = pg;
    const uint8_t* vc = pg + P * RB;
    const T* bnd = reinterpret_cast<const T*>(pg + 2 * P * RB);

    // ---- K side: q' = q * s_k / smax (A fragments), qz = q . lo_k ----
    uint32_t afr[NKS][2];
    float smax = 1.f, qz = 0.f;
    const float* tab = tabs + ui * TAB;
    if constexpr (KIND == 0) {
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        afr[ks][0] = qw[2 * ks];  // raw pages: q is the A operand as is
        afr[ks][1] = qw[2 * ks + 1];
      }
    } else {
      const float4* kn4 = reinterpret_cast<const float4*>(tab + j * QR);
      const float4* kl4 = reinterpret_cast<const float4*>(tab + D + j * QR);
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        const float4 f = kn4[ks], l = kl4[ks];
        const float2 q0 = DT<T>::to_f2(qw[2 * ks]), q1 = DT<T>::to_f2(qw[2 * ks + 1]);
        afr[ks][0] = pack2<MT>(q0.x * f.x, q0.y * f.y);
        afr[ks][1] = pack2<MT>(q1.x * f.z, q1.y * f.w);
        qz = fmaf(q0.x, l.x, fmaf(q0.y, l.y, fmaf(q1.x, l.z, fmaf(q1.y, l.w, qz))));
      }
      qz += __shfl_xor_sync(0xffffffffu, qz, 1);
      qz += __shfl_xor_sync(0xffffffffu, qz, 2);
      smax = tab[4 * D];
    }

    // ---- S = q' K^T for the tile's two n-tiles of 8 tokens ----
    float sc[2][2];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int nt = 2 * tt + h2;
      const int tok = 8 * nt + r;  // B operand: n = lane/4
      float c[4] = {0.f, 0.f, 0.f, 0.f};
      if constexpr (KIND == 1) {
        uint32_t wd[D / 32];
        const uint8_t* src = kc + tok * (D / 2) + j * (D / 8);
        if constexpr (D == 128) {
          uint4 v = *reinterpret_cast<const uint4*>(src);
          wd[0] = v.x; wd[1] = v.y; wd[2] = v.z; wd[3] = v.w;
        } else {
          uint2 v = *reinterpret_cast<const uint2*>(src);
          wd[0] = v.x; wd[1] = v.y;
        }
#pragma unroll
        for (int ks = 0; ks < NKS; ++ks) {
          int ri0 = 2 * ks, ri1 = 2 * ks + 1;
          uint32_t b0 = nib2h(wd[ri0 / 4], ri0 % 4), b1 = nib2h(wd[ri1 / 4], ri1 % 4);
#if defined(SK_DBG) && SK_DBG == 1
          c[0] += __uint_as_float(b0 ^ afr[ks][0]); c[1] += __uint_as_float(b1 ^ afr[ks][1]);
#else
          mma16816<MT>(c, afr[ks][0], 0u, afr[ks][1], 0u, b0, b1);
#endif
        }
      } else if constexpr (KIND == 2) {
        uint32_t wd[D / 16];
        const uint4* src = reinterpret_cast<const uint4*>(kc + tok * D + j * (D / 4));
#pragma unroll
        for (int i = 0; i < D / 64; ++i) {
          uint4 v = src[i];
          wd[4 * i] = v.x; wd[4 * i + 1] = v.y; wd[4 * i + 2] = v.z; wd[4 * i + 3] = v.w;
        }
#pragma unroll
        for (int ks = 0; ks < NKS; ++ks) {
          uint32_t b0 = byte2h(wd[ks], 0), b1 = byte2h(wd[ks], 1);
          mma16816<MT>(c, afr[ks][0], 0u, afr[ks][1], 0u, b0, b1);
        }
      } else {
        uint32_t wd[D / 8];
        const uint4* src = reinterpret_cast<const uint4*>(kc + tok * D * 2 + j * (D / 2));
#pragma unroll
        for (int i = 0; i < D / 32; ++i) {
          uint4 v = src[i];
          wd[4 * i] = v.x; wd[4 * i + 1] = v.y; wd[4 * i + 2] = v.z; wd[4 * i + 3] = v.w;
        }
#pragma unroll
        for (int ks = 0; ks < NKS; ++ks) mma16816<MT>(c, afr[ks][0], 0u, afr[ks][1], 0u, wd[2 * ks], wd[2 * ks + 1]);
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int t = 8 * nt + 2 * j + e;
        float v = (c[e] * smax + qz) * sl2;
        sc[h2][e] = t < tok_in_page ? v : -INFINITY;
      }
    }

    // ---- online softmax for row r over the 16 tokens (4 lanes j share a row) ----
    float tmax = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    const float m_new = attend ? fmaxf(m_run, tmax) : m_run;
    const float alpha = attend ? exp2f(m_run - m_new) : 1.f;  // exp2(-inf) = 0
    uint32_t pfr[2];
    float psum = 0.f;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
#if defined(SK_DBG) && SK_DBG == 3
      float p0 = attend ? (sc[h2][0] - m_new) : 0.f;
      float p1 = attend ? (sc[h2][1] - m_new) : 0.f;
#else
      float p0 = attend ? exp2f(sc[h2][0] - m_new) : 0.f;
      float p1 = attend ? exp2f(sc[h2][1] - m_new) : 0.f;
#endif
      uint32_t pk = pack2<MT>(p0, p1);
      float2 pr = unpack2<MT>(pk);  // the rounded values the MMA sees
      psum += pr.x + pr.y;
      pfr[h2] = pk;
    }
    l_run = l_run * alpha + psum;  // per-thread partial (tokens of lane j)
    m_run = m_new;
    float prow = psum;
    prow += __shfl_xor_sync(0xffffffffu, prow, 1);
    prow += __shfl_xor_sync(0xffffffffu, prow, 2);

    // ---- O += P V over the tile's 16 tokens: one k-step per channel n-tile ----
    const int ri0 = 2 * tt, ri1 = 2 * tt + 1;
#pragma unroll
    for (int cn = 0; cn < NCN; ++cn) {
      float c[4] = {0.f, 0.f, 0.f, 0.f};
      const int vl = 32 * cn + lane;  // (cn, lane) chunk
      uint32_t b0, b1;
      if constexpr (KIND == 1) {
        const uint32_t w = reinterpret_cast<const uint32_t*>(vc + vl * (P / 8))[ri0 / 4];
        b0 = nib2h(w, ri0 % 4);
        b1 = nib2h(w, ri1 % 4);
      } else if constexpr (KIND == 2) {
        const uint32_t w = reinterpret_cast<const uint32_t*>(vc + vl * (P / 4))[tt];
        b0 = byte2h(w, 0);
        b1 = byte2h(w, 1);
      } else {
        const uint2 w = reinterpret_cast<const uint2*>(vc + vl * (P / 2))[tt];
        b0 = w.x;
        b1 = w.y;
      }
#if defined(SK_DBG) && SK_DBG == 2
      c[0] = __uint_as_float(b0 ^ pfr[0]); c[1] = __uint_as_float(b1 ^ pfr[1]);
#else
      mma16816<MT>(c, pfr[0], 0u, pfr[1], 0u, b0, b1);
#endif
      float add0 = c[0], add1 = c[1];
      if constexpr (KIND != 0) {
        // channels 8cn+2j, +1 are adjacent in the V table (vbound order)
        const float2 sv = *reinterpret_cast<const float2*>(tab + 2 * D + j * QR + 2 * cn);
        const float2 lo = *reinterpret_cast<const float2*>(tab + 3 * D + j * QR + 2 * cn);
        add0 = fmaf(sv.x, c[0], lo.x * prow);
        add1 = fmaf(sv.y, c[1], lo.y * prow);
      }
      o[2 * cn] = fmaf(o[2 * cn], alpha, add0);
      o[2 * cn + 1] = fmaf(o[2 * cn + 1], alpha, add1);
    }
  }

  SK_WSTAMP(11);
  // ---- merge the 8 warps of this CTA (rows < kMaxRows) ----
  __syncthreads();  // page buffers are reused as the merge area
  SK_STAMP(2);
  float* sm_m = reinterpret_cast<float*>(smem);  // [kWarps][8]
  float* sm_l = sm_m + kWarps * kMaxRows;        // [kWarps][8]
  float* sm_o = sm_l + kWarps * kMaxRows;        // [kWarps][8][D]
  {
    float lt = l_run;
    lt += __shfl_xor_sync(0xffffffffu, lt, 1);
    lt += __shfl_xor_sync(0xffffffffu, lt, 2);
    if (j == 0) {
      sm_m[warp * kMaxRows + r] = m_run;
      sm_l[warp * kMaxRows + r] = lt;
    }
#pragma unroll
    for (int cn = 0; cn < NCN; ++cn)
#pragma unroll
      for (int e = 0; e < 2; ++e) sm_o[(warp * kMaxRows + r) * D + 8 * cn + 2 * j + e] = o[2 * cn + e];
  }
  __syncthreads();
  SK_STAMP(3);
  const int part_stride = 2 + D;
  float* part = prm.ws_part + ((int64_t)s * prm.max_splits + split) * kMaxRows * part_stride;
  // per-(warp, row) rescale factors once, then one FMA chain per output
  float* sm_f = sm_o + kWarps * kMaxRows * D;  // [kWarps][8]
  if (tid < G) {
    const int rr = tid;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sm_m[w * kMaxRows + rr]);
    float L = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float f = M == -INFINITY ? 0.f : exp2f(sm_m[w * kMaxRows + rr] - M);
      sm_f[w * kMaxRows + rr] = f;
      L += f * sm_l[w * kMaxRows + rr];
    }
    if (split < n_used) {
      part[rr * part_stride] = M;
      part[rr * part_stride + 1] = L;
    }
  }
  __syncthreads();
  if (split < n_used) {
    for (int i = tid; i < G * D; i += kDecThreads) {
      const int rr = i / D, c = i % D;
      float O = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) O = fmaf(sm_f[w * kMaxRows + rr], sm_o[(w * kMaxRows + rr) * D + c], O);
      part[rr * part_stride + 2 + c] = O;
    }
  }
  const T* kn = reinterpret_cast<const T*>(prm.k_new) + s * prm.new_ss;
  const T* vn = reinterpret_cast<const T*>(prm.v_new) + s * prm.new_ss;
  // ---- last CTA of the stream: merge splits + the new token, write ----
  __syncthreads();
  SK_STAMP(4);
  if (tid == 0) {
    __threadfence();
    uint32_t t = atomicAdd(prm.ws_ticket + s, 1u);
    s_last = (t == gridDim.x - 1);
    if (s_last) prm.ws_ticket[s] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  SK_STAMP(5);
  __threadfence();
  // Parallel merge of the n_used split partials (m, l, O[D]) + the new token:
  // stage the G rows of every split in smem with independent coalesced loads,
  // then one warp per row reduces (max, factors, denominator) and one thread
  // per (row, channel) sums the rescaled partial outputs.
  const int ps = part_stride;
  float* stg = reinterpret_cast<float*>(smem);  // [n_used][G * ps]
  float* row_l = stg + n_used * G * ps;         // [G]
  float* row_f = row_l + G;                     // [G] factor of the new token
  {
    const float* wsp = prm.ws_part + (int64_t)s * prm.max_splits * kMaxRows * ps;
    for (int sp = warp; sp < n_used; sp += kWarps)
      for (int idx = lane; idx < G * ps; idx += 32) stg[sp * G * ps + idx] = __ldcg(wsp + (int64_t)sp * kMaxRows * ps + idx);
  }
  __syncthreads();
  for (int rr = warp; rr < G; rr += kWarps) {
    const T* qrow = reinterpret_cast<const T*>(prm.q) + s * prm.q_ss + (int64_t)rr * prm.q_rs;
    float dot = 0.f;
    for (int c = lane; c < D; c += 32) dot = fmaf(DT<T>::to_f(qrow[c]), DT<T>::to_f(kn[c]), dot);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
    const float s_self = dot * sl2;
    float M = s_self;
    for (int sp = lane; sp < n_used; sp += 32) M = fmaxf(M, stg[(sp * G + rr) * ps]);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    float L = 0.f;
    for (int sp = lane; sp < n_used; sp += 32) {
      float* cell = stg + (sp * G + rr) * ps;
      const float pm = cell[0];
      const float f = pm == -INFINITY ? 0.f : exp2f(pm - M);
      L = fmaf(f, cell[1], L);
      cell[0] = f;  // the split's rescale factor for the output pass
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
    if (lane == 0) {
      const float fs = exp2f(s_self - M);
      row_l[rr] = L + fs;
      row_f[rr] = fs;
    }
  }
  __syncthreads();
  for (int i = tid; i < G * D; i += kDecThreads) {
    const int rr = i / D, c = i % D;
    float O = row_f[rr] * DT<T>::to_f(vn[c]);
    for (int sp = 0; sp < n_used; ++sp) {
      const float* cell = stg + (sp * G + rr) * ps;
      O = fmaf(cell[0], cell[2 + c], O);
    }
    O /= row_l[rr];
    const int64_t oi = s * prm.out_ss + (int64_t)rr * prm.out_rs + c;
    if (prm.out_dtype == SK_F32) reinterpret_cast<float*>(prm.out)[oi] = O;
    else if (prm.out_dtype == SK_F16) reinterpret_cast<__half*>(prm.out)[oi] = __float2half_rn(O);
    else reinterpret_cast<__nv_bfloat16*>(prm.out)[oi] = __float2bfloat16_rn(O);
  }
}

__host__ __device__ constexpr int slot_used(int kind, int D, int P) {
  return 2 * P * (kind == 0 ? 2 * D : (kind == 1 ? D / 2 : D)) + (kind == 0 ? 0 : 8 * D);
}

template <typename T, int KIND, int D, int P>
int launch_one(const DecodeParams& prm, dim3 grid, size_t smem_min, cudaStream_t st) {
  constexpr int SLOT = slot_used(KIND, D, P);
  size_t smem = (((size_t)prm.pps * SLOT + 15) & ~(size_t)15) + (size_t)prm.pps * (4 * D + 4) * 4;
  if (smem < smem_min) smem = smem_min;
  if (smem > 220 * 1024) {
    set_error("decode: pages_per_split too large for shared memory");
    return SK_EINVAL;
  }
  auto kern = decode_kernel<T, KIND, D, P>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, kDecThreads, smem, st>>>(prm);
  SK_CHECK_LAUNCH("decode_kernel");
  return SK_OK;
}

template <typename T, int KIND>
int launch_kind(const DecodeParams& prm, dim3 grid, size_t smem, cudaStream_t st) {
  const int D = prm.pv.D, P = prm.pv.P;
#define SK_DEC(DD, PP) if (D == DD && P == PP) return launch_one<T, KIND, DD, PP>(prm, grid, smem, st)
  SK_DEC(128, 64);
  SK_DEC(128, 32);
  SK_DEC(128, 128);
  SK_DEC(64, 64);
  SK_DEC(64, 32);
  SK_DEC(64, 128);
#undef SK_DEC
  set_error("decode: unsupported (head_dim, page_size); supported D in {64,128}, P in {32,64,128}");
  return SK_EUNSUPPORTED;
}

}  // namespace
}  // namespace sk

extern "C" int64_t sk_decode_workspace(int32_t n_streams, int32_t group_rows, int32_t head_dim, int32_t max_splits) {
  (void)group_rows;
  return (int64_t)n_streams * max_splits * sk::kMaxRows * (2 + head_dim) * 4 + (int64_t)n_streams * 4 + 256;
}

extern "C" int sk_decode_attn(const sk_pool* pool, int32_t n_streams, int32_t group_rows, const void* q,
                              int64_t q_stream_stride, int64_t q_row_stride, const void* k_new, const void* v_new,
                              int64_t new_stream_stride, const uint32_t* row_mask, const int32_t* sel,
                              const int32_t* sel_count, int32_t sel_stride, int32_t* tokens, float softmax_scale,
                              void* out, int64_t out_stream_stride, int64_t out_row_stride, int32_t out_dtype,
                              int32_t pages_per_split, int32_t max_splits, int32_t fuse_append, void* workspace,
                              int64_t workspace_bytes, void* stream) {
  using namespace sk;
  int rc = check_pool(pool);
  if (rc) return rc;
  SK_CHECK_ARG(n_streams >= 1, "decode: no streams");
  SK_CHECK_ARG(group_rows >= 1 && group_rows <= kMaxRows, "decode: group size must be in [1, 8]");
  SK_CHECK_ARG(pages_per_split >= 1 && pages_per_split <= kMaxPps && max_splits >= 1, "decode: bad split geometry");
  SK_CHECK_ARG(sel_stride <= kMaxSel, "decode: selection wider than 2048 pages");
  SK_CHECK_ARG(pool->sink + pool->local <= kMaxExtra, "decode: sink + local window too large");
  SK_CHECK_ARG(out_dtype == SK_F16 || out_dtype == SK_BF16 || out_dtype == SK_F32, "decode: bad out dtype");
  SK_CHECK_ARG(workspace_bytes >= sk_decode_workspace(n_streams, group_rows, pool->head_dim, max_splits),
               "decode: workspace too small");
  SK_CHECK_ARG(q && k_new && v_new && row_mask && sel && sel_count && tokens && out && workspace,
               "decode: NULL pointer");
  SK_CHECK_ARG(q_row_stride % 2 == 0 && q_stream_stride % 2 == 0, "decode: q strides must be even");
  DecodeParams prm;
  prm.pv = make_view(*pool);
  prm.G = group_rows;
  prm.q = q;
  prm.q_ss = q_stream_stride;
  prm.q_rs = q_row_stride;
  prm.k_new = k_new;
  prm.v_new = v_new;
  prm.new_ss = new_stream_stride;
  prm.row_mask = row_mask;
  prm.sel = sel;
  prm.sel_count = sel_count;
  prm.sel_stride = sel_stride;
  prm.tokens = tokens;
  prm.scale_log2 = softmax_scale * 1.4426950408889634f;
  prm.out = out;
  prm.out_ss = out_stream_stride;
  prm.out_rs = out_row_stride;
  prm.out_dtype = out_dtype;
  prm.pps = pages_per_split;
  prm.fuse_append = fuse_append;
  prm.max_splits = max_splits;
  prm.ws_part = static_cast<float*>(workspace);
  prm.ws_ticket = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(workspace) +
                                              (int64_t)n_streams * max_splits * kMaxRows * (2 + pool->head_dim) * 4);
  size_t smem_merge = (size_t)kWarps * kMaxRows * (3 + pool->head_dim) * 4;
  size_t smem_comb = ((size_t)max_splits * group_rows * (2 + pool->head_dim) + 2 * group_rows) * 4;
  size_t smem = smem_merge > smem_comb ? smem_merge : smem_comb;
  dim3 grid(max_splits, n_streams);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int kind = pool->bits == 0 ? 0 : (pool->bits <= 4 ? 1 : 2);
  int rc2;
  if (pool->dtype == SK_F16) {
    rc2 = kind == 0 ? launch_kind<__half, 0>(prm, grid, smem, st)
                    : (kind == 1 ? launch_kind<__half, 1>(prm, grid, smem, st) : launch_kind<__half, 2>(prm, grid, smem, st));
  } else {
    rc2 = kind == 0 ? launch_kind<__nv_bfloat16, 0>(prm, grid, smem, st)
                    : (kind == 1 ? launch_kind<__nv_bfloat16, 1>(prm, grid, smem, st)
                                 : launch_kind<__nv_bfloat16, 2>(prm, grid, smem, st));
  }
  if (rc2 != SK_OK || !fuse_append) return rc2;
  // the new token is appended by K1's one-token kernel right behind the
  // attention (stream order: every read of its page has completed)
  return append_launch(pool, n_streams, k_new, v_new, new_stream_stride, 0, tokens, 1, 1, st);
}

extern "C" int sk_debug_decode_times(unsigned long long* host_out) {
#ifdef SK_DECODE_TIMING
  return cudaMemcpyFromSymbol(host_out, sk::g_dec_times, sizeof(sk::g_dec_times)) == cudaSuccess ? 0 : -2;
#else
  (void)host_out;
  return -3;
#endif
}
