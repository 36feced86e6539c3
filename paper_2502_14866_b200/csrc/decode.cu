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
#include "sk_sm100.cuh"

namespace sk {
namespace {

constexpr int kDecThreads = 128;
constexpr int kWarps = kDecThreads / 32;
constexpr int kMaxRows = 8;
constexpr int kMaxExtra = 64;

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
// NBUF: pages staged per warp in shared memory by cp.async (0 = read the
// arena directly, 2 = double-buffered prefetch of the warp's next page).
template <typename T, int KIND, int D, int P, int NBUF>
__global__ void __launch_bounds__(kDecThreads) decode_kernel(DecodeParams prm) {
  using MT = typename std::conditional<KIND == 0, T, __half>::type;
  constexpr int NKS = D / 16;   // QK k-steps
  constexpr int NNT = P / 8;    // QK n-tiles (8 tokens)
  constexpr int NCN = D / 8;    // PV n-tiles (8 channels)
  constexpr int NPK = P / 16;   // PV k-steps (16 tokens)
  constexpr int QR = D / 4;     // q / o / bounds values per thread
  constexpr int RB = KIND == 0 ? 2 * D : (KIND == 1 ? D / 2 : D);  // code row bytes
  constexpr int SLOT_USED = 2 * P * RB + (KIND == 0 ? 0 : 8 * D);  // bytes of a slot the kernel reads
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_extra[kMaxExtra];
  __shared__ int s_nextra;
  __shared__ uint32_t s_last;

  const PoolView& pv = prm.pv;
  const int s = blockIdx.y, split = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 2, j = lane & 3;
  const int G = prm.G;
  const int n_tok = prm.tokens[s];
  const int n_pages = (n_tok + P - 1) / P;
  const uint32_t gmask = (G >= 32) ? 0xffffffffu : ((1u << G) - 1u);
  const uint32_t rmask = prm.row_mask[s] & gmask;
  const uint32_t smask = gmask & ~rmask;
  const int nsel = rmask ? prm.sel_count[s] : 0;
  const int32_t* sel = prm.sel + (int64_t)s * prm.sel_stride;
  const int sink_end = min(pv.sink, n_pages), local_start = max(n_pages - pv.local, 0);
  const int u_begin = split * prm.pps;
  uint8_t* wbuf = smem + warp * (NBUF > 0 ? NBUF : 1) * SLOT_USED;

  auto prefetch = [&](int p, int b) {
    const uint8_t* src = pv.slot_ptr(s, p);
    uint8_t* dst = wbuf + b * SLOT_USED;
    for (int i = lane; i < SLOT_USED / 16; i += 32) cp_async16(dst + 16 * i, src + 16 * i);
    cp_async_commit();
  };
  // the warp's first page can start streaming before the union is known
  int first_u = u_begin + warp;
  bool first_issued = false;
  if constexpr (NBUF > 0) {
    if (first_u < nsel && first_u < u_begin + prm.pps) {
      prefetch(sel[first_u], 0);
      first_issued = true;
    }
  }
  if (tid == 0) {
    int ne = 0;
    if (smask) {
      for (int p = 0; p < n_pages && ne < kMaxExtra; ++p) {
        if (p >= sink_end && p < local_start) {
          p = local_start - 1;
          continue;
        }
        if (!contains(sel, nsel, p)) s_extra[ne++] = p;
      }
    }
    s_nextra = ne;
  }
  __syncthreads();
  const int U = nsel + s_nextra;
  const int n_used = (U + prm.pps - 1) / prm.pps;
  const int u_end = min(U, u_begin + prm.pps);
  auto page_of = [&](int u, uint32_t& um) -> int {
    if (u < nsel) {
      int p = sel[u];
      um = rmask | ((smask && (p < sink_end || p >= local_start)) ? smask : 0u);
      return p;
    }
    um = smask;
    return s_extra[u - nsel];
  };

  // ---- per-thread row state: row r (lane/4), dims/channels of j (lane%4) ----
  const bool row_ok = r < G;
  float qf[QR];
  {
    const T* qrow = reinterpret_cast<const T*>(prm.q) + s * prm.q_ss + (int64_t)(row_ok ? r : 0) * prm.q_rs;
#pragma unroll
    for (int ri = 0; ri < D / 8; ++ri) {
      int d = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j;
      float2 v = DT<T>::to_f2(*reinterpret_cast<const uint32_t*>(qrow + d));
      qf[2 * ri] = row_ok ? v.x : 0.f;
      qf[2 * ri + 1] = row_ok ? v.y : 0.f;
    }
  }
  float o[QR];
#pragma unroll
  for (int i = 0; i < QR; ++i) o[i] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;
  const float sl2 = prm.scale_log2;
  const float inv_levels = KIND == 0 ? 1.f : 1.f / float((1 << pv.bits) - 1);

  int it = 0;
  for (int u = first_u; u < u_end; u += kWarps, ++it) {
    uint32_t um;
    const int p = page_of(u, um);
    const uint8_t* pg;
    if constexpr (NBUF > 0) {
      if (!first_issued || (NBUF == 1 && it > 0)) {
        prefetch(p, 0);
        first_issued = true;
      }
      const int un = u + kWarps;
      if (NBUF == 2 && un < u_end) {
        uint32_t um2;
        prefetch(page_of(un, um2), (it + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      pg = wbuf + (NBUF == 2 ? (it & 1) : 0) * SLOT_USED;
    } else {
      pg = pv.slot_ptr(s, p);
    }
    const int tok_in_page = min(P, n_tok - p * P);
    const uint8_t* kc = pg;
    const uint8_t* vc = pg + P * RB;
    const T* bnd = reinterpret_cast<const T*>(pg + 2 * P * RB);

    // ---- K side: q' = q * s_k / smax (A fragments), qz = q . lo_k ----
    uint32_t afr[NKS][2];
    float smax = 1.f, qz = 0.f;
    if constexpr (KIND == 0) {
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        afr[ks][0] = pack2<MT>(qf[4 * ks], qf[4 * ks + 1]);
        afr[ks][1] = pack2<MT>(qf[4 * ks + 2], qf[4 * ks + 3]);
      }
    } else {
      float sk[QR];
      const uint4* klo4 = reinterpret_cast<const uint4*>(bnd + j * QR);
      const uint4* khi4 = reinterpret_cast<const uint4*>(bnd + D + j * QR);
#pragma unroll
      for (int i = 0; i < QR / 8; ++i) {
        uint4 a = klo4[i], b = khi4[i];
        uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float2 lo = DT<T>::to_f2(aw[k]), hi = DT<T>::to_f2(bw[k]);
          int idx = 8 * i + 2 * k;
          float s0 = (hi.x - lo.x) * inv_levels, s1 = (hi.y - lo.y) * inv_levels;
          sk[idx] = s0 > 0.f ? s0 : 1.f;
          sk[idx + 1] = s1 > 0.f ? s1 : 1.f;
          qz = fmaf(qf[idx], lo.x, qz);
          qz = fmaf(qf[idx + 1], lo.y, qz);
        }
      }
      float mx = 0.f;
#pragma unroll
      for (int i = 0; i < QR; ++i) mx = fmaxf(mx, sk[i]);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      qz += __shfl_xor_sync(0xffffffffu, qz, 1);
      qz += __shfl_xor_sync(0xffffffffu, qz, 2);
      smax = mx;
      const float inv_mx = 1.f / mx;
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        afr[ks][0] = pack2<MT>(qf[4 * ks] * sk[4 * ks] * inv_mx, qf[4 * ks + 1] * sk[4 * ks + 1] * inv_mx);
        afr[ks][1] = pack2<MT>(qf[4 * ks + 2] * sk[4 * ks + 2] * inv_mx, qf[4 * ks + 3] * sk[4 * ks + 3] * inv_mx);
      }
    }

    // ---- S = q' K^T over the page's NNT n-tiles of 8 tokens ----
    float sc[NNT][2];
#pragma unroll
    for (int nt = 0; nt < NNT; ++nt) {
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
          mma16816<MT>(c, afr[ks][0], 0u, afr[ks][1], 0u, b0, b1);
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
        sc[nt][e] = t < tok_in_page ? v : -INFINITY;
      }
    }

    // ---- online softmax for row r (4 lanes j share a row) ----
    const bool attend = row_ok && ((um >> r) & 1u);
    float tmax = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < NNT; ++nt) tmax = fmaxf(tmax, fmaxf(sc[nt][0], sc[nt][1]));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    const float m_new = attend ? fmaxf(m_run, tmax) : m_run;
    const float alpha = attend ? exp2f(m_run - m_new) : 1.f;  // exp2(-inf) = 0
    uint32_t pfr[NPK][2];
    float psum = 0.f;
#pragma unroll
    for (int ks = 0; ks < NPK; ++ks) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int nt = 2 * ks + h;
        float p0 = attend ? exp2f(sc[nt][0] - m_new) : 0.f;
        float p1 = attend ? exp2f(sc[nt][1] - m_new) : 0.f;
        uint32_t pk = pack2<MT>(p0, p1);
        float2 pr = unpack2<MT>(pk);  // the rounded values the MMA sees
        psum += pr.x + pr.y;
        pfr[ks][h] = pk;
      }
    }
    l_run = l_run * alpha + psum;  // per-thread partial (tokens of lane j)
    m_run = m_new;
    float prow = psum;
    prow += __shfl_xor_sync(0xffffffffu, prow, 1);
    prow += __shfl_xor_sync(0xffffffffu, prow, 2);

    // ---- O += P V : C fragment row r, channels 8cn + 2j + {0,1} ----
    float sv[2 * NCN], vlo[2 * NCN];
    if constexpr (KIND != 0) {
      const uint4* vlo4 = reinterpret_cast<const uint4*>(bnd + 2 * D + j * QR);
      const uint4* vhi4 = reinterpret_cast<const uint4*>(bnd + 3 * D + j * QR);
#pragma unroll
      for (int i = 0; i < QR / 8; ++i) {
        uint4 a = vlo4[i], b = vhi4[i];
        uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float2 lo = DT<T>::to_f2(aw[k]), hi = DT<T>::to_f2(bw[k]);
          int idx = 8 * i + 2 * k;
          float s0 = (hi.x - lo.x) * inv_levels, s1 = (hi.y - lo.y) * inv_levels;
          sv[idx] = s0 > 0.f ? s0 : 1.f;
          sv[idx + 1] = s1 > 0.f ? s1 : 1.f;
          vlo[idx] = lo.x;
          vlo[idx + 1] = lo.y;
        }
      }
    }
#pragma unroll
    for (int cn = 0; cn < NCN; ++cn) {
      float c[4] = {0.f, 0.f, 0.f, 0.f};
      const int vl = 32 * cn + lane;  // (cn, lane) chunk
      if constexpr (KIND == 1) {
        constexpr int NW = P / 32;
        uint32_t wd[NW];
        const uint32_t* src = reinterpret_cast<const uint32_t*>(vc + vl * (P / 8));
        if constexpr (NW == 2) {
          uint2 v = *reinterpret_cast<const uint2*>(src);
          wd[0] = v.x; wd[1] = v.y;
        } else {
#pragma unroll
          for (int i = 0; i < NW; ++i) wd[i] = src[i];
        }
#pragma unroll
        for (int ks = 0; ks < NPK; ++ks) {
          int ri0 = 2 * ks, ri1 = 2 * ks + 1;
          mma16816<MT>(c, pfr[ks][0], 0u, pfr[ks][1], 0u, nib2h(wd[ri0 / 4], ri0 % 4), nib2h(wd[ri1 / 4], ri1 % 4));
        }
      } else if constexpr (KIND == 2) {
        constexpr int NW = P / 16;
        uint32_t wd[NW];
        const uint32_t* src = reinterpret_cast<const uint32_t*>(vc + vl * (P / 4));
#pragma unroll
        for (int i = 0; i < NW; ++i) wd[i] = src[i];
#pragma unroll
        for (int ks = 0; ks < NPK; ++ks)
          mma16816<MT>(c, pfr[ks][0], 0u, pfr[ks][1], 0u, byte2h(wd[ks], 0), byte2h(wd[ks], 1));
      } else {
        constexpr int NW = P / 8;
        uint32_t wd[NW];
        const uint32_t* src = reinterpret_cast<const uint32_t*>(vc + vl * (P / 2));
#pragma unroll
        for (int i = 0; i < NW; ++i) wd[i] = src[i];
#pragma unroll
        for (int ks = 0; ks < NPK; ++ks) mma16816<MT>(c, pfr[ks][0], 0u, pfr[ks][1], 0u, wd[2 * ks], wd[2 * ks + 1]);
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float add = KIND == 0 ? c[e] : fmaf(sv[2 * cn + e], c[e], vlo[2 * cn + e] * prow);
        o[2 * cn + e] = fmaf(o[2 * cn + e], alpha, add);
      }
    }
    if constexpr (NBUF > 0) __syncwarp();  // buffer may be refilled next iteration
  }

  // ---- merge the 4 warps of this CTA (rows < kMaxRows) ----
  __syncthreads();  // page buffers are reused as the merge area
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
  const int part_stride = 2 + D;
  float* part = prm.ws_part + ((int64_t)s * prm.max_splits + split) * kMaxRows * part_stride;
  if (split < n_used) {
    for (int i = tid; i < G * D; i += kDecThreads) {
      int rr = i / D, c = i % D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sm_m[w * kMaxRows + rr]);
      float L = 0.f, O = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        float f = M == -INFINITY ? 0.f : exp2f(sm_m[w * kMaxRows + rr] - M);
        L += f * sm_l[w * kMaxRows + rr];
        O += f * sm_o[(w * kMaxRows + rr) * D + c];
      }
      part[rr * part_stride + 2 + c] = O;
      if (c == 0) {
        part[rr * part_stride] = M;
        part[rr * part_stride + 1] = L;
      }
    }
  }
  const T* kn = reinterpret_cast<const T*>(prm.k_new) + s * prm.new_ss;
  const T* vn = reinterpret_cast<const T*>(prm.v_new) + s * prm.new_ss;
  // The new token joins an open page (t_old > 0): the only reader of that page
  // in this step is the unit holding page n_pages-1, so the CTA that owns it
  // appends right after its own reads -- off the critical serial tail.
  const bool opens_page = (n_tok % P) == 0;
  if (prm.fuse_append && !opens_page) {
    const int u_last = nsel > 0 ? nsel - 1 : U - 1;
    if (u_last >= u_begin && u_last < u_end) {
      __syncthreads();  // smem is reused by the append
      append_one_token<T>(pv, s, n_tok, kn, vn, smem);
    }
  }
  // ---- last CTA of the stream: merge splits + the new token, write ----
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    uint32_t t = atomicAdd(prm.ws_ticket + s, 1u);
    s_last = (t == gridDim.x - 1);
    if (s_last) prm.ws_ticket[s] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // stage every split's partial (m, l, O[D]) of this stream in smem with one
  // coalesced sweep (serialised L2 round trips would dominate the step)
  float* stage = reinterpret_cast<float*>(smem);  // [n_used][G][part_stride]
  {
    const int per_split = G * part_stride;
    const float* src = prm.ws_part + (int64_t)s * prm.max_splits * kMaxRows * part_stride;
    for (int i = tid; i < n_used * per_split; i += kDecThreads) {
      const int sp = i / per_split, rem = i % per_split;
      stage[i] = __ldcg(src + (int64_t)sp * kMaxRows * part_stride + rem);
    }
  }
  __syncthreads();
  for (int rr = warp; rr < G; rr += kWarps) {
    const T* qrow = reinterpret_cast<const T*>(prm.q) + s * prm.q_ss + (int64_t)rr * prm.q_rs;
    float dot = 0.f;
    for (int c = lane; c < D; c += 32) dot = fmaf(DT<T>::to_f(qrow[c]), DT<T>::to_f(kn[c]), dot);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
    const float s_self = dot * sl2;
    const float* pb = stage + rr * part_stride;
    const int sstride = G * part_stride;
    float M = s_self;
    for (int sp = 0; sp < n_used; ++sp) M = fmaxf(M, pb[sp * sstride]);
    float L = exp2f(s_self - M);
    for (int sp = 0; sp < n_used; ++sp) {
      const float pm = pb[sp * sstride];
      L += pm == -INFINITY ? 0.f : exp2f(pm - M) * pb[sp * sstride + 1];
    }
    const float inv_L = 1.f / L;
    const float fs = exp2f(s_self - M);
    for (int c = lane; c < D; c += 32) {
      float O = fs * DT<T>::to_f(vn[c]);
      for (int sp = 0; sp < n_used; ++sp) {
        const float pm = pb[sp * sstride];
        if (pm != -INFINITY) O = fmaf(exp2f(pm - M), pb[sp * sstride + 2 + c], O);
      }
      O *= inv_L;
      int64_t oi = s * prm.out_ss + (int64_t)rr * prm.out_rs + c;
      if (prm.out_dtype == SK_F32) reinterpret_cast<float*>(prm.out)[oi] = O;
      else if (prm.out_dtype == SK_F16) reinterpret_cast<__half*>(prm.out)[oi] = __float2half_rn(O);
      else reinterpret_cast<__nv_bfloat16*>(prm.out)[oi] = __float2bfloat16_rn(O);
    }
  }
  if (prm.fuse_append) {
    if (opens_page) {
      // a fresh page may reuse a streaming ring slot read in this step: only now is it free
      __syncthreads();
      append_page<T>(pv, s, n_tok / P, n_tok, n_tok + 1, kn, vn, 0, smem);
    }
    __syncthreads();
    if (tid == 0) prm.tokens[s] = n_tok + 1;
  }
}

__host__ __device__ constexpr int slot_used(int kind, int D, int P) {
  return 2 * P * (kind == 0 ? 2 * D : (kind == 1 ? D / 2 : D)) + (kind == 0 ? 0 : 8 * D);
}

template <typename T, int KIND, int D, int P>
int launch_one(const DecodeParams& prm, dim3 grid, size_t smem_min, cudaStream_t st) {
  constexpr int SLOT = slot_used(KIND, D, P);
  constexpr int NBUF = (2 * kWarps * SLOT <= 160 * 1024) ? 2 : ((kWarps * SLOT <= 160 * 1024) ? 1 : 0);
  size_t smem = (size_t)kWarps * (NBUF > 0 ? NBUF : 0) * SLOT;
  if (smem < smem_min) smem = smem_min;
  auto kern = decode_kernel<T, KIND, D, P, NBUF>;
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
  SK_CHECK_ARG(pages_per_split >= 1 && max_splits >= 1, "decode: bad split geometry");
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
  size_t smem_merge = (size_t)kWarps * kMaxRows * (2 + pool->head_dim) * 4;
  size_t smem_app = fuse_append ? append_smem_bytes(pool->head_dim, pool->page_size) : 0;
  size_t smem_one = append_one_smem_bytes(pool->head_dim, pool->page_size);
  if (smem_app < smem_one) smem_app = smem_one;
  size_t smem_comb = (size_t)max_splits * group_rows * (2 + pool->head_dim) * 4;
  if (smem_app < smem_comb) smem_app = smem_comb;
  size_t smem = smem_merge > smem_app ? smem_merge : smem_app;
  dim3 grid(max_splits, n_streams);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int kind = pool->bits == 0 ? 0 : (pool->bits <= 4 ? 1 : 2);
  if (pool->dtype == SK_F16) {
    if (kind == 0) return launch_kind<__half, 0>(prm, grid, smem, st);
    if (kind == 1) return launch_kind<__half, 1>(prm, grid, smem, st);
    return launch_kind<__half, 2>(prm, grid, smem, st);
  }
  if (kind == 0) return launch_kind<__nv_bfloat16, 0>(prm, grid, smem, st);
  if (kind == 1) return launch_kind<__nv_bfloat16, 1>(prm, grid, smem, st);
  return launch_kind<__nv_bfloat16, 2>(prm, grid, smem, st);
}
