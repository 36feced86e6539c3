// K3 -- split-KV decode attention over the selected pages (+ append).
//
// Replaces the per-head page loop of Engine.decode_step (reference
// engine.py:257-285), PhysicalPage.dequantize (cache.py:97-102) and
// merge_block (attn.py:191-229).
//
// Work decomposition (latency-first: a 128k decode step of one layer reads
// ~5 MB, under a microsecond of HBM time, so the kernel is built around the
// number of dependent round trips and the length of each warp's dependent
// compute chain, not bandwidth):
//   * grid (cps, streams): cps CTAs per stream (= one KV head of one
//     sequence), sized so that all the streams together fill the 148 SMs
//     (decode_cps: 18 per stream for 8 streams, 1 once the streams alone
//     fill the GPU).  The stream's page union -- the selection for retrieval
//     rows plus the sink/local window for streaming rows, each page carrying
//     the mask of group rows that attend it -- is cut into 32-token units
//     (two 16-token MMA tiles), dealt round-robin over the stream's
//     cps x 8 warps: at 128k each warp owns at most one unit;
//   * a warp issues every load of its unit straight into registers
//     (128-bit, coalesced: K1 writes the codes in the m16n8k16 fragment
//     order, sk_layout.cuh) before doing any math, then runs QK and PV as
//     m16n8k16 tensor-core MMAs on the stored codes through the
//     dequantisation algebra
//         q . khat_t = sum_d (q_d s_d) c_td + sum_d q_d lo_d
//         sum_t p_t vhat_tc = s_c sum_t p_t c_tc + lo_c sum_t p_t
//     (codes -> exact fp16 integers with one LOP3 + one HSUB2 per two),
//     TRANSPOSED so tokens / channels sit in the MMA's M dimension and the
//     <= 8 group rows in N: S^T = K q'^T, O^T += V^T P^T;
//   * one online-softmax state per (warp, row); the CTA's warps merge in
//     shared memory; with cps > 1 each CTA writes its partial (m, l, O) to
//     the workspace and the stream's last CTA (an acq_rel ticket) merges the
//     cps partials with log-sum-exp together with the new token's raw K/V
//     (engine.py:276-277) and writes the output.
// Round trips on the critical path: {tokens, selection, q} -> page table ->
// unit data -> (partial, ticket) -> partials.
#include <cstdlib>

#include "append_impl.cuh"
#include "sk_sm100.cuh"

namespace sk {
int append_launch(const sk_pool* pool, int n_streams, const void* k_src, const void* v_src, int64_t ss, int64_t ts,
                  int32_t* tokens, int m, int max_pages_touched, cudaStream_t st);
}  // namespace sk

namespace sk {
namespace {

constexpr int kDecThreads = 256;
constexpr int kWarps = kDecThreads / 32;
constexpr int kMaxRows = 8;    // group rows (query heads per KV head)
constexpr int kMaxExtra = 64;  // sink + local pages
constexpr int kMaxSel = 2048;  // selection entries staged in smem
constexpr int kMaxCps = 31;    // CTAs per stream (the finish gives each a lane, plus the new token)
constexpr int kUnitTok = 32;   // tokens per work unit when a stream spans several CTAs (two 16-token tiles)

// CTAs per stream: fill the SMs when the streams are few, never more CTAs
// than the stream's largest possible union needs (8 units per CTA).
inline int decode_cps(int n_streams, int max_units) {
  int c = device_sm_count() / n_streams;
  c = c < 1 ? 1 : (c > kMaxCps ? kMaxCps : c);
  const int need = (max_units + kWarps - 1) / kWarps;
  return c < need ? c : (need < 1 ? 1 : need);
}
// m[G], l[G], O[G][D], padded to 16 bytes (the last CTA bulk-copies the partials)
__host__ __device__ inline int64_t part_floats(int G, int D) { return (2ll * G + (int64_t)G * D + 3) / 4 * 4; }
inline int64_t ticket_bytes(int n_streams) { return ((int64_t)n_streams * 4 + 255) / 256 * 256; }

struct DecodeParams {
  PoolView pv;
  int G;
  const void* q;
  int64_t q_ss, q_rs;
  const void* k_new;
  const void* v_new;
  int64_t new_ss;
  const uint32_t* row_mask;
  const uint32_t* row_window;  // [stream][row] sink | local << 16 (pages), or NULL = the pool's window
  const int32_t* sel;
  const int32_t* sel_count;
  int sel_stride;
  const int32_t* tokens;
  float scale_log2;
  void* out;
  int64_t out_ss, out_rs;
  int out_dtype;
  uint32_t flags;    // SK_DECODE_* / SK_LAUNCH_PDL
  int cps;           // CTAs per stream (gridDim.x)
  float* part;       // [stream][cps][part_floats]
  uint32_t* ticket;  // [stream]
};

// Timing build only (-DSK_DEC_TIMING, tools/decode_stamp_probe.py): globaltimer
// stamps of each CTA's phases, read back with sk_debug_decode_stamps.
#ifdef SK_DEC_TIMING
__device__ uint64_t g_dec_stamps[4096][8];
#define DSTAMP(i)                                                                   \
  do {                                                                              \
    if (threadIdx.x == 0) {                                                         \
      uint64_t t_;                                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
      g_dec_stamps[(blockIdx.y * gridDim.x + blockIdx.x) & 4095][(i)] = t_;         \
    }                                                                               \
  } while (0)
// warp-level: globaltimer + clock64 around one unit's compute (CTA 0 of stream 0)
#define WSTAMP(i)                                                                          \
  do {                                                                                     \
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0 && blockIdx.y == 0) {                   \
      uint64_t t_, c_;                                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_));                                   \
      g_dec_stamps[4000 + (threadIdx.x >> 5)][2 * (i)] = t_;                               \
      g_dec_stamps[4000 + (threadIdx.x >> 5)][2 * (i) + 1] = c_;                           \
    }                                                                                      \
  } while (0)
#else
#define DSTAMP(i) \
  do {            \
  } while (0)
#define WSTAMP(i) \
  do {            \
  } while (0)
#endif

// timing builds only (tools/ab_variant.sh): 2 = no ticket / merge of the
// partials, 3 = the last CTA skips the final merge, 4 = units only
#ifndef SK_DEC_ABLATE
#define SK_DEC_ABLATE 0
#endif
#ifndef SK_DEC_STAGE  // 0: the one-CTA-per-stream path loads pages straight into registers
#define SK_DEC_STAGE 1
#endif
#ifndef SK_DEC_MINB
#define SK_DEC_MINB 1
#endif

// m16n8k16 MMA, fp32 accumulate.
template <typename MT>
__device__ __forceinline__ void mma16816_full(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
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

// Code word -> fp16x2 MMA operand, with NO conversion arithmetic: the codes
// are used as fp16 SUBNORMALS (the tensor cores multiply subnormal fp16
// operands exactly; every product and partial sum stays a normal fp32).
// Nibble slot 0/2 (bits 0-3 / 8-11 of each 16-bit half) masks to n * 2^-24,
// slot 1/3 (bits 4-7 / 12-15) to 16 n * 2^-24 in place, so a word costs one
// shift (shared by slots 2 and 3) and four single-immediate LOP3s; the odd
// slots feed the MMA's second k-half (a2/a3), whose B operand carries the
// matching 1/16, and the accumulator is scaled back by 2^24 (kCodeUnscale).
// Round 2 formed exact fp16 integers (LOP3 into 1024 + n, then HSUB2/HFMA2):
// ptxas splits that LOP3 in two (one immediate per instruction), so a word
// cost 13 instructions instead of 5 (ncu, cfg4 K3: 27% of all instructions
// were LOP3, 14% HADD2).
constexpr float kCodeUnscale = 16777216.f;  // 2^24
constexpr float kOddSlot = 0.0625f;         // 1/16 on the B operand of the odd nibble slots
__device__ __forceinline__ uint32_t nib2h(uint32_t w, int slot) {
  const uint32_t x = slot >= 2 ? (w >> 8) : w;
  return x & ((slot & 1) ? 0x00F000F0u : 0x000F000Fu);
}
// byte pair (r2 = 0: bytes 0,1; r2 = 1: bytes 2,3) -> fp16x2 subnormals b * 2^-24
__device__ __forceinline__ uint32_t byte2h(uint32_t w, int r2) {
  return __byte_perm(w, 0u, r2 ? 0x4342 : 0x4140);  // {b, 0, b', 0}
}

// packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2 on sm_100): two lanes of
// scale / bias work per instruction in the per-page dequantisation algebra
__device__ __forceinline__ uint64_t x2(float x, float y) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ float2 x2f(uint64_t r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ uint64_t x2mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t x2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__device__ __forceinline__ uint4 ldg16(const void* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ uint2 ldg8(const void* p) { return __ldg(reinterpret_cast<const uint2*>(p)); }
// unit loads from global memory (SM = false) or from a page staged in shared
// memory by a bulk copy (SM = true)
template <bool SM>
__device__ __forceinline__ uint4 ldu16(const void* p) {
  if constexpr (SM) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(p)));
    return v;
  } else {
    return ldg16(p);
  }
}
template <bool SM>
__device__ __forceinline__ uint2 ldu8(const void* p) {
  if constexpr (SM) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(smem_u32(p)));
    return v;
  } else {
    return ldg8(p);
  }
}
template <bool SM>
__device__ __forceinline__ uint32_t ldu4(const void* p) {
  if constexpr (SM) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)));
    return v;
  } else {
    return __ldg(reinterpret_cast<const uint32_t*>(p));
  }
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

// movmatrix: transpose an 8x8 b16 matrix held in the standard fragment
// layout (thread l holds row l/4, columns 2(l%4), 2(l%4)+1).
__device__ __forceinline__ uint32_t transpose8x8(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// Per-(warp) online-softmax state of the thread's two group rows 2j, 2j+1
// and its output channels 16*ct + g + 8*h (g = lane/4, j = lane%4).
template <int D>
struct RowState {
  float m[2], l[2];
  float o[D / 16][4];  // [ct][2h + e]: channel 16ct + g + 8h, row 2j + e
};

// One 32-token unit (tiles tt0, tt0+1 of a page) for one warp, computed
// TRANSPOSED so that the 16-row MMA dimension carries tokens (QK) and
// channels (PV) and the group rows (<= 8) sit in N = 8: S^T = K q'^T and
// O^T += V^T P^T.  The A fragments are exactly the bytes K1 stores per
// (token, lane%4) and (channel tile, lane) (sk_layout.cuh); P goes from the
// S^T accumulator to the P^T operand with one movmatrix per 8x8.
// KIND: 0 raw pages (MMA in T), 1 nibble codes, 2 byte codes (MMA in fp16).
template <typename T, int KIND, int D, int P, int UT>
struct UnitData {
  static constexpr int RB = KIND == 0 ? 2 * D : (KIND == 1 ? D / 2 : D);
  static constexpr int KW = KIND == 1 ? D / 32 : (KIND == 2 ? D / 16 : D / 8);  // words per (token, lane%4)
  static constexpr int VW = KIND == 1 ? P / 32 : (KIND == 2 ? P / 16 : P / 8);  // words per (cn, lane), whole page
  static constexpr int VU = KIND == 1 ? UT / 2 : (KIND == 2 ? UT : 2 * UT);     // of them used by one unit
  uint32_t kw[UT][2][KW];
  uint32_t vw[D / 8][VU];
  uint32_t kb_lo[D / 8], kb_hi[D / 8], vb_lo[D / 8], vb_hi[D / 8];
};

// Every load of one 32-token unit (tiles tt0, tt0+1 of the page in slot pg),
// straight into registers -- issued before any math (one round trip), and
// for the first unit before the kernel's dependency wait (PDL prologue).
template <typename T, int KIND, int D, int P, int UT, bool SM = false>
__device__ __forceinline__ void unit_load(const uint8_t* pg, int tt0, UnitData<T, KIND, D, P, UT>& u) {
  using U = UnitData<T, KIND, D, P, UT>;
  constexpr int NCT = D / 16;
  constexpr int RB = U::RB, KW = U::KW, VW = U::VW, VU = U::VU;
  const int lane = threadIdx.x & 31, g = lane >> 2, j = lane & 3;
  const uint8_t* kc = pg;
  const uint8_t* vc = pg + P * RB;
  const T* bnd = reinterpret_cast<const T*>(pg + 2 * P * RB);
  // K codes of tokens 16tt + g + 8h (A rows), this lane's dim chunk j
#pragma unroll
  for (int i = 0; i < UT; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint8_t* src = kc + (16 * (tt0 + i) + 8 * h + g) * RB + j * (RB / 4);
      if constexpr (KW == 2) {
        const uint2 v = ldu8<SM>(src);
        u.kw[i][h][0] = v.x; u.kw[i][h][1] = v.y;
      } else {
#pragma unroll
        for (int w = 0; w < KW / 4; ++w) {
          const uint4 v = ldu16<SM>(src + 16 * w);
          u.kw[i][h][4 * w] = v.x; u.kw[i][h][4 * w + 1] = v.y; u.kw[i][h][4 * w + 2] = v.z; u.kw[i][h][4 * w + 3] = v.w;
        }
      }
    }
  // V codes of the unit's tokens: chunk (cn, lane), cn = 2ct + h
  const int w0 = KIND == 1 ? tt0 / 2 : (KIND == 2 ? tt0 : 2 * tt0);  // first word of the unit
#pragma unroll
  for (int cn = 0; cn < 2 * NCT; ++cn) {
    const uint8_t* src = vc + ((32 * cn + lane) * VW + w0) * 4;
    if constexpr (VU == 1) {
      u.vw[cn][0] = ldu4<SM>(src);
    } else if constexpr (VU == 2) {
      const uint2 v = ldu8<SM>(src);
      u.vw[cn][0] = v.x; u.vw[cn][1] = v.y;
    } else {
#pragma unroll
      for (int w = 0; w < VU / 4; ++w) {
        const uint4 v = ldu16<SM>(src + 16 * w);
        u.vw[cn][4 * w] = v.x; u.vw[cn][4 * w + 1] = v.y; u.vw[cn][4 * w + 2] = v.z; u.vw[cn][4 * w + 3] = v.w;
      }
    }
  }
  // bounds: K in kbound order (this lane's dims at j*D/4), V in vbound order
  // (channels 16ct + g + 8h at (g/2)*D/4 + 4ct + 2h + g%2)
  if constexpr (KIND != 0) {
#pragma unroll
    for (int i = 0; i < D / 32; ++i) {
      const uint4 a = ldu16<SM>(bnd + j * (D / 4) + 8 * i), b = ldu16<SM>(bnd + D + j * (D / 4) + 8 * i);
      const uint4 c = ldu16<SM>(bnd + 2 * D + (g >> 1) * (D / 4) + 8 * i);
      const uint4 d = ldu16<SM>(bnd + 3 * D + (g >> 1) * (D / 4) + 8 * i);
      u.kb_lo[4 * i] = a.x; u.kb_lo[4 * i + 1] = a.y; u.kb_lo[4 * i + 2] = a.z; u.kb_lo[4 * i + 3] = a.w;
      u.kb_hi[4 * i] = b.x; u.kb_hi[4 * i + 1] = b.y; u.kb_hi[4 * i + 2] = b.z; u.kb_hi[4 * i + 3] = b.w;
      u.vb_lo[4 * i] = c.x; u.vb_lo[4 * i + 1] = c.y; u.vb_lo[4 * i + 2] = c.z; u.vb_lo[4 * i + 3] = c.w;
      u.vb_hi[4 * i] = d.x; u.vb_hi[4 * i + 1] = d.y; u.vb_hi[4 * i + 2] = d.z; u.vb_hi[4 * i + 3] = d.w;
    }
  }
}

// One 32-token unit (tiles tt0, tt0+1 of a page) for one warp, computed
// TRANSPOSED so that the 16-row MMA dimension carries tokens (QK) and
// channels (PV) and the group rows (<= 8) sit in N = 8: S^T = K q'^T and
// O^T += V^T P^T.  The A fragments are exactly the bytes K1 stores per
// (token, lane%4) and (channel tile, lane) (sk_layout.cuh); P goes from the
// S^T accumulator to the P^T operand with one movmatrix per 8x8.
// KIND: 0 raw pages (MMA in T), 1 nibble codes, 2 byte codes (MMA in fp16).
template <typename T, int KIND, int D, int P, int UT>
__device__ __forceinline__ void unit_compute(const UnitData<T, KIND, D, P, UT>& u, int tt0, int tok_in_page,
                                             uint32_t att_mask, const uint32_t (&qw)[D / 8], float sl2,
                                             float inv_levels, RowState<D>& st) {
  using MT = typename std::conditional<KIND == 0, T, __half>::type;
  constexpr int NKS = D / 16;  // QK k-steps (16 dims)
  constexpr int NCT = D / 16;  // PV M-tiles (16 channels)
  constexpr int TT = UT;       // 16-token tiles per unit
  const int lane = threadIdx.x & 31, g = lane >> 2, j = lane & 3;
  const auto& kw = u.kw;
  const auto& vw = u.vw;
  const auto& kb_lo = u.kb_lo;
  const auto& kb_hi = u.kb_hi;
  const auto& vb_lo = u.vb_lo;
  const auto& vb_hi = u.vb_hi;

  // ---- K side: B = q'^T with q' = q * s_k / smax (row g), qz_r = q_r . lo_k --------
  uint32_t bq[NKS][2];
  float smax = 1.f, qz = 0.f;
  if constexpr (KIND == 0) {
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks) {
      bq[ks][0] = qw[2 * ks];
      bq[ks][1] = qw[2 * ks + 1];
    }
  } else {
    // s_k = (hi - lo) / levels per channel; a constant channel (s_k = 0) has
    // all-zero codes, so its scale never reaches the score
    uint64_t qs2[D / 8];  // (q s_k) channel pairs
    uint64_t qz2 = x2(0.f, 0.f);
    float mx = 0.f;
    const uint64_t il2 = x2(inv_levels, inv_levels), m12 = x2(-1.f, -1.f);
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const float2 lo = DT<T>::to_f2(kb_lo[i]), hi = DT<T>::to_f2(kb_hi[i]), q = DT<T>::to_f2(qw[i]);
      const uint64_t lo2 = x2(lo.x, lo.y), q2 = x2(q.x, q.y);
      const uint64_t s2 = x2mul(x2fma(lo2, m12, x2(hi.x, hi.y)), il2);
      const float2 sf = x2f(s2);
      mx = fmax3(mx, sf.x, sf.y);
      qs2[i] = x2mul(q2, s2);
      qz2 = x2fma(q2, lo2, qz2);
    }
    const float2 qzf = x2f(qz2);
    qz = qzf.x + qzf.y;
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    qz += __shfl_xor_sync(0xffffffffu, qz, 1);
    qz += __shfl_xor_sync(0xffffffffu, qz, 2);  // qz of row g
    mx = mx > 0.f ? mx : 1.f;                    // every channel constant
    smax = mx;
    const float inv = 1.f / mx, inv1 = KIND == 1 ? inv * kOddSlot : inv;  // k-half 1 = odd nibble slots
    const uint64_t i0 = x2(inv, inv), i1 = x2(inv1, inv1);
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks) {
      const float2 a = x2f(x2mul(qs2[2 * ks], i0)), b = x2f(x2mul(qs2[2 * ks + 1], i1));
      bq[ks][0] = pack2<MT>(a.x, a.y);
      bq[ks][1] = pack2<MT>(b.x, b.y);
    }
  }
  // the S^T accumulator holds rows 2j, 2j+1: fetch their qz from lanes 8j, 8j+4
  const float qz0 = __shfl_sync(0xffffffffu, qz, 8 * j), qz1 = __shfl_sync(0xffffffffu, qz, 8 * j + 4);

  // codes enter the MMA as subnormals: undo their 2^-24 with the page scale
  // (fp16 scales cannot overflow by it; bf16 ones keep a separate exact multiply)
  float smax_u = smax;
  if constexpr (KIND != 0) {
    if constexpr (std::is_same<T, __half>::value) smax_u = smax * kCodeUnscale;
  }
  constexpr float kAccU = (KIND != 0 && !std::is_same<T, __half>::value) ? kCodeUnscale : 1.f;

  // ---- S^T = K q'^T: tile i gives tokens 16(tt0+i) + g (+8), rows 2j, 2j+1 ---------
  float sc[TT][4];
#pragma unroll
  for (int i = 0; i < TT; ++i) {
    float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks) {
      uint32_t a0, a1, a2, a3;  // (tok g, dims lo) (tok g+8, lo) (tok g, hi) (tok g+8, hi)
      const int ri0 = 2 * ks, ri1 = 2 * ks + 1;
      if constexpr (KIND == 1) {
        a0 = nib2h(kw[i][0][ri0 / 4], ri0 % 4);
        a1 = nib2h(kw[i][1][ri0 / 4], ri0 % 4);
        a2 = nib2h(kw[i][0][ri1 / 4], ri1 % 4);
        a3 = nib2h(kw[i][1][ri1 / 4], ri1 % 4);
      } else if constexpr (KIND == 2) {
        a0 = byte2h(kw[i][0][ks], 0);
        a1 = byte2h(kw[i][1][ks], 0);
        a2 = byte2h(kw[i][0][ks], 1);
        a3 = byte2h(kw[i][1][ks], 1);
      } else {
        a0 = kw[i][0][ri0];
        a1 = kw[i][1][ri0];
        a2 = kw[i][0][ri1];
        a3 = kw[i][1][ri1];
      }
      mma16816_full<MT>(c, a0, a1, a2, a3, bq[ks][0], bq[ks][1]);
    }
    if constexpr (kAccU != 1.f) {
#pragma unroll
      for (int e = 0; e < 4; ++e) c[e] *= kAccU;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool ok = 16 * (tt0 + i) + 8 * h + g < tok_in_page;
      sc[i][2 * h] = ok ? (c[2 * h] * smax_u + qz0) * sl2 : -INFINITY;
      sc[i][2 * h + 1] = ok ? (c[2 * h + 1] * smax_u + qz1) * sl2 : -INFINITY;
    }
  }

  // ---- per-row unit max, rescale, probabilities -----------------------------------
  float tmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int i = 0; i < TT; ++i) {
    tmax[0] = fmax3(tmax[0], sc[i][0], sc[i][2]);
    tmax[1] = fmax3(tmax[1], sc[i][1], sc[i][3]);
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    tmax[e] = fmaxf(tmax[e], __shfl_xor_sync(0xffffffffu, tmax[e], 4));
    tmax[e] = fmaxf(tmax[e], __shfl_xor_sync(0xffffffffu, tmax[e], 8));
    tmax[e] = fmaxf(tmax[e], __shfl_xor_sync(0xffffffffu, tmax[e], 16));
  }
  bool att[2];
  float alpha[2], m_new[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    att[e] = (att_mask >> (2 * j + e)) & 1u;
    m_new[e] = att[e] ? fmaxf(st.m[e], tmax[e]) : st.m[e];
    alpha[e] = att[e] ? exp2f(st.m[e] - m_new[e]) : 1.f;  // exp2(-inf) = 0
  }
  uint32_t pb[TT][2];  // P^T B fragments: (tokens 2j.., row g) / (tokens 2j+8.., row g)
  float psum[2] = {0.f, 0.f};
#pragma unroll
  for (int i = 0; i < TT; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float p0 = att[0] ? fast_exp2(sc[i][2 * h] - m_new[0]) : 0.f;
      const float p1 = att[1] ? fast_exp2(sc[i][2 * h + 1] - m_new[1]) : 0.f;
      // tokens 8..15 of the tile (h = 1) meet the odd nibble slots: P / 16 there
      const float ps = (KIND == 1 && h == 1) ? kOddSlot : 1.f;
      const uint32_t pk = pack2<MT>(p0 * ps, p1 * ps);  // (token 16tt + 8h + g, rows 2j, 2j+1)
      const float2 pr = unpack2<MT>(pk);               // the rounded values the MMA sees
      psum[0] = fmaf(pr.x, 1.f / ps, psum[0]);
      psum[1] = fmaf(pr.y, 1.f / ps, psum[1]);
      pb[i][h] = transpose8x8(pk);
    }
  float prow[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    st.l[e] = st.l[e] * alpha[e] + psum[e];  // per-thread partial (tokens of lane g)
    st.m[e] = m_new[e];
    prow[e] = psum[e];
    prow[e] += __shfl_xor_sync(0xffffffffu, prow[e], 4);
    prow[e] += __shfl_xor_sync(0xffffffffu, prow[e], 8);
    prow[e] += __shfl_xor_sync(0xffffffffu, prow[e], 16);
  }

  // ---- O^T = alpha O^T + s_v (V^T P^T) + lo_v sum(P) -----------------------------
  const uint64_t prow2 = x2(prow[0], prow[1]), alpha2 = x2(alpha[0], alpha[1]);
  const uint32_t vsel = (g & 1) ? 0x7632u : 0x5410u;  // {lo, hi} halves of this lane's channel
  const float inv_v = std::is_same<T, __half>::value ? inv_levels * kCodeUnscale : inv_levels;
#pragma unroll
  for (int ct = 0; ct < NCT; ++ct) {
    float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < TT; ++i) {
      uint32_t a0, a1, a2, a3;  // (ch g, tok lo) (ch g+8, lo) (ch g, hi) (ch g+8, hi)
      if constexpr (KIND == 1) {  // word i/2 of the unit, slots 2(i%2), 2(i%2)+1: tile tt0+i
        a0 = nib2h(vw[2 * ct][i / 2], 2 * (i % 2));
        a1 = nib2h(vw[2 * ct + 1][i / 2], 2 * (i % 2));
        a2 = nib2h(vw[2 * ct][i / 2], 2 * (i % 2) + 1);
        a3 = nib2h(vw[2 * ct + 1][i / 2], 2 * (i % 2) + 1);
      } else if constexpr (KIND == 2) {
        a0 = byte2h(vw[2 * ct][i], 0);
        a1 = byte2h(vw[2 * ct + 1][i], 0);
        a2 = byte2h(vw[2 * ct][i], 1);
        a3 = byte2h(vw[2 * ct + 1][i], 1);
      } else {
        a0 = vw[2 * ct][2 * i];
        a1 = vw[2 * ct + 1][2 * i];
        a2 = vw[2 * ct][2 * i + 1];
        a3 = vw[2 * ct + 1][2 * i + 1];
      }
      mma16816_full<MT>(c, a0, a1, a2, a3, pb[i][0], pb[i][1]);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint64_t add = x2(c[2 * h], c[2 * h + 1]);
      if constexpr (KIND != 0) {
        // channel 16ct + 8h + g: half g%2 of vbound words (g/2)*D/4 + 2*(2ct+h)
        const float2 b = DT<T>::to_f2(__byte_perm(vb_lo[2 * ct + h], vb_hi[2 * ct + h], vsel));  // (lo_c, hi_c)
        const float sc_ = (b.y - b.x) * inv_v;  // a constant channel's codes are 0: any scale
        if constexpr (kAccU != 1.f) add = x2mul(add, x2(kAccU, kAccU));
        add = x2fma(x2(sc_, sc_), add, x2mul(x2(b.x, b.x), prow2));
      }
      const float2 o = x2f(x2fma(x2(st.o[ct][2 * h], st.o[ct][2 * h + 1]), alpha2, add));
      st.o[ct][2 * h] = o.x;
      st.o[ct][2 * h + 1] = o.y;
    }
  }
}

// Merge of a stream's partials (m, l, O over channel c) with the new token
// (score s_new, value v_c) and write of the normalised output.
template <typename T>
__device__ __forceinline__ void finish_out(const DecodeParams& prm, int s, int rr, int c, float M, float L, float O) {
  const int64_t oi = s * prm.out_ss + (int64_t)rr * prm.out_rs + c;
  O /= L;
  if (prm.out_dtype == SK_F32) reinterpret_cast<float*>(prm.out)[oi] = O;
  else if (prm.out_dtype == SK_F16) reinterpret_cast<__half*>(prm.out)[oi] = __float2half_rn(O);
  else reinterpret_cast<__nv_bfloat16*>(prm.out)[oi] = __float2bfloat16_rn(O);
}

// Bytes of a page slot a unit reads: codes of K and V, then the four bound rows.
template <int KIND, int D, int P>
__host__ __device__ constexpr int slot_used_bytes() {
  return (KIND == 0 ? 4 * P * D : (KIND == 1 ? P * D : 2 * P * D)) + (KIND == 0 ? 0 : 8 * D);
}
// STAGE (one CTA per stream, whole-page units): each warp streams its pages
// through two shared-memory buffers filled by bulk copies, the next page in
// flight while the current one computes.
template <int KIND, int D, int P, int UT>
__host__ __device__ constexpr bool stage_fits() {
  return KIND == 1 && P == 16 * UT && 2 * kWarps * slot_used_bytes<KIND, D, P>() <= 160 * 1024;
}

template <typename T, int KIND, int D, int P, int UT, bool STAGE = false>
__global__ void __launch_bounds__(kDecThreads, SK_DEC_MINB) decode_kernel(const __grid_constant__ DecodeParams prm) {
  constexpr int UPP = P / (16 * UT);  // units per page
  constexpr int kSlotUsed = slot_used_bytes<KIND, D, P>();
  static_assert(!STAGE || stage_fits<KIND, D, P, UT>(), "staged decode needs whole-page units that fit");
  __shared__ uint64_t s_sbar[STAGE ? 2 * kWarps : 1];
  __shared__ int s_sel[kMaxSel];
  __shared__ int s_extra[kWarps][kMaxExtra];
  __shared__ float s_m[kWarps][kMaxRows], s_l[kWarps][kMaxRows];
  __shared__ __align__(16) float s_o[kWarps][kMaxRows][D];
  __shared__ float s_self[kMaxRows];
  __shared__ uint32_t s_last;
  __shared__ uint64_t s_bar;
  extern __shared__ __align__(16) float s_part[];  // last CTA: [cps][part_floats] (dynamic)
  DSTAMP(0);
  const PoolView& pv = prm.pv;
  const int s = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 2, g = r, j = lane & 3;
  const int G = prm.G;

  // Programmatic dependent launch (SK_LAUNCH_PDL): let the next kernel's CTAs
  // start their own prologue as SMs free up, and read nothing the previous
  // kernel may write -- q, the new token, and (unless SK_DECODE_SEL_READY)
  // the selection -- before griddepcontrol.wait.
  const bool pdl = prm.flags & SK_LAUNCH_PDL;
  const bool early_sel = !pdl || (prm.flags & SK_DECODE_SEL_READY);
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // ---- round trip 1: header and selection (independent loads) ---------------
  const int n_tok = prm.tokens[s];
  const uint32_t rm_raw = prm.row_mask[s];
  // per-row streaming windows (HeadProfile.sink_blocks / local_blocks, engine.py:264-267)
  uint32_t win = (uint32_t)pv.sink | ((uint32_t)pv.local << 16);
  if (prm.row_window != nullptr && lane < G) win = __ldg(prm.row_window + (int64_t)s * G + lane);
  if (!early_sel) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int cnt_raw = prm.sel_count[s];
  const int32_t* sel = prm.sel + (int64_t)s * prm.sel_stride;
  const int sel_w = min(prm.sel_stride, kMaxSel);
  for (int i = tid; i < sel_w; i += kDecThreads) s_sel[i] = __ldcg(sel + i);
  const int n_pages = (n_tok + pv.P - 1) / pv.P;
  const uint32_t gmask = (G >= 32) ? 0xffffffffu : ((1u << G) - 1u);
  const uint32_t rmask = rm_raw & gmask;
  const uint32_t smask = gmask & ~rmask;
  const int nsel = rmask ? min(cnt_raw, sel_w) : 0;
  // lane r (< G) holds row r's window; the union over streaming rows is
  // [0, max sink) u [n - max local, n), and each page carries the mask of
  // the streaming rows whose own window contains it
  const bool srow = lane < G && ((smask >> lane) & 1u);
  const int my_sink = srow ? min((int)(win & 0xFFFFu), n_pages) : 0;
  const int my_loc = srow ? max(n_pages - (int)(win >> 16), 0) : n_pages;
  int sink_end = my_sink, local_start = my_loc;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    sink_end = max(sink_end, __shfl_xor_sync(0xffffffffu, sink_end, off));
    local_start = min(local_start, __shfl_xor_sync(0xffffffffu, local_start, off));
  }
  // streaming rows attending page pg (warp-uniform pg)
  auto win_rows = [&](int pg) -> uint32_t {
    return __ballot_sync(0xffffffffu, srow && (pg < my_sink || pg >= my_loc));
  };
  __syncthreads();
  DSTAMP(1);
  // ---- the stream's page union: selection + sink/local pages it lacks.  Each
  //      warp derives it itself (a ballot over <= 32 candidates against the
  //      staged selection), so no second CTA barrier sits on the critical path.
  int* w_extra = s_extra[warp];
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
      if (extra && pos < kMaxExtra) w_extra[pos] = p;
      ne += __popc(bal);
    }
    ne = min(ne, kMaxExtra);
  }
  __syncwarp();
  const int NU = (nsel + ne) * UPP;  // 32-token units of the union

  // ---- this warp's units: u = warp index in the stream + k * (cps * kWarps) ----
  RowState<D> st;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    st.m[e] = -INFINITY;
    st.l[e] = 0.f;
  }
#pragma unroll
  for (int ct = 0; ct < D / 16; ++ct)
#pragma unroll
    for (int i = 0; i < 4; ++i) st.o[ct][i] = 0.f;
  const float sl2 = prm.scale_log2;
  const float inv_levels = KIND == 0 ? 1.f : 1.f / float((1 << pv.bits) - 1);
  auto unit_page = [&](int u, uint32_t& um) -> int {
    const int pi = u / UPP;
    const int pg = pi < nsel ? s_sel[pi] : w_extra[pi - nsel];
    um = (pi < nsel ? rmask : 0u) | (smask ? win_rows(pg) : 0u);
    return pg;
  };
  const int ustride = prm.cps * kWarps;
  int u = blockIdx.x * kWarps + warp;
  int pg_next = 0;
  uint32_t um_next = 0;
  const uint8_t* slot_next = nullptr;
  UnitData<T, KIND, D, P, UT> ud;
  uint64_t* sbar = s_sbar + 2 * warp;
  uint8_t* sbuf = reinterpret_cast<uint8_t*>(s_part) + (size_t)warp * 2 * kSlotUsed;
  // the slots of the warp's units k0 .. k0+31 (unit u0 + k * ustride), lane k - k0
  // each: one page-table round trip per 32 units instead of one per unit
  const int u0 = u;
  const uint8_t* lane_slot = nullptr;
  auto fetch_slots = [&](int k0) {
    const int ul = u0 + (k0 + lane) * ustride;
    if (ul < NU) {
      const int pi = ul / UPP;
      lane_slot = pv.slot_ptr(s, pi < nsel ? s_sel[pi] : w_extra[pi - nsel]);
    }
  };
  // warp-wide: lane 0 bulk-copies the page slot of the warp's k-th unit into buffer b
  auto stage_unit = [&](int k, int b) {
    if ((k & 31) == 0) fetch_slots(k);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(
        __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(lane_slot), k & 31));
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the warp's reads of b precede the copy
      mbar_arrive_expect_tx(sbar + b, kSlotUsed);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(sbuf + b * kSlotUsed)),
                   "l"(src), "r"(kSlotUsed), "r"(smem_u32(sbar + b))
                   : "memory");
    }
  };
  if constexpr (STAGE) {
    if (lane == 0) {
      mbar_init(sbar, 1);
      mbar_init(sbar + 1, 1);
      fence_barrier_init();
    }
    __syncwarp();
    if (u < NU) stage_unit(0, 0);
    if (u + ustride < NU) stage_unit(1, 1);
  } else if (u < NU) {
    pg_next = unit_page(u, um_next);
    slot_next = pv.slot_ptr(s, pg_next);  // round trip 2 (page table)
    if (16 * UT * (u % UPP) < min(P, n_tok - pg_next * P)) unit_load<T, KIND, D, P, UT>(slot_next, UT * (u % UPP), ud);
  }
  if (pdl && early_sel) asm volatile("griddepcontrol.wait;" ::: "memory");
  // ---- q and the new token: the previous kernel's outputs in a model --------
  const bool row_ok = r < G;
  uint32_t qw[D / 8];  // this lane's q values of row r (pairs, input dtype)
  {
    const T* qrow = reinterpret_cast<const T*>(prm.q) + s * prm.q_ss + (int64_t)(row_ok ? r : 0) * prm.q_rs;
#pragma unroll
    for (int ri = 0; ri < D / 8; ++ri) {
      const int d = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j;
      qw[ri] = row_ok ? __ldcg(reinterpret_cast<const uint32_t*>(qrow + d)) : 0u;
    }
  }
  // the new token's raw K and warp w's q row (w < G): loaded now, scored after
  // the units (engine.py:276-277 merges the new token last)
  T qs_self[D / 32], ks_self[D / 32];
  const T* vn = reinterpret_cast<const T*>(prm.v_new) + s * prm.new_ss;
  float v_own[(kMaxRows * D + kDecThreads - 1) / kDecThreads];  // v_new of this thread's output elements
#pragma unroll
  for (int k = 0; k < (kMaxRows * D + kDecThreads - 1) / kDecThreads; ++k) {  // element tid + k * kDecThreads
    const int i = tid + k * kDecThreads;
    v_own[k] = i < G * D ? DT<T>::to_f(__ldcg(vn + i % D)) : 0.f;
  }
  if (warp < G) {
    const T* qrow = reinterpret_cast<const T*>(prm.q) + s * prm.q_ss + (int64_t)warp * prm.q_rs;
    const T* kn = reinterpret_cast<const T*>(prm.k_new) + s * prm.new_ss;
#pragma unroll
    for (int i = 0; i < D / 32; ++i) {
      qs_self[i] = __ldcg(qrow + lane + 32 * i);
      ks_self[i] = __ldcg(kn + lane + 32 * i);
    }
  }
  bool first = true;
  if constexpr (STAGE) {
    for (int it = 0; u < NU; u += ustride, ++it) {
      uint32_t um;
      const int pg = unit_page(u, um), b = it & 1;
      const int tok_in_page = min(P, n_tok - pg * P);
      mbar_wait(sbar + b, (it >> 1) & 1);
      unit_load<T, KIND, D, P, UT, true>(sbuf + b * kSlotUsed, 0, ud);
      unit_compute<T, KIND, D, P, UT>(ud, 0, tok_in_page, um & gmask, qw, sl2, inv_levels, st);
      if (u + 2 * ustride < NU) {
        __syncwarp();
        stage_unit(it + 2, b);
      }
    }
  }
  for (; !STAGE && u < NU; u += ustride) {
    const int pg = pg_next;
    const uint32_t um = um_next;
    const uint8_t* slot = slot_next;
    const int un = u + ustride;
    if (un < NU) {  // next unit's table entry + its bytes into L2 while this one computes
      pg_next = unit_page(un, um_next);
      slot_next = pv.slot_ptr(s, pg_next);
      constexpr int kSlotUsed = (KIND == 0 ? 4 * P * D : (KIND == 1 ? P * D : 2 * P * D)) + (KIND == 0 ? 0 : 8 * D);
      for (int off = lane * 128; off < kSlotUsed; off += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(slot_next + off));
    }
    const int tok_in_page = min(P, n_tok - pg * P), tt0 = UT * (u % UPP);
    if (16 * tt0 < tok_in_page) {  // a unit past the open page's last token holds nothing
      if (!first) unit_load<T, KIND, D, P, UT>(slot, tt0, ud);
      WSTAMP(0);
      unit_compute<T, KIND, D, P, UT>(ud, tt0, tok_in_page, um & gmask, qw, sl2, inv_levels, st);
      WSTAMP(1);
    }
    first = false;
  }
  if (warp < G) {
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < D / 32; ++i) dot = fmaf(DT<T>::to_f(qs_self[i]), DT<T>::to_f(ks_self[i]), dot);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
    if (lane == 0) s_self[warp] = dot * prm.scale_log2;
  }
  DSTAMP(2);
  if (SK_DEC_ABLATE == 4) return;

  // ---- merge the CTA's warps ---------------------------------------------------
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    float lt = st.l[e];
    lt += __shfl_xor_sync(0xffffffffu, lt, 4);
    lt += __shfl_xor_sync(0xffffffffu, lt, 8);
    lt += __shfl_xor_sync(0xffffffffu, lt, 16);
    if (g == 0) {
      s_m[warp][2 * j + e] = st.m[e];
      s_l[warp][2 * j + e] = lt;
    }
  }
#pragma unroll
  for (int ct = 0; ct < D / 16; ++ct)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e) s_o[warp][2 * j + e][16 * ct + 8 * h + g] = st.o[ct][2 * h + e];
  __syncthreads();
  DSTAMP(3);
  // every thread merges the warps for its own output elements (no serial
  // per-row step, one barrier): M = max_w m_w, O = sum_w 2^(m_w - M) O_w
  const int64_t PF = part_floats(G, D);
  float* mine = prm.part + ((int64_t)s * prm.cps + blockIdx.x) * PF;
  constexpr int kEl = (kMaxRows * D + kDecThreads - 1) / kDecThreads;  // output elements per thread
#pragma unroll
  for (int k = 0; k < kEl; ++k) {
    const int i = tid + k * kDecThreads;
    if (i >= G * D) break;
    const int rr = i / D, c = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, s_m[w][rr]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float f = M == -INFINITY ? 0.f : fast_exp2(s_m[w][rr] - M);
      L = fmaf(f, s_l[w][rr], L);
      O = fmaf(f, s_o[w][rr][c], O);
    }
    if (prm.cps == 1) {  // the CTA holds the whole stream: finish with the new token
      const float s_new = s_self[rr], Mt = fmaxf(M, s_new);
      const float f = M == -INFINITY ? 0.f : fast_exp2(M - Mt), fs = fast_exp2(s_new - Mt);
      finish_out<T>(prm, s, rr, c, Mt, fmaf(f, L, fs), fmaf(f, O, fs * v_own[k]));
    } else {
      mine[2 * G + i] = O;
      if (c == 0) {
        mine[rr] = M;
        mine[G + rr] = L;
      }
    }
  }
  if (prm.cps == 1) {
    DSTAMP(6);
    return;
  }
  if (SK_DEC_ABLATE == 2) return;
  // ---- partial -> workspace; the stream's last CTA merges them -----------------
  __syncthreads();
  if (tid == 0) {  // bar.sync + a gpu-scope acq_rel RMW: releases this partial, acquires the others
    uint32_t t;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(prm.ticket + s) : "memory");
    s_last = (t == (uint32_t)prm.cps - 1);
    if (s_last) {
      prm.ticket[s] = 0;  // re-arm for the next launch
      // every partial of the stream (contiguous) -> shared memory, one bulk copy
      // (generic-proxy writes of the other CTAs, acquired above, read by the async proxy)
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const uint32_t bytes = (uint32_t)(prm.cps * PF * 4);
      mbar_init(&s_bar, 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(&s_bar, bytes);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(s_part)),
                   "l"(prm.part + (int64_t)s * prm.cps * PF), "r"(bytes), "r"(smem_u32(&s_bar))
                   : "memory");
    }
  }
  __syncthreads();
  DSTAMP(4);
  if (!s_last) return;
  mbar_wait(&s_bar, 0);
  DSTAMP(5);
  if (SK_DEC_ABLATE == 3) return;
  // per-(row, partial) merge factors 2^(m_b - M) once -- warp rr, lane b (the new
  // token's at b = cps) -- and the reciprocal of each row's normaliser L
  const int cps = prm.cps;
  float* s_f = &s_o[0][0][0];  // [G][cps + 1] (s_o is free now)
  float* s_rl = s_f + G * (kMaxCps + 1);
  if (warp < G) {
    const int rr = warp;
    const float s_new = s_self[rr];
    const float pm = lane < cps ? s_part[lane * PF + rr] : (lane == cps ? s_new : -INFINITY);
    float M = pm;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    const float f = pm == -INFINITY ? 0.f : fast_exp2(pm - M);
    float L = lane < cps ? f * s_part[lane * PF + G + rr] : (lane == cps ? f : 0.f);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
    if (lane <= cps) s_f[rr * (kMaxCps + 1) + lane] = f;
    if (lane == 0) s_rl[rr] = 1.f / L;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kEl; ++k) {
    const int i = tid + k * kDecThreads;
    if (i >= G * D) break;
    const int rr = i / D, c = i % D;
    const float* f = s_f + rr * (kMaxCps + 1);
    float O[4] = {f[cps] * v_own[k], 0.f, 0.f, 0.f};  // four independent chains
#pragma unroll
    for (int b = 0; b < kMaxCps; ++b)
      if (b < cps) O[b & 3] = fmaf(f[b], s_part[b * PF + 2 * G + i], O[b & 3]);
    finish_out<T>(prm, s, rr, c, 0.f, 1.f / s_rl[rr], (O[0] + O[1]) + (O[2] + O[3]));
  }
  DSTAMP(6);
}

template <typename T, int KIND, int D, int P, int UT, bool STAGE = false>
int launch_ut(const DecodeParams& prm, int n_streams, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(prm.cps, n_streams, 1);
  cfg.blockDim = dim3(kDecThreads, 1, 1);
  cfg.dynamicSmemBytes = STAGE ? (size_t)2 * kWarps * slot_used_bytes<KIND, D, P>()
                               : (prm.cps > 1 ? (size_t)prm.cps * part_floats(prm.G, D) * 4 : 0);
  if (cfg.dynamicSmemBytes > 0)  // static + dynamic exceeds the 48 KB default
    cudaFuncSetAttribute(decode_kernel<T, KIND, D, P, UT, STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)cfg.dynamicSmemBytes);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (prm.flags & SK_LAUNCH_PDL) ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, decode_kernel<T, KIND, D, P, UT, STAGE>, prm);
  if (e != cudaSuccess) {
    set_error(std::string("decode_kernel: ") + cudaGetErrorString(e));
    return SK_ECUDA;
  }
  SK_CHECK_LAUNCH("decode_kernel");
  return SK_OK;
}

// Unit size: 32 tokens when a stream's units are spread over several CTAs
// (latency); whole 64-token pages when one CTA holds the stream (many units
// per warp: the per-unit bounds, q' and sum setup is paid once per page).
template <typename T, int KIND, int D, int P>
int launch_one(const DecodeParams& prm, int n_streams, cudaStream_t st) {
  constexpr int UT_BIG = (P >= 64 && KIND == 1) ? 4 : 2;  // raw / byte codes: registers only fit 2 tiles
  if (prm.cps == 1 && UT_BIG != 2) {
    if constexpr (SK_DEC_STAGE && stage_fits<KIND, D, P, UT_BIG>())
      return launch_ut<T, KIND, D, P, UT_BIG, true>(prm, n_streams, st);
    return launch_ut<T, KIND, D, P, UT_BIG>(prm, n_streams, st);
  }
  return launch_ut<T, KIND, D, P, 2>(prm, n_streams, st);
}

template <typename T, int KIND>
int launch_kind(const DecodeParams& prm, int n_streams, cudaStream_t st) {
  const int D = prm.pv.D, P = prm.pv.P;
#define SK_DEC(DD, PP) if (D == DD && P == PP) return launch_one<T, KIND, DD, PP>(prm, n_streams, st)
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

extern "C" int64_t sk_decode_workspace(int32_t n_streams, int32_t group_rows, int32_t head_dim) {
  using namespace sk;
  if (n_streams < 1 || group_rows < 1 || head_dim < 1) return 0;
  // n x decode_cps(n) <= max(SMs, n): one buffer also serves launches over a subset of the streams
  const int64_t parts = (int64_t)(device_sm_count() > n_streams ? device_sm_count() : n_streams) + kMaxCps;
  return ticket_bytes(n_streams) + parts * part_floats(group_rows, head_dim) * 4;
}

extern "C" int sk_decode_attn(const sk_pool* pool, int32_t n_streams, int32_t group_rows, const void* q,
                              int64_t q_stream_stride, int64_t q_row_stride, const void* k_new, const void* v_new,
                              int64_t new_stream_stride, const uint32_t* row_mask, const uint32_t* row_window,
                              const int32_t* sel, const int32_t* sel_count, int32_t sel_stride, int32_t* tokens,
                              float softmax_scale, void* out, int64_t out_stream_stride, int64_t out_row_stride,
                              int32_t out_dtype, uint32_t flags, void* workspace, int64_t workspace_bytes,
                              void* stream) {
  using namespace sk;
  int rc = check_pool(pool);
  if (rc) return rc;
  SK_CHECK_ARG(n_streams >= 1 && n_streams <= 65535, "decode: stream count must be in [1, 65535]");
  SK_CHECK_ARG(group_rows >= 1 && group_rows <= kMaxRows, "decode: group size must be in [1, 8]");
  SK_CHECK_ARG(sel_stride >= 1 && sel_stride <= kMaxSel, "decode: selection width must be in [1, 2048]");
  SK_CHECK_ARG(pool->sink + pool->local <= kMaxExtra, "decode: sink + local window too large");
  SK_CHECK_ARG(out_dtype == SK_F16 || out_dtype == SK_BF16 || out_dtype == SK_F32, "decode: bad out dtype");
  SK_CHECK_ARG(q && k_new && v_new && row_mask && sel && sel_count && tokens && out, "decode: NULL pointer");
  SK_CHECK_ARG(q_row_stride % 2 == 0 && q_stream_stride % 2 == 0, "decode: q strides must be even");
  SK_CHECK_ARG(reinterpret_cast<uintptr_t>(pool->arena) % 16 == 0 && pool->slot_bytes % 16 == 0,
               "decode: arena slots must be 16-byte aligned");
  SK_CHECK_ARG(pool->page_size % kUnitTok == 0, "decode: page size must be a multiple of 32");
  SK_CHECK_ARG(workspace != nullptr &&
                   workspace_bytes >= sk_decode_workspace(n_streams, group_rows, pool->head_dim),
               "decode: workspace missing or smaller than sk_decode_workspace()");
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
  prm.row_window = row_window;
  prm.sel = sel;
  prm.sel_count = sel_count;
  prm.sel_stride = sel_stride;
  prm.tokens = tokens;
  prm.scale_log2 = softmax_scale * 1.4426950408889634f;
  prm.out = out;
  prm.out_ss = out_stream_stride;
  prm.out_rs = out_row_stride;
  prm.out_dtype = out_dtype;
  prm.flags = flags;
  // units: at most the selection width (+ the window) pages of P / 32 units each
  prm.cps = decode_cps(n_streams, (sel_stride + pool->sink + pool->local) * (pool->page_size / kUnitTok));
  prm.ticket = static_cast<uint32_t*>(workspace);
  prm.part = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + ticket_bytes(n_streams));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int kind = pool->bits == 0 ? 0 : (pool->bits <= 4 ? 1 : 2);
  int rc2;
  if (pool->dtype == SK_F16) {
    rc2 = kind == 0 ? launch_kind<__half, 0>(prm, n_streams, st)
                    : (kind == 1 ? launch_kind<__half, 1>(prm, n_streams, st) : launch_kind<__half, 2>(prm, n_streams, st));
  } else {
    rc2 = kind == 0 ? launch_kind<__nv_bfloat16, 0>(prm, n_streams, st)
                    : (kind == 1 ? launch_kind<__nv_bfloat16, 1>(prm, n_streams, st)
                                 : launch_kind<__nv_bfloat16, 2>(prm, n_streams, st));
  }
  if (rc2 != SK_OK || !(flags & SK_DECODE_APPEND)) return rc2;
  // the new token is appended by K1's one-token kernel right behind the
  // attention (stream order: every read of its page has completed)
  return append_launch(pool, n_streams, k_new, v_new, new_stream_stride, 0, tokens, 1, 1, st);
}

#ifdef SK_DEC_TIMING
extern "C" int sk_debug_decode_stamps(uint64_t* host_out) {  // 4096 x 8 u64
  return cudaMemcpyFromSymbol(host_out, sk::g_dec_stamps, sizeof(sk::g_dec_stamps)) == cudaSuccess ? 0 : 1;
}
extern "C" int sk_debug_decode_stamps_clear() {
  static uint64_t zero[4096][8];
  return cudaMemcpyToSymbol(sk::g_dec_stamps, zero, sizeof(zero)) == cudaSuccess ? 0 : 1;
}
#endif
