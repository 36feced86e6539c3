// K4 -- block-sparse causal prefill attention, tcgen05 + TMEM + TMA (sm_100a).
//
// Replaces blockwise_attention (reference attn.py:245-324) as driven by
// Engine.prefill (engine.py:152-168): every (head, 64-row query tile) visits
// only its scheduled 64-key tiles -- range(diag+1) for retrieval heads, the
// sink + local Lambda window for streaming heads -- with the element-wise
// causal mask on tiles that cross the diagonal (attn.py:315-319) and an
// online softmax over the visited tiles (attn.py:191-229).
//
// One CTA = one 256-row query block of one head: two 128-row tcgen05 tiles
// (four reference query tiles; per-64-row "quarter" flags on every segment
// keep their schedules distinct) that share one K/V stream.  Warp roles:
//   warp 0      TMA producer: both Q tiles once, then K/V 64-key blocks into
//               a kNS-stage ring (SWIZZLE_128B, mbarrier complete_tx)
//   warp 1      MMA issuer (one elected thread), per key block j:
//                 S_t,j = Q_t K_j^T   (M=128, N=64, K=D) for t = 0, 1 into
//                 double-buffered TMEM, then O_t += P_t,j-1 V_j-1 (M=128,
//                 N=D, K=64; V is an MN-major operand), so the tensor core
//                 always has the other tile's work while one tile's softmax
//                 runs (FA4-style ping-pong)
//   warps 2..5  softmax of tile 0, warps 6..9 softmax of tile 1: one thread
//               per query row reads S from TMEM (tcgen05.ld 32x32b), masks
//               only blocks that need it, exp2 with the scale folded into
//               one FFMA2 per pair, writes P (fp16/bf16) into a swizzled
//               K-major smem tile; O is rescaled in TMEM only when the
//               running max grows by more than 2^8 (exact: the stale max is a
//               shared reference point)
// TMEM: S[tile][buf] at columns tile*128 + buf*64, O[tile] at 256 + tile*128.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>

#include "sk_common.cuh"
#include "sk_layout.cuh"
#include "sk_sm100.cuh"

namespace sk {
namespace {

#ifndef SK_TMEM_P
#define SK_TMEM_P 1
#endif
constexpr bool kTmemP = SK_TMEM_P;   // P stored over its S columns in TMEM (A operand of PV)
constexpr int kNS = kTmemP ? 5 : 3;  // K/V pipeline stages (the smem P tiles make room for two more)
constexpr int kPfThreads = 320;    // 10 warps
constexpr int kItemRows = 256;     // two 128-row tiles
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr uint32_t kFlagCausal = 1u << 4, kFlagMasks = 1u << 5;
#ifndef SK_POLY_FROM
#define SK_POLY_FROM 64  // elements [SK_POLY_FROM, 64) of a row use exp2_poly2 (64 = off)
#endif
constexpr int kPolyFrom = SK_POLY_FROM;

// K/V stages when K/V are dequantised from the page pool (PAGED): one
// fewer, the room holds the producer's page-bounds tables
constexpr int kNSPaged = 4;

template <int D, int NS = kNS, bool PAGED = false>
struct PfSmem {
  static constexpr int NC = D / 64;  // 128-byte column chunks
  alignas(1024) uint8_t q[2][NC][128 * 128];
  alignas(1024) uint8_t kv[NS][2][NC][64 * 128];
  alignas(kTmemP ? 16 : 1024) uint8_t p[kTmemP ? 1 : 2][kTmemP ? 1 : 2][kTmemP ? 16 : 128 * 128];
  alignas(16) uint8_t bnd[PAGED ? 4 : 1][PAGED ? 4 * D * 2 : 16];  // raw page bounds / (scale, lo) tables
  // PAGED, 64-token pages: bulk-copied KV4 page slots, two blocks ahead of the dequantiser
  alignas(128) uint8_t stage[PAGED ? 3 : 1][PAGED ? 64 * D + 8 * D : 16];
  uint64_t stage_full[PAGED ? 3 : 1];
  uint64_t q_full;
  uint64_t kv_full[NS];
  uint64_t kv_empty[NS];
  uint64_t s_full[2][2];
  uint64_t p_full[2][2];
  uint64_t p_empty[2][2];
  uint64_t o_done[2];
  uint32_t tmem_base;
};

struct PfParams {
  void* out;
  int n_q, n_kv, n_heads, n_kv_heads, group;
  float scale_log2;
  const sk_prefill_item* items;
  const uint32_t* segs;
  const uint64_t* row_masks;
  // PAGED (chunked prefill over the page pool): keys [0, hist) are the pool's
  // KV4 pages (stream = KV head), keys [hist, n_kv) the chunk's raw k / v
  // [n_kv - hist][n_kv_heads][D]
  PoolView pv;
  int hist;
  const void* kc;
  const void* vc;
};

// Walks an item's segments block by block.
struct SegWalk {
  const uint32_t* segs;
  int seg, seg_end, i;
  uint32_t first, count, flags, mask_base;
  __device__ SegWalk(const uint32_t* s, int b, int n) : segs(s), seg(b), seg_end(b + n), i(0) { load(); }
  __device__ void load() {
    if (seg < seg_end) {
      first = segs[3 * seg];
      uint32_t w = segs[3 * seg + 1];
      count = w & 0xFFFFFFu;
      flags = w >> 24;
      mask_base = segs[3 * seg + 2];
    } else {
      count = 0;
    }
  }
  __device__ bool done() const { return seg >= seg_end; }
  __device__ int block() const { return int(first) + i; }
  __device__ void next() {
    if (++i >= int(count)) {
      i = 0;
      ++seg;
      load();
    }
  }
};

// packed fp32x2 helpers (FFMA2 / FADD2 on sm_100)
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(uint64_t r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^x for a pair, x <= ~8, on the FMA pipe: Cody-Waite split x = n + f with
// the 1.5*2^23 rounding trick (n lands in the low mantissa bits), a degree-3
// minimax polynomial for 2^f on [-1/2, 1/2] (max relative error 7.5e-5, below
// half an fp16 ulp of P), and n added straight into the exponent field.
__device__ __forceinline__ float2 exp2_poly2(uint64_t x2) {
  float2 x = f2_unpack(x2);
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const uint64_t xc = f2_pack(x.x, x.y);
  const uint64_t magic = f2_pack(12582912.f, 12582912.f);
  const uint64_t j = f2_add(xc, magic);
  const uint64_t n = f2_add(j, f2_pack(-12582912.f, -12582912.f));
  const uint64_t f = f2_fma(n, f2_pack(-1.f, -1.f), xc);
  uint64_t p = f2_fma(f2_pack(0.055171654f, 0.055171654f), f, f2_pack(0.24261115f, 0.24261115f));
  p = f2_fma(p, f, f2_pack(0.69326097f, 0.69326097f));
  p = f2_fma(p, f, f2_pack(0.99992806f, 0.99992806f));
  const float2 pv = f2_unpack(p), jv = f2_unpack(j);
  return make_float2(__int_as_float(__float_as_int(pv.x) + (__float_as_int(jv.x) << 23)),
                     __int_as_float(__float_as_int(pv.y) + (__float_as_int(jv.y) << 23)));
}

// A operand in TMEM (P), B in shared memory (V): D[tmem] (+)= A[tmem] * B
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// A 4-bit code as an exact float without I2F (a conversion would share the
// XU pipe with the softmax's MUFU.EX2): 2^23 + n, less 2^23.
__device__ __forceinline__ float nib_f(uint32_t w, int shift) {
  return __uint_as_float(0x4B000000u | ((w >> shift) & 0xFu)) - 8388608.f;
}
// The two codes at bits [shift, +4) and [shift + 16, +4) of w, dequantised as
// a pair with packed fp32 ops: PRMT builds 2^23 + n for both, one FADD2
// removes 2^23 (exact), one FFMA2 applies (scale, lo) -- the same single
// fp32 fma per value as K1b -- and the pair is rounded to T.
template <typename T>
__device__ __forceinline__ uint32_t nib_pair(uint32_t w, int shift, uint64_t sc2, uint64_t lo2) {
  const uint32_t x = (w >> shift) & 0x000F000Fu;
  const uint64_t f = f2_pack(__uint_as_float(__byte_perm(x, 0x4B000000u, 0x7540)),
                             __uint_as_float(__byte_perm(x, 0x4B000000u, 0x7542)));
  const float2 v = f2_unpack(f2_fma(f2_add(f, f2_pack(-8388608.f, -8388608.f)), sc2, lo2));
  return std::is_same<T, __nv_bfloat16>::value ? pack_bf162(v.x, v.y) : pack_half2(v.x, v.y);
}

// Producer warps 10-13 of the PAGED kernel: K/V block j of the item is built in
// the stage's smem tiles in the layouts the MMAs read -- K row-major
// [key][D] (SWIZZLE_128B, as TMA writes it), V K-major [D][64 keys] (its rows
// are the pool's channel-major code runs) -- from the KV4 pages (dequantised:
// code * scale + lo in fp32, rounded to T: the values PhysicalPage.dequantize
// casts to the attention dtype, identical to K1b and K3) or from the chunk's
// raw k / v; keys past n_kv are zero.  Thread i: K token i/2, dims
// [(i%2) D/2, +D/2); V channel i % D, keys [(i/D) 64D/128, +64D/128).
template <typename T, int D, int P, int NS>
__device__ __forceinline__ void paged_block(PfSmem<D, NS, true>& sm, const PfParams& prm, int kvh, int st, int key0,
                                            int tid) {
  constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
  constexpr int UPT = D / 16;                // K units (8 dims) per thread
  constexpr int VKEYS = D == 128 ? 64 : 32;  // V keys per thread
  constexpr int PPB = 64 / P;                // pages per block
  constexpr int BCH = 4 * D * 2 / 16;        // 16-byte chunks of one page's bounds
  constexpr int RW = P / 8;                  // words of a channel's code run in a page (4 lanes x P/32)
  const PoolView& pv = prm.pv;
  const int hist = prm.hist;
  const int page0 = key0 / P;
  // ---- issue every load first: bounds -> smem, K codes / raw row and the
  //      channel's V code runs -> registers
  for (int x = tid; x < PPB * BCH; x += 128) {
    const int pg = x / BCH;
    if ((page0 + pg) * P < hist) {
      const uint8_t* bsrc = pv.bounds(pv.slot_ptr(kvh, page0 + pg));
      *reinterpret_cast<uint4*>(&sm.bnd[pg][(x % BCH) * 16]) = *reinterpret_cast<const uint4*>(bsrc + (x % BCH) * 16);
    }
  }
  const int t = tid >> 1, hd = tid & 1, kpos = key0 + t;
  uint32_t kwv[4][UPT / 4];
  uint4 kraw[UPT];
  if (kpos < hist) {
    const uint8_t* kc = pv.slot_ptr(kvh, kpos / P) + (kpos % P) * (D / 2);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int w = 0; w < UPT / 4; ++w)
        kwv[j][w] = *reinterpret_cast<const uint32_t*>(kc + j * (D / 8) + (hd * (UPT / 4) + w) * 4);
  } else if (kpos < prm.n_kv) {
    const T* src = reinterpret_cast<const T*>(prm.kc) + ((int64_t)(kpos - hist) * prm.n_kv_heads + kvh) * D + hd * (D / 2);
#pragma unroll
    for (int u = 0; u < UPT; ++u) kraw[u] = *reinterpret_cast<const uint4*>(src + 8 * u);
  }
  const int c = tid % D, kh = tid / D, kb0 = key0 + kh * VKEYS;
  uint32_t vrun[PPB][RW];
#pragma unroll
  for (int pg = 0; pg < PPB; ++pg) {
    if ((page0 + pg) * P < hist) {
      const uint8_t* run = pv.v_codes(pv.slot_ptr(kvh, page0 + pg)) + (32 * (c / 8) + 4 * (c % 8)) * (P / 8);
#pragma unroll
      for (int q = 0; q < RW / 4; ++q) {
        const uint4 v4 = *reinterpret_cast<const uint4*>(run + 16 * q);
        vrun[pg][4 * q] = v4.x; vrun[pg][4 * q + 1] = v4.y; vrun[pg][4 * q + 2] = v4.z; vrun[pg][4 * q + 3] = v4.w;
      }
    }
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");  // bounds staged
  // ---- K: dequantise (or copy) the thread's 8-dim units into the swizzled row
  uint8_t* kt = &sm.kv[st][0][0][0];
  const int kpg = kpos / P - page0;
#pragma unroll
  for (int u = 0; u < UPT; ++u) {
    const int m = hd * UPT + u;  // 8-dim unit of the row
    uint4 outv = make_uint4(0u, 0u, 0u, 0u);
    if (kpos < hist) {
      const T* bt = reinterpret_cast<const T*>(&sm.bnd[kpg][0]);
      uint32_t pk[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t wd = kwv[j][u / 4];
        const int bp = j * (D / 4) + 2 * m;  // kbound_pos of dims 8m+2j, 8m+2j+1
        float x2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float lo = DT<T>::to_f(bt[bp + e]), hi = DT<T>::to_f(bt[D + bp + e]);
          float sc = (hi - lo) / 15.f;
          sc = sc > 0.f ? sc : 1.f;
          x2[e] = fmaf(nib_f(wd, 4 * (m % 4) + 16 * e), sc, lo);
        }
        pk[j] = kBF16 ? pack_bf162(x2[0], x2[1]) : pack_half2(x2[0], x2[1]);
      }
      outv = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    } else if (kpos < prm.n_kv) {
      outv = kraw[u];
    }
    const int d0 = 8 * m, chk = d0 / 64, un = (d0 % 64) / 8;
    *reinterpret_cast<uint4*>(kt + chk * (64 * 128) + t * 128 + ((un ^ (t & 7)) << 4)) = outv;
  }
  // ---- V: the channel's keys, K-major row c (64 keys x 2 B, swizzled 16 B units)
  uint8_t* vr = &sm.kv[st][1][0][0] + c * 128;
  const int vbp = ((c % 8) / 2) * (D / 4) + (c / 8) * 2 + (c % 2);  // vbound_pos(c)
#pragma unroll
  for (int q8 = 0; q8 < VKEYS / 8; ++q8) {
    uint32_t pk[4];
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      float x2[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = kb0 + 8 * q8 + 2 * e2 + e;
        float val = 0.f;
        if (key < hist) {
          const int pg = key / P - page0, tin = key % P;
          const T* bt = reinterpret_cast<const T*>(&sm.bnd[pg][0]);
          const float lo = DT<T>::to_f(bt[2 * D + vbp]), hi = DT<T>::to_f(bt[3 * D + vbp]);
          float sc = (hi - lo) / 15.f;
          sc = sc > 0.f ? sc : 1.f;
          const uint32_t wd = vrun[pg][((tin % 8) / 2) * (P / 32) + tin / 32];
          val = fmaf(nib_f(wd, 4 * ((tin / 8) % 4) + 16 * (tin % 2)), sc, lo);
        } else if (key < prm.n_kv) {
          val = DT<T>::to_f(reinterpret_cast<const T*>(prm.vc)[((int64_t)(key - hist) * prm.n_kv_heads + kvh) * D + c]);
        }
        x2[e] = val;
      }
      pk[e2] = kBF16 ? pack_bf162(x2[0], x2[1]) : pack_half2(x2[0], x2[1]);
    }
    const int un = (kh * VKEYS) / 8 + q8;
    *reinterpret_cast<uint4*>(vr + ((un ^ (c & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
  fence_proxy_async_smem();  // generic-proxy smem writes -> the tensor core's async proxy
  asm volatile("bar.sync 1, 128;" ::: "memory");  // every thread's tile writes (and bounds reads) done
}

// Fast path of the paged producer for blocks lying wholly in the history:
// the loads of block j+1 (bound values of this thread's dim / channel, K codes,
// V code runs) are issued before block j is dequantised; per-page (scale, lo)
// tables in smem are formed once per block (one fp32 division per dim, the
// formula of K1b), so a code costs an extract, a conversion and an FMA.
template <typename T, int D, int P>
struct PagedRegs {
  static constexpr int UPT = D / 16, RW = P / 8, PPB = 64 / P;
  uint32_t kw[4][UPT / 4];   // K codes of the thread's token, its dim half
  uint32_t vrun[PPB][RW];    // V code runs of the thread's channel
  uint32_t kb[PPB][2];       // K lo / hi (raw T bits) of dim tid (D = 128) or tid % D
  uint32_t vb[PPB][2];       // V lo / hi of channel tid % D
};
template <typename T, int D, int P>
__device__ __forceinline__ void paged_prefetch(const PfParams& prm, int kvh, int key0, int tid, PagedRegs<T, D, P>& r) {
  using R = PagedRegs<T, D, P>;
  const PoolView& pv = prm.pv;
  const int page0 = key0 / P;
  const int t = tid >> 1, hd = tid & 1, kpos = key0 + t;
  const uint8_t* kc = pv.slot_ptr(kvh, kpos / P) + (kpos % P) * (D / 2);
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int w = 0; w < R::UPT / 4; ++w)
      r.kw[j][w] = __ldg(reinterpret_cast<const uint32_t*>(kc + j * (D / 8) + (hd * (R::UPT / 4) + w) * 4));
  const int c = tid % D;
  const int kbp = kbound_pos(c, D), vbp = vbound_pos(c, D);
#pragma unroll
  for (int pg = 0; pg < R::PPB; ++pg) {
    const uint8_t* slot = pv.slot_ptr(kvh, page0 + pg);
    const uint8_t* run = pv.v_codes(const_cast<uint8_t*>(slot)) + (32 * (c / 8) + 4 * (c % 8)) * (P / 8);
#pragma unroll
    for (int q = 0; q < R::RW / 4; ++q) {
      const uint4 v4 = __ldg(reinterpret_cast<const uint4*>(run + 16 * q));
      r.vrun[pg][4 * q] = v4.x; r.vrun[pg][4 * q + 1] = v4.y; r.vrun[pg][4 * q + 2] = v4.z; r.vrun[pg][4 * q + 3] = v4.w;
    }
    const uint16_t* b = reinterpret_cast<const uint16_t*>(pv.bounds(const_cast<uint8_t*>(slot)));
    r.kb[pg][0] = __ldg(b + kbp);
    r.kb[pg][1] = __ldg(b + D + kbp);
    r.vb[pg][0] = __ldg(b + 2 * D + vbp);
    r.vb[pg][1] = __ldg(b + 3 * D + vbp);
  }
}
template <typename T>
__device__ __forceinline__ float2 scale_lo(uint32_t lo_bits, uint32_t hi_bits) {  // K1b's (scale, lo)
  const uint16_t l16 = (uint16_t)lo_bits, h16 = (uint16_t)hi_bits;
  const float lo = DT<T>::to_f(*reinterpret_cast<const T*>(&l16)), hi = DT<T>::to_f(*reinterpret_cast<const T*>(&h16));
  const float sc = (hi - lo) / 15.f;
  return make_float2(sc > 0.f ? sc : 1.f, lo);
}
template <typename T, int D, int P, int NS>
__device__ __forceinline__ void paged_fast(PfSmem<D, NS, true>& sm, int st, int tid, const PagedRegs<T, D, P>& r,
                                           const float2* ktab /* [PPB][D] (scale, lo) */) {
  using R = PagedRegs<T, D, P>;
  constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
  constexpr int VKEYS = D == 128 ? 64 : 32;
  const int t = tid >> 1, hd = tid & 1;
  const int kpg = t / P;
  uint8_t* kt = &sm.kv[st][0][0][0];
#pragma unroll
  for (int u = 0; u < R::UPT; ++u) {
    const int m = hd * R::UPT + u;
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t wd = r.kw[j][u / 4];
      const float4 sl = *reinterpret_cast<const float4*>(&ktab[kpg * D + 8 * m + 2 * j]);  // dims 8m+2j, +1
      const float x0 = fmaf(nib_f(wd, 4 * (u % 4)), sl.x, sl.y);  // m % 4 == u % 4
      const float x1 = fmaf(nib_f(wd, 4 * (u % 4) + 16), sl.z, sl.w);
      pk[j] = kBF16 ? pack_bf162(x0, x1) : pack_half2(x0, x1);
    }
    const int d0 = 8 * m, chk = d0 / 64, un = (d0 % 64) / 8;
    *reinterpret_cast<uint4*>(kt + chk * (64 * 128) + t * 128 + ((un ^ (t & 7)) << 4)) =
        make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
  const int c = tid % D, kh = tid / D;
  uint8_t* vr = &sm.kv[st][1][0][0] + c * 128;
  float2 vsl[R::PPB];
#pragma unroll
  for (int pg = 0; pg < R::PPB; ++pg) vsl[pg] = scale_lo<T>(r.vb[pg][0], r.vb[pg][1]);
#pragma unroll
  for (int q8 = 0; q8 < VKEYS / 8; ++q8) {
    uint32_t pk[4];
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      float x2[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int kr = 8 * q8 + 2 * e2 + e;  // key within the thread's VKEYS (compile-time)
        // D = 128: kh == 0 and every index below is a compile-time register index;
        // D = 64: kh selects the page (P = 32) or the word (P = 64)
        const int kb = (D == 128 ? 0 : VKEYS) + kr;
        const int pg1 = kb / P, tin1 = kb % P, pg0 = kr / P, tin0 = kr % P;
        const uint32_t w0 = r.vrun[pg0][((tin0 % 8) / 2) * (P / 32) + tin0 / 32];
        const uint32_t w1 = r.vrun[pg1][((tin1 % 8) / 2) * (P / 32) + tin1 / 32];
        const bool hi = D != 128 && kh == 1;
        const uint32_t wd = hi ? w1 : w0;
        const int tin = hi ? tin1 : tin0;
        const float2 sl = hi ? vsl[pg1] : vsl[pg0];
        x2[e] = fmaf(nib_f(wd, 4 * ((tin / 8) % 4) + 16 * (tin % 2)), sl.x, sl.y);
      }
      pk[e2] = kBF16 ? pack_bf162(x2[0], x2[1]) : pack_half2(x2[0], x2[1]);
    }
    const int un = (kh * VKEYS) / 8 + q8;
    *reinterpret_cast<uint4*>(vr + ((un ^ (c & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
}

// Fast path for 64-token pages: the block's page slot (codes + bounds, one
// contiguous 64 D + 8 D bytes) arrives by one 1-D bulk copy issued two blocks
// ahead; the dequantiser reads everything from shared memory.
template <typename T, int D, int NS>
__device__ __forceinline__ void paged_staged(PfSmem<D, NS, true>& sm, int st, int tid, const uint8_t* slot,
                                             float2* ktab) {
  constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
  constexpr int P = 64, UPT = D / 16, VKEYS = D == 128 ? 64 : 32;
  const uint16_t* b = reinterpret_cast<const uint16_t*>(slot + 2 * P * (D / 2));
  if (tid < D) ktab[tid] = scale_lo<T>(b[kbound_pos(tid, D)], b[D + kbound_pos(tid, D)]);
  const int c = tid % D, kh = tid / D;
  const float2 vsl = scale_lo<T>(b[2 * D + vbound_pos(c, D)], b[3 * D + vbound_pos(c, D)]);
  const int t = tid >> 1, hd = tid & 1;
  uint32_t kw[4][UPT / 4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int w = 0; w < UPT / 4; ++w)
      kw[j][w] = *reinterpret_cast<const uint32_t*>(slot + t * (D / 2) + j * (D / 8) + (hd * (UPT / 4) + w) * 4);
  uint32_t vrun[8];
  {
    const uint8_t* run = slot + P * (D / 2) + (32 * (c / 8) + 4 * (c % 8)) * (P / 8);
    const uint4 a = *reinterpret_cast<const uint4*>(run), bb = *reinterpret_cast<const uint4*>(run + 16);
    vrun[0] = a.x; vrun[1] = a.y; vrun[2] = a.z; vrun[3] = a.w; vrun[4] = bb.x; vrun[5] = bb.y; vrun[6] = bb.z; vrun[7] = bb.w;
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");  // K (scale, lo) table complete
  uint8_t* kt = &sm.kv[st][0][0][0];
#pragma unroll
  for (int u = 0; u < UPT; ++u) {
    const int m = hd * UPT + u;
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 sl = *reinterpret_cast<const float4*>(&ktab[8 * m + 2 * j]);  // dims 8m+2j, +1
      pk[j] = nib_pair<T>(kw[j][u / 4], 4 * (u % 4), f2_pack(sl.x, sl.z), f2_pack(sl.y, sl.w));  // m%4 == u%4
    }
    const int d0 = 8 * m, chk = d0 / 64, un = (d0 % 64) / 8;
    *reinterpret_cast<uint4*>(kt + chk * (64 * 128) + t * 128 + ((un ^ (t & 7)) << 4)) =
        make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
  uint8_t* vr = &sm.kv[st][1][0][0] + c * 128;
  const uint64_t vsc2 = f2_pack(vsl.x, vsl.x), vlo2 = f2_pack(vsl.y, vsl.y);
#pragma unroll
  for (int q8 = 0; q8 < VKEYS / 8; ++q8) {
    uint32_t pk[4];
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      // keys tin = kh*VKEYS + tr, tr + 1 of the page share word ((tin%8)/2)*2 + tin/32 -- a
      // register index fixed at compile time (kh only picks between two words when D = 64) --
      // at bit offsets 4((tin/8)%4) and +16
      const int tr = 8 * q8 + 2 * e2;
      const int wi = ((tr % 8) / 2) * 2 + (D == 128 ? tr / 32 : 0);
      const uint32_t wd = (D == 128 || kh == 0) ? vrun[wi] : vrun[wi + 1];
      pk[e2] = nib_pair<T>(wd, 4 * ((tr / 8) % 4), vsc2, vlo2);
    }
    const int un = (kh * VKEYS) / 8 + q8;
    *reinterpret_cast<uint4*>(vr + ((un ^ (c & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
}

// A block wholly inside the chunk: its raw K and V rows, copied 16 bytes at a
// time into the same row-major SWIZZLE_128B tiles TMA would write (the MMA
// reads this block's V as MN-major); keys past n_kv are zero.
template <typename T, int D, int NS>
__device__ __forceinline__ void chunk_rows(PfSmem<D, NS, true>& sm, const PfParams& prm, int kvh, int st, int key0,
                                           int tid) {
  constexpr int UPR = D / 8;  // 16-byte units per row
  for (int x = tid; x < 2 * 64 * UPR; x += 128) {
    const int which = x / (64 * UPR), t = (x / UPR) % 64, u = x % UPR;
    const int key = key0 + t;
    uint4 val = make_uint4(0u, 0u, 0u, 0u);
    if (key < prm.n_kv) {
      const T* src = reinterpret_cast<const T*>(which ? prm.vc : prm.kc) +
                     ((int64_t)(key - prm.hist) * prm.n_kv_heads + kvh) * D + 8 * u;
      val = *reinterpret_cast<const uint4*>(src);
    }
    const int chk = u / 8, un = u % 8;
    *reinterpret_cast<uint4*>(&sm.kv[st][which][chk][0] + t * 128 + ((un ^ (t & 7)) << 4)) = val;
  }
  fence_proxy_async_smem();
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

template <typename T, int D, bool PAGED = false, int PP = 64>
__global__ void __launch_bounds__(PAGED ? kPfThreads + 128 : kPfThreads, 1)
    prefill_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                   const __grid_constant__ CUtensorMap tv, const __grid_constant__ PfParams prm) {
  constexpr int NS = PAGED ? kNSPaged : kNS;
  using Sm = PfSmem<D, NS, PAGED>;
  constexpr int NC = Sm::NC;
  constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
  constexpr uint32_t kTmemCols = 512;
  constexpr uint32_t kOCol = 256;
  extern __shared__ uint8_t smem_raw[];
  Sm& sm = *reinterpret_cast<Sm*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const int warp = warp_id_uniform(), lane = threadIdx.x & 31;
  const sk_prefill_item item = prm.items[blockIdx.x];
  const int kvh = item.head / prm.group;
  int n_blocks = 0;
  for (int sgi = 0; sgi < item.seg_count; ++sgi) n_blocks += prm.segs[3 * (item.seg_begin + sgi) + 1] & 0xFFFFFFu;

  if (threadIdx.x == 0) {
    mbar_init(&sm.q_full, 1);
    if (PAGED)
      for (int i = 0; i < 3; ++i) mbar_init(&sm.stage_full[i], 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(&sm.s_full[t][b], 1);
        mbar_init(&sm.p_full[t][b], 4);
        mbar_init(&sm.p_empty[t][b], 1);
      }
      mbar_init(&sm.o_done[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (elect_one()) {
      tma_prefetch_desc(&tq);
      tma_prefetch_desc(&tk);
      tma_prefetch_desc(&tv);
      mbar_arrive_expect_tx(&sm.q_full, 2 * NC * 128 * 128);
      for (int t = 0; t < 2; ++t)
        for (int c = 0; c < NC; ++c) tma_load_3d(sm.q[t][c], &tq, &sm.q_full, 64 * c, item.head, item.row0 + 128 * t);
      int j = 0;
      for (SegWalk w(prm.segs, item.seg_begin, item.seg_count); !PAGED && !w.done(); w.next(), ++j) {
        const int st = j % NS;
        if (j >= NS) mbar_wait(&sm.kv_empty[st], ((j / NS) - 1) & 1);
        mbar_arrive_expect_tx(&sm.kv_full[st], 2 * NC * 64 * 128);
        const int key0 = w.block() * 64;
        for (int c = 0; c < NC; ++c) {
          tma_load_3d(sm.kv[st][0][c], &tk, &sm.kv_full[st], 64 * c, kvh, key0);
          tma_load_3d(sm.kv[st][1][c], &tv, &sm.kv_full[st], 64 * c, kvh, key0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------ MMA issuer --------------------------------
    constexpr uint32_t idesc_s = make_idesc_f16(128, 64, kBF16, false, false);
    constexpr uint32_t idesc_o = make_idesc_f16(128, D, kBF16, false, true);     // V MN-major (TMA)
    constexpr uint32_t idesc_o_km = make_idesc_f16(128, D, kBF16, false, false); // V K-major (paged producer)
    // PAGED: which stage holds a K-major V (a block built by the producer warps)
    uint32_t kmaj = 0;  // bit st: stage st holds a K-major V
    SegWalk mw(prm.segs, item.seg_begin, item.seg_count);
    mbar_wait(&sm.q_full, 0);
    tc_fence_after();
    auto issue_s = [&](int t, int jj) {  // S_t,jj = Q_t K_jj^T into TMEM buffer jj&1
      const int st = jj % NS;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          uint64_t a = make_sdesc_sw128(smem_u32(sm.q[t][kk / 4]) + (kk % 4) * 32, 16, 1024);
          uint64_t b = make_sdesc_sw128(smem_u32(sm.kv[st][0][kk / 4]) + (kk % 4) * 32, 16, 1024);
          mma_f16_ss(tmem + t * 128 + (jj & 1) * 64, a, b, idesc_s, kk > 0);
        }
        mma_commit(&sm.s_full[t][jj & 1]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int t, int jj) {  // O_t += P_t,jj V_jj
      const int st = jj % NS;
      mbar_wait(&sm.p_full[t][jj & 1], (jj >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          // V: MN-major [key][D] as TMA writes it, or K-major [D][key] from the paged producer
          const bool km = PAGED && ((kmaj >> st) & 1u);
          uint64_t b = km ? make_sdesc_sw128(smem_u32(sm.kv[st][1][0]) + kk * 32, 16, 1024)
                          : make_sdesc_sw128(smem_u32(sm.kv[st][1][0]) + kk * 2048, 64 * 128, 1024);
          if (kTmemP) {
            mma_f16_ts(tmem + kOCol + t * 128, tmem + t * 128 + (jj & 1) * 64 + kk * 8, b, km ? idesc_o_km : idesc_o,
                       (jj > 0 || kk > 0) ? 1u : 0u);
          } else {
            uint64_t a = make_sdesc_sw128(smem_u32(sm.p[kTmemP ? 0 : t][jj & 1]) + kk * 32, 16, 1024);
            mma_f16_ss(tmem + kOCol + t * 128, a, b, idesc_o, (jj > 0 || kk > 0) ? 1u : 0u);
          }
        }
        if (!kTmemP) mma_commit(&sm.p_empty[t][jj & 1]);  // P in TMEM: no smem P buffer to release
        mma_commit(&sm.o_done[t]);
        if (t == 1) mma_commit(&sm.kv_empty[st]);
      }
      __syncwarp();
    };
    auto wait_kv = [&](int jj) {  // blocks are waited in order: record block jj's V layout for its PV
      if (PAGED) {
        const uint32_t bit = 1u << (jj % NS);
        kmaj = (mw.block() * 64 < prm.hist) ? (kmaj | bit) : (kmaj & ~bit);
        mw.next();
      }
      mbar_wait(&sm.kv_full[jj % NS], (jj / NS) & 1);
      tc_fence_after();
    };
    // S_t,j reuses the TMEM buffer of S_t,j-2, whose softmax finished before
    // PV_t,j-2 could be issued -- and every order below issues PV_t,j-2 first.
#ifndef SK_PF_ORDER
#define SK_PF_ORDER 0
#endif
    if (SK_PF_ORDER == 0) {  // S_0,j S_1,j | PV_0,j-1 PV_1,j-1
      for (int j = 0; j < n_blocks; ++j) {
        wait_kv(j);
        issue_s(0, j);
        issue_s(1, j);
        if (j > 0) {
          issue_pv(0, j - 1);
          issue_pv(1, j - 1);
        }
      }
      if (n_blocks > 0) {
        issue_pv(0, n_blocks - 1);
        issue_pv(1, n_blocks - 1);
      }
    } else {  // S_0,j+1 | PV_0,j | S_1,j+1 | PV_1,j (tile softmaxes staggered)
      if (n_blocks > 0) {
        wait_kv(0);
        issue_s(0, 0);
        issue_s(1, 0);
      }
      for (int j = 0; j < n_blocks; ++j) {
        const bool more = j + 1 < n_blocks;
        if (more) {
          wait_kv(j + 1);
          issue_s(0, j + 1);
        }
        issue_pv(0, j);
        if (more) issue_s(1, j + 1);
        issue_pv(1, j);
      }
    }
  } else if (PAGED && warp >= 10) {
    // ------------------------- paged K/V producer (PAGED) -------------------------
    if constexpr (PAGED && PP == 64) {
      // 64-token pages: page j's slot is bulk-copied two blocks ahead (one
      // thread issues, page-table entry loaded one block before that)
      const int tid = threadIdx.x - 320;
      float2* ktab = reinterpret_cast<float2*>(&sm.bnd[0][0]);  // [2][D] (scale, lo) of K
      const uint32_t slot_bytes = 64 * D + 8 * D;
      auto whole = [&](int block) { return (block + 1) * 64 <= prm.hist; };
      SegWalk w(prm.segs, item.seg_begin, item.seg_count);
      SegWalk wi = w;  // issue cursor, two blocks ahead
      const uint8_t* nxt_slot = nullptr;
      auto issue = [&](int jj) {  // bulk copy of block jj (cursor wi) if it is a history block
        if (!wi.done() && whole(wi.block())) {
          mbar_arrive_expect_tx(&sm.stage_full[jj % 3], slot_bytes);
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_u32(sm.stage[jj % 3])),
                       "l"(prm.pv.slot_ptr(kvh, wi.block())), "r"(slot_bytes), "r"(smem_u32(&sm.stage_full[jj % 3]))
                       : "memory");
        }
        if (!wi.done()) wi.next();
      };
      if (tid == 0) {
        issue(0);
        issue(1);
      }
      for (int j = 0; !w.done(); ++j) {
        const int st = j % NS, block = w.block();
        if (tid == 0) issue(j + 2);  // the slot j + 2 - 3 = j - 1 was released by block j-1's last barrier
        if (j >= NS) mbar_wait(&sm.kv_empty[st], ((j / NS) - 1) & 1);
        if (block * 64 >= prm.hist) {  // wholly in the chunk: raw rows, row-major K and V
          chunk_rows<T, D, NS>(sm, prm, kvh, st, block * 64, tid);
          if (tid == 0) mbar_arrive(&sm.kv_full[st]);
          w.next();
          continue;
        }
#ifndef SK_PAGED_NOOP  // timing experiment only: 1 = the producer writes nothing
#define SK_PAGED_NOOP 0
#endif
        if (SK_PAGED_NOOP) {
          if (whole(block)) mbar_wait(&sm.stage_full[j % 3], (j / 3) & 1);
          asm volatile("bar.sync 1, 128;" ::: "memory");
        } else if (whole(block)) {
          mbar_wait(&sm.stage_full[j % 3], (j / 3) & 1);
          paged_staged<T, D, NS>(sm, st, tid, sm.stage[j % 3], ktab + (j & 1) * D);
          fence_proxy_async_smem();
          asm volatile("bar.sync 1, 128;" ::: "memory");
        } else {
          paged_block<T, D, PP, NS>(sm, prm, kvh, st, block * 64, tid);
        }
        if (tid == 0) mbar_arrive(&sm.kv_full[st]);
        w.next();
      }
      (void)nxt_slot;
    } else if constexpr (PAGED) {
      const int tid = threadIdx.x - 320;
      float2* ktab = reinterpret_cast<float2*>(&sm.bnd[0][0]);  // [2 buffers][PPB][D] (scale, lo) of K
      constexpr int PPB = 64 / PP;
      PagedRegs<T, D, PP> cur, nxt;
      SegWalk w(prm.segs, item.seg_begin, item.seg_count);
      auto whole = [&](int block) { return (block + 1) * 64 <= prm.hist; };
      if (!w.done() && whole(w.block())) paged_prefetch<T, D, PP>(prm, kvh, w.block() * 64, tid, cur);
      for (int j = 0; !w.done(); ++j) {
        const int st = j % NS, block = w.block();
        SegWalk wn = w;
        wn.next();
        if (block * 64 >= prm.hist) {  // wholly in the chunk: raw rows, row-major K and V
          if (j >= NS) mbar_wait(&sm.kv_empty[st], ((j / NS) - 1) & 1);
          chunk_rows<T, D, NS>(sm, prm, kvh, st, block * 64, tid);
          if (tid == 0) mbar_arrive(&sm.kv_full[st]);
          w = wn;
          continue;
        }
        if (whole(block)) {
          // K (scale, lo) of this block's page(s) -> table j&1 (dim tid % D)
          if (tid < D)
#pragma unroll
            for (int pg = 0; pg < PPB; ++pg)
              ktab[((j & 1) * PPB + pg) * D + tid] = scale_lo<T>(cur.kb[pg][0], cur.kb[pg][1]);
        }
        if (!wn.done() && whole(wn.block())) paged_prefetch<T, D, PP>(prm, kvh, wn.block() * 64, tid, nxt);
        if (j >= NS) mbar_wait(&sm.kv_empty[st], ((j / NS) - 1) & 1);
        if (whole(block)) {
          asm volatile("bar.sync 1, 128;" ::: "memory");  // table j&1 complete
          paged_fast<T, D, PP, NS>(sm, st, tid, cur, ktab + (j & 1) * PPB * D);
          fence_proxy_async_smem();
          asm volatile("bar.sync 1, 128;" ::: "memory");
        } else {
          paged_block<T, D, PP, NS>(sm, prm, kvh, st, block * 64, tid);
        }
        if (tid == 0) mbar_arrive(&sm.kv_full[st]);
        cur = nxt;
        w = wn;
      }
    }
  } else {
    // ------------------------------ softmax -----------------------------------
    const int t = (warp - 2) >> 2;   // tile of this warpgroup
    const int quarter = warp & 3;    // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;  // row within the tile
    const uint32_t trow = tmem + (uint32_t(quarter * 32) << 16);
    const uint32_t s_col = t * 128, o_col = kOCol + t * 128;
    const int pos = item.row0 + 128 * t + row + (prm.n_kv - prm.n_q);
    const uint32_t q_bit = 1u << (2 * t + (row >> 6));
    const float sl2 = prm.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;
    int j = 0;
    for (SegWalk w(prm.segs, item.seg_begin, item.seg_count); !w.done(); w.next(), ++j) {
      mbar_wait(&sm.s_full[t][j & 1], (j >> 1) & 1);
      tc_fence_after();
      float s[64];
      {
        uint32_t r[64];
        tmem_ld_x32(trow + s_col + (j & 1) * 64, r);
        tmem_ld_x32(trow + s_col + (j & 1) * 64 + 32, r + 32);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 64; ++i) s[i] = __uint_as_float(r[i]);
      }
      const uint32_t fl = w.flags;
      const bool active = fl & q_bit;
      const int col0 = w.block() * 64;
      const int lim = (fl & kFlagCausal) ? pos - col0 : 64;  // columns c <= lim visible
      float mx;
      if (active && lim >= 63 && !(fl & kFlagMasks)) {
        // fast path (almost every block): the whole row is visible; the max
        // is taken on raw scores (scale > 0 commutes with max)
        float tm[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) tm[g] = fmax3(s[8 * g], s[8 * g + 1], s[8 * g + 2]);
#pragma unroll
        for (int g = 0; g < 8; ++g) tm[g] = fmax3(tm[g], s[8 * g + 3], s[8 * g + 4]);
#pragma unroll
        for (int g = 0; g < 8; ++g) tm[g] = fmax3(tm[g], s[8 * g + 5], s[8 * g + 6]);
#pragma unroll
        for (int g = 0; g < 8; ++g) tm[g] = fmaxf(tm[g], s[8 * g + 7]);
        mx = fmax3(fmax3(tm[0], tm[1], tm[2]), fmax3(tm[3], tm[4], tm[5]), fmaxf(tm[6], tm[7])) * sl2;
      } else {
        uint64_t emask = ~0ull;
        if (fl & kFlagMasks) emask = prm.row_masks[(int64_t)(w.mask_base + w.i) * kItemRows + 128 * t + row];
        mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const bool ok = active && i <= lim && ((emask >> i) & 1ull);
          s[i] = ok ? s[i] : -INFINITY;
          mx = fmaxf(mx, s[i]);
        }
        mx *= sl2;
      }
      // lazy rescale: only when the max grows by more than 2^threshold
      const float m_new = fmaxf(m_run, mx);
      const bool need = (m_run != -INFINITY) && (m_new > m_run + kRescaleThreshold);
      if (m_run == -INFINITY) m_run = m_new;
      const bool rescale = __any_sync(0xffffffffu, need);
      if (rescale) {
        if (j > 0) mbar_wait(&sm.o_done[t], (j - 1) & 1);  // PV_{j-1} landed in O
        tc_fence_after();
        const float alpha = need ? exp2f(m_run - m_new) : 1.f;
#pragma unroll
        for (int c = 0; c < D; c += 16) {
          uint32_t r[16];
          tmem_ld_x16(trow + o_col + c, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st_x16(trow + o_col + c, r);
        }
        tmem_wait_st();
        if (need) {
          l_run *= alpha;
          m_run = m_new;
        }
      }
      // p = 2^(s*scale - m): one FFMA2 per pair + one MUFU.EX2 each (-inf -> 0)
      const float shift = m_run == -INFINITY ? 0.f : m_run;
      const uint64_t sl2x2 = f2_pack(sl2, sl2), nsh = f2_pack(-shift, -shift);
      uint64_t rs[4] = {0ull, 0ull, 0ull, 0ull};
      uint32_t pk[32];
#pragma unroll
      const bool fast = active && lim >= 63 && !(fl & kFlagMasks);  // every s[i] finite
      for (int i = 0; i < 64; i += 2) {
        const uint64_t x2 = f2_fma(f2_pack(s[i], s[i + 1]), sl2x2, nsh);
        float p0, p1;
        if (kPolyFrom <= i && fast) {  // part of the exponentials on the FMA pipe
          const float2 pp = exp2_poly2(x2);
          p0 = pp.x;
          p1 = pp.y;
        } else {
          const float2 e = f2_unpack(x2);
          p0 = fast_exp2(e.x);
          p1 = fast_exp2(e.y);
        }
        rs[(i / 2) & 3] = f2_add(rs[(i / 2) & 3], f2_pack(p0, p1));
        pk[i / 2] = kBF16 ? pack_bf162(p0, p1) : pack_half2(p0, p1);
      }
      {
        const float2 a = f2_unpack(f2_add(f2_add(rs[0], rs[1]), f2_add(rs[2], rs[3])));
        l_run += a.x + a.y;
      }
      // every o_done phase is waited exactly once: phase j-1 here (PV_{j-1} ran
      // while this softmax did; the wait is almost always already satisfied)
      if (j > 0 && !rescale) mbar_wait(&sm.o_done[t], (j - 1) & 1);
      if (kTmemP) {
        // P over the first 32 columns of this S buffer: S_t,j+2 (the next
        // writer) is issued after PV_t,j, and tcgen05 MMAs run in order
        tmem_st_x32(trow + s_col + (j & 1) * 64, pk);
        tmem_wait_st();
      } else {
        if (j >= 2) mbar_wait(&sm.p_empty[t][j & 1], ((j >> 1) - 1) & 1);
        uint8_t* prow = sm.p[kTmemP ? 0 : t][j & 1] + row * 128;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint4 v = make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
          *reinterpret_cast<uint4*>(prow + ((ch ^ (row & 7)) << 4)) = v;
        }
        fence_proxy_async_smem();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.p_full[t][j & 1]);
    }
    // epilogue: O / l -> out.  o_done completes one phase per PV; phases
    // 0..n-2 were waited in the loop, so the last one is next.
    if (n_blocks > 0) {
      mbar_wait(&sm.o_done[t], (n_blocks - 1) & 1);
      tc_fence_after();
    }
    const int grow = item.row0 + 128 * t + row;
    const float inv_l = l_run > 0.f ? 1.f / l_run : 0.f;
    T* orow = reinterpret_cast<T*>(prm.out) + ((int64_t)grow * prm.n_heads + item.head) * D;
#pragma unroll
    for (int c = 0; c < D; c += 16) {
      uint32_t r[16];
      tmem_ld_x16(trow + o_col + c, r);
      tmem_wait_ld();
      uint32_t pk[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float a = __uint_as_float(r[2 * i]) * inv_l, b = __uint_as_float(r[2 * i + 1]) * inv_l;
        pk[i] = kBF16 ? pack_bf162(a, b) : pack_half2(a, b);
      }
      if (grow < prm.n_q) {
        *reinterpret_cast<uint4*>(orow + c) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(orow + c + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 3-D map over a token-major [rows][heads][D] tensor; box = 64 channels x 1 head x box_rows.
int make_map(CUtensorMap* m, const void* base, int dtype, int D, int heads, int rows, int box_rows) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SK_ECUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)heads * D * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, dtype == SK_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                  const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return SK_ECUDA;
  }
  return SK_OK;
}

template <typename T, int D, bool PAGED = false, int PP = 64>
int launch_prefill(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const PfParams& prm,
                   int n_items, cudaStream_t st) {
  size_t smem = sizeof(PfSmem<D, PAGED ? kNSPaged : kNS, PAGED>) + 1024;
  auto kern = prefill_kernel<T, D, PAGED, PP>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<n_items, PAGED ? kPfThreads + 128 : kPfThreads, smem, st>>>(tq, tk, tv, prm);
  SK_CHECK_LAUNCH("prefill_kernel");
  return SK_OK;
}

}  // namespace
}  // namespace sk

extern "C" int sk_prefill_attn(int32_t dtype, const void* q, const void* k, const void* v, void* out, int32_t n_q,
                               int32_t n_kv, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim,
                               float softmax_scale, const sk_prefill_item* items, int32_t n_items,
                               const uint32_t* segs, const uint64_t* row_masks, void* stream) {
  using namespace sk;
  SK_CHECK_ARG(dtype == SK_F16 || dtype == SK_BF16, "prefill: dtype must be f16 or bf16");
  SK_CHECK_ARG(head_dim == 64 || head_dim == 128, "prefill: head_dim must be 64 or 128 (pad smaller dims)");
  SK_CHECK_ARG(n_q >= 1 && n_kv >= n_q, "prefill: history must cover queries");
  SK_CHECK_ARG(n_heads >= 1 && n_kv_heads >= 1 && n_heads % n_kv_heads == 0,
               "prefill: query head count is not a multiple of KV head count");
  SK_CHECK_ARG(q && k && v && out && items && segs, "prefill: NULL pointer");
  SK_CHECK_ARG((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) %
                       16 == 0,
               "prefill: q/k/v must be 16-byte aligned");
  if (n_items == 0) return SK_OK;
  CUtensorMap tq, tk, tv;
  int rc;
  if ((rc = make_map(&tq, q, dtype, head_dim, n_heads, n_q, 128))) return rc;
  if ((rc = make_map(&tk, k, dtype, head_dim, n_kv_heads, n_kv, 64))) return rc;
  if ((rc = make_map(&tv, v, dtype, head_dim, n_kv_heads, n_kv, 64))) return rc;
  PfParams prm = {};
  prm.out = out;
  prm.n_q = n_q;
  prm.n_kv = n_kv;
  prm.n_heads = n_heads;
  prm.n_kv_heads = n_kv_heads;
  prm.group = n_heads / n_kv_heads;
  prm.scale_log2 = softmax_scale * 1.4426950408889634f;
  prm.items = items;
  prm.segs = segs;
  prm.row_masks = row_masks;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == SK_F16)
    return head_dim == 128 ? launch_prefill<__half, 128>(tq, tk, tv, prm, n_items, st)
                           : launch_prefill<__half, 64>(tq, tk, tv, prm, n_items, st);
  return head_dim == 128 ? launch_prefill<__nv_bfloat16, 128>(tq, tk, tv, prm, n_items, st)
                         : launch_prefill<__nv_bfloat16, 64>(tq, tk, tv, prm, n_items, st);
}

extern "C" int sk_prefill_attn_paged(const sk_pool* pool, int32_t n_kv_heads, int32_t hist_tokens, const void* q,
                                     const void* k_chunk, const void* v_chunk, void* out, int32_t n_q,
                                     int32_t n_heads, float softmax_scale, const sk_prefill_item* items,
                                     int32_t n_items, const uint32_t* segs, const uint64_t* row_masks,
                                     void* stream) {
  using namespace sk;
  int rc = check_pool(pool);
  if (rc) return rc;
  SK_CHECK_ARG(pool->bits >= 1 && pool->bits <= 4, "prefill paged: the pool must hold <= 4-bit codes (KV4)");
  SK_CHECK_ARG(pool->page_size == 32 || pool->page_size == 64, "prefill paged: page size must be 32 or 64");
  SK_CHECK_ARG(hist_tokens >= 1 && n_q >= 1, "prefill paged: empty history or chunk");
  SK_CHECK_ARG((int64_t)(hist_tokens + pool->page_size - 1) / pool->page_size <= pool->max_pages,
               "prefill paged: more history than the pool holds");
  SK_CHECK_ARG(n_heads >= 1 && n_kv_heads >= 1 && n_heads % n_kv_heads == 0,
               "prefill paged: query head count is not a multiple of KV head count");
  SK_CHECK_ARG(q && k_chunk && v_chunk && out && items && segs, "prefill paged: NULL pointer");
  SK_CHECK_ARG((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k_chunk) |
                reinterpret_cast<uintptr_t>(v_chunk) | reinterpret_cast<uintptr_t>(pool->arena)) % 16 == 0,
               "prefill paged: q/k/v/arena must be 16-byte aligned");
  if (n_items == 0) return SK_OK;
  const int D = pool->head_dim, dtype = pool->dtype;
  CUtensorMap tq, tk, tv;  // K/V maps are not read by the paged kernel (the producer warps are)
  if ((rc = make_map(&tq, q, dtype, D, n_heads, n_q, 128))) return rc;
  if ((rc = make_map(&tk, k_chunk, dtype, D, n_kv_heads, n_q, 64))) return rc;
  if ((rc = make_map(&tv, v_chunk, dtype, D, n_kv_heads, n_q, 64))) return rc;
  PfParams prm = {};
  prm.out = out;
  prm.n_q = n_q;
  prm.n_kv = hist_tokens + n_q;
  prm.n_heads = n_heads;
  prm.n_kv_heads = n_kv_heads;
  prm.group = n_heads / n_kv_heads;
  prm.scale_log2 = softmax_scale * 1.4426950408889634f;
  prm.items = items;
  prm.segs = segs;
  prm.row_masks = row_masks;
  prm.pv = make_view(*pool);
  prm.hist = hist_tokens;
  prm.kc = k_chunk;
  prm.vc = v_chunk;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define SK_PG(TT, DD)                                                                             \
  return pool->page_size == 64 ? launch_prefill<TT, DD, true, 64>(tq, tk, tv, prm, n_items, st) \
                               : launch_prefill<TT, DD, true, 32>(tq, tk, tv, prm, n_items, st)
  if (dtype == SK_F16) {
    if (D == 128) SK_PG(__half, 128);
    SK_PG(__half, 64);
  }
  if (D == 128) SK_PG(__nv_bfloat16, 128);
  SK_PG(__nv_bfloat16, 64);
#undef SK_PG
}
