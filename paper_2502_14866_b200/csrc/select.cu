// K2 -- hierarchical page selection (LServe Eq. 2).
//
// Replaces score_pages / _stacked_stats / pinned_pages / select_pages
// (reference selector.py:39-108) in ONE kernel, grid (page chunks, streams).
// The reference ranks pages by an fp64 score; fp64 on every page is what made
// the round-1 kernel slow (conversions + DFMA + fp64 butterflies, 38 us for
// the 33.6 MB of a 128k layer).  Here the exact fp64 score is only computed
// where it can change the answer:
//
// Phase A (every CTA, HBM-bound).  Eq. 2 as a tensor-core contraction:
//     score(j, r) = sum_c q-_rc kmin_jc + q+_rc kmax_jc
//   (q- = min(q, 0), q+ = max(q, 0): one of the two products is exactly 0,
//   so each term is the reference's max(q kmax, q kmin)).  A = the stats rows
//   of 16 logical pages (M) over the 2D channels [kmin | kmax] (K), loaded
//   straight from HBM into registers, 128-bit and fully coalesced; B = the
//   retrieval rows' [q- | q+] (N = 8 rows per n-tile), staged once per CTA in
//   shared memory in the same channel permutation as A.  m16n8k16 MMAs with
//   fp32 accumulation: every product of two fp16/bf16 values is exact in
//   fp32, only the sums round.  A second MMA of |A| and |B| gives
//   sum_c |q_c k_c|, and the page's error bound is
//       err = 2^-12 * sum|t| + 1e-30
//   (fp32 summation of <= 256 exact terms errs by < 256 * 2^-23 * sum|t| =
//   2^-15 sum|t| even with truncating accumulation: 8x margin; the absolute
//   term covers underflow).  A non-finite bound (bf16 overflow) makes the
//   page undecidable in fp32 -> err = inf.  The physical page keeps the max
//   score / max bound over its logical pages and rows: (score, err) -> ws.
//
// Phase B (the stream's last CTA, found with an acq_rel ticket).  With T =
//   the K'-th largest approximate score (K' = K - |pins|, located by
//   value-linear histogram passes over [min, max] of the approximate scores)
//   and E = the largest bound:
//     approx > T + 2E  -> certainly among the top K' (true score > true K'-th)
//     approx < T - 2E  -> certainly not
//     otherwise        -> the band: rescored EXACTLY in fp64 (the round-1
//                         arithmetic, sum_c q+ kmax + q- kmin, bit-identical
//                         to the reference on fp16/bf16-valued inputs --
//                         SURVEY Appendix A.4) and ranked by (score desc,
//                         page index asc), selector.py:106.
//   A typical 128k band holds a handful of pages.  If it exceeds kBandCap
//   (massive ties, overflow) every page is scored exactly and the exact
//   radix select of round 1 (topk_exact) decides: slower, same answer.
// Output: pins + chosen pages, ascending (block scan over page order).
#include <cstdlib>

#include "sk_common.cuh"
#include "sk_sm100.cuh"

namespace sk {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRows = 32;         // retrieval rows per stream (group rows)
constexpr int kBandCap = 256;        // band pages resolved by the fast path
constexpr int kRadixBits = 11;       // fast-path radix digit (2048 bins)
constexpr int kNB = 1 << kRadixBits;
constexpr float kErrRel = 1.0f / 4096.0f;  // 2^-12
constexpr float kErrAbs = 1e-30f;

struct SelParams {
  PoolView pv;
  const void* q;
  int64_t q_ss, q_rs;
  const uint32_t* row_mask;
  const int32_t* tokens;
  const uint8_t* invoke;
  int K;            // budget pages
  int group_rows;
  float2* approx;   // [stream][ws_pages] (fp32 score, error bound) of phase A
  double* exact;    // [stream][ws_pages] fp64 scores of the slow path
  uint32_t* ticket;
  int ws_pages;
  int tiles_per_warp;
  int32_t* sel_out;
  int32_t* sel_count;
  int sel_stride;
  int smem_bytes;
  uint32_t flags;  // SK_LAUNCH_PDL
};

__device__ __forceinline__ bool is_pin(int i, int n) { return i == 0 || i == n - 1 || i == (n - 2 > 0 ? n - 2 : 0); }
__device__ __forceinline__ int n_pins(int n) { return n <= 1 ? 1 : (n == 2 ? 2 : 3); }  // selector.py:75-78

// Order-preserving unsigned images (larger value -> larger key; never 0 for a
// finite value, so 0 marks "not a candidate").
__device__ __forceinline__ uint64_t order_key(double x) {
  x = x + 0.0;  // -0.0 -> +0.0 (equal scores tie on the index, like Python's sort)
  uint64_t u = __double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ uint32_t order_key32(float x) {
  x = x + 0.0f;
  uint32_t u = __float_as_uint(x);
  return (u >> 31) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key32_value(uint32_t k) {
  return __uint_as_float((k >> 31) ? (k & 0x7FFFFFFFu) : ~k);
}

template <typename T>
__device__ __forceinline__ void mma_f32(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
  if constexpr (std::is_same<T, __half>::value) {
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

__device__ __forceinline__ uint4 ldg_stream(const void* p) {  // read once: no L1 allocation
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// |x| of both halves.  volatile: keeps the masking inside the n-tile loop
// (hoisted, the 2 x 2D/2 masked words would double the live registers).
__device__ __forceinline__ uint32_t abs2(uint32_t x) {
  uint32_t y;
  asm volatile("and.b32 %0, %1, 0x7FFF7FFF;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t word_of(const uint4& v, int w) {
  return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

// NV values per lane; after the call lane l holds the full-warp sum of value
// index (l >> (5 - log2 NV)) in v[0].  Step OFF halves the live values: the
// lane with bit OFF set keeps the upper half, its partner the lower half.
// Every value is summed over the xor tree 16, 8, 4, 2, 1 -- the same
// pairing as a plain xor reduction.
template <int NV, int OFF>
struct Butterfly {
  static __device__ __forceinline__ void run(double* v, int lane) {
    if constexpr (NV > 1) {
      const bool upper = lane & OFF;
#pragma unroll
      for (int i = 0; i < NV / 2; ++i) {
        double send = upper ? v[i] : v[i + NV / 2];
        double keep = upper ? v[i + NV / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);
      }
      if constexpr (OFF > 1) Butterfly<NV / 2, OFF / 2>::run(v, lane);
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], OFF);
      if constexpr (OFF > 1) Butterfly<1, OFF / 2>::run(v, lane);
    }
  }
};

// ---- exact fp64 physical-page score (warp-cooperative) ------------------------
// max over the retrieval rows and the page's logical pages of
// sum_c q_c * (q_c > 0 ? kmax_c : kmin_c), each lane summing its D/32
// channels in order before the butterfly -- the round-1 arithmetic.
template <typename T, int D>
__device__ double exact_page_score(const PoolView& pv, int s, int page, int n_log, const T* qs, int64_t q_rs,
                                   const int* row_idx, int rows) {
  constexpr int CPL = D / 32;
  using W = typename std::conditional<CPL == 4, uint2, uint32_t>::type;  // CPL values of T
  const int lane = threadIdx.x & 31;
  const int LP = pv.P / pv.L;
  const int la = page * LP, nl = min(la + LP, n_log) - la;
  const int V = rows * nl;
  double best = -INFINITY;
  for (int v0 = 0; v0 < V; v0 += 8) {
    W wq[8], wmin[8], wmax[8];  // every load of the chunk issued before any math
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int vi = min(v0 + jj, V - 1);
      const int r = vi / nl, l = la + vi % nl;
      const T* st = reinterpret_cast<const T*>(pv.stats_ptr(s, l)) + lane * CPL;
      wq[jj] = *reinterpret_cast<const W*>(qs + (int64_t)row_idx[r] * q_rs + lane * CPL);
      wmin[jj] = __ldcg(reinterpret_cast<const W*>(st));
      wmax[jj] = __ldcg(reinterpret_cast<const W*>(st + D));
    }
    double v[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const T* qv = reinterpret_cast<const T*>(&wq[jj]);
      const T* kn = reinterpret_cast<const T*>(&wmin[jj]);
      const T* kx = reinterpret_cast<const T*>(&wmax[jj]);
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const double qd = (double)DT<T>::to_f(qv[c]);
        acc = fma(qd, (double)DT<T>::to_f(qd > 0.0 ? kx[c] : kn[c]), acc);
      }
      v[jj] = acc;
    }
    Butterfly<8, 16>::run(v, lane);
    double mine = (v0 + (lane >> 2) < V) ? v[0] : -INFINITY;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) mine = fmax(mine, __shfl_xor_sync(0xffffffffu, mine, off));
    best = fmax(best, mine);
  }
  return best;
}

// ---- phase A: approximate scores + bounds of this warp's tiles ----------------
// Tile = 16 logical pages.  Thread (g = lane/4, t = lane%4) holds logical
// pages g and g+8 of the tile, bytes [64i + 16t, +16) of each 2D-channel row
// for i < 2D/32 (a load instruction covers 8 x 64 contiguous bytes), and
// k-step ks uses words 2(ks&1), 2(ks&1)+1 of chunk ks/2 -- i.e. the channel
// permutation ch(ks, k) = (ks/2)*32 + t*8 + 4(ks&1) + {0,1 | 2,3}; bfrag holds
// q' = [q- | q+] of every group row in the same permutation.  A warp's first
// tile is loaded straight into registers, the following ones arrive by 1-D
// bulk copies into the warp's shared-memory slot; every address is clamped
// to the stream's allocated stats rows (not its token count), so the first
// loads issue before the kernel has read anything.
template <typename T, int D>
__device__ __forceinline__ void load_tile(const SelParams& p, int s, int rows_alloc, int ti, uint4 (&a)[2][D / 16]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int l0 = ti * 16 + g, l1 = l0 + 8;
  const T* r0 = reinterpret_cast<const T*>(p.pv.stats_ptr(s, min(l0, rows_alloc - 1))) + t * 8;
  const T* r1 = reinterpret_cast<const T*>(p.pv.stats_ptr(s, min(l1, rows_alloc - 1))) + t * 8;
#pragma unroll
  for (int i = 0; i < D / 16; ++i) {
    a[0][i] = ldg_stream(r0 + i * 32);
    a[1][i] = ldg_stream(r1 + i * 32);
  }
}
template <int D>
__device__ __forceinline__ void lds_tile(const uint8_t* tile, uint4 (&a)[2][D / 16]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const uint8_t* r0 = tile + g * (4 * D) + t * 16;  // a row: 2D values of 2 bytes
  const uint8_t* r1 = r0 + 8 * (4 * D);
#pragma unroll
  for (int i = 0; i < D / 16; ++i) {
    a[0][i] = *reinterpret_cast<const uint4*>(r0 + i * 64);
    a[1][i] = *reinterpret_cast<const uint4*>(r1 + i * 64);
  }
}
__device__ __forceinline__ void bulk_tile(uint8_t* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  mbar_arrive_expect_tx(bar, bytes);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint32_t tile_bytes(int ti, int rows_alloc, int D) {
  return (uint32_t)(min(16, rows_alloc - ti * 16) * 4 * D);
}

template <typename T, int D, int NT>
__device__ __forceinline__ void score_tiles(const SelParams& p, int s, int n_log, int n_pages, uint32_t rmask,
                                            int rows_alloc, int tile_hint, const uint2* bfrag, float2* approx,
                                            uint4 (&a)[2][D / 16], uint8_t* slot, uint64_t* bar) {
  constexpr int KS = D / 8;  // k-steps over 2D channels
  const int LP = p.pv.P / p.pv.L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int n_tiles = (n_log + 15) >> 4;
  const int tile0 = (blockIdx.x * kWarps + warp) * p.tiles_per_warp;
  const int tile1 = min(tile0 + p.tiles_per_warp, n_tiles);
  const int tile1_hint = min(tile0 + p.tiles_per_warp, tile_hint);  // tiles whose copies were issued
  float run_v = -INFINITY, run_e = 0.f;  // LP = 32: a page spans two tiles of this warp
  int ti = tile0;
  for (; ti < tile1; ++ti) {
    const int l0 = ti * 16 + g, l1 = l0 + 8;
    if (ti != tile0) {  // tile ti sits in the slot; refill it with ti + 1 once every lane holds ti
      mbar_wait(bar, (ti - tile0 - 1) & 1);
      lds_tile<D>(slot, a);
      __syncwarp();
      if (lane == 0 && ti + 1 < tile1_hint)
        bulk_tile(slot, p.pv.stats_ptr(s, (ti + 1) * 16), tile_bytes(ti + 1, rows_alloc, D), bar);
    }
    // n-tiles innermost: each k-step's |A| words are formed once and die with
    // it; two accumulator chains (even / odd k-steps) halve the MMA latency chain
    constexpr int CH = NT <= 2 ? 2 : 1;  // accumulator chains (registers allowing)
    float c[NT][2][4], m[NT][2][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 4; ++e) c[nt][h][e] = m[nt][h][e] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int i = ks >> 1, w = (ks & 1) * 2;
      const uint32_t a0 = word_of(a[0][i], w), a1 = word_of(a[1][i], w);
      const uint32_t a2 = word_of(a[0][i], w + 1), a3 = word_of(a[1][i], w + 1);
      const uint32_t m0 = abs2(a0), m1 = abs2(a1), m2 = abs2(a2), m3 = abs2(a3);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const uint2 b = bfrag[(nt * KS + ks) * 32 + lane];
        mma_f32<T>(c[nt][ks % CH], a0, a1, a2, a3, b.x, b.y);
        mma_f32<T>(m[nt][ks % CH], m0, m1, m2, m3, abs2(b.x), abs2(b.y));
      }
    }
    // accumulator: c0/c1 = (page g, group rows 2t, 2t+1), c2/c3 = (page g+8, ...);
    // only the retrieval rows (bits of rmask) count
    float v0 = -INFINITY, v1 = -INFINITY, e0 = 0.f, e1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = nt * 8 + 2 * t + e;
        if (col >= 32 || !((rmask >> col) & 1u)) continue;
        const float c0 = c[nt][0][e] + c[nt][1][e], c2 = c[nt][0][2 + e] + c[nt][1][2 + e];
        const float ma = m[nt][0][e] + m[nt][1][e], mb = m[nt][0][2 + e] + m[nt][1][2 + e];
        const bool f0 = isfinite(ma), f1 = isfinite(mb);
        v0 = fmaxf(v0, f0 ? c0 : 0.f);
        e0 = fmaxf(e0, f0 ? fmaf(ma, kErrRel, kErrAbs) : INFINITY);
        v1 = fmaxf(v1, f1 ? c2 : 0.f);
        e1 = fmaxf(e1, f1 ? fmaf(mb, kErrRel, kErrAbs) : INFINITY);
      }
    if (l0 >= n_log) { v0 = -INFINITY; e0 = 0.f; }
    if (l1 >= n_log) { v1 = -INFINITY; e1 = 0.f; }
    // rows: reduce over the quad
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      v0 = fmaxf(v0, __shfl_xor_sync(0xffffffffu, v0, off));
      v1 = fmaxf(v1, __shfl_xor_sync(0xffffffffu, v1, off));
      e0 = fmaxf(e0, __shfl_xor_sync(0xffffffffu, e0, off));
      e1 = fmaxf(e1, __shfl_xor_sync(0xffffffffu, e1, off));
    }
    float2* out = approx + (int64_t)s * p.ws_pages;
    if (LP < 16) {
      // logical pages of one physical page: lanes whose g differ in the low log2(LP) bits
      for (int off = 4; off < 4 * LP; off <<= 1) {
        v0 = fmaxf(v0, __shfl_xor_sync(0xffffffffu, v0, off));
        v1 = fmaxf(v1, __shfl_xor_sync(0xffffffffu, v1, off));
        e0 = fmaxf(e0, __shfl_xor_sync(0xffffffffu, e0, off));
        e1 = fmaxf(e1, __shfl_xor_sync(0xffffffffu, e1, off));
      }
      if (t == 0 && g % LP == 0) {
        const int pg0 = l0 / LP, pg1 = l1 / LP;
        if (l0 < n_log && pg0 < p.ws_pages) out[pg0] = make_float2(v0, e0);
        if (l1 < n_log && pg1 < p.ws_pages) out[pg1] = make_float2(v1, e1);
      }
    } else {
      float v = fmaxf(v0, v1), e = fmaxf(e0, e1);
#pragma unroll
      for (int off = 4; off <= 16; off <<= 1) {
        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
        e = fmaxf(e, __shfl_xor_sync(0xffffffffu, e, off));
      }
      run_v = fmaxf(run_v, v);
      run_e = fmaxf(run_e, e);
      const int tpp = LP / 16;
      if ((ti % tpp) == tpp - 1 || ti == n_tiles - 1) {
        const int pg = ti / tpp;
        if (lane == 0 && pg < n_pages && pg < p.ws_pages) out[pg] = make_float2(run_v, run_e);
        run_v = -INFINITY;
        run_e = 0.f;
      }
    }
  }
  // a copy issued for a tile past the token count must land before the CTA exits
  if (lane == 0 && ti < tile1_hint && ti > tile0) mbar_wait(bar, (ti - tile0 - 1) & 1);
  else if (lane == 0 && ti == tile0 && tile0 + 1 < tile1_hint) mbar_wait(bar, 0);
}

// Block-wide exclusive scan of one value per thread in thread order; returns
// the thread's exclusive prefix and the block total.
__device__ __forceinline__ uint32_t block_scan(uint32_t x, uint32_t* warp_tot, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = x;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = lane < kWarps ? warp_tot[lane] : 0u;
    uint32_t ti = t;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, ti, off);
      if (lane >= off) ti += o;
    }
    if (lane < kWarps) warp_tot[lane] = ti - t;  // exclusive warp offsets
    if (lane == kWarps - 1) warp_tot[kWarps] = ti;
  }
  __syncthreads();
  const uint32_t res = warp_tot[warp] + incl - x;
  total = warp_tot[kWarps];
  __syncthreads();
  return res;
}

// Exclusive scan of one value per thread in thread order with ONE barrier:
// warp-inclusive shuffles, warp totals through shared memory, and each thread
// adds the totals of the warps before its own.  warp_tot must not be read
// again by the caller (no trailing barrier).
__device__ __forceinline__ uint32_t block_scan1(uint32_t x, uint32_t* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = x;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  uint32_t base = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) base += w < warp ? warp_tot[w] : 0u;
  return base + incl - x;
}

// ---- exact top-k (slow path): every non-pinned page scored in fp64 ------------
// Pins, then the best K-|pins| others by (score desc, index asc), ascending.
// Keys staged in shared memory when they fit, else re-read from the slots.
__device__ void topk_exact(int n, int K, const double* scores, uint64_t* s_keys, int stage_cap, int32_t* sel_out,
                           int32_t* sel_count) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t whist[kWarps * 256];
  __shared__ uint32_t warp_tot[kWarps + 1];
  __shared__ uint64_t s_max[kWarps], s_min[kWarps];
  __shared__ uint32_t sh_bin, sh_kk, sh_done;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool staged = n <= stage_cap;
  auto key_at = [&](int i) -> uint64_t {
    if (staged) return s_keys[i];
    return is_pin(i, n) ? 0ull : order_key(__ldcg(scores + i));
  };
  uint64_t kmax = 0, kmin = ~0ull;
  for (int i = tid; i < n; i += kThreads) {
    const uint64_t k = is_pin(i, n) ? 0ull : order_key(__ldcg(scores + i));
    if (staged) s_keys[i] = k;
    if (k) {
      kmax = k > kmax ? k : kmax;
      kmin = k < kmin ? k : kmin;
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, kmax, off), b = __shfl_xor_sync(0xffffffffu, kmin, off);
    kmax = a > kmax ? a : kmax;
    kmin = b < kmin ? b : kmin;
  }
  if (lane == 0) {
    s_max[warp] = kmax;
    s_min[warp] = kmin;
  }
  if (tid == 0) {
    sh_kk = K - n_pins(n);
    sh_done = 0;
  }
  __syncthreads();
  kmax = 0;
  kmin = ~0ull;
  for (int w = 0; w < kWarps; ++w) {
    kmax = s_max[w] > kmax ? s_max[w] : kmax;
    kmin = s_min[w] < kmin ? s_min[w] : kmin;
  }
  const int common = kmax == kmin ? 64 : __clzll(kmax ^ kmin);
  int shift = 56 - 8 * (common / 8);
  uint64_t mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
  uint64_t prefix = kmax & mask;
  bool done = false;
  if (common == 64) {  // every candidate has the same key: the lowest indices win
    mask = ~0ull;
    prefix = kmax;
    shift = -8;
  }
  const int kpt = (n + kThreads - 1) / kThreads;
  const int i0 = tid * kpt, i1 = min(n, i0 + kpt);
  for (; shift >= 0; shift -= 8) {
    for (int b = tid; b < kWarps * 256; b += kThreads) whist[b] = 0;
    __syncthreads();
    for (int i = i0; i < i1; ++i) {
      const uint64_t key = key_at(i);
      if (key && (key & mask) == prefix) atomicAdd(&whist[warp * 256 + (uint32_t(key >> shift) & 255u)], 1u);
    }
    __syncthreads();
    {
      uint32_t h = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) h += whist[w * 256 + tid];
      hist[tid] = h;
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t kk = sh_kk;
      uint32_t sum = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) sum += hist[255 - 8 * lane - b];
      uint32_t incl = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      const uint32_t excl = incl - sum;
      const uint32_t ballot = __ballot_sync(0xffffffffu, incl >= kk);
      const int first = __ffs(ballot) - 1;
      if (lane == first) {
        uint32_t cum = excl;
        for (int b = 0; b < 8; ++b) {
          const uint32_t h = hist[255 - 8 * lane - b];
          if (cum + h >= kk) {
            sh_bin = 255 - 8 * lane - b;
            sh_kk = kk - cum;
            sh_done = (h == kk - cum) ? 1u : 0u;
            break;
          }
          cum += h;
        }
      }
    }
    __syncthreads();
    prefix |= (uint64_t)sh_bin << shift;
    mask |= (uint64_t)0xFF << shift;
    done = sh_done;
    __syncthreads();
    if (done) break;
  }
  const bool all_equal_taken = done;
  const uint32_t take_eq = sh_kk;
  uint32_t n_eq = 0;
  for (int i = i0; i < i1; ++i) {
    const uint64_t key = key_at(i);
    n_eq += (key && !is_pin(i, n) && (key & mask) == prefix) ? 1u : 0u;
  }
  uint32_t tot;
  uint32_t eq_rank = block_scan(n_eq, warp_tot, tot);
  uint32_t n_take = 0;
  for (int i = i0; i < i1; ++i) {
    const uint64_t key = key_at(i);
    const bool pinned = is_pin(i, n);
    const uint64_t km = key & mask;
    const bool cand = !pinned && key != 0;
    bool take = pinned || (cand && km > prefix);
    if (cand && km == prefix) take = take || all_equal_taken || eq_rank++ < take_eq;
    n_take += take ? 1u : 0u;
  }
  uint32_t out_pos = block_scan(n_take, warp_tot, tot);
  eq_rank -= n_eq;  // replay the same decisions to write them
  for (int i = i0; i < i1; ++i) {
    const uint64_t key = key_at(i);
    const bool pinned = is_pin(i, n);
    const uint64_t km = key & mask;
    const bool cand = !pinned && key != 0;
    bool take = pinned || (cand && km > prefix);
    if (cand && km == prefix) take = take || all_equal_taken || eq_rank++ < take_eq;
    if (take) sel_out[out_pos++] = i;
  }
  if (tid == kThreads - 1) *sel_count = out_pos;
}

// ---- phase B, fast path ----------------------------------------------------------
// Returns false (nothing written) when the band is larger than kBandCap.
#ifdef SK_SEL_TIMING  // timing builds only: globaltimer stamps of phase B into the f64 scratch
#define SK_STAMP(i)                                                                               \
  do {                                                                                            \
    if (threadIdx.x == 0) {                                                                       \
      uint64_t t_;                                                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                      \
      reinterpret_cast<uint64_t*>(p.exact)[(int64_t)s * p.ws_pages + (i)] = t_;                   \
    }                                                                                             \
  } while (0)
// CTA-level phase-A stamps: [stream][8 + 3 * blockIdx.x + i] of the same scratch
#define SK_CSTAMP(i)                                                                                        \
  do {                                                                                                      \
    if (threadIdx.x == 0) {                                                                                 \
      uint64_t t_;                                                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                                \
      reinterpret_cast<uint64_t*>(p.exact)[(int64_t)s * p.ws_pages + 8 + 3 * blockIdx.x + (i)] = t_;        \
    }                                                                                                       \
  } while (0)
#else
#define SK_STAMP(i) \
  do {              \
  } while (0)
#define SK_CSTAMP(i) \
  do {               \
  } while (0)
#endif

// The K'-th largest approximate score is located by 11-bit radix passes over
// the order-preserving 32-bit images (thread t holds pages [t*kpt, +kpt)),
// from the first bit where the candidates differ, and only until its bin is
// narrower than 2E: any T in the bin [lo_b, hi_b] then gives
//   certain-in   approx > hi_b + 2E   (true score > true K'-th score)
//   certain-out  approx < lo_b - 2E
// and the band in between is rescored exactly.  Counters and the band list
// use shared-memory atomics (the list order is irrelevant: the rank compares
// (exact score, page index)); one block scan orders the output.
template <typename T, int D, int KPT>
__device__ bool topk_filtered(const SelParams& p, int s, int n, int n_log, const T* qs, const int* row_idx, int rows,
                              uint32_t* hist2) {
  constexpr int BPT = kNB / kThreads;  // bins per thread (8)
  __shared__ uint32_t wtot[kWarps + 1];
  __shared__ uint32_t s_max[kWarps], s_min[kWarps], s_emax[kWarps];
  __shared__ uint32_t sh_bin, sh_kk, s_nb, s_nin;
  __shared__ int band_idx[kBandCap];
  __shared__ uint64_t band_key[kBandCap];
  __shared__ uint32_t chosen_bits[64 * kThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float2* approx = p.approx + (int64_t)s * p.ws_pages;
  const int kpt = (n + kThreads - 1) / kThreads;
  const int i0 = tid * kpt;
  uint32_t key[KPT];
  float emax = 0.f;
  uint32_t kmax = 0, kmin = ~0u;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const int i = i0 + j;
    key[j] = 0;
    if (j < kpt && i < n && !is_pin(i, n)) {
      const float2 ae = __ldcg(approx + i);
      key[j] = order_key32(ae.x);
      emax = fmaxf(emax, ae.y);
      kmax = max(kmax, key[j]);
      kmin = min(kmin, key[j]);
    }
  }
  for (int b = tid; b < kNB; b += kThreads) hist2[b] = 0;
  for (int b = tid; b < (n + 31) / 32; b += kThreads) chosen_bits[b] = 0;
  if (tid == 0) s_nb = s_nin = 0;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, off));
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, off));
    emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, off));
  }
  if (lane == 0) {
    s_max[warp] = kmax;
    s_min[warp] = kmin;
    s_emax[warp] = __float_as_uint(emax);
  }
  SK_STAMP(1);
  __syncthreads();
  kmax = 0;
  kmin = ~0u;
  emax = 0.f;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    kmax = max(kmax, s_max[w]);
    kmin = min(kmin, s_min[w]);
    emax = fmaxf(emax, __uint_as_float(s_emax[w]));
  }
  const double w2 = 2.0 * (double)emax * (1.0 + 0x1p-20);  // 2E, widened for the threshold roundings
  uint32_t kk = p.K - n_pins(n);                            // K' >= 1 here
  const uint32_t kq = kk;
  // Value-linear passes: bin b of [vlo, vhi] holds x with
  // floor((x - vlo) * kNB / (vhi - vlo)) = b (double arithmetic, monotone in x),
  // so keys spread over the bins by value -- few share a histogram counter,
  // where the top bits of the order keys put most pages in a handful of bins.
  // A pass finds the bin of the K'-th largest remaining candidate; the next
  // pass splits that bin.  It stops once the bin is narrower than 2E or holds
  // few candidates (or after 3 passes): the band [lo - 2E, hi + 2E] around it
  // is rescored exactly whatever its width.
  double vlo = (double)key32_value(kmin), vhi = (double)key32_value(kmax);
  uint32_t cand = 0;  // bit j: key j still inside the current bin
#pragma unroll
  for (int j = 0; j < KPT; ++j) cand |= key[j] ? (1u << j) : 0u;
  __shared__ uint32_t sh_cnt;
  bool done = !(vhi - vlo > w2) || !isfinite(vhi - vlo);
  int cur = 0;
  for (int pass = 0; pass < 3 && !done; ++pass) {
    const double scale = (double)kNB / (vhi - vlo);
    auto bin_of = [&](uint32_t k) -> int {
      const int b = (int)(((double)key32_value(k) - vlo) * scale);
      return b < 0 ? 0 : (b > kNB - 1 ? kNB - 1 : b);
    };
    uint32_t* h = hist2 + cur * kNB;
#pragma unroll
    for (int j = 0; j < KPT; ++j)
      if ((cand >> j) & 1u) atomicAdd(&h[bin_of(key[j])], 1u);
    uint32_t* hn = hist2 + (cur ^ 1) * kNB;
    for (int b = tid; b < kNB; b += kThreads) hn[b] = 0;
    __syncthreads();  // A: histogram complete
    uint32_t loc[BPT], sum = 0;
#pragma unroll
    for (int e = 0; e < BPT; ++e) {
      loc[e] = h[kNB - 1 - BPT * tid - e];
      sum += loc[e];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();  // B: warp totals
    uint32_t excl = incl - sum;
#pragma unroll
    for (int w3 = 0; w3 < kWarps; ++w3) excl += w3 < warp ? wtot[w3] : 0u;
    if (excl < kk && kk <= excl + sum) {
      uint32_t cum = excl;
#pragma unroll
      for (int e = 0; e < BPT; ++e) {
        if (cum + loc[e] >= kk && cum < kk) {
          sh_bin = kNB - 1 - BPT * tid - e;
          sh_kk = kk - cum;
          sh_cnt = loc[e];
        }
        cum += loc[e];
      }
    }
    __syncthreads();  // C: boundary bin published
    const int bs = (int)sh_bin;
    kk = sh_kk;
#pragma unroll
    for (int j = 0; j < KPT; ++j)
      if (((cand >> j) & 1u) && bin_of(key[j]) != bs) cand &= ~(1u << j);
    // the bin's value range, widened by the rounding of the bin formula
    const double w = 1.0 / scale, delta = (vhi - vlo) * 0x1p-40;
    const double nlo = vlo + bs * w - delta, nhi = vlo + (bs + 1) * w + delta;
    vlo = nlo;
    vhi = nhi;
    cur ^= 1;
    done = !(vhi - vlo > w2) || sh_cnt <= 16u;
  }
  SK_STAMP(2);
  const double hiT = vhi + w2, loT = vlo - w2;
  uint64_t inb = 0, bnd = 0;
  uint32_t c_in = 0;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    if (!key[j]) continue;
    const double x = (double)key32_value(key[j]);
    if (x > hiT) {
      inb |= 1ull << j;
      ++c_in;
    } else if (x >= loT) {
      bnd |= 1ull << j;
      const uint32_t slot = atomicAdd(&s_nb, 1u);
      if (slot < (uint32_t)kBandCap) band_idx[slot] = i0 + j;
    }
  }
  c_in = __reduce_add_sync(0xffffffffu, c_in);
  if (lane == 0 && c_in) atomicAdd(&s_nin, c_in);
  __syncthreads();
  const uint32_t nb = s_nb, n_in = s_nin;
  SK_STAMP(3);
  if (nb > (uint32_t)kBandCap) return false;
  const uint32_t need = kq - n_in;  // in [1, nb]
  if (need < nb) {
    for (uint32_t b = warp; b < nb; b += kWarps) {
      const double sc = exact_page_score<T, D>(p.pv, s, band_idx[b], n_log, qs, p.q_rs, row_idx, rows);
      if (lane == 0) band_key[b] = order_key(sc);
    }
    __syncthreads();
    if (tid < (int)nb) {
      const uint64_t mk = band_key[tid];
      const int mi = band_idx[tid];
      uint32_t rank = 0;
      for (uint32_t b = 0; b < nb; ++b) {
        const uint64_t o = band_key[b];
        rank += (o > mk || (o == mk && band_idx[b] < mi)) ? 1u : 0u;
      }
      if (rank < need) atomicOr(&chosen_bits[mi >> 5], 1u << (mi & 31));
    }
    __syncthreads();
  }
  SK_STAMP(4);
  // ordered compaction: pins, certain-in, chosen band pages
  const bool all_band = need >= nb;
  int32_t* sel_out = p.sel_out + (int64_t)s * p.sel_stride;
  auto taken = [&](int j) -> bool {
    const int i = i0 + j;
    if (j >= kpt || i >= n) return false;
    if (is_pin(i, n) || ((inb >> j) & 1ull)) return true;
    return ((bnd >> j) & 1ull) && (all_band || ((chosen_bits[i >> 5] >> (i & 31)) & 1u));
  };
  uint32_t n_take = 0;
#pragma unroll
  for (int j = 0; j < KPT; ++j) n_take += taken(j);
  uint32_t pos = block_scan1(n_take, wtot);
#pragma unroll
  for (int j = 0; j < KPT; ++j)
    if (taken(j)) sel_out[pos++] = i0 + j;
  if (tid == kThreads - 1) p.sel_count[s] = pos;
  SK_STAMP(5);
  return true;
}

// Dynamic shared memory: [per-warp tile slots | B fragments]; phase B reuses
// the slots for its radix histograms.
template <int D>
__host__ __device__ constexpr int sel_slot_bytes() { return 16 * 4 * D; }  // one tile
template <int D>
__host__ __device__ constexpr int sel_smem_bytes() {
  return kWarps * sel_slot_bytes<D>() + 4 * (D / 8) * 32 * 8 > 2 * kNB * 4
             ? kWarps * sel_slot_bytes<D>() + 4 * (D / 8) * 32 * 8
             : 2 * kNB * 4;
}

template <typename T, int D>
__global__ void __launch_bounds__(kThreads, 2) select_kernel(const __grid_constant__ SelParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int row_idx[kMaxRows];
  __shared__ uint32_t is_last;
  __shared__ uint64_t tile_bar[kWarps];
  constexpr int KS = D / 8;
  const int s = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool pdl = p.flags & SK_LAUNCH_PDL;
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  SK_CSTAMP(0);
  // ---- issued before anything is read: the warp's first tile (registers) and
  //      its second (bulk copy into the warp's slot), addressed by the stream's
  //      allocated stats rows; then the header -------------------------------
  const int LP = p.pv.P / p.pv.L;
  const int rows_alloc = p.pv.max_pages * LP;
  const int tile_hint = (min(p.ws_pages * LP, rows_alloc) + 15) >> 4;
  const int tile0 = (blockIdx.x * kWarps + warp) * p.tiles_per_warp;
  const int tile1_hint = min(tile0 + p.tiles_per_warp, tile_hint);
  uint8_t* slot = smem + warp * sel_slot_bytes<D>();
  uint4 a0[2][D / 16];
  if (tile0 < tile1_hint) load_tile<T, D>(p, s, rows_alloc, tile0, a0);
  const bool copy1 = tile0 + 1 < tile1_hint;
  if (lane == 0) {
    mbar_init(&tile_bar[warp], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the init, before the async proxy uses it
    if (copy1) bulk_tile(slot, p.pv.stats_ptr(s, (tile0 + 1) * 16), tile_bytes(tile0 + 1, rows_alloc, D), &tile_bar[warp]);
  }
  auto drain = [&]() {  // a CTA leaving early still owns its in-flight copy
    if (lane == 0 && copy1) mbar_wait(&tile_bar[warp], 0);
  };
  const uint8_t inv = p.invoke != nullptr ? p.invoke[s] : 1;
  const uint32_t gmask = p.group_rows >= 32 ? 0xffffffffu : ((1u << p.group_rows) - 1u);
  const uint32_t rmask = p.row_mask[s] & gmask;
  const int n_tok = p.tokens[s];
  // ---- q of every group row (the previous kernel's output in a model: after
  //      the dependency wait), this thread's B-fragment entries --------------
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const T* qs = reinterpret_cast<const T*>(p.q) + s * p.q_ss;
  const int NT = (p.group_rows + 7) >> 3;
  // entry e = (nt, ks, lane) of the B fragments: 4 consecutive channels of group row nt*8 + lane/4
  auto q_entry = [&](int e) -> uint2 {
    const int nt = e / (KS * 32), ks = (e / 32) % KS, ln = e & 31;
    const int r = nt * 8 + (ln >> 2), tt = ln & 3;
    const int ch = (ks >> 1) * 32 + tt * 8 + (ks & 1) * 4;  // in [0, 2D); 4 channels of one half
    return r < p.group_rows ? __ldcg(reinterpret_cast<const uint2*>(qs + (int64_t)r * p.q_rs + (ch % D)))
                            : make_uint2(0u, 0u);
  };
  constexpr int kEnt = (KS * 32 + kThreads - 1) / kThreads;  // the first n-tile's entries, loaded now
  uint2 qraw[kEnt];
#pragma unroll
  for (int k = 0; k < kEnt; ++k) qraw[k] = tid + k * kThreads < KS * 32 ? q_entry(tid + k * kThreads) : make_uint2(0u, 0u);
  if (inv == 0 || rmask == 0) {
    drain();
    return;
  }
  const int P = p.pv.P, L = p.pv.L;
  const int n_pages = min((n_tok + P - 1) / P, p.ws_pages);
  const int n_log = min((n_tok + L - 1) / L, n_pages * LP);
  int32_t* sel_out = p.sel_out + (int64_t)s * p.sel_stride;
  const int npins = n_pins(n_pages);
  if (n_pages <= 0 || p.K >= n_pages || p.K <= npins) {  // selector.py:98-103: no scoring
    if (n_pages > 0 && blockIdx.x == 0) {
      if (p.K >= n_pages) {
        for (int i = tid; i < n_pages; i += kThreads) sel_out[i] = i;
      } else if (tid == 0) {  // pins {0, n-2, n-1}, ascending and deduplicated
        sel_out[0] = 0;
        if (n_pages >= 2) sel_out[npins - 1] = n_pages - 1;
        if (n_pages >= 3) sel_out[1] = n_pages - 2;
      }
      if (tid == 0) p.sel_count[s] = p.K >= n_pages ? n_pages : npins;
    }
    drain();
    return;
  }
  const int rows = __popc(rmask);
  if (tid == 0) {  // retrieval rows, for phase B's exact rescoring
    uint32_t m = rmask;
    for (int r = 0; r < rows; ++r) {
      row_idx[r] = __ffs(m) - 1;
      m &= m - 1;
    }
  }
  // ---- B fragments: q' = [q- | q+] of every group row, A's channel permutation
  uint2* bfrag = reinterpret_cast<uint2*>(smem + kWarps * sel_slot_bytes<D>());
  for (int e = tid; e < NT * KS * 32; e += kThreads) {
    const int k = e / kThreads;
    const int ks = (e / 32) % KS, tt = e & 3;
    const bool neg_half = ((ks >> 1) * 32 + tt * 8) < D;  // kmin channels take q-, kmax channels q+
    const uint2 raw = k < kEnt ? qraw[k < kEnt ? k : 0] : q_entry(e);
    uint32_t w[2] = {raw.x, raw.y};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t o = 0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t x = (w[h] >> (16 * c)) & 0xFFFFu;
        if (((x & 0x8000u) != 0) == neg_half) o |= x << (16 * c);
      }
      w[h] = o;
    }
    bfrag[e] = make_uint2(w[0], w[1]);
  }
  __syncthreads();
  SK_CSTAMP(1);
  // ---- phase A
  float2* approx = p.approx;
  switch (NT) {
    case 1: score_tiles<T, D, 1>(p, s, n_log, n_pages, rmask, rows_alloc, tile_hint, bfrag, approx, a0, slot, &tile_bar[warp]); break;
    case 2: score_tiles<T, D, 2>(p, s, n_log, n_pages, rmask, rows_alloc, tile_hint, bfrag, approx, a0, slot, &tile_bar[warp]); break;
    case 3: score_tiles<T, D, 3>(p, s, n_log, n_pages, rmask, rows_alloc, tile_hint, bfrag, approx, a0, slot, &tile_bar[warp]); break;
    default: score_tiles<T, D, 4>(p, s, n_log, n_pages, rmask, rows_alloc, tile_hint, bfrag, approx, a0, slot, &tile_bar[warp]); break;
  }
  // ---- CTA ticket: the stream's last CTA runs phase B
#ifndef SK_SEL_ABLATE  // timing builds only (tools/ab_variant.sh): 1 = phase A only, 2 = no phase B
#define SK_SEL_ABLATE 0
#endif
  __syncthreads();
  SK_CSTAMP(2);
  if (SK_SEL_ABLATE == 1) return;
  if (tid == 0) {  // bar.sync + a gpu-scope acq_rel RMW: releases the CTA's slots, acquires the others'
    uint32_t t;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(p.ticket + s) : "memory");
    is_last = (t == gridDim.x - 1);
    if (is_last) p.ticket[s] = 0;  // re-arm for the next invocation
  }
  __syncthreads();
  if (!is_last || SK_SEL_ABLATE == 2) return;
  uint32_t* hist2 = reinterpret_cast<uint32_t*>(smem);
  SK_STAMP(0);
  bool ok = false;
#ifdef SK_SEL_TWICE  // timing experiment: a second identical phase B (warm instruction cache), stamped
  if (n_pages <= 8 * kThreads) {
    topk_filtered<T, D, 8>(p, s, n_pages, n_log, qs, row_idx, rows, hist2);
    __syncthreads();
  }
#endif
  if (n_pages <= 8 * kThreads) ok = topk_filtered<T, D, 8>(p, s, n_pages, n_log, qs, row_idx, rows, hist2);
  else if (n_pages <= 16 * kThreads) ok = topk_filtered<T, D, 16>(p, s, n_pages, n_log, qs, row_idx, rows, hist2);
  else if (n_pages <= 32 * kThreads) ok = topk_filtered<T, D, 32>(p, s, n_pages, n_log, qs, row_idx, rows, hist2);
  else if (n_pages <= 64 * kThreads) ok = topk_filtered<T, D, 64>(p, s, n_pages, n_log, qs, row_idx, rows, hist2);
  if (ok) return;
  // ---- slow path: exact fp64 score of every non-pinned page, exact radix select
  __syncthreads();
  double* exact = p.exact + (int64_t)s * p.ws_pages;
  for (int i = warp; i < n_pages; i += kWarps) {
    if (is_pin(i, n_pages)) continue;
    const double sc = exact_page_score<T, D>(p.pv, s, i, n_log, qs, p.q_rs, row_idx, rows);
    if (lane == 0) exact[i] = sc;
  }
  __syncthreads();
  topk_exact(n_pages, p.K, exact, reinterpret_cast<uint64_t*>(smem), p.smem_bytes / 8, sel_out, p.sel_count + s);
}

// ---- sk_score_pages: exact fp64 scores of every page (score_pages) -------------
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) score_kernel(const __grid_constant__ SelParams p, double* out,
                                                          int out_stride) {
  __shared__ int row_idx[kMaxRows];
  const int s = blockIdx.y;
  const uint32_t gmask = p.group_rows >= 32 ? 0xffffffffu : ((1u << p.group_rows) - 1u);
  const uint32_t rmask = p.row_mask[s] & gmask;
  const int rows = __popc(rmask);
  if (threadIdx.x == 0) {
    uint32_t m = rmask;
    for (int r = 0; r < rows; ++r) {
      row_idx[r] = __ffs(m) - 1;
      m &= m - 1;
    }
  }
  __syncthreads();
  const int n_tok = p.tokens[s];
  const int n_pages = min((n_tok + p.pv.P - 1) / p.pv.P, out_stride);
  const int n_log = (n_tok + p.pv.L - 1) / p.pv.L;
  const T* qs = reinterpret_cast<const T*>(p.q) + s * p.q_ss;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = blockIdx.x * kWarps + warp; i < n_pages; i += gridDim.x * kWarps) {
    const double sc = rows ? exact_page_score<T, D>(p.pv, s, i, n_log, qs, p.q_rs, row_idx, rows) : -INFINITY;
    if (lane == 0) out[(int64_t)s * out_stride + i] = sc;
  }
}


template <typename T, int D>
int select_launch(const SelParams& p0, int n_streams, int max_pages, cudaStream_t st) {
  SelParams p = p0;
  const int LP = p.pv.P / p.pv.L;
  const int n_tiles = (max_pages * LP + 15) / 16;
  // ~2 CTAs per SM in total, as c equal chunks per stream (c = 2 SMs / streams,
  // so the grid is one wave: cfg4's 128 streams take 2 chunks each, 256 CTAs,
  // not 3 uneven ones spilling into a second wave); each warp streams
  // tiles_per_warp tiles (8 KB each)
  const int sms = device_sm_count();
  const int chunks = 2 * sms / n_streams > 1 ? 2 * sms / n_streams : 1;
  int tpw = (n_tiles + kWarps * chunks - 1) / (kWarps * chunks);
  tpw = tpw < 1 ? 1 : tpw;
  if (LP > 16) tpw = (tpw + LP / 16 - 1) / (LP / 16) * (LP / 16);  // a page's tiles stay in one warp
  p.tiles_per_warp = tpw;
  constexpr int kSmemBytes = sel_smem_bytes<D>();
  p.smem_bytes = kSmemBytes;
  cudaFuncSetAttribute(select_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((n_tiles + kWarps * tpw - 1) / (kWarps * tpw), n_streams, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (p.flags & SK_LAUNCH_PDL) ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, select_kernel<T, D>, p);
  if (e != cudaSuccess) {
    set_error(std::string("select_kernel: ") + cudaGetErrorString(e));
    return SK_ECUDA;
  }
  SK_CHECK_LAUNCH("select_kernel");
  return SK_OK;
}

}  // namespace
}  // namespace sk

extern "C" int64_t sk_select_scores_offset(int32_t n_streams) { return ((int64_t)n_streams * 4 + 255) / 256 * 256; }

extern "C" int64_t sk_select_workspace(int32_t n_streams, int32_t max_pages) {
  return sk_select_scores_offset(n_streams) + (int64_t)n_streams * max_pages * 16;  // tickets + 2 x 8 B per page
}

namespace {
int fill_params(sk::SelParams& p, const sk_pool* pool, int32_t n_streams, int32_t group_rows, const void* q,
                int64_t q_ss, int64_t q_rs, const uint32_t* row_mask, const int32_t* tokens) {
  using namespace sk;
  int rc = check_pool(pool);
  if (rc) return rc;
  SK_CHECK_ARG(pool->stats != nullptr, "select: pool has no stats");
  SK_CHECK_ARG(n_streams >= 1 && n_streams <= 65535 && group_rows >= 1 && group_rows <= kMaxRows,
               "select: bad stream/row counts");
  SK_CHECK_ARG(q && row_mask && tokens, "select: NULL pointer");
  SK_CHECK_ARG(reinterpret_cast<uintptr_t>(pool->stats) % 16 == 0, "select: stats must be 16-byte aligned");
  SK_CHECK_ARG(reinterpret_cast<uintptr_t>(q) % 8 == 0 && q_ss % 4 == 0 && q_rs % 4 == 0,
               "select: q must be 8-byte aligned with strides a multiple of 4 elements");
  p = SelParams{};
  p.pv = make_view(*pool);
  p.q = q;
  p.q_ss = q_ss;
  p.q_rs = q_rs;
  p.row_mask = row_mask;
  p.tokens = tokens;
  p.group_rows = group_rows;
  return SK_OK;
}
}  // namespace

extern "C" int sk_select_pages(const sk_pool* pool, int32_t n_streams, int32_t group_rows, const void* q,
                               int64_t q_stream_stride, int64_t q_row_stride, const uint32_t* row_mask,
                               const int32_t* tokens, const uint8_t* invoke, int32_t budget_pages,
                               int32_t max_pages_hint, int32_t* sel_out, int32_t* sel_count, int32_t sel_stride,
                               void* workspace, int64_t workspace_bytes, uint32_t flags, void* stream) {
  using namespace sk;
  SelParams p;
  int rc = fill_params(p, pool, n_streams, group_rows, q, q_stream_stride, q_row_stride, row_mask, tokens);
  if (rc) return rc;
  SK_CHECK_ARG(budget_pages >= 1, "select: budget below one page");
  SK_CHECK_ARG(max_pages_hint >= 1 && max_pages_hint <= pool->max_pages, "select: bad max_pages_hint");
  SK_CHECK_ARG(sel_stride >= budget_pages || sel_stride >= max_pages_hint, "select: sel_stride too small");
  SK_CHECK_ARG(workspace_bytes >= sk_select_workspace(n_streams, max_pages_hint), "select: workspace too small");
  SK_CHECK_ARG(sel_out && sel_count && workspace, "select: NULL pointer");
  p.invoke = invoke;
  p.K = budget_pages;
  p.ticket = static_cast<uint32_t*>(workspace);
  p.approx = reinterpret_cast<float2*>(static_cast<uint8_t*>(workspace) + sk_select_scores_offset(n_streams));
  p.exact = reinterpret_cast<double*>(p.approx + (int64_t)n_streams * max_pages_hint);
  p.ws_pages = max_pages_hint;
  p.sel_out = sel_out;
  p.sel_count = sel_count;
  p.sel_stride = sel_stride;
  p.flags = flags;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool f16 = pool->dtype == SK_F16;
  if (pool->head_dim == 128)
    return f16 ? select_launch<__half, 128>(p, n_streams, max_pages_hint, st)
               : select_launch<__nv_bfloat16, 128>(p, n_streams, max_pages_hint, st);
  return f16 ? select_launch<__half, 64>(p, n_streams, max_pages_hint, st)
             : select_launch<__nv_bfloat16, 64>(p, n_streams, max_pages_hint, st);
}

extern "C" int sk_score_pages(const sk_pool* pool, int32_t n_streams, int32_t group_rows, const void* q,
                              int64_t q_stream_stride, int64_t q_row_stride, const uint32_t* row_mask,
                              const int32_t* tokens, double* scores_out, int32_t out_stride, void* stream) {
  using namespace sk;
  SelParams p;
  int rc = fill_params(p, pool, n_streams, group_rows, q, q_stream_stride, q_row_stride, row_mask, tokens);
  if (rc) return rc;
  SK_CHECK_ARG(scores_out != nullptr && out_stride >= 1, "score: bad output");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int blocks = (out_stride + kWarps - 1) / kWarps;
  dim3 grid(blocks < 1024 ? blocks : 1024, n_streams);
  const bool f16 = pool->dtype == SK_F16;
  if (pool->head_dim == 128) {
    if (f16) score_kernel<__half, 128><<<grid, kThreads, 0, st>>>(p, scores_out, out_stride);
    else score_kernel<__nv_bfloat16, 128><<<grid, kThreads, 0, st>>>(p, scores_out, out_stride);
  } else {
    if (f16) score_kernel<__half, 64><<<grid, kThreads, 0, st>>>(p, scores_out, out_stride);
    else score_kernel<__nv_bfloat16, 64><<<grid, kThreads, 0, st>>>(p, scores_out, out_stride);
  }
  SK_CHECK_LAUNCH("score_kernel");
  return SK_OK;
}
