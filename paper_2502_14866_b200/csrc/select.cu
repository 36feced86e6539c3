// K2 -- hierarchical page selection (LServe Eq. 2).
//
// Replaces score_pages / _stacked_stats / pinned_pages / select_pages
// (reference selector.py:39-108) in ONE kernel, grid (page chunks, streams):
//
// Scoring (HBM-bound).  Each warp owns kPagesPerWarp consecutive physical
//   pages and streams their contiguous (k_min, k_max) rows through a
//   double-buffered pair of shared-memory slots with 1-D bulk copies
//   (cp.async.bulk, mbarrier completion): the copy of batch i+1 is in flight
//   while batch i is scored, so the selector's 33.6 MB at 128k is read at
//   close to HBM rate by ~1 CTA per SM.  Each lane scores its D/32 channels
//   of every logical page in fp64:
//       score(r, j) = sum_c q+_rc * kmax_jc + q-_rc * kmin_jc
//   (q+ = max(q,0), q- = min(q,0): one of the two products is exactly 0, so
//   each term equals the reference's max(q*kmax, q*kmin); fp16 products are
//   exact in fp64 and the sums are exact for fp16-valued inputs, matching
//   the reference's BLAS centre/radius form bit-for-bit -- SURVEY Appendix
//   A.4).  A multi-value butterfly reduces all (row, logical page) sums of
//   the warp at once; the physical-page score is their max over retrieval
//   rows and logical pages.  Only the stream's retrieval rows are computed.
//
// Top-k (the last CTA of each stream, found with an acq_rel ticket).  Radix
//   select of the (K - |pins|)-th largest score among non-pinned pages on the
//   order-preserving 64-bit image of the fp64 score, starting at the first
//   byte where the candidates' keys differ; ties go to the lower page index
//   (selector.py:106); union with the pins; ascending compaction by a
//   block-wide scan over page order.
#include <cstdlib>

#include "sk_common.cuh"
#include "sk_sm100.cuh"

namespace sk {
namespace {

constexpr int kScoreThreads = 256;
constexpr int kScoreWarps = kScoreThreads / 32;
constexpr int kBatchesPerWarp = 4;  // slots a warp streams through
constexpr int kTopkThreads = kScoreThreads;
constexpr int kTopkWarps = kTopkThreads / 32;

__device__ __forceinline__ int pins_of(int n, int* pin) {  // selector.py:75-78
  int c = 0;
  pin[c++] = 0;
  int a = n - 2 > 0 ? n - 2 : 0;
  if (a != 0) pin[c++] = a;
  if (n - 1 != 0 && n - 1 != a) pin[c++] = n - 1;
  return c;
}
__device__ __forceinline__ bool is_pin(int i, int n) { return i == 0 || i == n - 1 || i == (n - 2 > 0 ? n - 2 : 0); }

// Order-preserving unsigned image of a double (larger score -> larger key).
// Never 0 for a real score, so 0 marks "not a candidate".
__device__ __forceinline__ uint64_t order_key(double x) {
  x = x + 0.0;  // -0.0 -> +0.0 (equal scores tie on the index, like Python's sort)
  uint64_t u = __double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// NV values per lane; after the call lane l holds the full-warp sum of value
// index (l >> (5 - log2 NV)) in v[0].  Step OFF halves the live values: the
// lane with bit OFF set keeps the upper half, its partner the lower half.
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

// fp16/bf16 bit patterns -> exact doubles
template <typename T>
__device__ __forceinline__ void to_f64x4(uint2 w, double* o) {
  const float2 a = DT<T>::to_f2(w.x), b = DT<T>::to_f2(w.y);
  o[0] = a.x;
  o[1] = a.y;
  o[2] = b.x;
  o[3] = b.y;
}

// Retrieval rows [rbase, rbase + RMAX) for this lane's channels.  Up to two
// rows use the sign-select form max(q*kmax, q*kmin) = q * (q > 0 ? kmax :
// kmin): qa = q (fp64) and per 32-bit word of stats a mask picking k_max
// where q > 0, so each (row, channel) costs one conversion and one DFMA.
// Four rows share the converted k_min/k_max instead: qa = q+, qb = q-.
// Either way the fp64 sum sees exactly the same non-zero terms in the same
// order (sum over channels of q+*kmax + q-*kmin), so scores are identical.
template <typename T, int RMAX>
__device__ __forceinline__ void load_rows(const T* q, int64_t q_rs, uint32_t rmask, int rbase, int rows, int D,
                                          double (&qd)[RMAX][4], double (&qb)[RMAX][4], uint32_t (&qsel)[RMAX][2]) {
  const int lane = threadIdx.x & 31, cpl = D / 32;
  uint32_t mbits = rmask;
  for (int r = 0; r < rbase; ++r) mbits &= mbits - 1;
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    const int g = __ffs(mbits) - 1;
    const bool ok = rbase + r < rows && g >= 0;
    if (ok) mbits &= mbits - 1;
    const T* qr = q + (int64_t)(ok ? g : 0) * q_rs + lane * cpl;
    qsel[r][0] = qsel[r][1] = 0u;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double x = (ok && c < cpl) ? (double)DT<T>::to_f(qr[c]) : 0.0;
      if constexpr (RMAX <= 2) {
        qd[r][c] = x;
        if (x > 0.0) qsel[r][c >> 1] |= (c & 1) ? 0xFFFF0000u : 0x0000FFFFu;
      } else {
        qd[r][c] = x > 0.0 ? x : 0.0;
        qb[r][c] = x < 0.0 ? x : 0.0;
      }
    }
  }
}

template <typename T, int RMAX>
__device__ __forceinline__ void row_scores(uint2 wmin, uint2 wmax, const double (&qd)[RMAX][4],
                                           const double (&qb)[RMAX][4], const uint32_t (&qsel)[RMAX][2],
                                           double* acc_out) {
  if constexpr (RMAX > 2) {
    double kmin[4], kmax[4];
    to_f64x4<T>(wmin, kmin);
    to_f64x4<T>(wmax, kmax);
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc = fma(qd[r][c], kmax[c], acc);
        acc = fma(qb[r][c], kmin[c], acc);
      }
      acc_out[r] = acc;
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    uint2 w;
    w.x = (wmax.x & qsel[r][0]) | (wmin.x & ~qsel[r][0]);
    w.y = (wmax.y & qsel[r][1]) | (wmin.y & ~qsel[r][1]);
    double k[4];
    to_f64x4<T>(w, k);
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) acc = fma(qd[r][c], k[c], acc);
    acc_out[r] = acc;
  }
}

// Scores of the np pages staged in sbuf (nl_rel valid logical pages) for
// rows [rbase, rbase + RMAX); lane 0 writes (first row chunk) or max-merges
// (later chunks) each page's score into out[].  LPC logical pages per
// butterfly pass (RMAX * LPC <= 16).
template <typename T, int RMAX, int LPC>
__device__ __forceinline__ void score_batch(const uint8_t* sbuf, int np, int lp_per, int nl_rel, int D,
                                            const double (&qd)[RMAX][4], const double (&qb)[RMAX][4], const uint32_t (&qsel)[RMAX][2], int rbase,
                                            int rows, double* out) {
  constexpr int NV = RMAX * LPC;
  const int lane = threadIdx.x & 31;
  const int cpl = D / 32;
  const int row_bytes = 2 * D * 2;  // (k_min, k_max) of one logical page
  for (int pi = 0; pi < np; ++pi) {
    double best = -INFINITY;
    for (int l0 = 0; l0 < lp_per; l0 += LPC) {
      double v[NV];
#pragma unroll
      for (int jj = 0; jj < LPC; ++jj) {
        const int lrel = pi * lp_per + l0 + jj;
        const T* st = reinterpret_cast<const T*>(sbuf + (int64_t)min(lrel, nl_rel - 1) * row_bytes);
        uint2 wmin, wmax;
        if (cpl == 4) {
          wmin = *reinterpret_cast<const uint2*>(st + lane * 4);
          wmax = *reinterpret_cast<const uint2*>(st + D + lane * 4);
        } else {
          wmin = make_uint2(*reinterpret_cast<const uint32_t*>(st + lane * 2), 0u);
          wmax = make_uint2(*reinterpret_cast<const uint32_t*>(st + D + lane * 2), 0u);
        }
        double acc[RMAX];
        row_scores<T, RMAX>(wmin, wmax, qd, qb, qsel, acc);
#pragma unroll
        for (int r = 0; r < RMAX; ++r) v[r * LPC + jj] = acc[r];
      }
      Butterfly<NV, 16>::run(v, lane);
      const int idx = lane >> (6 - __ffs(NV));  // value index owned by this lane
      const int r = idx / LPC, jj = idx % LPC;
      const bool valid = rbase + r < rows && l0 + jj < lp_per && pi * lp_per + l0 + jj < nl_rel;
      double mine = valid ? v[0] : -INFINITY;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) mine = fmax(mine, __shfl_xor_sync(0xffffffffu, mine, off));
      best = fmax(best, mine);
    }
    if (lane == 0) out[pi] = rbase == 0 ? best : fmax(out[pi], best);
  }
}

// Grouped form for LP = P/L logical pages per physical page with RMAX * LP
// dividing 32: PG = 32 / (RMAX * LP) physical pages share one butterfly, so
// the dependent shuffle chain (5 butterfly levels + log2(32/PG) max levels)
// is paid once per PG pages instead of once per page.
template <typename T, int RMAX, int LP>
__device__ __forceinline__ void score_batch_grouped(const uint8_t* sbuf, int np, int nl_rel, int D,
                                                    const double (&qd)[RMAX][4], const double (&qb)[RMAX][4],
                                                    const uint32_t (&qsel)[RMAX][2], int rbase, int rows,
                                                    double* out) {
  constexpr int PG = 32 / (RMAX * LP);
  constexpr int NV = 32;
  const int lane = threadIdx.x & 31;
  const int cpl = D / 32;
  const int row_bytes = 2 * D * 2;
  for (int g0 = 0; g0 < np; g0 += PG) {
    double v[NV];
#pragma unroll
    for (int pg = 0; pg < PG; ++pg) {
#pragma unroll
      for (int lp = 0; lp < LP; ++lp) {
        const int lrel = (g0 + pg) * LP + lp;
        const T* st = reinterpret_cast<const T*>(sbuf + (int64_t)min(lrel, nl_rel - 1) * row_bytes);
        uint2 wmin, wmax;
        if (cpl == 4) {
          wmin = *reinterpret_cast<const uint2*>(st + lane * 4);
          wmax = *reinterpret_cast<const uint2*>(st + D + lane * 4);
        } else {
          wmin = make_uint2(*reinterpret_cast<const uint32_t*>(st + lane * 2), 0u);
          wmax = make_uint2(*reinterpret_cast<const uint32_t*>(st + D + lane * 2), 0u);
        }
        double acc[RMAX];
        row_scores<T, RMAX>(wmin, wmax, qd, qb, qsel, acc);
#pragma unroll
        for (int r = 0; r < RMAX; ++r) v[(pg * RMAX + r) * LP + lp] = acc[r];
      }
    }
    Butterfly<NV, 16>::run(v, lane);  // lane l now holds value l
    const int pg = lane / (RMAX * LP), r = (lane / LP) % RMAX, lp = lane % LP;
    const bool valid = rbase + r < rows && g0 + pg < np && (g0 + pg) * LP + lp < nl_rel;
    double mine = valid ? v[0] : -INFINITY;
#pragma unroll
    for (int off = 1; off < RMAX * LP; off <<= 1) mine = fmax(mine, __shfl_xor_sync(0xffffffffu, mine, off));
    if (lane % (RMAX * LP) == 0 && g0 + pg < np) out[g0 + pg] = rbase == 0 ? mine : fmax(out[g0 + pg], mine);
  }
}

template <typename T, int RMAX, int LPC>
__device__ __forceinline__ void score_rows(const uint8_t* sbuf, int np, int lp_per, int nl_rel, int D,
                                           const T* q, int64_t q_rs, uint32_t rmask, int rows, double* out) {
  for (int rb = 0; rb < rows; rb += RMAX) {
    double qd[RMAX][4], qb[RMAX][4];
    uint32_t qsel[RMAX][2];
    load_rows<T, RMAX>(q, q_rs, rmask, rb, rows, D, qd, qb, qsel);
    if constexpr (LPC * RMAX <= 32 && 32 % (LPC * RMAX) == 0 && 32 / (LPC * RMAX) > 1) {
      if (lp_per == LPC) {
        score_batch_grouped<T, RMAX, LPC>(sbuf, np, nl_rel, D, qd, qb, qsel, rb, rows, out);
        continue;
      }
    }
    score_batch<T, RMAX, LPC>(sbuf, np, lp_per, nl_rel, D, qd, qb, qsel, rb, rows, out);
  }
}

__device__ void topk_cta(int n, int K, const double* scores, uint64_t* s_keys, int stage_cap, int32_t* sel_out,
                         int32_t* sel_count);
constexpr int kRegTopkMax = 24 * kTopkThreads;                 // n <= 6144 pages (384k tokens at P=64)
constexpr int kRegTopkBits = 11;                               // radix digit: 2048 bins
constexpr int kRegTopkSmem = 2 * (1 << kRegTopkBits) * 4;      // two histograms
template <int KPT>
__device__ void topk_cta_reg(int n, int K, const double* scores, uint32_t* hist2, int32_t* sel_out,
                             int32_t* sel_count);

template <typename T, int LPC>
#ifndef SK_SEL_MINB
#define SK_SEL_MINB 1
#endif
#ifndef SK_SEL_LOG_PER_SLOT
#define SK_SEL_LOG_PER_SLOT 16
#endif
__global__ void __launch_bounds__(kScoreThreads, SK_SEL_MINB) select_kernel(PoolView pv, const T* __restrict__ q, int64_t q_ss,
                                                               int64_t q_rs, const uint32_t* __restrict__ row_mask,
                                                               const int32_t* __restrict__ tokens,
                                                               const uint8_t* __restrict__ invoke, int K,
                                                               double* ws_scores, uint32_t* ws_ticket,
                                                               int ws_pages, int pps, int32_t* sel_out_all,
                                                               int32_t* sel_count_all, int sel_stride,
                                                               int smem_bytes, int dbg) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar[kScoreWarps][2];
  __shared__ uint32_t is_last;
  const int s = blockIdx.y;
  if (invoke != nullptr && invoke[s] == 0) return;
  const uint32_t rmask = row_mask[s];
  if (rmask == 0) return;
  const int n_tok = tokens[s];
  const int P = pv.P, L = pv.L, D = pv.D, LP = P / L;
  const int n_pages = (n_tok + P - 1) / P;
  const int n_log = (n_tok + L - 1) / L;
  int32_t* sel_out = sel_out_all + (int64_t)s * sel_stride;
  double* scores = ws_scores + (int64_t)s * ws_pages;
  int pin[3];
  const int npins = pins_of(n_pages, pin);
  if (K >= n_pages || K <= npins) {  // selector.py:98-103: no scoring
    if (blockIdx.x == 0) {
      if (K >= n_pages) {
        for (int i = threadIdx.x; i < n_pages; i += blockDim.x) sel_out[i] = i;
      } else if (threadIdx.x == 0) {
        for (int i = 0; i < npins; ++i) sel_out[i] = pin[i];
      }
      if (threadIdx.x == 0) sel_count_all[s] = K >= n_pages ? n_pages : npins;
    }
    return;
  }
  // ---- scoring: the warp streams kBatchesPerWarp batches of pps pages -------
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t row_bytes = 2 * D * 2;
  const uint32_t slot = (uint32_t)pps * LP * row_bytes;
  const int wp0 = (blockIdx.x * kScoreWarps + warp) * pps * kBatchesPerWarp;  // warp's first page
  const int nb = (dbg == 1 || dbg == 3) ? 0 : max(0, min(kBatchesPerWarp, (n_pages - wp0 + pps - 1) / pps));
  uint8_t* wbuf = smem + (size_t)warp * 2 * slot;
  auto issue = [&](int b) {  // lane 0: bulk copy of batch b into slot b&1
    const int p0 = wp0 + b * pps;
    const int nl = min(min(pps, n_pages - p0) * LP, n_log - p0 * LP);
    mbar_arrive_expect_tx(&bar[warp][b & 1], nl * row_bytes);
    bulk_g2s(wbuf + (b & 1) * slot, pv.stats_ptr(s, p0 * LP), nl * row_bytes, &bar[warp][b & 1]);
  };
  if (lane == 0) {
    mbar_init(&bar[warp][0], 1);
    mbar_init(&bar[warp][1], 1);
    fence_barrier_init();
    if (nb > 0 && dbg != 5) issue(0);
    if (nb > 1 && dbg != 5) issue(1);
  }
  __syncwarp();
  const T* qs = q + s * q_ss;
  const int rows = __popc(rmask);
  for (int b = 0; b < nb; ++b) {
    const int p0 = wp0 + b * pps;
    const int np = min(pps, n_pages - p0);
    const int nl = min(np * LP, n_log - p0 * LP);
    if (dbg != 5) mbar_wait(&bar[warp][b & 1], (b >> 1) & 1);
    const uint8_t* sb = wbuf + (b & 1) * slot;
    if (dbg == 4) {
    } else if (rows == 1) score_rows<T, 1, (LPC < 16 ? LPC : 16)>(sb, np, LP, nl, D, qs, q_rs, rmask, rows, scores + p0);
    else if (rows == 2) score_rows<T, 2, (LPC < 8 ? LPC : 8)>(sb, np, LP, nl, D, qs, q_rs, rmask, rows, scores + p0);
    else score_rows<T, 4, (LPC < 4 ? LPC : 4)>(sb, np, LP, nl, D, qs, q_rs, rmask, rows, scores + p0);
    __syncwarp();  // every lane is done with the slot before it is refilled
    if (lane == 0 && b + 2 < nb && dbg != 5) issue(b + 2);
  }
  // ---- CTA ticket: the stream's last CTA runs the top-k --------------------------
  // bar.sync orders the CTA's score stores before thread 0's acq_rel fence +
  // relaxed atomic (the release pattern of CUTLASS's generic barrier)
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const uint32_t t = atomicAdd(ws_ticket + s, 1u);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    is_last = (t == gridDim.x - 1);
    if (is_last) ws_ticket[s] = 0;  // re-arm for the next invocation
  }
  __syncthreads();
  if (!is_last || dbg == 2 || dbg == 3) return;
  if (n_pages <= 16 * kTopkThreads && smem_bytes >= kRegTopkSmem && dbg != 7)  // keys per thread: as few as fit
    topk_cta_reg<16>(n_pages, K, scores, reinterpret_cast<uint32_t*>(smem), sel_out, sel_count_all + s);
  else if (n_pages <= kRegTopkMax && smem_bytes >= kRegTopkSmem && dbg != 7)
    topk_cta_reg<24>(n_pages, K, scores, reinterpret_cast<uint32_t*>(smem), sel_out, sel_count_all + s);
  else
    topk_cta(n_pages, K, scores, reinterpret_cast<uint64_t*>(smem), smem_bytes / 8, sel_out, sel_count_all + s);
}

// Block-wide exclusive scan of one value per thread (kTopkThreads threads)
// in thread order; returns the thread's exclusive prefix and the block total.
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
    const uint32_t t = lane < kTopkWarps ? warp_tot[lane] : 0u;
    uint32_t ti = t;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, ti, off);
      if (lane >= off) ti += o;
    }
    if (lane < kTopkWarps) warp_tot[lane] = ti - t;  // exclusive warp offsets
    if (lane == kTopkWarps - 1) warp_tot[kTopkWarps] = ti;
  }
  __syncthreads();
  const uint32_t res = warp_tot[warp] + incl - x;
  total = warp_tot[kTopkWarps];
  __syncthreads();
  return res;
}

// Top-k of one stream by the whole CTA (kTopkThreads threads); the trivial
// cases (every page / pins only) are handled by the caller.
__device__ void topk_cta(int n, int K, const double* scores, uint64_t* s_keys, int stage_cap, int32_t* sel_out,
                         int32_t* sel_count) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t whist[kTopkWarps * 256];
  __shared__ uint32_t warp_tot[kTopkWarps + 1];
  __shared__ uint64_t s_max[kTopkWarps], s_min[kTopkWarps];
  __shared__ uint32_t sh_bin, sh_kk, sh_done;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int pin[3];
  const int npins = pins_of(n, pin);
  const bool staged = n <= stage_cap;
  auto key_at = [&](int i) -> uint64_t {
    if (staged) return s_keys[i];
    return is_pin(i, n) ? 0ull : order_key(__ldcg(scores + i));
  };
  // keys + the candidates' max/min (to skip the leading bytes they share)
  uint64_t kmax = 0, kmin = ~0ull;
  constexpr int kU = 8;  // loads in flight per thread
  for (int base = 0; base < n; base += kU * kTopkThreads) {
    double sc[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = base + u * kTopkThreads + tid;
      sc[u] = i < n ? __ldcg(scores + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = base + u * kTopkThreads + tid;
      if (i >= n) continue;
      const uint64_t k = is_pin(i, n) ? 0ull : order_key(sc[u]);
      if (staged) s_keys[i] = k;
      if (k) {
        kmax = k > kmax ? k : kmax;
        kmin = k < kmin ? k : kmin;
      }
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
    sh_kk = K - npins;
    sh_done = 0;
  }
  __syncthreads();
  kmax = 0;
  kmin = ~0ull;
  for (int w = 0; w < kTopkWarps; ++w) {
    kmax = s_max[w] > kmax ? s_max[w] : kmax;
    kmin = s_min[w] < kmin ? s_min[w] : kmin;
  }
  // radix passes start at the first byte where the candidates differ
  const int common = kmax == kmin ? 64 : __clzll(kmax ^ kmin);
  int shift = 56 - 8 * (common / 8);
  uint64_t mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
  uint64_t prefix = kmax & mask;
  bool done = false;
  if (common == 64) {  // every candidate has the same key: the lowest indices win
    mask = ~0ull;
    prefix = kmax;
    done = false;
    shift = -8;
  }
  // thread t owns the consecutive indices [t*kpt, t*kpt + kpt): one pass over
  // its keys per radix digit, and page order is thread order for compaction
  const int kpt = (n + kTopkThreads - 1) / kTopkThreads;
  const int i0 = tid * kpt, i1 = min(n, i0 + kpt);
  for (; shift >= 0; shift -= 8) {
    for (int b = tid; b < kTopkWarps * 256; b += kTopkThreads) whist[b] = 0;
    __syncthreads();
    for (int i = i0; i < i1; ++i) {  // per-warp histograms: contention stays inside a warp
      const uint64_t key = key_at(i);
      if (key && (key & mask) == prefix) atomicAdd(&whist[warp * 256 + (uint32_t(key >> shift) & 255u)], 1u);
    }
    __syncthreads();
    {
      uint32_t h = 0;
#pragma unroll
      for (int w = 0; w < kTopkWarps; ++w) h += whist[w * 256 + tid];  // kTopkThreads == 256 bins
      hist[tid] = h;
    }
    __syncthreads();
    if (warp == 0) {
      // bins from the top: lane l covers bins 255-8l .. 248-8l
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
    __syncthreads();  // sh_* are rewritten by the next pass
    if (done) break;
  }
  const bool all_equal_taken = done;  // every key matching the prefix is selected
  const uint32_t take_eq = sh_kk;     // else: this many keys == prefix, lowest index first
  // ordered compaction: rank of equal keys, then output positions, by two
  // block-wide scans over thread (= page) order
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
  if (tid == kTopkThreads - 1) *sel_count = out_pos;
}

// Top-k of one stream, keys in registers (n <= kRegTopkMax).  Same result
// as topk_cta -- pins, then the best K-|pins| others by (score desc, index
// asc), ascending -- with far fewer block barriers: one shared 2048-bin
// histogram per 11-bit radix pass (random scores rarely collide, so no
// per-warp copies), double-buffered so zeroing the next one needs no extra
// barrier, the boundary bin found with one block scan (3 barriers per pass),
// and one packed scan (strict | equal counts) for the ordered compaction.
template <int KPT>
__device__ void topk_cta_reg(int n, int K, const double* scores, uint32_t* hist2, int32_t* sel_out,
                             int32_t* sel_count) {
  constexpr int NB = 1 << kRegTopkBits;
  constexpr int BPT = NB / kTopkThreads;  // bins per thread (8)
  __shared__ uint32_t wtot[kTopkWarps + 1];
  __shared__ uint64_t s_max[kTopkWarps], s_min[kTopkWarps];
  __shared__ uint32_t sh_bin, sh_kk, sh_done;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int pin[3];
  const int npins = pins_of(n, pin);
  const int kpt = (n + kTopkThreads - 1) / kTopkThreads;
  const int i0 = tid * kpt;
  uint64_t key[KPT];
  uint64_t kmax = 0, kmin = ~0ull;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const int i = i0 + j;
    key[j] = 0;
    if (j < kpt && i < n && !is_pin(i, n)) key[j] = order_key(__ldcg(scores + i));
    if (key[j]) {
      kmax = key[j] > kmax ? key[j] : kmax;
      kmin = key[j] < kmin ? key[j] : kmin;
    }
  }
  for (int b = tid; b < NB; b += kTopkThreads) hist2[b] = 0;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, kmax, off), c = __shfl_xor_sync(0xffffffffu, kmin, off);
    kmax = a > kmax ? a : kmax;
    kmin = c < kmin ? c : kmin;
  }
  if (lane == 0) {
    s_max[warp] = kmax;
    s_min[warp] = kmin;
  }
  __syncthreads();
  kmax = 0;
  kmin = ~0ull;
#pragma unroll
  for (int w = 0; w < kTopkWarps; ++w) {
    kmax = s_max[w] > kmax ? s_max[w] : kmax;
    kmin = s_min[w] < kmin ? s_min[w] : kmin;
  }
  uint32_t kk = K - npins;  // keys still to take at/below the current prefix
  // bits below `hi` are unresolved; the candidates agree on every bit above
  int hi = kmax == kmin ? 0 : 64 - __clzll(kmax ^ kmin);
  uint64_t mask = hi >= 64 ? 0ull : (~0ull << hi);
  uint64_t prefix = kmax & mask;
  int cur = 0;
  while (hi > 0) {
    const int w = hi < kRegTopkBits ? hi : kRegTopkBits;
    const int shift = hi - w;
    const uint32_t dm = (1u << w) - 1u;
    uint32_t* h = hist2 + cur * NB;
#pragma unroll
    for (int j = 0; j < KPT; ++j)
      if (key[j] && (key[j] & mask) == prefix) atomicAdd(&h[uint32_t(key[j] >> shift) & dm], 1u);
    uint32_t* hn = hist2 + (cur ^ 1) * NB;
    for (int b = tid; b < NB; b += kTopkThreads) hn[b] = 0;
    __syncthreads();  // A: histogram complete
    // thread t owns bins NB-1-BPT*t .. NB-BPT*(t+1), scanned from the top
    uint32_t loc[BPT], sum = 0;
#pragma unroll
    for (int e = 0; e < BPT; ++e) {
      loc[e] = h[NB - 1 - BPT * tid - e];
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
    for (int w2 = 0; w2 < kTopkWarps; ++w2) excl += w2 < warp ? wtot[w2] : 0u;
    if (excl < kk && kk <= excl + sum) {
      uint32_t cum = excl;
#pragma unroll
      for (int e = 0; e < BPT; ++e) {
        if (cum + loc[e] >= kk && cum < kk) {
          sh_bin = NB - 1 - BPT * tid - e;
          sh_kk = kk - cum;
          sh_done = loc[e] == kk - cum ? 1u : 0u;
        }
        cum += loc[e];
      }
    }
    __syncthreads();  // C: boundary bin published
    const uint32_t bin = sh_bin;
    kk = sh_kk;
    const bool done = sh_done;
    prefix |= (uint64_t)bin << shift;
    mask |= (uint64_t)dm << shift;
    hi = shift;
    cur ^= 1;
    if (done) break;  // every key of the boundary bin is taken
  }
  // ordered compaction: pins and keys above the prefix are taken; of the keys
  // equal to it, the kk lowest indices.  One scan of packed (taken | equal << 16).
  uint32_t n_take = 0, n_eq = 0;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const int i = i0 + j;
    if (j >= kpt || i >= n) continue;
    const uint64_t km = key[j] & mask;
    if (is_pin(i, n) || (key[j] && km > prefix)) ++n_take;
    else if (key[j] && km == prefix) ++n_eq;
  }
  uint32_t tot;
  const uint32_t ex = block_scan(n_take | (n_eq << 16), wtot, tot);
  uint32_t eq_rank = ex >> 16;
  uint32_t pos = (ex & 0xFFFFu) + (eq_rank < kk ? eq_rank : kk);
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const int i = i0 + j;
    if (j >= kpt || i >= n) continue;
    const uint64_t km = key[j] & mask;
    bool take = is_pin(i, n) || (key[j] && km > prefix);
    if (!take && key[j] && km == prefix) take = eq_rank++ < kk;
    if (take) sel_out[pos++] = i;
  }
  if (tid == kTopkThreads - 1) *sel_count = (tot & 0xFFFFu) + ((tot >> 16) < kk ? (tot >> 16) : kk);
}

template <typename T>
int select_dispatch(const PoolView& pv, int n_streams, const void* q, int64_t q_ss, int64_t q_rs,
                    const uint32_t* row_mask, const int32_t* tokens, const uint8_t* invoke, int K, int max_pages,
                    int32_t* sel_out, int32_t* sel_count, int sel_stride, double* scores, uint32_t* ticket,
                    cudaStream_t st) {
  const int LP = pv.P / pv.L;
  const int pps = LP >= SK_SEL_LOG_PER_SLOT ? 1 : SK_SEL_LOG_PER_SLOT / LP;  // pages per bulk copy
  const size_t slot = (size_t)pps * LP * 2 * pv.D * 2;
  size_t smem = 2 * kScoreWarps * slot;
  if (smem > 200 * 1024) {
    set_error("select: page/logical-page geometry needs too much shared memory");
    return SK_EUNSUPPORTED;
  }
  const int ppc = kScoreWarps * kBatchesPerWarp * pps;  // pages per CTA
  dim3 grid((max_pages + ppc - 1) / ppc, n_streams);
  const T* qt = static_cast<const T*>(q);
  // ablation builds for timing the phases (tools/decode_probe.py; never the shipped library):
  // -DSK_SEL_ABLATE=1 no scoring, 2 no top-k, 3 neither, 4 copies without scoring
#ifndef SK_SEL_ABLATE
#define SK_SEL_ABLATE 0
#endif
  const int dbg = SK_SEL_ABLATE;
#define SK_SEL(LPV)                                                                                          \
  do {                                                                                                       \
    cudaFuncSetAttribute(select_kernel<T, LPV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    select_kernel<T, LPV><<<grid, kScoreThreads, smem, st>>>(pv, qt, q_ss, q_rs, row_mask, tokens, invoke, K, \
                                                             scores, ticket, max_pages, pps, sel_out,         \
                                                             sel_count, sel_stride, (int)smem, dbg);          \
  } while (0)
  if (LP == 1) SK_SEL(1);
  else if (LP == 2) SK_SEL(2);
  else if (LP == 4) SK_SEL(4);
  else if (LP == 8) SK_SEL(8);
  else if (LP == 16) SK_SEL(16);
  else SK_SEL(32);
#undef SK_SEL
  SK_CHECK_LAUNCH("select_kernel");
  return SK_OK;
}

}  // namespace
}  // namespace sk

extern "C" int64_t sk_select_scores_offset(int32_t n_streams) { return ((int64_t)n_streams * 4 + 255) / 256 * 256; }

extern "C" int64_t sk_select_workspace(int32_t n_streams, int32_t max_pages) {
  return sk_select_scores_offset(n_streams) + (int64_t)n_streams * max_pages * 8;  // tickets + scores
}

extern "C" int sk_select_pages(const sk_pool* pool, int32_t n_streams, int32_t group_rows, const void* q,
                               int64_t q_stream_stride, int64_t q_row_stride, const uint32_t* row_mask,
                               const int32_t* tokens, const uint8_t* invoke, int32_t budget_pages,
                               int32_t max_pages_hint, int32_t* sel_out, int32_t* sel_count, int32_t sel_stride,
                               void* workspace, int64_t workspace_bytes, void* stream) {
  using namespace sk;
  int rc = check_pool(pool);
  if (rc) return rc;
  SK_CHECK_ARG(pool->stats != nullptr, "select: pool has no stats");
  SK_CHECK_ARG(n_streams >= 1 && n_streams <= 65535 && group_rows >= 1 && group_rows <= 32,
               "select: bad stream/row counts");
  SK_CHECK_ARG(budget_pages >= 1, "select: budget below one page");
  SK_CHECK_ARG(max_pages_hint >= 1 && max_pages_hint <= pool->max_pages, "select: bad max_pages_hint");
  SK_CHECK_ARG(sel_stride >= budget_pages || sel_stride >= max_pages_hint, "select: sel_stride too small");
  SK_CHECK_ARG(workspace_bytes >= sk_select_workspace(n_streams, max_pages_hint), "select: workspace too small");
  SK_CHECK_ARG(q && row_mask && tokens && sel_out && sel_count && workspace, "select: NULL pointer");
  SK_CHECK_ARG(reinterpret_cast<uintptr_t>(pool->stats) % 16 == 0, "select: stats must be 16-byte aligned");
  PoolView pv = make_view(*pool);
  // workspace = [tickets: n_streams x u32, padded to 256 B][scores: n_streams x max_pages_hint f64]; the
  // tickets sit at a fixed offset so one zeroed buffer serves any max_pages_hint it is large enough for
  uint32_t* ticket = static_cast<uint32_t*>(workspace);
  double* scores = reinterpret_cast<double*>(static_cast<uint8_t*>(workspace) + sk_select_scores_offset(n_streams));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (pool->dtype == SK_F16)
    return select_dispatch<__half>(pv, n_streams, q, q_stream_stride, q_row_stride, row_mask, tokens, invoke,
                                   budget_pages, max_pages_hint, sel_out, sel_count, sel_stride, scores, ticket, st);
  return select_dispatch<__nv_bfloat16>(pv, n_streams, q, q_stream_stride, q_row_stride, row_mask, tokens, invoke,
                                        budget_pages, max_pages_hint, sel_out, sel_count, sel_stride, scores, ticket,
                                        st);
}
