// K2 -- hierarchical page selection (LServe Eq. 2).
//
// Replaces score_pages / _stacked_stats / pinned_pages / select_pages
// (reference selector.py:39-108).  Two kernels:
//
// score_kernel (many CTAs per stream, HBM-bound).  Each warp owns
//   kPagesPerWarp physical pages; one lane issues a single 1-D bulk copy
//   (cp.async.bulk, mbarrier completion) of their contiguous (k_min, k_max)
//   rows into shared memory, so every byte of the selector's 33.6 MB at 128k
//   is requested in the first few hundred cycles of the CTA.  Each lane then
//   scores its D/32 channels of every logical page in fp64:
//       score(r, j) = sum_c q+_rc * kmax_jc + q-_rc * kmin_jc
//   (q+ = max(q,0), q- = min(q,0): one of the two products is exactly 0, so
//   each term equals the reference's max(q*kmax, q*kmin); fp16 products are
//   exact in fp64 and the sums are exact for fp16-valued inputs, matching
//   the reference's BLAS centre/radius form bit-for-bit -- SURVEY Appendix
//   A.4).  A multi-value butterfly reduces all (row, logical page) sums of
//   the warp at once; the physical-page score is their max over retrieval
//   rows and logical pages.  Only the stream's retrieval rows are computed
//   (RMAX = 1, 2 or 4 rows per pass).
//
// topk_kernel (one 1024-thread CTA per stream).  Radix select of the
//   (K - |pins|)-th largest score among non-pinned pages on the order-
//   preserving 64-bit image of the fp64 score, starting at the first byte
//   where the candidates' keys differ; ties go to the lower page index
//   (selector.py:106); union with the pins; ascending compaction by a
//   block-wide scan over page order.
#include <cstdlib>

#include "sk_common.cuh"
#include "sk_sm100.cuh"

namespace sk {
namespace {

constexpr int kScoreThreads = 256;
constexpr int kScoreWarps = kScoreThreads / 32;
constexpr int kPagesPerWarp = 4;
constexpr int kPagesPerCta = kScoreWarps * kPagesPerWarp;
constexpr int kTopkThreads = 1024;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kTopkStage = 8192;  // keys staged in shared memory (64 KB)

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

// Score the warp's pages for retrieval rows [rbase, rbase + RMAX) and fold
// them into best[].  LPC logical pages per butterfly pass (RMAX*LPC <= 16
// keeps two 256-thread CTAs resident per SM).
template <typename T, int RMAX, int LPC>
__device__ __forceinline__ void score_rows(const uint8_t* sbuf, int np, int lp_per, int n_log_rel, int D,
                                           const T* q, int64_t q_rs, uint32_t rmask, int rbase, int rows,
                                           double (&best)[kPagesPerWarp]) {
  constexpr int NV = RMAX * LPC;
  const int lane = threadIdx.x & 31;
  const int cpl = D / 32;  // channels per lane: 4 (D=128) or 2 (D=64)
  double qp[RMAX][4], qm[RMAX][4];
  {
    uint32_t mbits = rmask;
    for (int r = 0; r < rbase; ++r) mbits &= mbits - 1;
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      const int g = __ffs(mbits) - 1;
      const bool ok = rbase + r < rows && g >= 0;
      if (ok) mbits &= mbits - 1;
      const T* qr = q + (int64_t)(ok ? g : 0) * q_rs + lane * cpl;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double x = (ok && c < cpl) ? (double)DT<T>::to_f(qr[c]) : 0.0;
        qp[r][c] = x > 0.0 ? x : 0.0;
        qm[r][c] = x < 0.0 ? x : 0.0;
      }
    }
  }
  const int row_bytes = 2 * D * 2;  // (k_min, k_max) of one logical page
  for (int pi = 0; pi < np; ++pi) {
    for (int l0 = 0; l0 < lp_per; l0 += LPC) {
      double v[NV];
#pragma unroll
      for (int jj = 0; jj < LPC; ++jj) {
        const int lrel = pi * lp_per + l0 + jj;
        const T* st = reinterpret_cast<const T*>(sbuf + (int64_t)min(lrel, n_log_rel - 1) * row_bytes);
        uint2 wmin, wmax;
        if (cpl == 4) {
          wmin = *reinterpret_cast<const uint2*>(st + lane * 4);
          wmax = *reinterpret_cast<const uint2*>(st + D + lane * 4);
        } else {
          wmin = make_uint2(*reinterpret_cast<const uint32_t*>(st + lane * 2), 0u);
          wmax = make_uint2(*reinterpret_cast<const uint32_t*>(st + D + lane * 2), 0u);
        }
        double kmin[4], kmax[4];
        to_f64x4<T>(wmin, kmin);
        to_f64x4<T>(wmax, kmax);
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          double acc = 0.0;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            acc = fma(qp[r][c], kmax[c], acc);
            acc = fma(qm[r][c], kmin[c], acc);
          }
          v[r * LPC + jj] = acc;
        }
      }
      Butterfly<NV, 16>::run(v, lane);
      const int idx = lane >> (6 - __ffs(NV));  // value index owned by this lane
      const int r = idx / LPC, jj = idx % LPC;
      const bool valid = rbase + r < rows && l0 + jj < lp_per && pi * lp_per + l0 + jj < n_log_rel;
      double mine = valid ? v[0] : -INFINITY;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) mine = fmax(mine, __shfl_xor_sync(0xffffffffu, mine, off));
      best[pi] = fmax(best[pi], mine);
    }
  }
}

template <typename T, int LPC>
__global__ void __launch_bounds__(kScoreThreads, 2) score_kernel(PoolView pv, const T* __restrict__ q, int64_t q_ss,
                                                              int64_t q_rs, const uint32_t* __restrict__ row_mask,
                                                              const int32_t* __restrict__ tokens,
                                                              const uint8_t* __restrict__ invoke, int K,
                                                              double* ws_scores, int ws_pages) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar[kScoreWarps];
  const int s = blockIdx.y;
  if (invoke != nullptr && invoke[s] == 0) return;
  const uint32_t rmask = row_mask[s];
  if (rmask == 0) return;
  const int n_tok = tokens[s];
  const int P = pv.P, L = pv.L, D = pv.D, LP = P / L;
  const int n_pages = (n_tok + P - 1) / P;
  const int n_log = (n_tok + L - 1) / L;
  int pin[3];
  if (K >= n_pages || K <= pins_of(n_pages, pin)) return;  // trivial selection, no scores needed
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = (blockIdx.x * kScoreWarps + warp) * kPagesPerWarp;
  if (p0 >= n_pages) return;  // warp-level exit: nothing below synchronises the CTA
  const int np = min(kPagesPerWarp, n_pages - p0);
  const int lg0 = p0 * LP;
  const int nl = min(np * LP, n_log - lg0);  // valid logical pages of this warp
  const uint32_t row_bytes = 2 * D * 2;
  uint8_t* sbuf = smem + (size_t)warp * kPagesPerWarp * LP * row_bytes;
  if (lane == 0) {
    mbar_init(&bar[warp], 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(&bar[warp], nl * row_bytes);
    bulk_g2s(sbuf, pv.stats_ptr(s, lg0), nl * row_bytes, &bar[warp]);
  }
  __syncwarp();
  const T* qs = q + s * q_ss;
  const int rows = __popc(rmask);
  double best[kPagesPerWarp];
#pragma unroll
  for (int i = 0; i < kPagesPerWarp; ++i) best[i] = -INFINITY;
  mbar_wait(&bar[warp], 0);
  if (rows == 1) {
    score_rows<T, 1, (LPC < 16 ? LPC : 16)>(sbuf, np, LP, nl, D, qs, q_rs, rmask, 0, rows, best);
  } else if (rows == 2) {
    score_rows<T, 2, (LPC < 8 ? LPC : 8)>(sbuf, np, LP, nl, D, qs, q_rs, rmask, 0, rows, best);
  } else {
    for (int rb = 0; rb < rows; rb += 4)
      score_rows<T, 4, (LPC < 4 ? LPC : 4)>(sbuf, np, LP, nl, D, qs, q_rs, rmask, rb, rows, best);
  }
  if (lane < np) {
    double b = best[0];
#pragma unroll
    for (int i = 1; i < kPagesPerWarp; ++i)
      if (lane == i) b = best[i];
    ws_scores[(int64_t)s * ws_pages + p0 + lane] = b;
  }
}

// Block-wide exclusive scan of one value per thread (1024 threads) in thread
// order; returns the thread's exclusive prefix and the block total.
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
    const uint32_t t = warp_tot[lane];
    uint32_t ti = t;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, ti, off);
      if (lane >= off) ti += o;
    }
    warp_tot[lane] = ti - t;  // exclusive warp offsets
    if (lane == 31) warp_tot[32] = ti;
  }
  __syncthreads();
  const uint32_t res = warp_tot[warp] + incl - x;
  total = warp_tot[32];
  __syncthreads();
  return res;
}

__global__ void __launch_bounds__(kTopkThreads) topk_kernel(int P, const uint32_t* __restrict__ row_mask,
                                                            const int32_t* __restrict__ tokens,
                                                            const uint8_t* __restrict__ invoke, int K,
                                                            const double* __restrict__ ws_scores, int ws_pages,
                                                            int32_t* sel_out_all, int32_t* sel_count_all,
                                                            int sel_stride) {
  extern __shared__ uint64_t s_keys[];  // min(n, kTopkStage) keys
  __shared__ uint32_t hist[256];
  __shared__ uint32_t warp_tot[kTopkWarps + 1];
  __shared__ uint64_t s_max[kTopkWarps], s_min[kTopkWarps];
  __shared__ uint32_t sh_bin, sh_kk, sh_done;
  const int s = blockIdx.x;
  if (invoke != nullptr && invoke[s] == 0) return;
  if (row_mask[s] == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = (tokens[s] + P - 1) / P;
  int32_t* sel_out = sel_out_all + (int64_t)s * sel_stride;
  int32_t* sel_count = sel_count_all + s;
  int pin[3];
  const int npins = pins_of(n, pin);
  if (K >= n) {  // selector.py:98-100 -- every page, no scoring
    for (int i = tid; i < n; i += kTopkThreads) sel_out[i] = i;
    if (tid == 0) *sel_count = n;
    return;
  }
  if (K <= npins) {  // selector.py:101-103 -- pins only
    if (tid == 0) {
      for (int i = 0; i < npins; ++i) sel_out[i] = pin[i];
      *sel_count = npins;
    }
    return;
  }
  const double* scores = ws_scores + (int64_t)s * ws_pages;
  const bool staged = n <= kTopkStage;
  auto key_at = [&](int i) -> uint64_t {
    if (staged) return s_keys[i];
    return is_pin(i, n) ? 0ull : order_key(__ldcg(scores + i));
  };
  // keys + the candidates' max/min (to skip the leading bytes they share)
  uint64_t kmax = 0, kmin = ~0ull;
  for (int i = tid; i < n; i += kTopkThreads) {
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
  for (; shift >= 0; shift -= 8) {
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    for (int base = 0; base < n; base += kTopkThreads) {
      const int i = base + tid;
      bool live = false;
      uint32_t bin = 256u + lane;  // unique dummy bin for idle lanes
      if (i < n) {
        const uint64_t key = key_at(i);
        if (key && (key & mask) == prefix) {
          live = true;
          bin = uint32_t(key >> shift) & 255u;
        }
      }
      // warp-aggregated: one shared atomic per distinct bin per warp
      const uint32_t peers = __match_any_sync(0xffffffffu, bin);
      if (live && (__ffs(peers) - 1) == lane) atomicAdd(&hist[bin], uint32_t(__popc(peers)));
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
  // ordered compaction in chunks of 1024 consecutive page indices
  uint32_t eq_seen = 0, out_pos = 0;
  for (int base = 0; base < n; base += kTopkThreads) {
    const int i = base + tid;
    const bool valid = i < n;
    const bool pinned = valid && is_pin(i, n);
    const uint64_t key = valid ? key_at(i) : 0ull;
    const uint64_t km = key & mask;
    const bool cand = valid && !pinned && key != 0;
    const bool gt = cand && km > prefix;
    const bool eq = cand && km == prefix;
    uint32_t chunk_eq, chunk_take;
    const uint32_t before = eq_seen + block_scan(eq ? 1u : 0u, warp_tot, chunk_eq);
    const bool take = pinned || gt || (eq && (all_equal_taken || before < take_eq));
    const uint32_t pos = out_pos + block_scan(take ? 1u : 0u, warp_tot, chunk_take);
    if (take) sel_out[pos] = i;
    eq_seen += chunk_eq;
    out_pos += chunk_take;
  }
  if (tid == 0) *sel_count = out_pos;
}

template <typename T>
int select_dispatch(const PoolView& pv, int n_streams, const void* q, int64_t q_ss, int64_t q_rs,
                    const uint32_t* row_mask, const int32_t* tokens, const uint8_t* invoke, int K, int max_pages,
                    int32_t* sel_out, int32_t* sel_count, int sel_stride, double* scores, cudaStream_t st) {
  const int LP = pv.P / pv.L;
  const size_t smem = (size_t)kPagesPerCta * LP * 2 * pv.D * 2;
  if (smem > 200 * 1024) {
    set_error("select: page/logical-page geometry needs too much shared memory");
    return SK_EUNSUPPORTED;
  }
  dim3 grid((max_pages + kPagesPerCta - 1) / kPagesPerCta, n_streams);
  const T* qt = static_cast<const T*>(q);
  const int dbg = getenv("SK_SEL_DEBUG") ? atoi(getenv("SK_SEL_DEBUG")) : 0;  // temporary timing switch
  if (dbg != 2) {
#define SK_SCORE(LPV)                                                                                       \
  do {                                                                                                      \
    cudaFuncSetAttribute(score_kernel<T, LPV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    score_kernel<T, LPV><<<grid, kScoreThreads, smem, st>>>(pv, qt, q_ss, q_rs, row_mask, tokens, invoke, K, \
                                                            scores, max_pages);                              \
  } while (0)
  if (LP == 1) SK_SCORE(1);
  else if (LP == 2) SK_SCORE(2);
  else if (LP == 4) SK_SCORE(4);
  else if (LP == 8) SK_SCORE(8);
  else if (LP == 16) SK_SCORE(16);
  else SK_SCORE(32);
#undef SK_SCORE
  SK_CHECK_LAUNCH("score_kernel");
  }
  if (dbg == 1) return SK_OK;
  const int stage = max_pages < kTopkStage ? max_pages : kTopkStage;
  const size_t tsmem = (size_t)stage * 8;
  cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
  topk_kernel<<<n_streams, kTopkThreads, tsmem, st>>>(pv.P, row_mask, tokens, invoke, K, scores, max_pages, sel_out,
                                                      sel_count, sel_stride);
  SK_CHECK_LAUNCH("topk_kernel");
  return SK_OK;
}

}  // namespace
}  // namespace sk

extern "C" int64_t sk_select_workspace(int32_t n_streams, int32_t max_pages) {
  return (int64_t)n_streams * max_pages * 8 + 256;
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
  double* scores = static_cast<double*>(workspace);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (pool->dtype == SK_F16)
    return select_dispatch<__half>(pv, n_streams, q, q_stream_stride, q_row_stride, row_mask, tokens, invoke,
                                   budget_pages, max_pages_hint, sel_out, sel_count, sel_stride, scores, st);
  return select_dispatch<__nv_bfloat16>(pv, n_streams, q, q_stream_stride, q_row_stride, row_mask, tokens, invoke,
                                        budget_pages, max_pages_hint, sel_out, sel_count, sel_stride, scores, st);
}
