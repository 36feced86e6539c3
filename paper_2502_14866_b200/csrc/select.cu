// K2 -- hierarchical page selection (LServe Eq. 2).
//
// Replaces score_pages / _stacked_stats / pinned_pages / select_pages
// (reference selector.py:39-108).  Phase 1 (many CTAs per stream): one warp
// per physical page reads the (k_min, k_max) rows of its logical pages
// (coalesced, 8 B per lane), converts them to fp64 and accumulates
//     score(r, j) = sum_c q+_rc * kmax_jc + q-_rc * kmin_jc
// (q+ = max(q,0), q- = min(q,0): one of the two products is exactly 0, so
// each term equals the reference's max(q*kmax, q*kmin); fp16 products are
// exact in fp64 and the sums are exact for fp16-valued inputs, matching the
// reference's BLAS centre/radius form bit-for-bit -- Appendix A.4).  A
// multi-value butterfly reduces all (row, logical) sums at once; the page
// score is their max.  Phase 2 (the last CTA of each stream, found with an
// atomic ticket): radix select of the (K - |pins|)-th largest score among
// non-pinned pages, ties toward the lower page index (selector.py:106),
// union with the pins, ascending compaction.
#include "sk_common.cuh"

namespace sk {
namespace {

constexpr int kSelThreads = 256;
constexpr int kPagesPerWarp = 4;
constexpr int kPagesPerCta = (kSelThreads / 32) * kPagesPerWarp;

__device__ __forceinline__ int pins_of(int n, int* pin) {  // selector.py:75-78
  int c = 0;
  pin[c++] = 0;
  int a = n - 2 > 0 ? n - 2 : 0;
  if (a != 0) pin[c++] = a;
  if (n - 1 != 0 && n - 1 != a) pin[c++] = n - 1;
  return c;
}
__device__ __forceinline__ bool is_pin(int i, int n) { return i == 0 || i == n - 1 || i == (n - 2 > 0 ? n - 2 : 0); }

__device__ __forceinline__ uint64_t order_key(double x) {
  x = x + 0.0;  // -0.0 -> +0.0 (equal scores tie on the index, like Python's sort)
  uint64_t u = __double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

template <typename T>
__device__ __forceinline__ void load4(const T* p, double* out) {
  // 4 consecutive elements (8 bytes)
  uint2 w = *reinterpret_cast<const uint2*>(p);
  float2 a = DT<T>::to_f2(w.x), b = DT<T>::to_f2(w.y);
  out[0] = a.x;
  out[1] = a.y;
  out[2] = b.x;
  out[3] = b.y;
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

// Phase 1: physical page scores.  RMAX = max retrieval rows handled, LP = P/L.
template <typename T, int RMAX, int LP>
__device__ void score_pages_cta(const PoolView& pv, int s, int n_tok, const T* q, int64_t q_rs, uint32_t rmask,
                                double* scores) {
  constexpr int NV = RMAX * LP;  // power of two <= 32
  const int D = pv.D, L = pv.L, P = pv.P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_pages = (n_tok + P - 1) / P;
  const int n_log = (n_tok + L - 1) / L;
  const int cpl = D / 32;  // channels per lane: 4 (D=128) or 2 (D=64)
  // retrieval rows -> fp64 q+ / q- for this lane's channels
  double qp[RMAX][4], qm[RMAX][4];
  // retrieval row r = r-th set bit of rmask
  int rows = __popc(rmask) < RMAX ? __popc(rmask) : RMAX;
  uint32_t mbits = rmask;
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    int g = __ffs(mbits) - 1;
    if (r < rows) mbits &= mbits - 1;
    const T* qr = q + (int64_t)(g < 0 ? 0 : g) * q_rs + lane * cpl;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double x = (r < rows && c < cpl) ? (double)DT<T>::to_f(qr[c]) : 0.0;
      qp[r][c] = x > 0.0 ? x : 0.0;
      qm[r][c] = x < 0.0 ? x : 0.0;
    }
  }
  // each warp walks kPagesPerWarp pages; the next page's stats are loaded
  // while the current one is scored (register double buffer)
  uint2 wmin[2][LP], wmax[2][LP];
  auto load_page = [&](int p, int b) {
#pragma unroll
    for (int j = 0; j < LP; ++j) {
      const int lp = min(p * LP + j, n_log - 1);  // clamp: invalid entries are masked below
      const T* st = reinterpret_cast<const T*>(pv.stats_ptr(s, lp));
      if (cpl == 4) {
        wmin[b][j] = __ldcg(reinterpret_cast<const uint2*>(st + lane * 4));
        wmax[b][j] = __ldcg(reinterpret_cast<const uint2*>(st + D + lane * 4));
      } else {
        wmin[b][j] = make_uint2(__ldcg(reinterpret_cast<const uint32_t*>(st + lane * 2)), 0u);
        wmax[b][j] = make_uint2(__ldcg(reinterpret_cast<const uint32_t*>(st + D + lane * 2)), 0u);
      }
    }
  };
  const int p0 = blockIdx.x * kPagesPerCta + warp;
  constexpr int kStride = kSelThreads / 32;
  if (p0 < n_pages) load_page(p0, 0);
#pragma unroll
  for (int it = 0; it < kPagesPerWarp; ++it) {
    const int p = p0 + it * kStride;
    if (p >= n_pages) break;
    const int b = it & 1;
    if (it + 1 < kPagesPerWarp && p + kStride < n_pages) load_page(p + kStride, b ^ 1);
    double v[NV];
#pragma unroll
    for (int j = 0; j < LP; ++j) {
      float2 a0 = DT<T>::to_f2(wmin[b][j].x), a1 = DT<T>::to_f2(wmin[b][j].y);
      float2 b0 = DT<T>::to_f2(wmax[b][j].x), b1 = DT<T>::to_f2(wmax[b][j].y);
      const double kmin[4] = {a0.x, a0.y, a1.x, a1.y}, kmax[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc = fma(qp[r][c], kmax[c], acc);
          acc = fma(qm[r][c], kmin[c], acc);
        }
        v[r * LP + j] = acc;
      }
    }
    Butterfly<NV, 16>::run(v, lane);
    int idx = lane >> (5 - __ffs(NV) + 1);  // value index owned by this lane
    int r = idx / LP, j = idx % LP;
    double mine = (r < rows && p * LP + j < n_log) ? v[0] : -INFINITY;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) mine = fmax(mine, __shfl_xor_sync(0xffffffffu, mine, off));
    if (lane == 0) scores[p] = mine;
  }
}

// Phase 2: top-k of one stream (whole CTA).  `scores` may point to shared
// memory (staged) or global memory.
__device__ void topk_cta(const double* scores, int n, int K, int32_t* sel_out, int32_t* sel_count) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t sh_bin, sh_kk, sh_done, sh_base;
  __shared__ uint32_t warp_tot[kSelThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int pin[3];
  int npins = pins_of(n, pin);
  if (K >= n) {
    for (int i = tid; i < n; i += blockDim.x) sel_out[i] = i;
    if (tid == 0) *sel_count = n;
    return;
  }
  if (K <= npins) {
    if (tid == 0) {
      for (int i = 0; i < npins; ++i) sel_out[i] = pin[i];
      *sel_count = npins;
    }
    return;
  }
  const uint32_t want = K - npins;
  uint64_t prefix = 0, mask = 0;
  if (tid == 0) { sh_kk = want; sh_done = 0; }
  __syncthreads();
  for (int shift = 56; shift >= 0; shift -= 8) {
    hist[tid] = 0;  // kSelThreads == 256
    __syncthreads();
    // warp-aggregated: lanes holding the same bin elect one leader per bin,
    // so a pass where every key shares its top byte costs one shared atomic
    // per warp instead of n serialised ones on the same address
    for (int base = 0; base < n; base += blockDim.x) {
      const int i = base + tid;
      bool live = false;
      uint32_t bin = 256u + lane;  // unique dummy bin for inactive lanes
      if (i < n && !is_pin(i, n)) {
        const uint64_t key = order_key(scores[i]);
        if ((key & mask) == prefix) {
          live = true;
          bin = uint32_t(key >> shift) & 255u;
        }
      }
      const uint32_t peers = __match_any_sync(0xffffffffu, bin);
      if (live && (__ffs(peers) - 1) == lane) atomicAdd(&hist[bin], uint32_t(__popc(peers)));
    }
    __syncthreads();
    if (warp == 0) {
      // bins from the top: lane l covers bins 255-8l .. 248-8l
      uint32_t kk = sh_kk;
      uint32_t sum = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) sum += hist[255 - 8 * lane - b];
      uint32_t incl = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      uint32_t excl = incl - sum;
      uint32_t ballot = __ballot_sync(0xffffffffu, incl >= kk);
      int first = __ffs(ballot) - 1;
      if (lane == first) {
        uint32_t cum = excl;
        for (int b = 0; b < 8; ++b) {
          uint32_t h = hist[255 - 8 * lane - b];
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
    if (sh_done) break;
    __syncthreads();
  }
  const bool all_equal_taken = sh_done;  // every key matching the prefix is selected
  const uint32_t take_eq = sh_kk;        // else: this many keys == prefix, lowest index first
  // flags + ordered compaction, in chunks of blockDim.x indices
  uint32_t eq_seen = 0, out_pos = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    int i = base + tid;
    bool valid = i < n;
    bool pinned = valid && is_pin(i, n);
    uint64_t key = valid && !pinned ? order_key(scores[i]) : 0;
    uint64_t km = key & mask;
    bool gt = valid && !pinned && km > prefix;
    bool eq = valid && !pinned && km == prefix;
    // rank of eq among equal keys in index order
    uint32_t b_eq = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) warp_tot[warp] = __popc(b_eq);
    __syncthreads();
    uint32_t before = eq_seen;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    before += __popc(b_eq & ((1u << lane) - 1));
    uint32_t chunk_eq = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) chunk_eq += warp_tot[w];
    __syncthreads();
    bool take = pinned || gt || (eq && (all_equal_taken || before < take_eq));
    uint32_t b_take = __ballot_sync(0xffffffffu, take);
    if (lane == 0) warp_tot[warp] = __popc(b_take);
    __syncthreads();
    uint32_t pos = out_pos;
    for (int w = 0; w < warp; ++w) pos += warp_tot[w];
    pos += __popc(b_take & ((1u << lane) - 1));
    uint32_t chunk_take = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) chunk_take += warp_tot[w];
    if (take) sel_out[pos] = i;
    eq_seen += chunk_eq;
    out_pos += chunk_take;
    __syncthreads();
  }
  if (tid == 0) *sel_count = out_pos;
  (void)sh_base;
}

template <typename T, int RMAX, int LP>
__global__ void __launch_bounds__(kSelThreads) select_kernel(PoolView pv, const T* __restrict__ q, int64_t q_ss,
                                                             int64_t q_rs, const uint32_t* __restrict__ row_mask,
                                                             const int32_t* __restrict__ tokens,
                                                             const uint8_t* __restrict__ invoke, int K,
                                                             int32_t* sel_out, int32_t* sel_count, int sel_stride,
                                                             double* ws_scores, uint32_t* ws_ticket, int ws_pages,
                                                             int stage_smem) {
  const int s = blockIdx.y;
  if (invoke != nullptr && invoke[s] == 0) return;
  const uint32_t rmask = row_mask[s];
  if (rmask == 0) return;
  const int n_tok = tokens[s];
  const int n_pages = (n_tok + pv.P - 1) / pv.P;
  double* scores = ws_scores + (int64_t)s * ws_pages;
  int pin[3];
  const bool trivial = K >= n_pages || K <= pins_of(n_pages, pin);
  if (!trivial) score_pages_cta<T, RMAX, LP>(pv, s, n_tok, q + s * q_ss, q_rs, rmask, scores);
  // last CTA of this stream runs the top-k
  __shared__ uint32_t is_last;
  // CTA ticket: bar.sync orders the CTA's score stores before thread 0's
  // acq_rel fence + relaxed atomic (the release pattern of CUTLASS's
  // generic barrier; a seq_cst __threadfence per CTA serialises the grid)
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    uint32_t t = atomicAdd(ws_ticket + s, 1u);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    is_last = (t == gridDim.x - 1);
    if (is_last) ws_ticket[s] = 0;  // re-arm for the next invocation
  }
  __syncthreads();
  if (!is_last) return;
  extern __shared__ double s_scores[];
  const double* src = scores;
  if (stage_smem && !trivial) {
    for (int i = threadIdx.x; i < n_pages; i += blockDim.x) s_scores[i] = __ldcg(scores + i);
    __syncthreads();
    src = s_scores;
  }
  topk_cta(src, n_pages, K, sel_out + (int64_t)s * sel_stride, sel_count + s);
}

template <typename T>
int select_dispatch(const PoolView& pv, int n_streams, int group_rows, const void* q, int64_t q_ss, int64_t q_rs,
                    const uint32_t* row_mask, const int32_t* tokens, const uint8_t* invoke, int K, int max_pages,
                    int32_t* sel_out, int32_t* sel_count, int sel_stride, double* scores, uint32_t* ticket,
                    cudaStream_t st) {
  const int LP = pv.P / pv.L;
  dim3 grid((max_pages + kPagesPerCta - 1) / kPagesPerCta, n_streams);
  const T* qt = static_cast<const T*>(q);
  const size_t smem = (size_t)max_pages * 8;
  const int stage = smem <= 160 * 1024 ? 1 : 0;
#define SK_SEL(R, LPV)                                                                                         \
  do {                                                                                                         \
    if (stage)                                                                                                 \
      cudaFuncSetAttribute(select_kernel<T, R, LPV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    select_kernel<T, R, LPV><<<grid, kSelThreads, stage ? smem : 0, st>>>(                                    \
        pv, qt, q_ss, q_rs, row_mask, tokens, invoke, K, sel_out, sel_count, sel_stride, scores, ticket,       \
        max_pages, stage);                                                                                     \
  } while (0)
  int rows = group_rows;
  if (LP == 4 && rows <= 4) SK_SEL(4, 4);
  else if (LP == 4 && rows <= 8) SK_SEL(8, 4);
  else if (LP == 1 && rows <= 8) SK_SEL(8, 1);
  else if (LP == 2 && rows <= 8) SK_SEL(8, 2);
  else if (LP == 8 && rows <= 4) SK_SEL(4, 8);
  else if (LP == 16 && rows <= 2) SK_SEL(2, 16);
  else if (LP == 32 && rows <= 1) SK_SEL(1, 32);
  else {
    set_error("select: unsupported (group rows, P/L) combination");
    return SK_EUNSUPPORTED;
  }
#undef SK_SEL
  SK_CHECK_LAUNCH("select_kernel");
  return SK_OK;
}

}  // namespace
}  // namespace sk

extern "C" int64_t sk_select_workspace(int32_t n_streams, int32_t max_pages) {
  return (int64_t)n_streams * max_pages * 8 + (int64_t)n_streams * 4 + 256;
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
  SK_CHECK_ARG(n_streams >= 1 && group_rows >= 1 && group_rows <= 32, "select: bad stream/row counts");
  SK_CHECK_ARG(budget_pages >= 1, "select: budget below one page");
  SK_CHECK_ARG(max_pages_hint >= 1 && max_pages_hint <= pool->max_pages, "select: bad max_pages_hint");
  SK_CHECK_ARG(sel_stride >= budget_pages || sel_stride >= max_pages_hint, "select: sel_stride too small");
  SK_CHECK_ARG(workspace_bytes >= sk_select_workspace(n_streams, max_pages_hint), "select: workspace too small");
  SK_CHECK_ARG(q && row_mask && tokens && sel_out && sel_count && workspace, "select: NULL pointer");
  PoolView pv = make_view(*pool);
  double* scores = static_cast<double*>(workspace);
  uint32_t* ticket = reinterpret_cast<uint32_t*>(scores + (int64_t)n_streams * max_pages_hint);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (pool->dtype == SK_F16)
    return select_dispatch<__half>(pv, n_streams, group_rows, q, q_stream_stride, q_row_stride, row_mask, tokens,
                                   invoke, budget_pages, max_pages_hint, sel_out, sel_count, sel_stride, scores,
                                   ticket, st);
  return select_dispatch<__nv_bfloat16>(pv, n_streams, group_rows, q, q_stream_stride, q_row_stride, row_mask,
                                        tokens, invoke, budget_pages, max_pages_hint, sel_out, sel_count,
                                        sel_stride, scores, ticket, st);
}
