/*
 * sparsekv_b200.h -- C ABI of the B200 (sm_100a) LServe sparse-attention hot path.
 *
 * The reference (`sparsekv`, /root/reference/pkg/src/sparsekv) is a pure
 * Python/numpy package with no FFI; its drop-in boundary is the Python API
 * in __init__.py:23-56.  This header is the native layer *beneath* that API:
 * the host package `paper_2502_14866_b200` (same names, same argument
 * meaning and errors as the reference) binds these entry points with
 * ctypes.  Each entry point cites the reference computation it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every pointer argument documented as
 *    "device" is a CUDA device pointer; `stream` is a cudaStream_t (NULL =
 *    legacy default stream).  All calls are asynchronous and stream-ordered.
 *  - The library never allocates device memory: callers pass buffers and
 *    workspaces (the required workspace size is returned by the *_workspace
 *    query functions).
 *  - Return value: SK_OK (0) or a negative status; sk_last_error() returns
 *    a thread-local message for the last failure.
 *  - A "stream" of the KV store (not to be confused with a CUDA stream) is
 *    one (sequence, KV head) pair: index s = seq * n_kv_heads + kv_head.
 */
#ifndef SPARSEKV_B200_H
#define SPARSEKV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SK_OK 0
#define SK_EINVAL (-1)       /* invalid argument / shape -> ValueError */
#define SK_ECUDA (-2)        /* CUDA launch or runtime error -> RuntimeError */
#define SK_EUNSUPPORTED (-3) /* valid but unsupported on this build/device */

#define SK_F16 0
#define SK_BF16 1
#define SK_F32 2

#define SK_KIND_DENSE 0     /* dense pool: keeps every page, carries key stats */
#define SK_KIND_STREAMING 1 /* streaming pool: keeps sink + local pages only */

/*
 * Paged KV store of one attention layer (possibly many sequences).
 * Replaces cache.py:143-329 (HeadPages / TwoWayCache / PhysicalPage /
 * PageTable / PageStats) with device-resident pools.
 *
 * Arena slot layout (slot_bytes = sk_slot_bytes(...)):
 *   [0, P*R)        K codes, one row of R bytes per token
 *   [P*R, 2*P*R)    V codes
 *   [2*P*R, +8*D)   bits>0 only: k_lo[D], k_hi[D], v_lo[D], v_hi[D] in `dtype`
 * where R = D/2 (bits<=4, two codes per byte, channel 2j in the low nibble
 * of byte j), D (5<=bits<=8, one byte per code) or 2*D (bits=0: raw values).
 * scale = (hi-lo)/(2^bits-1) (1 where hi==lo) and zero = lo reproduce the
 * reference's per-page, per-channel quantiser (cache.py:20-51) exactly,
 * because lo/hi are min/max of values that are exact in `dtype`.
 */
typedef struct sk_pool {
  int32_t dtype;             /* SK_F16 or SK_BF16: raw K/V, bounds, stats, staging */
  int32_t head_dim;          /* D (padded: 64 or 128) */
  int32_t page_size;         /* physical page P (tokens), <= 128 */
  int32_t logical_page;      /* logical page L, divides P */
  int32_t bits;              /* 0 = raw pages, 2..8 = KV-b codes */
  int32_t max_pages;         /* page-table row width per stream */
  int32_t sink;              /* streaming window: sink pages (heads.py:107-125) */
  int32_t local;             /* streaming window: local pages */
  int64_t slot_bytes;        /* bytes per arena slot */
  void* arena;               /* device [n_slots][slot_bytes] */
  const int32_t* page_table; /* device [n_streams][max_pages]: page index -> arena slot (-1 none) */
  void* stats;               /* device [n_streams][max_pages*P/L][2][D]: (k_min, k_max) per logical page */
  void* staging;             /* device [n_streams][2][P][D]: raw K, V of each stream's open page */
  const uint8_t* kind;       /* device [n_streams]: SK_KIND_DENSE / SK_KIND_STREAMING */
} sk_pool;

/* Library identity and health. */
const char* sk_version(void);
const char* sk_last_error(void);
/* 1 if device `dev` is an sm_100 part this build can run on, else 0. */
int sk_device_supported(int dev);
/* Bytes per arena slot for a pool geometry. */
int64_t sk_slot_bytes(int32_t head_dim, int32_t page_size, int32_t bits, int32_t dtype);

/*
 * K1 -- append m tokens to every stream (bulk prefill ingest or one decode
 * token).  Replaces HeadPages.append -> _rebuild_open_page -> quantize_page
 * + PageStats.from_keys -> _evict_outside_window (cache.py:189-261).
 * For each stream s and each page touched by tokens [tokens[s], tokens[s]+m):
 * rebuilds the page from the raw open-page staging plus the new tokens,
 * recomputes lo/hi, codes (fp64 round-half-even, bit-exact with numpy) and,
 * for dense streams, the logical-page (k_min, k_max); stores the raw tail
 * of a partial last page in staging.  Streaming-pool pages that the append
 * would evict are skipped.  Afterwards tokens[s] += m.
 *   k_src/v_src: device, element (s, t, c) at src + s*src_stream_stride +
 *                t*src_token_stride + c, in pool->dtype.
 *   tokens:      device [n_streams] token counts before the append (updated).
 *   max_pages_touched: upper bound on pages one stream touches (host-known).
 * Caller guarantees page_table[s][p] is set for every touched page p.
 */
int sk_append_pages(const sk_pool* pool, int32_t n_streams, const void* k_src, const void* v_src,
                    int64_t src_stream_stride, int64_t src_token_stride, int32_t* tokens, int32_t m_tokens,
                    int32_t max_pages_touched, void* stream);

/*
 * K1, decode step: one new token for every stream of n_layers pools that share
 * dtype, head_dim, page_size and bits, in ONE launch (the appends of several
 * layers of a decode step).  Layer l: pools[l] (host array), tokens[l] (host
 * array of device counters, advanced by one); k / v of layer l, stream s at
 * k_src / v_src + l*src_layer_stride + s*src_stream_stride (elements).  Same
 * result as n_layers sk_append_pages(..., m_tokens = 1, ...) calls.
 */
int sk_append_token_layers(const sk_pool* pools, int32_t n_layers, int32_t n_streams, const void* k_src,
                           const void* v_src, int64_t src_layer_stride, int64_t src_stream_stride,
                           int32_t* const* tokens, void* stream);

/*
 * K1b -- pool gather (chunked prefill).  Dequantises the resident pages of
 * streams [0, n_streams) (first n_tokens tokens, every stream holds that
 * many) into a token-major history: element (s, t, c) of K / V at
 * k_out / v_out + t*out_token_stride + s*out_stream_stride + c, in
 * pool->dtype, value code*scale + lo (PhysicalPage.dequantize,
 * cache.py:54-56 / :97-102, cast to the attention dtype as engine.py:250-262
 * does); raw pools (bits 0) are copied.  Evicted pages of streaming streams
 * are not written.  No reference entry point: the reference has no
 * continued prefill; this is the device half of Engine.prefill_chunk.
 */
int sk_gather_pages(const sk_pool* pool, int32_t n_streams, int32_t n_tokens, void* k_out, void* v_out,
                    int64_t out_stream_stride, int64_t out_token_stride, void* stream);

/* Launch flags (sk_select_pages / sk_decode_attn). */
#define SK_DECODE_APPEND 1u    /* decode: append the new token behind the attention */
#define SK_LAUNCH_PDL 2u       /* programmatic dependent launch (see each entry point) */
#define SK_DECODE_SEL_READY 4u /* decode: the selection predates the previous kernel */

/*
 * K2 -- hierarchical page selection (Eq. 2).  Replaces
 * score_pages / select_pages / pinned_pages (selector.py:39-108) and the
 * call site engine.py:237-255.  For every stream with invoke[s] != 0 and a
 * non-zero retrieval row mask: scores every logical page as
 * sum_c max(q_c*kmax_c, q_c*kmin_c), takes the max over the retrieval rows
 * and over the logical pages of each physical page, then selects
 * K = budget_pages pages: all pages if K >= n; the pins {0, n-2, n-1} if
 * K <= |pins|; else pins + the best K-|pins| others ordered by
 * (score desc, page index asc).  Output is ascending.  The ranking is the
 * reference's fp64 one, bit for bit: every page is scored on the tensor
 * cores in fp32 with a rigorous error bound, and the pages whose bound
 * straddles the K-th score are rescored exactly in fp64.
 *   q:         device; row r of stream s at q + s*q_stream_stride + r*q_row_stride.
 *   row_mask:  device [n_streams] bit r set = group row r (< group_rows <= 32) is a retrieval row.
 *   tokens:    device [n_streams] tokens currently in each stream.
 *   invoke:    device [n_streams] (NULL = all).
 *   sel_out:   device [n_streams][sel_stride] ascending page indices.
 *   sel_count: device [n_streams].
 *   max_pages_hint: >= ceil(max tokens / P), sizes the grid.
 *   flags: SK_LAUNCH_PDL launches as a programmatic dependent of the previous kernel on
 *          the stream (CUDA-graph decode): stats, tokens, row masks and invoke flags are
 *          read before the dependency wait, so the previous kernel must not write them;
 *          q after it.
 */
/* Workspace bytes: [u32 ticket per stream, padded to 256 B | (f32 score,
 * f32 error bound) per (stream, page < max_pages) | f64 scratch per (stream,
 * page)].  Zero it once; the kernel re-arms its tickets, so one buffer serves
 * every launch with a max_pages_hint it fits.  The (score, bound) pairs of
 * the last launch start at sk_select_scores_offset(n). */
int64_t sk_select_workspace(int32_t n_streams, int32_t max_pages);
int64_t sk_select_scores_offset(int32_t n_streams);
int sk_select_pages(const sk_pool* pool, int32_t n_streams, int32_t group_rows, const void* q,
                    int64_t q_stream_stride, int64_t q_row_stride, const uint32_t* row_mask,
                    const int32_t* tokens, const uint8_t* invoke, int32_t budget_pages, int32_t max_pages_hint,
                    int32_t* sel_out, int32_t* sel_count, int32_t sel_stride, void* workspace,
                    int64_t workspace_bytes, uint32_t flags, void* stream);

/*
 * score_pages (selector.py:39-72): the exact fp64 physical-page score of
 * every page p < min(ceil(tokens[s]/P), out_stride) of every stream, max over
 * the retrieval rows of row_mask[s] (-inf for a stream without one), into
 * scores_out[s*out_stride + p].  Same arithmetic as K2's exact rescoring.
 */
int sk_score_pages(const sk_pool* pool, int32_t n_streams, int32_t group_rows, const void* q,
                   int64_t q_stream_stride, int64_t q_row_stride, const uint32_t* row_mask,
                   const int32_t* tokens, double* scores_out, int32_t out_stride, void* stream);

/*
 * K3 -- split-KV decode attention over the selected pages.  Replaces the
 * per-head page loop of Engine.decode_step (engine.py:257-281) with
 * PhysicalPage.dequantize (cache.py:97-102) and merge_block
 * (attn.py:191-229).  Per stream, group row r attends: the stream's
 * selection (retrieval rows, bit r of row_mask[s] set) or the sink+local
 * window of the current page count (streaming rows, streaming_schedule at
 * qt = page_count - 1, heads.py:107-125), then the raw new token
 * in-register.  Pages are dequantised on the fly; the union of the
 * stream's pages is cut into 32-token units spread over several CTAs, whose
 * partials are merged with log-sum-exp by the stream's last CTA.
 *   row_window: device [n_streams][group_rows] u32 = sink_blocks | local_blocks << 16
 *               of each streaming row (its HeadProfile), or NULL for the pool's window.
 *               A streaming-pool stream only holds the pool's window: the caller must
 *               not ask for more (the reference raises "evicted" there).
 *   flags: SK_DECODE_APPEND appends k_new/v_new (K1, one token) right behind the
 *          attention on the same stream (a second launch) and increments tokens[s];
 *          SK_LAUNCH_PDL launches as a programmatic dependent of the previous kernel on
 *          the stream (CUDA-graph decode): the pool, tokens and page table -- and, with
 *          SK_DECODE_SEL_READY, the selection -- are read before the dependency wait, so
 *          the previous kernel must not write them; q / k_new / v_new are read after it.
 *   out: element (s, r, c) at out + s*out_stream_stride + r*out_row_stride + c, type out_dtype.
 *   workspace: device, >= sk_decode_workspace(n_streams, group_rows, head_dim) bytes,
 *              zeroed once (tickets re-arm themselves); launches that share one
 *              workspace must be stream-ordered.  Page size: a multiple of 32.
 */
int64_t sk_decode_workspace(int32_t n_streams, int32_t group_rows, int32_t head_dim);
int sk_decode_attn(const sk_pool* pool, int32_t n_streams, int32_t group_rows, const void* q,
                   int64_t q_stream_stride, int64_t q_row_stride, const void* k_new, const void* v_new,
                   int64_t new_stream_stride, const uint32_t* row_mask, const uint32_t* row_window,
                   const int32_t* sel, const int32_t* sel_count, int32_t sel_stride, int32_t* tokens,
                   float softmax_scale, void* out, int64_t out_stream_stride, int64_t out_row_stride,
                   int32_t out_dtype, uint32_t flags, void* workspace, int64_t workspace_bytes,
                   void* stream);

/*
 * K4 -- block-sparse causal prefill attention on tcgen05 tensor cores.
 * Replaces blockwise_attention (attn.py:245-324) driven by Engine.prefill's
 * schedules (engine.py:152-168).  q [n_q][n_heads][D], k/v [n_kv][n_kv_heads][D]
 * token-major (device, `dtype`), out like q.  Query row i sees key columns
 * <= n_kv - n_q + i.  Each work item is one 256-row query block of one head
 * (four of the reference's 64-row query tiles, computed as two 128-row
 * tensor-core tiles sharing one K/V stream) and a list of segments of
 * consecutive 64-key blocks; the host builds items and segments from the
 * per-(head, query tile) schedules (the paper's block iterator,
 * PAPER.md:296-297) and orders items heaviest first.
 *
 * Segment = 3 x uint32: { first_block, count | flags << 24, mask_base } with
 *   flags bits 0..3: query rows [64q, 64q+64) of the item (quarter q) attend
 *                    these key blocks
 *   flags bit 4:     apply the element-wise causal mask (column > row position)
 *   flags bit 5:     explicit per-row column masks: block first_block+i uses
 *                    row_masks[(mask_base + i) * 256 + row] (bit c = column c
 *                    allowed; generic tile sizes).
 */
typedef struct sk_prefill_item {
  int32_t head;      /* query head */
  int32_t row0;      /* first query row of the 256-row block */
  int32_t seg_begin; /* first segment (index into segs, in units of segments) */
  int32_t seg_count; /* number of segments */
} sk_prefill_item;

int sk_prefill_attn(int32_t dtype, const void* q, const void* k, const void* v, void* out, int32_t n_q,
                    int32_t n_kv, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim, float softmax_scale,
                    const sk_prefill_item* items, int32_t n_items, const uint32_t* segs,
                    const uint64_t* row_masks, void* stream);

/*
 * K4 over the page pool (chunked prefill): the same attention
 * as sk_prefill_attn on an (n_q, hist_tokens + n_q) plan, with keys
 * [0, hist_tokens) read from the pool's KV4 pages through its page table
 * (stream = KV head), dequantised by producer warps straight into the
 * kernel's shared-memory K/V tiles -- code * scale + lo in fp32 rounded to
 * the pool dtype, the values PhysicalPage.dequantize casts to the attention
 * dtype (cache.py:97-102, engine.py:250-262) -- and keys [hist_tokens, +n_q)
 * from the chunk's raw k_chunk / v_chunk [n_q][n_kv_heads][head_dim].  No
 * history buffer is materialised.  q / out [n_q][n_heads][head_dim] in the
 * pool dtype.  Pools with <= 4-bit codes and page size 32 or 64.
 */
int sk_prefill_attn_paged(const sk_pool* pool, int32_t n_kv_heads, int32_t hist_tokens, const void* q,
                          const void* k_chunk, const void* v_chunk, void* out, int32_t n_q, int32_t n_heads,
                          float softmax_scale, const sk_prefill_item* items, int32_t n_items,
                          const uint32_t* segs, const uint64_t* row_masks, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEKV_B200_H */
