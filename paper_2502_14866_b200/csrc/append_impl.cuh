// Device-side page rebuild shared by K1 (append.cu) and K3's fused append
// (decode.cu).  See append.cu for the reference mapping.
#pragma once
#include "sk_common.cuh"
#include "sk_layout.cuh"

namespace sk {

__host__ __device__ inline size_t append_smem_bytes(int D, int P) {
  return (size_t)2 * P * D * 2 + 6 * D * sizeof(double) + 4 * D * sizeof(float);
}

// code = clip(round_half_even((x - lo) / scale), 0, levels), computed so the
// result equals numpy's fp64 np.round((x-lo)/scale) exactly: a multiply by
// the reciprocal is exact enough unless the quotient sits within 1e-9 of a
// .5 tie, in which case the correctly rounded division decides.
__device__ __forceinline__ uint32_t quant_code(double x, double lo, double scale, double inv, int levels) {
  double d = x - lo;  // exact: x, lo are fp16/bf16 values
  double t = d * inv;
  double r = rint(t);
  if (fabs(fabs(t - r) - 0.5) < 1e-9) r = rint(__ddiv_rn(d, scale));
  r = fmin(fmax(r, 0.0), double(levels));
  return uint32_t(r);
}
// The same code from an fp32 quotient: t32 = (x - lo) * (1/scale) in fp32 is
// within |t| * 2^-22 < 2^-14 of the fp64 quotient (t <= 255), so its rounding
// agrees with numpy's whenever t32 is farther than 2^-10 from a .5 tie; the
// (rare) near-tie quotients take the fp64 path above.
__device__ __forceinline__ uint32_t quant_code32(float x, float lo32, float inv32, double lo, double scale,
                                                 double inv, int levels) {
  const float t = (x - lo32) * inv32;
  const float r = rintf(t);
  if (fabsf(fabsf(t - r) - 0.5f) < 0x1p-10f) return quant_code((double)x, lo, scale, inv, levels);
  return (uint32_t)fminf(fmaxf(r, 0.f), (float)levels);
}

// The raw tokens of a partial last page (n1 % P != 0) -> the stream's staging
// rows, straight from the source (every tail token is new).  Whole CTA.
template <typename T>
__device__ void write_tail_from_src(const PoolView& pv, int s, int n0, int n1, const T* __restrict__ src_k,
                                    const T* __restrict__ src_v, int64_t src_ts) {
  constexpr int vec = 8;
  const int D = pv.D, P = pv.P;
  T* wk = reinterpret_cast<T*>(pv.staging_ptr(s, 0));
  T* wv = reinterpret_cast<T*>(pv.staging_ptr(s, 1));
  const int tail0 = (n1 - 1) / P * P;  // > n0
  for (int i = threadIdx.x; i < (n1 - tail0) * (D / vec); i += blockDim.x) {
    const int tl = i / (D / vec), c = (i % (D / vec)) * vec;
    const int64_t off = (int64_t)(tail0 + tl - n0) * src_ts + c;
    *reinterpret_cast<uint4*>(wk + tl * D + c) = *reinterpret_cast<const uint4*>(src_k + off);
    *reinterpret_cast<uint4*>(wv + tl * D + c) = *reinterpret_cast<const uint4*>(src_v + off);
  }
}

// Rebuild page p of stream s after tokens [n0, n1) were appended: raw page
// -> smem, bounds, codes (fragment-native layout, sk_layout.cuh), logical
// stats, staging.  Whole CTA.  src_k/src_v point at the stream's first new
// token.  Returns without work for streaming-pool pages this append evicts.
template <typename T>
__device__ void append_page(const PoolView& pv, int s, int p, int n0, int n1, const T* __restrict__ src_k,
                            const T* __restrict__ src_v, int64_t src_ts, uint8_t* smem) {
  const int D = pv.D, P = pv.P;
  const bool streaming = pv.kind[s] == SK_KIND_STREAMING;
  const int count = (n1 + P - 1) / P;
  constexpr int vec = 8;  // 16-byte vectors
  // The staging page holds the raw tokens of the stream's open page.  The
  // CTA of the first touched page (p_open) is the only one that reads it;
  // when the append ends in a different, partial page, that same CTA (not
  // the last page's) writes the new tail into staging once its own read is
  // done -- so no two CTAs of one launch touch staging unordered.
  const int p_open = n0 / P, p_last = (n1 - 1) / P;
  const bool tail_by_open = p == p_open && p_last != p_open && (n1 % P) != 0;
  auto write_tail_from_src = [&]() { sk::write_tail_from_src<T>(pv, s, n0, n1, src_k, src_v, src_ts); };
  if (streaming && p >= pv.sink && p < count - pv.local) {  // evicted by the end of this append
    if (tail_by_open) write_tail_from_src();
    return;
  }

  const int t0 = p * P;
  const int t1 = min(t0 + P, n1);
  const int ntok = t1 - t0;
  T* rk = reinterpret_cast<T*>(smem);                    // [P][D]
  T* rv = rk + P * D;                                    // [P][D]
  double* s_lo = reinterpret_cast<double*>(rv + P * D);  // [2][D]
  double* s_sc = s_lo + 2 * D;                           // [2][D]
  double* s_inv = s_sc + 2 * D;                          // [2][D]
  float* s_lo32 = reinterpret_cast<float*>(s_inv + 2 * D);  // [2][D]
  float* s_inv32 = s_lo32 + 2 * D;                           // [2][D]

  // 1. raw page -> smem (staging for positions < n0, new tokens otherwise)
  const T* stg_k = reinterpret_cast<const T*>(pv.staging_ptr(s, 0));
  const T* stg_v = reinterpret_cast<const T*>(pv.staging_ptr(s, 1));
  for (int i = threadIdx.x; i < ntok * (D / vec); i += blockDim.x) {
    int tl = i / (D / vec), c = (i % (D / vec)) * vec;
    int t = t0 + tl;
    uint4 kk, vv;
    if (t < n0) {
      kk = *reinterpret_cast<const uint4*>(stg_k + tl * D + c);
      vv = *reinterpret_cast<const uint4*>(stg_v + tl * D + c);
    } else {
      int64_t off = (int64_t)(t - n0) * src_ts + c;
      kk = *reinterpret_cast<const uint4*>(src_k + off);
      vv = *reinterpret_cast<const uint4*>(src_v + off);
    }
    *reinterpret_cast<uint4*>(rk + tl * D + c) = kk;
    *reinterpret_cast<uint4*>(rv + tl * D + c) = vv;
  }
  __syncthreads();
  if (tail_by_open) write_tail_from_src();  // staging reads of this CTA are complete

  uint8_t* slot = pv.slot_ptr(s, p);
  uint8_t* kc = pv.k_codes(slot);
  uint8_t* vc = pv.v_codes(slot);
  const int bits = pv.bits;
  if (bits > 0) {
    // 2. per-channel bounds for K (which=0) and V (which=1)
    T* bnd = reinterpret_cast<T*>(pv.bounds(slot));
    const int levels = (1 << bits) - 1;
    // channel pair (2q, 2q+1) of K (q < D/2) or V: 256/D threads split its
    // tokens, 32-bit loads, then a shuffle across those adjacent lanes
    {
      const int tpp = blockDim.x / D;  // threads per channel pair (2 at D = 128)
      const int pair = threadIdx.x / tpp, sp = threadIdx.x % tpp;
      const int which = pair / (D / 2), c = 2 * (pair % (D / 2));
      const T* raw = which ? rv : rk;
      float lo0 = INFINITY, hi0 = -INFINITY, lo1 = INFINITY, hi1 = -INFINITY;
      for (int t = sp; t < ntok; t += tpp) {
        const float2 x = DT<T>::to_f2(*reinterpret_cast<const uint32_t*>(raw + t * D + c));
        lo0 = fminf(lo0, x.x);
        hi0 = fmaxf(hi0, x.x);
        lo1 = fminf(lo1, x.y);
        hi1 = fmaxf(hi1, x.y);
      }
      for (int off = 1; off < tpp; off <<= 1) {
        lo0 = fminf(lo0, __shfl_xor_sync(0xffffffffu, lo0, off));
        hi0 = fmaxf(hi0, __shfl_xor_sync(0xffffffffu, hi0, off));
        lo1 = fminf(lo1, __shfl_xor_sync(0xffffffffu, lo1, off));
        hi1 = fmaxf(hi1, __shfl_xor_sync(0xffffffffu, hi1, off));
      }
      if (sp < 2) {
        const int ch = c + sp;
        const float lo = sp ? lo1 : lo0, hi = sp ? hi1 : hi0;
        const int i = which * D + ch;
        const int pos = which ? vbound_pos(ch, D) : kbound_pos(ch, D);
        bnd[(2 * which) * D + pos] = DT<T>::from_f(lo);  // exact: lo/hi are T values
        bnd[(2 * which + 1) * D + pos] = DT<T>::from_f(hi);
        double sc = ((double)hi - (double)lo) / levels;
        if (!(sc > 0.0)) sc = 1.0;
        s_lo[i] = lo;
        s_sc[i] = sc;
        s_inv[i] = 1.0 / sc;
        s_lo32[i] = lo;
        s_inv32[i] = (float)(1.0 / sc);
      }
    }
    __syncthreads();
    // 3. codes, written one 32-bit word at a time in the fragment-native
    //    layout (sk_layout.cuh); padding tokens of a partial page get code 0.
    auto code_at = [&](int which, int t, int c) -> uint32_t {
      if (t >= ntok) return 0u;
      const T* raw = which ? rv : rk;
      int i = which * D + c;
      return quant_code32(DT<T>::to_f(raw[t * D + c]), s_lo32[i], s_inv32[i], s_lo[i], s_sc[i], s_inv[i], levels);
    };
    uint32_t* kw = reinterpret_cast<uint32_t*>(kc);
    uint32_t* vw = reinterpret_cast<uint32_t*>(vc);
    if (bits <= 4) {
      // K: blockDim is a multiple of the D/8 words of a token, so a thread keeps
      // one (j, w) -- the same 8 dims (4 adjacent pairs) -- for every token it
      // codes: their (lo, 1/scale) stay in registers, raw values load as pairs
      const int kwords = P * D / 8, wpc = D / 32;  // words per (token, j) chunk
      {
        const int rem = threadIdx.x % (D / 8), j = rem / wpc, w = rem % wpc;
        int dp[4];
        float lo32[8], inv32[8];
#pragma unroll
        for (int slot = 0; slot < 4; ++slot) {
          const int ri = 4 * w + slot;
          dp[slot] = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            lo32[2 * slot + e] = s_lo32[dp[slot] + e];
            inv32[2 * slot + e] = s_inv32[dp[slot] + e];
          }
        }
        for (int wi = threadIdx.x; wi < kwords; wi += blockDim.x) {
          const int t = wi / (D / 8);
          uint32_t word = 0;
          if (t < ntok) {
#pragma unroll
            for (int slot = 0; slot < 4; ++slot) {
              const float2 x = DT<T>::to_f2(*reinterpret_cast<const uint32_t*>(rk + t * D + dp[slot]));
              const uint32_t c0 = quant_code32(x.x, lo32[2 * slot], inv32[2 * slot], s_lo[dp[slot]], s_sc[dp[slot]],
                                               s_inv[dp[slot]], levels);
              const uint32_t c1 = quant_code32(x.y, lo32[2 * slot + 1], inv32[2 * slot + 1], s_lo[dp[slot] + 1],
                                               s_sc[dp[slot] + 1], s_inv[dp[slot] + 1], levels);
              word |= (c0 << (4 * slot)) | (c1 << (4 * slot + 16));
            }
          }
          kw[wi] = word;
        }
      }
      // V: a thread codes whole (channel tile, lane) chunks -- one channel each
      const int vwpl = P / 32;  // words per (cn, lane)
      for (int cl = threadIdx.x; cl < (D / 8) * 32; cl += blockDim.x) {
        const int cn = cl / 32, lane = cl % 32;
        const int c = 8 * cn + lane / 4, j = lane % 4, i = D + c;
        const float lo = s_lo32[i], inv = s_inv32[i];
        for (int w = 0; w < vwpl; ++w) {
          uint32_t word = 0;
#pragma unroll
          for (int slot = 0; slot < 4; ++slot)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int ri = 4 * w + slot, t = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j + e;
              if (t < ntok)
                word |= quant_code32(DT<T>::to_f(rv[t * D + c]), lo, inv, s_lo[i], s_sc[i], s_inv[i], levels)
                        << (4 * slot + 16 * e);
            }
          vw[cl * vwpl + w] = word;
        }
      }
    } else {
      const int kwords = P * D / 4, wpc = D / 16;
      for (int wi = threadIdx.x; wi < kwords; wi += blockDim.x) {
        int t = wi / (D / 4), rem = wi % (D / 4), j = rem / wpc, w = rem % wpc;
        uint32_t word = 0;
#pragma unroll
        for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            int ri = 2 * w + r2, d = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j + e;
            word |= code_at(0, t, d) << (8 * (2 * r2 + e));
          }
        kw[wi] = word;
      }
      const int vwpl = P / 16;
      for (int wi = threadIdx.x; wi < kwords; wi += blockDim.x) {
        int cn = wi / (32 * vwpl), rem = wi % (32 * vwpl), lane = rem / vwpl, w = rem % vwpl;
        int c = 8 * cn + lane / 4, j = lane % 4;
        uint32_t word = 0;
#pragma unroll
        for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            int ri = 2 * w + r2, t = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j + e;
            word |= code_at(1, t, c) << (8 * (2 * r2 + e));
          }
        vw[wi] = word;
      }
    }
  } else {
    // raw pages: permuted copy of the page's tokens
    T* kr = reinterpret_cast<T*>(kc);
    T* vr = reinterpret_cast<T*>(vc);
    if (ntok < P) {
      for (int i = threadIdx.x; i < 2 * P * pv.row_bytes / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(kc)[i] = 0u;
      __syncthreads();
    }
    for (int i = threadIdx.x; i < ntok * D; i += blockDim.x) {
      int tl = i / D, c = i % D;
      kr[kpos_raw(tl, c, D)] = rk[tl * D + c];
      vr[vpos_raw(tl, c, P)] = rv[tl * D + c];
    }
  }
  // 4. logical-page key stats (dense pool only)
  if (!streaming && pv.stats != nullptr) {
    const int L = pv.L;
    const int nlog = (ntok + L - 1) / L;
    for (int i = threadIdx.x; i < nlog * D; i += blockDim.x) {
      int j = i / D, c = i % D;
      int a = j * L, b = min(a + L, ntok);
      float lo = DT<T>::to_f(rk[a * D + c]), hi = lo;
      for (int t = a + 1; t < b; ++t) {
        float x = DT<T>::to_f(rk[t * D + c]);
        lo = fminf(lo, x);
        hi = fmaxf(hi, x);
      }
      T* st = reinterpret_cast<T*>(pv.stats_ptr(s, p * (P / L) + j));
      st[c] = DT<T>::from_f(lo);
      st[D + c] = DT<T>::from_f(hi);
    }
  }
  // 5. a partial page at the end keeps its raw tokens in staging (written
  //    here only when it is also the open page; otherwise by p_open's CTA)
  if (t1 == n1 && (n1 % P) != 0 && p == p_open) {
    T* wk = reinterpret_cast<T*>(pv.staging_ptr(s, 0));
    T* wv = reinterpret_cast<T*>(pv.staging_ptr(s, 1));
    int first = max(n0, t0) - t0;
    for (int i = threadIdx.x; i < (ntok - first) * (D / vec); i += blockDim.x) {
      int tl = first + i / (D / vec), c = (i % (D / vec)) * vec;
      *reinterpret_cast<uint4*>(wk + tl * D + c) = *reinterpret_cast<const uint4*>(rk + tl * D + c);
      *reinterpret_cast<uint4*>(wv + tl * D + c) = *reinterpret_cast<const uint4*>(rv + tl * D + c);
    }
  }
}


// Decode-step append of ONE token to stream s holding n_tok tokens, for an
// open page that already holds t_old = n_tok % P > 0 tokens, split over the
// kAppendParts CTAs of a cluster (latency: one CTA per stream was a long
// serial chain).  Part q < 4 re-codes the K words of page tokens
// [q P/4, (q+1) P/4), part q >= 4 the V words of channels
// [(q-4) D/4, (q-3) D/4).  Every part recomputes the bounds it needs from the
// raw staging copy plus the new token and re-codes its words in full, so no
// code word is read back: bit-identical to append_page() (a full rebuild of
// the page, cache.py:211-251).  Part 0 also writes the K bounds, the open
// logical page's key stats and the K staging row; part 4 the V staging row.
constexpr int kAppendParts = 8;
__host__ __device__ inline size_t append_part_smem_bytes(int D, int P) {
  return (size_t)P * D * 2 + (size_t)2 * 256 * 4 + (size_t)3 * D * 8;
}

template <typename T>
__device__ void append_one_part(const PoolView& pv, int s, int part, int n_tok, const T* __restrict__ kn,
                                const T* __restrict__ vn, uint8_t* smem) {
  const int D = pv.D, P = pv.P;
  const int t_old = n_tok % P, p = n_tok / P, nt = t_old + 1;  // tokens in the page after the append
  const bool isv = part >= 4;
  const int q = part & 3;
  const int c0 = isv ? q * (D / 4) : 0, nc = isv ? D / 4 : D;  // channels this part needs
  const T* stg = reinterpret_cast<const T*>(pv.staging_ptr(s, isv ? 1 : 0));
  const T* xn = isv ? vn : kn;
  T* raw = reinterpret_cast<T*>(smem);                                // [nt][nc]
  float* pmin = reinterpret_cast<float*>(raw + (size_t)P * D);        // [256]
  float* pmax = pmin + 256;                                           // [256]
  double* lo = reinterpret_cast<double*>(pmax + 256);                 // [nc]
  double* sc = lo + D;
  double* inv = sc + D;
  const int levels = (1 << pv.bits) - 1;
  // 1. raw page (staging rows + the new token) -> smem, 16-byte vectors
  const int vpr = nc / 8;  // vectors per row
  for (int i = threadIdx.x; i < nt * vpr; i += blockDim.x) {
    const int t = i / vpr, c = (i % vpr) * 8;
    const T* src = t < t_old ? stg + (int64_t)t * D + c0 + c : xn + c0 + c;
    *reinterpret_cast<uint4*>(raw + t * nc + c) = *reinterpret_cast<const uint4*>(src);
  }
  __syncthreads();
  // 2. per-channel bounds over the page's tokens: 256 / nc token splits per channel
  {
    const int ns = 256 / nc, c = threadIdx.x % nc, sp = threadIdx.x / nc;
    float mn = INFINITY, mx = -INFINITY;
    if (sp < ns)
      for (int t = sp; t < nt; t += ns) {
        const float x = DT<T>::to_f(raw[t * nc + c]);
        mn = fminf(mn, x);
        mx = fmaxf(mx, x);
      }
    pmin[threadIdx.x] = mn;
    pmax[threadIdx.x] = mx;
    __syncthreads();
    if (threadIdx.x < nc) {
      for (int k = 1; k < ns; ++k) {
        mn = fminf(mn, pmin[k * nc + c]);
        mx = fmaxf(mx, pmax[k * nc + c]);
      }
      double scl = ((double)mx - (double)mn) / levels;
      if (!(scl > 0.0)) scl = 1.0;
      lo[c] = mn;
      sc[c] = scl;
      inv[c] = 1.0 / scl;
      if (isv || part == 0) {  // exact: lo/hi are T values
        T* bnd = reinterpret_cast<T*>(pv.bounds(pv.slot_ptr(s, p)));
        const int ch = c0 + c;
        const int pos = isv ? vbound_pos(ch, D) : kbound_pos(ch, D);
        bnd[(isv ? 2 : 0) * D + pos] = DT<T>::from_f(mn);
        bnd[(isv ? 3 : 1) * D + pos] = DT<T>::from_f(mx);
      }
    }
    __syncthreads();
  }
  auto code_at = [&](int t, int c) -> uint32_t {  // c relative to c0; padding tokens -> 0
    if (t >= nt) return 0u;
    return quant_code((double)DT<T>::to_f(raw[t * nc + c]), lo[c], sc[c], inv[c], levels);
  };
  // 3. this part's code words, fragment-native layout (sk_layout.cuh)
  uint8_t* slot = pv.slot_ptr(s, p);
  const bool nib = pv.bits <= 4;
  if (!isv) {
    uint32_t* kw = reinterpret_cast<uint32_t*>(pv.k_codes(slot));
    const int wpt = nib ? D / 8 : D / 4, wpc = nib ? D / 32 : D / 16;  // words per token / per (token, j)
    const int tq = P / 4, tfirst = q * tq;
    for (int wi = threadIdx.x; wi < tq * wpt; wi += blockDim.x) {
      const int t = tfirst + wi / wpt, rem = wi % wpt, j = rem / wpc, w = rem % wpc;
      uint32_t word = 0;
      if (nib) {
#pragma unroll
        for (int slt = 0; slt < 4; ++slt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int ri = 4 * w + slt, d = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j + e;
            word |= code_at(t, d) << (4 * slt + 16 * e);
          }
      } else {
#pragma unroll
        for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int ri = 2 * w + r2, d = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j + e;
            word |= code_at(t, d) << (8 * (2 * r2 + e));
          }
      }
      kw[t * wpt + rem] = word;
    }
  } else {
    uint32_t* vw = reinterpret_cast<uint32_t*>(pv.v_codes(slot));
    const int vwl = nib ? P / 32 : P / 16;  // words per (cn, lane)
    const int cn0 = c0 / 8, ncn = nc / 8;
    for (int wi = threadIdx.x; wi < ncn * 32 * vwl; wi += blockDim.x) {
      const int cnl = wi / (32 * vwl), rem = wi % (32 * vwl), lane = rem / vwl, w = rem % vwl;
      const int c = 8 * cnl + lane / 4, j = lane % 4;  // relative channel
      uint32_t word = 0;
      if (nib) {
#pragma unroll
        for (int slt = 0; slt < 4; ++slt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int ri = 4 * w + slt, t = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j + e;
            word |= code_at(t, c) << (4 * slt + 16 * e);
          }
      } else {
#pragma unroll
        for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int ri = 2 * w + r2, t = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j + e;
            word |= code_at(t, c) << (8 * (2 * r2 + e));
          }
      }
      vw[(cn0 + cnl) * 32 * vwl + rem] = word;
    }
  }
  // 4. part 0: key stats of the open logical page (dense pool); parts 0 / 4: the staging row
  if (part == 0 && pv.kind[s] == SK_KIND_DENSE && pv.stats != nullptr) {
    const int L = pv.L, jl = t_old / L;
    T* st = reinterpret_cast<T*>(pv.stats_ptr(s, p * (P / L) + jl));
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
      float mn = INFINITY, mx = -INFINITY;
      for (int t = jl * L; t < nt; ++t) {
        const float x = DT<T>::to_f(raw[t * nc + c]);
        mn = fminf(mn, x);
        mx = fmaxf(mx, x);
      }
      st[c] = DT<T>::from_f(mn);
      st[D + c] = DT<T>::from_f(mx);
    }
  }
  if ((part == 0 || part == 4) && t_old + 1 < P) {
    T* w = reinterpret_cast<T*>(pv.staging_ptr(s, isv ? 1 : 0));
    for (int c = threadIdx.x; c < D; c += blockDim.x) w[t_old * D + c] = xn[c];
  }
}

}  // namespace sk
