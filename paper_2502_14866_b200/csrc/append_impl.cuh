// Device-side page rebuild shared by K1 (append.cu) and K3's fused append
// (decode.cu).  See append.cu for the reference mapping.
#pragma once
#include "sk_common.cuh"
#include "sk_layout.cuh"

namespace sk {

__host__ __device__ inline size_t append_one_smem_bytes(int D, int P) {
  return (size_t)2 * D * (4 + 3 * 8) + ((2 * D + 15) & ~15) + (size_t)2 * P * D * 2;
}
__host__ __device__ inline size_t append_smem_bytes(int D, int P) {
  return (size_t)2 * P * D * 2 + 6 * D * sizeof(double);
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
  auto write_tail_from_src = [&]() {
    T* wk = reinterpret_cast<T*>(pv.staging_ptr(s, 0));
    T* wv = reinterpret_cast<T*>(pv.staging_ptr(s, 1));
    const int tail0 = p_last * P;  // > n0: every tail token is new
    for (int i = threadIdx.x; i < (n1 - tail0) * (D / vec); i += blockDim.x) {
      const int tl = i / (D / vec), c = (i % (D / vec)) * vec;
      const int64_t off = (int64_t)(tail0 + tl - n0) * src_ts + c;
      *reinterpret_cast<uint4*>(wk + tl * D + c) = *reinterpret_cast<const uint4*>(src_k + off);
      *reinterpret_cast<uint4*>(wv + tl * D + c) = *reinterpret_cast<const uint4*>(src_v + off);
    }
  };
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
    for (int i = threadIdx.x; i < 2 * D; i += blockDim.x) {
      int which = i / D, c = i % D;
      const T* raw = which ? rv : rk;
      float lo = DT<T>::to_f(raw[c]), hi = lo;
      for (int t = 1; t < ntok; ++t) {
        float x = DT<T>::to_f(raw[t * D + c]);
        lo = fminf(lo, x);
        hi = fmaxf(hi, x);
      }
      int pos = which ? vbound_pos(c, D) : kbound_pos(c, D);
      bnd[(2 * which) * D + pos] = DT<T>::from_f(lo);  // exact: lo/hi are T values
      bnd[(2 * which + 1) * D + pos] = DT<T>::from_f(hi);
      double sc = ((double)hi - (double)lo) / levels;
      if (!(sc > 0.0)) sc = 1.0;
      s_lo[i] = lo;
      s_sc[i] = sc;
      s_inv[i] = 1.0 / sc;
    }
    __syncthreads();
    // 3. codes, written one 32-bit word at a time in the fragment-native
    //    layout (sk_layout.cuh); padding tokens of a partial page get code 0.
    auto code_at = [&](int which, int t, int c) -> uint32_t {
      if (t >= ntok) return 0u;
      const T* raw = which ? rv : rk;
      int i = which * D + c;
      return quant_code((double)DT<T>::to_f(raw[t * D + c]), s_lo[i], s_sc[i], s_inv[i], levels);
    };
    uint32_t* kw = reinterpret_cast<uint32_t*>(kc);
    uint32_t* vw = reinterpret_cast<uint32_t*>(vc);
    if (bits <= 4) {
      const int kwords = P * D / 8, wpc = D / 32;  // words per (token, j) chunk
      for (int wi = threadIdx.x; wi < kwords; wi += blockDim.x) {
        int t = wi / (D / 8), rem = wi % (D / 8), j = rem / wpc, w = rem % wpc;
        uint32_t word = 0;
#pragma unroll
        for (int slot = 0; slot < 4; ++slot)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            int ri = 4 * w + slot, d = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j + e;
            word |= code_at(0, t, d) << (4 * slot + 16 * e);
          }
        kw[wi] = word;
      }
      const int vwpl = P / 32;  // words per (cn, lane)
      for (int wi = threadIdx.x; wi < kwords; wi += blockDim.x) {
        int cn = wi / (32 * vwpl), rem = wi % (32 * vwpl), lane = rem / vwpl, w = rem % vwpl;
        int c = 8 * cn + lane / 4, j = lane % 4;
        uint32_t word = 0;
#pragma unroll
        for (int slot = 0; slot < 4; ++slot)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            int ri = 4 * w + slot, t = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j + e;
            word |= code_at(1, t, c) << (4 * slot + 16 * e);
          }
        vw[wi] = word;
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
// open page that already has t_old = n_tok % P > 0 tokens.  Bit-identical
// to append_page(): a channel whose min/max did not move keeps its lo and
// scale, so only the new token's code changes; channels whose bounds moved
// are re-coded for every token of the page from the raw staging copy.
// Whole CTA; smem >= append_one_smem_bytes(D, P).
template <typename T>
__device__ void append_one_token(const PoolView& pv, int s, int n_tok, const T* __restrict__ kn,
                                 const T* __restrict__ vn, uint8_t* smem) {
  const int D = pv.D, P = pv.P;
  const int t_old = n_tok % P;
  const int p = n_tok / P;
  if (t_old == 0 || pv.bits == 0) {
    append_page<T>(pv, s, p, n_tok, n_tok + 1, kn, vn, 0, smem);
    return;
  }
  const bool dense = pv.kind[s] == SK_KIND_DENSE;
  uint8_t* slot = pv.slot_ptr(s, p);
  T* bnd = reinterpret_cast<T*>(pv.bounds(slot));
  const T* stg[2] = {reinterpret_cast<const T*>(pv.staging_ptr(s, 0)),
                     reinterpret_cast<const T*>(pv.staging_ptr(s, 1))};
  float* xnew = reinterpret_cast<float*>(smem);   // [2][D]
  double* lo = reinterpret_cast<double*>(xnew + 2 * D);  // [2][D]
  double* sc = lo + 2 * D;
  double* inv = sc + 2 * D;
  uint8_t* chg = reinterpret_cast<uint8_t*>(inv + 2 * D);  // [2][D]
  T* raw = reinterpret_cast<T*>(chg + ((2 * D + 15) & ~15));  // [2][t_old][D] staged raw tokens
  const int levels = (1 << pv.bits) - 1;
  // the open page's raw tokens -> smem (one coalesced sweep; code_at reads them often)
  for (int i = threadIdx.x; i < 2 * t_old * (D / 8); i += blockDim.x) {
    const int which = i / (t_old * (D / 8)), rem = i % (t_old * (D / 8));
    *reinterpret_cast<uint4*>(raw + (which * t_old) * D + rem * 8) =
        *reinterpret_cast<const uint4*>(stg[which] + rem * 8);
  }
  for (int i = threadIdx.x; i < 2 * D; i += blockDim.x) {
    const int which = i / D, c = i % D;
    const float x = DT<T>::to_f((which ? vn : kn)[c]);
    const int pos = which ? vbound_pos(c, D) : kbound_pos(c, D);
    const float olo = DT<T>::to_f(bnd[2 * which * D + pos]), ohi = DT<T>::to_f(bnd[(2 * which + 1) * D + pos]);
    const float nlo = fminf(olo, x), nhi = fmaxf(ohi, x);
    const bool changed = (nlo != olo) || (nhi != ohi);
    if (changed) {
      bnd[2 * which * D + pos] = DT<T>::from_f(nlo);
      bnd[(2 * which + 1) * D + pos] = DT<T>::from_f(nhi);
    }
    double scl = ((double)nhi - (double)nlo) / levels;
    if (!(scl > 0.0)) scl = 1.0;
    xnew[i] = x;
    lo[i] = nlo;
    sc[i] = scl;
    inv[i] = 1.0 / scl;
    chg[i] = changed;
  }
  __syncthreads();
  auto code_at = [&](int which, int t, int c) -> uint32_t {
    if (t > t_old) return 0u;  // padding slots of the page
    const float x = t == t_old ? xnew[which * D + c] : DT<T>::to_f(raw[(which * t_old + t) * D + c]);
    const int i = which * D + c;
    return quant_code((double)x, lo[i], sc[i], inv[i], levels);
  };
  uint32_t* kw = reinterpret_cast<uint32_t*>(pv.k_codes(slot));
  uint32_t* vw = reinterpret_cast<uint32_t*>(pv.v_codes(slot));
  const bool nib = pv.bits <= 4;
  const int cpw = nib ? 8 : 4;                      // codes per 32-bit word
  const int wpt = nib ? D / 8 : D / 4;              // K words per token
  const int wpc = nib ? D / 32 : D / 16;            // K words per (token, j) chunk
  const int vwl = nib ? P / 32 : P / 16;            // V words per (cn, lane)
  // (q-th code of a word) -> (register index offset, e, bit position)
  auto qmap = [&](int w, int q, int& ri, int& e, int& bit) {
    if (nib) {
      const int slt = q >> 1;
      e = q & 1;
      ri = 4 * w + slt;
      bit = 4 * slt + 16 * e;
    } else {
      const int r2 = q >> 1;
      e = q & 1;
      ri = 2 * w + r2;
      bit = 8 * (2 * r2 + e);
    }
  };
  const uint32_t cmask = nib ? 0xFu : 0xFFu;
  // K: words of tokens 0..t_old (token t_old fully rewritten, others only if a channel moved)
  for (int wi = threadIdx.x; wi < (t_old + 1) * wpt; wi += blockDim.x) {
    const int t = wi / wpt, rem = wi % wpt, j = rem / wpc, w = rem % wpc;
    uint32_t word = t == t_old ? 0u : kw[t * wpt + rem];
    bool dirty = t == t_old;
    for (int q = 0; q < cpw; ++q) {
      int ri, e, bit;
      qmap(w, q, ri, e, bit);
      const int d = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j + e;
      if (t == t_old || chg[d]) {
        word = (word & ~(cmask << bit)) | (code_at(0, t, d) << bit);
        dirty = true;
      }
    }
    if (dirty) kw[t * wpt + rem] = word;
  }
  // V: a moved channel rewrites all its words; otherwise only the nibble/byte of token t_old
  const int vwords = P * D / cpw;
  for (int wi = threadIdx.x; wi < vwords; wi += blockDim.x) {
    const int cn = wi / (32 * vwl), rem = wi % (32 * vwl), lane = rem / vwl, w = rem % vwl;
    const int c = 8 * cn + lane / 4, j = lane % 4;
    const bool moved = chg[D + c];
    uint32_t word = moved ? 0u : vw[wi];
    bool dirty = moved;
    for (int q = 0; q < cpw; ++q) {
      int ri, e, bit;
      qmap(w, q, ri, e, bit);
      const int t = 16 * (ri / 2) + 8 * (ri % 2) + 2 * j + e;
      if (moved || t == t_old) {
        word = (word & ~(cmask << bit)) | (code_at(1, t, c) << bit);
        dirty = true;
      }
    }
    if (dirty) vw[wi] = word;
  }
  // logical-page key stats of the page's open logical page (dense pool)
  if (dense && pv.stats != nullptr) {
    const int L = pv.L;
    T* st = reinterpret_cast<T*>(pv.stats_ptr(s, p * (P / L) + t_old / L));
    const bool fresh = (t_old % L) == 0;
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
      const float x = xnew[c];
      if (fresh) {
        st[c] = DT<T>::from_f(x);
        st[D + c] = DT<T>::from_f(x);
      } else {
        st[c] = DT<T>::from_f(fminf(DT<T>::to_f(st[c]), x));
        st[D + c] = DT<T>::from_f(fmaxf(DT<T>::to_f(st[D + c]), x));
      }
    }
  }
  // raw staging of the open page (unless the page is now full)
  if (t_old + 1 < P) {
    T* wk = reinterpret_cast<T*>(pv.staging_ptr(s, 0));
    T* wv = reinterpret_cast<T*>(pv.staging_ptr(s, 1));
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
      wk[t_old * D + c] = kn[c];
      wv[t_old * D + c] = vn[c];
    }
  }
}

}  // namespace sk
