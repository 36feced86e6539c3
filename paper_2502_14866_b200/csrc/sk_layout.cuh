// Fragment-native page layout shared by K1 (writer), K3 (reader) and the
// host-side views (paper_2502_14866_b200/layout.py mirrors these formulas).
//
// Decode runs on m16n8k16 tensor-core fragments (f16 in, f32 accumulate):
//   S   = q'  x K^T : B[k=dim][n=token]   thread: token = lane/4, dims 16s+8h+2j+e
//   O  += P   x V   : B[k=token][n=chan]  thread: chan  = 8cn+lane/4, tokens 16ks+8h+2j+e
// (j = lane%4, e in {0,1}).  K1 stores codes so that each thread's B
// registers for a page are contiguous bytes, and a 32-bit word holds four
// fp16x2 registers as nibbles: register `slot` of a word takes bits
// [4*slot, 4*slot+4) for its low half and [16+4*slot, ...) for its high half,
// so one LOP3 ((w >> 4*slot) & 0x000F000F | 0x64006400) plus one HSUB2 gives
// the two codes as exact fp16 integers.
#pragma once
#include <cstdint>

namespace sk {

// ---- K codes: token t, dim d -------------------------------------------------
// row of D/2 bytes per token (bits<=4); chunk j (D/8 bytes) per lane%4.
__host__ __device__ inline void kpos_nib(int t, int d, int D, int& byte, int& shift) {
  int s = d / 16, h = (d % 16) / 8, j = (d % 8) / 2, e = d % 2;
  int ri = 2 * s + h, w = ri / 4, slot = ri % 4;
  int bit = 4 * slot + 16 * e;
  byte = t * (D / 2) + j * (D / 8) + w * 4 + bit / 8;
  shift = bit % 8;
}
// 8-bit codes: register = 2 bytes (e=0 low byte, e=1 high byte).
__host__ __device__ inline int kpos_byte(int t, int d, int D) {
  int s = d / 16, h = (d % 16) / 8, j = (d % 8) / 2, e = d % 2;
  int ri = 2 * s + h;
  return t * D + j * (D / 4) + ri * 2 + e;
}
// raw 16-bit values: register = 2 elements.  Returns element index.
__host__ __device__ inline int kpos_raw(int t, int d, int D) {
  int s = d / 16, h = (d % 16) / 8, j = (d % 8) / 2, e = d % 2;
  int ri = 2 * s + h;
  return t * D + j * (D / 4) + ri * 2 + e;
}

// ---- V codes: token t, channel c --------------------------------------------
// [cn = c/8][lane = 4*(c%8) + (t%8)/2][P/8 bytes] (bits<=4; requires P%32==0)
__host__ __device__ inline void vpos_nib(int t, int c, int P, int& byte, int& shift) {
  int cn = c / 8, c8 = c % 8;
  int ks = t / 16, h = (t % 16) / 8, j = (t % 8) / 2, e = t % 2;
  int lane = 4 * c8 + j;
  int ri = 2 * ks + h, w = ri / 4, slot = ri % 4;
  int bit = 4 * slot + 16 * e;
  byte = (cn * 32 + lane) * (P / 8) + w * 4 + bit / 8;
  shift = bit % 8;
}
__host__ __device__ inline int vpos_byte(int t, int c, int P) {
  int cn = c / 8, c8 = c % 8;
  int ks = t / 16, h = (t % 16) / 8, j = (t % 8) / 2, e = t % 2;
  int lane = 4 * c8 + j;
  int ri = 2 * ks + h;
  return (cn * 32 + lane) * (P / 4) + ri * 2 + e;
}
__host__ __device__ inline int vpos_raw(int t, int c, int P) {  // element index
  int cn = c / 8, c8 = c % 8;
  int ks = t / 16, h = (t % 16) / 8, j = (t % 8) / 2, e = t % 2;
  int lane = 4 * c8 + j;
  int ri = 2 * ks + h;
  return (cn * 32 + lane) * (P / 4) + ri * 2 + e;
}

// ---- page bounds: [k_lo | k_hi | v_lo | v_hi], each D elements --------------
// K bounds follow the q' A-fragment dims of lane%4 = j: index j*(D/4) + ri*2 + e
// with d = 16*(ri/2) + 8*(ri%2) + 2j + e.  V bounds follow the PV C-fragment
// channels of j: index j*(D/4) + cn*2 + e with c = 8*cn + 2j + e.
__host__ __device__ inline int kbound_pos(int d, int D) {
  int s = d / 16, h = (d % 16) / 8, j = (d % 8) / 2, e = d % 2;
  return j * (D / 4) + (2 * s + h) * 2 + e;
}
__host__ __device__ inline int vbound_pos(int c, int D) {
  int cn = c / 8, j = (c % 8) / 2, e = c % 2;
  return j * (D / 4) + cn * 2 + e;
}

}  // namespace sk
