// Standalone probe: validates the hand-written tcgen05 / TMA / UMMA-descriptor
// encodings in sk_sm100.cuh on a real B200 before the prefill kernel uses
// them.  One CTA computes S = Q K^T (128x64, D=128, K-major SW128 operands
// loaded by TMA), writes P = fp16(S * 0.125) into shared memory in the
// SW128 K-major layout, then O = P V with V as an MN-major SW128 operand.
// Prints max-abs errors against a host fp32 reference.  Exit 0 = pass.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2502_14866_b200/csrc/sk_sm100.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(2);} } while (0)

using namespace sk;

struct Smem {
  alignas(1024) uint8_t q[2][128 * 128];  // 2 d-chunks x 128 rows x 128B
  alignas(1024) uint8_t k[2][64 * 128];
  alignas(1024) uint8_t v[2][64 * 128];
  alignas(1024) uint8_t p[128 * 128];
  uint64_t bar_load, bar_mma;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(128) probe(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                                             const __grid_constant__ CUtensorMap tv, float* s_out, float* o_out,
                                             int lbo_v, int sbo_v) {
  extern __shared__ uint8_t raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&sm.bar_load, 1);
    mbar_init(&sm.bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tbase = sm.tmem_base;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&sm.bar_load, 2 * 128 * 128 + 4 * 64 * 128);
    for (int c = 0; c < 2; ++c) {
      tma_load_3d(sm.q[c], &tq, &sm.bar_load, 64 * c, 0, 0);
      tma_load_3d(sm.k[c], &tk, &sm.bar_load, 64 * c, 0, 0);
      tma_load_3d(sm.v[c], &tv, &sm.bar_load, 64 * c, 0, 0);
    }
  }
  mbar_wait(&sm.bar_load, 0);
  // S = Q K^T : M=128, N=64, K=128 (8 steps of 16)
  if (warp == 0) {
    tc_fence_after();
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc_f16(128, 64, false, false, false);
      for (int kk = 0; kk < 8; ++kk) {
        uint64_t a = make_sdesc_sw128(smem_u32(sm.q[kk / 4]) + (kk % 4) * 32, 16, 1024);
        uint64_t b = make_sdesc_sw128(smem_u32(sm.k[kk / 4]) + (kk % 4) * 32, 16, 1024);
        mma_f16_ss(tbase, a, b, idesc, kk > 0);
      }
      mma_commit(&sm.bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&sm.bar_mma, 0);
  tc_fence_after();
  int row = warp * 32 + lane;
  uint32_t lane_base = tbase + (uint32_t(warp * 32) << 16);
  float srow[64];
  for (int c = 0; c < 64; c += 16) {
    uint32_t r[16];
    tmem_ld_x16(lane_base + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) srow[c + i] = __uint_as_float(r[i]);
  }
  for (int c = 0; c < 64; ++c) s_out[row * 64 + c] = srow[c];
  // P = fp16(S/8) -> smem SW128 K-major (row r: 8 chunks of 16B, chunk ^= r&7)
  for (int ch = 0; ch < 8; ++ch) {
    uint4 w;
    w.x = pack_half2(srow[ch * 8 + 0] * 0.125f, srow[ch * 8 + 1] * 0.125f);
    w.y = pack_half2(srow[ch * 8 + 2] * 0.125f, srow[ch * 8 + 3] * 0.125f);
    w.z = pack_half2(srow[ch * 8 + 4] * 0.125f, srow[ch * 8 + 5] * 0.125f);
    w.w = pack_half2(srow[ch * 8 + 6] * 0.125f, srow[ch * 8 + 7] * 0.125f);
    *reinterpret_cast<uint4*>(sm.p + row * 128 + ((ch ^ (row & 7)) << 4)) = w;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  // O = P V : M=128, N=128, K=64 (4 steps); V is MN-major (d contiguous)
  if (warp == 0) {
    tc_fence_after();
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc_f16(128, 128, false, false, true);
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t a = make_sdesc_sw128(smem_u32(sm.p) + kk * 32, 16, 1024);
        uint64_t b = make_sdesc_sw128(smem_u32(sm.v[0]) + kk * 2048, lbo_v, sbo_v);
        mma_f16_ss(tbase + 64, a, b, idesc, kk > 0);
      }
      mma_commit(&sm.bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&sm.bar_mma, 1);
  tc_fence_after();
  for (int c = 0; c < 128; c += 16) {
    uint32_t r[16];
    tmem_ld_x16(lane_base + 64 + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) o_out[row * 128 + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tbase);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static CUtensorMap make_map(void* base, int rows, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {128, 1, (cuuint64_t)rows};
  cuuint64_t strides[2] = {128 * 2, 128 * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, base, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(2); }
  return m;
}

int main() {
  int n_q = 128, n_k = 64, d = 128;
  std::vector<__half> hq(n_q * d), hk(n_k * d), hv(n_k * d);
  std::vector<float> fq(n_q * d), fk(n_k * d), fv(n_k * d);
  srand(1);
  auto rnd = [] { return (rand() / (float)RAND_MAX) * 2.f - 1.f; };
  for (int i = 0; i < n_q * d; ++i) { hq[i] = __float2half(rnd()); fq[i] = __half2float(hq[i]); }
  for (int i = 0; i < n_k * d; ++i) { hk[i] = __float2half(rnd()); fk[i] = __half2float(hk[i]); }
  for (int i = 0; i < n_k * d; ++i) { hv[i] = __float2half(rnd()); fv[i] = __half2float(hv[i]); }
  __half *dq, *dk, *dv; float *ds, *dout;
  CK(cudaMalloc(&dq, n_q * d * 2)); CK(cudaMalloc(&dk, n_k * d * 2)); CK(cudaMalloc(&dv, n_k * d * 2));
  CK(cudaMalloc(&ds, n_q * n_k * 4)); CK(cudaMalloc(&dout, n_q * d * 4));
  CK(cudaMemcpy(dq, hq.data(), n_q * d * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dk, hk.data(), n_k * d * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, hv.data(), n_k * d * 2, cudaMemcpyHostToDevice));
  CUtensorMap tq = make_map(dq, n_q, 128), tk = make_map(dk, n_k, 64), tv = make_map(dv, n_k, 64);
  size_t smem = sizeof(Smem) + 1024;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // reference
  std::vector<float> s_ref(n_q * n_k), o_ref(n_q * d, 0.f);
  for (int i = 0; i < n_q; ++i)
    for (int j = 0; j < n_k; ++j) {
      float a = 0; for (int c = 0; c < d; ++c) a += fq[i * d + c] * fk[j * d + c];
      s_ref[i * n_k + j] = a;
    }
  for (int i = 0; i < n_q; ++i)
    for (int j = 0; j < n_k; ++j) {
      float p = __half2float(__float2half(s_ref[i * n_k + j] * 0.125f));
      for (int c = 0; c < d; ++c) o_ref[i * d + c] += p * fv[j * d + c];
    }
  int variants[2][2] = {{8192, 1024}, {1024, 8192}};
  int rc = 1;
  for (auto& vnt : variants) {
    CK(cudaMemset(ds, 0, n_q * n_k * 4)); CK(cudaMemset(dout, 0, n_q * d * 4));
    probe<<<1, 128, smem>>>(tq, tk, tv, ds, dout, vnt[0], vnt[1]);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> s(n_q * n_k), o(n_q * d);
    CK(cudaMemcpy(s.data(), ds, s.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost));
    double es = 0, eo = 0, ms = 0, mo = 0;
    for (size_t i = 0; i < s.size(); ++i) { es = fmax(es, fabs(s[i] - s_ref[i])); ms = fmax(ms, fabs(s_ref[i])); }
    for (size_t i = 0; i < o.size(); ++i) { eo = fmax(eo, fabs(o[i] - o_ref[i])); mo = fmax(mo, fabs(o_ref[i])); }
    printf("V desc LBO=%d SBO=%d : S maxerr %.3e (max %.2f)  O maxerr %.3e (max %.2f)\n", vnt[0], vnt[1], es, ms, eo, mo);
    if (es < 1e-2 && eo < 1e-2) rc = 0;
  }
  printf(rc == 0 ? "PROBE PASS\n" : "PROBE FAIL\n");
  return rc;
}
