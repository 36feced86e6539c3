// Micro-benchmark: mma.sync m16n8k16 (f16 -> f32) latency and throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(float* out, int iters, long long* cyc) {
  float c[CH][4] = {};
  unsigned a0 = threadIdx.x, a1 = 0, a2 = threadIdx.x * 3, a3 = 0, b0 = 0x3c003c00u, b1 = threadIdx.x;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int h = 0; h < CH; ++h)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[h][0]), "+f"(c[h][1]), "+f"(c[h][2]), "+f"(c[h][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  float s = 0;
  for (int h = 0; h < CH; ++h) s += c[h][0] + c[h][1] + c[h][2] + c[h][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
void run(int warps) {
  float* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8);
  int iters = 1000;
  k<CH><<<1, 32 * warps>>>(o, iters, c);
  cudaDeviceSynchronize();
  k<CH><<<1, 32 * warps>>>(o, iters, c);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("chains=%d warps/CTA=%d: %.1f cycles per mma per warp (issue interval %.1f per SM)\n", CH, warps,
         double(h) / (iters * CH), double(h) / (iters * CH * warps));
}
int main() {
  run<1>(1); run<4>(1); run<8>(1); run<16>(1);
  run<8>(4); run<8>(8); run<8>(16);
  return 0;
}
