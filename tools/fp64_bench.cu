// Micro-benchmark: fp64 FMA and f32->f64 conversion throughput per SM on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma(double* out, int iters, long long* cyc) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001 + i;
  const double b = 1.0000001, c = 0.999;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void cvt(double* out, int iters, long long* cyc) {
  float f[8];
  double a[8];
  for (int i = 0; i < 8; ++i) { f[i] = threadIdx.x * 0.001f + i; a[i] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] += (double)f[i]; f[i] = __int_as_float(__float_as_int(f[i]) ^ 1); }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 8);
  int iters = 2000;
  for (int threads : {32, 128, 256, 512, 1024}) {
    dfma<<<1, threads>>>(o, iters, c); cudaDeviceSynchronize();
    dfma<<<1, threads>>>(o, iters, c); long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA threads=%d: %.2f lane-FMAs/clk/SM\n", threads, double(threads) * iters * 8 / h);
    cvt<<<1, threads>>>(o, iters, c); cudaDeviceSynchronize();
    cvt<<<1, threads>>>(o, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("CVT+DADD threads=%d: %.2f lane-ops/clk/SM (per cvt+dadd pair)\n", threads, double(threads) * iters * 8 / h);
  }
  return 0;
}
