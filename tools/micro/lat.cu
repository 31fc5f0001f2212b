#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsqrt_fast(double a) {
  double r = (double)rsqrtf((float)a);
  r = r * (1.5 - 0.5 * a * r * r);
  r = r * (1.5 - 0.5 * a * r * r);
  return r;
}
__global__ void k(double x, long long* clk, double* out) {
  __shared__ double s[64];
  double a = x, b = x * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) a = fma(a, b, 0.125);
  long long t1 = clock64();
  double c = x;
  for (int i = 0; i < 64; ++i) c = rsqrt_fast(c + 1.0);
  long long t2 = clock64();
  double d = x;
  for (int i = 0; i < 64; ++i) d = 1.0 / sqrt(d + 1.0);
  long long t3 = clock64();
  s[threadIdx.x] = a;
  double e = 0;
  for (int i = 0; i < 64; ++i) { __syncthreads(); e += s[(threadIdx.x + i) & 63]; s[threadIdx.x] = e; }
  long long t4 = clock64();
  if (threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; clk[3] = t4 - t3; }
  out[threadIdx.x] = a + c + d + e;
}
int main() {
  long long* dc; double* o; cudaMalloc(&dc, 64); cudaMalloc(&o, 64 * 8);
  for (int r = 0; r < 2; ++r) {
    k<<<1, 64>>>(1.1, dc, o); cudaDeviceSynchronize();
    long long c[4]; cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
    printf("DFMA dep %.1f cyc, rsqrt_fast %.1f cyc, 1/sqrt %.1f cyc, smem+barrier step %.1f cyc\n", c[0] / 256.0, c[1] / 64.0, c[2] / 64.0, c[3] / 64.0);
  }
}
