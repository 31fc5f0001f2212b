#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double x, long long* clk, double* out, int nw) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = x + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < 256; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 1.0000001, 0.5);
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[0] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[threadIdx.x] = s;
}
int main() {
  long long* dc; double* o; cudaMalloc(&dc, 64); cudaMalloc(&o, 1024 * 8);
  for (int nt : {32, 128, 256, 1024}) {
    k<<<1, nt>>>(1.1, dc, o, nt / 32); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    double fma_per_clk = (double)nt * 256 * 8 / c;
    printf("%4d threads: %lld cycles for %d DFMA/thread -> %.1f DFMA/clk/SM\n", nt, c, 256 * 8, fma_per_clk);
  }
}
