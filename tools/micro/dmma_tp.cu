// DMMA (mma.sync.m8n8k4.f64) throughput and latency on one SM: W warps, C independent
// accumulator chains per warp, operands in registers (a) or loaded from shared memory
// per k-step (b). Prints DMMA per clock per SM and flop/clk/SM (512 flop per DMMA).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int C, bool SMEM>
__global__ void k(long long* clk, double* out, int iters) {
  __shared__ double s[8][64 * 8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * 64 * 8; i += blockDim.x) (&s[0][0])[i] = 1e-3 * (i % 17);
  double c[C][2];
#pragma unroll
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1.0 + lane * 1e-6, b = 0.5;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) {
      if (SMEM) {
        a = s[w & 7][((it * C + i) * 32 + lane) & 511];
        b = s[(w + 1) & 7][((it * C + i) * 32 + lane + 7) & 511];
      }
      dmma(c[i][0], c[i][1], a, b);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  double t = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) t += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int C, bool SMEM>
void run(int warps, int grid) {
  long long* dc; double* o;
  cudaMalloc(&dc, grid * 8); cudaMalloc(&o, (size_t)grid * warps * 32 * 8);
  const int iters = 4096 / C;
  k<C, SMEM><<<grid, warps * 32>>>(dc, o, iters);
  k<C, SMEM><<<grid, warps * 32>>>(dc, o, iters);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  double per = (double)warps * iters * C / c;
  printf("%s C=%d warps=%2d grid=%3d: %.3f DMMA/clk/SM (%.1f flop/clk/SM; %.1f TF/s @1.965GHz x148)\n",
         SMEM ? "smem" : "regs", C, warps, grid, per, per * 512, per * 512 * 1.965e9 * 148 / 1e12);
  cudaFree(dc); cudaFree(o);
}
int main() {
  for (int w : {1, 4, 8, 16, 32}) { run<1, false>(w, 1); run<2, false>(w, 1); run<4, false>(w, 1); run<8, false>(w, 1); }
  for (int w : {4, 8, 16}) { run<4, true>(w, 1); run<8, true>(w, 1); }
  run<4, false>(8, 148); run<8, false>(16, 148);
  return 0;
}
