// Microbenchmark of the 64x64 POTRF + inverse block kernel's phases (clock64).
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>
constexpr int TB = 64;
__device__ __forceinline__ double rsqrt_fast(double a) {
  double r = (double)rsqrtf((float)a);
  r = r * (1.5 - 0.5 * a * r * r);
  r = r * (1.5 - 0.5 * a * r * r);
  return r;
}
__global__ void __launch_bounds__(256) k(const double* Ain, double* Lout, long long* clk) {
  extern __shared__ double dyn[];
  double(*A)[TB + 1] = reinterpret_cast<double(*)[TB + 1]>(dyn);
  __shared__ double L[TB][TB + 1];
  __shared__ double cb[2][TB];
  __shared__ double pr[2];
  const int tid = threadIdx.x;
  long long t0 = clock64();
  for (int e = tid; e < TB * TB; e += 256) {
    const int c = e / TB, r = e % TB;
    double v = Ain[c * TB + r];
    A[r][c] = v;
    if (c == 0) cb[0][r] = v;
    if (e == 0) pr[0] = rsqrt_fast(v);
  }
  __syncthreads();
  long long t1 = clock64();
  const int r = tid & 63, cg = tid >> 6;
  for (int j = 0; j < TB; ++j) {
    const double* col = cb[j & 1];
    double* nxt = cb[(j + 1) & 1];
    const double rj = pr[j & 1];
    const double ajj = col[j];
    if (r >= j && cg == 0) L[r][j] = (r == j) ? ajj * rj : col[r] * rj;
    if (r > j) {
      const double lr = col[r] * rj * rj;
      int c = j + 1 + cg;
      if (cg == 0) {
        const double v = A[r][c] - lr * col[c];
        A[r][c] = v;
        nxt[r] = v;
        if (r == j + 1) pr[(j + 1) & 1] = rsqrt_fast(v);
        c += 4;
      }
      for (; c <= r; c += 4) A[r][c] -= lr * col[c];
    }
    __syncthreads();
  }
  long long t2 = clock64();
  for (int e = tid; e < TB * TB; e += 256) Lout[e] = L[e % TB][e / TB];
  __syncthreads();
  long long t3 = clock64();
  if (tid == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; }
}
// variant: only barriers
__global__ void __launch_bounds__(256) kb(long long* clk) {
  long long t0 = clock64();
  for (int j = 0; j < 64; ++j) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[0] = t1 - t0;
}
int main() {
  double h[TB * TB];
  for (int i = 0; i < TB; ++i) for (int j = 0; j < TB; ++j) h[j * TB + i] = (i == j ? 100.0 : 1.0 / (1 + abs(i - j)));
  double *dA, *dL; long long* dc; cudaMalloc(&dA, sizeof h); cudaMalloc(&dL, sizeof h); cudaMalloc(&dc, 64);
  cudaMemcpy(dA, h, sizeof h, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TB * (TB + 1) * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); k<<<16, 256, TB * (TB + 1) * 8>>>(dA, dL, dc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c[3]; cudaMemcpy(c, dc, 24, cudaMemcpyDeviceToHost);
    printf("potrf: %.1f us  load %lld  chol %lld  store %lld cycles\n", ms * 1e3, c[0], c[1], c[2]);
  }
  kb<<<1, 256>>>(dc); cudaDeviceSynchronize(); long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("64 barriers: %lld cycles\n", c);
  return 0;
}
