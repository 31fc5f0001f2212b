// Blocked (8-column panels) 64x64 POTRF in shared memory.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int TB = 64, PW = 8;
__device__ __forceinline__ double rsqrt_fast(double a) {
  double r = (double)rsqrtf((float)a);
  r = r * (1.5 - 0.5 * a * r * r);
  r = r * (1.5 - 0.5 * a * r * r);
  return r;
}
__global__ void __launch_bounds__(256) k(const double* F, int ld, int b, double* Fout, long long* clk) {
  extern __shared__ double dyn[];
  double(*A)[TB + 1] = reinterpret_cast<double(*)[TB + 1]>(dyn);
  __shared__ double L[TB][TB + 1];
  const int tid = threadIdx.x;
  long long t0 = clock64();
  for (int e = tid; e < TB * TB; e += 256) {
    const int c = e / TB, r = e % TB;
    double v;
    if (r < b && c < b) v = (r >= c) ? F[(long long)c * ld + r] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    A[r][c] = v;
  }
  __syncthreads();
  long long t1 = clock64();
  for (int p0 = 0; p0 < TB; p0 += PW) {
    for (int j = p0; j < p0 + PW; ++j) {
      const double ajj = A[j][j];
      const double rj = ajj > 0.0 ? rsqrt_fast(ajj) : 1.0;
      const double rj2 = rj * rj;
      // scaled column j into L; in-panel update of columns j+1..p0+PW-1
      const int ncol = p0 + PW - 1 - j;  // columns j+1 .. p0+PW-1
      for (int e = tid; e < TB * (ncol + 1); e += 256) {
        const int r = e & 63, q = e >> 6;  // q = 0: column j itself
        if (q == 0) {
          if (r >= j) L[r][j] = A[r][j] * rj;
        } else {
          const int c = j + q;
          if (r >= c) A[r][c] -= A[r][j] * A[c][j] * rj2;
        }
      }
      __syncthreads();
    }
    // trailing update: rows/cols >= p0+PW, c <= r: A[r][c] -= sum_k L[r][k] L[c][k]
    const int t0r = p0 + PW, n = TB - t0r;
    for (int e = tid; e < n * n; e += 256) {
      const int rr = e % n, cc = e / n;
      if (cc > rr) continue;
      const int r = t0r + rr, c = t0r + cc;
      double s = 0.0;
#pragma unroll
      for (int kk = 0; kk < PW; ++kk) s += L[r][p0 + kk] * L[c][p0 + kk];
      A[r][c] -= s;
    }
    __syncthreads();
  }
  long long t2 = clock64();
  for (int e = tid; e < TB * TB; e += 256) {
    const int c = e / TB, rr = e % TB;
    if (rr < b && c < b && rr >= c) Fout[(long long)c * ld + rr] = L[rr][c];
  }
  if (tid == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; }
}
int main() {
  static double h[TB * TB];
  for (int i = 0; i < TB; ++i) for (int j = 0; j < TB; ++j) h[j * TB + i] = (i == j ? 100.0 : 1.0 / (1 + abs(i - j)));
  double *dA, *dL; long long* dc; cudaMalloc(&dA, sizeof h); cudaMalloc(&dL, sizeof h); cudaMalloc(&dc, 64);
  cudaMemcpy(dA, h, sizeof h, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TB * (TB + 1) * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); k<<<16, 256, TB * (TB + 1) * 8>>>(dA, TB, TB, dL, dc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c[2]; cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
    printf("potrf3: %.1f us  load %lld  chol %lld cycles\n", ms * 1e3, c[0], c[1]);
  }
  static double Lh[TB*TB]; cudaMemcpy(Lh, dL, sizeof Lh, cudaMemcpyDeviceToHost);
  double e1m = 0;
  for (int i = 0; i < TB; ++i) for (int j = 0; j <= i; ++j) {
    double s = 0; for (int m = 0; m <= j; ++m) s += Lh[m*TB+i] * Lh[m*TB+j];
    e1m = fmax(e1m, fabs(s - h[j*TB+i]));
  }
  printf("max |LL^T - A| %.2e\n", e1m);
}
