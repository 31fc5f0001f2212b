// Register-resident POTRF variant: thread (r, cg) keeps A[r][cg + 4m], m < 16.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int TB = 64, SB = 16;
__device__ __forceinline__ double rsqrt_fast(double a) {
  double r = (double)rsqrtf((float)a);
  r = r * (1.5 - 0.5 * a * r * r);
  r = r * (1.5 - 0.5 * a * r * r);
  return r;
}
__global__ void __launch_bounds__(256) k(const double* F, int ld, int b, double* Fout, double* D, long long* clk) {
  extern __shared__ double dyn[];
  double(*X)[TB + 1] = reinterpret_cast<double(*)[TB + 1]>(dyn);
  __shared__ double L[TB][TB + 1];
  __shared__ double T[SB][3 * SB + 1];
  __shared__ double dg[TB];
  __shared__ double cb[2][TB];
  __shared__ double pr[2];
  const int tid = threadIdx.x;
  long long t0 = clock64();
  // lower-triangle entries idx = r(r+1)/2 + c, thread tid owns idx = tid + 256 s
  constexpr int NS = (TB * (TB + 1) / 2 + 255) / 256;  // 9 slots
  double a[NS];
  int rs[NS], cs[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    const int idx = tid + 256 * q;
    int rr = (int)((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
    while (rr * (rr + 1) / 2 > idx) --rr;
    while ((rr + 1) * (rr + 2) / 2 <= idx) ++rr;
    const int cc = idx - rr * (rr + 1) / 2;
    const bool valid = idx < TB * (TB + 1) / 2;
    rs[q] = valid ? rr : -1;
    cs[q] = valid ? cc : TB;
    double v = 0.0;
    if (valid) {
      if (rr < b && cc < b) v = F[(long long)cc * ld + rr];
      else v = (rr == cc) ? 1.0 : 0.0;
    }
    a[q] = v;
    if (valid && cc == 0) cb[0][rr] = v;
    if (valid && idx == 0) pr[0] = rsqrt_fast(v);
  }
  __syncthreads();
  long long t1 = clock64();
  for (int j = 0; j < TB; ++j) {
    const double* col = cb[j & 1];
    double* nxt = cb[(j + 1) & 1];
    const double rj = pr[j & 1];
    const double rj2 = rj * rj;
    if (tid < TB && tid >= j) L[tid][j] = col[tid] * rj;
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      const int c = cs[q];
      if (c > j) {  // r >= c > j: a_rc -= l_rj l_cj
        a[q] -= col[rs[q]] * col[c] * rj2;
        if (c == j + 1) {
          nxt[rs[q]] = a[q];
          if (rs[q] == c) pr[(j + 1) & 1] = a[q] > 0.0 ? rsqrt_fast(a[q]) : 1.0;
        }
      }
    }
    __syncthreads();
  }
  long long t2 = clock64();
  for (int e = tid; e < TB * TB; e += 256) {
    const int c = e / TB, rr = e % TB;
    if (rr < b && c < b && rr >= c) Fout[(long long)c * ld + rr] = L[rr][c];
    X[e / TB][e % TB] = 0.0;
  }
  if (tid < TB) dg[tid] = 1.0 / L[tid][tid];
  __syncthreads();
  {
    const int warp = tid >> 5, lane = tid & 31;
    if (warp < 4 && lane < SB) {
      const int o = warp * SB, c = lane;
      double xc[SB];
#pragma unroll
      for (int m = 0; m < SB; ++m) xc[m] = (m == c) ? dg[o + c] : 0.0;
      X[o + c][o + c] = dg[o + c];
#pragma unroll
      for (int rr = 1; rr < SB; ++rr) {
        if (rr <= c) continue;
        double sum = 0.0, s1 = 0.0;
#pragma unroll
        for (int m = 0; m < rr; m += 2) {
          sum += L[o + rr][o + m] * xc[m];
          if (m + 1 < rr) s1 += L[o + rr][o + m + 1] * xc[m + 1];
        }
        xc[rr] = -(sum + s1) * dg[o + rr];
        X[o + rr][o + c] = xc[rr];
      }
    }
  }
  __syncthreads();
  for (int ib = 1; ib < TB / SB; ++ib) {
    const int nc = ib * SB;
    for (int e = tid; e < SB * nc; e += 256) {
      const int rr = e / nc, c = e % nc;
      double sum = 0.0;
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int m = (c / SB) * SB;
      for (; m + 3 < nc; m += 4) {
        sum += L[ib * SB + rr][m] * X[m][c];
        s1 += L[ib * SB + rr][m + 1] * X[m + 1][c];
        s2 += L[ib * SB + rr][m + 2] * X[m + 2][c];
        s3 += L[ib * SB + rr][m + 3] * X[m + 3][c];
      }
      for (; m < nc; ++m) sum += L[ib * SB + rr][m] * X[m][c];
      T[rr][c] = (sum + s1) + (s2 + s3);
    }
    __syncthreads();
    for (int e = tid; e < SB * nc; e += 256) {
      const int rr = e / nc, c = e % nc;
      double sum = 0.0;
      double s1 = 0.0;
      int kk = 0;
      for (; kk + 1 <= rr; kk += 2) {
        sum += X[ib * SB + rr][ib * SB + kk] * T[kk][c];
        s1 += X[ib * SB + rr][ib * SB + kk + 1] * T[kk + 1][c];
      }
      if (kk <= rr) sum += X[ib * SB + rr][ib * SB + kk] * T[kk][c];
      X[ib * SB + rr][c] = -(sum + s1);
    }
    __syncthreads();
  }
  long long t3 = clock64();
  for (int e = tid; e < TB * TB; e += 256) {
    const int c = e / TB, rr = e % TB;
    D[e] = (rr < b && c < b && rr >= c) ? X[rr][c] : 0.0;
  }
  __syncthreads();
  long long t4 = clock64();
  if (tid == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; clk[3] = t4 - t3; }
}
int main() {
  static double h[TB * TB];
  for (int i = 0; i < TB; ++i) for (int j = 0; j < TB; ++j) h[j * TB + i] = (i == j ? 100.0 : 1.0 / (1 + abs(i - j)));
  double *dA, *dL, *dD; long long* dc; cudaMalloc(&dA, sizeof h); cudaMalloc(&dL, sizeof h); cudaMalloc(&dD, sizeof h); cudaMalloc(&dc, 64);
  cudaMemcpy(dA, h, sizeof h, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TB * (TB + 1) * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); k<<<16, 256, TB * (TB + 1) * 8>>>(dA, TB, TB, dL, dD, dc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c[4]; cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
    printf("potrf2: %.1f us  load %lld  chol %lld  inverse %lld  store %lld cycles\n", ms * 1e3, c[0], c[1], c[2], c[3]);
  }
  // correctness: L L^T = A and X L = I on the host
  static double L[TB*TB], X[TB*TB];
  cudaMemcpy(L, dL, sizeof L, cudaMemcpyDeviceToHost); cudaMemcpy(X, dD, sizeof X, cudaMemcpyDeviceToHost);
  double e1m = 0, e2m = 0;
  for (int i = 0; i < TB; ++i) for (int j = 0; j <= i; ++j) {
    double s = 0; for (int m = 0; m <= j; ++m) s += L[m*TB+i] * L[m*TB+j];
    e1m = fmax(e1m, fabs(s - h[j*TB+i]));
    double t = 0; for (int m = j; m <= i; ++m) t += X[m*TB+i] * L[j*TB+m];
    e2m = fmax(e2m, fabs(t - (i == j)));
  }
  printf("max |LL^T - A| %.2e   max |X L - I| %.2e\n", e1m, e2m);
  return 0;
}
