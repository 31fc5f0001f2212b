// Row-in-registers 64x64 POTRF + triangular inverse, 128 threads: thread (r, h) owns the
// columns c = 2i + h (i < 32) of row r, h = warp-uniform half. One barrier per elimination
// step; the next pivot column is updated first and published through a double-buffered
// smem column; the next pivot's rsqrt is computed by every lane of the owning half (no
// divergence) and stored by its owner after the remaining updates.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
constexpr int TB = 64, NT = 128;
__device__ __forceinline__ double rsqrt_h(double a) {
  // float seed + one third-order correction: relative error ~ e^3, e ~ 2^-22
  const double r0 = (double)rsqrtf((float)a);
  const double e = fma(-a * r0, r0, 1.0);
  return fma(r0 * e, fma(0.375, e, 0.5), r0);
}
template <int H>
__device__ __forceinline__ void chol_half(double (&a)[32], int r, double (*cb)[TB], double* pr, double* dg, bool& ok) {
  // Entries above the diagonal (c > r) are never read; they are updated unconditionally
  // (any value, even non-finite) so that the update is branch- and select-free.
#pragma unroll
  for (int j = 0; j < TB; ++j) {
    const double rj = pr[j & 1];
    const double* col = cb[j & 1];
    double* nxt = cb[(j + 1) & 1];
    const double cr = col[r];
    const double s = cr * rj * rj;  // a_r[j] / a_jj
    if ((j & 1) == H) {
      if (r >= j) a[j >> 1] = cr * rj;  // L[r][j]
    }
    if (j + 1 < TB) {
      if (((j + 1) & 1) == H) {
        const int i1 = (j + 1) >> 1;
        a[i1] = fma(-s, col[j + 1], a[i1]);
        nxt[r] = a[i1];
        const double v = a[i1];
        const double rn = rsqrt_h(v);
        if (r == j + 1) {
          pr[(j + 1) & 1] = rn;
          dg[j + 1] = rn;
          ok = ok && (v > 0.0);
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = 2 * i + H;
        if (c >= j + 2) a[i] = fma(-s, col[c], a[i]);
      }
      if (r >= 32) {
#pragma unroll
        for (int i = 16; i < 32; ++i) {
          const int c = 2 * i + H;
          if (c >= j + 2) a[i] = fma(-s, col[c], a[i]);
        }
      }
    }
    __syncthreads();
  }
}
__global__ void __launch_bounds__(NT) k(const double* F, int ld, int b, double* Fout, double* Dout, int* bad,
                                        long long* clk) {
  __shared__ double cb[2][TB];
  __shared__ double pr[2];
  __shared__ double dg[TB];  // 1 / L[j][j] = the pivots' rsqrt
  __shared__ double Ls[TB][TB + 1];
  const int t = threadIdx.x, r = t & 63, h = t >> 6;
  long long t0 = clock64();
  double a[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int c = 2 * i + h;
    double v;
    if (r < b && c < b) v = (c <= r) ? F[(long long)c * ld + r] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    a[i] = v;
  }
  bool ok = true;
  if (h == 0) {
    cb[0][r] = a[0];
    if (r == 0) {
      pr[0] = rsqrt_h(a[0]);
      dg[0] = pr[0];
      ok = a[0] > 0.0;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (h == 0) chol_half<0>(a, r, cb, pr, dg, ok);
  else chol_half<1>(a, r, cb, pr, dg, ok);
  long long t2 = clock64();
  if (!ok) atomicOr(bad, 1);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int c = 2 * i + h;
    if (r < b && c < b && c <= r) Fout[(long long)c * ld + r] = a[i];
    Ls[r][c] = (c <= r) ? a[i] : 0.0;
  }
  __syncthreads();
  // X = L^-1 by 32-blocks: X11 = L11^-1, X22 = L22^-1 (warp 0 / warp 1, lane = column),
  // then X21 = -X22 (L21 X11).
  // X = L^-1 by columns: thread pair (c, hf), c = t >> 1, forward-substitutes column c;
  // each half sums the k of its parity, the pair combines with a shuffle. X[m][c]
  // (m > c) is kept in the strictly upper part of Ls at Ls[c][m]; X[c][c] = dg[c].
  {
    const int c = t >> 1, hf = t & 1;
    const int m0 = (t & ~31) >> 1;  // the warp's smallest column: uniform trip counts
#pragma unroll 1
    for (int m = m0 + 1; m < TB; ++m) {
      double s0 = 0.0, s1 = 0.0;
      int k = c + 1 + hf;
      if (hf == 0 && m > c) s0 = Ls[m][c] * dg[c];
#pragma unroll 2
      for (; k + 2 < m; k += 4) {
        s0 = fma(Ls[m][k], Ls[c][k], s0);
        s1 = fma(Ls[m][k + 2], Ls[c][k + 2], s1);
      }
      if (k < m) s0 = fma(Ls[m][k], Ls[c][k], s0);
      double sum = s0 + s1;
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      if (hf == 0 && m > c) Ls[c][m] = -sum * dg[m];
      __syncwarp();
    }
  }
  __syncthreads();
  long long t2a = clock64();
  long long t2b = t2a;
  for (int e = t; e < TB * TB; e += NT) {
    const int c = e >> 6, m = e & 63;
    Dout[e] = (m >= c && m < b && c < b) ? ((m == c) ? dg[c] : Ls[c][m]) : 0.0;
  }
  long long t3 = clock64();
  if (t == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; clk[3] = t2a - t2; clk[4] = t2b - t2a; }
}
int main() {
  static double h[TB * TB];
  for (int i = 0; i < TB; ++i) for (int j = 0; j < TB; ++j) h[j * TB + i] = (i == j ? 100.0 : 1.0 / (1 + abs(i - j)));
  double *dA, *dL, *dD; long long* dc; int* db;
  cudaMalloc(&dA, sizeof h); cudaMalloc(&dL, sizeof h); cudaMalloc(&dD, sizeof h); cudaMalloc(&dc, 64); cudaMalloc(&db, 4);
  cudaMemset(db, 0, 4);
  cudaMemcpy(dA, h, sizeof h, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); k<<<16, NT>>>(dA, TB, TB, dL, dD, db, dc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c[5]; cudaMemcpy(c, dc, 40, cudaMemcpyDeviceToHost);
    printf("potrf4: %.1f us  load %lld  chol %lld  inv %lld (diag %lld T %lld) cycles (%s)\n", ms * 1e3, c[0], c[1], c[2], c[3], c[4],
           cudaGetErrorString(cudaGetLastError()));
  }
  static double Lh[TB * TB], Dh[TB * TB];
  cudaMemcpy(Lh, dL, sizeof Lh, cudaMemcpyDeviceToHost);
  cudaMemcpy(Dh, dD, sizeof Dh, cudaMemcpyDeviceToHost);
  double e1m = 0, e2m = 0;
  for (int i = 0; i < TB; ++i) for (int j = 0; j <= i; ++j) {
    double s = 0; for (int m = 0; m <= j; ++m) s += Lh[m * TB + i] * Lh[m * TB + j];
    e1m = fmax(e1m, fabs(s - h[j * TB + i]));
  }
  for (int i = 0; i < TB; ++i) for (int j = 0; j < TB; ++j) {
    double s = 0; for (int m = 0; m < TB; ++m) s += (m <= i ? Lh[m * TB + i] : 0.0) * Dh[j * TB + m];
    e2m = fmax(e2m, fabs(s - (i == j)));
  }
  int bh; cudaMemcpy(&bh, db, 4, cudaMemcpyDeviceToHost);
  printf("max |LL^T - A| %.2e   max |L X - I| %.2e  bad %d\n", e1m, e2m, bh);
}
