// 64x64 POTRF + inverse with compact code (the fully unrolled variant is instruction-fetch
// bound: straight-line code executed once per CTA). 128 threads, thread (r, h) owns the
// columns jb + 2i + h (i < 32) of row r in registers; the outer loop over 8-column panels
// is rolled, the 8 steps of a panel are unrolled, and the register window shifts by 4 per
// panel. Above-diagonal entries are updated unconditionally (never read; the published
// pivot column is zero above the diagonal so nothing non-finite can appear).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
constexpr int TB = 64, NT = 128, PW = 8;
__device__ __forceinline__ double rsqrt_h(double a) {
  const double r0 = (double)rsqrtf((float)a);
  const double e = fma(-a * r0, r0, 1.0);
  return fma(r0 * e, fma(0.375, e, 0.5), r0);
}
struct Smem {
  double cb[2][2 * TB];  // published pivot column (zero tail for the shifted window)
  double pr[2];
  double dg[TB];         // 1 / L[j][j]
  double L[TB][TB + 1];
  double X[TB][TB + 1];
};
template <int H>
__device__ __forceinline__ void chol(double (&a)[32], int r, Smem& S, bool& ok) {
#pragma unroll 1
  for (int jb = 0; jb < TB; jb += PW) {
#pragma unroll
    for (int jj = 0; jj < PW; ++jj) {
      const int j = jb + jj;
      const double rj = S.pr[jj & 1];
      const double* col = S.cb[jj & 1];
      double* nxt = S.cb[(jj + 1) & 1];
      const double cr = col[r];
      const double s = cr * rj * rj;
      if ((jj & 1) == H) a[jj >> 1] = cr * rj;  // L[r][j] (finalised; valid for r >= j)
      if (((jj + 1) & 1) == H) {                // the next pivot column first
        const int i1 = (jj + 1) >> 1;
        a[i1] = fma(-s, col[j + 1], a[i1]);
        const double v = a[i1];
        nxt[r] = (r > j) ? v : 0.0;
        const double rn = rsqrt_h(v);
        if (r == j + 1) {
          S.pr[(jj + 1) & 1] = rn;
          S.dg[j + 1] = rn;
          ok = ok && (v > 0.0);
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int c = 2 * i + H;  // relative to jb
        if (c >= jj + 2) a[i] = fma(-s, col[jb + c], a[i]);
      }
      __syncthreads();
    }
    // retire the panel's 4 columns of this half, shift the window by 4
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = jb + 2 * i + H;
      S.L[r][c] = (c <= r) ? a[i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 28; ++i) a[i] = a[i + 4];
#pragma unroll
    for (int i = 28; i < 32; ++i) a[i] = 0.0;
  }
}
__global__ void __launch_bounds__(NT) k(const double* F, int ld, int b, double* Fout, double* Dout, int* bad,
                                        long long* clk) {
  extern __shared__ double dyn[];
  Smem& S = *reinterpret_cast<Smem*>(dyn);
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
  S.cb[0][TB + r] = 0.0;
  S.cb[1][TB + r] = 0.0;
  bool ok = true;
  if (h == 0) {
    S.cb[0][r] = a[0];
    if (r == 0) {
      S.pr[0] = rsqrt_h(a[0]);
      S.dg[0] = S.pr[0];
      ok = a[0] > 0.0;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (h == 0) chol<0>(a, r, S, ok);
  else chol<1>(a, r, S, ok);
  __syncthreads();
  long long t2 = clock64();
  if (!ok) atomicOr(bad, 1);
  // L out (coalesced column-major)
  for (int e = t; e < TB * TB; e += NT) {
    const int c = e >> 6, m = e & 63;
    if (m >= c && m < b && c < b) Fout[(long long)c * ld + m] = S.L[m][c];
  }
  // ---- X = L^-1 ----
  // (1) diagonal 16-blocks: thread t < 64: block q = t >> 4, column cc = t & 15
  if (t < 64) {
    const int o = (t >> 4) * 16, cc = t & 15;
    double x[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < m; kk += 2) {
        s0 = fma(S.L[o + m][o + kk], x[kk], s0);
        if (kk + 1 < m) s1 = fma(S.L[o + m][o + kk + 1], x[kk + 1], s1);
      }
      x[m] = ((m == cc ? 1.0 : 0.0) - (s0 + s1)) * S.dg[o + m];
    }
#pragma unroll
    for (int m = 0; m < 16; ++m) S.X[o + m][o + cc] = x[m];
  }
  __syncthreads();
  // (2) block rows I = 1..3: X[I][c] = -Xd[I] * (sum_{k in [16 J, 16 I)} L[I rows][k] X[k][c]), c < 16 I
  //     T goes to the (dead) upper part of X: T[rr][c] at X[c][16 I + rr]? use L's upper part instead.
#pragma unroll 1
  for (int I = 1; I < 4; ++I) {
    const int nc = 16 * I;
    for (int e = t; e < 16 * nc; e += NT) {
      const int rr = e / nc, c = e - rr * nc;
      const int k0 = c & ~15;
      double s0 = 0.0, s1 = 0.0;
      for (int kk = k0; kk < nc; kk += 2) {
        s0 = fma(S.L[nc + rr][kk], S.X[kk][c], s0);
        s1 = fma(S.L[nc + rr][kk + 1], S.X[kk + 1][c], s1);
      }
      S.L[c][nc + rr] = s0 + s1;  // T[rr][c], stored transposed in L's upper triangle (c < nc <= nc + rr)
    }
    __syncthreads();
    for (int e = t; e < 16 * nc; e += NT) {
      const int rr = e / nc, c = e - rr * nc;
      double s0 = 0.0, s1 = 0.0;
      int m = 0;
      for (; m + 1 <= rr; m += 2) {
        s0 = fma(S.X[nc + rr][nc + m], S.L[c][nc + m], s0);
        s1 = fma(S.X[nc + rr][nc + m + 1], S.L[c][nc + m + 1], s1);
      }
      if (m <= rr) s0 = fma(S.X[nc + rr][nc + m], S.L[c][nc + m], s0);
      S.X[nc + rr][c] = -(s0 + s1);
    }
    __syncthreads();
  }
  long long t3 = clock64();
  for (int e = t; e < TB * TB; e += NT) {
    const int c = e >> 6, m = e & 63;
    Dout[e] = (m >= c && m < b && c < b) ? S.X[m][c] : 0.0;
  }
  if (t == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; }
}
int main() {
  static double h[TB * TB];
  for (int i = 0; i < TB; ++i) for (int j = 0; j < TB; ++j) h[j * TB + i] = (i == j ? 100.0 : 1.0 / (1 + abs(i - j)));
  double *dA, *dL, *dD; long long* dc; int* db;
  cudaMalloc(&dA, sizeof h); cudaMalloc(&dL, sizeof h); cudaMalloc(&dD, sizeof h); cudaMalloc(&dc, 64); cudaMalloc(&db, 4);
  cudaMemset(db, 0, 4);
  cudaMemcpy(dA, h, sizeof h, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 4; ++rep) {
    const int nb = rep < 3 ? 16 : 296;
    cudaEventRecord(e0); k<<<nb, NT, sizeof(Smem)>>>(dA, TB, TB, dL, dD, db, dc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c[3]; cudaMemcpy(c, dc, 24, cudaMemcpyDeviceToHost);
    printf("potrf5 (%d CTAs): %.1f us  load %lld  chol %lld  inv %lld cycles (%s)\n", nb, ms * 1e3, c[0], c[1], c[2],
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaMemset(db, 0, 4);
  k<<<1, NT, sizeof(Smem)>>>(dA, TB, TB, dL, dD, db, dc);
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
