#include <cstdio>
#include <cuda_runtime.h>
constexpr int TB = 64;
__device__ __forceinline__ double rsqrt_fast(double a) {
  double r = (double)rsqrtf((float)a);
  r = r * (1.5 - 0.5 * a * r * r);
  r = r * (1.5 - 0.5 * a * r * r);
  return r;
}
template <int V>
__global__ void __launch_bounds__(256) k(double x, long long* clk, double* out) {
  __shared__ double cb[2][TB];
  __shared__ double pr[2];
  __shared__ double A[TB][TB + 1];
  const int tid = threadIdx.x, r = tid & 63, cg = tid >> 6;
  for (int e = tid; e < TB * TB; e += 256) A[e / TB][e % TB] = (e / TB == e % TB) ? 100.0 : 0.5;
  if (tid < TB) cb[0][tid] = 100.0;
  if (tid == 0) pr[0] = 0.1;
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
  for (int j = 0; j < TB; ++j) {
    const double* col = cb[j & 1];
    double* nxt = cb[(j + 1) & 1];
    const double rj = pr[j & 1];
    if (V >= 1 && r > j) {
      const double lr = col[r] * rj * rj;
      for (int c = j + 1 + cg; c <= r; c += 4) A[r][c] -= lr * col[c];
    }
    if (V >= 2 && cg == 0) nxt[r] = A[r][j + 1 < TB ? j + 1 : j];
    if (tid == j + 1) pr[(j + 1) & 1] = rsqrt_fast(col[tid] + rj);
    acc += rj;
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) clk[V] = t1 - t0;
  out[tid] = acc + A[r][r];
}
// register-resident rows (thread (r, cg) owns a[m] = A[r][cg + 4m]); branch-free update
template <int MODE>  // 0 full, 1 no rsqrt (pivot = constant), 2 no select (column from a[0]), 3 no update
__global__ void __launch_bounds__(256) kreg(long long* clk, double* out) {
  __shared__ double cb[2][TB];
  __shared__ double pr[2];
  const int tid = threadIdx.x, r = tid & 63, cg = tid >> 6;
  double a[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = (cg + 4 * m == r) ? 100.0 : 0.5;
  if (tid < TB) cb[0][tid] = 100.0;
  if (tid == 0) pr[0] = 0.1;
  __syncthreads();
  long long t0 = clock64();
  for (int j = 0; j < TB; ++j) {
    const double* col = cb[j & 1];
    double* nxt = cb[(j + 1) & 1];
    const double rj = pr[j & 1];
    const double lr = (r > j) ? col[r] * rj * rj : 0.0;
    if (MODE != 3) {
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int c = cg + 4 * m;
        const double cc = col[c];
        const double upd = fma(-lr, cc, a[m]);
        a[m] = (c > j && c <= r) ? upd : a[m];
      }
    }
    const int own = (j + 1) & 3, m1 = (j + 1) >> 2;
    double v = a[0];
    if (MODE != 2) {
#pragma unroll
      for (int m = 1; m < 16; ++m) v = (m == m1) ? a[m] : v;
    }
    if (cg == own && j + 1 < TB) {
      nxt[r] = v;
      if (r == j + 1) pr[(j + 1) & 1] = (MODE == 1) ? v * 0.001 : rsqrt_fast(v);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) clk[3 + MODE] = t1 - t0;
  double s2 = 0;
#pragma unroll
  for (int m = 0; m < 16; ++m) s2 += a[m];
  out[tid] = s2;
}
int main() {
  long long* dc; double* o; cudaMalloc(&dc, 64); cudaMalloc(&o, 256 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 256>>>(1.1, dc, o); k<1><<<1, 256>>>(1.1, dc, o); k<2><<<1, 256>>>(1.1, dc, o);
    kreg<0><<<1, 256>>>(dc, o); kreg<1><<<1, 256>>>(dc, o); kreg<2><<<1, 256>>>(dc, o); kreg<3><<<1, 256>>>(dc, o);
    cudaDeviceSynchronize();
    long long c[7]; cudaMemcpy(c, dc, 56, cudaMemcpyDeviceToHost);
    printf("reg: full %.0f  no-rsqrt %.0f  no-select %.0f  no-update %.0f cycles/step\n", c[3] / 64.0, c[4] / 64.0, c[5] / 64.0, c[6] / 64.0);
  }
}
