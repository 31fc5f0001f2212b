// DMMA rate of the chunk pass's inner loops alone (operands from shared memory, the same
// swizzled layouts and fragment mapping as pcg.cu sym_chunks), 8 warps per CTA, one CTA
// per SM, no tile streaming. Variants: SYNC = __syncthreads per tile.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pass_rate pass_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int TB = 64, NC = 16;
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int SYNC, int UNR>
__global__ void __launch_bounds__(256, 1) kpass(double* out, int tiles) {
  __shared__ __align__(16) double T[TB * TB];
  __shared__ __align__(16) double X[TB * NC];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  for (int e = tid; e < TB * TB; e += 256) T[e] = 1e-3 * (e % 97);
  for (int e = tid; e < TB * NC; e += 256) X[e] = 1e-2 * (e % 31);
  __syncthreads();
  const int q4 = warp & 3, r0 = 16 * q4 + g;
  const bool tw = warp >= 4;
  int acol[4];
  for (int kl = 0; kl < 4; ++kl) acol[kl] = 4 * (kl ^ (g & 3)) + t4;
  const int at0 = t4 * TB + (r0 ^ (t4 << 2)), at1 = t4 * TB + ((r0 + 8) ^ (t4 << 2));
  const int xb0 = t4 * NC + (g ^ (t4 << 2)), xb1 = t4 * NC + ((g ^ (t4 << 2)) ^ 8);
  double acc[2][2][2] = {};
  for (int t = 0; t < tiles; ++t) {
    if (!tw) {
#pragma unroll UNR
      for (int k0 = 0; k0 < TB; k0 += 4) {
        const double* An = T + r0 * TB + (k0 & ~15) + acol[(k0 >> 2) & 3];
        const double a0 = An[0], a1 = An[8 * TB];
        const double b0 = X[xb0 + k0 * NC], b1 = X[xb1 + k0 * NC];
        dmma(acc[0][0][0], acc[0][0][1], a0, b0);
        dmma(acc[0][1][0], acc[0][1][1], a1, b0);
        dmma(acc[1][0][0], acc[1][0][1], a0, b1);
        dmma(acc[1][1][0], acc[1][1][1], a1, b1);
      }
    } else {
#pragma unroll UNR
      for (int k0 = 0; k0 < TB; k0 += 4) {
        const double a0 = T[at0 + k0 * TB], a1 = T[at1 + k0 * TB];
        const double b0 = X[xb0 + k0 * NC], b1 = X[xb1 + k0 * NC];
        dmma(acc[0][0][0], acc[0][0][1], a0, b0);
        dmma(acc[0][1][0], acc[0][1][1], a1, b0);
        dmma(acc[1][0][0], acc[1][0][1], a0, b1);
        dmma(acc[1][1][0], acc[1][1][1], a1, b1);
      }
    }
    if (SYNC) __syncthreads();
  }
  double s = 0;
  for (int e = 0; e < 8; ++e) s += acc[e >> 2][(e >> 1) & 1][e & 1];
  if (s == 1234.5) out[0] = s;
}
template <typename K>
void run(const char* name, K k) {
  double* out;
  cudaMalloc(&out, 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int tiles = 20000;
  k<<<nsm, 256>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<nsm, 256>>>(out, tiles);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = (double)nsm * tiles * 2.0 * (2.0 * TB * TB * NC);  // N + T per tile
  printf("%-24s %7.2f TFLOP/s  %.3f us/tile  err=%s\n", name, fl / (ms * 1e-3) / 1e12, ms * 1e3 / tiles,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run("nosync unroll8", kpass<0, 8>);
  run("sync unroll8", kpass<1, 8>);
  run("nosync unroll16", kpass<0, 16>);
  run("sync unroll16", kpass<1, 16>);
  run("nosync unroll4", kpass<0, 4>);
  return 0;
}
