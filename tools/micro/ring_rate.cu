// Tile-stream ring of the chunk pass in isolation: 32 KB tiles from a large global array
// (each CTA its own contiguous range; DRAM) by cp.async.bulk + mbarrier into an S-deep
// ring, 8 warps, per tile optionally the pass's DMMA loops (N warps 0-3, T warps 4-7),
// slot release by arrival counting (last warp issues the slot's next copy) or by
// __syncthreads + thread 0. Reports us per tile.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ring_rate ring_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int TB = 64, NC = 16, TE = TB * TB;
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  do {
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void issue_copy(double* dst, const double* src, uint64_t* bar, unsigned long long pol) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(TE * 8) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
               ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(TE * 8), "r"(b), "l"(pol) : "memory");
}
template <int S, bool COMPUTE, bool SYNCREL>
__global__ void __launch_bounds__(256, 1) kring(const double* __restrict__ tiles, int ntiles, double* out) {
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;
  double* X = sm + S * TE;
  __shared__ uint64_t full[S];
  __shared__ unsigned rel[S];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  for (int e = tid; e < TB * NC; e += 256) X[e] = 1e-2 * (e % 31);
  if (tid == 0)
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      rel[s] = 0;
    }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const double* src = tiles + (long long)blockIdx.x * ntiles * TE;
  if (tid == 0)
    for (int i = 0; i < S && i < ntiles; ++i) issue_copy(ring + i * TE, src + (long long)i * TE, &full[i], pol);
  const int q4 = warp & 3, r0 = 16 * q4 + g;
  const bool tw = warp >= 4;
  int acol[4];
  for (int kl = 0; kl < 4; ++kl) acol[kl] = 4 * (kl ^ (g & 3)) + t4;
  const int at0 = t4 * TB + (r0 ^ (t4 << 2)), at1 = t4 * TB + ((r0 + 8) ^ (t4 << 2));
  const int xb0 = t4 * NC + (g ^ (t4 << 2)), xb1 = t4 * NC + ((g ^ (t4 << 2)) ^ 8);
  double acc[2][2][2] = {};
  for (int i = 0; i < ntiles; ++i) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1);
    const double* T = ring + s * TE;
    if (COMPUTE) {
      if (!tw) {
#pragma unroll 8
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
#pragma unroll 8
        for (int k0 = 0; k0 < TB; k0 += 4) {
          const double a0 = T[at0 + k0 * TB], a1 = T[at1 + k0 * TB];
          const double b0 = X[xb0 + k0 * NC], b1 = X[xb1 + k0 * NC];
          dmma(acc[0][0][0], acc[0][0][1], a0, b0);
          dmma(acc[0][1][0], acc[0][1][1], a1, b0);
          dmma(acc[1][0][0], acc[1][0][1], a0, b1);
          dmma(acc[1][1][0], acc[1][1][1], a1, b1);
        }
      }
    } else {
      acc[0][0][0] += T[tid];
    }
    if (SYNCREL) {
      __syncthreads();
      if (tid == 0 && i + S < ntiles) issue_copy(ring + s * TE, src + (long long)(i + S) * TE, &full[s], pol);
    } else {
      __syncwarp();
      if (lane == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;\n" : "=r"(old)
                     : "r"((unsigned)__cvta_generic_to_shared(&rel[s])) : "memory");
        if (old == 8u * (i / S) + 7u && i + S < ntiles) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          issue_copy(ring + s * TE, src + (long long)(i + S) * TE, &full[s], pol);
        }
      }
    }
  }
  double sacc = 0;
  for (int e = 0; e < 8; ++e) sacc += acc[e >> 2][(e >> 1) & 1][e & 1];
  if (sacc == 1234.5) out[0] = sacc;
}
template <int S, bool C, bool SR>
void run(const double* tiles, int ntiles, double* out, int nsm) {
  auto k = kring<S, C, SR>;
  const int smem = (S * TE + TB * NC) * 8;
  cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<nsm, 256, smem>>>(tiles, 8, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<nsm, 256, smem>>>(tiles, ntiles, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("S=%d compute=%d syncrel=%d: %.3f us/tile, %.0f GB/s  err=%s\n", S, (int)C, (int)SR, ms * 1e3 / ntiles,
         (double)nsm * ntiles * TE * 8 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int ntiles = 200;  // 148 x 200 x 32 KB = 970 MB: DRAM
  double *tiles, *out;
  cudaMalloc(&tiles, (size_t)nsm * ntiles * TE * 8);
  cudaMemset(tiles, 0, (size_t)nsm * ntiles * TE * 8);
  cudaMalloc(&out, 8);
  run<2, false, false>(tiles, ntiles, out, nsm);
  run<3, false, false>(tiles, ntiles, out, nsm);
  run<4, false, false>(tiles, ntiles, out, nsm);
  run<6, false, false>(tiles, ntiles, out, nsm);
  run<2, true, false>(tiles, ntiles, out, nsm);
  run<3, true, false>(tiles, ntiles, out, nsm);
  run<4, true, false>(tiles, ntiles, out, nsm);
  run<6, true, false>(tiles, ntiles, out, nsm);
  run<3, true, true>(tiles, ntiles, out, nsm);
  run<6, true, true>(tiles, ntiles, out, nsm);
  return 0;
}
