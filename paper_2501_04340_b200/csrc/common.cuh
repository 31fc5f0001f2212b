// Device helpers shared by the CUDA translation units of libietidp.so.
#pragma once
#include <cuda_runtime.h>

#include "handle.h"
#include "impl.h"

namespace ieti {

// FP64 tensor-core MMA (sm_80+ DMMA; on sm_100a it lowers to SASS DMMA):
// D(8x8) += A(8x4, row) * B(4x8, col).  Fragments (PTX ISA, mma.m8n8k4 .f64):
//   a0 = A[lane>>2][lane&3], b0 = B[lane&3][lane>>2],
//   {d0,d1} = D[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Swizzled position of element (r, m) of a TB x TB row-major tile: the 4-double
// groups of a row are XOR-permuted by (r & 3), so that the 16 lanes of each half-warp
// of an 8-byte DMMA fragment load -- 4 rows x 4 consecutive columns, row-wise
// (A = S) or column-wise (A = S^T) -- hit 16 distinct bank pairs (measured: the
// previous (r & 7) permutation of 16-byte chunks left every LDS.64 2-way
// conflicted, ncu profiles/r02_pcg_c5_chunk_raw.txt). The loop's tiles
// (L_II, L_II^-1, W_k = S_II^-1, S_II) are STORED in this layout in global memory,
// so that a tile moves into shared memory as one contiguous 32 KB copy (one
// cp.async.bulk, or linear 16-byte cp.async).
__device__ __forceinline__ int swz(int r, int m) { return r * TB + (m ^ ((r & 3) << 2)); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

inline int grid_for(long long n, int block, int cap = 148 * 16) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// Every kernel launch is counted; with IETIDP_TRACE=<file> set, an event is also
// recorded after it (per-launch device durations, written by the API at the end of
// factor / solve; a diagnostics aid, off by default).
#define IETI_LAUNCHED(h)                                                   \
  do {                                                                     \
    (h)->launches++;                                                       \
    if ((h)->trace.on) (h)->trace.mark((h)->stream, __FILE__, __LINE__);   \
  } while (0)
#define IETI_LAUNCHED_SIDE(h) \
  do {                        \
    (h)->launches++;          \
  } while (0)

#define IETI_CHECK_LAUNCH() IETI_CUDA(cudaGetLastError())

}  // namespace ieti
