// Batched supernodal (multifrontal) Cholesky of every subdomain's K_rr^(k)
// (SURVEY §8(a) a3).
//
// All supernodes of one elimination-tree level, over ALL subdomains, are one
// batch. Per level:
//   1. zero the level's fronts and scatter the original entries of K_rr;
//   2. extend-add the children's update matrices (one launch per child slot:
//      deterministic, no atomics);
//   3. right-looking partial Cholesky over the pivot columns in TB-wide panels:
//      POTRF of the TB x TB diagonal block (+ its inverse Dinv), TRSM of the
//      panel as a DMMA GEMM with Dinv^T, DMMA SYRK/GEMM trailing update of the
//      rest of the front (remaining pivots and the update block).
// The root front of subdomain k holds r_I, so its factor is L_II with
// L_II L_II^T = S_{r_I r_I} (F2).
#include <climits>

#include "common.cuh"

namespace ieti {

__global__ void k_scatter(long long n, const long long* __restrict__ dst, const int* __restrict__ src,
                          const double* __restrict__ vals, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[dst[i]] = vals[src[i]];
}

// Work item (child c, column range [a, b)): F_parent[rel[i], rel[j]] += U_c[i, j].
__global__ void k_extend_add(const Work* __restrict__ work, const SnDev* __restrict__ sn,
                             const int* __restrict__ rel, double* __restrict__ pool) {
  const Work w = work[blockIdx.x];
  const SnDev c = sn[w.sn];
  const SnDev p = sn[c.parent];
  const int nu = c.f - c.npiv;
  const double* U = pool + c.front_off + (long long)c.npiv * c.ld + c.npiv;
  double* F = pool + p.front_off;
  const int* rl = rel + c.rel_off;
  for (int j = w.a; j < w.b; ++j) {
    const long long pc = (long long)rl[j] * p.ld;
    const double* Uj = U + (long long)j * c.ld;
    for (int i = j + threadIdx.x; i < nu; i += blockDim.x) F[pc + rl[i]] += Uj[i];
  }
}

// POTRF of the diagonal block of panel w.a of front w.sn, and its inverse.
// Dynamic smem: A[TB][TB+1], X[TB][TB+1].
__global__ void __launch_bounds__(256) k_potrf(const Work* __restrict__ work, const SnDev* __restrict__ sn,
                                               double* __restrict__ pool, double* __restrict__ dinv,
                                               int* __restrict__ err) {
  extern __shared__ double sm[];
  double(*A)[TB + 1] = reinterpret_cast<double(*)[TB + 1]>(sm);
  double(*X)[TB + 1] = reinterpret_cast<double(*)[TB + 1]>(sm + TB * (TB + 1));
  __shared__ int bad;
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const int p0 = w.a * TB;
  const int b = min(TB, s.npiv - p0);
  double* F = pool + s.front_off + (long long)p0 * s.ld + p0;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < TB * TB; e += blockDim.x) {
    int c = e / TB, r = e % TB;  // column-major walk: coalesced along r
    double v;
    if (r < b && c < b) v = (r >= c) ? F[(long long)c * s.ld + r] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    A[r][c] = v;
    X[r][c] = 0.0;
  }
  __syncthreads();
  // right-looking unblocked Cholesky (column j)
  for (int j = 0; j < TB; ++j) {
    if (tid == 0) {
      double d = A[j][j];
      if (!(d > 0.0)) {
        bad = 1;
        d = 1.0;
      }
      A[j][j] = sqrt(d);
    }
    __syncthreads();
    const double inv = 1.0 / A[j][j];
    for (int i = j + 1 + tid; i < TB; i += blockDim.x) A[i][j] *= inv;
    __syncthreads();
    // trailing update: rows i > j, columns j < c <= i
    {
      const int r = tid & 63, cg = tid >> 6;  // 64 rows x 4 column groups
      if (r > j) {
        const double lij = A[r][j];
        for (int c = j + 1 + cg; c <= r; c += 4) A[r][c] -= lij * A[c][j];
      }
    }
    __syncthreads();
  }
  if (tid == 0 && bad) atomicMin(err, s.sub);
  // write back L (lower) of the valid b x b block
  for (int e = tid; e < TB * TB; e += blockDim.x) {
    int c = e / TB, r = e % TB;
    if (r < b && c < b && r >= c) F[(long long)c * s.ld + r] = A[r][c];
  }
  // X = A^-1 (lower), row by row: X[i][c] = -(sum_{m=c}^{i-1} A[i][m] X[m][c]) / A[i][i]
  if (tid < TB) X[tid][tid] = 1.0 / A[tid][tid];
  __syncthreads();
  for (int i = 1; i < TB; ++i) {
    const int c = tid >> 2, part = tid & 3;  // 64 columns x 4 partial sums
    double sum = 0.0;
    if (c < i)
      for (int m = c + part; m < i; m += 4) sum += A[i][m] * X[m][c];
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    if (c < i && part == 0) X[i][c] = -sum * X[i][i];
    __syncthreads();
  }
  double* D = dinv + s.dinv_off + (long long)w.a * TILE_ELEMS;  // column-major TB x TB
  for (int e = tid; e < TB * TB; e += blockDim.x) {
    int c = e / TB, r = e % TB;
    D[e] = (r < b && c < b && r >= c) ? X[r][c] : 0.0;
  }
}

// DMMA tile GEMM on a front: C(TB x TB) = / -= A(TB x kb) * B(TB x kb)^T, 4 warps
// each owning a 32 x 32 quadrant (4 x 4 m8n8 blocks).
//   MODE 0 (TRSM):   rows tile w.b below the diagonal block; A = panel rows,
//                    B = Dinv (row j, col m = Dinv[j][m]); C overwrites A.
//   MODE 1 (update): tile pair (ti, tj) = (w.b >> 16, w.b & 0xffff) of the
//                    trailing matrix; A = panel rows ti, B = panel rows tj; C -= .
// Dynamic smem: As[TB][72], Bs[TB][72] (k-major; stride 72 = conflict-free frags).
constexpr int KS = 72;
template <int MODE>
__global__ void __launch_bounds__(128) k_panel_gemm(const Work* __restrict__ work, const SnDev* __restrict__ sn,
                                                    double* __restrict__ pool, const double* __restrict__ dinv) {
  extern __shared__ double sm[];
  double* As = sm;
  double* Bs = sm + TB * KS;
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const int p0 = w.a * TB;
  const int kb = min(TB, s.npiv - p0);
  const int start = p0 + kb;
  double* F = pool + s.front_off;
  const long long ld = s.ld;
  int ti, tj;
  if (MODE == 0) {
    ti = w.b;
    tj = 0;
  } else {
    ti = w.b >> 16;
    tj = w.b & 0xffff;
  }
  const int r0 = start + ti * TB;  // first front row of the C tile
  const int c0 = start + tj * TB;  // MODE 1: first front column of the C tile
  const int tid = threadIdx.x;
  // load A: As[k][r] = F[p0 + k][r0 + r]
  for (int e = tid; e < TB * TB; e += 128) {
    int k = e / TB, r = e % TB;
    double v = 0.0;
    if (k < kb && r0 + r < s.f) v = F[(long long)(p0 + k) * ld + r0 + r];
    As[k * KS + r] = v;
  }
  if (MODE == 0) {
    const double* D = dinv + s.dinv_off + (long long)w.a * TILE_ELEMS;
    for (int e = tid; e < TB * TB; e += 128) {
      int k = e / TB, j = e % TB;
      Bs[k * KS + j] = D[e];  // D column-major: D[j + TB*k] = Dinv[j][k]
    }
  } else {
    for (int e = tid; e < TB * TB; e += 128) {
      int k = e / TB, r = e % TB;
      double v = 0.0;
      if (k < kb && c0 + r < s.f) v = F[(long long)(p0 + k) * ld + c0 + r];
      Bs[k * KS + r] = v;
    }
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int kend = (kb + 3) & ~3;
  for (int k0 = 0; k0 < kend; k0 += 4) {
    double a[4], bb[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = As[(k0 + t) * KS + wm + i * 8 + g];
#pragma unroll
    for (int j = 0; j < 4; ++j) bb[j] = Bs[(k0 + t) * KS + wn + j * 8 + g];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
  }
  if (MODE == 0) __syncthreads();  // (As is not re-read; kept for clarity of the in-place write)
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int rr = wm + i * 8 + g;
        const int cc = wn + j * 8 + 2 * t + q;
        const int R = r0 + rr;
        if (R >= s.f) continue;
        if (MODE == 0) {
          if (cc < kb) F[(long long)(p0 + cc) * ld + R] = acc[i][j][q];
        } else {
          const int C = c0 + cc;
          if (C < s.f && R >= C) F[(long long)C * ld + R] -= acc[i][j][q];
        }
      }
}

// General batched tile GEMM (DMMA): C = (+/-) A * B (+ C) on one <= TB x TB tile
// per CTA, K looped in TB chunks; column-major operands in three base arrays
// (GemmWork). Used for the partitioned inverse L11^-1 (recursive doubling).
template <int NEG_BIT_UNUSED>
__global__ void __launch_bounds__(128) k_tgemm(const GemmWork* __restrict__ work, const double* __restrict__ Ab,
                                               const double* __restrict__ Bb, double* __restrict__ Cb) {
  extern __shared__ double sm[];
  double* As = sm;            // [k][r], stride KS
  double* Bs = sm + TB * KS;  // [k][c], stride KS
  const GemmWork w = work[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kk = 0; kk < w.kdim; kk += TB) {
    const int kb = min(TB, w.kdim - kk);
    __syncthreads();
    for (int e = tid; e < TB * TB; e += 128) {
      const int k = e / TB, r = e % TB;  // A column k contiguous in r
      As[k * KS + r] = (k < kb && r < w.m) ? Ab[w.a_off + (long long)(kk + k) * w.lda + r] : 0.0;
    }
    for (int e = tid; e < TB * TB; e += 128) {
      const int c = e / TB, k = e % TB;  // B column c contiguous in k
      Bs[k * KS + c] = (k < kb && c < w.n) ? Bb[w.b_off + (long long)c * w.ldb + kk + k] : 0.0;
    }
    __syncthreads();
    const int kend = (kb + 3) & ~3;
    for (int k0 = 0; k0 < kend; k0 += 4) {
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[(k0 + t) * KS + wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[(k0 + t) * KS + wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
    }
  }
  const double sgn = (w.mode & 1) ? -1.0 : 1.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = wm + i * 8 + g, c = wn + j * 8 + 2 * t + q;
        if (r < w.m && c < w.n) {
          double* C = Cb + w.c_off + (long long)c * w.ldc + r;
          *C = (w.mode & 2) ? *C + sgn * acc[i][j][q] : sgn * acc[i][j][q];
        }
      }
}

// Diagonal TB-blocks of L11^-1 are the Dinv blocks of the panels.
__global__ void k_inv_copy(const Work* __restrict__ work, const SnDev* __restrict__ sn, const double* __restrict__ dinv,
                           double* __restrict__ ipool) {
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const int p0 = w.a * TB, b = min(TB, s.npiv - p0);
  const double* D = dinv + s.dinv_off + (long long)w.a * TILE_ELEMS;
  double* I = ipool + s.inv_off + (long long)p0 * s.ldi + p0;
  for (int e = threadIdx.x; e < TILE_ELEMS; e += blockDim.x) {
    const int c = e / TB, r = e % TB;
    if (r < b && c < b) I[(long long)c * s.ldi + r] = D[e];
  }
}

static void set_smem(const void* f, int bytes) {
  IETI_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void run_factor(ietidp_s* h) {
  cudaStream_t st = h->stream;
  const Plan& P = h->plan;
  static bool attr = false;
  const int sm_potrf = 2 * TB * (TB + 1) * sizeof(double);
  const int sm_gemm = 2 * TB * KS * sizeof(double);
  if (!attr) {
    set_smem((const void*)k_potrf, sm_potrf);
    set_smem((const void*)k_panel_gemm<0>, sm_gemm);
    set_smem((const void*)k_panel_gemm<1>, sm_gemm);
    set_smem((const void*)k_tgemm<0>, sm_gemm);
    attr = true;
  }
  static const int init_flags[2] = {INT_MAX, 1};  // failing subdomain (min), coarse OK
  IETI_CUDA(cudaMemcpyAsync(h->err_flag.p, init_flags, 2 * sizeof(int), cudaMemcpyHostToDevice, st));
  const Work* W = reinterpret_cast<const Work*>(h->d_work.p);
  for (int L = 0; L <= P.max_level; ++L) {
    const LevelPlan& lp = P.levels[L];
    if (lp.front_end > lp.front_begin)
      IETI_CUDA(cudaMemsetAsync(h->pool.p + lp.front_begin, 0,
                                (lp.front_end - lp.front_begin) * sizeof(double), st));
    long long ne = lp.scat_end - lp.scat_begin;
    if (ne > 0) {
      k_scatter<<<grid_for(ne, 256), 256, 0, st>>>(ne, h->sc_front_dst.p + lp.scat_begin,
                                                   h->sc_front_src.p + lp.scat_begin, h->kval.p, h->pool.p);
      IETI_LAUNCHED(h);
    }
    for (auto& ea : lp.ea) {
      k_extend_add<<<ea.second, 128, 0, st>>>(W + ea.first, h->d_sn.p, h->d_rel.p, h->pool.p);
      IETI_LAUNCHED(h);
    }
    for (auto& pn : lp.panels) {
      if (pn.potrf_n) {
        k_potrf<<<pn.potrf_n, 256, sm_potrf, st>>>(W + pn.potrf_off, h->d_sn.p, h->pool.p, h->dinv.p,
                                                  h->err_flag.p);
        IETI_LAUNCHED(h);
      }
      if (pn.trsm_n) {
        k_panel_gemm<0><<<pn.trsm_n, 128, sm_gemm, st>>>(W + pn.trsm_off, h->d_sn.p, h->pool.p, h->dinv.p);
        IETI_LAUNCHED(h);
      }
      if (pn.upd_n) {
        k_panel_gemm<1><<<pn.upd_n, 128, sm_gemm, st>>>(W + pn.upd_off, h->d_sn.p, h->pool.p, h->dinv.p);
        IETI_LAUNCHED(h);
      }
    }
  }
  // partitioned inverse L11^-1 of every factored supernode (all at once)
  if (P.inv_copy_n) {
    k_inv_copy<<<P.inv_copy_n, 256, 0, st>>>(W + P.inv_copy_off, h->d_sn.p, h->dinv.p, h->ipool.p);
    IETI_LAUNCHED(h);
  }
  for (size_t r = 0; r < P.inv_rounds.size(); ++r) {
    const auto& rg = P.inv_rounds[r];
    if (!rg.second) continue;
    const bool step1 = (r % 2) == 0;
    k_tgemm<0><<<rg.second, 128, sm_gemm, st>>>(h->d_gwork.p + rg.first, step1 ? h->pool.p : h->ipool.p,
                                                step1 ? h->ipool.p : h->tpool.p, step1 ? h->tpool.p : h->ipool.p);
    IETI_LAUNCHED(h);
  }
  IETI_CHECK_LAUNCH();
}

}  // namespace ieti
