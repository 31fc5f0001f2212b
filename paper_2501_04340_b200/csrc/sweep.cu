// Batched multifrontal triangular sweeps with the supernodal factor:
// X_k <- K_rr^(k)^-1 X_k for every subdomain at once, multi-RHS
// (coarse basis K_rr^-1 K_rP, y = K_rr^-1 j_r, recovery
// a_r = K_rr^-1(...) of Eq. (9)).
//
// X_k is row-major (n_r x ncols) in the subdomain's r ordering. One CTA per
// supernode, all supernodes of a level (all subdomains) in one launch.
// Forward (leaves -> root): the front vector v = [x_piv; 0] plus the children's
// update vectors (fixed child order, deterministic), y_piv = L11^-1 v_piv using
// the inverted diagonal blocks, v_upd -= L21 y_piv is kept for the parent.
// Backward (root -> leaves): x_piv = L11^-T (y_piv - L21^T x_rows).
#include "common.cuh"

namespace ieti {

constexpr int SW_THREADS = 256;

__global__ void __launch_bounds__(SW_THREADS)
    k_sweep_fwd(const int* __restrict__ lst, const SnDev* __restrict__ sn, const SubDev* __restrict__ sub,
                const int* __restrict__ rel, const int* __restrict__ children, const double* __restrict__ pool,
                const double* __restrict__ dinv, double* __restrict__ X, double* __restrict__ Wv, int ncols) {
  extern __shared__ double ys[];  // TB x ncols
  const SnDev s = sn[lst[blockIdx.x]];
  const SubDev d = sub[s.sub];
  const int tid = threadIdx.x;
  double* v = Wv + s.vec_off * ncols;
  double* x = X + (d.x_off + s.c0) * ncols;
  const int np = s.npiv * ncols, nf = s.f * ncols;
  for (int e = tid; e < nf; e += SW_THREADS) v[e] = (e < np) ? x[e] : 0.0;
  __syncthreads();
  for (int ci = 0; ci < s.nchild; ++ci) {
    const SnDev c = sn[children[s.child_off + ci]];
    const int nu = c.f - c.npiv;
    const double* uc = Wv + (c.vec_off + c.npiv) * ncols;
    const int* rl = rel + c.rel_off;
    for (int e = tid; e < nu * ncols; e += SW_THREADS) {
      int i = e / ncols, cc = e - i * ncols;
      v[rl[i] * ncols + cc] += uc[e];
    }
    __syncthreads();
  }
  const double* F = pool + s.front_off;
  for (int p0 = 0, kp = 0; p0 < s.npiv; p0 += TB, ++kp) {
    const int b = min(TB, s.npiv - p0);
    const double* D = dinv + s.dinv_off + (long long)kp * TILE_ELEMS;  // col-major
    for (int e = tid; e < b * ncols; e += SW_THREADS) {
      int r = e / ncols, cc = e - r * ncols;
      double sum = 0.0;
      for (int m = 0; m <= r; ++m) sum += D[r + TB * m] * v[(p0 + m) * ncols + cc];
      ys[e] = sum;
    }
    __syncthreads();
    for (int e = tid; e < b * ncols; e += SW_THREADS) v[p0 * ncols + e] = ys[e];
    // rows below the block: v[i] -= L[i, p0:p0+b] * y
    for (int i = p0 + b + tid; i < s.f; i += SW_THREADS) {
      for (int c0 = 0; c0 < ncols; c0 += 8) {
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int cn = min(8, ncols - c0);
        for (int m = 0; m < b; ++m) {
          const double l = F[(long long)(p0 + m) * s.ld + i];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < cn) acc[q] += l * ys[m * ncols + c0 + q];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < cn) v[i * ncols + c0 + q] -= acc[q];
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < np; e += SW_THREADS) x[e] = v[e];
}

__global__ void __launch_bounds__(SW_THREADS)
    k_sweep_bwd(const int* __restrict__ lst, const SnDev* __restrict__ sn, const SubDev* __restrict__ sub,
                const int* __restrict__ rows, const double* __restrict__ pool, const double* __restrict__ dinv,
                double* __restrict__ X, double* __restrict__ Wv, int ncols) {
  extern __shared__ double ys[];  // TB x ncols
  const SnDev s = sn[lst[blockIdx.x]];
  const SubDev d = sub[s.sub];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = SW_THREADS / 32;
  double* v = Wv + s.vec_off * ncols;
  double* x = X + (d.x_off + s.c0) * ncols;
  const double* Xs = X + d.x_off * ncols;
  const int nu = s.f - s.npiv;
  const int* rw = rows + s.rows_off;
  for (int e = tid; e < s.f * ncols; e += SW_THREADS) {
    int i = e / ncols, cc = e - i * ncols;
    v[e] = (i < s.npiv) ? x[e] : Xs[rw[i - s.npiv] * ncols + cc];
  }
  __syncthreads();
  const double* F = pool + s.front_off;
  // t = y - L21^T x_rows : warp per pivot column
  if (nu > 0) {
    for (int i = warp; i < s.npiv; i += nwarps) {
      const double* Li = F + (long long)i * s.ld + s.npiv;
      for (int c0 = 0; c0 < ncols; c0 += 8) {
        const int cn = min(8, ncols - c0);
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int j = lane; j < nu; j += 32) {
          const double l = Li[j];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < cn) acc[q] += l * v[(s.npiv + j) * ncols + c0 + q];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          double a = warp_sum(acc[q]);
          if (lane == 0 && q < cn) v[i * ncols + c0 + q] -= a;
        }
      }
    }
    __syncthreads();
  }
  const int npan = (s.npiv + TB - 1) / TB;
  for (int kp = npan - 1; kp >= 0; --kp) {
    const int p0 = kp * TB;
    const int b = min(TB, s.npiv - p0);
    const double* D = dinv + s.dinv_off + (long long)kp * TILE_ELEMS;  // col-major
    // x_b = Dinv^T t_b : x[r] = sum_{m >= r} D[m][r] t[m]
    for (int e = tid; e < b * ncols; e += SW_THREADS) {
      int r = e / ncols, cc = e - r * ncols;
      double sum = 0.0;
      for (int m = r; m < b; ++m) sum += D[m + TB * r] * v[(p0 + m) * ncols + cc];
      ys[e] = sum;
    }
    __syncthreads();
    for (int e = tid; e < b * ncols; e += SW_THREADS) v[p0 * ncols + e] = ys[e];
    // earlier pivots: t[i] -= sum_m L11[p0+m][i] x_b[m], warp per column i < p0
    for (int i = warp; i < p0; i += nwarps) {
      const double* Li = F + (long long)i * s.ld + p0;
      for (int c0 = 0; c0 < ncols; c0 += 8) {
        const int cn = min(8, ncols - c0);
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int m = lane; m < b; m += 32) {
          const double l = Li[m];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < cn) acc[q] += l * ys[m * ncols + c0 + q];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          double a = warp_sum(acc[q]);
          if (lane == 0 && q < cn) v[i * ncols + c0 + q] -= a;
        }
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < s.npiv * ncols; e += SW_THREADS) x[e] = v[e];
}

// X <- K_rr^-1 X for all subdomains (row-major X, ncols columns).
void run_sweeps(ietidp_s* h, double* X, int ncols) {
  cudaStream_t st = h->stream;
  const Plan& P = h->plan;
  const int smem = TB * ncols * sizeof(double);
  if (smem > 48 * 1024) {
    IETI_CUDA(cudaFuncSetAttribute((const void*)k_sweep_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    IETI_CUDA(cudaFuncSetAttribute((const void*)k_sweep_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  for (int L = 0; L <= P.max_level; ++L) {
    const LevelPlan& lp = P.levels[L];
    if (!lp.sn_n) continue;
    k_sweep_fwd<<<lp.sn_n, SW_THREADS, smem, st>>>(h->d_level_sn.p + lp.sn_off, h->d_sn.p, h->d_sub.p, h->d_rel.p,
                                                   h->d_children.p, h->pool.p, h->dinv.p, X, h->vecw.p, ncols);
    IETI_LAUNCHED(h);
  }
  for (int L = P.max_level; L >= 0; --L) {
    const LevelPlan& lp = P.levels[L];
    if (!lp.sn_n) continue;
    k_sweep_bwd<<<lp.sn_n, SW_THREADS, smem, st>>>(h->d_level_sn.p + lp.sn_off, h->d_sn.p, h->d_sub.p, h->d_rows.p,
                                                   h->pool.p, h->dinv.p, X, h->vecw.p, ncols);
    IETI_LAUNCHED(h);
  }
  IETI_CHECK_LAUNCH();
}

}  // namespace ieti
