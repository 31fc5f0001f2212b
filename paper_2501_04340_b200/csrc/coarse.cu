// Coarse set-up, RHS and recovery:
//   X_k = K_rr^-1 [K_rP | j_r]                      (multifrontal sweeps)
//   S_PP = sum_k C_k^T (K_PP - K_Pr X_P) C_k       (SPD sign)
//   ftilde = sum_k C_k^T (j_P - K_Pr y_k)           (SPD sign)
//   G_k = X_k[r_I, P],  e = sum_k B y_k[r_I]
//   S_PP = L L^T, S_PP^-1 = L^-T L^-1 (one CTA)
//   d_DP = e - G S_PP^-1 ftilde                     (R1)
// plus the Dirichlet-scaling weights, the tile-major repacking of L_II for the
// loop, and the recovery p = S_PP^-1(ftilde + G^T lambda) (Eq. 8),
// a_r = K_rr^-1 (j_r - K_rP C_k p - B_r^T lambda) (Eq. 9).
#include <climits>

#include "common.cuh"

namespace ieti {

void run_sweeps(ietidp_s* h, double* X, int ncols);
void bgather_public(ietidp_s* h, int ncols, const double* x, const double* z, double coef, double* out);
void coarse_apply_public(ietidp_s* h, int ncols, const double* gk, const double* add, double* z);
__global__ void k_scatter(long long n, const long long* __restrict__ dst, const int* __restrict__ src,
                          const double* __restrict__ vals, double* __restrict__ out);

// Local coarse blocks, one CTA per subdomain (warp per output entry).
__global__ void __launch_bounds__(256)
    k_coarse_local(const SubDev* __restrict__ sub, int ncx, int nPmax, int nrhs, const double* __restrict__ X0,
                   const double* __restrict__ X, const double* __restrict__ kpp, const double* __restrict__ jp,
                   double* __restrict__ sloc, double* __restrict__ floc, double* __restrict__ G,
                   double* __restrict__ yI) {
  const SubDev d = sub[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* x0 = X0 + d.x_off * ncx;
  const double* x = X + d.x_off * ncx;
  const int nP = d.nP;
  // S_loc[a][b] = K_PP[a][b] - sum_i K_rP[i][a] X[i][b];  f_loc[a][c] = j_P[a][c] - sum_i K_rP[i][a] y[i][c]
  const int nent = nP * nP + nP * nrhs;
  for (int e = warp; e < nent; e += 8) {
    int a, col;
    bool isS = e < nP * nP;
    if (isS) {
      a = e / nP;
      col = e - a * nP;
    } else {
      int f = e - nP * nP;
      a = f / nrhs;
      col = nPmax + (f - a * nrhs);
    }
    double s = 0.0;
    for (int i = lane; i < d.nr; i += 32) s += x0[(long long)i * ncx + a] * x[(long long)i * ncx + col];
    s = warp_sum(s);
    if (lane == 0) {
      if (isS) sloc[d.sloc_off + e] = kpp[d.kpp_off + e] - s;
      else {
        int f = e - nP * nP;
        floc[d.floc_off + f] = jp[d.jp_off + f] - s;
      }
    }
  }
  // G_k = X[r_I rows, P cols] (row-major nI x nP); y_I (e-part)
  for (int e = threadIdx.x; e < d.nI * nP; e += blockDim.x) {
    const int a = e / nP, b = e - a * nP;
    G[d.g_off + e] = x[(long long)(d.nV + a) * ncx + b];
  }
  for (int e = threadIdx.x; e < d.nI * nrhs; e += blockDim.x) {
    const int a = e / nrhs, c = e - a * nrhs;
    yI[(d.rI_off + a) * nrhs + c] = x[(long long)(d.nV + a) * ncx + nPmax + c];
  }
}

// S_PP assembly (deterministic: fixed contribution lists), symmetrisation,
// Cholesky, inverse, and zc0 = S^-1 ftilde. One CTA of 1024 threads; the lower
// triangle lives packed in shared memory (n(n+1)/2 doubles).
__device__ __forceinline__ int pk(int i, int j) { return i * (i + 1) / 2 + j; }

__global__ void __launch_bounds__(1024)
    k_coarse_factor(int n, int nrhs, const int* __restrict__ scoef_ptr, const int* __restrict__ scoef_src,
                    const double* __restrict__ sloc, const int* __restrict__ pcon_ptr,
                    const int* __restrict__ pcon_src, const double* __restrict__ floc, double* __restrict__ S,
                    double* __restrict__ Sinv, double* __restrict__ ftil, double* __restrict__ zc0,
                    int* __restrict__ err) {
  extern __shared__ double Lp[];  // n(n+1)/2
  __shared__ double tmp[1024];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < n * n; e += blockDim.x) {
    double s = 0.0;
    for (int q = scoef_ptr[e]; q < scoef_ptr[e + 1]; ++q) s += sloc[scoef_src[q]];
    S[e] = s;
  }
  for (int e = tid; e < n * nrhs; e += blockDim.x) {
    const int g = e / nrhs, c = e - g * nrhs;
    double s = 0.0;
    for (int q = pcon_ptr[g]; q < pcon_ptr[g + 1]; ++q) s += floc[(long long)pcon_src[q] * nrhs + c];
    ftil[e] = s;
  }
  __syncthreads();
  for (int e = tid; e < n * (n + 1) / 2; e += blockDim.x) {
    int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while (pk(i, 0) > e) --i;
    while (pk(i + 1, 0) <= e) ++i;
    const int j = e - pk(i, 0);
    Lp[e] = 0.5 * (S[i * n + j] + S[j * n + i]);
  }
  __syncthreads();
  // Cholesky (right-looking)
  for (int j = 0; j < n; ++j) {
    if (tid == 0) {
      double dd = Lp[pk(j, j)];
      if (!(dd > 0.0)) {
        bad = 1;
        dd = 1.0;
      }
      Lp[pk(j, j)] = sqrt(dd);
    }
    __syncthreads();
    const double inv = 1.0 / Lp[pk(j, j)];
    for (int i = j + 1 + tid; i < n; i += blockDim.x) Lp[pk(i, j)] *= inv;
    __syncthreads();
    for (int i = j + 1 + (tid >> 3); i < n; i += (blockDim.x >> 3)) {
      const double lij = Lp[pk(i, j)];
      for (int c = j + 1 + (tid & 7); c <= i; c += 8) Lp[pk(i, c)] -= lij * Lp[pk(c, j)];
    }
    __syncthreads();
  }
  if (tid == 0 && bad) atomicMin(err + 1, 0);
  // in-place inverse of the lower factor (LAPACK trti2, lower, backward)
  for (int j = n - 1; j >= 0; --j) {
    if (tid == 0) Lp[pk(j, j)] = 1.0 / Lp[pk(j, j)];
    __syncthreads();
    const double ajj = -Lp[pk(j, j)];
    for (int i = j + 1 + tid; i < n; i += blockDim.x) tmp[i] = Lp[pk(i, j)];
    __syncthreads();
    // X[i][j] = ajj * sum_{m=j+1}^{i} Xinv[i][m] tmp[m]
    for (int base = j + 1; base < n; base += (blockDim.x >> 3)) {  // warp-uniform trip count
      const int i = base + (tid >> 3);
      double s = 0.0;
      if (i < n)
        for (int m = j + 1 + (tid & 7); m <= i; m += 8) s += Lp[pk(i, m)] * tmp[m];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      if (i < n && (tid & 7) == 0) Lp[pk(i, j)] = ajj * s;
    }
    __syncthreads();
  }
  // S^-1 = X^T X, X = L^-1 lower: Sinv[i][j] = sum_{m >= max(i,j)} X[m][i] X[m][j]
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    double s = 0.0;
    for (int m = max(i, j); m < n; ++m) s += Lp[pk(m, i)] * Lp[pk(m, j)];
    Sinv[e] = s;
  }
  __syncthreads();
  for (int e = tid; e < n * nrhs; e += blockDim.x) {
    const int i = e / nrhs, c = e - i * nrhs;
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += Sinv[i * n + j] * ftil[j * nrhs + c];
    zc0[e] = s;
  }
}

// Dirichlet scaling weights (R5).
__global__ void k_scaling(int m, const LamDev* __restrict__ lam, const int* __restrict__ kdiag_src,
                          const double* __restrict__ kval, double* __restrict__ kdiag, double* __restrict__ delta,
                          int stiffness) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    const int a = lam[j].slot[0], b = lam[j].slot[1];
    const double ka = kval[kdiag_src[a]], kb = kval[kdiag_src[b]];
    kdiag[a] = ka;
    kdiag[b] = kb;
    if (stiffness) {
      delta[a] = kb / (ka + kb);
      delta[b] = ka / (ka + kb);
    } else {
      delta[a] = 0.5;
      delta[b] = 0.5;
    }
  }
}

// Repack L_II (root front of every subdomain) into row-major TB x TB tiles
// (row-block order), and the inverted diagonal blocks likewise.
__global__ void __launch_bounds__(256)
    k_pack_LII(const SubDev* __restrict__ sub, const SnDev* __restrict__ sn, const double* __restrict__ pool,
               const double* __restrict__ dinv, double* __restrict__ tiles, double* __restrict__ dtiles, int maxnt) {
  const int k = blockIdx.x / maxnt, i = blockIdx.x % maxnt;
  const SubDev d = sub[k];
  if (d.nI == 0 || i >= d.nt) return;
  const SnDev s = sn[d.root];
  const double* F = pool + s.front_off;
  for (int j = 0; j <= i; ++j) {
    double* T = tiles + d.tile_off + (long long)(i * (i + 1) / 2 + j) * TILE_ELEMS;
    for (int e = threadIdx.x; e < TILE_ELEMS; e += blockDim.x) {
      const int c = e / TB, r = e % TB;  // read column-major (coalesced), write transposed
      const int R = i * TB + r, C = j * TB + c;
      double v = 0.0;
      if (R < d.nI && C < d.nI && R >= C) v = F[(long long)C * s.ld + R];
      T[r * TB + c] = v;
    }
  }
  const double* D = dinv + s.dinv_off + (long long)i * TILE_ELEMS;  // col-major
  double* Dt = dtiles + d.dtile_off + (long long)i * TILE_ELEMS;
  for (int e = threadIdx.x; e < TILE_ELEMS; e += blockDim.x) {
    const int c = e / TB, r = e % TB;
    Dt[r * TB + c] = D[e];
  }
}

// G_k^T (B_I^T lambda), per subdomain (recovery).
__global__ void __launch_bounds__(256)
    k_gt_lambda(const SubDev* __restrict__ sub, const double* __restrict__ G, const int* __restrict__ slot_lam,
                const float* __restrict__ slot_sign, const double* __restrict__ lam, double* __restrict__ gk,
                int ncols) {
  const SubDev d = sub[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = warp; e < d.nP * ncols; e += 8) {
    const int p = e / ncols, c = e - p * ncols;
    double s = 0.0;
    for (int a = lane; a < d.nI; a += 32) {
      const int slot = (int)d.rI_off + a;
      s += G[d.g_off + (long long)a * d.nP + p] * (double)slot_sign[slot] * lam[(long long)slot_lam[slot] * ncols + c];
    }
    s = warp_sum(s);
    if (lane == 0) gk[(long long)(d.prim_off + p) * ncols + c] = s;
  }
}

// Recovery RHS: Xr = j_r - K_rP C_k p - B_r^T lambda   (row-major nr x nrhs)
__global__ void __launch_bounds__(256)
    k_rec_rhs(const SubDev* __restrict__ sub, int ncx, int nPmax, int nrhs, const double* __restrict__ X0,
              const int* __restrict__ prim_gid, const double* __restrict__ pc, const int* __restrict__ slot_lam,
              const float* __restrict__ slot_sign, const double* __restrict__ lam, double* __restrict__ Xr) {
  const SubDev d = sub[blockIdx.x];
  for (int e = threadIdx.x; e < d.nr * nrhs; e += blockDim.x) {
    const int i = e / nrhs, c = e - i * nrhs;
    const double* x0 = X0 + (d.x_off + i) * ncx;
    double v = x0[nPmax + c];
    for (int q = 0; q < d.nP; ++q) v -= x0[q] * pc[(long long)prim_gid[d.prim_off + q] * nrhs + c];
    if (i >= d.nV) {
      const int slot = (int)d.rI_off + i - d.nV;
      v -= (double)slot_sign[slot] * lam[(long long)slot_lam[slot] * nrhs + c];
    }
    Xr[(d.x_off + i) * nrhs + c] = v;
  }
}

// u^(k): r DOFs from a_r, primal DOFs from C_k p, tree DOFs 0 (n_k x nrhs col-major)
__global__ void __launch_bounds__(256)
    k_assemble_u(const SubDev* __restrict__ sub, int nrhs, const int* __restrict__ perm, const int* __restrict__ prim_dof,
                 const int* __restrict__ prim_gid, const double* __restrict__ Xr, const double* __restrict__ pc,
                 const long long* __restrict__ u_off, double* __restrict__ U) {
  const SubDev d = sub[blockIdx.x];
  double* u = U + u_off[blockIdx.x];
  for (int e = threadIdx.x; e < d.nr * nrhs; e += blockDim.x) {
    const int i = e / nrhs, c = e - i * nrhs;
    u[perm[d.perm_off + i] + (long long)c * d.nk] = Xr[(d.x_off + i) * nrhs + c];
  }
  for (int e = threadIdx.x; e < d.nP * nrhs; e += blockDim.x) {
    const int q = e / nrhs, c = e - q * nrhs;
    u[prim_dof[d.prim_off + q] + (long long)c * d.nk] = pc[(long long)prim_gid[d.prim_off + q] * nrhs + c];
  }
}

static void scatter(ietidp_s* h, const DevBuf<long long>& dst, const DevBuf<int>& src, const double* vals, double* out) {
  if (!dst.n) return;
  k_scatter<<<grid_for((long long)dst.n, 256), 256, 0, h->stream>>>((long long)dst.n, dst.p, src.p, vals, out);
  IETI_LAUNCHED(h);
}

// After run_factor: scaling weights, L_II tiles, coarse problem, d_DP.
void run_coarse(ietidp_s* h) {
  cudaStream_t s = h->stream;
  const Plan& P = h->plan;
  const int nrhs = h->nrhs, ng = h->n_primal;
  if (h->n_lambda) {
    k_scaling<<<grid_for(h->n_lambda, 256), 256, 0, s>>>(h->n_lambda, h->lam.p, h->kdiag_src.p, h->kval.p, h->kdiag.p,
                                                        h->delta.p, h->opt.scaling == IETIDP_SCALE_STIFFNESS);
    IETI_LAUNCHED(h);
  }
  int maxnt = 0;
  for (auto& d : h->h_sub) maxnt = std::max(maxnt, d.nt);
  if (maxnt) {
    k_pack_LII<<<h->n_sub * maxnt, 256, 0, s>>>(h->d_sub.p, h->d_sn.p, h->pool.p, h->dinv.p, h->tiles.p, h->dtiles.p,
                                                maxnt);
    IETI_LAUNCHED(h);
  }
  // right-hand sides of the coarse sweep: [K_rP | j_r]
  h->X0.zero(s);
  h->kpp.zero(s);
  h->jp.zero(s);
  scatter(h, h->sc_x0_dst, h->sc_x0_src, h->kval.p, h->X0.p);
  scatter(h, h->sc_fx_dst, h->sc_fx_src, h->fval.p, h->X0.p);
  scatter(h, h->sc_kpp_dst, h->sc_kpp_src, h->kval.p, h->kpp.p);
  scatter(h, h->sc_fp_dst, h->sc_fp_src, h->fval.p, h->jp.p);
  if (h->X0.n) IETI_CUDA(cudaMemcpyAsync(h->X.p, h->X0.p, h->X0.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  run_sweeps(h, h->X.p, P.ncx);
  k_coarse_local<<<h->n_sub, 256, 0, s>>>(h->d_sub.p, P.ncx, P.nPmax, nrhs, h->X0.p, h->X.p, h->kpp.p, h->jp.p,
                                          h->sloc.p, h->floc.p, h->G.p, h->xI.p);
  IETI_LAUNCHED(h);
  if (ng > 0) {
    const int smem = ng * (ng + 1) / 2 * sizeof(double);
    if (smem > 220 * 1024) throw Error(IETIDP_E_ARG, "coarse problem too large for the one-CTA coarse factorisation");
    IETI_CUDA(cudaFuncSetAttribute((const void*)k_coarse_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_coarse_factor<<<1, 1024, smem, s>>>(ng, nrhs, h->scoef_ptr.p, h->scoef_src.p, h->sloc.p, h->pcon_ptr.p,
                                          h->pcon_src.p, h->floc.p, h->S.p, h->Sinv.p, h->ftil.p, h->zc0.p,
                                          h->err_flag.p);
    IETI_LAUNCHED(h);
  }
  // d = e - G S^-1 ftilde
  if (h->n_lambda) bgather_public(h, nrhs, h->xI.p, ng ? h->zc0.p : nullptr, -1.0, h->d_vec.p);
  IETI_CHECK_LAUNCH();
}

void run_recover(ietidp_s* h) {
  cudaStream_t s = h->stream;
  const Plan& P = h->plan;
  const int nrhs = h->nrhs, ng = h->n_primal;
  if (ng > 0) {
    if (h->n_lambda) {
      k_gt_lambda<<<h->n_sub, 256, 0, s>>>(h->d_sub.p, h->G.p, h->slot_lam.p, h->slot_sign.p, h->lam_vec.p, h->gk.p,
                                           nrhs);
      IETI_LAUNCHED(h);
    } else {
      h->gk.zero(s);
    }
    coarse_apply_public(h, nrhs, h->gk.p, h->ftil.p, h->zc.p);
  }
  k_rec_rhs<<<h->n_sub, 256, 0, s>>>(h->d_sub.p, P.ncx, P.nPmax, nrhs, h->X0.p, h->d_prim_gid.p, h->zc.p,
                                     h->slot_lam.p, h->slot_sign.p, h->lam_vec.p, h->Xr.p);
  IETI_LAUNCHED(h);
  run_sweeps(h, h->Xr.p, nrhs);
  h->U.zero(s);
  k_assemble_u<<<h->n_sub, 256, 0, s>>>(h->d_sub.p, nrhs, h->d_perm.p, h->d_prim_dof.p, h->d_prim_gid.p, h->Xr.p,
                                        h->zc.p, h->d_uoff.p, h->U.p);
  IETI_LAUNCHED(h);
  IETI_CHECK_LAUNCH();
}

}  // namespace ieti
