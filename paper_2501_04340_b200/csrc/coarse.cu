// Coarse set-up, RHS and recovery, with the primal
// DOFs ordered last:
//   S_loc^(k) = K_PP - K_Pr K_rr^-1 K_rP  is the assembled P front (factor.cu);
//   ftilde^(k) = j_P - K_Pr K_rr^-1 j_r   is the P rows of the forward sweep;
//   S_PP = sum_k C_k^T S_loc C_k, ftilde = sum_k C_k^T ftilde^(k)
//   S_PP = L L^T, S_PP^-1 = L^-T L^-1 (one CTA)
//   d_DP = e - G S_PP^-1 ftilde = sum_k B_I L_II^-T (y_I - L_PI^T C_k S^-1 ftilde)
//          with y_I the r_I rows of L^-1 j                       (R1, F2')
// plus the Dirichlet-scaling weights and the tile-major repacking of L_II,
// L_II^-1 and L_PI for the loop. Recovery (Eqs. 8-9):
//   p = S_PP^-1 (ftilde + G^T lambda),  G^T lambda = sum_k C_k^T L_PI L_II^-1 B_I^T lambda,
//   a_r = L^-T (L^-1 j_r - L_Pr^T C_k p - [0; L_II^-1 B_I^T lambda])  (one backward sweep
//   with the P rows set to p).
#include <climits>

#include "common.cuh"

namespace ieti {

void run_sweeps(ietidp_s* h, double* X, bool fwd, bool bwd);
void launch_form_G(ietidp_s* h);
void loop_fwd(ietidp_s* h, int ncols, const double* v, double* y, bool partials, const void* st);
void loop_bwd(ietidp_s* h, int ncols, const double* y, const double* z, double zsign, double* x, const void* st);
void bgather(ietidp_s* h, int ncols, const double* x, const double* weight, double* out, const double* dotv,
             double* partial, const void* st);
void coarse_apply(ietidp_s* h, int ncols, const double* add, double* z, const void* st, bool sym_rows = false);
__global__ void k_scatter(long long n, const long long* __restrict__ dst, const int* __restrict__ src,
                          const double* __restrict__ vals, double* __restrict__ out);

// S_PP = sum_k C_k^T S_loc C_k from the P fronts, ftilde = sum_k C_k^T ftilde^(k)
// from the forward-swept loads (deterministic: fixed contribution lists), symmetrisation,
// Cholesky, inverse, and zc0 = S^-1 ftilde. One CTA of 1024 threads; the lower
// triangle lives packed in shared memory (n(n+1)/2 doubles).
__device__ __forceinline__ int pk(int i, int j) { return i * (i + 1) / 2 + j; }

// S_PP = sum_k C_k^T S_loc^(k) C_k from the P fronts, and ftilde = sum_k C_k^T ftilde^(k):
// element-parallel over all CTAs (the gathers), ahead of the one-CTA factorisation
__global__ void __launch_bounds__(256)
    k_coarse_assemble(int n, int nrhs, const int* __restrict__ scoef_ptr, const long long* __restrict__ scoef_src,
                      const double* __restrict__ pool, const int* __restrict__ pcon_ptr,
                      const int* __restrict__ pcon_sub, const int* __restrict__ pcon_q,
                      const SubDev* __restrict__ sub, const double* __restrict__ Xf, double* __restrict__ S,
                      double* __restrict__ ftil) {
  const long long tot = (long long)n * n + (long long)n * nrhs;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    if (e < (long long)n * n) {
      double s = 0.0;
      for (int q = scoef_ptr[e]; q < scoef_ptr[e + 1]; ++q) s += pool[scoef_src[q]];
      S[e] = s;
    } else {
      const long long f = e - (long long)n * n;
      const int g = (int)(f / nrhs), c = (int)(f - (long long)g * nrhs);
      double s = 0.0;
      for (int q = pcon_ptr[g]; q < pcon_ptr[g + 1]; ++q) {
        const SubDev& d = sub[pcon_sub[q]];
        s += Xf[(d.x_off + d.nr + pcon_q[q]) * nrhs + c];
      }
      ftil[f] = s;
    }
  }
}

__global__ void __launch_bounds__(1024)
    k_coarse_factor(int n, int nrhs, const int* __restrict__ scoef_ptr, const long long* __restrict__ scoef_src,
                    const double* __restrict__ pool, const int* __restrict__ pcon_ptr,
                    const int* __restrict__ pcon_sub, const int* __restrict__ pcon_q, const SubDev* __restrict__ sub,
                    const double* __restrict__ Xf, double* __restrict__ S, double* __restrict__ Sinv,
                    double* __restrict__ ftil, double* __restrict__ zc0, int* __restrict__ err) {
  extern __shared__ double Lp[];  // n(n+1)/2
  __shared__ double tmp[1024], tsc[1024];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  (void)scoef_ptr;
  (void)scoef_src;
  (void)pool;
  (void)pcon_ptr;
  (void)pcon_sub;
  (void)pcon_q;
  (void)sub;
  (void)Xf;
  __syncthreads();
  for (int e = tid; e < n * (n + 1) / 2; e += blockDim.x) {
    int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while (pk(i, 0) > e) --i;
    while (pk(i + 1, 0) <= e) ++i;
    const int j = e - pk(i, 0);
    Lp[e] = 0.5 * (S[i * n + j] + S[j * n + i]);
  }
  __syncthreads();
  // S_PP^-1 by the symmetric sweep operator (Gauss-Jordan without pivoting on the SPD
  // matrix, packed lower storage): sweeping pivot k maps
  //   a_kk -> -1/a_kk,  a_ik -> a_ik / a_kk,  a_ij -> a_ij - a_ik a_jk / a_kk  (i, j != k);
  // after all n pivots the matrix holds -S^-1. The pivots are the Schur-complement
  // diagonals: one that is not positive means S_PP is not SPD. Two barriers per pivot.
  constexpr int EPT = 32;  // packed entries per thread (n <= 255)
  int pij[EPT];  // (i << 16) | j of this thread's packed entries, -1 past the end
  const int ne = n * (n + 1) / 2;
#pragma unroll
  for (int m = 0; m < EPT; ++m) {
    const int e = tid + m * 1024;
    pij[m] = -1;
    if (e < ne) {
      int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (pk(i, 0) > e) --i;
      while (pk(i + 1, 0) <= e) ++i;
      pij[m] = (i << 16) | (e - pk(i, 0));
    }
  }
  for (int k = 0; k < n; ++k) {
    double akk = Lp[pk(k, k)];
    if (!(akk > 0.0)) {
      if (tid == 0) bad = 1;
      akk = 1.0;
    }
    const double inv = 1.0 / akk;
    // column k of the current matrix (0 at k itself) and its scaled copy
    for (int i = tid; i < n; i += blockDim.x) {
      const double t = (i == k) ? 0.0 : Lp[i > k ? pk(i, k) : pk(k, i)];
      tmp[i] = t;
      tsc[i] = t * inv;
    }
    __syncthreads();
    // a_ij -= (a_ik / a_kk) a_jk for every entry (row / column k unchanged: t_k = 0)
#pragma unroll
    for (int m = 0; m < EPT; ++m) {
      if (pij[m] < 0) continue;
      const int e = tid + m * 1024;
      Lp[e] = fma(-tsc[pij[m] >> 16], tmp[pij[m] & 0xffff], Lp[e]);
    }
    __syncthreads();
    // then row / column k: a_ik / a_kk, and -1 / a_kk on the diagonal
    for (int i = tid; i < n; i += blockDim.x) Lp[i > k ? pk(i, k) : pk(k, i)] = (i == k) ? -inv : tsc[i];
    __syncthreads();
  }
  if (tid == 0 && bad) atomicMin(err + 1, 0);
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    Sinv[e] = -Lp[i >= j ? pk(i, j) : pk(j, i)];
  }
  __syncthreads();
  for (int e = tid; e < n * nrhs; e += blockDim.x) {
    const int i = e / nrhs, c = e - i * nrhs;
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += Sinv[i * n + j] * ftil[j * nrhs + c];
    zc0[e] = s;
  }
}

// ---------------------------------------------------------------------------
// Larger coarse problems (n_gp > COARSE_CTA_MAX: n_gp grows with the
// number of subdomains): S_PP^-1 by the BLOCKED sweep operator on the full n x n
// matrix in global memory (row-major A = S_PP, TB-blocks). Sweeping block K:
//   A_KK -> -A_KK^-1,  A_KJ -> A_KK^-1 A_KJ,  A_IK -> A_IK A_KK^-1,
//   A_IJ -> A_IJ - A_IK A_KK^-1 A_KJ   (I, J != K);
// after all blocks A = -S_PP^-1 (the block form of the scalar sweep of k_coarse_factor).
// Per block: the pivot block's inverse (one CTA, scalar sweep in shared memory; a
// pivot that is not positive means S_PP is not SPD), T_K* = A_KK^-1 A_K* (a tile per
// block), the update of every other tile (DMMA), then row / column K.
// ---------------------------------------------------------------------------
constexpr int COARSE_CTA_MAX = 230;  // the one-CTA packed factorisation above up to this size

__global__ void __launch_bounds__(256) k_bsw_pivot(int n, int K, const double* __restrict__ A, double* __restrict__ D,
                                                  int* __restrict__ err) {
  __shared__ double M[TB][TB + 1];
  __shared__ double col[TB], scol[TB];
  const int tid = threadIdx.x, k0 = K * TB, b = min(TB, n - k0);
  for (int e = tid; e < TILE_ELEMS; e += 256) {
    const int r = e >> 6, c = e & (TB - 1);
    M[r][c] = (r < b && c < b) ? A[(long long)(k0 + r) * n + k0 + c] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  bool bad = false;
  for (int k = 0; k < TB; ++k) {
    double akk = M[k][k];
    if (!(akk > 0.0)) {
      bad = true;
      akk = 1.0;
    }
    const double inv = 1.0 / akk;
    if (tid < TB) {
      const double t = (tid == k) ? 0.0 : M[tid][k];
      col[tid] = t;
      scol[tid] = t * inv;
    }
    __syncthreads();
    for (int e = tid; e < TILE_ELEMS; e += 256) {
      const int r = e >> 6, c = e & (TB - 1);
      M[r][c] = fma(-scol[r], col[c], M[r][c]);
    }
    __syncthreads();
    if (tid < TB) {
      M[tid][k] = (tid == k) ? -inv : scol[tid];
      M[k][tid] = (tid == k) ? -inv : scol[tid];
    }
    __syncthreads();
  }
  if (bad && tid == 0) atomicMin(err + 1, 0);
  for (int e = tid; e < TILE_ELEMS; e += 256) D[e] = -M[e >> 6][e & (TB - 1)];  // A_KK^-1 (row-major)
}

// C(64 x 64 tile) = op of A-tile (row-major, lda) times B-tile (row-major, ldb), DMMA,
// 4 warps x 32 x 32; tiles staged in shared memory (zero padded). mode 0: C = A B,
// 1: C -= A B.
constexpr int BSW_SMEM = 2 * TB * (TB + 1) * (int)sizeof(double);  // two staged tiles (dynamic)
__device__ __forceinline__ void bsw_tile_mma(const double* A, long long lda, int am, int ak, const double* B,
                                             long long ldb, int bn, double* C, long long ldc, int cm, int cn,
                                             int mode, double (*As)[TB + 1], double (*Bs)[TB + 1]) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  for (int e = tid; e < TILE_ELEMS; e += 128) {
    const int r = e >> 6, c = e & (TB - 1);
    As[r][c] = (r < am && c < ak) ? A[r * lda + c] : 0.0;
    Bs[r][c] = (r < ak && c < bn) ? B[r * ldb + c] : 0.0;
  }
  __syncthreads();
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double acc[4][4][2] = {};
#pragma unroll 4
  for (int k0 = 0; k0 < TB; k0 += 4) {
    double a[4], bb[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = As[wm + 8 * i + g][k0 + t];
#pragma unroll
    for (int j = 0; j < 4; ++j) bb[j] = Bs[k0 + t][wn + 8 * j + g];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = wm + 8 * i + g, c = wn + 8 * j + 2 * t + e;
        if (r < cm && c < cn) {
          double* p = C + r * ldc + c;
          *p = mode ? *p - acc[i][j][e] : acc[i][j][e];
        }
      }
  __syncthreads();
}

// T_KJ = A_KK^-1 A_KJ for every block J (J = K included: unused)
__global__ void __launch_bounds__(128) k_bsw_row(int n, int K, const double* __restrict__ A,
                                                const double* __restrict__ D, double* __restrict__ T) {
  extern __shared__ double bsm[];
  auto As = reinterpret_cast<double(*)[TB + 1]>(bsm);
  auto Bs = reinterpret_cast<double(*)[TB + 1]>(bsm + TB * (TB + 1));
  const int J = blockIdx.x, k0 = K * TB, j0 = J * TB;
  const int bk = min(TB, n - k0), bj = min(TB, n - j0);
  bsw_tile_mma(D, TB, bk, bk, A + (long long)k0 * n + j0, n, bj, T + j0, n, bk, bj, 0, As, Bs);
}

// A_IJ -= A_IK T_KJ for I, J != K
__global__ void __launch_bounds__(128) k_bsw_update(int n, int nb, int K, double* __restrict__ A,
                                                   const double* __restrict__ T) {
  extern __shared__ double bsm[];
  auto As = reinterpret_cast<double(*)[TB + 1]>(bsm);
  auto Bs = reinterpret_cast<double(*)[TB + 1]>(bsm + TB * (TB + 1));
  const int I = blockIdx.x / nb, J = blockIdx.x % nb;
  if (I == K || J == K) return;
  const int i0 = I * TB, j0 = J * TB, k0 = K * TB;
  const int bi = min(TB, n - i0), bj = min(TB, n - j0), bk = min(TB, n - k0);
  bsw_tile_mma(A + (long long)i0 * n + k0, n, bi, bk, T + j0, n, bj, A + (long long)i0 * n + j0, n, bi, bj, 1, As,
               Bs);
}

// row / column K: A_KJ = T_KJ, A_JK = T_KJ^T (J != K), A_KK = -A_KK^-1
__global__ void __launch_bounds__(256) k_bsw_fix(int n, int K, double* __restrict__ A, const double* __restrict__ D,
                                                const double* __restrict__ T) {
  const int k0 = K * TB, bk = min(TB, n - k0);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)bk * n;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / n), c = (int)(e - (long long)r * n);
    if (c >= k0 && c < k0 + bk) {
      A[(long long)(k0 + r) * n + c] = -D[r * TB + (c - k0)];
    } else {
      const double v = T[(long long)r * n + c];
      A[(long long)(k0 + r) * n + c] = v;
      A[(long long)c * n + k0 + r] = v;
    }
  }
}

// S = 1/2 (S + S^T) into A; afterwards Sinv = -A, zc0 = Sinv ftilde
__global__ void k_bsw_init(int n, const double* __restrict__ S, double* __restrict__ A) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e - (long long)i * n);
    A[e] = 0.5 * (S[(long long)i * n + j] + S[(long long)j * n + i]);
  }
}
__global__ void k_bsw_finish(int n, int nrhs, const double* __restrict__ A, double* __restrict__ Sinv,
                             const double* __restrict__ ftil, double* __restrict__ zc0) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x)
    Sinv[e] = -A[e];
}
__global__ void k_bsw_z(int n, int nrhs, const double* __restrict__ Sinv, const double* __restrict__ ftil,
                        double* __restrict__ zc0) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = warp; e < n * nrhs; e += nw) {
    const int i = e / nrhs, c = e - i * nrhs;
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s += Sinv[(long long)i * n + j] * ftil[j * nrhs + c];
    s = warp_sum(s);
    if (lane == 0) zc0[e] = s;
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

// Sharded mode (ietidp_shard.h): the K diagonal of each multiplier's local side(s) into
// kd2[2j + (sign < 0)] (zero where the side lives on another rank); after the sum over the
// ranks both sides are known everywhere and the weights follow as in k_scaling.
__global__ void k_sh_kdiag(int m, const LamDev* __restrict__ lam, const int* __restrict__ kdiag_src,
                           const double* __restrict__ kval, double* __restrict__ kd2) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    double v[2] = {0.0, 0.0};
    for (int q = 0; q < 2; ++q)
      if (lam[j].sign[q] != 0.f) v[lam[j].sign[q] < 0.f ? 1 : 0] = kval[kdiag_src[lam[j].slot[q]]];
    kd2[2 * j] = v[0];
    kd2[2 * j + 1] = v[1];
  }
}
__global__ void k_sh_delta(int m, const LamDev* __restrict__ lam, const double* __restrict__ kd2,
                           double* __restrict__ kdiag, double* __restrict__ delta, int stiffness) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x)
    for (int q = 0; q < 2; ++q) {
      if (lam[j].sign[q] == 0.f) continue;
      const int a = lam[j].slot[q], side = lam[j].sign[q] < 0.f ? 1 : 0;
      const double mine = kd2[2 * j + side], other = kd2[2 * j + 1 - side];
      kdiag[a] = mine;
      delta[a] = stiffness ? other / (mine + other) : 0.5;
    }
}

// Sum of a device buffer over the ranks of a sharded solve (the caller's all-reduce).
void sh_sum(ietidp_s* h, double* buf, long long n) {
  if (!h->shard || n <= 0) return;
  if (h->sh_allreduce(h->sh_ctx, buf, (int64_t)n, (void*)h->stream) != 0)
    throw Error(IETIDP_E_CUDA, "the all-reduce callback of the sharded solve failed");
  h->sh_reduced_doubles += n;
}

// Repack the r_I root front of every subdomain for the loop: L_II^-1 (and, for the
// triangular loop, L_II) as row-major TB x TB lower tiles (row-block order), L_PI as
// nP x nI row-major. One CTA per (subdomain, lower tile); the tile is transposed
// through shared memory. The CTAs of the tiles (i, 0) also write L_PI's columns of
// block i.
__global__ void __launch_bounds__(256)
    k_pack(const SubDev* __restrict__ sub, const SnDev* __restrict__ sn, const int* __restrict__ rows,
           const double* __restrict__ pool, const double* __restrict__ ipool, double* __restrict__ tiles,
           double* __restrict__ itiles, double* __restrict__ lpi, int maxnt, int want_tiles) {
  __shared__ double S[TB][TB + 1];
  const int ntl = maxnt * (maxnt + 1) / 2;
  const int k = blockIdx.x / ntl, t = blockIdx.x % ntl;
  int i = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while (i * (i + 1) / 2 > t) --i;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  const int j = t - i * (i + 1) / 2;
  const SubDev d = sub[k];
  if (d.nI == 0 || i >= d.nt) return;
  const SnDev s = sn[d.root];
  const double* F = pool + s.front_off;
  const double* I = ipool + s.inv_off;
  const long long toff = d.tile_off + (long long)t * TILE_ELEMS;
  for (int pass = want_tiles ? 0 : 1; pass < 2; ++pass) {
    const double* M = pass ? I : F;
    const long long ld = pass ? s.ldi : s.ld;
    for (int e = threadIdx.x; e < TILE_ELEMS; e += blockDim.x) {
      const int c = e >> 6, r = e & (TB - 1);  // coalesced column reads into smem
      const int R = i * TB + r, C = j * TB + c;
      S[c][r] = (R < d.nI && C < d.nI && R >= C) ? M[(long long)C * ld + R] : 0.0;
    }
    __syncthreads();
    double* T = (pass ? itiles : tiles) + toff;
    for (int e = threadIdx.x; e < TILE_ELEMS; e += blockDim.x)  // row writes, swizzled (common.cuh swz)
      T[swz(e >> 6, e & (TB - 1))] = S[e & (TB - 1)][e >> 6];
    __syncthreads();
  }
  if (j != 0) return;
  // L_PI: the root's update rows are P positions (>= nr)
  const int nu = s.f - s.npiv;
  const int* rw = rows + s.rows_off;
  for (int e = threadIdx.x; e < d.nP * TB; e += blockDim.x) {
    const int q = e / TB, a = i * TB + e % TB;
    if (a < d.nI) lpi[d.lpi_off + (long long)q * d.nI + a] = 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nu * TB; e += blockDim.x) {
    const int rho = e / TB, a = i * TB + e % TB;
    if (a < d.nI) {
      const int q = rw[rho] - d.nr;
      lpi[d.lpi_off + (long long)q * d.nI + a] = F[(long long)a * s.ld + s.npiv + rho];
    }
  }
}

// y_I (slot vector) <- the r_I rows of X
__global__ void k_gather_I(const SubDev* __restrict__ sub, int nrhs, const double* __restrict__ X,
                           double* __restrict__ y) {
  const SubDev d = sub[blockIdx.x];
  for (int e = threadIdx.x; e < d.nI * nrhs; e += blockDim.x) {
    const int a = e / nrhs, c = e % nrhs;
    y[(d.rI_off + a) * nrhs + c] = X[(d.x_off + d.nV + a) * nrhs + c];
  }
}

// Recovery input of the backward sweep: P rows <- C_k p, r_I rows -= L_II^-1 B_I^T lambda
__global__ void k_rec_prep(const SubDev* __restrict__ sub, int nrhs, const int* __restrict__ prim_gid,
                           const double* __restrict__ pc, const double* __restrict__ ylam, double* __restrict__ X) {
  const SubDev d = sub[blockIdx.x];
  for (int e = threadIdx.x; e < d.nP * nrhs; e += blockDim.x) {
    const int q = e / nrhs, c = e % nrhs;
    X[(d.x_off + d.nr + q) * nrhs + c] = pc[(long long)prim_gid[d.prim_off + q] * nrhs + c];
  }
  for (int e = threadIdx.x; e < d.nI * nrhs; e += blockDim.x) {
    const int a = e / nrhs, c = e % nrhs;
    X[(d.x_off + d.nV + a) * nrhs + c] -= ylam[(d.rI_off + a) * nrhs + c];
  }
}

// u^(k): every non-tree DOF from X (r and P positions), tree DOFs 0 (n_k x nrhs col-major)
__global__ void __launch_bounds__(256)
    k_assemble_u(const SubDev* __restrict__ sub, int nrhs, const int* __restrict__ perm, const double* __restrict__ X,
                 const long long* __restrict__ u_off, double* __restrict__ U) {
  const SubDev d = sub[blockIdx.x];
  double* u = U + u_off[blockIdx.x];
  for (int e = threadIdx.x; e < d.ne * nrhs; e += blockDim.x) {
    const int i = e / nrhs, c = e % nrhs;
    u[perm[d.perm_off + i] + (long long)c * d.nk] = X[(d.x_off + i) * nrhs + c];
  }
}

// After run_factor: scaling weights, loop tiles, forward sweep of the loads,
// coarse problem, d_DP.
void run_coarse(ietidp_s* h) {
  cudaStream_t s = h->stream;
  const int nrhs = h->nrhs, ng = h->n_primal;
  const int nlev = h->plan.max_level + 1;
  (void)nlev;  // the factorisation's streams have joined the caller's stream
  if (h->n_lambda && h->shard) {  // the partner's K diagonal may live on another rank
    if (h->sh_kd2.n == 0) h->sh_kd2.alloc(2 * (size_t)h->n_lambda);
    k_sh_kdiag<<<grid_for(h->n_lambda, 256), 256, 0, s>>>(h->n_lambda, h->lam.p, h->kdiag_src.p, h->kval.p, h->sh_kd2.p);
    IETI_LAUNCHED(h);
    sh_sum(h, h->sh_kd2.p, 2LL * h->n_lambda);
    k_sh_delta<<<grid_for(h->n_lambda, 256), 256, 0, s>>>(h->n_lambda, h->lam.p, h->sh_kd2.p, h->kdiag.p, h->delta.p,
                                                          h->opt.scaling == IETIDP_SCALE_STIFFNESS);
    IETI_LAUNCHED(h);
  } else if (h->n_lambda) {
    k_scaling<<<grid_for(h->n_lambda, 256), 256, 0, s>>>(h->n_lambda, h->lam.p, h->kdiag_src.p, h->kval.p, h->kdiag.p,
                                                        h->delta.p, h->opt.scaling == IETIDP_SCALE_STIFFNESS);
    IETI_LAUNCHED(h);
  }
  int maxnt = 0;
  for (auto& d : h->h_sub) maxnt = std::max(maxnt, d.nt);
  if (maxnt) {
    k_pack<<<h->n_sub * (maxnt * (maxnt + 1) / 2), 256, 0, s>>>(h->d_sub.p, h->d_sn.p, h->d_rows.p, h->pool.p, h->ipool.p, h->tiles.p,
                                            h->itiles.p, h->lpi.p, maxnt, h->opt.loop == IETIDP_LOOP_TRIANGULAR);
    IETI_LAUNCHED(h);
    if (ng > 0) launch_form_G(h);
  }
  // loads -> X (position order), forward sweep: X = L^-1 j, P rows = ftilde^(k)
  if (!h->fwd_in_factor) {
    h->Xf.zero(s);
    if (h->sc_fx_dst.n) {
      k_scatter<<<grid_for((long long)h->sc_fx_dst.n, 256), 256, 0, s>>>((long long)h->sc_fx_dst.n, h->sc_fx_dst.p,
                                                                        h->sc_fx_src.p, h->fval.p, h->Xf.p);
      IETI_LAUNCHED(h);
    }
    run_sweeps(h, h->Xf.p, true, false);
  }
  if (ng > 0) {
    k_coarse_assemble<<<grid_for((long long)ng * (ng + nrhs), 256), 256, 0, s>>>(
        ng, nrhs, h->scoef_ptr.p, h->scoef_src.p, h->pool.p, h->pcon_ptr.p, h->pcon_sub.p, h->pcon_q.p, h->d_sub.p,
        h->Xf.p, h->S.p, h->ftil.p);
    IETI_LAUNCHED(h);
    if (h->shard) {  // S_PP and ftilde are sums over all subdomains
      sh_sum(h, h->S.p, (long long)ng * ng);
      sh_sum(h, h->ftil.p, (long long)ng * nrhs);
    }
    // one CTA up to 127 primal DOFs; above, the blocked sweep operator over all SMs is quicker
    // (C5, n_gp = 177: coarse set-up 1.38 -> 1.10 ms; C3, 145: 0.74 -> 0.64 ms); sharded: always
    // (S_PP comes from the sum over the ranks, not from the local P fronts)
    static const int one_cta_max = getenv("IETIDP_COARSE_CTA_MAX") ? atoi(getenv("IETIDP_COARSE_CTA_MAX")) : 127;
    if (ng <= std::min(COARSE_CTA_MAX, one_cta_max) && !h->shard) {
      const int smem = ng * (ng + 1) / 2 * sizeof(double);
      IETI_CUDA(cudaFuncSetAttribute((const void*)k_coarse_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_coarse_factor<<<1, 1024, smem, s>>>(ng, nrhs, h->scoef_ptr.p, h->scoef_src.p, h->pool.p, h->pcon_ptr.p,
                                            h->pcon_sub.p, h->pcon_q.p, h->d_sub.p, h->Xf.p, h->S.p, h->Sinv.p,
                                            h->ftil.p, h->zc0.p, h->err_flag.p);
      IETI_LAUNCHED(h);
    } else {  // blocked sweep operator over all SMs
      const int nb = (ng + TB - 1) / TB;
      if (h->bsw_A.n < (size_t)ng * ng) {
        h->bsw_A.alloc((size_t)ng * ng);
        h->bsw_T.alloc((size_t)TB * ng);
        h->bsw_D.alloc(TILE_ELEMS);
      }
      IETI_CUDA(cudaFuncSetAttribute((const void*)k_bsw_row, cudaFuncAttributeMaxDynamicSharedMemorySize, BSW_SMEM));
      IETI_CUDA(cudaFuncSetAttribute((const void*)k_bsw_update, cudaFuncAttributeMaxDynamicSharedMemorySize, BSW_SMEM));
      k_bsw_init<<<grid_for((long long)ng * ng, 256), 256, 0, s>>>(ng, h->S.p, h->bsw_A.p);
      IETI_LAUNCHED(h);
      for (int K = 0; K < nb; ++K) {
        k_bsw_pivot<<<1, 256, 0, s>>>(ng, K, h->bsw_A.p, h->bsw_D.p, h->err_flag.p);
        k_bsw_row<<<nb, 128, BSW_SMEM, s>>>(ng, K, h->bsw_A.p, h->bsw_D.p, h->bsw_T.p);
        k_bsw_update<<<nb * nb, 128, BSW_SMEM, s>>>(ng, nb, K, h->bsw_A.p, h->bsw_T.p);
        k_bsw_fix<<<grid_for((long long)TB * ng, 256), 256, 0, s>>>(ng, K, h->bsw_A.p, h->bsw_D.p, h->bsw_T.p);
        for (int q = 0; q < 4; ++q) IETI_LAUNCHED(h);
      }
      k_bsw_finish<<<grid_for((long long)ng * ng, 256), 256, 0, s>>>(ng, nrhs, h->bsw_A.p, h->Sinv.p, h->ftil.p,
                                                                      h->zc0.p);
      k_bsw_z<<<grid_for((long long)ng * nrhs * 32, 256), 256, 0, s>>>(ng, nrhs, h->Sinv.p, h->ftil.p, h->zc0.p);
      IETI_LAUNCHED(h);
      IETI_LAUNCHED(h);
    }
  }
  // d = sum_k B_I L_II^-T (y_I - L_PI^T C_k S^-1 ftilde)
  if (h->n_lambda) {
    k_gather_I<<<h->n_sub, 256, 0, s>>>(h->d_sub.p, nrhs, h->Xf.p, h->yI.p);
    IETI_LAUNCHED(h);
    loop_bwd(h, nrhs, h->yI.p, ng ? h->zc0.p : nullptr, -1.0, h->xI.p, nullptr);
    bgather(h, nrhs, h->xI.p, nullptr, h->d_vec.p, nullptr, nullptr, nullptr);  // (sharded: summed over the ranks inside)
  }
  IETI_CHECK_LAUNCH();
}

void run_recover(ietidp_s* h) {
  cudaStream_t s = h->stream;
  const int nrhs = h->nrhs, ng = h->n_primal;
  if (h->n_lambda) loop_fwd(h, nrhs, h->lam_vec.p, h->yI.p, true, nullptr);
  if (ng > 0) {
    if (!h->n_lambda) h->gpart.zero(s);
    coarse_apply(h, nrhs, h->ftil.p, h->zc.p, nullptr);
  }
  IETI_CUDA(cudaMemcpyAsync(h->Xr.p, h->Xf.p, h->Xf.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (!h->n_lambda) h->yI.zero(s);
  k_rec_prep<<<h->n_sub, 256, 0, s>>>(h->d_sub.p, nrhs, h->d_prim_gid.p, h->zc.p, h->yI.p, h->Xr.p);
  IETI_LAUNCHED(h);
  run_sweeps(h, h->Xr.p, false, true);
  h->U.zero(s);
  k_assemble_u<<<h->n_sub, 256, 0, s>>>(h->d_sub.p, nrhs, h->d_perm.p, h->Xr.p, h->d_uoff.p, h->U.p);
  IETI_LAUNCHED(h);
  IETI_CHECK_LAUNCH();
}

}  // namespace ieti
