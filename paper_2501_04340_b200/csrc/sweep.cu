// Batched multifrontal triangular sweeps with the supernodal factor and the
// partitioned inverse L11^-1 of every supernode:
//   forward  (leaves -> root): v = [x_piv; 0] + children's update vectors,
//            y_piv = L11^-1 v_piv, v_upd -= L21 y_piv (kept for the parent);
//            the P (coarse) supernode only assembles: x_P = j_P - K_Pr K_rr^-1 j_r
//            = ftilde^(k) (SPD sign);
//   backward (root -> leaves): x_piv = L11^-T (y_piv - L21^T x_rows).
// Used for y = K_rr^-1 j_r at set-up (a5) and for the recovery Eq. (9) (a7).
// X is row-major (ne rows per subdomain) x ldx columns, in position order.
// Every step is a batched GEMV over tiles of all supernodes of a level: no
// sequential dependency inside a supernode, so the top fronts spread over many SMs.
#include "common.cuh"

namespace ieti {

constexpr int SWT = 256;

// F1: assemble the front vector (one CTA per supernode of the level).
template <int NCB>
__global__ void __launch_bounds__(SWT)
    k_fs_assemble(const int* __restrict__ lst, const SnDev* __restrict__ sn, const SubDev* __restrict__ sub,
                  const int* __restrict__ rel, const int* __restrict__ children, double* __restrict__ X,
                  double* __restrict__ Wv, int ldx, int cofs) {
  const SnDev s = sn[lst[blockIdx.x]];
  const SubDev d = sub[s.sub];
  const int ncl = min(NCB, ldx - cofs);
  double* v = Wv + s.vec_off * NCB;
  double* x = X + (d.x_off + s.c0) * ldx + cofs;
  for (int e = threadIdx.x; e < s.f * NCB; e += SWT) {
    const int i = e / NCB, c = e % NCB;
    v[e] = (i < s.npiv && c < ncl) ? x[(long long)i * ldx + c] : 0.0;
  }
  __syncthreads();
  for (int ci = 0; ci < s.nchild; ++ci) {
    const SnDev ch = sn[children[s.child_off + ci]];
    const int nu = ch.f - ch.npiv;
    const double* uc = Wv + (ch.vec_off + ch.npiv) * NCB;
    const int* rl = rel + ch.rel_off;
    for (int e = threadIdx.x; e < nu * NCB; e += SWT) {
      const int i = e / NCB, c = e % NCB;
      v[rl[i] * NCB + c] += uc[e];
    }
    __syncthreads();
  }
  if (s.coarse)
    for (int e = threadIdx.x; e < s.npiv * ncl; e += SWT) {
      const int i = e / ncl, c = e % ncl;
      x[(long long)i * ldx + c] = v[i * NCB + c];
    }
}

// F2 (MODE 0): y[tile rows] = L11^-1[tile rows, :] v_piv  -> X
// F3 (MODE 1): v_upd[tile rows] -= L21[tile rows, :] y    -> Wv
// 64 rows x 4 k-groups per CTA; the K vector is staged in shared memory by chunks.
template <int MODE, int NCB>
__global__ void __launch_bounds__(SWT)
    k_fs_gemv(const Work* __restrict__ work, const SnDev* __restrict__ sn, const SubDev* __restrict__ sub,
              const double* __restrict__ pool, const double* __restrict__ ipool, double* __restrict__ X,
              double* __restrict__ Wv, int ldx, int cofs) {
  __shared__ double xs[TB][NCB];
  __shared__ double red[4][TB][NCB];
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const SubDev d = sub[s.sub];
  const int ncl = min(NCB, ldx - cofs);
  const int r = threadIdx.x & 63, kg = threadIdx.x >> 6;
  const int row0 = w.a * TB;
  const int nrows = (MODE == 0) ? s.npiv : s.f - s.npiv;
  const int R = row0 + r;
  const int kend = (MODE == 0) ? min(s.npiv, row0 + TB) : s.npiv;  // L11^-1 lower: k < tile end
  const double* Amat;
  long long lda;
  if (MODE == 0) {
    Amat = ipool + s.inv_off + R;
    lda = s.ldi;
  } else {
    Amat = pool + s.front_off + s.npiv + R;
    lda = s.ld;
  }
  const double* vin = (MODE == 0) ? Wv + s.vec_off * NCB : nullptr;       // v_piv
  const double* yin = (MODE == 1) ? X + (d.x_off + s.c0) * ldx + cofs : nullptr;  // y
  double acc[NCB];
#pragma unroll
  for (int c = 0; c < NCB; ++c) acc[c] = 0.0;
  for (int k0 = 0; k0 < kend; k0 += TB) {
    __syncthreads();
    for (int e = threadIdx.x; e < TB * NCB; e += SWT) {
      const int k = e / NCB, c = e % NCB;
      double v = 0.0;
      if (k0 + k < kend) v = (MODE == 0) ? vin[(k0 + k) * NCB + c] : (c < ncl ? yin[(long long)(k0 + k) * ldx + c] : 0.0);
      xs[k][c] = v;
    }
    __syncthreads();
    if (R < nrows) {
      const int kn = min(TB, kend - k0);
      for (int k = kg; k < kn; k += 4) {
        const double a = Amat[(long long)(k0 + k) * lda];
#pragma unroll
        for (int c = 0; c < NCB; ++c) acc[c] += a * xs[k][c];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < NCB; ++c) red[kg][r][c] = acc[c];
  __syncthreads();
  if (kg == 0 && R < nrows) {
#pragma unroll
    for (int c = 0; c < NCB; ++c) {
      const double v = red[0][r][c] + red[1][r][c] + red[2][r][c] + red[3][r][c];
      if (MODE == 0) {
        if (c < ncl) X[(d.x_off + s.c0 + R) * ldx + cofs + c] = v;
      } else {
        Wv[(s.vec_off + s.npiv + R) * NCB + c] -= v;
      }
    }
  }
}

// B1 (MODE 0): t[cols] = y[cols] - L21[:, cols]^T x_rows      -> Wv (pivot rows)
// B2 (MODE 1): x[cols] = L11^-T[cols, :] t = sum_{r>=c} Linv[r][c] t[r] -> X
// One warp per pivot column (lanes over the contiguous column), 8 columns per warp.
template <int MODE, int NCB>
__global__ void __launch_bounds__(SWT)
    k_bs_gemv(const Work* __restrict__ work, const SnDev* __restrict__ sn, const SubDev* __restrict__ sub,
              const int* __restrict__ rows, const double* __restrict__ pool, const double* __restrict__ ipool,
              double* __restrict__ X, double* __restrict__ Wv, int ldx, int cofs) {
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const SubDev d = sub[s.sub];
  const int ncl = min(NCB, ldx - cofs);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nu = s.f - s.npiv;
  double* Xs = X + d.x_off * ldx + cofs;
  double* t = Wv + s.vec_off * NCB;
  for (int cc = warp; cc < TB; cc += SWT / 32) {
    const int col = w.a * TB + cc;
    if (col >= s.npiv) break;
    double acc[NCB];
#pragma unroll
    for (int c = 0; c < NCB; ++c) acc[c] = 0.0;
    if (MODE == 0) {
      const double* Lc = pool + s.front_off + (long long)col * s.ld + s.npiv;
      const int* rw = rows + s.rows_off;
      for (int q0 = 0; q0 < nu; q0 += 128) {  // 4 independent rows per lane
        double l[4];
        const double* xr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = q0 + lane + 32 * u;
          l[u] = q < nu ? Lc[q] : 0.0;
          xr[u] = q < nu ? Xs + (long long)rw[q] * ldx : Xs;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int c = 0; c < NCB; ++c)
            if (c < ncl) acc[c] += l[u] * xr[u][c];
      }
    } else {
      const double* Ic = ipool + s.inv_off + (long long)col * s.ldi;
      const bool from_t = nu > 0;
      for (int q0 = col; q0 < s.npiv; q0 += 128) {
        double l[4];
        int qq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          qq[u] = q0 + lane + 32 * u;
          l[u] = qq[u] < s.npiv ? Ic[qq[u]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (qq[u] >= s.npiv) continue;
#pragma unroll
          for (int c = 0; c < NCB; ++c) {
            const double tv = from_t ? t[qq[u] * NCB + c] : (c < ncl ? Xs[(long long)(s.c0 + qq[u]) * ldx + c] : 0.0);
            acc[c] += l[u] * tv;
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NCB; ++c) acc[c] = warp_sum(acc[c]);
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < NCB; ++c) {
        if (MODE == 0) {
          t[col * NCB + c] = (c < ncl ? Xs[(long long)(s.c0 + col) * ldx + c] : 0.0) - acc[c];
        } else if (c < ncl) {
          Xs[(long long)(s.c0 + col) * ldx + c] = acc[c];
        }
      }
    }
  }
}

template <int NCB>
static void sweeps_t(ietidp_s* h, double* X, bool fwd, bool bwd, int cofs) {
  cudaStream_t st = h->stream;
  const Plan& P = h->plan;
  const Work* W = reinterpret_cast<const Work*>(h->d_work.p);
  const int ldx = h->nrhs;
  if (fwd)
    for (int L = 0; L <= P.max_level; ++L) {
      const LevelPlan& lp = P.levels[L];
      if (!lp.sn_n) continue;
      k_fs_assemble<NCB><<<lp.sn_n, SWT, 0, st>>>(h->d_level_sn.p + lp.sn_off, h->d_sn.p, h->d_sub.p, h->d_rel.p,
                                                  h->d_children.p, X, h->vecw.p, ldx, cofs);
      IETI_LAUNCHED(h);
      if (lp.fs_n) {
        k_fs_gemv<0, NCB><<<lp.fs_n, SWT, 0, st>>>(W + lp.fs_off, h->d_sn.p, h->d_sub.p, h->pool.p, h->ipool.p, X,
                                                   h->vecw.p, ldx, cofs);
        IETI_LAUNCHED(h);
      }
      if (lp.fu_n) {
        k_fs_gemv<1, NCB><<<lp.fu_n, SWT, 0, st>>>(W + lp.fu_off, h->d_sn.p, h->d_sub.p, h->pool.p, h->ipool.p, X,
                                                   h->vecw.p, ldx, cofs);
        IETI_LAUNCHED(h);
      }
    }
  if (bwd)
    for (int L = P.max_level; L >= 0; --L) {
      const LevelPlan& lp = P.levels[L];
      if (lp.bt_n) {
        k_bs_gemv<0, NCB><<<lp.bt_n, SWT, 0, st>>>(W + lp.bt_off, h->d_sn.p, h->d_sub.p, h->d_rows.p, h->pool.p,
                                                   h->ipool.p, X, h->vecw.p, ldx, cofs);
        IETI_LAUNCHED(h);
      }
      if (lp.bx_n) {
        k_bs_gemv<1, NCB><<<lp.bx_n, SWT, 0, st>>>(W + lp.bx_off, h->d_sn.p, h->d_sub.p, h->d_rows.p, h->pool.p,
                                                   h->ipool.p, X, h->vecw.p, ldx, cofs);
        IETI_LAUNCHED(h);
      }
    }
  IETI_CHECK_LAUNCH();
}

// Forward sweep of one level for every column (nrhs <= 16), on stream st: used by the
// factorisation's side stream, level by level as the partitioned inverse completes.
template <int NCB>
static void fwd_level_t(ietidp_s* h, double* X, int L, cudaStream_t st) {
  const LevelPlan& lp = h->plan.levels[L];
  const Work* W = reinterpret_cast<const Work*>(h->d_work.p);
  const int ldx = h->nrhs;
  if (!lp.sn_n) return;
  k_fs_assemble<NCB><<<lp.sn_n, SWT, 0, st>>>(h->d_level_sn.p + lp.sn_off, h->d_sn.p, h->d_sub.p, h->d_rel.p,
                                              h->d_children.p, X, h->vecw.p, ldx, 0);
  IETI_LAUNCHED_SIDE(h);
  if (lp.fs_n) {
    k_fs_gemv<0, NCB><<<lp.fs_n, SWT, 0, st>>>(W + lp.fs_off, h->d_sn.p, h->d_sub.p, h->pool.p, h->ipool.p, X,
                                               h->vecw.p, ldx, 0);
    IETI_LAUNCHED_SIDE(h);
  }
  if (lp.fu_n) {
    k_fs_gemv<1, NCB><<<lp.fu_n, SWT, 0, st>>>(W + lp.fu_off, h->d_sn.p, h->d_sub.p, h->pool.p, h->ipool.p, X,
                                               h->vecw.p, ldx, 0);
    IETI_LAUNCHED_SIDE(h);
  }
}
void fwd_sweep_level(ietidp_s* h, double* X, int L, cudaStream_t st) {
  const int n = h->nrhs;
  if (n == 1) fwd_level_t<1>(h, X, L, st);
  else if (n == 2) fwd_level_t<2>(h, X, L, st);
  else if (n <= 4) fwd_level_t<4>(h, X, L, st);
  else if (n <= 8) fwd_level_t<8>(h, X, L, st);
  else fwd_level_t<16>(h, X, L, st);
}

// X (ne rows per subdomain x nrhs) <- L^-1 X (forward) and/or L^-T X (backward).
void run_sweeps(ietidp_s* h, double* X, bool fwd, bool bwd) {
  const int nc = h->nrhs;
  for (int c0 = 0; c0 < nc; c0 += 16) {
    const int n = nc - c0;
    if (n == 1) sweeps_t<1>(h, X, fwd, bwd, c0);
    else if (n == 2) sweeps_t<2>(h, X, fwd, bwd, c0);
    else if (n <= 4) sweeps_t<4>(h, X, fwd, bwd, c0);
    else if (n <= 8) sweeps_t<8>(h, X, fwd, bwd, c0);
    else sweeps_t<16>(h, X, fwd, bwd, c0);
  }
}

}  // namespace ieti
