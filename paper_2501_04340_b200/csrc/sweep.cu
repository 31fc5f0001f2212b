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
  if constexpr (NCB == 16) {
    // 16 columns: the tile product on the FP64 tensor pipe. Warp w owns rows 8w .. 8w+7 of the
    // tile and both 8-column halves: per 4-deep k step one global load of the A fragment
    // (A[8w + lane/4][k + lane%4], 8 consecutive rows of a column: 64-byte segments), two
    // shared-memory loads of the staged vector rows and two DMMAs; eight steps' loads in flight.
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int Rw = row0 + 8 * warp + g;
    const bool rok = Rw < nrows;
    const double* Aw = (MODE == 0) ? ipool + s.inv_off + Rw : pool + s.front_off + s.npiv + Rw;
    double dacc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int k0 = 0; k0 < kend; k0 += TB) {
      __syncthreads();
      for (int e = threadIdx.x; e < TB * NCB; e += SWT) {
        const int k = e / NCB, c = e % NCB;
        double v = 0.0;
        if (k0 + k < kend) v = (MODE == 0) ? vin[(k0 + k) * NCB + c] : (c < ncl ? yin[(long long)(k0 + k) * ldx + c] : 0.0);
        xs[k][c] = v;
      }
      __syncthreads();
      const int kn = min(TB, kend - k0);
      for (int kb = 0; kb < kn; kb += 32) {
        double a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = kb + 4 * u + t4;
          a[u] = (rok && k < kn) ? Aw[(long long)(k0 + k) * lda] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = kb + 4 * u + t4;
          if (kb + 4 * u < kn) {
            const int kk = min(k, TB - 1);
            dmma8x8x4(dacc[0][0], dacc[0][1], a[u], xs[kk][g]);
            dmma8x8x4(dacc[1][0], dacc[1][1], a[u], xs[kk][8 + g]);
          }
        }
      }
    }
    if (rok) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int c = 8 * hh + 2 * t4 + q;
          if (MODE == 0) {
            if (c < ncl) X[(d.x_off + s.c0 + Rw) * ldx + cofs + c] = dacc[hh][q];
          } else {
            Wv[(s.vec_off + s.npiv + Rw) * NCB + c] -= dacc[hh][q];
          }
        }
    }
    return;
  }
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

// Backward sweep, first step, split over BS_RB-row chunks of L21 (many CTAs, short
// dependent chains): partial[rc][col] = L21[chunk rc, col]^T x_rows[chunk rc] for the 64
// pivot columns of tile w.a. The chunk's x rows are gathered once into shared memory;
// warp w takes columns w, w+8, ..., two at a time, lanes over the contiguous rows.
template <int NCB>
__global__ void __launch_bounds__(SWT)
    k_bs_partial(const Work* __restrict__ work, const SnDev* __restrict__ sn, const SubDev* __restrict__ sub,
                 const int* __restrict__ rows, const double* __restrict__ pool, const double* __restrict__ X,
                 double* __restrict__ bpart, int ldx, int cofs) {
  constexpr int XS = NCB | 1;  // odd row stride: conflict-free column reads
  __shared__ double xs[BS_RB][XS];
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const SubDev d = sub[s.sub];
  const int ncl = min(NCB, ldx - cofs);
  const int nu = s.f - s.npiv;
  const int q0 = w.b * BS_RB, nq = min(BS_RB, nu - q0);
  const int* rw = rows + s.rows_off + q0;
  const double* Xs = X + d.x_off * ldx + cofs;
  for (int e = threadIdx.x; e < BS_RB * NCB; e += SWT) {
    const int q = e / NCB, c = e - q * NCB;
    xs[q][c] = (q < nq && c < ncl) ? Xs[(long long)rw[q] * ldx + c] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (NCB == 16) {
    // 16 columns: partial[col][c] = sum_q L21[q][col] x[q][c] on the FP64 tensor pipe; warp w owns
    // the pivot columns 8w .. 8w+7 of the tile (fragment rows), lanes%4 the 4 rows q of a step;
    // eight steps' loads in flight, no shuffle reductions
    const int g = lane >> 2, t4 = lane & 3;
    const int col = w.a * TB + 8 * warp + g;
    const bool cok = col < s.npiv;
    const double* Lc = pool + s.front_off + (long long)col * s.ld + s.npiv + q0;
    double dacc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int kb = 0; kb < nq; kb += 32) {
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = kb + 4 * u + t4;
        a[u] = (cok && q < nq) ? Lc[q] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (kb + 4 * u < nq) {
          const int qq = min(kb + 4 * u + t4, BS_RB - 1);
          dmma8x8x4(dacc[0][0], dacc[0][1], a[u], xs[qq][g]);
          dmma8x8x4(dacc[1][0], dacc[1][1], a[u], xs[qq][8 + g]);
        }
    }
    if (cok) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2)
          bpart[s.bp_off + ((long long)w.b * s.npiv + col) * NCB + 8 * hh + 2 * t4 + q2] = dacc[hh][q2];
    }
    return;
  }
  for (int cc = warp; cc < TB; cc += 2 * (SWT / 32)) {
    double acc[2][NCB];
    bool okc[2];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      okc[h2] = w.a * TB + cc + h2 * (SWT / 32) < s.npiv;
#pragma unroll
      for (int c = 0; c < NCB; ++c) acc[h2][c] = 0.0;
    }
    if (!okc[0]) break;
    double l[2][BS_RB / 32];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int col = w.a * TB + cc + h2 * (SWT / 32);
      const double* Lc = pool + s.front_off + (long long)col * s.ld + s.npiv + q0;
#pragma unroll
      for (int u = 0; u < BS_RB / 32; ++u) {
        const int q = lane + 32 * u;
        l[h2][u] = (okc[h2] && q < nq) ? Lc[q] : 0.0;
      }
    }
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
      for (int u = 0; u < BS_RB / 32; ++u)
#pragma unroll
        for (int c = 0; c < NCB; ++c) acc[h2][c] += l[h2][u] * xs[lane + 32 * u][c];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
#pragma unroll
      for (int c = 0; c < NCB; ++c) acc[h2][c] = warp_sum(acc[h2][c]);
      const int col = w.a * TB + cc + h2 * (SWT / 32);
      if (lane == 0 && okc[h2]) {
#pragma unroll
        for (int c = 0; c < NCB; ++c) bpart[s.bp_off + ((long long)w.b * s.npiv + col) * NCB + c] = acc[h2][c];
      }
    }
  }
}

// Backward sweep, second step, split over BS_RB-row chunks of L11^-1:
// partial[rc][col] = sum_{r in chunk rc, r >= col} Linv[r][col] t[r], t from Wv (or,
// for a supernode without update rows, the X pivot rows themselves).
template <int NCB>
__global__ void __launch_bounds__(SWT)
    k_bx_partial(const Work* __restrict__ work, const SnDev* __restrict__ sn, const SubDev* __restrict__ sub,
                 const double* __restrict__ ipool, const double* __restrict__ X, const double* __restrict__ Wv,
                 double* __restrict__ bpart, int ldx, int cofs) {
  constexpr int XS = NCB | 1;
  __shared__ double ts[BS_RB][XS];
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const SubDev d = sub[s.sub];
  const int ncl = min(NCB, ldx - cofs);
  const int r0 = w.b * BS_RB, nr = min(BS_RB, s.npiv - r0);
  const bool from_t = s.f > s.npiv;
  const double* Xs = X + d.x_off * ldx + cofs;
  (void)Wv;
  // t = y - L21^T x_rows: the pivot rows of X minus the step-1 partials (fixed order)
  const int nchu = (s.f - s.npiv + BS_RB - 1) / BS_RB;
  for (int e = threadIdx.x; e < BS_RB * NCB; e += SWT) {
    const int q = e / NCB, c = e - q * NCB;
    double v = 0.0;
    if (q < nr && c < ncl) {
      double p = 0.0;
      if (from_t)
        for (int rc = 0; rc < nchu; ++rc) p += bpart[s.bp_off + ((long long)rc * s.npiv + r0 + q) * NCB + c];
      v = Xs[(long long)(s.c0 + r0 + q) * ldx + c] - p;
    }
    ts[q][c] = v;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (NCB == 16) {  // as k_bs_partial: partial[col][c] = sum_{r >= col} Linv[r][col] t[r][c] by DMMA
    const int g = lane >> 2, t4 = lane & 3;
    const int col = w.a * TB + 8 * warp + g;
    const bool cok = col < s.npiv;
    const double* Ic = ipool + s.inv_off + (long long)col * s.ldi + r0;
    double dacc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int kb = 0; kb < nr; kb += 32) {
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = kb + 4 * u + t4;
        a[u] = (cok && q < nr && r0 + q >= col) ? Ic[q] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (kb + 4 * u < nr) {
          const int qq = min(kb + 4 * u + t4, BS_RB - 1);
          dmma8x8x4(dacc[0][0], dacc[0][1], a[u], ts[qq][g]);
          dmma8x8x4(dacc[1][0], dacc[1][1], a[u], ts[qq][8 + g]);
        }
    }
    if (cok) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2)
          bpart[s.bp_off + ((long long)(nchu + w.b) * s.npiv + col) * NCB + 8 * hh + 2 * t4 + q2] = dacc[hh][q2];
    }
    return;
  }
  for (int cc = warp; cc < TB; cc += 2 * (SWT / 32)) {
    double acc[2][NCB];
    bool okc[2];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      okc[h2] = w.a * TB + cc + h2 * (SWT / 32) < s.npiv;
#pragma unroll
      for (int c = 0; c < NCB; ++c) acc[h2][c] = 0.0;
    }
    if (!okc[0]) break;
    double l[2][BS_RB / 32];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int col = w.a * TB + cc + h2 * (SWT / 32);
      const double* Ic = ipool + s.inv_off + (long long)col * s.ldi + r0;
#pragma unroll
      for (int u = 0; u < BS_RB / 32; ++u) {
        const int q = lane + 32 * u;
        l[h2][u] = (okc[h2] && q < nr && r0 + q >= col) ? Ic[q] : 0.0;
      }
    }
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
      for (int u = 0; u < BS_RB / 32; ++u)
#pragma unroll
        for (int c = 0; c < NCB; ++c) acc[h2][c] += l[h2][u] * ts[lane + 32 * u][c];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
#pragma unroll
      for (int c = 0; c < NCB; ++c) acc[h2][c] = warp_sum(acc[h2][c]);
      const int col = w.a * TB + cc + h2 * (SWT / 32);
      if (lane == 0 && okc[h2]) {
#pragma unroll
        for (int c = 0; c < NCB; ++c)
          bpart[s.bp_off + ((long long)(nchu + w.b) * s.npiv + col) * NCB + c] = acc[h2][c];
      }
    }
  }
}

// x[col] = sum over the row chunks rc >= col's tile of the partials (fixed order) -> X
template <int NCB>
__global__ void __launch_bounds__(SWT)
    k_bx_red(const Work* __restrict__ work, const SnDev* __restrict__ sn, const SubDev* __restrict__ sub,
             const double* __restrict__ bpart, double* __restrict__ X, int ldx, int cofs) {
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const SubDev d = sub[s.sub];
  const int ncl = min(NCB, ldx - cofs);
  const int nch = (s.npiv + BS_RB - 1) / BS_RB, nchu = (s.f - s.npiv + BS_RB - 1) / BS_RB;
  double* Xs = X + d.x_off * ldx + cofs;
  for (int e = threadIdx.x; e < TB * NCB; e += SWT) {
    const int cc = e / NCB, c = e - cc * NCB;
    const int col = w.a * TB + cc;
    if (col >= s.npiv || c >= ncl) continue;
    double v = 0.0;
    for (int rc = w.a * TB / BS_RB; rc < nch; ++rc)
      v += bpart[s.bp_off + ((long long)(nchu + rc) * s.npiv + col) * NCB + c];
    Xs[(long long)(s.c0 + col) * ldx + c] = v;
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
        k_bs_partial<NCB><<<lp.bt_n, SWT, 0, st>>>(W + lp.bt_off, h->d_sn.p, h->d_sub.p, h->d_rows.p, h->pool.p, X,
                                                   h->bpart.p, ldx, cofs);
        IETI_LAUNCHED(h);
      }
      if (lp.bx_n) {
        k_bx_partial<NCB><<<lp.bx_n, SWT, 0, st>>>(W + lp.bx_off, h->d_sn.p, h->d_sub.p, h->ipool.p, X, h->vecw.p,
                                                   h->bpart.p, ldx, cofs);
        IETI_LAUNCHED(h);
        k_bx_red<NCB><<<lp.bxr_n, SWT, 0, st>>>(W + lp.bxr_off, h->d_sn.p, h->d_sub.p, h->bpart.p, X, ldx, cofs);
        IETI_LAUNCHED(h);
      }
    }
  IETI_CHECK_LAUNCH();
}

// Forward sweep of one level for every column (nrhs <= 16), on stream st: used by the
// factorisation's side stream, level by level as the partitioned inverse completes.
template <int NCB>
static void fwd_level_t(ietidp_s* h, double* X, const LevelPlan& lp, cudaStream_t st) {
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
void fwd_sweep_lp(ietidp_s* h, double* X, const LevelPlan& lp, cudaStream_t st) {
  const int n = h->nrhs;
  if (n == 1) fwd_level_t<1>(h, X, lp, st);
  else if (n == 2) fwd_level_t<2>(h, X, lp, st);
  else if (n <= 4) fwd_level_t<4>(h, X, lp, st);
  else if (n <= 8) fwd_level_t<8>(h, X, lp, st);
  else fwd_level_t<16>(h, X, lp, st);
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
