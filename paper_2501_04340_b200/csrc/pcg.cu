// The PCG loop on F_DP lambda = d_DP.
//
// Per iteration (all on device, one CUDA-graph while-loop, no host sync):
//   k_local<SOLVE>  per subdomain: b = B_I^T p (gather), g_k = G_k^T b,
//                   x = L_II^-T L_II^-1 b (tile-streamed, inverted diagonal tiles)
//   k_coarse        g = sum_k C_k g_k, z = S_PP^-1 g            (one CTA)
//   k_bgather       q = sum_k B_I (x_k + G_k C_k^T z), partial p.q
//   k_cg_alpha      alpha, lambda += alpha p, r -= alpha q, partial r.r
//   k_local<PREC>   b = B_D^T r, z_loc = L_II (L_II^T b)        (F2)
//   k_bgather       z = sum_k B_D z_loc, partial r.z
//   k_cg_beta       beta, p = z + beta p
//   k_ctl           iteration counts, stop test, graph condition
// Vectors are interleaved: v[j * ncols + c]. Dot products are fixed-order
// two-stage reductions (per-block partials, reduced redundantly by consumers),
// so results are bit-reproducible run to run.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace ieti {

struct PcgState {
  int it, done, max_iter, fixed, ncols, pad0;
  double tol;
  int active[IETIDP_MAX_RHS];
  int iters[IETIDP_MAX_RHS];
  double rz[IETIDP_MAX_RHS];
  double r0[IETIDP_MAX_RHS];
};

constexpr int NBLK = 296;  // blocks of the vector kernels = 2 x 148 SMs
constexpr int VT = 256;    // threads of the vector kernels

// ---------------------------------------------------------------------------
// Per-subdomain tile-streamed kernel
// ---------------------------------------------------------------------------
enum StepKind { ACC_N = 0, ACC_T = 1, DIAG_N = 2, DIAG_T = 3, LAST_N = 4, LAST_T = 5 };

struct Step {
  int src;   // >= 0: tile index into tiles; < 0: -1-index into dtiles
  short kind, blk;  // blk: input vector block (ACC), or the finalised block
};

constexpr int MAX_STEPS = 2 * (32 * 33 / 2 + 32);

__device__ __forceinline__ void load_tile_async(double* dst, const double* src, int tid, int nthreads) {
  for (int q = tid; q < TB * TB / 2; q += nthreads) {
    const int r = q >> 5, c = q & 31;
    cp_async16(dst + r * TB + ((c ^ (r & 7)) << 1), src + r * TB + 2 * c);
  }
}

// MODE 0: x = L^-T L^-1 b (F-apply local part), also g_k = G_k^T b.
// MODE 1: z = L L^T b (Dirichlet preconditioner local part).
// NCP = 1: DFMA path (warp owns 8 rows, lanes split columns);
// NCP = 8/16: DMMA path (warp owns 8 output rows, NCP/8 column blocks).
template <int MODE, int NCP, int STAGES>
__global__ void __launch_bounds__(256, 1)
    k_local(const SubDev* __restrict__ sub, const double* __restrict__ tiles, const double* __restrict__ dtiles,
            const double* __restrict__ G, const int* __restrict__ slot_lam, const float* __restrict__ slot_sign,
            const double* __restrict__ weight, const double* __restrict__ vin, double* __restrict__ vout,
            double* __restrict__ gk, int ncols, int c_off, const PcgState* __restrict__ st,
            const double* __restrict__ rr_part, int check) {
  extern __shared__ __align__(16) double smem[];
  constexpr int VS = (NCP == 1) ? 1 : NCP + 4;
  __shared__ Step steps[MAX_STEPS];
  __shared__ int nsteps_s;
  __shared__ double red[8][TB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncl = min(NCP, ncols - c_off);  // columns handled by this launch

  if (st) {
    if (st->done) return;
    if (MODE == 1 && check && !st->fixed) {
      // convergence of the columns after this iteration's r update (any active?)
      __shared__ int any_s;
      if (tid == 0) any_s = 0;
      __syncthreads();
      if (tid < st->ncols && st->active[tid]) {
        double s = 0.0;
        for (int b = 0; b < NBLK; ++b) s += rr_part[b * st->ncols + tid];
        if (!(sqrt(s) <= st->tol * st->r0[tid])) atomicOr(&any_s, 1);
      }
      __syncthreads();
      if (!any_s) return;
    }
  }
  const SubDev d = sub[blockIdx.x];
  if (d.nI == 0) return;
  const int nt = d.nt;
  double* ring = smem;
  double* vec = smem + STAGES * TILE_ELEMS;
  double* scratch = vec + nt * TB * VS;

  // ---- step list ----
  if (tid == 0) {
    int n = 0;
    auto T = [](int i, int j) { return i * (i + 1) / 2 + j; };
    const int tb = (int)(d.tile_off / TILE_ELEMS), db = (int)(d.dtile_off / TILE_ELEMS);
    if (MODE == 0) {
      for (int i = 0; i < nt; ++i) {
        for (int j = 0; j < i; ++j) steps[n++] = {tb + T(i, j), ACC_N, (short)j};
        steps[n++] = {-1 - (db + i), DIAG_N, (short)i};
      }
      for (int i = nt - 1; i >= 0; --i) {
        for (int j = nt - 1; j > i; --j) steps[n++] = {tb + T(j, i), ACC_T, (short)j};
        steps[n++] = {-1 - (db + i), DIAG_T, (short)i};
      }
    } else {
      for (int j = 0; j < nt; ++j) {
        for (int i = nt - 1; i > j; --i) steps[n++] = {tb + T(i, j), ACC_T, (short)i};
        steps[n++] = {tb + T(j, j), LAST_T, (short)j};
      }
      for (int i = nt - 1; i >= 0; --i) {
        for (int j = 0; j < i; ++j) steps[n++] = {tb + T(i, j), ACC_N, (short)j};
        steps[n++] = {tb + T(i, i), LAST_N, (short)i};
      }
    }
    nsteps_s = n;
  }
  // ---- gather b (with sign and weight) ----
  const int nrow = nt * TB;
  for (int e = tid; e < nrow * VS; e += 256) {
    const int a = e / VS, c = e - a * VS;
    double v = 0.0;
    if (a < d.nI && c < ncl) {
      const int slot = (int)d.rI_off + a;
      const double w = weight ? weight[slot] : 1.0;
      v = (double)slot_sign[slot] * w * vin[(long long)slot_lam[slot] * ncols + c_off + c];
    }
    vec[e] = v;
  }
  __syncthreads();
  const int nsteps = nsteps_s;
  // ---- prologue prefetch (overlaps with g_k below) ----
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nsteps) {
      const Step sp = steps[s];
      const double* src = sp.src >= 0 ? tiles + (long long)sp.src * TILE_ELEMS : dtiles + (long long)(-1 - sp.src) * TILE_ELEMS;
      load_tile_async(ring + s * TILE_ELEMS, src, tid, 256);
    }
    cp_async_commit();
  }
  // ---- coarse: g_k = G_k^T b (MODE 0) ----
  if (MODE == 0 && gk && d.nP > 0) {
    const double* Gk = G + d.g_off;
    for (int pc = warp; pc < d.nP * ncl; pc += 8) {
      const int pi = pc / ncl, c = pc - pi * ncl;
      double acc = 0.0;
      for (int a = lane; a < d.nI; a += 32) acc += Gk[(long long)a * d.nP + pi] * vec[a * VS + c];
      acc = warp_sum(acc);
      if (lane == 0) gk[(long long)(d.prim_off + pi) * ncols + c_off + c] = acc;
    }
  }

  // accumulators
  double accN[8];   // DFMA: per-lane partial row sums (rows 8w+rr)
  double accT[2];   // DFMA: per-warp partial column sums (cols lane, lane+32)
  double acc[NCP == 1 ? 1 : NCP / 8][2];  // DMMA: rows 8w+g, cols nb*8+2t+q
#pragma unroll
  for (int i = 0; i < 8; ++i) accN[i] = 0.0;
  accT[0] = accT[1] = 0.0;
#pragma unroll
  for (int i = 0; i < (NCP == 1 ? 1 : NCP / 8); ++i) acc[i][0] = acc[i][1] = 0.0;
  const int g = lane >> 2, t4 = lane & 3;

  for (int s = 0; s < nsteps; ++s) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int sn = s + STAGES - 1;
      if (sn < nsteps) {
        const Step sp = steps[sn];
        const double* src = sp.src >= 0 ? tiles + (long long)sp.src * TILE_ELEMS : dtiles + (long long)(-1 - sp.src) * TILE_ELEMS;
        load_tile_async(ring + (sn % STAGES) * TILE_ELEMS, src, tid, 256);
      }
      cp_async_commit();
    }
    const double* Tt = ring + (s % STAGES) * TILE_ELEMS;
    const Step sp = steps[s];
    double* vb = vec + sp.blk * TB * VS;
    if constexpr (NCP == 1) {
      // ------------------------- DFMA path -------------------------
      if (sp.kind == ACC_N || sp.kind == LAST_N) {
        const double x0 = vb[lane], x1 = vb[lane + 32];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int r = warp * 8 + rr;
          accN[rr] += Tt[swz(r, lane)] * x0 + Tt[swz(r, lane + 32)] * x1;
        }
        if (sp.kind == LAST_N) {
          double full[8];
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) full[rr] = warp_sum(accN[rr]);
          __syncthreads();
          if (lane < 8) {
            double v = full[0];
#pragma unroll
            for (int rr = 1; rr < 8; ++rr)
              if (lane == rr) v = full[rr];
            vb[warp * 8 + lane] = v;
          }
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) accN[rr] = 0.0;
        }
      } else if (sp.kind == ACC_T || sp.kind == LAST_T) {
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int r = warp * 8 + rr;
          const double xr = vb[r];
          accT[0] += Tt[swz(r, lane)] * xr;
          accT[1] += Tt[swz(r, lane + 32)] * xr;
        }
        if (sp.kind == LAST_T) {
          red[warp][lane] = accT[0];
          red[warp][lane + 32] = accT[1];
          __syncthreads();
          if (tid < TB) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) v += red[w][tid];
            vb[tid] = v;
          }
          accT[0] = accT[1] = 0.0;
        }
      } else if (sp.kind == DIAG_N) {
        // t = b_i - sum_j L_ij y_j ; y_i = Dinv_i t
        double full[8];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) full[rr] = warp_sum(accN[rr]);
        if (lane < 8) {
          double v = full[0];
#pragma unroll
          for (int rr = 1; rr < 8; ++rr)
            if (lane == rr) v = full[rr];
          scratch[warp * 8 + lane] = vb[warp * 8 + lane] - v;
        }
        __syncthreads();
        const double t0 = scratch[lane], t1 = scratch[lane + 32];
        double y[8];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int r = warp * 8 + rr;
          y[rr] = warp_sum(Tt[swz(r, lane)] * t0 + Tt[swz(r, lane + 32)] * t1);
        }
        if (lane < 8) {
          double v = y[0];
#pragma unroll
          for (int rr = 1; rr < 8; ++rr)
            if (lane == rr) v = y[rr];
          vb[warp * 8 + lane] = v;
        }
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) accN[rr] = 0.0;
      } else {  // DIAG_T: t = y_i - sum_{j>i} L_ji^T x_j ; x_i = Dinv_i^T t
        red[warp][lane] = accT[0];
        red[warp][lane + 32] = accT[1];
        __syncthreads();
        if (tid < TB) {
          double v = 0.0;
#pragma unroll
          for (int w = 0; w < 8; ++w) v += red[w][tid];
          scratch[tid] = vb[tid] - v;
        }
        __syncthreads();
        double p0 = 0.0, p1 = 0.0;
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int r = warp * 8 + rr;
          const double tr = scratch[r];
          p0 += Tt[swz(r, lane)] * tr;
          p1 += Tt[swz(r, lane + 32)] * tr;
        }
        red[warp][lane] = p0;
        red[warp][lane + 32] = p1;
        __syncthreads();
        if (tid < TB) {
          double v = 0.0;
#pragma unroll
          for (int w = 0; w < 8; ++w) v += red[w][tid];
          vb[tid] = v;
        }
        accT[0] = accT[1] = 0.0;
      }
    } else {
      // ------------------------- DMMA path -------------------------
      constexpr int NB = NCP / 8;
      const bool trans = (sp.kind == ACC_T || sp.kind == LAST_T);
      if (sp.kind == ACC_N || sp.kind == ACC_T || sp.kind == LAST_N || sp.kind == LAST_T) {
#pragma unroll 4
        for (int k0 = 0; k0 < TB; k0 += 4) {
          const double a = trans ? Tt[swz(k0 + t4, warp * 8 + g)] : Tt[swz(warp * 8 + g, k0 + t4)];
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) dmma8x8x4(acc[nb][0], acc[nb][1], a, vb[(k0 + t4) * VS + nb * 8 + g]);
        }
        if (sp.kind == LAST_N || sp.kind == LAST_T) {
          __syncthreads();
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            vb[(warp * 8 + g) * VS + nb * 8 + 2 * t4] = acc[nb][0];
            vb[(warp * 8 + g) * VS + nb * 8 + 2 * t4 + 1] = acc[nb][1];
            acc[nb][0] = acc[nb][1] = 0.0;
          }
        }
      } else {
        // DIAG: t = v_i - acc -> scratch ; v_i = D t (N) or D^T t (T)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int idx = (warp * 8 + g) * VS + nb * 8 + 2 * t4 + q;
            scratch[idx] = vb[idx] - acc[nb][q];
            acc[nb][q] = 0.0;
          }
        __syncthreads();
        const bool tr = (sp.kind == DIAG_T);
#pragma unroll 4
        for (int k0 = 0; k0 < TB; k0 += 4) {
          const double a = tr ? Tt[swz(k0 + t4, warp * 8 + g)] : Tt[swz(warp * 8 + g, k0 + t4)];
#pragma unroll
          for (int nb = 0; nb < NB; ++nb)
            dmma8x8x4(acc[nb][0], acc[nb][1], a, scratch[(k0 + t4) * VS + nb * 8 + g]);
        }
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          vb[(warp * 8 + g) * VS + nb * 8 + 2 * t4] = acc[nb][0];
          vb[(warp * 8 + g) * VS + nb * 8 + 2 * t4 + 1] = acc[nb][1];
          acc[nb][0] = acc[nb][1] = 0.0;
        }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  for (int e = tid; e < d.nI * ncl; e += 256) {
    const int a = e / ncl, c = e - a * ncl;
    vout[(d.rI_off + a) * ncols + c_off + c] = vec[a * VS + c];
  }
}

// ---------------------------------------------------------------------------
// Vector kernels
// ---------------------------------------------------------------------------
__device__ __forceinline__ int pow2ge(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Block reduction of per-thread column partials (thread column c = tid % P2);
// writes partial[blockIdx.x * ncols + c].
__device__ void block_col_reduce(double v, int ncols, int P2, double* partial) {
  __shared__ double red[VT];
  const int tid = threadIdx.x;
  red[tid] = v;
  __syncthreads();
  for (int s = VT / 2; s >= P2; s >>= 1) {
    if (tid < s) red[tid] += red[tid + s];
    __syncthreads();
  }
  if (tid < ncols) partial[blockIdx.x * ncols + tid] = red[tid];
}

// out[j][c] = sum_{2 slots} sign * w * (x[slot][c] + coef * G_k[row] . z[C_k^T][c])
template <bool COARSE>
__global__ void __launch_bounds__(VT)
    k_bgather(int m, int ncols, const LamDev* __restrict__ lam, const double* __restrict__ x,
              const double* __restrict__ weight, const long long* __restrict__ slot_goff,
              const int* __restrict__ slot_np, const int* __restrict__ slot_poff, const double* __restrict__ G,
              const int* __restrict__ prim_gid, const double* __restrict__ z, double coef, double* __restrict__ out,
              const double* __restrict__ dotv, double* __restrict__ partial, const PcgState* __restrict__ st) {
  if (st && st->done) return;
  const int P2 = pow2ge(ncols);
  const int c = threadIdx.x % P2, rl = threadIdx.x / P2, R = VT / P2;
  double dot = 0.0;
  if (c < ncols) {
    for (int j = blockIdx.x * R + rl; j < m; j += gridDim.x * R) {
      const LamDev L = lam[j];
      double val = 0.0;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int a = L.slot[q];
        double xv = x[(long long)a * ncols + c];
        if (COARSE) {
          const int np = slot_np[a];
          const double* Gr = G + slot_goff[a];
          const int* gid = prim_gid + slot_poff[a];
          double s = 0.0;
          for (int p = 0; p < np; ++p) s += Gr[p] * z[gid[p] * ncols + c];
          xv += coef * s;
        }
        val += (double)L.sign[q] * (weight ? weight[a] : 1.0) * xv;
      }
      out[(long long)j * ncols + c] = val;
      if (dotv) dot += val * dotv[(long long)j * ncols + c];
    }
  }
  if (partial) block_col_reduce(dot, ncols, P2, partial);
}

// z = S^-1 (add + sum_k C_k g_k)  (one CTA)
__global__ void __launch_bounds__(1024)
    k_coarse(int ng, int ncols, const int* __restrict__ pcon_ptr, const int* __restrict__ pcon_src,
             const double* __restrict__ gk, const double* __restrict__ add, const double* __restrict__ Sinv,
             double* __restrict__ z, const PcgState* __restrict__ st) {
  if (st && st->done) return;
  extern __shared__ double gs[];  // ng x ncols
  for (int e = threadIdx.x; e < ng * ncols; e += blockDim.x) {
    const int gi = e / ncols, c = e - gi * ncols;
    double s = add ? add[e] : 0.0;
    for (int q = pcon_ptr[gi]; q < pcon_ptr[gi + 1]; ++q) s += gk[(long long)pcon_src[q] * ncols + c];
    gs[e] = s;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int e = warp; e < ng * ncols; e += nw) {
    const int i = e / ncols, c = e - i * ncols;
    double s = 0.0;
    for (int j = lane; j < ng; j += 32) s += Sinv[(long long)i * ng + j] * gs[j * ncols + c];
    s = warp_sum(s);
    if (lane == 0) z[e] = s;
  }
}

__device__ void reduce_cols(const double* part, int nblk, int ncols, double* out_smem) {
  // thread c < ncols sums column c in fixed order
  if (threadIdx.x < ncols) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[b * ncols + threadIdx.x];
    out_smem[threadIdx.x] = s;
  }
}

__device__ void active_after(const PcgState* st, const double* rr_part, int* act) {
  __shared__ double rr[IETIDP_MAX_RHS];
  reduce_cols(rr_part, NBLK, st->ncols, rr);
  __syncthreads();
  if (threadIdx.x < st->ncols) {
    const int c = threadIdx.x;
    int a = st->active[c];
    if (a && !st->fixed && sqrt(rr[c]) <= st->tol * st->r0[c]) a = 0;
    act[c] = a;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(VT)
    k_cg_alpha(int m, PcgState* __restrict__ st, const double* __restrict__ pq_part, double* __restrict__ lam,
               double* __restrict__ r, const double* __restrict__ p, const double* __restrict__ q,
               double* __restrict__ rr_part) {
  if (st->done) return;
  const int ncols = st->ncols;
  __shared__ double pq[IETIDP_MAX_RHS], alpha[IETIDP_MAX_RHS];
  reduce_cols(pq_part, NBLK, ncols, pq);
  __syncthreads();
  if (threadIdx.x < ncols) {
    const int c = threadIdx.x;
    alpha[c] = st->active[c] ? st->rz[c] / pq[c] : 0.0;
  }
  __syncthreads();
  const int P2 = pow2ge(ncols);
  const int c = threadIdx.x % P2, rl = threadIdx.x / P2, R = VT / P2;
  double acc = 0.0;
  if (c < ncols) {
    const bool act = st->active[c];
    const double a = alpha[c];
    for (int j = blockIdx.x * R + rl; j < m; j += gridDim.x * R) {
      const long long e = (long long)j * ncols + c;
      double rv = r[e];
      if (act) {
        lam[e] += a * p[e];
        rv -= a * q[e];
        r[e] = rv;
      }
      acc += rv * rv;
    }
  }
  block_col_reduce(acc, ncols, P2, rr_part);
}

__global__ void __launch_bounds__(VT)
    k_cg_beta(int m, const PcgState* __restrict__ st, const double* __restrict__ rr_part,
              const double* __restrict__ rz_part, double* __restrict__ p, const double* __restrict__ z) {
  if (st->done) return;
  const int ncols = st->ncols;
  __shared__ int act[IETIDP_MAX_RHS];
  __shared__ double rz[IETIDP_MAX_RHS], beta[IETIDP_MAX_RHS];
  active_after(st, rr_part, act);
  reduce_cols(rz_part, NBLK, ncols, rz);
  __syncthreads();
  if (threadIdx.x < ncols) beta[threadIdx.x] = rz[threadIdx.x] / st->rz[threadIdx.x];
  __syncthreads();
  const int P2 = pow2ge(ncols);
  const int c = threadIdx.x % P2, rl = threadIdx.x / P2, R = VT / P2;
  if (c < ncols && act[c]) {
    const double b = beta[c];
    for (int j = blockIdx.x * R + rl; j < m; j += gridDim.x * R) {
      const long long e = (long long)j * ncols + c;
      p[e] = z[e] + b * p[e];
    }
  }
}

__global__ void k_ctl(PcgState* __restrict__ st, const double* __restrict__ rr_part, const double* __restrict__ rz_part,
                      unsigned long long handle, int use_graph) {
  if (st->done) {
    if (use_graph && threadIdx.x == 0) cudaGraphSetConditional((cudaGraphConditionalHandle)handle, 0);
    return;
  }
  const int ncols = st->ncols;
  __shared__ int act[IETIDP_MAX_RHS];
  __shared__ double rz[IETIDP_MAX_RHS];
  active_after(st, rr_part, act);
  reduce_cols(rz_part, NBLK, ncols, rz);
  __syncthreads();
  if (threadIdx.x == 0) {
    int any = 0;
    for (int c = 0; c < ncols; ++c) {
      if (st->active[c]) st->iters[c]++;
      if (act[c]) st->rz[c] = rz[c];
      st->active[c] = act[c];
      any |= act[c];
    }
    st->it++;
    int stop = !any || (st->fixed ? st->it >= st->fixed : st->it >= st->max_iter);
    if (stop) st->done = 1;
    if (use_graph) cudaGraphSetConditional((cudaGraphConditionalHandle)handle, stop ? 0u : 1u);
  }
}

// ---- initialisation ----
__global__ void __launch_bounds__(VT) k_init(int m, int ncols, const double* __restrict__ d, double* __restrict__ lam,
                                             double* __restrict__ r, double* __restrict__ rr_part) {
  const int P2 = pow2ge(ncols);
  const int c = threadIdx.x % P2, rl = threadIdx.x / P2, R = VT / P2;
  double acc = 0.0;
  if (c < ncols)
    for (int j = blockIdx.x * R + rl; j < m; j += gridDim.x * R) {
      const long long e = (long long)j * ncols + c;
      lam[e] = 0.0;
      r[e] = d[e];
      acc += d[e] * d[e];
    }
  block_col_reduce(acc, ncols, P2, rr_part);
}

__global__ void k_init_ctl(PcgState* st, const double* __restrict__ rr_part, int ncols, int m, double tol,
                           int max_iter, int fixed) {
  __shared__ double rr[IETIDP_MAX_RHS];
  reduce_cols(rr_part, NBLK, ncols, rr);
  __syncthreads();
  if (threadIdx.x == 0) {
    st->it = 0;
    st->ncols = ncols;
    st->tol = tol;
    st->max_iter = max_iter;
    st->fixed = fixed;
    int any = 0;
    for (int c = 0; c < ncols; ++c) {
      st->r0[c] = sqrt(rr[c]);
      st->active[c] = (m > 0 && st->r0[c] > 0.0) ? 1 : 0;
      st->iters[c] = 0;
      st->rz[c] = 0.0;
      any |= st->active[c];
    }
    if (max_iter <= 0 && !fixed) any = 0;
    st->done = any ? 0 : 1;
  }
}

__global__ void __launch_bounds__(VT) k_init_p(int m, const PcgState* __restrict__ st, const double* __restrict__ z,
                                               double* __restrict__ p) {
  const long long n = (long long)m * st->ncols;
  for (long long e = blockIdx.x * (long long)VT + threadIdx.x; e < n; e += (long long)gridDim.x * VT) p[e] = z[e];
}

__global__ void k_init_rz(PcgState* st, const double* __restrict__ rz_part) {
  __shared__ double rz[IETIDP_MAX_RHS];
  reduce_cols(rz_part, NBLK, st->ncols, rz);
  __syncthreads();
  if (threadIdx.x < st->ncols) st->rz[threadIdx.x] = rz[threadIdx.x];
}

__global__ void __launch_bounds__(VT) k_resid(int m, int ncols, const double* __restrict__ d,
                                              const double* __restrict__ Fl, double* __restrict__ part) {
  const int P2 = pow2ge(ncols);
  const int c = threadIdx.x % P2, rl = threadIdx.x / P2, R = VT / P2;
  double acc = 0.0;
  if (c < ncols)
    for (int j = blockIdx.x * R + rl; j < m; j += gridDim.x * R) {
      const long long e = (long long)j * ncols + c;
      const double v = d[e] - Fl[e];
      acc += v * v;
    }
  block_col_reduce(acc, ncols, P2, part);
}

__global__ void k_transpose(int rows, int ncols, const double* __restrict__ in, double* __restrict__ out, int to_inter) {
  const long long n = (long long)rows * ncols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / ncols, c = e - j * ncols;
    if (to_inter) out[e] = in[c * rows + j];
    else out[c * rows + j] = in[e];
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
struct LocalCfg {
  int ncp, stages, smem;
};

static LocalCfg local_cfg(const ietidp_s* h, int ncols) {
  const int nt = (h->plan.max_nI + TB - 1) / TB;
  LocalCfg c{};
  if (ncols == 1) {
    c.ncp = 1;
    c.stages = 3;
    c.smem = (c.stages * TILE_ELEMS + nt * TB * 1 + TB * 1) * 8;
    return c;
  }
  const int ncps[2] = {16, 8};
  for (int ncp : ncps) {
    if (ncp == 16 && ncols <= 8) continue;
    const int vs = ncp + 4;
    for (int stages = 3; stages >= 2; --stages) {
      int bytes = (stages * TILE_ELEMS + nt * TB * vs + TB * vs) * 8;
      if (bytes <= 200 * 1024) return {ncp, stages, bytes};
    }
  }
  throw Error(IETIDP_E_ARG, "interface block too large for the shared-memory loop kernel");
}

template <int MODE, int NCP, int STAGES>
static void launch_local_t(ietidp_s* h, const LocalCfg& cfg, const double* weight, const double* vin, double* vout,
                           double* gk, int ncols, int c_off, const PcgState* st, const double* rr_part, int check) {
  auto kern = k_local<MODE, NCP, STAGES>;
  IETI_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, cfg.smem));
  const double* tl = h->tiles.p;
  kern<<<h->n_sub, 256, cfg.smem, h->stream>>>(h->d_sub.p, tl, h->dtiles.p, h->G.p, h->slot_lam.p, h->slot_sign.p,
                                               weight, vin, vout, gk, ncols, c_off, st, rr_part, check);
  IETI_LAUNCHED(h);
}

template <int MODE>
static void launch_local(ietidp_s* h, const double* weight, const double* vin, double* vout, double* gk, int ncols,
                         const PcgState* st, const double* rr_part, int check) {
  const LocalCfg cfg = local_cfg(h, ncols);
  for (int c0 = 0; c0 < ncols; c0 += cfg.ncp) {
    if (cfg.ncp == 1) launch_local_t<MODE, 1, 3>(h, cfg, weight, vin, vout, gk, ncols, c0, st, rr_part, check);
    else if (cfg.ncp == 16 && cfg.stages == 3) launch_local_t<MODE, 16, 3>(h, cfg, weight, vin, vout, gk, ncols, c0, st, rr_part, check);
    else if (cfg.ncp == 16) launch_local_t<MODE, 16, 2>(h, cfg, weight, vin, vout, gk, ncols, c0, st, rr_part, check);
    else if (cfg.stages == 3) launch_local_t<MODE, 8, 3>(h, cfg, weight, vin, vout, gk, ncols, c0, st, rr_part, check);
    else launch_local_t<MODE, 8, 2>(h, cfg, weight, vin, vout, gk, ncols, c0, st, rr_part, check);
  }
}

// out = sum_k B (x + coef G z) with optional weight; optional dot partials with dotv.
static void bgather(ietidp_s* h, int ncols, const double* x, const double* weight, const double* z, double coef,
                    double* out, const double* dotv, double* partial, const PcgState* st) {
  if (h->n_lambda == 0) return;
  const int grid = NBLK;
  if (z && h->n_primal > 0)
    k_bgather<true><<<grid, VT, 0, h->stream>>>(h->n_lambda, ncols, h->lam.p, x, weight, h->slot_goff.p, h->slot_np.p, h->slot_poff.p,
                                                h->G.p, h->d_prim_gid.p, z, coef, out, dotv, partial, st);
  else
    k_bgather<false><<<grid, VT, 0, h->stream>>>(h->n_lambda, ncols, h->lam.p, x, weight, nullptr, nullptr, nullptr,
                                                 nullptr, nullptr, nullptr, 0.0, out, dotv, partial, st);
  IETI_LAUNCHED(h);
}

static void coarse_apply(ietidp_s* h, int ncols, const double* gk, const double* add, double* z, const PcgState* st) {
  if (h->n_primal == 0) return;
  const int smem = h->n_primal * ncols * 8;
  if (smem > 48 * 1024)
    IETI_CUDA(cudaFuncSetAttribute((const void*)k_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_coarse<<<1, 1024, smem, h->stream>>>(h->n_primal, ncols, h->pcon_ptr.p, h->pcon_src.p, gk, add, h->Sinv.p, z, st);
  IETI_LAUNCHED(h);
}

// y = F_DP x (interleaved, ncols columns)
static void apply_F_inter(ietidp_s* h, int ncols, const double* x, double* y, const PcgState* st, const double* dotv,
                          double* partial) {
  if (h->n_lambda == 0) return;
  launch_local<0>(h, nullptr, x, h->xI.p, h->n_primal ? h->gk.p : nullptr, ncols, st, nullptr, 0);
  coarse_apply(h, ncols, h->gk.p, nullptr, h->zc.p, st);
  bgather(h, ncols, h->xI.p, nullptr, h->n_primal ? h->zc.p : nullptr, 1.0, y, dotv, partial, st);
}

static void apply_M_inter(ietidp_s* h, int ncols, const double* x, double* y, const PcgState* st, const double* rr_part,
                          int check, const double* dotv, double* partial) {
  if (h->n_lambda == 0) return;
  launch_local<1>(h, h->delta.p, x, h->zI.p, nullptr, ncols, st, rr_part, check);
  bgather(h, ncols, h->zI.p, h->delta.p, nullptr, 0.0, y, dotv, partial, st);
}

void run_apply_F(ietidp_s* h, int ncols, const double* x, double* y) {
  apply_F_inter(h, ncols, x, y, nullptr, nullptr, nullptr);
  IETI_CHECK_LAUNCH();
}
void run_apply_M(ietidp_s* h, int ncols, const double* x, double* y) {
  apply_M_inter(h, ncols, x, y, nullptr, nullptr, 0, nullptr, nullptr);
  IETI_CHECK_LAUNCH();
}

// exported for coarse.cu (d = e - G S^-1 ftilde)
void bgather_public(ietidp_s* h, int ncols, const double* x, const double* z, double coef, double* out) {
  bgather(h, ncols, x, nullptr, z, coef, out, nullptr, nullptr, nullptr);
}
void coarse_apply_public(ietidp_s* h, int ncols, const double* gk, const double* add, double* z) {
  coarse_apply(h, ncols, gk, add, z, nullptr);
}

static int body_launches(ietidp_s* h, int ncols) {
  const LocalCfg cfg = local_cfg(h, ncols);
  const int chunks = (ncols + cfg.ncp - 1) / cfg.ncp;
  return 2 * chunks + (h->n_primal ? 1 : 0) + 2 + 3;
}

static void iteration_body(ietidp_s* h, PcgState* st, int use_graph) {
  const int nc = h->nrhs, m = h->n_lambda;
  double* pq_part = h->partial.p;
  double* rr_part = h->partial.p + NBLK * nc;
  double* rz_part = h->partial.p + 2 * NBLK * nc;
  apply_F_inter(h, nc, h->p_vec.p, h->q_vec.p, st, h->p_vec.p, pq_part);
  k_cg_alpha<<<NBLK, VT, 0, h->stream>>>(m, st, pq_part, h->lam_vec.p, h->r_vec.p, h->p_vec.p, h->q_vec.p, rr_part);
  IETI_LAUNCHED(h);
  apply_M_inter(h, nc, h->r_vec.p, h->z_vec.p, st, rr_part, 1, h->r_vec.p, rz_part);
  k_cg_beta<<<NBLK, VT, 0, h->stream>>>(m, st, rr_part, rz_part, h->p_vec.p, h->z_vec.p);
  IETI_LAUNCHED(h);
  k_ctl<<<1, 64, 0, h->stream>>>(st, rr_part, rz_part, (unsigned long long)h->cond_handle, use_graph);
  IETI_LAUNCHED(h);
}

static bool build_graph(ietidp_s* h, PcgState* st) {
  if (h->graph_exec && h->graph_ncols == h->nrhs) return true;
  cudaGraph_t graph;
  IETI_CUDA(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle handle;
  IETI_CUDA(cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  IETI_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  h->cond_handle = (unsigned long long)handle;
  long long before = h->launches;
  IETI_CUDA(cudaStreamBeginCaptureToGraph(h->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  iteration_body(h, st, 1);
  cudaGraph_t captured;
  IETI_CUDA(cudaStreamEndCapture(h->stream, &captured));
  h->launches = before;  // captured, not launched
  cudaGraphExec_t exec;
  IETI_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  h->graph = graph;
  h->graph_exec = exec;
  h->graph_ncols = h->nrhs;
  return true;
}

void destroy_graph(ietidp_s* h) {
  if (h->graph_exec) cudaGraphExecDestroy((cudaGraphExec_t)h->graph_exec);
  if (h->graph) cudaGraphDestroy((cudaGraph_t)h->graph);
  h->graph_exec = h->graph = nullptr;
}

void run_solve(ietidp_s* h) {
  const int nc = h->nrhs, m = h->n_lambda;
  PcgState* st = reinterpret_cast<PcgState*>(h->state.p);
  double* rr_part = h->partial.p + NBLK * nc;
  double* rz_part = h->partial.p + 2 * NBLK * nc;
  cudaStream_t s = h->stream;
  IETI_CUDA(cudaMemsetAsync(h->partial.p, 0, h->partial.n * sizeof(double), s));
  if (m > 0) {
    k_init<<<NBLK, VT, 0, s>>>(m, nc, h->d_vec.p, h->lam_vec.p, h->r_vec.p, rr_part);
    IETI_LAUNCHED(h);
  }
  k_init_ctl<<<1, 64, 0, s>>>(st, rr_part, nc, m, h->opt.tol, h->opt.max_iter, h->opt.fixed_iters);
  IETI_LAUNCHED(h);
  if (m > 0) {
    apply_M_inter(h, nc, h->r_vec.p, h->z_vec.p, st, rr_part, 0, h->r_vec.p, rz_part);
    k_init_p<<<NBLK, VT, 0, s>>>(m, st, h->z_vec.p, h->p_vec.p);
    IETI_LAUNCHED(h);
    k_init_rz<<<1, 64, 0, s>>>(st, rz_part);
    IETI_LAUNCHED(h);
    build_graph(h, st);
    IETI_CUDA(cudaGraphLaunch((cudaGraphExec_t)h->graph_exec, s));
  }
  IETI_CHECK_LAUNCH();
}

// After run_solve: read the state; count graph-launched kernels; true residual.
void finish_solve(ietidp_s* h, ietidp_report* rep) {
  const int nc = h->nrhs, m = h->n_lambda;
  PcgState hs;
  IETI_CUDA(cudaMemcpyAsync(&hs, h->state.p, sizeof(PcgState), cudaMemcpyDeviceToHost, h->stream));
  IETI_CUDA(cudaStreamSynchronize(h->stream));
  if (m > 0) h->launches += (long long)body_launches(h, nc) * std::max(hs.it, 1);
  for (int c = 0; c < nc; ++c) {
    rep->iters[c] = hs.iters[c];
    rep->converged[c] = h->opt.fixed_iters ? 1 : !hs.active[c];
  }
  // true residual ||d - F lambda|| / ||d||
  if (m > 0) {
    double* part = h->partial.p + 3 * NBLK * nc;
    apply_F_inter(h, nc, h->lam_vec.p, h->tmp_out.p, nullptr, nullptr, nullptr);
    k_resid<<<NBLK, VT, 0, h->stream>>>(m, nc, h->d_vec.p, h->tmp_out.p, part);
    IETI_LAUNCHED(h);
    std::vector<double> hp((size_t)NBLK * nc);
    IETI_CUDA(cudaMemcpyAsync(hp.data(), part, hp.size() * 8, cudaMemcpyDeviceToHost, h->stream));
    IETI_CUDA(cudaStreamSynchronize(h->stream));
    for (int c = 0; c < nc; ++c) {
      double s = 0.0;
      for (int b = 0; b < NBLK; ++b) s += hp[(size_t)b * nc + c];
      rep->rel_residual[c] = hs.r0[c] > 0 ? std::sqrt(s) / hs.r0[c] : 0.0;
    }
  } else {
    for (int c = 0; c < nc; ++c) rep->rel_residual[c] = 0.0;
  }
}

void transpose_in(ietidp_s* h, int rows, int ncols, const double* colmajor, double* inter) {
  k_transpose<<<grid_for((long long)rows * ncols, 256), 256, 0, h->stream>>>(rows, ncols, colmajor, inter, 1);
  IETI_LAUNCHED(h);
}
void transpose_out(ietidp_s* h, int rows, int ncols, const double* inter, double* colmajor) {
  k_transpose<<<grid_for((long long)rows * ncols, 256), 256, 0, h->stream>>>(rows, ncols, inter, colmajor, 0);
  IETI_LAUNCHED(h);
}

}  // namespace ieti
