// The PCG loop on F_DP lambda = d_DP.
//
// With the P (primal) DOFs ordered after r_I, the local
// and coarse parts of F_DP only need the trailing blocks L_II and L_PI:
//   G_k^T b = L_PI L_II^-1 b,   G_k z = L_II^-T L_PI^T z        (F2')
// so   F_DP p = sum_k B_I L_II^-T ( L_II^-1 b_k + L_PI^T C_k z ),
//      z = S_PP^-1 sum_k C_k^T L_PI L_II^-1 b_k,   b_k = B_I^(k)T p.
// Per iteration (one CUDA-graph while-loop, no host sync):
//   k_tmv<FWD>   y_k = L_II^-1 b_k (tiles of the stored inverse), g partials
//   k_coarse     z = S_PP^-1 g                                  (one CTA)
//   k_tmv<BWD>   x_k = L_II^-T (y_k + L_PI^T z_k)
//   k_bgather    q = sum_k B x_k, partial p.q
//   k_cg_alpha   alpha; lambda += alpha p; r -= alpha q; partial r.r
//   k_tmv<PRE1>  s_k = L_II^T B_D^(k)T r
//   k_tmv<PRE2>  z_k = L_II s_k
//   k_bgather    z = sum_k B_D z_k, partial r.z
//   k_cg_beta    beta; p = z + beta p
//   k_ctl        iteration counts, stop test, graph condition
// Each k_tmv CTA owns one subdomain's block pair (i, nt-1-i) of output rows
// (FWD, PRE2: block rows of a lower triangle) or columns (BWD, PRE1), streams
// its tiles through a cp.async ring and writes finished blocks: no reductions
// across CTAs. Vectors are interleaved v[j * ncols + c]; dot products are
// fixed-order two-stage reductions (bit-reproducible run to run).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <string>

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

enum TmvMode { FWD = 0, BWD = 1, PRE1 = 2, PRE2 = 3 };

// (the tile is stored swizzled in global memory: a linear copy)
__device__ __forceinline__ void load_tile_async(double* dst, const double* src, int tid) {
#pragma unroll 4
  for (int q = tid; q < TB * TB / 2; q += 256) cp_async16(dst + 2 * q, src + 2 * q);
}
// the same with an L2 eviction-priority hint (createpolicy: 1 = evict_last, 2 = evict_first)
__device__ __forceinline__ void load_tile_async_hint(double* dst, const double* src, int tid, int hint) {
  if (hint == 0) {
    load_tile_async(dst, src, tid);
    return;
  }
  unsigned long long pol;
  if (hint == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll 4
  for (int q = tid; q < TB * TB / 2; q += 256) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + 2 * q);
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src + 2 * q),
                 "l"(pol));
  }
}

struct TmvArgs {
  const LoopWork* work;
  const SubDev* sub;
  const double* tiles;     // L_II tiles (PRE1/PRE2) or L_II^-1 tiles (FWD/BWD)
  const double* lpi;       // L_PI (nP x nI row-major)
  const int* slot_lam;
  const float* slot_sign;
  const int* prim_gid;
  const double* weight;    // PRE1: scaling weights per slot (nullable)
  const double* vin;       // FWD/PRE1: lambda-space vector; BWD: y (slots); PRE2: s (slots)
  const double* z;         // BWD: coarse solution (n_primal x ncols) or null
  double zsign;
  double* vout;            // slot vector
  double* gpart;           // FWD/SYM: coarse partials [cta][nPmax][ncols] (nullable)
  const double* gmat;      // SYM: G_k (n_I x n_P row-major) for the coarse partials
  double* spart;           // SYM: partial blocks of the transposed tile products
  const long long* pboff;  // SYM: first partial block of each (subdomain, block) (SlotRed)
  const SymWork* swork;    // SYM: work items (row segments)
  int maxseg;              // SYM: segments per block row (npart layout)
  int l2hint;              // SYM: L2 eviction priority of the tile stream (0 none, 1 last, 2 first)
  int slot_in;             // FWD/PRE1/SYM: vin is already in slot order (B^T, weights applied)
  int nPmax, ncols, c_off;
  int nt_max;              // SYM (chunk pass): largest number of TB-blocks of a subdomain (x staging)
  int n_sub;               // number of subdomains (chunk-mode coarse phase)
  const SymChunk* chunks;  // SYM (chunk pass): the chunks of the several-RHS pass
  const long long* cpb;    // SYM (chunk pass): first partial block of each (subdomain, block)
  const int* cfirst;       // SYM (chunk pass): rank of the first chunk writing (subdomain, block)
  const PcgState* st;
  const double* rr_part;   // PRE1 inside the loop: convergence test
  int check;
  unsigned long long* tl;  // diagnostics (IETIDP_DBG_TL): CTA 0's timeline of one pass
  int dbg;                 // experiments only (IETIDP_DBG_PASS): bits: 1 every tile read is tile 0, 2 no DMMA, 4 no TMEM in T, 8 no x staging, 16 no write-out
};

// Asynchronous gather of rows [lo, hi) of a slot-ordered vector (row-major,
// A.ncols columns) into vec (stride VS, columns [0, ncl) of the chunk c_off):
// cp.async of every element (8 bytes, 16 where aligned), zero padding written
// directly. The caller commits it with the first tile prefetches.
template <int VS>
__device__ __forceinline__ void gather_async(double* vec, int lo, int hi, const SubDev& d, const TmvArgs& A, int ncl) {
  const int tid = threadIdx.x;
  const int nrow = hi - lo;
  const bool pair16 = (ncl % 2 == 0) && (A.ncols % 2 == 0) && (A.c_off % 2 == 0) && (VS % 2 == 0);
  if (pair16) {
    const int hp = VS / 2;  // 16-byte pairs per row
    for (int e = tid; e < nrow * hp; e += 256) {
      const int a = lo + e / hp, cp = (e % hp) * 2;
      double* dst = vec + (a - lo) * VS + cp;
      if (a < d.nI && cp < ncl)
        cp_async16(dst, A.vin + (d.rI_off + a) * (long long)A.ncols + A.c_off + cp);
      else {
        dst[0] = 0.0;
        dst[1] = 0.0;
      }
    }
  } else {
    for (int e = tid; e < nrow * VS; e += 256) {
      const int a = lo + e / VS, c = e % VS;
      double* dst = vec + (a - lo) * VS + c;
      if (a < d.nI && c < ncl) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa),
                     "l"(A.vin + (d.rI_off + a) * (long long)A.ncols + A.c_off + c));
      } else {
        *dst = 0.0;
      }
    }
  }
}

// Gather the input rows [lo, hi) of one subdomain into shared memory
// (vec[(a - lo) * VS + c]): from the lambda-space vector through B^T (sign, optional
// weight) when LAMBDA, else from a slot vector (plus, for BWD, zsign * L_PI^T z_k
// with z_k staged in zs). VS == 1: thread per row; VS > 1: warp per row, lanes over
// columns, slot metadata loaded once per row, four rows in flight per warp.
template <int VS, bool LAMBDA, bool BWDZ>
__device__ __forceinline__ void gather_rows(double* vec, int lo, int hi, const SubDev& d, const TmvArgs& A, int ncl,
                                            const double* zs, int NCPz) {
  const int tid = threadIdx.x;
  if (VS == 1) {
    for (int a = lo + tid; a < hi; a += 256) {
      double v = 0.0;
      if (a < d.nI && ncl > 0) {
        const long long slot = d.rI_off + a;
        if (LAMBDA) {
          const double w = A.weight ? A.weight[slot] : 1.0;
          v = (double)A.slot_sign[slot] * w * A.vin[(long long)A.slot_lam[slot] * A.ncols + A.c_off];
        } else {
          v = A.vin[slot * A.ncols + A.c_off];
          if (BWDZ) {
            const double* lp = A.lpi + d.lpi_off + a;
            double s2 = 0.0;
#pragma unroll 4
            for (int q = 0; q < d.nP; ++q) s2 += lp[(long long)q * d.nI] * zs[q * NCPz];
            v += A.zsign * s2;
          }
        }
      }
      vec[a - lo] = v;
    }
    return;
  }
  const int warp = tid >> 5, lane = tid & 31;
  for (int a0 = lo + warp * 4; a0 < hi; a0 += 32) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int a = a0 + u;
      v[u] = 0.0;
      if (a < hi && a < d.nI && lane < ncl) {
        const long long slot = d.rI_off + a;
        if (LAMBDA) {
          const double w = A.weight ? A.weight[slot] : 1.0;
          v[u] = (double)A.slot_sign[slot] * w * A.vin[(long long)A.slot_lam[slot] * A.ncols + A.c_off + lane];
        } else {
          v[u] = A.vin[slot * A.ncols + A.c_off + lane];
          if (BWDZ) {
            const double* lp = A.lpi + d.lpi_off + a;
            double s2 = 0.0;
#pragma unroll 4
            for (int q = 0; q < d.nP; ++q) s2 += lp[(long long)q * d.nI] * zs[q * NCPz + lane];
            v[u] += A.zsign * s2;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (a0 + u < hi && lane < VS) vec[(a0 + u - lo) * VS + lane] = v[u];
  }
}

// One work item (subdomain block pair) of a tile-streamed operator.
template <int MODE, int NCP, int STAGES>
__device__ __forceinline__ void tmv_item(const TmvArgs& A, int item, double* smem) {
  constexpr bool TRANS = (MODE == BWD || MODE == PRE1);
  constexpr int VS = (NCP == 1) ? 1 : NCP + 4;
  constexpr int NB = (NCP == 1) ? 1 : NCP / 8;
  __shared__ double red[8][TB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncl = min(NCP, A.ncols - A.c_off);
  __syncthreads();  // shared memory of the previous item is free
  const LoopWork lw = A.work[item];
  const SubDev d = A.sub[lw.sub];
  const int nt = d.nt;
  const int ob[2] = {lw.blk0, lw.blk1};
  const int nob = lw.nblk;
  // input rows needed: N-op (FWD, PRE2) blocks [0, max ob], T-op (BWD, PRE1) blocks [min ob, nt)
  const int bmin = min(ob[0], ob[nob - 1]), bmax = max(ob[0], ob[nob - 1]);
  const int lo = TRANS ? bmin * TB : 0;
  const int hi = TRANS ? nt * TB : (bmax + 1) * TB;
  double* ring = smem;
  double* vec = smem + STAGES * TILE_ELEMS;  // rows [lo, hi)
  double* outb = vec + (hi - lo) * VS;       // one finished output block (FWD partials)

  // ---- input vector ----
  double* zs = outb + TB * VS;  // BWD: z_k (nP x NCP)
  if (MODE == BWD && A.z) {
    for (int e = tid; e < d.nP * NCP; e += 256) {
      const int q = e / NCP, c = e % NCP;
      zs[e] = c < ncl ? A.z[(long long)A.prim_gid[d.prim_off + q] * A.ncols + A.c_off + c] : 0.0;
    }
    __syncthreads();
  }
  if ((MODE == FWD || MODE == PRE1) && !A.slot_in) gather_rows<VS, true, false>(vec, lo, hi, d, A, ncl, zs, NCP);
  else if (MODE == BWD && A.z) gather_rows<VS, false, true>(vec, lo, hi, d, A, ncl, zs, NCP);
  else gather_async<VS>(vec, lo, hi, d, A, ncl);  // committed with the first tile
  // ---- tile schedule: per output block o, N: (o, 0..o), T: (o..nt-1, o) ----
  auto ntiles_of = [&](int o) { return TRANS ? nt - o : o + 1; };
  const int n0 = ntiles_of(ob[0]);
  const int nsteps = n0 + (nob == 2 ? ntiles_of(ob[1]) : 0);
  auto tile_ptr = [&](int s) {
    const int which = s < n0 ? 0 : 1;
    const int o = ob[which], k = which ? s - n0 : s;
    const int i = TRANS ? o + k : o, j = TRANS ? o : k;
    return A.tiles + d.tile_off + (long long)(i * (i + 1) / 2 + j) * TILE_ELEMS;
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nsteps) load_tile_async(ring + s * TILE_ELEMS, tile_ptr(s), tid);
    cp_async_commit();
  }
  double gacc[2] = {0.0, 0.0};  // FWD coarse partials of (q, c) = ((tid + 256 u) / NCP, (tid + 256 u) % NCP)
  double accN[8], accT[2], acc[NB][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) accN[i] = 0.0;
  accT[0] = accT[1] = 0.0;
#pragma unroll
  for (int i = 0; i < NB; ++i) acc[i][0] = acc[i][1] = 0.0;
  const int g = lane >> 2, t4 = lane & 3;

  for (int s = 0; s < nsteps; ++s) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int sn = s + STAGES - 1;
      if (sn < nsteps) load_tile_async(ring + (sn % STAGES) * TILE_ELEMS, tile_ptr(sn), tid);
      cp_async_commit();
    }
    const double* Tt = ring + (s % STAGES) * TILE_ELEMS;
    const int which = s < n0 ? 0 : 1;
    const int o = ob[which], k = which ? s - n0 : s;
    const int inblk = TRANS ? o + k : k;  // input vector block
    const double* vb = vec + (inblk * TB - lo) * VS;
    const bool last = (k == ntiles_of(o) - 1);
    if constexpr (NCP == 1) {
      if (!TRANS) {
        const double x0 = vb[lane], x1 = vb[lane + 32];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int r = warp * 8 + rr;
          accN[rr] += Tt[swz(r, lane)] * x0 + Tt[swz(r, lane + 32)] * x1;
        }
      } else {
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int r = warp * 8 + rr;
          const double xr = vb[r];
          accT[0] += Tt[swz(r, lane)] * xr;
          accT[1] += Tt[swz(r, lane + 32)] * xr;
        }
      }
      if (last) {
        // finished output block o -> outb (64 values)
        if (!TRANS) {
          double full[8];
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) full[rr] = warp_sum(accN[rr]);
          if (lane < 8) {
            double v = full[0];
#pragma unroll
            for (int rr = 1; rr < 8; ++rr)
              if (lane == rr) v = full[rr];
            outb[warp * 8 + lane] = v;
          }
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) accN[rr] = 0.0;
          __syncthreads();
        } else {
          red[warp][lane] = accT[0];
          red[warp][lane + 32] = accT[1];
          __syncthreads();
          if (tid < TB) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) v += red[w][tid];
            outb[tid] = v;
          }
          accT[0] = accT[1] = 0.0;
          __syncthreads();
        }
      }
    } else {
#pragma unroll 4
      for (int k0 = 0; k0 < TB; k0 += 4) {
        const double a = TRANS ? Tt[swz(k0 + t4, warp * 8 + g)] : Tt[swz(warp * 8 + g, k0 + t4)];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) dmma8x8x4(acc[nb][0], acc[nb][1], a, vb[(k0 + t4) * VS + nb * 8 + g]);
      }
      if (last) {
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          outb[(warp * 8 + g) * VS + nb * 8 + 2 * t4] = acc[nb][0];
          outb[(warp * 8 + g) * VS + nb * 8 + 2 * t4 + 1] = acc[nb][1];
          acc[nb][0] = acc[nb][1] = 0.0;
        }
        __syncthreads();
      }
    }
    if (last) {
      // write the finished block; FWD also accumulates the coarse partial L_PI y
      for (int e = tid; e < TB * ncl; e += 256) {
        const int r = e / ncl, c = e % ncl;
        const int a = o * TB + r;
        if (a < d.nI) A.vout[(d.rI_off + a) * A.ncols + A.c_off + c] = outb[r * VS + c];
      }
      if (MODE == FWD && A.gpart && d.nP > 0) {
        double* gs = outb + TB * VS;  // nP x TB (L_PI columns of this block)
        const int na = min(TB, d.nI - o * TB);
        for (int e = tid; e < d.nP * TB; e += 256) {
          const int q = e / TB, r = e % TB;
          gs[e] = r < na ? A.lpi[d.lpi_off + (long long)q * d.nI + o * TB + r] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int e = tid + 256 * u;
          if (e < d.nP * NCP) {
            const int q = e / NCP, c = e % NCP;
            for (int r = 0; r < na; ++r) gacc[u] += gs[q * TB + r] * outb[r * VS + c];
          }
        }
      }
      __syncthreads();
    }
  }
  cp_async_wait<0>();
  if (MODE == FWD && A.gpart)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = tid + 256 * u;
      if (e >= d.nP * NCP) break;
      const int q = e / NCP, c = e % NCP;
      if (c < ncl) A.gpart[((long long)item * A.nPmax + q) * A.ncols + A.c_off + c] = gacc[u];
    }
}

// One work item of a symmetric matrix held as lower TB-tiles (diagonal tiles full):
// y = S x in ONE pass. For each own block row o, tile (o, j) contributes S_oj x_j to
// y_o (kept in registers) and, for j < o, S_oj^T x_o to y_j (written as partial
// block (o, j), summed later in a fixed order by sym_reduce). The input x is
// gathered from the lambda-space vector (sign, optional weight); the F-apply also
// accumulates the coarse partial G_k^T x of its own rows.
template <int NCP, int STAGES>
__device__ __forceinline__ void sym_item(const TmvArgs& A, int item, double* smem) {
  // One row segment (o, j0..j1) of the symmetric lower tile matrix:
  //   N: npart[o][seg] = sum_j S_oj x_j        (the row product, partial over the segment)
  //   T: spart(o, j)   = S_oj^T x_o, j < o     (the transposed products, per tile)
  // plus, for the first segment of a row, the coarse partial G_k[rows o]^T x_o.
  constexpr int VS = (NCP == 1) ? 1 : NCP + 4;
  constexpr int NB = (NCP == 1) ? 1 : NCP / 8;
  __shared__ double red[2][8][TB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncl = min(NCP, A.ncols - A.c_off);
  __syncthreads();
  const SymWork sw = A.swork[item];
  const SubDev d = A.sub[sw.sub];
  const int o = sw.o, j0 = sw.j0, j1 = sw.j1, nsteps = j1 - j0 + 1;
  const bool xo_sep = j1 < o;
  double* ring = smem;
  double* vec = smem + STAGES * TILE_ELEMS;  // blocks j0..j1, then block o if separate
  double* xo = xo_sep ? vec + nsteps * TB * VS : vec + (o - j0) * TB * VS;
  if (A.slot_in) {
    gather_async<VS>(vec, j0 * TB, (j1 + 1) * TB, d, A, ncl);  // committed with the first tile
    if (xo_sep) gather_async<VS>(xo, o * TB, (o + 1) * TB, d, A, ncl);
  } else {
    gather_rows<VS, true, false>(vec, j0 * TB, (j1 + 1) * TB, d, A, ncl, nullptr, NCP);
    if (xo_sep) gather_rows<VS, true, false>(xo, o * TB, (o + 1) * TB, d, A, ncl, nullptr, NCP);
  }
  auto tile_ptr = [&](int st) {
    return A.tiles + d.tile_off + (long long)(o * (o + 1) / 2 + j0 + st) * TILE_ELEMS;
  };
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nsteps) load_tile_async(ring + st * TILE_ELEMS, tile_ptr(st), tid);
    cp_async_commit();
  }
  cp_async_wait<STAGES - 2>();  // group 0: the gathered input and tile 0
  __syncthreads();              // vec complete
  // coarse partial of block row o (first segment only): G_k[rows o]^T x_o
  double gacc[2] = {0.0, 0.0};
  if (A.gpart && d.nP > 0 && sw.seg == 0) {
    double* gs = xo + TB * VS;  // TB x nP
    const int na = min(TB, d.nI - o * TB);
    const double* Gb = A.gmat + d.g_off + (long long)o * TB * d.nP;
    for (int e = tid; e < na * d.nP; e += 256) gs[e] = Gb[e];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = tid + 256 * u;
      if (e < d.nP * NCP) {
        const int q = e / NCP, c = e % NCP;
        for (int r = 0; r < na; ++r) gacc[u] += gs[r * d.nP + q] * xo[r * VS + c];
      }
    }
    __syncthreads();
  }
  double accN[8], acc[NB][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) accN[i] = 0.0;
#pragma unroll
  for (int i = 0; i < NB; ++i) acc[i][0] = acc[i][1] = 0.0;
  const int g = lane >> 2, t4 = lane & 3;
  double* pend = nullptr;  // NCP == 1: T partial of the previous tile still in red[]
  for (int st = 0; st < nsteps; ++st) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if constexpr (NCP == 1) {
      if (pend && tid < TB) {
        double v = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < 8; ++w2) v += red[(st - 1) & 1][w2][tid];
        pend[(long long)tid * A.ncols] = v;
      }
      pend = nullptr;
    }
    {
      const int sn = st + STAGES - 1;
      if (sn < nsteps) load_tile_async(ring + (sn % STAGES) * TILE_ELEMS, tile_ptr(sn), tid);
      cp_async_commit();
    }
    const double* Tt = ring + (st % STAGES) * TILE_ELEMS;
    const int j = j0 + st;
    const bool diag = (j == o);
    const double* xj = vec + st * TB * VS;
    double* pblk = A.spart + ((A.pboff[d.blk0 + j] + j / SYM_SEG + o - j) * TB) * A.ncols + A.c_off;
    if constexpr (NCP == 1) {
      {  // N: y_o += S_oj x_j
        const double x0 = xj[lane], x1 = xj[lane + 32];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int r = warp * 8 + rr;
          accN[rr] += Tt[swz(r, lane)] * x0 + Tt[swz(r, lane + 32)] * x1;
        }
      }
      if (!diag) {  // T: partial (o, j) = S_oj^T x_o, reduced over the warps at the next step
        double p0 = 0.0, p1 = 0.0;
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int r = warp * 8 + rr;
          const double xr = xo[r];
          p0 += Tt[swz(r, lane)] * xr;
          p1 += Tt[swz(r, lane + 32)] * xr;
        }
        red[st & 1][warp][lane] = p0;
        red[st & 1][warp][lane + 32] = p1;
        pend = pblk;
      }
    } else {
#pragma unroll 4
      for (int k0 = 0; k0 < TB; k0 += 4) {
        const double a = Tt[swz(warp * 8 + g, k0 + t4)];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) dmma8x8x4(acc[nb][0], acc[nb][1], a, xj[(k0 + t4) * VS + nb * 8 + g]);
      }
      if (!diag) {
        double pt[NB][2];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) pt[nb][0] = pt[nb][1] = 0.0;
#pragma unroll 4
        for (int k0 = 0; k0 < TB; k0 += 4) {
          const double a = Tt[swz(k0 + t4, warp * 8 + g)];
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) dmma8x8x4(pt[nb][0], pt[nb][1], a, xo[(k0 + t4) * VS + nb * 8 + g]);
        }
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int c = nb * 8 + 2 * t4 + q;
            if (c < ncl) pblk[(long long)(warp * 8 + g) * A.ncols + c] = pt[nb][q];
          }
      }
    }
  }
  double* nb_out = A.spart + ((A.pboff[d.blk0 + o] + sw.seg) * TB) * A.ncols + A.c_off;
  if constexpr (NCP == 1) {
    __syncthreads();
    if (pend && tid < TB) {
      double v = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < 8; ++w2) v += red[(nsteps - 1) & 1][w2][tid];
      pend[(long long)tid * A.ncols] = v;
    }
    double full[8];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) full[rr] = warp_sum(accN[rr]);
    if (lane < 8) {
      double v = full[0];
#pragma unroll
      for (int rr = 1; rr < 8; ++rr)
        if (lane == rr) v = full[rr];
      nb_out[(long long)(warp * 8 + lane) * A.ncols] = v;
    }
  } else {
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = nb * 8 + 2 * t4 + q;
        if (c < ncl) nb_out[(long long)(warp * 8 + g) * A.ncols + c] = acc[nb][q];
      }
  }
  cp_async_wait<0>();
  if (A.gpart && sw.seg == 0)
    for (int u = 0; u < 2; ++u) {
      const int e = tid + 256 * u;
      if (e >= d.nP * NCP) break;
      const int q = e / NCP, c = e % NCP;
      if (c < ncl) A.gpart[((long long)(d.blk0 + o) * A.nPmax + q) * A.ncols + A.c_off + c] = gacc[u];
    }
}

// The symmetric pass over a CTA's list of row-segment items as ONE tile stream: the
// cp.async ring runs across item boundaries (the next item's input rows are gathered
// into the other of NVB vector buffers together with its first tile), so there is no
// pipeline refill per item. Same arithmetic and outputs as sym_item (slot_in only).
template <int NCP, int STAGES>
__device__ __forceinline__ void sym_stream(const TmvArgs& A, const int* items, int nitems, double* smem) {
  constexpr int VS = (NCP == 1) ? 1 : NCP + 4;
  constexpr int NB = (NCP == 1) ? 1 : NCP / 8;
  // vector buffers: at most STAGES items are in flight (the consumed one and up to
  // STAGES - 1 issued ahead, each with at least one tile), so STAGES buffers suffice
  constexpr int NVB = STAGES;
  constexpr int VROWS = (SYM_SEG + 1) * TB;
  __shared__ double red[2][8][TB];
  __shared__ SymWork s_sw[NVB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncl = min(NCP, A.ncols - A.c_off);
  if (nitems == 0) return;
  double* ring = smem;
  double* vbase = smem + STAGES * TILE_ELEMS;
  double* gs = vbase + NVB * VROWS * VS;  // TB x nP coarse rows
  __syncthreads();
  // issue cursor: (item ii, step is) of the next tile to prefetch
  int ii = 0, is = 0;
  auto nsteps_of = [&](const SymWork& w) { return w.j1 - w.j0 + 1; };
  SymWork wi = A.swork[items[0]];
  auto issue = [&](int gslot) {  // prefetch the next tile (and, at an item's first tile, its input rows)
    if (ii < nitems) {
      const SubDev d = A.sub[wi.sub];
      if (is == 0) {
        double* vec = vbase + (ii % NVB) * VROWS * VS;
        const int nst = nsteps_of(wi);
        gather_async<VS>(vec, wi.j0 * TB, (wi.j1 + 1) * TB, d, A, ncl);
        if (wi.j1 < wi.o) gather_async<VS>(vec + nst * TB * VS, wi.o * TB, (wi.o + 1) * TB, d, A, ncl);
        if (tid == 0) s_sw[ii % NVB] = wi;
      }
      load_tile_async_hint(ring + gslot * TILE_ELEMS,
                           A.tiles + d.tile_off + (long long)(wi.o * (wi.o + 1) / 2 + wi.j0 + is) * TILE_ELEMS, tid,
                           A.l2hint);
      if (++is == nsteps_of(wi)) {
        is = 0;
        if (++ii < nitems) wi = A.swork[items[ii]];
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) issue(st);
  double accN[8], acc[NB][2];
  double gacc[2] = {0.0, 0.0};
  const int g = lane >> 2, t4 = lane & 3;
  double* pend = nullptr;
  int pend_buf = 0;
  int gt = 0;  // global tile counter of the CTA
  for (int k = 0; k < nitems; ++k) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();  // item k's input rows and first tile are in; s_sw[k] visible
    const SymWork sw = s_sw[k % NVB];
    const SubDev d = A.sub[sw.sub];
    const int o = sw.o, j0 = sw.j0, nst = nsteps_of(sw);
    double* vec = vbase + (k % NVB) * VROWS * VS;
    double* xo = (sw.j1 < o) ? vec + nst * TB * VS : vec + (o - j0) * TB * VS;
    gacc[0] = gacc[1] = 0.0;
    if (A.gpart && d.nP > 0 && sw.seg == 0) {  // coarse partial of block row o
      const int na = min(TB, d.nI - o * TB);
      const double* Gb = A.gmat + d.g_off + (long long)o * TB * d.nP;
      for (int e = tid; e < na * d.nP; e += 256) gs[e] = Gb[e];
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = tid + 256 * u;
        if (e < d.nP * NCP) {
          const int q = e / NCP, c = e % NCP;
          for (int r = 0; r < na; ++r) gacc[u] += gs[r * d.nP + q] * xo[r * VS + c];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) accN[i] = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int st = 0; st < nst; ++st, ++gt) {
      if (st > 0) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
      }
      if constexpr (NCP == 1) {
        if (pend && tid < TB) {
          double v = 0.0;
#pragma unroll
          for (int w2 = 0; w2 < 8; ++w2) v += red[pend_buf][w2][tid];
          pend[(long long)tid * A.ncols] = v;
        }
        pend = nullptr;
      }
      const int j = j0 + st;
      const long long pbj = __ldg(A.pboff + d.blk0 + j);  // before the issue: latency hidden
      issue((gt + STAGES - 1) % STAGES);
      const double* Tt = ring + (gt % STAGES) * TILE_ELEMS;
      const bool diag = (j == o);
      const double* xj = vec + st * TB * VS;
      double* pblk = A.spart + ((pbj + j / SYM_SEG + o - j) * TB) * A.ncols + A.c_off;
      if constexpr (NCP == 1) {
        {
          const double x0 = xj[lane], x1 = xj[lane + 32];
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) {
            const int r = warp * 8 + rr;
            accN[rr] += Tt[swz(r, lane)] * x0 + Tt[swz(r, lane + 32)] * x1;
          }
        }
        if (!diag) {
          double p0 = 0.0, p1 = 0.0;
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) {
            const int r = warp * 8 + rr;
            const double xr = xo[r];
            p0 += Tt[swz(r, lane)] * xr;
            p1 += Tt[swz(r, lane + 32)] * xr;
          }
          red[gt & 1][warp][lane] = p0;
          red[gt & 1][warp][lane + 32] = p1;
          pend = pblk;
          pend_buf = gt & 1;
        }
      } else {
#pragma unroll 4
        for (int k0 = 0; k0 < TB; k0 += 4) {
          const double a = Tt[swz(warp * 8 + g, k0 + t4)];
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) dmma8x8x4(acc[nb][0], acc[nb][1], a, xj[(k0 + t4) * VS + nb * 8 + g]);
        }
        if (!diag) {
          double pt[NB][2];
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) pt[nb][0] = pt[nb][1] = 0.0;
#pragma unroll 4
          for (int k0 = 0; k0 < TB; k0 += 4) {
            const double a = Tt[swz(k0 + t4, warp * 8 + g)];
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) dmma8x8x4(pt[nb][0], pt[nb][1], a, xo[(k0 + t4) * VS + nb * 8 + g]);
          }
#pragma unroll
          for (int nb = 0; nb < NB; ++nb)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int c = nb * 8 + 2 * t4 + q;
              if (c < ncl) pblk[(long long)(warp * 8 + g) * A.ncols + c] = pt[nb][q];
            }
        }
      }
    }
    // item done: its row-segment partial and coarse partial
    double* nb_out = A.spart + ((A.pboff[d.blk0 + o] + sw.seg) * TB) * A.ncols + A.c_off;
    if constexpr (NCP == 1) {
      double full[8];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) full[rr] = warp_sum(accN[rr]);
      if (lane < 8) {
        double v = full[0];
#pragma unroll
        for (int rr = 1; rr < 8; ++rr)
          if (lane == rr) v = full[rr];
        nb_out[(long long)(warp * 8 + lane) * A.ncols] = v;
      }
    } else {
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int c = nb * 8 + 2 * t4 + q;
          if (c < ncl) nb_out[(long long)(warp * 8 + g) * A.ncols + c] = acc[nb][q];
        }
    }
    if (A.gpart && sw.seg == 0)
      for (int u = 0; u < 2; ++u) {
        const int e = tid + 256 * u;
        if (e >= d.nP * NCP) break;
        const int q = e / NCP, c = e % NCP;
        if (c < ncl) A.gpart[((long long)(d.blk0 + o) * A.nPmax + q) * A.ncols + A.c_off + c] = gacc[u];
      }
  }
  if constexpr (NCP == 1) {
    __syncthreads();
    if (pend && tid < TB) {
      double v = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < 8; ++w2) v += red[pend_buf][w2][tid];
      pend[(long long)tid * A.ncols] = v;
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// ---------------------------------------------------------------------------
// The several-RHS symmetric pass (16 columns): chunks of whole tile ranges, the
// transposed products accumulated on chip in tensor memory.
//
// y = S x for a symmetric matrix held as lower TB-tiles (diagonal tiles full). The
// CTA's chunks are contiguous tile ranges of one subdomain in lower row-major order,
// so the CTA's tile stream is ONE contiguous range of the tile array: a thread issues
// one 32 KB cp.async.bulk per tile into a STAGES-deep ring (mbarrier completion, L2
// evict_first). For tile (o, j), with DMMA m8n8k4 on 16 x 16 warp fragments (four
// independent accumulation chains per warp: the DMMA latency is covered):
//   N (warps 0-3): S_oj x_j  -> rows o, warp q = rows 16q .. 16q+15, accumulated in
//      registers over the row;
//   T (warps 4-7): S_oj^T x_o -> rows j (j < o), warp 4+q = rows 16q .. 16q+15,
//      accumulated in TENSOR MEMORY: block j's fragment (8 doubles per thread) is
//      loaded (tcgen05.ld), extended by the DMMA chain and stored back (tcgen05.st),
//      so the chunk's transposed products never leave the SM.
// At the diagonal tile the N warps finish the row's chain (it becomes block o's
// accumulator) while the T warps form the coarse partial G_k[rows o]^T x_o of the F-apply.
// The warps are not synchronised per tile: each releases a ring slot when it is done with
// it (the last of the eight issues the slot's next copy), and T warp q waits for N warp q
// (a release/acquire counter of its diagonals) only before its first tile (o', j) of a
// block j whose row lies in the chunk, so it runs on into the next row while the N warps
// finish a diagonal.
// At the end of the chunk every block j <= o_b is written once as the chunk's partial
// block (then zeroed); the gathers sum the (typically 1-3) partial blocks of a slot in
// chunk order (deterministic).
// The chunk's input blocks x_0..x_ob are staged in shared memory (16 columns, 4-double
// groups XOR-swizzled by (r & 3): conflict-free DMMA B fragments, ch_xpos). Tensor
// memory: lanes = the warp's quadrant (32 (w & 3) + lane), columns 16 j + 8 h + [0, 8)
// hold half h (RHS columns 8h .. 8h+7) of block j: up to 32 blocks (n_I <= 2048).
// ---------------------------------------------------------------------------
constexpr int CH_NC = 16;                 // columns per chunk pass
constexpr int CH_XBLK = TB * CH_NC;       // doubles per staged input block
constexpr int CH_TMEM_COLS = 512;

__device__ __forceinline__ int ch_xpos(int r, int c) { return r * CH_NC + (c ^ ((r & 3) << 2)); }

__device__ __forceinline__ void cp_async_z16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tm_ld8(unsigned taddr, double (&v)[2][2]) {
  unsigned r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i >> 1][i & 1] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}
// issue only (the caller waits with tm_wait_ld before reading r)
__device__ __forceinline__ void tm_ld8_issue(unsigned taddr, unsigned (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_st8(unsigned taddr, const double (&v)[2][2]) {
  unsigned r[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double x = v[i >> 1][i & 1];
    r[2 * i] = (unsigned)__double2loint(x);
    r[2 * i + 1] = (unsigned)__double2hiint(x);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// Per-CTA state of the chunk passes (shared memory): the ring's mbarriers, the tensor
// memory base and the running count of tiles streamed (ring slot and phase parity).
struct ChunkCtl {
  uint64_t full[4];
  unsigned rel[4];   // per ring slot: warps done with it, counted over all its uses
  unsigned diag[4];  // per quadrant: diagonal tiles whose row accumulator N warp q has stored
  long long pb[32];  // the chunk's partial block of each block row (write-out)
  unsigned tmem;
  unsigned streamed;
  unsigned ncall, ntl;  // diagnostics: pass calls, timeline entries
};

// Tile (o, j) of chunk tiles: row o of lower row-major index t.
__device__ __forceinline__ int o0_of(int t);
__device__ __forceinline__ int tri_row(int t) {
  int o = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while (o * (o + 1) / 2 > t) --o;
  while ((o + 1) * (o + 2) / 2 <= t) ++o;
  return o;
}

__device__ __forceinline__ int o0_of(int t) { return tri_row(t); }

__device__ __forceinline__ void tl_mark(const TmvArgs& A, ChunkCtl* ctl, bool rec, int ev, int a, int b) {
  if (rec) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned k = ctl->ntl++;
    if (k < 2048) {
      A.tl[2 * k] = t;
      A.tl[2 * k + 1] = ((unsigned long long)ev << 32) | ((unsigned)a << 16) | (unsigned)b;
    }
  }
}
template <int STAGES>
__device__ __forceinline__ void sym_chunks(const TmvArgs& A, const SymChunk* ch, int nch, double* smem, ChunkCtl* ctl) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int ncl = min(CH_NC, A.ncols - A.c_off);
  double* ring = smem;
  double* xb = smem + STAGES * TILE_ELEMS;
  double* gs = xb + A.nt_max * CH_XBLK;  // G_k rows of the current block row (TB x nP), F-apply
  if (nch == 0) return;
  // diagnostics: CTA 0, thread 0 (N warp 0) records its timeline of pass call 100 and 101
  const bool rec = A.tl && blockIdx.x == 0 && tid == 0 && (ctl->ncall == 100 || ctl->ncall == 101);
  tl_mark(A, ctl, rec, 0, ctl->ncall, nch);
  const long long g0 = ch[0].gtile;
  const int ntiles = (int)(ch[nch - 1].gtile + (ch[nch - 1].t1 - ch[nch - 1].t0) - g0);
  const unsigned base = ctl->streamed;
  // tensor memory: lanes = the warp's quadrant q = w & 3 (rows 16q .. 16q+15 of a block),
  // block j at columns 16 j .. 16 j + 15 (columns 0-7 of the RHS, then 8-15; 4 doubles each)
  const int q4 = warp & 3, r0 = 16 * q4 + g;
  const bool tw = warp >= 4;
  const unsigned tq = ctl->tmem + ((unsigned)(32 * q4) << 16);
  // fragment offsets (doubles) with the swizzles resolved once: for k-step k0 (a multiple
  // of 4), A = S rows r0 (+8): swz(r0, k0 + t4) = r0 TB + (k0 & ~15) + acol[(k0 >> 2) & 3];
  // A = S^T: swz(k0 + t4, r0 (+8)) = at0 (at1) + k0 TB; B = x: ch_xpos(k0 + t4, g (+8)) =
  // xb0 (xb1) + k0 CH_NC
  int acol[4];
#pragma unroll
  for (int kl = 0; kl < 4; ++kl) acol[kl] = 4 * (kl ^ (g & 3)) + t4;
  const int at0 = t4 * TB + (r0 ^ (t4 << 2)), at1 = t4 * TB + ((r0 + 8) ^ (t4 << 2));
  const int xb0 = t4 * CH_NC + (g ^ (t4 << 2)), xb1 = t4 * CH_NC + ((g ^ (t4 << 2)) ^ 8);
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int i) {
    const unsigned s = (base + i) % STAGES;
    mbar_expect_tx(&ctl->full[s], TILE_ELEMS * 8);
    bulk_g2s(ring + s * TILE_ELEMS, A.tiles + ((A.dbg & 1) ? (g0 + (i & 1)) * TILE_ELEMS : (g0 + i) * TILE_ELEMS), TILE_ELEMS * 8, &ctl->full[s], pol);
  };
  if (tid == 0)
    for (int i = 0; i < min(STAGES, ntiles); ++i) issue(i);
  int i = 0;  // tile counter of the CTA's stream
  for (int c = 0; c < nch; ++c) {
    const SymChunk C = ch[c];
    const SubDev d = A.sub[C.sub];
    const int ob = tri_row(C.t1 - 1);
    const bool coarse = A.gpart && d.nP > 0;
    auto stage_g = [&](int row, int t0, int nt) {  // G_k rows of block row `row` (threads t0 of nt)
      const int na = min(TB, d.nI - row * TB);
      const double* Gb = A.gmat + d.g_off + (long long)row * TB * d.nP;
      for (int e = t0; e < na * d.nP; e += nt) gs[e] = __ldg(Gb + e);
    };
    if (coarse) stage_g(o0_of(C.t0), tid, 256);
    if (tid <= ob) ctl->pb[tid] = A.cpb[d.blk0 + tid] + (C.rank - A.cfirst[d.blk0 + tid]);  // partial blocks
    // stage x_0 .. x_ob (16-byte pairs; rows beyond n_I and columns beyond ncl are zero)
    {
      const double* src = A.vin + d.rI_off * A.ncols + A.c_off;
      const int nrow = (ob + 1) * TB;
      const bool vec2 = ((A.ncols | A.c_off) & 1) == 0;
      for (int e = tid; e < ((A.dbg & 8) ? 0 : nrow * (CH_NC / 2)); e += 256) {
        const int r = e >> 3, cp = (e & 7) * 2;
        double* dst = xb + (r >> 6) * CH_XBLK + ch_xpos(r & (TB - 1), cp);
        if (r < d.nI && cp + 1 < ncl && vec2) {
          cp_async16(dst, src + (long long)r * A.ncols + cp);
        } else {
          dst[0] = (r < d.nI && cp < ncl) ? src[(long long)r * A.ncols + cp] : 0.0;
          dst[1] = (r < d.nI && cp + 1 < ncl) ? src[(long long)r * A.ncols + cp + 1] : 0.0;
        }
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
    }
    tl_mark(A, ctl, rec, 1, c, ob);
    // N warps (0-3): rows 16q .. 16q+15 of the row's product (all 16 columns, registers,
    // acc[nb][mb], x_j, then x_o at the diagonal tile); T warps (4-7): rows 16q .. 16q+15 of
    // block j's transposed product (tensor memory), and at the diagonal tile the coarse
    // partial. Four independent DMMA chains per warp. The warps are not synchronised per
    // tile: each releases a ring slot when done with it (the last of the eight issues the
    // slot's next copy), and T warp q waits for N warp q at each diagonal (release/acquire
    // counter diag[q]) before it touches the block the N warp has just stored.
    double acc[2][2][2] = {};
    unsigned ndiag = ctl->diag[q4];  // diagonals of this quadrant so far (the warps are in step here)
    const unsigned ndiag0 = ndiag;
    unsigned tr[2][8];
    int preb = -1;  // T warps: block whose accumulator load (tr) is in flight
    int o = tri_row(C.t0), j = C.t0 - o * (o + 1) / 2;
    // T warps: block j >= o0 starts from N warp q's diagonal store (row j of this chunk);
    // blocks below o0 start from zero. synced = the highest block already waited for.
    const int o0 = o;
    int synced = o0 - 1;
    auto wait_block = [&](int jb) {  // N warp q has stored block jb (diagonal jb of the chunk)
      if (jb <= synced) return;
      const unsigned want = ndiag0 + (unsigned)(jb - o0 + 1);
      unsigned have;
      do {
        asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];\n"
                     : "=r"(have)
                     : "r"((unsigned)__cvta_generic_to_shared(&ctl->diag[q4]))
                     : "memory");
      } while ((int)(have - want) < 0);
      __syncwarp();
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      synced = jb;
    };
    for (int t = C.t0; t < C.t1; ++t, ++i) {
      const unsigned s = (base + i) % STAGES;
      mbar_wait(&ctl->full[s], ((base + i) / STAGES) & 1);
      tl_mark(A, ctl, rec, 2, o, j);
      const double* Tt = ring + s * TILE_ELEMS;
      const double* xo = xb + o * CH_XBLK;
      if (!tw) {  // N: S_oj x_j (x_o on the diagonal)
        const double* xj = xb + j * CH_XBLK;
#pragma unroll 8
        for (int k0 = 0; k0 < ((A.dbg & 2) ? 0 : TB); k0 += 4) {
          const double* An = Tt + r0 * TB + (k0 & ~15) + acol[(k0 >> 2) & 3];  // swz(r0, k0 + t4)
          const double a0 = An[0], a1 = An[8 * TB];
          const double b0 = xj[xb0 + k0 * CH_NC], b1 = xj[xb1 + k0 * CH_NC];
          dmma8x8x4(acc[0][0][0], acc[0][0][1], a0, b0);
          dmma8x8x4(acc[0][1][0], acc[0][1][1], a1, b0);
          dmma8x8x4(acc[1][0][0], acc[1][0][1], a0, b1);
          dmma8x8x4(acc[1][1][0], acc[1][1][1], a1, b1);
        }
        if (j == o) {
          // the row's chain is block o's accumulator (zero until now: block o only receives
          // later rows' transposed products)
          tm_st8(tq + 16 * o, acc[0]);
          tm_st8(tq + 16 * o + 8, acc[1]);
          tm_wait_st();
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          __syncwarp();
          if (lane == 0)  // diagonals done by this N warp (release: the block's stores before it)
            asm volatile("st.release.cta.shared::cta.u32 [%0], %1;\n" ::"r"(
                             (unsigned)__cvta_generic_to_shared(&ctl->diag[q4])),
                         "r"(ndiag + 1)
                         : "memory");
          ++ndiag;
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e >> 2][(e >> 1) & 1][e & 1] = 0.0;
        }
      } else if (j < o) {  // T: S_oj^T x_o onto block j's accumulator
        if (preb != j) wait_block(j);
        if (preb != j && !(A.dbg & 4)) {
          tm_ld8_issue(tq + 16 * j, tr[0]);
          tm_ld8_issue(tq + 16 * j + 8, tr[1]);
        }
        if (!(A.dbg & 4)) tm_wait_ld();
        double pt[2][2][2];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
          for (int e = 0; e < 4; ++e)
            pt[h2][e >> 1][e & 1] = __hiloint2double((int)tr[h2][2 * e + 1], (int)tr[h2][2 * e]);
#pragma unroll 8
        for (int k0 = 0; k0 < ((A.dbg & 2) ? 0 : TB); k0 += 4) {
          const double a0 = Tt[at0 + k0 * TB], a1 = Tt[at1 + k0 * TB];  // swz(k0 + t4, r0 (+ 8))
          const double b0 = xo[xb0 + k0 * CH_NC], b1 = xo[xb1 + k0 * CH_NC];
          dmma8x8x4(pt[0][0][0], pt[0][0][1], a0, b0);
          dmma8x8x4(pt[0][1][0], pt[0][1][1], a1, b0);
          dmma8x8x4(pt[1][0][0], pt[1][0][1], a0, b1);
          dmma8x8x4(pt[1][1][0], pt[1][1][1], a1, b1);
        }
        if ((A.dbg & 4)) {
#pragma unroll
          for (int e = 0; e < 8; ++e) tr[e >> 2][(e & 3) * 2] += __double2loint(pt[e >> 2][(e >> 1) & 1][e & 1]);
        } else {
        tm_st8(tq + 16 * j, pt[0]);
        tm_st8(tq + 16 * j + 8, pt[1]);
        }
        preb = -1;
        if (j + 1 < o && j + 1 <= synced && t + 1 < C.t1 && !(A.dbg & 4)) {  // the next tile's block, in flight
          tm_ld8_issue(tq + 16 * (j + 1), tr[0]);
          tm_ld8_issue(tq + 16 * (j + 1) + 8, tr[1]);
          preb = j + 1;
        }
        tm_wait_st();
      } else {  // T warps at the diagonal tile
        if (coarse) {
          // coarse partial of block row o (F-apply): G_k[rows o]^T x_o, G staged in shared
          // memory (two outputs per thread in flight; each sum in row order)
          const int tt = tid - 128, n = d.nP * CH_NC, na = min(TB, d.nI - o * TB);
          double* gp = A.gpart + (long long)(d.blk0 + o) * A.nPmax * A.ncols + A.c_off;
          for (int e0 = tt; e0 < n; e0 += 256) {
            const int e1 = e0 + 128;
            const int q0 = e0 / CH_NC, c0 = e0 % CH_NC, q1 = e1 / CH_NC, c1 = e1 % CH_NC;
            double ga0 = 0.0, ga1 = 0.0;
            if (e1 < n) {
#pragma unroll 4
              for (int r = 0; r < na; ++r) {
                ga0 += gs[r * d.nP + q0] * xo[ch_xpos(r, c0)];
                ga1 += gs[r * d.nP + q1] * xo[ch_xpos(r, c1)];
              }
            } else {
#pragma unroll 4
              for (int r = 0; r < na; ++r) ga0 += gs[r * d.nP + q0] * xo[ch_xpos(r, c0)];
            }
            if (c0 < ncl) gp[q0 * A.ncols + c0] = ga0;
            if (e1 < n && c1 < ncl) gp[q1 * A.ncols + c1] = ga1;
          }
          asm volatile("bar.sync 5, 128;\n" ::: "memory");  // every T warp is done with gs
          if (t + 1 < C.t1) stage_g(o + 1, tt, 128);
          asm volatile("bar.sync 5, 128;\n" ::: "memory");  // G rows of row o + 1 staged
        }
        // no wait here: block o is needed only at tile (o + 1, o), the last of the next
        // row (wait_block), so the T warps run on into row o + 1 while the N warps finish
        // the diagonal
        if (t + 1 < C.t1 && 0 <= synced) {  // the next tile is (o + 1, 0)
          tm_ld8_issue(tq, tr[0]);
          tm_ld8_issue(tq + 8, tr[1]);
          preb = 0;
        }
      }
      // release ring slot s: the last of the eight warps to be done with it issues the
      // slot's next copy (arrivals counted per use: use u of slot s ends at 8u + 8)
      __syncwarp();
      if (lane == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;\n"
                     : "=r"(old)
                     : "r"((unsigned)__cvta_generic_to_shared(&ctl->rel[s]))
                     : "memory");
        if (old == 8u * ((base + i) / STAGES) + 7u && i + STAGES < ntiles) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          issue(i + STAGES);
        }
      }
      if (++j > o) {
        ++o;
        j = 0;
      }
    }
    // a chunk that ends inside a row: the row's N partial joins block o's accumulator
    if (j != 0 && !tw) {
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        double v[2][2];
        tm_ld8(tq + 16 * o + 8 * h2, v);
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e >> 1][e & 1] += acc[h2][e >> 1][e & 1];
        tm_st8(tq + 16 * o + 8 * h2, v);
      }
      tm_wait_st();
    }
    tl_mark(A, ctl, rec, 3, o, j);
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    tl_mark(A, ctl, rec, 4, o, j);
    // write the chunk's partial blocks 0..ob (warp: quadrant q, columns 8 (w >> 2) ..),
    // zero the accumulators
    // (partial block indices staged at chunk start)
    const double zero[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int h2 = warp >> 2;
    for (int jb = 0; jb <= ((A.dbg & 16) ? -1 : ob); ++jb) {
      double v[2][2];
      tm_ld8(tq + 16 * jb + 8 * h2, v);
      tm_st8(tq + 16 * jb + 8 * h2, zero);
      const long long pb = ctl->pb[jb];
#pragma unroll
      for (int mb = 0; mb < 2; ++mb) {
        double* out = A.spart + (pb * TB + r0 + 8 * mb) * A.ncols + A.c_off;
        const int cc = h2 * 8 + 2 * t4;
        if (cc + 1 < ncl && ((A.ncols | A.c_off) & 1) == 0) {
          *reinterpret_cast<double2*>(out + cc) = make_double2(v[mb][0], v[mb][1]);
        } else {
          if (cc < ncl) out[cc] = v[mb][0];
          if (cc + 1 < ncl) out[cc + 1] = v[mb][1];
        }
      }
    }
    tm_wait_st();
    __syncthreads();  // x blocks reused by the next chunk
  }
  tl_mark(A, ctl, rec, 5, 0, 0);
  if (tid == 0) {
    ctl->streamed = base + ntiles;
    ctl->ncall++;
  }
  __syncthreads();
}

// y_j = sum over the row segments of the N-partials + sum_{i > j} partial (i, j),
// for one (subdomain, block) work item (fixed order).
__device__ __forceinline__ void sym_reduce_item(const TmvArgs& A, int k, int j) {
  const SubDev d = A.sub[k];
  const int nc = A.ncols;
  const int cnt = (j / SYM_SEG + 1) + (d.nt - 1 - j);
  const double* P0 = A.spart + A.pboff[d.blk0 + j] * TB * nc;
  for (int e = threadIdx.x; e < TB * nc; e += 256) {
    const int r = e / nc, c = e - r * nc;
    const int a = j * TB + r;
    if (a >= d.nI) continue;
    double v = 0.0;
    for (int p = 0; p < cnt; ++p) v += P0[((long long)p * TB + r) * nc + c];
    A.vout[(d.rI_off + a) * nc + c] = v;
  }
}

template <int NCP, int STAGES>
__global__ void __launch_bounds__(256, 1) k_sym(const TmvArgs A) {
  extern __shared__ __align__(16) double smem[];
  sym_item<NCP, STAGES>(A, blockIdx.x, smem);
}

// The symmetric pass as a launch of its own with the persistent kernel's structure: a
// resident grid, every CTA streaming its longest-processing-time list of row-segment items
// through one tile ring (no pipeline refill per item; two CTAs per SM with one RHS).
template <int NCP, int STAGES>
__global__ void __launch_bounds__(256, NCP == 1 ? 2 : 1)
    k_sym_stream(const TmvArgs A, const int* __restrict__ cta_ptr, const int* __restrict__ cta_items);

__global__ void __launch_bounds__(256) k_sym_reduce(const TmvArgs A, const int2* __restrict__ blk) {
  const int2 kb = blk[blockIdx.x];
  sym_reduce_item(A, kb.x, kb.y);
}

template <int MODE, int NCP, int STAGES>
__global__ void __launch_bounds__(256, 1) k_tmv(const TmvArgs A) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int any_s;
  const int tid = threadIdx.x;
  if (A.st) {
    if (A.st->done) return;
    if (MODE == PRE1 && A.check && !A.st->fixed) {
      if (tid == 0) any_s = 0;
      __syncthreads();
      if (tid < A.st->ncols && A.st->active[tid]) {
        double s = 0.0;
        for (int b = 0; b < NBLK; ++b) s += A.rr_part[b * A.st->ncols + tid];
        if (!(sqrt(s) <= A.st->tol * A.st->r0[tid])) atomicOr(&any_s, 1);
      }
      __syncthreads();
      if (!any_s) return;
    }
  }
  tmv_item<MODE, NCP, STAGES>(A, blockIdx.x, smem);
}

// ---------------------------------------------------------------------------
// Vector kernels
// ---------------------------------------------------------------------------
__device__ __forceinline__ int pow2ge(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

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

// out[j][c] = sum_{2 slots} sign * w * (x[slot][c] + G_k[slot row] . z[C_k^T][c])
// (+ partial dot with dotv). The coarse term is the explicit loop's G_k z.
struct CoarseTerm {
  const long long* goff;
  const int *np, *poff, *prim_gid;
  const double *G, *z;
};

__device__ __forceinline__ double coarse_term(const CoarseTerm& ct, int a, int ncols, int c) {
  const int np = ct.np[a];
  const double* Gr = ct.G + ct.goff[a];
  const int* gid = ct.prim_gid + ct.poff[a];
  double s = 0.0;
  int q = 0;
  // four terms' loads in flight (gid -> z is a dependent pair); additions in order
  for (; q + 4 <= np; q += 4) {
    int g4[4];
    double G4[4], z4[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      g4[t] = gid[q + t];
      G4[t] = Gr[q + t];
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) z4[t] = ct.z[(long long)g4[t] * ncols + c];
#pragma unroll
    for (int t = 0; t < 4; ++t) s += G4[t] * z4[t];
  }
  for (; q < np; ++q) s += Gr[q] * ct.z[(long long)gid[q] * ncols + c];
  return s;
}

__global__ void __launch_bounds__(VT)
    k_bgather(int m, int ncols, const LamDev* __restrict__ lam, const double* __restrict__ x,
              const double* __restrict__ weight, double* __restrict__ out, const double* __restrict__ dotv,
              double* __restrict__ partial, const PcgState* __restrict__ st, CoarseTerm ct) {
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
        if (ct.z) xv += coarse_term(ct, a, ncols, c);
        val += (double)L.sign[q] * (weight ? weight[a] : 1.0) * xv;
      }
      out[(long long)j * ncols + c] = val;
      if (dotv) dot += val * dotv[(long long)j * ncols + c];
    }
  }
  if (partial) block_col_reduce(dot, ncols, P2, partial);
}

// z = S^-1 (add + sum_k C_k sum_{cta of k} gpart)   (one CTA)
__global__ void __launch_bounds__(1024)
    k_coarse(int ng, int ncols, int nPmax, const int* __restrict__ pcon_ptr, const int* __restrict__ pcon_sub,
             const int* __restrict__ pcon_q, const int* __restrict__ sub_cta0, const int* __restrict__ sub_ncta,
             const double* __restrict__ gpart, const double* __restrict__ add, const double* __restrict__ Sinv,
             double* __restrict__ z, const PcgState* __restrict__ st) {
  if (st && st->done) return;
  extern __shared__ double gs[];  // ng x ncols
  for (int e = threadIdx.x; e < ng * ncols; e += blockDim.x) {
    const int gi = e / ncols, c = e - gi * ncols;
    double s = add ? add[e] : 0.0;
    for (int q = pcon_ptr[gi]; q < pcon_ptr[gi + 1]; ++q) {
      const int k = pcon_sub[q], lq = pcon_q[q];
      for (int cta = sub_cta0[k]; cta < sub_cta0[k] + sub_ncta[k]; ++cta)
        s += gpart[((long long)cta * nPmax + lq) * ncols + c];
    }
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

// out[c] = sum over the blocks' partials of column c: a warp per column, lane l adds the
// blocks l, l + 32, ... (independent loads in flight), then the xor-shuffle tree -- a fixed
// order, so every CTA (and every rank of a sharded solve) gets bitwise the same sums. Called
// by all threads of the block.
__device__ void reduce_cols(const double* part, int nblk, int ncols, double* out_smem) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = warp; c < ncols; c += nw) {
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += part[b * ncols + c];
    s = warp_sum(s);
    if (lane == 0) out_smem[c] = s;
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
               double* __restrict__ rr_part, double* __restrict__ coef, int coef_ld) {
  if (st->done) return;
  const int ncols = st->ncols;
  __shared__ double pq[IETIDP_MAX_RHS], alpha[IETIDP_MAX_RHS];
  reduce_cols(pq_part, NBLK, ncols, pq);
  __syncthreads();
  if (threadIdx.x < ncols) {
    const int c = threadIdx.x;
    alpha[c] = st->active[c] ? st->rz[c] / pq[c] : 0.0;
    if (blockIdx.x == 0 && st->active[c] && st->iters[c] < coef_ld) coef[c * coef_ld + st->iters[c]] = alpha[c];
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
              const double* __restrict__ rz_part, double* __restrict__ p, const double* __restrict__ z,
              double* __restrict__ coef, int coef_ld) {
  if (st->done) return;
  const int ncols = st->ncols;
  __shared__ int act[IETIDP_MAX_RHS];
  __shared__ double rz[IETIDP_MAX_RHS], beta[IETIDP_MAX_RHS];
  active_after(st, rr_part, act);
  reduce_cols(rz_part, NBLK, ncols, rz);
  __syncthreads();
  if (threadIdx.x < ncols) {
    const int c = threadIdx.x;
    beta[c] = rz[c] / st->rz[c];
    // iteration index j = st->iters[c] (k_ctl increments it after this kernel)
    if (blockIdx.x == 0 && act[c] && st->iters[c] < coef_ld) coef[(ncols + c) * coef_ld + st->iters[c]] = beta[c];
  }
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

// true relative dual residual per column: sqrt(sum of the k_resid partials) / ||r_0||
__global__ void k_resid_ratio(const double* __restrict__ part, const PcgState* __restrict__ st,
                              double* __restrict__ out) {
  // a warp per column, lanes over the per-block partials (loads in flight together)
  const int nc = st->ncols, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < nc; c += blockDim.x >> 5) {
    double v = 0.0;
    for (int b = lane; b < NBLK; b += 32) v += part[b * nc + c];
    v = warp_sum(v);
    if (lane == 0) out[c] = st->r0[c] > 0 ? sqrt(v) / st->r0[c] : 0.0;
  }
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
// Persistent PCG: the whole loop in ONE cooperative launch (one CTA per SM),
// phases separated by a grid-wide barrier. Each CTA keeps its own copy of the
// per-column CG scalars, reduced redundantly and in a fixed order from the
// per-CTA partials, so all CTAs take identical decisions (bit-reproducible).
// ---------------------------------------------------------------------------
struct PcgArgs {
  TmvArgs fwd, bwd, pre1, pre2;  // triangular loop
  TmvArgs wsym, ssym;            // explicit loop: W = S_II^-1, S_II
  CoarseTerm ct;                 // explicit loop: G_k z in the gather
  const int2* blk;               // (subdomain, block) items of the partial reduction
  const LamDev* lam;
  const double* delta;
  double *lamv, *r, *p, *q, *z;
  const double* d;
  double *xI, *zI;
  double *pslot, *rslot;  // B^T p and B_D^T r in slot order (operator inputs)
  const int *pcon_ptr, *pcon_sub, *pcon_q, *sub_cta0, *sub_ncta;
  const double *gpart, *Sinv;
  double* zc;
  double* part;  // [3][grid][ncols]: p.q, r.r, r.z partials
  PcgState* st;
  unsigned* bar;  // [0] arrivals, [1] generation
  double tol;
  int m, ncols, ng, nPmax, max_iter, fixed, n_items, ncp, n_blk;
  const int *cta_ptr, *cta_items;  // this CTA's work items (tile-balanced, longest first)
  unsigned long long* prof;        // optional (IETIDP_PCG_PROF): %globaltimer at every barrier
  const SlotRed* slot_red;         // explicit loop: partial sums folded into the gathers
  const int *gsrc_ptr, *gsrc;      // coarse partial rows per global primal
  double* gc;                      // coarse right-hand side g (larger coarse problems)
  int fold;                        // one column: fold the symmetric partials into the gathers
  int fold_multi;                  // ... and with several columns too
  long long n_slots;
  double* coef;  // PCG coefficients: alpha_j of column c at coef[c*coef_ld + j], beta_j at coef[(ncols+c)*coef_ld + j]
  int coef_ld;
  const GatherRec* grec;        // chunk pass: per multiplier row, its slots' partial lists and signs
  const double* wrec;           // chunk pass: per multiplier row, the two slots' scaling weights delta
  double* gzv;                  // chunk pass: G_k z_k per slot (n_slots x ncols), added by the gather of q
  int chunk;                   // several RHS: the chunk pass (sym_chunks) replaces the row-segment pass
  int smem_doubles;            // dynamic shared memory of the launch (doubles)
  int stop;                    // ietidp_stop: 0 ||r|| <= tol ||r0||, 1 sqrt(r.z) <= tol sqrt(r0.z0)
  const int* chunk_ptr;        // chunk pass: this CTA's chunks chunk_list[chunk_ptr[b] .. chunk_ptr[b+1])
  const SymChunk* chunk_list;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ int g_prof_n;  // barrier counter of the profiled launch (CTA 0)

// Grid barrier of the persistent kernel: arrival counter bar[0], generation bar[1].
// Thread 0 of each CTA arrives with an acquire-release atomic (cumulative over the
// CTA's writes ordered before it by __syncthreads), the last arrival resets the
// counter and publishes the next generation with a release; the others poll the
// generation with acquire loads.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g, old;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    if (old == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
      } while (cur == g);
    }
  }
  __syncthreads();
}

// Column sums of the CTAs' partials, computed by the whole CTA (every thread loads a
// share, then a fixed-shape tree in shared memory: deterministic); out[c], c < ncols,
// is valid for every thread on return.
__device__ void colsum_all(const double* part, int ncols, double* out) {
  __shared__ double red[VT];
  const int tid = threadIdx.x, P2 = pow2ge(ncols);
  const int c = tid % P2, g = tid / P2, G = VT / P2;
  double v = 0.0;
  if (c < ncols)
    for (int b = g; b < (int)gridDim.x; b += G) v += __ldcg(part + b * ncols + c);
  red[tid] = v;
  __syncthreads();
  for (int st = VT / 2; st >= P2; st >>= 1) {
    if (tid < st) red[tid] += red[tid + st];
    __syncthreads();
  }
  if (tid < ncols) out[tid] = red[tid];
  __syncthreads();
}

template <int MODE, int NCP, int STAGES>
__device__ __forceinline__ void tmv_phase(TmvArgs A, const int* cta_ptr, const int* cta_items, int ncp, double* smem) {
  for (int c0 = 0; c0 < A.ncols; c0 += ncp) {
    A.c_off = c0;
    for (int e = cta_ptr[blockIdx.x]; e < cta_ptr[blockIdx.x + 1]; ++e)
      tmv_item<MODE, NCP, STAGES>(A, cta_items[e], smem);
  }
}

template <int NCP, int STAGES>
__device__ __forceinline__ void sym_phase(TmvArgs A, const int* cta_ptr, const int* cta_items, int ncp, double* smem) {
  for (int c0 = 0; c0 < A.ncols; c0 += ncp) {
    A.c_off = c0;
    const int beg = cta_ptr[blockIdx.x], end = cta_ptr[blockIdx.x + 1];
    sym_stream<NCP, STAGES>(A, cta_items + beg, end - beg, smem);
  }
}

template <int NCP, int STAGES>
__global__ void __launch_bounds__(256, NCP == 1 ? 2 : 1)
    k_sym_stream(const TmvArgs A, const int* __restrict__ cta_ptr, const int* __restrict__ cta_items) {
  extern __shared__ __align__(16) double smem[];
  sym_phase<NCP, STAGES>(A, cta_ptr, cta_items, NCP, smem);
}

__shared__ ChunkCtl g_chunk_ctl;  // per CTA (chunk pass): ring mbarriers, tensor memory, stream count

// The symmetric pass of the persistent kernel: the chunk pass (several RHS) or the
// row-segment stream.
template <int NCP, int STAGES, bool CH = false>
__device__ __forceinline__ void sym_pass(const PcgArgs& P, TmvArgs A, double* smem) {
  if constexpr (NCP == 16 && CH) {
    {
      const int beg = P.chunk_ptr[blockIdx.x], end = P.chunk_ptr[blockIdx.x + 1];
      for (int c0 = 0; c0 < A.ncols; c0 += CH_NC) {
        A.c_off = c0;
        sym_chunks<STAGES>(A, P.chunk_list + beg, end - beg, smem, &g_chunk_ctl);
      }
      return;
    }
  } else {
    sym_phase<NCP, STAGES>(A, P.cta_ptr, P.cta_items, P.ncp, smem);
  }
}

__device__ __forceinline__ double sym_value(const double* spart, const SlotRed* sred, long long a, int nc, int c);

// y = the reduced symmetric pass, element-parallel over (slot, column) (same order as
// sym_value / sym_reduce_item)
__device__ __forceinline__ void reduce_phase(const TmvArgs& A, const SlotRed* sred, long long n_slots) {
  const long long n = n_slots * A.ncols;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long st = (long long)TB * A.ncols;
  // four elements per thread, their partials loaded together (the sum of each element
  // stays in index order, as in sym_value)
  for (long long e0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; e0 < n; e0 += 4 * stride) {
    const double* P0[4];
    int cnt[4], maxc = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long e = e0 + u * stride;
      cnt[u] = 0;
      P0[u] = A.spart;
      if (e < n) {
        const long long a = e / A.ncols;
        const SlotRed sr = sred[a];
        P0[u] = A.spart + sr.base * A.ncols + (e - a * A.ncols);
        cnt[u] = sr.cnt;
        maxc = max(maxc, sr.cnt);
      }
    }
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int p = 0; p < maxc; ++p) {
      double t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] = p < cnt[u] ? P0[u][p * st] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (p < cnt[u]) v[u] += t[u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (e0 + u * stride < n) A.vout[e0 + u * stride] = v[u];
  }
}

// z = S_PP^-1 sum of the coarse partials: every CTA assembles g, each computes a
// slice of the rows of z.
__device__ __forceinline__ void coarse_phase(const PcgArgs& P, double* smem) {
  const int nc = P.ncols, tid = threadIdx.x, nb = gridDim.x;
  double* g = smem;  // ng x nc
  const int warp = tid >> 5, lane = tid & 31;
  __syncthreads();
  for (int e = warp; e < P.ng * nc; e += VT / 32) {
    const int gi = e / nc, c = e - gi * nc;
    double sacc = 0.0;
    for (int q = P.gsrc_ptr[gi] + lane; q < P.gsrc_ptr[gi + 1]; q += 32)
      sacc += __ldcg(P.gpart + (long long)P.gsrc[q] * nc + c);
    sacc = warp_sum(sacc);
    if (lane == 0) g[e] = sacc;
  }
  __syncthreads();
  for (int e = blockIdx.x * 8 + warp; e < P.ng * nc; e += nb * 8) {
    const int i = e / nc, c = e - i * nc;
    double sacc = 0.0;
    for (int j = lane; j < P.ng; j += 32) sacc += P.Sinv[(long long)i * P.ng + j] * g[j * nc + c];
    sacc = warp_sum(sacc);
    if (lane == 0) P.zc[e] = sacc;
  }
}

// z = S_PP^-1 g, computed by every CTA into shared memory (ng x nc; redundant, no barrier)
// -- for coarse problems up to COARSE_LOCAL_MAX primal DOFs (S_PP^-1 read by every CTA)
constexpr int COARSE_LOCAL_MAX = 32;
__device__ __forceinline__ void coarse_local(const PcgArgs& P, double* zs) {
  const int nc = P.ncols, tid = threadIdx.x;
  double* g = zs + P.ng * nc;
  __syncthreads();
  // g[gi][c]: a warp per (gi, c), lanes over the flattened partial rows (fixed order)
  const int warp = tid >> 5, lane = tid & 31;
  for (int e = warp; e < P.ng * nc; e += VT / 32) {
    const int gi = e / nc, c = e - gi * nc;
    double sacc = 0.0;
    for (int q = P.gsrc_ptr[gi] + lane; q < P.gsrc_ptr[gi + 1]; q += 32)
      sacc += __ldcg(P.gpart + (long long)P.gsrc[q] * nc + c);
    sacc = warp_sum(sacc);
    if (lane == 0) g[e] = sacc;
  }
  __syncthreads();
  for (int e = tid; e < P.ng * nc; e += VT) {
    const int i = e / nc, c = e - i * nc;
    double sacc = 0.0;
    for (int j = 0; j < P.ng; ++j) sacc += P.Sinv[(long long)i * P.ng + j] * g[j * nc + c];
    zs[e] = sacc;
  }
  __syncthreads();
}

// Larger coarse problems: g (warp per entry) and then z = S_PP^-1 g (warp per row),
// both spread over the CTAs, through global memory.
__device__ __forceinline__ void coarse_spread(const PcgArgs& P) {
  // a warp per entry (gi, c), lanes over the flattened partial rows (each lane's rows in
  // order, then the butterfly); the warp's entries, their row indices and the first four
  // rows of each lane are loaded together
  const int nc = P.ncols, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = P.ng * nc, W = gridDim.x * (VT / 32);
  constexpr int K = 3, M = 4;
  for (int eb = blockIdx.x * (VT / 32) + warp; eb < n; eb += K * W) {
    int lo[K], hi[K], cc[K], idx[K][M];
    double v[K][M];
#pragma unroll
    for (int u = 0; u < K; ++u) {
      const int e = eb + u * W;
      lo[u] = hi[u] = 0;
      cc[u] = 0;
      if (e < n) {
        const int gi = e / nc;
        cc[u] = e - gi * nc;
        lo[u] = P.gsrc_ptr[gi];
        hi[u] = P.gsrc_ptr[gi + 1];
      }
    }
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int q = lo[u] + lane + 32 * m;
        idx[u][m] = q < hi[u] ? P.gsrc[q] : -1;
      }
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int m = 0; m < M; ++m) v[u][m] = idx[u][m] >= 0 ? __ldcg(P.gpart + (long long)idx[u][m] * nc + cc[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      const int e = eb + u * W;
      double sacc = 0.0;
#pragma unroll
      for (int m = 0; m < M; ++m)
        if (idx[u][m] >= 0) sacc += v[u][m];
      for (int q = lo[u] + lane + 32 * M; q < hi[u]; q += 32) sacc += __ldcg(P.gpart + (long long)P.gsrc[q] * nc + cc[u]);
      sacc = warp_sum(sacc);
      if (lane == 0 && e < n) P.gc[e] = sacc;
    }
  }
}
__device__ __forceinline__ void coarse_spread_z(const PcgArgs& P) {
  const int nc = P.ncols, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = blockIdx.x * (VT / 32) + warp; e < P.ng * nc; e += gridDim.x * (VT / 32)) {
    const int i = e / nc, c = e - i * nc;
    double sacc = 0.0;
    for (int j = lane; j < P.ng; j += 32) sacc += P.Sinv[(long long)i * P.ng + j] * __ldcg(P.gc + j * nc + c);
    sacc = warp_sum(sacc);
    if (lane == 0) P.zc[e] = sacc;
  }
}

// y[slot][c] of a symmetric pass: the row-segment partials plus the transposed partials
// (the same fixed order as sym_reduce_item)
__device__ __forceinline__ double sym_value_sr(const double* spart, const SlotRed& sr, int nc, int c);
__device__ __forceinline__ double sym_value(const double* spart, const SlotRed* sred, long long a, int nc, int c) {
  return sym_value_sr(spart, sred[a], nc, c);
}
__device__ __forceinline__ double sym_value_sr(const double* spart, const SlotRed& sr, int nc, int c) {
  const double* P0 = spart + sr.base * nc + c;
  const long long st = (long long)TB * nc;
  double v0 = 0.0;
  int p = 0;
  // the partials in order; four loads in flight (the additions stay in order)
  for (; p + 4 <= sr.cnt; p += 4) {
    const double a0 = P0[p * st], a1 = P0[(p + 1) * st], a2 = P0[(p + 2) * st], a3 = P0[(p + 3) * st];
    v0 = (((v0 + a0) + a1) + a2) + a3;
  }
  for (; p < sr.cnt; ++p) v0 += P0[p * st];
  return v0;
}

// out = sum_k B (w) (x + G z), with the per-CTA partial of out . dotv
template <int UR = 1>
__device__ __forceinline__ void bgather_phase(const PcgArgs& P, const double* x, const double* w, double* out,
                                              const double* dotv, double* part, bool coarse,
                                              const TmvArgs* fold = nullptr, const double* zs = nullptr) {
  const int nc = P.ncols, P2 = pow2ge(nc);
  const int c = threadIdx.x % P2, rl = threadIdx.x / P2, R = VT / P2;
  double dot = 0.0;
  if (UR > 1 && !fold && !zs) {
    // UR rows per thread in flight (loads first); the row order of the dot partial is
    // that of a one-row loop
    const int stride = gridDim.x * R;
    if (c < nc)
      for (int j0 = blockIdx.x * R + rl; j0 < P.m; j0 += UR * stride) {
        LamDev L4[UR];
        double dv[UR], xv[UR][2], wv[UR][2];
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const int j = j0 + u * stride;
          if (j < P.m) {
            L4[u] = P.lam[j];
            dv[u] = dotv[(long long)j * nc + c];
          }
        }
#pragma unroll
        for (int u = 0; u < UR; ++u)
          if (j0 + u * stride < P.m)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int a = L4[u].slot[q];
              xv[u][q] = x[(long long)a * nc + c];
              wv[u][q] = w ? w[a] : 1.0;
            }
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const int j = j0 + u * stride;
          if (j >= P.m) continue;
          double val = 0.0;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            double x1 = xv[u][q];
            if (coarse) x1 += coarse_term(P.ct, L4[u].slot[q], nc, c);
            val += (double)L4[u].sign[q] * wv[u][q] * x1;
          }
          out[(long long)j * nc + c] = val;
          dot += val * dv[u];
        }
      }
    block_col_reduce(dot, nc, P2, part);
    return;
  }
  if (c < nc)
    for (int j = blockIdx.x * R + rl; j < P.m; j += gridDim.x * R) {
      const LamDev L = P.lam[j];
      double val = 0.0;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int a = L.slot[q];
        double xv = fold ? sym_value(fold->spart, P.slot_red, a, nc, c) : x[(long long)a * nc + c];
        if (coarse) {
          if (zs) {  // G_k[slot row] . z (z in shared memory)
            const int np = P.ct.np[a];
            const double* Gr = P.ct.G + P.ct.goff[a];
            const int* gid = P.ct.prim_gid + P.ct.poff[a];
            double sc = 0.0;
            for (int q2 = 0; q2 < np; ++q2) sc += Gr[q2] * zs[gid[q2] * nc + c];
            xv += sc;
          } else {
            xv += coarse_term(P.ct, a, nc, c);
          }
        }
        val += (double)L.sign[q] * (w ? w[a] : 1.0) * xv;
      }
      out[(long long)j * nc + c] = val;
      dot += val * dotv[(long long)j * nc + c];
    }
  block_col_reduce(dot, nc, P2, part);
}

// ---- chunk mode (several RHS): coarse correction and folded gathers ----

// After the coarse right-hand side g (P.gc, ng x nc) is complete: every CTA takes its
// subdomains, forms z_k = (S_PP^-1 g)[C_k rows] (S_PP^-1 rows and g staged in shared
// memory) and writes G_k z_k per slot (P.gzv); the gather of q = sum_k B (W_k p_k +
// G_k z_k) adds it to the slot's first chunk partial (F_DP = W +
// G S_PP^-1 G^T, SURVEY F1 signs).
__device__ __forceinline__ void coarse_gz_phase(const PcgArgs& P, const TmvArgs& A, double* smem, int smem_doubles) {
  const int nc = P.ncols, ng = P.ng, tid = threadIdx.x;
  double* gs = smem;               // g: ng x nc
  double* srow = gs + ng * nc;     // the subdomain's nP rows of S_PP^-1 (nP x ng)
  double* zk = srow + P.nPmax * ng;  // z_k: nP x nc
  double* gG = zk + P.nPmax * nc;    // G_k rows, a chunk at a time (rows x nP)
  const int gcap = smem_doubles - (int)(gG - smem);
  for (int e = tid; e < ng * nc; e += VT) gs[e] = __ldcg(P.gc + e);
  for (int k = blockIdx.x; k < A.n_sub; k += gridDim.x) {
    const SubDev d = A.sub[k];
    if (d.nP == 0 || d.nI == 0) continue;
    __syncthreads();  // gs complete (first), srow / zk / gG free (later)
    const int* gid = A.prim_gid + d.prim_off;
    for (int e = tid; e < d.nP * ng; e += VT) {
      const int q = e / ng, j = e - q * ng;
      srow[e] = __ldg(P.Sinv + (long long)gid[q] * ng + j);
    }
    const int rows = min(d.nI, gcap / d.nP);  // G rows per chunk
    const double* Gk = A.gmat + d.g_off;
    int a0 = 0;
    // first chunk of G_k in flight while z_k is formed
    for (int e = tid; e < rows * d.nP; e += VT) gG[e] = __ldg(Gk + e);
    __syncthreads();
    for (int e = tid; e < d.nP * nc; e += VT) {
      const int q = e / nc, c = e - q * nc;
      double acc = 0.0;
#pragma unroll 4
      for (int j = 0; j < ng; ++j) acc += srow[q * ng + j] * gs[j * nc + c];
      zk[e] = acc;
    }
    __syncthreads();
    const int P2 = pow2ge(nc), c = tid % P2, rl = tid / P2, R = VT / P2;
    while (true) {
      const int na = min(rows, d.nI - a0);
      if (c < nc)
        for (int a = rl; a < na; a += R) {
          const double* Gr = gG + a * d.nP;
          double acc = 0.0;
          for (int q = 0; q < d.nP; ++q) acc += Gr[q] * zk[q * nc + c];
          P.gzv[(d.rI_off + a0 + a) * nc + c] = acc;  // (G_k z_k) of the slot; the gather adds it to partial 0
        }
      a0 += na;
      if (a0 >= d.nI) break;
      __syncthreads();
      for (int e = tid; e < min(rows, d.nI - a0) * d.nP; e += VT) gG[e] = __ldg(Gk + (long long)a0 * d.nP + e);
      __syncthreads();
    }
  }
}

// out[j][c] = sum_{2 slots} sign (w) sum_{p < cnt} partial_p[slot][c], plus the per-CTA
// partial of out . dotv; UR multiplier rows per thread in flight (metadata, then all
// partial loads, then the sums in index order: the same arithmetic as sym_value).
template <int UR>
__device__ __forceinline__ void gather_fold(const PcgArgs& P, const double* spart, bool weighted, double* out,
                                            const double* dotv, double* part, const double* gzv = nullptr) {
  const int nc = P.ncols, P2 = pow2ge(nc);
  const int c = threadIdx.x % P2, rl = threadIdx.x / P2, R = VT / P2;
  const long long st = (long long)TB * nc;
  constexpr int CM = 4;  // partials per slot loaded together (more: a loop)
  double dot = 0.0;
  const int stride = gridDim.x * R;
  if (c < nc)
    for (int j0 = blockIdx.x * R + rl; j0 < P.m; j0 += UR * stride) {
      GatherRec g[UR];
      double w[UR][2], dv[UR];
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const int j = j0 + u * stride;
        if (j < P.m) {
          g[u] = P.grec[j];
          dv[u] = dotv[(long long)j * nc + c];
          if (weighted) {
            w[u][0] = P.wrec[2 * j];
            w[u][1] = P.wrec[2 * j + 1];
          } else {
            w[u][0] = w[u][1] = 1.0;
          }
        } else {
          g[u].cnt[0] = g[u].cnt[1] = 0;
        }
      }
      double v[UR][2][CM];
#pragma unroll
      for (int u = 0; u < UR; ++u)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double* p0 = spart + g[u].base[q] * nc + c;
#pragma unroll
          for (int p = 0; p < CM; ++p) v[u][q][p] = p < g[u].cnt[q] ? __ldcg(p0 + p * st) : 0.0;
        }
      if (gzv) {  // the coarse term joins the first partial of each slot
#pragma unroll
        for (int u = 0; u < UR; ++u)
#pragma unroll
          for (int q = 0; q < 2; ++q)
            if (g[u].cnt[q] > 0) v[u][q][0] += __ldcg(gzv + (long long)g[u].slot[q] * nc + c);
      }
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const int j = j0 + u * stride;
        if (j >= P.m) continue;
        double val = 0.0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          double y = 0.0;
#pragma unroll
          for (int p = 0; p < CM; ++p)
            if (p < g[u].cnt[q]) y += v[u][q][p];
          for (int p = CM; p < g[u].cnt[q]; ++p) y += __ldcg(spart + g[u].base[q] * nc + c + p * st);
          val += (double)g[u].sign[q] * w[u][q] * y;
        }
        out[(long long)j * nc + c] = val;
        dot += val * dv[u];
      }
    }
  block_col_reduce(dot, nc, P2, part);
}

// write B^T v (optionally weighted) of lambda-row j, column c into the slot vector
__device__ __forceinline__ void to_slots(const PcgArgs& P, long long j, int c, double v, const double* w, double* out) {
  const LamDev L = P.lam[j];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int a = L.slot[q];
    out[(long long)a * P.ncols + c] = (double)L.sign[q] * (w ? w[a] : 1.0) * v;
  }
}

// grid barrier of the PCG kernel; with P.prof, CTA 0 records the time of arrival
__device__ __forceinline__ void pcg_barrier(const PcgArgs& P) {
  if (P.prof && blockIdx.x == 0 && threadIdx.x == 0) {
    const int i = g_prof_n++;
    if (i < 4096) P.prof[i] = gtimer();
  }
  grid_barrier(P.bar);
}

// Set-up of the chunk pass in a CTA: ring mbarriers, the tensor-memory allocation, zeroed
// accumulators (the persistent kernel does it once; the sharded loop's pass kernels per launch).
template <int STAGES>
__device__ __forceinline__ void chunk_prologue() {
  const int tid = threadIdx.x;
  // ring mbarriers and the tensor-memory accumulators
  if (tid == 0) {
    for (int s2 = 0; s2 < STAGES; ++s2) {
      mbar_init(&g_chunk_ctl.full[s2], 1);
      g_chunk_ctl.rel[s2] = 0;
    }
    for (int q = 0; q < 4; ++q) g_chunk_ctl.diag[q] = 0;
    g_chunk_ctl.streamed = 0;
    g_chunk_ctl.ncall = g_chunk_ctl.ntl = 0;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if ((tid >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&g_chunk_ctl.tmem)),
                 "n"(CH_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int w = tid >> 5;
  const unsigned tb = g_chunk_ctl.tmem + ((unsigned)(32 * (w & 3)) << 16) + 8u * (w >> 2);
  const double zero[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int jb = 0; jb < 32; ++jb) tm_st8(tb + 16 * jb, zero);
  tm_wait_st();
  __syncthreads();
}
__device__ __forceinline__ void chunk_epilogue() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(g_chunk_ctl.tmem), "n"(CH_TMEM_COLS));
}

template <int NCP, int STAGES, bool EXPL, bool CH>
__device__ __forceinline__ void apply_F_phases(const PcgArgs& P, double* smem, double* pq) {
  if constexpr (EXPL && CH) {
    {
      // chunk mode: W pass | g | z_k, G_k z_k into the partials | folded gather of q
      sym_pass<NCP, STAGES, true>(P, P.wsym, smem);
      pcg_barrier(P);
      if (P.ng > 0) {
        coarse_spread(P);
        pcg_barrier(P);
        coarse_gz_phase(P, P.wsym, smem, P.smem_doubles);
        pcg_barrier(P);
      }
      gather_fold<2>(P, P.wsym.spart, false, P.q, P.p, pq, P.ng > 0 ? P.gzv : nullptr);
      return;
    }
  } else if constexpr (EXPL) {
    // W pass; then every CTA solves the coarse problem itself and folds the pass's
    // partial sums into the gather (no reduction phase, one barrier)
    // one column: the partial sums are folded into the gather; several: a reduction
    // phase (a slot shared by several multipliers would be summed repeatedly)
    const bool fold = P.fold && (P.ncols == 1 || P.fold_multi);
    const bool row1 = P.ncols == 1 && P.ng > 0 && P.ng <= COARSE_LOCAL_MAX && fold && P.m <= (int)gridDim.x * VT;
    const bool row1s = P.ncols == 1 && P.ng > COARSE_LOCAL_MAX && fold && P.m <= (int)gridDim.x * VT;  // spread coarse
    const int j = blockIdx.x * VT + threadIdx.x;
    LamDev L{};
    SlotRed sr[2] = {};
    sym_pass<NCP, STAGES>(P, P.wsym, smem);
    if ((row1 || row1s) && j < P.m) {  // static row data, loaded ahead of the barrier
      L = P.lam[j];
      sr[0] = P.slot_red[L.slot[0]];
      sr[1] = P.slot_red[L.slot[1]];
    }
    pcg_barrier(P);
    if (row1s) {
      // one row per thread: folded operator values first (in flight across the coarse
      // phases and their barriers), then the coarse term G_k z from the spread solve
      double pre[2] = {0.0, 0.0};
      if (j < P.m) {
#pragma unroll
        for (int q = 0; q < 2; ++q) pre[q] = sym_value_sr(P.wsym.spart, sr[q], 1, 0);
      }
      coarse_spread(P);
      pcg_barrier(P);
      coarse_spread_z(P);
      pcg_barrier(P);
      double dot = 0.0;
      if (j < P.m) {
        double val = 0.0;
#pragma unroll
        for (int q = 0; q < 2; ++q) val += (double)L.sign[q] * (pre[q] + coarse_term(P.ct, L.slot[q], 1, 0));
        P.q[j] = val;
        dot = val * P.p[j];
      }
      block_col_reduce(dot, 1, 1, pq);
      return;
    }
    if (!fold) reduce_phase(P.wsym, P.slot_red, P.n_slots);
    if (row1) {
      // one row per thread: the row's folded operator value is loaded first, so that
      // its latency chain overlaps the per-CTA coarse solve; then the coarse term
      double pre[2] = {0.0, 0.0}, sg[2] = {0.0, 0.0};
      if (j < P.m) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          pre[q] = sym_value_sr(P.wsym.spart, sr[q], 1, 0);
          sg[q] = (double)L.sign[q];
        }
      }
      coarse_local(P, smem);  // small coarse problem: every CTA solves it (no barrier)
      double dot = 0.0;
      if (j < P.m) {
        double val = 0.0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int a = L.slot[q];
          const int np = P.ct.np[a];
          const double* Gr = P.ct.G + P.ct.goff[a];
          const int* gid = P.ct.prim_gid + P.ct.poff[a];
          double sc = 0.0;
          for (int q2 = 0; q2 < np; ++q2) sc += Gr[q2] * smem[gid[q2]];
          val += sg[q] * (pre[q] + sc);
        }
        P.q[j] = val;
        dot = val * P.p[j];
      }
      block_col_reduce(dot, 1, 1, pq);
    } else if (P.ng > 0 && P.ng <= COARSE_LOCAL_MAX) {
      if (!fold) pcg_barrier(P);
      coarse_local(P, smem);  // small coarse problem: every CTA solves it (no barrier)
      bgather_phase(P, P.xI, nullptr, P.q, P.p, pq, true, fold ? &P.wsym : nullptr, smem);
    } else {
      if (P.ng > 0) {  // g, then the rows of z, spread over the CTAs
        coarse_spread(P);
        pcg_barrier(P);
        coarse_spread_z(P);
      }
      if (P.ng > 0 || !fold) pcg_barrier(P);
      bgather_phase<NCP == 1 ? 1 : 2>(P, P.xI, nullptr, P.q, P.p, pq, P.ng > 0, fold ? &P.wsym : nullptr);
    }
  } else {
    tmv_phase<FWD, NCP, STAGES>(P.fwd, P.cta_ptr, P.cta_items, P.ncp, smem);
    pcg_barrier(P);
    if (P.ng > 0) {
      coarse_phase(P, smem);
      pcg_barrier(P);
    }
    tmv_phase<BWD, NCP, STAGES>(P.bwd, P.cta_ptr, P.cta_items, P.ncp, smem);
    pcg_barrier(P);
    bgather_phase(P, P.xI, nullptr, P.q, P.p, pq, false);
  }
}

template <int NCP, int STAGES, bool EXPL, bool CH>
__device__ __forceinline__ void apply_M_phases(const PcgArgs& P, double* smem, double* rz) {
  if constexpr (EXPL && CH) {  // chunk mode: S pass | folded, weighted gather of z
    sym_pass<NCP, STAGES, true>(P, P.ssym, smem);
    pcg_barrier(P);
    gather_fold<2>(P, P.ssym.spart, true, P.z, P.r, rz);
    return;
  } else if constexpr (EXPL) {
    const bool row1 = P.ncols == 1 && P.fold && P.m <= (int)gridDim.x * VT;
    const int j = blockIdx.x * VT + threadIdx.x;
    LamDev L{};
    SlotRed sr[2] = {};
    double w2[2] = {0.0, 0.0};
    sym_pass<NCP, STAGES>(P, P.ssym, smem);
    if (row1 && j < P.m) {  // static row data, loaded ahead of the barrier
      L = P.lam[j];
      sr[0] = P.slot_red[L.slot[0]];
      sr[1] = P.slot_red[L.slot[1]];
      w2[0] = P.delta[L.slot[0]];
      w2[1] = P.delta[L.slot[1]];
    }
    pcg_barrier(P);
    if (row1) {  // z = B_D (S r) row by row, r.z partials (same order as bgather_phase)
      double dot = 0.0;
      if (j < P.m) {
        double val = 0.0;
#pragma unroll
        for (int q = 0; q < 2; ++q) val += (double)L.sign[q] * w2[q] * sym_value_sr(P.ssym.spart, sr[q], 1, 0);
        P.z[j] = val;
        dot = val * P.r[j];
      }
      block_col_reduce(dot, 1, 1, rz);
    } else if (P.fold && (P.ncols == 1 || P.fold_multi)) {
      bgather_phase(P, P.zI, P.delta, P.z, P.r, rz, false, &P.ssym);
    } else {
      reduce_phase(P.ssym, P.slot_red, P.n_slots);
      pcg_barrier(P);
      bgather_phase<NCP == 1 ? 1 : 2>(P, P.zI, P.delta, P.z, P.r, rz, false);
    }
  } else {
    tmv_phase<PRE1, NCP, STAGES>(P.pre1, P.cta_ptr, P.cta_items, P.ncp, smem);
    pcg_barrier(P);
    tmv_phase<PRE2, NCP, STAGES>(P.pre2, P.cta_ptr, P.cta_items, P.ncp, smem);
    pcg_barrier(P);
    bgather_phase(P, P.zI, P.delta, P.z, P.r, rz, false);
  }
}

// ---- the chunk-mode phases as launches of their own (sharded solve, several RHS): the same
// device functions as the persistent kernel's phases, a kernel boundary where that has a grid
// barrier, so that the sums over the ranks can run between them ----
template <int STAGES, int WHICH>  // WHICH 0: W = S_II^-1 (F-apply), 1: S_II (preconditioner)
__global__ void __launch_bounds__(256, 1) k_ch_pass(const PcgArgs P) {
  extern __shared__ __align__(16) double smem[];
  if (P.st->done) return;
  chunk_prologue<STAGES>();
  sym_pass<16, STAGES, true>(P, WHICH ? P.ssym : P.wsym, smem);
  chunk_epilogue();
}
__global__ void __launch_bounds__(256, 1) k_ch_g(const PcgArgs P) {
  if (P.st->done) return;
  coarse_spread(P);
}
__global__ void __launch_bounds__(256, 1) k_ch_zk(const PcgArgs P) {
  extern __shared__ __align__(16) double smem[];
  if (P.st->done) return;
  coarse_gz_phase(P, P.wsym, smem, P.smem_doubles);
}
template <int WHICH>
__global__ void __launch_bounds__(256, 1) k_ch_gather(const PcgArgs P, double* scratch) {
  if (P.st->done) return;
  if (WHICH) gather_fold<2>(P, P.ssym.spart, true, P.z, P.r, scratch);
  else gather_fold<2>(P, P.wsym.spart, false, P.q, P.p, scratch, P.ng > 0 ? P.gzv : nullptr);
}

template <int NCP, int STAGES, bool EXPL, bool CH = false>
__global__ void __launch_bounds__(256, NCP == 1 ? 2 : 1) k_pcg(const PcgArgs P) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double s_rz[IETIDP_MAX_RHS], s_r0[IETIDP_MAX_RHS], s_coef[IETIDP_MAX_RHS], s_sum[IETIDP_MAX_RHS];
  __shared__ double s_rz0[IETIDP_MAX_RHS];  // r_0 . z_0 (preconditioned stopping criterion)
  __shared__ int s_act[IETIDP_MAX_RHS], s_new[IETIDP_MAX_RHS], s_iters[IETIDP_MAX_RHS];
  __shared__ int s_any;
  const int tid = threadIdx.x, nb = gridDim.x, nc = P.ncols, m = P.m;
  double* pq = P.part;
  double* rr = P.part + nb * nc;
  double* rz = P.part + 2 * nb * nc;
  const int P2 = pow2ge(nc);
  const int cc = tid % P2, rl = tid / P2, R = VT / P2;
  auto rows = [&](auto&& f) {  // this CTA's share of the lambda-space rows, column cc
    if (cc < nc)
      for (int j = blockIdx.x * R + rl; j < m; j += nb * R) f((long long)j * nc + cc, j);
  };
  if constexpr (NCP == 16 && EXPL && CH) chunk_prologue<STAGES>();
  // ---- init: lambda = 0, r = d, r0 = ||d|| ----
  {
    double acc = 0.0;
    rows([&](long long e, int j) {
      P.lamv[e] = 0.0;
      const double dv = P.d[e];
      P.r[e] = dv;
      to_slots(P, j, cc, dv, P.delta, P.rslot);
      acc += dv * dv;
    });
    block_col_reduce(acc, nc, P2, rr);
  }
  pcg_barrier(P);
  colsum_all(rr, nc, s_sum);
  if (tid < nc) {
    s_r0[tid] = sqrt(s_sum[tid]);
    s_act[tid] = (m > 0 && s_r0[tid] > 0.0) ? 1 : 0;
    s_iters[tid] = 0;
    s_rz[tid] = 0.0;
  }
  __syncthreads();
  int it = 0;
  bool run = false;
  for (int c = 0; c < nc; ++c) run |= s_act[c] != 0;
  if (!P.fixed && P.max_iter <= 0) run = false;
  if (run) {
    // z = M r, rz = r.z, p = z
    apply_M_phases<NCP, STAGES, EXPL, CH>(P, smem, rz);
    pcg_barrier(P);
    colsum_all(rz, nc, s_sum);
    if (tid < nc) s_rz[tid] = s_rz0[tid] = s_sum[tid];
    rows([&](long long e, int j) {
      const double zv = P.z[e];
      P.p[e] = zv;
      to_slots(P, j, cc, zv, nullptr, P.pslot);
    });
    pcg_barrier(P);
  }
  // one column, one multiplier row per thread: the vector phases preload their row
  // data (slots, scaling, r, p) ahead of the grid barrier and issue the load of the
  // freshly computed vector before the column sum (same arithmetic as the general path)
  const bool fast1 = nc == 1 && m <= (int)gridDim.x * VT;
  constexpr int UR = NCP == 1 ? 1 : 4;  // rows in flight per thread in the vector phases
  const int jr = blockIdx.x * VT + tid;
  const bool myrow = fast1 && jr < m;
  while (run) {
    apply_F_phases<NCP, STAGES, EXPL, CH>(P, smem, pq);  // q = F p
    LamDev Lr{};
    double r_pre = 0.0, p_pre = 0.0, d0 = 0.0, d1 = 0.0;
    if (myrow) {
      Lr = P.lam[jr];
      r_pre = P.r[jr];
      p_pre = P.p[jr];
      d0 = P.delta[Lr.slot[0]];
      d1 = P.delta[Lr.slot[1]];
    }
    pcg_barrier(P);
    // alpha, lambda and r
    const double qv = myrow ? P.q[jr] : 0.0;
    colsum_all(pq, nc, s_sum);
    if (tid < nc) {
      s_coef[tid] = s_act[tid] ? s_rz[tid] / s_sum[tid] : 0.0;
      if (blockIdx.x == 0 && s_act[tid] && s_iters[tid] < P.coef_ld) P.coef[tid * P.coef_ld + s_iters[tid]] = s_coef[tid];
    }
    __syncthreads();
    if (fast1) {
      double acc = 0.0;
      if (myrow) {
        double rv = r_pre;
        if (s_act[0]) {
          const double a = s_coef[0];
          P.lamv[jr] += a * p_pre;
          rv -= a * qv;
          P.r[jr] = rv;
        }
        P.rslot[Lr.slot[0]] = (double)Lr.sign[0] * d0 * rv;
        P.rslot[Lr.slot[1]] = (double)Lr.sign[1] * d1 * rv;
        acc = rv * rv;
      }
      block_col_reduce(acc, 1, 1, rr);
    } else {
      // four rows per thread in flight (all loads first); the same arithmetic and
      // accumulation order as a one-row loop
      double acc = 0.0;
      const bool act = cc < nc && s_act[cc];
      const double a = cc < nc ? s_coef[cc] : 0.0;
      const int stride = nb * R;
      if (cc < nc)
        for (int j0 = blockIdx.x * R + rl; j0 < m; j0 += UR * stride) {
          double rv[UR], pv[UR], qv4[UR], lv[UR], w0[UR], w1[UR];
          LamDev L4[UR];
#pragma unroll
          for (int u = 0; u < UR; ++u) {
            const int j = j0 + u * stride;
            if (j < m) {
              const long long e = (long long)j * nc + cc;
              rv[u] = P.r[e];
              pv[u] = P.p[e];
              qv4[u] = P.q[e];
              lv[u] = P.lamv[e];
              L4[u] = P.lam[j];
            }
          }
#pragma unroll
          for (int u = 0; u < UR; ++u)
            if (j0 + u * stride < m) {
              w0[u] = P.delta[L4[u].slot[0]];
              w1[u] = P.delta[L4[u].slot[1]];
            }
#pragma unroll
          for (int u = 0; u < UR; ++u) {
            const int j = j0 + u * stride;
            if (j >= m) continue;
            const long long e = (long long)j * nc + cc;
            double r1 = rv[u];
            if (act) {
              P.lamv[e] = lv[u] + a * pv[u];
              r1 -= a * qv4[u];
              P.r[e] = r1;
            }
            P.rslot[(long long)L4[u].slot[0] * nc + cc] = (double)L4[u].sign[0] * w0[u] * r1;
            P.rslot[(long long)L4[u].slot[1] * nc + cc] = (double)L4[u].sign[1] * w1[u] * r1;
            acc += r1 * r1;
          }
        }
      block_col_reduce(acc, nc, P2, rr);
    }
    pcg_barrier(P);
    // stop test (identical in every CTA)
    if (tid == 0) s_any = 0;
    colsum_all(rr, nc, s_sum);
    if (tid < nc) {
      int a = s_act[tid];
      if (s_act[tid]) s_iters[tid]++;
      if (a && !P.fixed && P.stop == 0 && sqrt(s_sum[tid]) <= P.tol * s_r0[tid]) a = 0;
      s_new[tid] = a;
      if (a) atomicOr(&s_any, 1);
    }
    __syncthreads();
    ++it;
    if (P.fixed ? it >= P.fixed : (!s_any || it >= P.max_iter)) {
      if (tid < nc) s_act[tid] = s_new[tid];
      break;
    }
    apply_M_phases<NCP, STAGES, EXPL, CH>(P, smem, rz);  // z = M r
    double p_old = 0.0;
    if (myrow) p_old = P.p[jr];
    pcg_barrier(P);
    // beta, p
    const double zv = myrow ? P.z[jr] : 0.0;
    colsum_all(rz, nc, s_sum);
    if (P.stop == 1 && !P.fixed) {
      // preconditioned criterion, tested after the preconditioner (identical in every CTA)
      __syncthreads();
      if (tid == 0) s_any = 0;
      __syncthreads();
      if (tid < nc) {
        if (s_new[tid] && sqrt(fmax(s_sum[tid], 0.0)) <= P.tol * sqrt(s_rz0[tid])) s_new[tid] = 0;
        if (s_new[tid]) atomicOr(&s_any, 1);
      }
      __syncthreads();
      if (!s_any) {
        if (tid < nc) s_act[tid] = s_new[tid];
        break;
      }
    }
    if (tid < nc) {
      const double rzn = s_sum[tid];
      s_coef[tid] = rzn / s_rz[tid];
      if (s_new[tid]) {
        s_rz[tid] = rzn;
        if (blockIdx.x == 0 && s_iters[tid] - 1 < P.coef_ld) P.coef[(nc + tid) * P.coef_ld + s_iters[tid] - 1] = s_coef[tid];
      }
    }
    __syncthreads();
    if (fast1) {
      if (myrow) {
        double pv = p_old;
        if (s_new[0]) {
          pv = zv + s_coef[0] * pv;
          P.p[jr] = pv;
        }
        P.pslot[Lr.slot[0]] = (double)Lr.sign[0] * 1.0 * pv;
        P.pslot[Lr.slot[1]] = (double)Lr.sign[1] * 1.0 * pv;
      }
    } else {
      const bool act = cc < nc && s_new[cc];
      const double bta = cc < nc ? s_coef[cc] : 0.0;
      const int stride = nb * R;
      if (cc < nc)
        for (int j0 = blockIdx.x * R + rl; j0 < m; j0 += UR * stride) {
          double pv[UR], zv4[UR];
          LamDev L4[UR];
#pragma unroll
          for (int u = 0; u < UR; ++u) {
            const int j = j0 + u * stride;
            if (j < m) {
              const long long e = (long long)j * nc + cc;
              pv[u] = P.p[e];
              zv4[u] = P.z[e];
              L4[u] = P.lam[j];
            }
          }
#pragma unroll
          for (int u = 0; u < UR; ++u) {
            const int j = j0 + u * stride;
            if (j >= m) continue;
            const long long e = (long long)j * nc + cc;
            double p1 = pv[u];
            if (act) {
              p1 = zv4[u] + bta * p1;
              P.p[e] = p1;
            }
            P.pslot[(long long)L4[u].slot[0] * nc + cc] = (double)L4[u].sign[0] * 1.0 * p1;
            P.pslot[(long long)L4[u].slot[1] * nc + cc] = (double)L4[u].sign[1] * 1.0 * p1;
          }
        }
    }
    if (tid < nc) s_act[tid] = s_new[tid];
    pcg_barrier(P);
  }
  if constexpr (NCP == 16 && EXPL && CH) chunk_epilogue();
  if (blockIdx.x == 0 && tid == 0) {
    P.st->it = it;
    P.st->done = 1;
    P.st->ncols = nc;
    for (int c = 0; c < nc; ++c) {
      P.st->iters[c] = s_iters[c];
      P.st->active[c] = s_act[c];
      P.st->r0[c] = s_r0[c];
      P.st->rz[c] = s_rz[c];
    }
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
struct TmvCfg {
  int ncp, stages, smem;
};

// sym: the explicit loop's symmetric passes (row-segment items); else the block-pair
// items of the triangular operators
// big: a launch of its own without static shared memory (k_tmv) may use the whole 227 KB
static TmvCfg tmv_cfg(const ietidp_s* h, int ncols, bool sym = false, bool big = false) {
  const int nt = (h->plan.max_nI + TB - 1) / TB;
  const int npg = std::max(h->plan.nPmax, 16);  // staged coarse rows: TB x nP (at least 16)
  if (ncols == 1) {
    if (sym) {
      // row-segment items streamed through one ring (sym_stream): STAGES tiles and
      // STAGES input buffers of SYM_SEG + 1 blocks; two stages keep two CTAs per SM
      int st = 2;
      if (getenv("IETIDP_STAGES1")) {
        const int e = atoi(getenv("IETIDP_STAGES1"));
        st = (e == 3 || e == 5) ? e : 2;
      }
      return {1, st, (st * TILE_ELEMS + st * (SYM_SEG + 1) * TB + TB * npg) * 8};
    }
    // many work items: 3 stages (two CTAs per SM hide each other's barriers);
    // few (C2: 128 items): 5 stages, one deep-pipelined CTA per SM
    int st = h->n_loopwork >= 2 * 148 ? 3 : 5;
    if (getenv("IETIDP_STAGES1")) st = atoi(getenv("IETIDP_STAGES1")) == 5 ? 5 : 3;
    return {1, st, (st * TILE_ELEMS + nt * TB + TB + TB * npg) * 8};
  }
  for (int ncp : {16, 8}) {
    if (ncp == 16 && ncols <= 8) continue;
    const int vs = ncp + 4;
    for (int stages = 3; stages >= 2; --stages) {
      int bytes = sym ? (stages * TILE_ELEMS + stages * (SYM_SEG + 1) * TB * vs + TB * npg) * 8
                      : (stages * TILE_ELEMS + nt * TB * vs + TB * vs + TB * npg) * 8;
      if (bytes <= (big && !sym ? 226 : 210) * 1024) return {ncp, stages, bytes};
    }
  }
  throw Error(IETIDP_E_ARG, "interface block too large for the shared-memory loop kernels");
}

static TmvArgs sym_args(ietidp_s* h, const double* tiles, int ncols) {
  TmvArgs a{};
  a.work = h->d_loopwork.p;
  a.sub = h->d_sub.p;
  a.tiles = tiles;
  a.slot_lam = h->slot_lam.p;
  a.slot_sign = h->slot_sign.p;
  a.prim_gid = h->d_prim_gid.p;
  a.gmat = h->G.p;
  a.spart = h->spart.p;
  a.pboff = h->d_pboff.p;
  a.swork = h->d_symwork.p;
  a.maxseg = h->sym_maxseg;
  a.nPmax = std::max(h->plan.nPmax, 1);
  a.ncols = ncols;
  return a;
}

static CoarseTerm coarse_term_args(ietidp_s* h) {
  CoarseTerm ct{};
  if (h->n_primal == 0) return ct;
  ct.goff = h->slot_goff.p;
  ct.np = h->slot_np.p;
  ct.poff = h->slot_poff.p;
  ct.prim_gid = h->d_prim_gid.p;
  ct.G = h->G.p;
  ct.z = h->zc.p;
  return ct;
}

template <int MODE, int NCP, int STAGES>
static void launch_tmv_t(ietidp_s* h, const TmvCfg& cfg, TmvArgs a) {
  auto kern = k_tmv<MODE, NCP, STAGES>;
  IETI_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, cfg.smem));
  kern<<<h->n_loopwork, 256, cfg.smem, h->stream>>>(a);
  IETI_LAUNCHED(h);
}

template <int MODE>
static void launch_tmv(ietidp_s* h, TmvArgs a) {
  if (h->n_loopwork == 0) return;
  const TmvCfg cfg = tmv_cfg(h, a.ncols, false, true);  // C5: 16 columns in one pass (212 KB) instead of two of 8
  a.work = h->d_loopwork.p;
  a.sub = h->d_sub.p;
  a.tiles = (MODE == FWD || MODE == BWD) ? h->itiles.p : h->tiles.p;
  a.lpi = h->lpi.p;
  a.slot_lam = h->slot_lam.p;
  a.slot_sign = h->slot_sign.p;
  a.prim_gid = h->d_prim_gid.p;
  a.nPmax = std::max(h->plan.nPmax, 1);
  for (int c0 = 0; c0 < a.ncols; c0 += cfg.ncp) {
    a.c_off = c0;
    if (cfg.ncp == 1 && cfg.stages == 5) launch_tmv_t<MODE, 1, 5>(h, cfg, a);
    else if (cfg.ncp == 1) launch_tmv_t<MODE, 1, 3>(h, cfg, a);
    else if (cfg.ncp == 16 && cfg.stages == 3) launch_tmv_t<MODE, 16, 3>(h, cfg, a);
    else if (cfg.ncp == 16) launch_tmv_t<MODE, 16, 2>(h, cfg, a);
    else if (cfg.stages == 3) launch_tmv_t<MODE, 8, 3>(h, cfg, a);
    else launch_tmv_t<MODE, 8, 2>(h, cfg, a);
  }
}

static int tmv_launches(const ietidp_s* h, int ncols) {
  const TmvCfg cfg = tmv_cfg(h, ncols, false, true);
  return (ncols + cfg.ncp - 1) / cfg.ncp;
}

// ---- sharded mode (ietidp_shard.h) ----
// per-column partial dot products of two replicated multiplier-space vectors, in the layout
// of k_bgather's fused partials (partial[block * ncols + c], NBLK blocks)
__global__ void __launch_bounds__(VT) k_sh_dotpart(int m, int ncols, const double* __restrict__ a,
                                                   const double* __restrict__ b, double* __restrict__ partial,
                                                   const PcgState* __restrict__ st) {
  if (st && st->done) return;
  const int P2 = pow2ge(ncols);
  const int c = threadIdx.x % P2, rl = threadIdx.x / P2, R = VT / P2;
  double dot = 0.0;
  if (c < ncols)
    for (int j = blockIdx.x * R + rl; j < m; j += gridDim.x * R) dot += a[(long long)j * ncols + c] * b[(long long)j * ncols + c];
  block_col_reduce(dot, ncols, P2, partial);
}
// g[gi][c] = (add +) sum of the coarse partial rows of the local subdomains, one thread per
// entry over the whole grid (k_coarse does this part in one CTA: 340 us for C5's 177 x 16)
__global__ void __launch_bounds__(256)
    k_sh_gsum(int ng, int ncols, int nPmax, const int* __restrict__ pcon_ptr, const int* __restrict__ pcon_sub,
              const int* __restrict__ pcon_q, const int* __restrict__ sub_cta0, const int* __restrict__ sub_ncta,
              const double* __restrict__ gpart, const double* __restrict__ add, double* __restrict__ g,
              const PcgState* __restrict__ st) {
  if (st && st->done) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ng * ncols; e += gridDim.x * blockDim.x) {
    const int gi = e / ncols, c = e - gi * ncols;
    double s = add ? add[e] : 0.0;
    for (int q = pcon_ptr[gi]; q < pcon_ptr[gi + 1]; ++q) {
      const int k = pcon_sub[q], lq = pcon_q[q];
      for (int cta = sub_cta0[k]; cta < sub_cta0[k] + sub_ncta[k]; ++cta)
        s += gpart[((long long)cta * nPmax + lq) * ncols + c];
    }
    g[e] = s;
  }
}
// z = S^-1 (add + g), a warp per entry
__global__ void __launch_bounds__(256) k_sh_coarse_solve(int ng, int ncols, const double* __restrict__ Sinv,
                                                        const double* __restrict__ g, const double* __restrict__ add,
                                                        double* __restrict__ z, const PcgState* __restrict__ st) {
  if (st && st->done) return;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = warp; e < ng * ncols; e += nw) {
    const int i = e / ncols, c = e - i * ncols;
    double s = 0.0;
    for (int j = lane; j < ng; j += 32)
      s += Sinv[(long long)i * ng + j] * (g[j * ncols + c] + (add ? add[j * ncols + c] : 0.0));
    s = warp_sum(s);
    if (lane == 0) z[e] = s;
  }
}
// after a local gather into the multiplier space: sum over the ranks, then the dot partials
static void sh_finish_gather(ietidp_s* h, int ncols, double* out, const double* dotv, double* partial, const PcgState* st) {
  sh_sum(h, out, (long long)h->n_lambda * ncols);
  if (dotv && partial) {
    k_sh_dotpart<<<NBLK, VT, 0, h->stream>>>(h->n_lambda, ncols, out, dotv, partial, st);
    IETI_LAUNCHED(h);
  }
}

// y_k = L_II^-1 B_I^T v (per slot) and the coarse partials L_PI y_k
void loop_fwd(ietidp_s* h, int ncols, const double* v, double* y, bool partials, const void* stv) {
  const PcgState* st = static_cast<const PcgState*>(stv);
  TmvArgs a{};
  a.vin = v;
  a.vout = y;
  a.gpart = (partials && h->n_primal) ? h->gpart.p : nullptr;
  a.ncols = ncols;
  a.st = st;
  launch_tmv<FWD>(h, a);
}
// x_k = L_II^-T (y_k + zsign L_PI^T z_k)
void loop_bwd(ietidp_s* h, int ncols, const double* y, const double* z, double zsign, double* x, const void* stv) {
  const PcgState* st = static_cast<const PcgState*>(stv);
  TmvArgs a{};
  a.vin = y;
  a.z = h->n_primal ? z : nullptr;
  a.zsign = zsign;
  a.vout = x;
  a.ncols = ncols;
  a.st = st;
  launch_tmv<BWD>(h, a);
}

void bgather(ietidp_s* h, int ncols, const double* x, const double* weight, double* out, const double* dotv,
             double* partial, const void* stv) {
  const PcgState* st = static_cast<const PcgState*>(stv);
  if (h->n_lambda == 0) return;
  if (h->shard) {
    k_bgather<<<NBLK, VT, 0, h->stream>>>(h->n_lambda, ncols, h->lam.p, x, weight, out, nullptr, nullptr, st,
                                          CoarseTerm{});
    IETI_LAUNCHED(h);
    sh_finish_gather(h, ncols, out, dotv, partial, st);
    return;
  }
  k_bgather<<<NBLK, VT, 0, h->stream>>>(h->n_lambda, ncols, h->lam.p, x, weight, out, dotv, partial, st,
                                        CoarseTerm{});
  IETI_LAUNCHED(h);
}

// z = S^-1 (add + sum of the coarse partials)
void coarse_apply(ietidp_s* h, int ncols, const double* add, double* z, const void* stv, bool sym_rows = false) {
  const PcgState* st = static_cast<const PcgState*>(stv);
  if (h->n_primal == 0) return;
  // coarse partial rows per subdomain: (subdomain, block) rows of the symmetric pass, or
  // the block-pair items of the triangular operators
  const int* r0 = sym_rows ? h->sub_blk0.p : h->sub_cta0.p;
  const int* rn = sym_rows ? h->sub_nt.p : h->sub_ncta.p;
  // g over the whole grid, then z = S_PP^-1 g with a warp per entry (the same sums, in the same
  // order, as the one-CTA k_coarse; IETIDP_COARSE_1CTA=1 forces that kernel). Sharded: g is
  // summed over the ranks in between (S_PP^-1 is replicated), `add` after it.
  // (with few entries -- one RHS -- the single launch is quicker: C2 43 vs 51 us per F-apply)
  static const bool force_1cta = getenv("IETIDP_COARSE_1CTA") && atoi(getenv("IETIDP_COARSE_1CTA")) == 1;
  const bool one_cta = force_1cta || (long long)h->n_primal * ncols < 1024;
  if (h->shard || !one_cta) {
    k_sh_gsum<<<grid_for((long long)h->n_primal * ncols, 256), 256, 0, h->stream>>>(
        h->n_primal, ncols, std::max(h->plan.nPmax, 1), h->pcon_ptr.p, h->pcon_sub.p, h->pcon_q.p, r0, rn, h->gpart.p,
        h->shard ? nullptr : add, h->gc.p, st);
    IETI_LAUNCHED(h);
    sh_sum(h, h->gc.p, (long long)h->n_primal * ncols);
    k_sh_coarse_solve<<<grid_for((long long)h->n_primal * ncols * 32, 256), 256, 0, h->stream>>>(
        h->n_primal, ncols, h->Sinv.p, h->gc.p, h->shard ? add : nullptr, z, st);
    IETI_LAUNCHED(h);
    return;
  }
  const int smem = h->n_primal * ncols * 8;
  if (smem > 48 * 1024)
    IETI_CUDA(cudaFuncSetAttribute((const void*)k_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_coarse<<<1, 1024, smem, h->stream>>>(h->n_primal, ncols, std::max(h->plan.nPmax, 1), h->pcon_ptr.p,
                                         h->pcon_sub.p, h->pcon_q.p, r0, rn, h->gpart.p, add,
                                         h->Sinv.p, z, st);
  IETI_LAUNCHED(h);
}

// Work items over `grid` resident CTAs: longest processing time first (ptr/items lists).
static void lpt_lists(const ietidp_s* h, int grid, std::vector<int>& ptr, std::vector<int>& items) {
  const bool expl = h->opt.loop == IETIDP_LOOP_EXPLICIT;  // items: row segments, or block pairs
  const int nitems = expl ? h->n_symwork : h->n_loopwork;
  std::vector<std::pair<int, int>> cost(nitems);
  for (int i = 0; i < nitems; ++i) cost[i] = {expl ? h->h_symwork[i].cost : h->h_loopwork[i].cost, i};
  std::sort(cost.begin(), cost.end(), [](auto& x, auto& y) { return x.first > y.first || (x.first == y.first && x.second < y.second); });
  std::vector<std::vector<int>> lists(grid);
  std::vector<std::pair<long long, int>> heap;
  for (int b = 0; b < grid; ++b) heap.push_back({0, b});
  auto cmp = [](auto& x, auto& y) { return x.first > y.first || (x.first == y.first && x.second > y.second); };
  std::make_heap(heap.begin(), heap.end(), cmp);
  for (auto& c : cost) {
    std::pop_heap(heap.begin(), heap.end(), cmp);
    heap.back().first += c.first;
    lists[heap.back().second].push_back(c.second);
    std::push_heap(heap.begin(), heap.end(), cmp);
  }
  ptr.assign(grid + 1, 0);
  items.clear();
  for (int b = 0; b < grid; ++b) {
    items.insert(items.end(), lists[b].begin(), lists[b].end());
    ptr[b + 1] = (int)items.size();
  }
}

// IETIDP_SYM_STREAM=0: one CTA per item (round 1's launch) instead of the streamed pass
static bool sym_stream_enabled() {
  static const bool on = !(getenv("IETIDP_SYM_STREAM") && atoi(getenv("IETIDP_SYM_STREAM")) == 0);
  return on;
}

// out[slot][c] = sign * weight * x[multiplier of the slot][c]: B^T x (or B_D^T x) in slot order,
// the input form of the streamed pass
__global__ void __launch_bounds__(256) k_to_slots(long long n_slots, int ncols, const int* __restrict__ slot_lam,
                                                  const float* __restrict__ slot_sign, const double* __restrict__ weight,
                                                  const double* __restrict__ x, double* __restrict__ out,
                                                  const PcgState* __restrict__ st) {
  if (st && st->done) return;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n_slots * ncols;
       e += (long long)gridDim.x * blockDim.x) {
    const long long a = e / ncols;
    const int c = (int)(e - a * ncols);
    out[e] = (double)slot_sign[a] * (weight ? weight[a] : 1.0) * x[(long long)slot_lam[a] * ncols + c];
  }
}

template <int NCP, int STAGES>
static void launch_sym_t(ietidp_s* h, const TmvCfg& cfg, TmvArgs a) {
  if (a.slot_in && sym_stream_enabled() && h->opt.loop == IETIDP_LOOP_EXPLICIT) {
    auto kern = k_sym_stream<NCP, STAGES>;
    IETI_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, cfg.smem));
    int per_sm = 0, nsm = 0;
    IETI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, cfg.smem));
    IETI_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->opt.device));
    if (per_sm >= 1) {
      const int grid = std::min(nsm * per_sm, 1024);
      if (h->lpt2_grid != grid) {
        std::vector<int> ptr, items;
        lpt_lists(h, grid, ptr, items);
        h->cta_ptr2.upload(ptr, h->stream);
        h->cta_items2.upload(items, h->stream);
        IETI_CUDA(cudaStreamSynchronize(h->stream));  // the host vectors go out of scope
        h->lpt2_grid = grid;
      }
      kern<<<grid, 256, cfg.smem, h->stream>>>(a, h->cta_ptr2.p, h->cta_items2.p);
      IETI_LAUNCHED(h);
      return;
    }
  }
  auto kern = k_sym<NCP, STAGES>;
  IETI_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, cfg.smem));
  kern<<<h->n_symwork, 256, cfg.smem, h->stream>>>(a);
  IETI_LAUNCHED(h);
}

// y = S x for the symmetric tile matrix `tiles` (explicit loop), into the slot vector a.vout
static void sym_apply(ietidp_s* h, TmvArgs a) {
  if (h->n_symwork == 0) return;
  const TmvCfg cfg = tmv_cfg(h, a.ncols, true);
  if (!a.slot_in && sym_stream_enabled() && h->n_slots > 0) {  // the streamed pass reads slot order
    if (h->pslot.n < (size_t)h->n_slots * h->nrhs) {
      h->pslot.alloc((size_t)h->n_slots * h->nrhs);
      h->rslot.alloc((size_t)h->n_slots * h->nrhs);
    }
    k_to_slots<<<grid_for((long long)h->n_slots * a.ncols, 256), 256, 0, h->stream>>>(
        h->n_slots, a.ncols, h->slot_lam.p, h->slot_sign.p, a.weight, a.vin, h->pslot.p, a.st);
    IETI_LAUNCHED(h);
    a.vin = h->pslot.p;
    a.slot_in = 1;
    a.weight = nullptr;
  }
  for (int c0 = 0; c0 < a.ncols; c0 += cfg.ncp) {
    a.c_off = c0;
    if (cfg.ncp == 1 && cfg.stages == 2) launch_sym_t<1, 2>(h, cfg, a);
    else if (cfg.ncp == 1 && cfg.stages == 5) launch_sym_t<1, 5>(h, cfg, a);
    else if (cfg.ncp == 1) launch_sym_t<1, 3>(h, cfg, a);
    else if (cfg.ncp == 16 && cfg.stages == 3) launch_sym_t<16, 3>(h, cfg, a);
    else if (cfg.ncp == 16) launch_sym_t<16, 2>(h, cfg, a);
    else if (cfg.stages == 3) launch_sym_t<8, 3>(h, cfg, a);
    else launch_sym_t<8, 2>(h, cfg, a);
  }
  a.c_off = 0;
  if (h->n_blk) {
    k_sym_reduce<<<h->n_blk, 256, 0, h->stream>>>(a, h->d_blk.p);
    IETI_LAUNCHED(h);
  }
}

// y = F_DP x (interleaved, ncols columns)
static void apply_F_inter(ietidp_s* h, int ncols, const double* x, double* y, const PcgState* st, const double* dotv,
                          double* partial) {
  if (h->n_lambda == 0) return;
  if (h->opt.loop == IETIDP_LOOP_EXPLICIT) {
    TmvArgs a = sym_args(h, h->wtiles.p, ncols);
    a.vin = x;
    a.vout = h->xI.p;
    a.gpart = h->n_primal ? h->gpart.p : nullptr;
    sym_apply(h, a);
    coarse_apply(h, ncols, nullptr, h->zc.p, st, true);
    CoarseTerm ct = coarse_term_args(h);
    if (h->shard) {
      k_bgather<<<NBLK, VT, 0, h->stream>>>(h->n_lambda, ncols, h->lam.p, h->xI.p, nullptr, y, nullptr, nullptr, st, ct);
      IETI_LAUNCHED(h);
      sh_finish_gather(h, ncols, y, dotv, partial, st);
      return;
    }
    k_bgather<<<NBLK, VT, 0, h->stream>>>(h->n_lambda, ncols, h->lam.p, h->xI.p, nullptr, y, dotv, partial, st, ct);
    IETI_LAUNCHED(h);
    return;
  }
  loop_fwd(h, ncols, x, h->yI.p, true, st);
  coarse_apply(h, ncols, nullptr, h->zc.p, st);
  loop_bwd(h, ncols, h->yI.p, h->zc.p, 1.0, h->xI.p, st);
  bgather(h, ncols, h->xI.p, nullptr, y, dotv, partial, st);
}

// y = M_D^-1 x
static void apply_M_inter(ietidp_s* h, int ncols, const double* x, double* y, const PcgState* st, const double* rr_part,
                          int check, const double* dotv, double* partial) {
  if (h->n_lambda == 0) return;
  if (h->opt.loop == IETIDP_LOOP_EXPLICIT) {
    TmvArgs a = sym_args(h, h->stiles.p, ncols);
    a.vin = x;
    a.weight = h->delta.p;
    a.vout = h->zI.p;
    sym_apply(h, a);
    bgather(h, ncols, h->zI.p, h->delta.p, y, dotv, partial, st);
    return;
  }
  TmvArgs a{};
  a.vin = x;
  a.weight = h->delta.p;
  a.vout = h->sI.p;
  a.ncols = ncols;
  a.st = st;
  a.rr_part = rr_part;
  a.check = check;
  launch_tmv<PRE1>(h, a);
  TmvArgs b{};
  b.vin = h->sI.p;
  b.vout = h->zI.p;
  b.ncols = ncols;
  b.st = st;
  launch_tmv<PRE2>(h, b);
  bgather(h, ncols, h->zI.p, h->delta.p, y, dotv, partial, st);
}

static bool apply_F_chunk(ietidp_s* h, int ncols, const double* x, double* y);  // below (needs the chunk kernels)
void run_apply_F(ietidp_s* h, int ncols, const double* x, double* y) {
  if (!apply_F_chunk(h, ncols, x, y)) apply_F_inter(h, ncols, x, y, nullptr, nullptr, nullptr);
  IETI_CHECK_LAUNCH();
}
void run_apply_M(ietidp_s* h, int ncols, const double* x, double* y) {
  apply_M_inter(h, ncols, x, y, nullptr, nullptr, 0, nullptr, nullptr);
  IETI_CHECK_LAUNCH();
}

static int body_launches(ietidp_s* h, int ncols) {
  if (h->opt.loop == IETIDP_LOOP_EXPLICIT)  // per pass: slot order, pass, reduction, gather; coarse g and z; 3 CG kernels
    return 2 * (tmv_launches(h, ncols) + 3) + (h->n_primal ? 2 : 0) + 3;
  return 4 * tmv_launches(h, ncols) + (h->n_primal ? 2 : 0) + 2 + 3;
}

static void iteration_body(ietidp_s* h, PcgState* st, int use_graph) {
  const int nc = h->nrhs, m = h->n_lambda;
  double* pq_part = h->partial.p;
  double* rr_part = h->partial.p + NBLK * nc;
  double* rz_part = h->partial.p + 2 * NBLK * nc;
  apply_F_inter(h, nc, h->p_vec.p, h->q_vec.p, st, h->p_vec.p, pq_part);
  k_cg_alpha<<<NBLK, VT, 0, h->stream>>>(m, st, pq_part, h->lam_vec.p, h->r_vec.p, h->p_vec.p, h->q_vec.p, rr_part,
                                        h->cgcoef.p, h->coef_ld);
  IETI_LAUNCHED(h);
  apply_M_inter(h, nc, h->r_vec.p, h->z_vec.p, st, rr_part, 1, h->r_vec.p, rz_part);
  k_cg_beta<<<NBLK, VT, 0, h->stream>>>(m, st, rr_part, rz_part, h->p_vec.p, h->z_vec.p, h->cgcoef.p, h->coef_ld);
  IETI_LAUNCHED(h);
  k_ctl<<<1, 64, 0, h->stream>>>(st, rr_part, rz_part, (unsigned long long)h->cond_handle, use_graph);
  IETI_LAUNCHED(h);
}

static void build_graph(ietidp_s* h, PcgState* st) {
  if (h->graph_exec) return;
  // set the kernels' shared-memory attributes outside the capture
  (void)tmv_cfg(h, h->nrhs);
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
}

void destroy_graph(ietidp_s* h) {
  if (h->graph_exec) cudaGraphExecDestroy((cudaGraphExec_t)h->graph_exec);
  if (h->graph) cudaGraphDestroy((cudaGraph_t)h->graph);
  h->graph_exec = h->graph = nullptr;
}

static TmvArgs base_args(ietidp_s* h, int mode, int ncols) {
  TmvArgs a{};
  a.work = h->d_loopwork.p;
  a.sub = h->d_sub.p;
  a.tiles = (mode == FWD || mode == BWD) ? h->itiles.p : h->tiles.p;
  a.lpi = h->lpi.p;
  a.slot_lam = h->slot_lam.p;
  a.slot_sign = h->slot_sign.p;
  a.prim_gid = h->d_prim_gid.p;
  a.nPmax = std::max(h->plan.nPmax, 1);
  a.ncols = ncols;
  return a;
}

__global__ void k_wrec(int m, const LamDev* __restrict__ lam, const double* __restrict__ delta,
                       double* __restrict__ wrec) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m) {
    wrec[2 * j] = delta[lam[j].slot[0]];
    wrec[2 * j + 1] = delta[lam[j].slot[1]];
  }
}

// Plan of the chunk pass for `grid` CTAs: the tiles of all subdomains in order (lower
// row-major within a subdomain; weight 1 for a diagonal tile, which has only the row
// product, 2 otherwise) cut into `grid` contiguous ranges of equal weight; a range
// splits into one chunk per subdomain it touches.
static void plan_chunks(ietidp_s* h, int grid, int nc) {
  const int ns = h->n_sub;
  long long W = 0;
  for (int k = 0; k < ns; ++k) {
    const long long nt = h->h_sub[k].nt;
    W += nt * nt;  // nt diagonal tiles (1) + nt(nt-1)/2 off-diagonal (2)
  }
  std::vector<std::vector<SymChunk>> lists(grid);
  std::vector<int> nchunk(ns, 0);
  std::vector<std::vector<std::pair<int, int>>> sub_chunks(ns);  // (t0, t1) per rank
  long long cum = 0;
  int b = 0;
  for (int k = 0; k < ns; ++k) {
    const SubDev& d = h->h_sub[k];
    const int T = d.nt * (d.nt + 1) / 2;
    bool open = false;
    for (int t = 0, o = 0, j = 0; t < T; ++t) {
      if (!open) {
        lists[b].push_back({k, t, t, nchunk[k]++, d.tile_off / TILE_ELEMS + t});
        sub_chunks[k].push_back({t, t});
        open = true;
      }
      lists[b].back().t1 = t + 1;
      sub_chunks[k].back().second = t + 1;
      cum += (j == o) ? 1 : 2;
      if (b < grid - 1 && cum * grid >= W * (b + 1)) {
        ++b;
        open = false;
      }
      if (++j > o) {
        ++o;
        j = 0;
      }
    }
  }
  std::vector<int> ptr(grid + 1, 0);
  std::vector<SymChunk> all;
  for (int c = 0; c < grid; ++c) {
    all.insert(all.end(), lists[c].begin(), lists[c].end());
    ptr[c + 1] = (int)all.size();
  }
  auto row_of = [](int t) {
    int o = 0;
    while ((o + 1) * (o + 2) / 2 <= t) ++o;
    return o;
  };
  std::vector<long long> cpb;
  std::vector<int> cfirst;
  std::vector<SlotRed> sred(std::max(h->n_slots, 1));
  long long pb = 0;
  for (int k = 0; k < ns; ++k) {
    const SubDev& d = h->h_sub[k];
    const int C = (int)sub_chunks[k].size();
    std::vector<int> cnt(d.nt);
    for (int j = 0; j < d.nt; ++j) {
      int cf = C;
      for (int c = 0; c < C; ++c)
        if (row_of(sub_chunks[k][c].second - 1) >= j) {
          cf = c;
          break;
        }
      cfirst.push_back(cf);
      cpb.push_back(pb);
      cnt[j] = C - cf;
      pb += cnt[j];
    }
    for (int a = 0; a < d.nI; ++a) {
      const int j = a / TB;
      sred[d.rI_off + a] = {cpb[d.blk0 + j] * TB + a % TB, cnt[j], 0};
    }
  }
  h->chunk_ptr.upload(ptr, h->stream);
  h->chunk_list.upload(all, h->stream);
  h->chunk_cpb.upload(cpb, h->stream);
  h->chunk_cfirst.upload(cfirst, h->stream);
  h->chunk_slot_red.upload(sred, h->stream);
  std::vector<GatherRec> grec(std::max(h->n_lambda, 1));
  for (int j = 0; j < h->n_lambda; ++j) {
    const LamDev& L = h->h_lam[j];
    for (int q = 0; q < 2; ++q) {
      grec[j].base[q] = sred[L.slot[q]].base;
      grec[j].cnt[q] = sred[L.slot[q]].cnt;
      grec[j].sign[q] = L.sign[q];
      grec[j].slot[q] = L.slot[q];
    }
  }
  h->chunk_grec.upload(grec, h->stream);
  h->chunk_wrec.alloc(2 * (size_t)std::max(h->n_lambda, 1));
  h->chunk_spart.alloc((size_t)std::max(pb, 1LL) * TB * nc);
  h->chunk_grid = grid;
}

// run_solve_persistent in "prepare only" mode (the sharded chunk loop): launch_pcg_t fills the
// kernel arguments and plans, hands them out here and does not launch
struct PrepareOnly {
  PcgArgs* out = nullptr;
  int grid = 0, smem = 0, stages = 0;
  bool chunk = false;
};
static thread_local PrepareOnly g_prepare;  // per host thread: handles may be driven concurrently

template <int NCP, int STAGES, bool EXPL, bool CH = false>
static bool launch_pcg_t(ietidp_s* h, const TmvCfg& cfg, const PcgArgs& a) {
  auto kern = k_pcg<NCP, STAGES, EXPL, CH>;
  IETI_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, cfg.smem));
  int per_sm = 0, nsm = 0;
  IETI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, cfg.smem));
  IETI_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->opt.device));
  if (per_sm < 1) return false;
  const int grid = std::min(nsm * per_sm, 1024);
  if (h->lpt_grid != grid) {  // items over the persistent CTAs: longest processing time first
    std::vector<int> ptr, items;
    lpt_lists(h, grid, ptr, items);
    h->cta_ptr.upload(ptr, h->stream);
    h->cta_items.upload(items, h->stream);
    h->lpt_grid = grid;
  }
  PcgArgs args = a;
  args.cta_ptr = h->cta_ptr.p;
  args.cta_items = h->cta_items.p;
  if (args.chunk) {
    if (h->chunk_grid != grid) plan_chunks(h, grid, args.ncols);
    args.chunk_ptr = h->chunk_ptr.p;
    args.chunk_list = h->chunk_list.p;
    for (TmvArgs* t : {&args.wsym, &args.ssym}) {
      t->nt_max = (h->plan.max_nI + TB - 1) / TB;
      t->spart = h->chunk_spart.p;
      t->cpb = h->chunk_cpb.p;
      t->cfirst = h->chunk_cfirst.p;
    }
    args.slot_red = h->chunk_slot_red.p;
    args.smem_doubles = cfg.smem / 8;
    args.grec = h->chunk_grec.p;
    args.wrec = h->chunk_wrec.p;
    if (h->chunk_gzv.n < (size_t)h->n_slots * args.ncols) h->chunk_gzv.alloc(std::max<size_t>(1, (size_t)h->n_slots * args.ncols));
    args.gzv = h->chunk_gzv.p;
    args.wsym.n_sub = args.ssym.n_sub = h->n_sub;
    if (h->n_lambda)  // the two slots' scaling weights per multiplier row (delta: set by the factorisation)
      k_wrec<<<grid_for(h->n_lambda, 256), 256, 0, h->stream>>>(h->n_lambda, h->lam.p, h->delta.p, h->chunk_wrec.p);
    IETI_LAUNCHED(h);
    args.fold = 1;
    args.fold_multi = 1;  // the gathers sum the (few) chunk partials of each slot
  }
  if (g_prepare.out) {  // sharded loop: the arguments and the launch shape, no launch
    *g_prepare.out = args;
    g_prepare.grid = grid;
    g_prepare.smem = cfg.smem;
    g_prepare.stages = STAGES;
    g_prepare.chunk = CH && args.chunk;
    return true;
  }
  const char* prof_env = getenv("IETIDP_PCG_PROF");
  DevBuf<unsigned long long>& prof = h->pcg_prof;  // per handle, on the handle's device
  if (prof_env) {
    if (!prof.p) prof.alloc(4096);
    const int zero = 0;
    IETI_CUDA(cudaMemcpyToSymbolAsync(g_prof_n, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, h->stream));
    args.prof = prof.p;
  }
  if (args.wsym.tl) IETI_CUDA(cudaMemsetAsync(args.wsym.tl, 0, 4096 * sizeof(unsigned long long), h->stream));
  void* params[] = {&args};
  IETI_CUDA(cudaLaunchCooperativeKernel((const void*)kern, grid, 256, params, cfg.smem, h->stream));
  IETI_LAUNCHED(h);
  if (args.wsym.tl) {
    std::vector<unsigned long long> t(4096);
    IETI_CUDA(cudaStreamSynchronize(h->stream));
    IETI_CUDA(cudaMemcpy(t.data(), args.wsym.tl, sizeof(unsigned long long) * 4096, cudaMemcpyDeviceToHost));
    static const char* ev[] = {"pass", "xstaged", "tile", "loopend", "synced", "end"};
    for (int k = 0; k < 2048 && t[2 * k]; ++k) {
      const unsigned long long c = t[2 * k + 1];
      fprintf(stderr, "tl %8.3f us %-8s %4u %4u\n", (t[2 * k] - t[0]) * 1e-3, ev[(c >> 32) & 7],
              (unsigned)((c >> 16) & 0xffff), (unsigned)(c & 0xffff));
    }
  }
  if (prof_env) {
    // per-barrier intervals of CTA 0, averaged by position in the iteration (diagnostics)
    std::vector<unsigned long long> t(4096);
    int n = 0;
    IETI_CUDA(cudaStreamSynchronize(h->stream));
    IETI_CUDA(cudaMemcpyFromSymbol(&n, g_prof_n, sizeof(int)));
    IETI_CUDA(cudaMemcpy(t.data(), prof.p, sizeof(unsigned long long) * std::min(n, 4096), cudaMemcpyDeviceToHost));
    n = std::min(n, 4096);
    const int ng_ = h->n_primal, nc = a.fwd.ncols ? a.fwd.ncols : h->nrhs;
    const bool nofold = (nc > 1 && !args.fold_multi) || !args.fold;
    const int per = args.chunk ? (ng_ > 0 ? 8 : 6)
                    : EXPL ? 6 + (nofold ? 2 : 0) + (ng_ > COARSE_LOCAL_MAX ? 1 + (nofold ? 0 : 1) : 0) : 9,
              skip = EXPL ? 4 + (nofold ? 1 : 0) : 5;
    std::vector<double> acc(per, 0.0);
    int cnt = 0;
    for (int i = skip; i + per < n; i += per, ++cnt)
      for (int q = 0; q < per; ++q) acc[q] += (double)(t[i + q + 1] - t[i + q]) * 1e-3;
    fprintf(stderr, "pcg profile: %d barriers, grid %d; us per phase (avg over %d iterations):", n, grid, cnt);
    for (int q = 0; q < per; ++q) fprintf(stderr, " %.2f", cnt ? acc[q] / cnt : 0.0);
    fprintf(stderr, "\n");
  }
  return true;
}

// The whole PCG loop as one persistent cooperative kernel.
static bool run_solve_persistent(ietidp_s* h) {
  const int nc = h->nrhs, m = h->n_lambda;
  if (m == 0 || h->n_loopwork == 0) return false;
  TmvCfg cfg = tmv_cfg(h, nc, h->opt.loop == IETIDP_LOOP_EXPLICIT);
  // the explicit loop's per-CTA coarse solve keeps g and z (2 ng nc doubles) in shared memory
  const int zbytes = 2 * h->n_primal * nc * (int)sizeof(double);
  if (h->opt.loop == IETIDP_LOOP_EXPLICIT && zbytes > cfg.smem) {
    if (zbytes > 200 * 1024) return false;
    cfg.smem = zbytes;
  }
  if (h->gbar.n == 0) h->gbar.alloc(2);
  h->gbar.zero(h->stream);
  PcgArgs a{};
  if (h->pslot.n == 0) {
    h->pslot.alloc((size_t)std::max(h->n_slots, 1) * nc);
    h->rslot.alloc((size_t)std::max(h->n_slots, 1) * nc);
  }
  a.pslot = h->pslot.p;  // B^T p in slot order, written by the CG vector phases
  a.rslot = h->rslot.p;  // B_D^T r in slot order
  a.fwd = base_args(h, FWD, nc);
  a.fwd.vin = a.pslot;
  a.fwd.slot_in = 1;
  a.fwd.vout = h->yI.p;
  a.fwd.gpart = h->n_primal ? h->gpart.p : nullptr;
  a.bwd = base_args(h, BWD, nc);
  a.bwd.vin = h->yI.p;
  a.bwd.z = h->n_primal ? h->zc.p : nullptr;
  a.bwd.zsign = 1.0;
  a.bwd.vout = h->xI.p;
  a.pre1 = base_args(h, PRE1, nc);
  a.pre1.vin = a.rslot;
  a.pre1.slot_in = 1;
  a.pre1.vout = h->sI.p;
  a.pre2 = base_args(h, PRE2, nc);
  a.pre2.vin = h->sI.p;
  a.pre2.vout = h->zI.p;
  a.wsym = sym_args(h, h->wtiles.p, nc);
  a.wsym.vin = a.pslot;
  a.wsym.slot_in = 1;
  a.wsym.vout = h->xI.p;
  a.wsym.gpart = h->n_primal ? h->gpart.p : nullptr;
  a.ssym = sym_args(h, h->stiles.p, nc);
  {
    // one RHS with S_II's tiles smaller than ~2/3 of the L2: keep them resident across
    // iterations (evict_last) and stream W_k's past them (evict_first)
    const double sbytes = (double)h->stiles.n * sizeof(double);
    int l2 = 0;
    IETI_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->opt.device));
    const double keep_frac = getenv("IETIDP_L2KEEP") ? atof(getenv("IETIDP_L2KEEP")) : 0.66;
    const bool keep = nc == 1 && sbytes < keep_frac * l2 && !(getenv("IETIDP_L2HINT") && atoi(getenv("IETIDP_L2HINT")) == 0);
    a.ssym.l2hint = keep ? 1 : 0;
    a.wsym.l2hint = keep ? 2 : 0;
    // several RHS: both operators' tiles streamed with evict_first so that more of the
    // symmetric-pass partials stay in the L2 for the reduction (C5 PCG 118.8 -> 117.2 ms,
    // bit-identical; IETIDP_L2MULTI=0 turns it off)
    if (nc > 1 && !(getenv("IETIDP_L2MULTI") && atoi(getenv("IETIDP_L2MULTI")) == 0))
      a.ssym.l2hint = a.wsym.l2hint = 2;
  }
  a.ssym.vin = a.rslot;
  a.ssym.slot_in = 1;
  a.ssym.vout = h->zI.p;
  a.ct = coarse_term_args(h);
  a.slot_red = h->slot_red.p;
  a.gsrc_ptr = h->gsrc_ptr.p;
  a.gsrc = h->gsrc.p;
  a.gc = h->gc.p;
  a.n_slots = h->n_slots;
  a.fold = !(getenv("IETIDP_FOLD") && atoi(getenv("IETIDP_FOLD")) == 0);
  a.wsym.dbg = a.ssym.dbg = getenv("IETIDP_DBG_PASS") ? atoi(getenv("IETIDP_DBG_PASS")) : 0;
  if (getenv("IETIDP_DBG_TL")) {  // diagnostics: CTA 0's timeline of two passes (stderr after the solve)
    if (!h->dbg_tl.p) h->dbg_tl.alloc(4096);
    a.wsym.tl = a.ssym.tl = h->dbg_tl.p;
  }
  a.fold_multi = getenv("IETIDP_FOLD_MULTI") && atoi(getenv("IETIDP_FOLD_MULTI")) == 1;
  a.blk = h->d_blk.p;
  a.n_blk = h->n_blk;
  a.lam = h->lam.p;
  a.delta = h->delta.p;
  a.lamv = h->lam_vec.p;
  a.r = h->r_vec.p;
  a.p = h->p_vec.p;
  a.q = h->q_vec.p;
  a.z = h->z_vec.p;
  a.d = h->d_vec.p;
  a.xI = h->xI.p;
  a.zI = h->zI.p;
  a.pcon_ptr = h->pcon_ptr.p;
  a.pcon_sub = h->pcon_sub.p;
  a.pcon_q = h->pcon_q.p;
  a.sub_cta0 = h->sub_cta0.p;
  a.sub_ncta = h->sub_ncta.p;
  a.gpart = h->gpart.p;
  a.Sinv = h->Sinv.p;
  a.zc = h->zc.p;
  a.part = h->partial.p;
  a.st = reinterpret_cast<PcgState*>(h->state.p);
  a.bar = h->gbar.p;
  a.tol = h->opt.tol;
  a.m = m;
  a.ncols = nc;
  a.ng = h->n_primal;
  a.nPmax = std::max(h->plan.nPmax, 1);
  a.max_iter = h->opt.max_iter;
  a.fixed = h->opt.fixed_iters;
  a.stop = h->opt.stop;
  a.coef = h->cgcoef.p;
  a.coef_ld = h->coef_ld;
  a.n_items = h->opt.loop == IETIDP_LOOP_EXPLICIT ? h->n_symwork : h->n_loopwork;
  a.ncp = cfg.ncp;
  {
    // several RHS: the chunk pass (tensor-memory accumulators, bulk-copied tile stream;
    // IETIDP_CHUNK=0 selects the row-segment pass)
    const int nt = (h->plan.max_nI + TB - 1) / TB;
    const bool want = h->opt.loop == IETIDP_LOOP_EXPLICIT && cfg.ncp == 16 && nt <= 32 &&
                      !(getenv("IETIDP_CHUNK") && atoi(getenv("IETIDP_CHUNK")) == 0);
    if (want) {
      const int gsz = TB * std::max(h->plan.nPmax, 1);  // staged G_k rows
      int stages = 3;
      int bytes = (stages * TILE_ELEMS + nt * CH_XBLK + gsz) * 8;
      if (bytes > 210 * 1024) {
        stages = 2;
        bytes = (stages * TILE_ELEMS + nt * CH_XBLK + gsz) * 8;
      }
      const int npm = std::max(h->plan.nPmax, 1);
      const int gz = (h->n_primal * nc + npm * h->n_primal + npm * nc + TB * npm) * (int)sizeof(double);
      if (bytes <= 210 * 1024 && bytes >= gz) {
        a.chunk = 1;
        cfg.stages = stages;
        cfg.smem = bytes;
      }
    }
  }
  if (h->n_primal * nc * 8 > cfg.smem) return false;
  if (h->opt.loop == IETIDP_LOOP_EXPLICIT) {
    if (cfg.ncp == 1 && cfg.stages == 2) return launch_pcg_t<1, 2, true>(h, cfg, a);
    if (cfg.ncp == 1 && cfg.stages == 5) return launch_pcg_t<1, 5, true>(h, cfg, a);
    if (cfg.ncp == 1) return launch_pcg_t<1, 3, true>(h, cfg, a);
    if (cfg.ncp == 16 && a.chunk && cfg.stages == 3) return launch_pcg_t<16, 3, true, true>(h, cfg, a);
    if (cfg.ncp == 16 && a.chunk) return launch_pcg_t<16, 2, true, true>(h, cfg, a);
    if (cfg.ncp == 16 && cfg.stages == 3) return launch_pcg_t<16, 3, true>(h, cfg, a);
    if (cfg.ncp == 16) return launch_pcg_t<16, 2, true>(h, cfg, a);
    if (cfg.stages == 3) return launch_pcg_t<8, 3, true>(h, cfg, a);
    return launch_pcg_t<8, 2, true>(h, cfg, a);
  }
  if (cfg.ncp == 1 && cfg.stages == 5) return launch_pcg_t<1, 5, false>(h, cfg, a);
  if (cfg.ncp == 1) return launch_pcg_t<1, 3, false>(h, cfg, a);
  if (cfg.ncp == 16 && cfg.stages == 3) return launch_pcg_t<16, 3, false>(h, cfg, a);
  if (cfg.ncp == 16) return launch_pcg_t<16, 2, false>(h, cfg, a);
  if (cfg.stages == 3) return launch_pcg_t<8, 3, false>(h, cfg, a);
  return launch_pcg_t<8, 2, false>(h, cfg, a);
}

// ietidp_apply_F on all 16 columns: the chunk pass and its phases as launches of their own
// (the kernels of the sharded loop), with the persistent kernel's plans -- W pass | g | z_k,
// G_k z_k | folded gather -- instead of the row-segment stream (C5: 268 -> ~170 us per apply).
// IETIDP_FAPPLY_CHUNK=0 keeps the stream.
static bool apply_F_chunk(ietidp_s* h, int ncols, const double* x, double* y) {
  if (h->shard || ncols != 16 || ncols != h->nrhs || h->opt.loop != IETIDP_LOOP_EXPLICIT || h->n_lambda == 0) return false;
  static const bool off = getenv("IETIDP_FAPPLY_CHUNK") && atoi(getenv("IETIDP_FAPPLY_CHUNK")) == 0;
  if (off) return false;
  if (!h->fa_tried) {
    h->fa_tried = true;
    PcgArgs A{};
    g_prepare.out = &A;
    g_prepare.chunk = false;
    bool ok = false;
    try {
      ok = run_solve_persistent(h);
    } catch (...) {
      g_prepare.out = nullptr;
      throw;
    }
    g_prepare.out = nullptr;
    if (ok && g_prepare.chunk) {
      h->fa_args.resize(sizeof(PcgArgs));
      memcpy(h->fa_args.data(), &A, sizeof(PcgArgs));
      h->fa_grid = g_prepare.grid;
      h->fa_smem = g_prepare.smem;
      h->fa_stages = g_prepare.stages;
      h->fa_state.alloc(sizeof(PcgState) / sizeof(double) + 1);
      h->fa_state.zero(h->stream);  // a state that is never "done"
    }
  }
  if (h->fa_args.empty()) return false;
  PcgArgs A;
  memcpy(&A, h->fa_args.data(), sizeof(PcgArgs));
  A.st = reinterpret_cast<PcgState*>(h->fa_state.p);
  A.q = y;
  A.p = const_cast<double*>(x);  // (read only: the gather's dot partials, discarded)
  cudaStream_t s = h->stream;
  const int grid = h->fa_grid, smem = h->fa_smem;
  k_to_slots<<<grid_for((long long)h->n_slots * ncols, 256), 256, 0, s>>>(h->n_slots, ncols, h->slot_lam.p, h->slot_sign.p,
                                                                         nullptr, x, h->pslot.p, nullptr);
  IETI_LAUNCHED(h);
  if (h->fa_stages == 3) {
    IETI_CUDA(cudaFuncSetAttribute((const void*)k_ch_pass<3, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_ch_pass<3, 0><<<grid, 256, smem, s>>>(A);
  } else {
    IETI_CUDA(cudaFuncSetAttribute((const void*)k_ch_pass<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_ch_pass<2, 0><<<grid, 256, smem, s>>>(A);
  }
  IETI_LAUNCHED(h);
  if (h->n_primal) {
    k_ch_g<<<grid, 256, 0, s>>>(A);
    IETI_LAUNCHED(h);
    IETI_CUDA(cudaFuncSetAttribute((const void*)k_ch_zk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_ch_zk<<<grid, 256, smem, s>>>(A);
    IETI_LAUNCHED(h);
  }
  k_ch_gather<0><<<grid, 256, 0, s>>>(A, h->partial.p + 3 * NBLK * ncols);
  IETI_LAUNCHED(h);
  return true;
}

void run_solve(ietidp_s* h) {
  const int nc = h->nrhs, m = h->n_lambda;
  PcgState* st = reinterpret_cast<PcgState*>(h->state.p);
  double* rr_part = h->partial.p + NBLK * nc;
  double* rz_part = h->partial.p + 2 * NBLK * nc;
  cudaStream_t s = h->stream;
  IETI_CUDA(cudaMemsetAsync(h->partial.p, 0, h->partial.n * sizeof(double), s));
  const char* mode = getenv("IETIDP_PCG");
  h->pcg_persistent = false;
  if (!h->shard && !(mode && std::string(mode) == "graph") && run_solve_persistent(h)) {
    h->pcg_persistent = true;
    IETI_CHECK_LAUNCH();
    return;
  }
  if (h->opt.stop != IETIDP_STOP_RESIDUAL && m > 0)
    throw Error(IETIDP_E_ARG, "the preconditioned stopping criterion needs the persistent PCG kernel");
  // sharded, 16 RHS: the chunk pass and its phases as separate launches (the persistent
  // kernel's device functions), IETIDP_SHARD_CHUNK=0 keeps the row-segment stream
  PcgArgs CA{};
  bool ch = false;
  if (h->shard && m > 0 && h->opt.loop == IETIDP_LOOP_EXPLICIT &&
      !(getenv("IETIDP_SHARD_CHUNK") && atoi(getenv("IETIDP_SHARD_CHUNK")) == 0)) {
    g_prepare.out = &CA;
    g_prepare.chunk = false;
    bool ok = false;
    try {
      ok = run_solve_persistent(h);
    } catch (...) {
      g_prepare.out = nullptr;
      throw;
    }
    g_prepare.out = nullptr;
    ch = ok && g_prepare.chunk;
  }
  const int cgrid = g_prepare.grid, csmem = g_prepare.smem, cstages = g_prepare.stages;
  double* gscratch = h->partial.p + 3 * NBLK * nc;
  auto to_slots = [&](const double* x, const double* w, double* out) {
    k_to_slots<<<grid_for((long long)h->n_slots * nc, 256), 256, 0, s>>>(h->n_slots, nc, h->slot_lam.p, h->slot_sign.p, w, x,
                                                                        out, st);
    IETI_LAUNCHED(h);
  };
  auto ch_pass = [&](int which) {
    auto set = [&](const void* k) { IETI_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem)); };
    if (cstages == 3) {
      if (which) { set((const void*)k_ch_pass<3, 1>); k_ch_pass<3, 1><<<cgrid, 256, csmem, s>>>(CA); }
      else { set((const void*)k_ch_pass<3, 0>); k_ch_pass<3, 0><<<cgrid, 256, csmem, s>>>(CA); }
    } else {
      if (which) { set((const void*)k_ch_pass<2, 1>); k_ch_pass<2, 1><<<cgrid, 256, csmem, s>>>(CA); }
      else { set((const void*)k_ch_pass<2, 0>); k_ch_pass<2, 0><<<cgrid, 256, csmem, s>>>(CA); }
    }
    IETI_LAUNCHED(h);
  };
  auto ch_apply_F = [&]() {  // q = F_DP p, p.q partials
    to_slots(h->p_vec.p, nullptr, h->pslot.p);
    ch_pass(0);
    if (h->n_primal) {
      k_ch_g<<<cgrid, 256, 0, s>>>(CA);
      IETI_LAUNCHED(h);
      sh_sum(h, h->gc.p, (long long)h->n_primal * nc);
      IETI_CUDA(cudaFuncSetAttribute((const void*)k_ch_zk, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem));
      k_ch_zk<<<cgrid, 256, csmem, s>>>(CA);
      IETI_LAUNCHED(h);
    }
    k_ch_gather<0><<<cgrid, 256, 0, s>>>(CA, gscratch);
    IETI_LAUNCHED(h);
    sh_finish_gather(h, nc, h->q_vec.p, h->p_vec.p, h->partial.p, st);
  };
  auto ch_apply_M = [&]() {  // z = M_D^-1 r, r.z partials
    to_slots(h->r_vec.p, h->delta.p, h->rslot.p);
    ch_pass(1);
    k_ch_gather<1><<<cgrid, 256, 0, s>>>(CA, gscratch);
    IETI_LAUNCHED(h);
    sh_finish_gather(h, nc, h->z_vec.p, h->r_vec.p, rz_part, st);
  };
  auto ch_body = [&]() {
    ch_apply_F();
    k_cg_alpha<<<NBLK, VT, 0, s>>>(m, st, h->partial.p, h->lam_vec.p, h->r_vec.p, h->p_vec.p, h->q_vec.p, rr_part,
                                  h->cgcoef.p, h->coef_ld);
    IETI_LAUNCHED(h);
    ch_apply_M();
    k_cg_beta<<<NBLK, VT, 0, s>>>(m, st, rr_part, rz_part, h->p_vec.p, h->z_vec.p, h->cgcoef.p, h->coef_ld);
    IETI_LAUNCHED(h);
    k_ctl<<<1, 64, 0, s>>>(st, rr_part, rz_part, 0ull, 0);
    IETI_LAUNCHED(h);
  };
  if (m > 0) {
    k_init<<<NBLK, VT, 0, s>>>(m, nc, h->d_vec.p, h->lam_vec.p, h->r_vec.p, rr_part);
    IETI_LAUNCHED(h);
  }
  k_init_ctl<<<1, 64, 0, s>>>(st, rr_part, nc, m, h->opt.tol, h->opt.max_iter, h->opt.fixed_iters);
  IETI_LAUNCHED(h);
  if (m > 0) {
    if (ch) ch_apply_M();
    else apply_M_inter(h, nc, h->r_vec.p, h->z_vec.p, st, rr_part, 0, h->r_vec.p, rz_part);
    k_init_p<<<NBLK, VT, 0, s>>>(m, st, h->z_vec.p, h->p_vec.p);
    IETI_LAUNCHED(h);
    k_init_rz<<<1, 64, 0, s>>>(st, rz_part);
    IETI_LAUNCHED(h);
    if (h->shard) {
      // The all-reduce is the caller's, so the loop is driven from the host. Every rank reads
      // the same replicated state and takes the same decision. The stop flag of iteration i is
      // read after iteration i + 1 has been enqueued (one iteration of look-ahead keeps the GPU
      // fed while the host waits); the extra iteration launched past convergence is a no-op:
      // every kernel returns at once when st->done is set, and the sums over the ranks then
      // touch only q and z, which nothing reads afterwards.
      int* flag = nullptr;  // pinned {it, done}
      IETI_CUDA(cudaMallocHost(&flag, 2 * sizeof(int)));
      cudaEvent_t fev = nullptr;
      try {
        IETI_CUDA(cudaEventCreateWithFlags(&fev, cudaEventDisableTiming));
        flag[0] = flag[1] = 0;
        IETI_CUDA(cudaMemcpyAsync(flag, st, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
        IETI_CUDA(cudaStreamSynchronize(s));
        auto body = [&]() {
          if (ch) ch_body();
          else iteration_body(h, st, 0);
        };
        if (!flag[1]) {
          body();
          IETI_CUDA(cudaMemcpyAsync(flag, st, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
          IETI_CUDA(cudaEventRecord(fev, s));
          for (;;) {
            body();                                  // the next iteration, speculatively
            IETI_CUDA(cudaEventSynchronize(fev));    // the flag after the previous one
            if (flag[1]) break;
            IETI_CUDA(cudaMemcpyAsync(flag, st, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
            IETI_CUDA(cudaEventRecord(fev, s));
          }
        }
        IETI_CUDA(cudaStreamSynchronize(s));
      } catch (...) {
        if (fev) cudaEventDestroy(fev);
        cudaFreeHost(flag);
        throw;
      }
      cudaEventDestroy(fev);
      cudaFreeHost(flag);
      IETI_CHECK_LAUNCH();
      return;
    }
    build_graph(h, st);
    IETI_CUDA(cudaGraphLaunch((cudaGraphExec_t)h->graph_exec, s));
  }
  IETI_CHECK_LAUNCH();
}

void finish_solve(ietidp_s* h, ietidp_report* rep) {
  const int nc = h->nrhs, m = h->n_lambda;
  PcgState hs;
  IETI_CUDA(cudaMemcpyAsync(&hs, h->state.p, sizeof(PcgState), cudaMemcpyDeviceToHost, h->stream));
  IETI_CUDA(cudaStreamSynchronize(h->stream));
  if (m > 0 && !h->pcg_persistent) h->launches += (long long)body_launches(h, nc) * std::max(hs.it, 1);
  for (int c = 0; c < nc; ++c) {
    rep->iters[c] = hs.iters[c];
    rep->converged[c] = h->opt.fixed_iters ? 1 : !hs.active[c];
  }
  if (m > 0) {
    double* part = h->partial.p + 3 * NBLK * nc;
    apply_F_inter(h, nc, h->lam_vec.p, h->tmp_out.p, nullptr, nullptr, nullptr);
    k_resid<<<NBLK, VT, 0, h->stream>>>(m, nc, h->d_vec.p, h->tmp_out.p, part);
    IETI_LAUNCHED(h);
    double* ratio = h->cond_out.p;  // scratch (nc doubles), rewritten by the condition estimate
    k_resid_ratio<<<1, 512, 0, h->stream>>>(part, reinterpret_cast<const PcgState*>(h->state.p), ratio);
    IETI_LAUNCHED(h);
    IETI_CUDA(cudaMemcpyAsync(rep->rel_residual, ratio, (size_t)nc * sizeof(double), cudaMemcpyDeviceToHost,
                              h->stream));
    IETI_CUDA(cudaStreamSynchronize(h->stream));
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

// ---------------------------------------------------------------------------
// Condition estimate (SPEC estimate_condition; "cond(M_D^-1 S) with the
// largest and smallest absolute eigenvalue omega_max, omega_min"; SURVEY §8(c) Q25:
// Lanczos from the PCG alpha/beta). k PCG iterations of column c define the Lanczos
// tridiagonal of the preconditioned operator (the CG-Lanczos relation):
//   T_jj = 1/alpha_j + beta_{j-1}/alpha_{j-1}   (beta_{-1} = 0),
//   T_{j,j+1}^2 = beta_j / alpha_j^2,           j = 0..k-1 (beta_0..beta_{k-2} used).
// Its extreme eigenvalues (Ritz values) are found by multisection on the Sturm count
// (number of negative pivots of T - xI = number of eigenvalues below x): one CTA per
// column, threads 0..127 refine omega_min and 128..255 omega_max, 128 points per round.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int sturm_below(const double* a, const double* b2, int k, double x, double pivmin) {
  int cnt = 0;
  double d = a[0] - x;
  if (fabs(d) < pivmin) d = -pivmin;
  cnt += d < 0.0;
  for (int i = 1; i < k; ++i) {
    d = (a[i] - x) - b2[i - 1] / d;
    if (fabs(d) < pivmin) d = -pivmin;
    cnt += d < 0.0;
  }
  return cnt;
}

__global__ void __launch_bounds__(256) k_lanczos_cond(const PcgState* __restrict__ st, const double* __restrict__ coef,
                                                      int ld, double* __restrict__ out) {
  extern __shared__ double sm[];
  const int c = blockIdx.x, nc = gridDim.x, tid = threadIdx.x;
  const int k = min(st->iters[c], ld);
  double* a = sm;       // diagonal of T (k)
  double* b2 = sm + ld; // squared off-diagonal (k - 1)
  __shared__ double s_lo[2], s_hi[2], s_red[2][256];
  __shared__ int s_cnt[256];
  if (k == 0) {
    if (tid == 0) out[3 * c] = out[3 * c + 1] = out[3 * c + 2] = 0.0;
    return;
  }
  const double* al = coef + (size_t)c * ld;
  const double* be = coef + (size_t)(nc + c) * ld;
  for (int j = tid; j < k; j += blockDim.x) {
    a[j] = 1.0 / al[j] + (j > 0 ? be[j - 1] / al[j - 1] : 0.0);
    if (j < k - 1) b2[j] = be[j] / (al[j] * al[j]);
  }
  __syncthreads();
  // Gershgorin interval and the largest squared off-diagonal (pivot floor, as LAPACK's pivmin)
  double glo = INFINITY, ghi = -INFINITY, bmax = 0.0;
  for (int j = tid; j < k; j += blockDim.x) {
    const double r = (j > 0 ? sqrt(b2[j - 1]) : 0.0) + (j < k - 1 ? sqrt(b2[j]) : 0.0);
    glo = fmin(glo, a[j] - r);
    ghi = fmax(ghi, a[j] + r);
    if (j < k - 1) bmax = fmax(bmax, b2[j]);
  }
  s_red[0][tid] = glo;
  s_red[1][tid] = ghi;
  s_cnt[tid] = 0;
  __syncthreads();
  if (tid == 0) {
    for (int t = 1; t < blockDim.x; ++t) {
      glo = fmin(glo, s_red[0][t]);
      ghi = fmax(ghi, s_red[1][t]);
    }
    const double w = fmax(ghi - glo, fabs(ghi)) * 1e-14 + 1e-300;
    s_lo[0] = s_lo[1] = glo - w;
    s_hi[0] = s_hi[1] = ghi + w;
  }
  __syncthreads();
  s_red[0][tid] = bmax;
  __syncthreads();
  if (tid == 0)
    for (int t = 1; t < blockDim.x; ++t) s_red[0][0] = fmax(s_red[0][0], s_red[0][t]);
  __syncthreads();
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, s_red[0][0]);
  const int half = tid >> 7, lane = tid & 127;
  // half 0: eigenvalue index 0 (omega_min), half 1: index k-1 (omega_max); the
  // eigenvalue with index e lies where the count crosses from <= e to >= e+1
  const int e = half ? k - 1 : 0;
  for (int round = 0; round < 12; ++round) {
    const double lo = s_lo[half], hi = s_hi[half];
    const double x = lo + (hi - lo) * (double)(lane + 1) / 129.0;
    s_cnt[tid] = sturm_below(a, b2, k, x, pivmin) >= e + 1;
    __syncthreads();
    if (lane == 0) {
      int i = 0;
      while (i < 128 && !s_cnt[tid + i]) ++i;
      const double nlo = i == 0 ? lo : lo + (hi - lo) * (double)i / 129.0;
      const double nhi = i == 128 ? hi : lo + (hi - lo) * (double)(i + 1) / 129.0;
      s_lo[half] = nlo;
      s_hi[half] = nhi;
    }
    __syncthreads();
    if (s_hi[0] - s_lo[0] <= 2e-16 * fabs(s_hi[0]) && s_hi[1] - s_lo[1] <= 2e-16 * fabs(s_hi[1])) break;
  }
  if (tid == 0) {
    const double wmin = 0.5 * (s_lo[0] + s_hi[0]), wmax = 0.5 * (s_lo[1] + s_hi[1]);
    out[3 * c] = wmin;
    out[3 * c + 1] = wmax;
    out[3 * c + 2] = wmax / wmin;
  }
}

void run_estimate_condition(ietidp_s* h, double* omega_min, double* omega_max, double* cond) {
  const int nc = h->nrhs, ld = h->coef_ld;
  const size_t smem = 2 * (size_t)ld * sizeof(double);
  if (smem > 48 * 1024)
    IETI_CUDA(cudaFuncSetAttribute(k_lanczos_cond, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_lanczos_cond<<<nc, 256, smem, h->stream>>>(reinterpret_cast<const PcgState*>(h->state.p), h->cgcoef.p, ld,
                                               h->cond_out.p);
  IETI_LAUNCHED(h);
  IETI_CHECK_LAUNCH();
  std::vector<double> o(3 * (size_t)nc);
  IETI_CUDA(cudaMemcpyAsync(o.data(), h->cond_out.p, o.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  IETI_CUDA(cudaStreamSynchronize(h->stream));
  for (int c = 0; c < nc; ++c) {
    if (omega_min) omega_min[c] = o[3 * c];
    if (omega_max) omega_max[c] = o[3 * c + 1];
    if (cond) cond[c] = o[3 * c + 2];
  }
}

}  // namespace ieti
