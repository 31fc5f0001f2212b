// Batched supernodal (multifrontal) Cholesky of every subdomain's K_rr^(k) with
// the primal DOFs ordered last.
//
// All supernodes of one elimination-tree level, over ALL subdomains, are one
// batch. Per level:
//   (all fronts are zeroed and K's entries scattered once, up front)
//   1. left-looking partial Cholesky over the pivot columns in TB-wide panels:
//      (a) panel columns -= L[rows, 0:p0] L[panel, 0:p0]^T   (DMMA GEMM, long K)
//      (b) POTRF of the TB x TB diagonal block and its inverse Dinv
//      (c) rows below the diagonal block: L = A Dinv^T      (DMMA GEMM)
//   2. update block: parent[rel] += F22 - L21 L21^T           (DMMA GEMM, K = npiv,
//      the multifrontal extend-add fused into its epilogue; one launch per child
//      slot: deterministic, no atomics)
// The P supernode of each subdomain is assembled but not factored: it ends as
// S_loc = K_PP - K_Pr K_rr^-1 K_rP. Afterwards every pivot block is inverted
// (partitioned inverse, recursive doubling with the same GEMM kernel).
#include <climits>

#include "common.cuh"

namespace ieti {

__global__ void k_scatter(long long n, const long long* __restrict__ dst, const int* __restrict__ src,
                          const double* __restrict__ vals, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[dst[i]] = vals[src[i]];
}

// 1/sqrt(a) in FP64 without the slow-path sqrt and divide: a float MUFU seed
// (~2^-23) refined by two Newton steps r <- r (3 - a r^2) / 2 (~2^-46, ~2^-92:
// within rounding of the correctly rounded value). The pivot chain of POTRF runs
// through this once per column, so its latency sets the kernel's.
__device__ __forceinline__ double rsqrt_fast(double a) {
  if (!(a > 1e-30 && a < 1e30)) return 1.0 / sqrt(a);
  double r = (double)rsqrtf((float)a);
  r = r * (1.5 - 0.5 * a * r * r);
  r = r * (1.5 - 0.5 * a * r * r);
  return r;
}

// POTRF of the diagonal block of panel w.a of front w.sn, and its inverse.
// Cholesky: one barrier per elimination step. Step j reads the pivot column from a
// double-buffered copy `cb` (static smem, so the trailing update's loads and stores
// to A stay in flight) and the pivot's reciprocal square root `pr`, which the thread
// that updates the next diagonal entry computes ahead (hidden behind the update).
// Inverse: the four 16 x 16 diagonal blocks are inverted by four warps, the
// off-diagonal blocks follow in three block-row steps (X_ib,jb = -X_ib,ib sum L X).
constexpr int POTRF_T = 256;
constexpr int SB = 16;  // sub-block of the inverse
__global__ void __launch_bounds__(POTRF_T) k_potrf(const Work* __restrict__ work, const SnDev* __restrict__ sn,
                                                   double* __restrict__ pool, double* __restrict__ dinv,
                                                   int* __restrict__ err) {
  extern __shared__ double sm[];
  double(*A)[TB + 1] = reinterpret_cast<double(*)[TB + 1]>(sm);  // working copy, then X = L^-1
  __shared__ double L[TB][TB + 1];
  __shared__ double T[SB][3 * SB + 1];  // scratch (L X) of one block row: 16 x 48
  __shared__ double dg[TB];
  __shared__ double cb[2][TB];
  __shared__ double pr[2];
  __shared__ int bad;
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const int p0 = w.a * TB;
  const int b = min(TB, s.npiv - p0);
  double* F = pool + s.front_off + (long long)p0 * s.ld + p0;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int e = tid; e < TB * TB; e += POTRF_T) {
    const int c = e / TB, r = e % TB;  // column-major walk: coalesced along r
    double v;
    if (r < b && c < b) v = (r >= c) ? F[(long long)c * s.ld + r] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    A[r][c] = v;
    if (c == 0) cb[0][r] = v;
    if (e == 0) {
      const bool ok = v > 0.0;
      if (!ok) bad = 1;
      pr[0] = ok ? rsqrt_fast(v) : 1.0;
    }
  }
  __syncthreads();
  const int r = tid & 63, cg = tid >> 6;  // 64 rows x 4 column groups
  for (int j = 0; j < TB; ++j) {
    const double* col = cb[j & 1];
    double* nxt = cb[(j + 1) & 1];
    const double rj = pr[j & 1];
    const double ajj = col[j];
    if (r >= j && cg == 0) L[r][j] = (r == j) ? ajj * rj : col[r] * rj;
    if (r > j) {
      const double lr = col[r] * rj * rj;
      int c = j + 1 + cg;
      if (cg == 0) {  // column j+1: the next pivot column
        const double v = A[r][c] - lr * col[c];
        A[r][c] = v;
        nxt[r] = v;
        if (r == j + 1) {  // the next pivot: its rsqrt ahead of the barrier
          const bool ok = v > 0.0;
          if (!ok) bad = 1;
          pr[(j + 1) & 1] = ok ? rsqrt_fast(v) : 1.0;
        }
        c += 4;
      }
      for (; c + 12 <= r; c += 16) {
        const double a0 = A[r][c], a1 = A[r][c + 4], a2 = A[r][c + 8], a3 = A[r][c + 12];
        const double b0 = col[c], b1 = col[c + 4], b2 = col[c + 8], b3 = col[c + 12];
        A[r][c] = a0 - lr * b0;
        A[r][c + 4] = a1 - lr * b1;
        A[r][c + 8] = a2 - lr * b2;
        A[r][c + 12] = a3 - lr * b3;
      }
      for (; c <= r; c += 4) A[r][c] -= lr * col[c];
    }
    __syncthreads();
  }
  if (tid == 0 && bad) atomicMin(err, s.sub);
  for (int e = tid; e < TB * TB; e += POTRF_T) {
    const int c = e / TB, rr = e % TB;
    if (rr < b && c < b && rr >= c) F[(long long)c * s.ld + rr] = L[rr][c];
  }
  // ---- X = L^-1 ----
  double(*X)[TB + 1] = A;
  for (int e = tid; e < TB * TB; e += POTRF_T) X[e / TB][e % TB] = 0.0;
  if (tid < TB) dg[tid] = 1.0 / L[tid][tid];
  __syncthreads();
  {
    // diagonal 16-blocks: warp wb < 4 inverts block wb; lane c < 16 solves column c
    const int warp = tid >> 5, lane = tid & 31;
    if (warp < 4 && lane < SB) {
      const int o = warp * SB, c = lane;
      double xc[SB];  // column c of the block inverse, in registers
#pragma unroll
      for (int m = 0; m < SB; ++m) xc[m] = (m == c) ? dg[o + c] : 0.0;
      X[o + c][o + c] = dg[o + c];
#pragma unroll
      for (int rr = 1; rr < SB; ++rr) {
        if (rr <= c) continue;
        double sum = 0.0;
#pragma unroll
        for (int m = 0; m < rr; ++m) sum += L[o + rr][o + m] * xc[m];  // xc[m] = 0 for m < c
        xc[rr] = -sum * dg[o + rr];
        X[o + rr][o + c] = xc[rr];
      }
    }
  }
  __syncthreads();
  for (int ib = 1; ib < TB / SB; ++ib) {
    // T[r][c] = sum_m L[ib*16 + r][m] X[m][c] over the block rows jb..ib-1 of X
    const int nc = ib * SB;
    for (int e = tid; e < SB * nc; e += POTRF_T) {
      const int rr = e / nc, c = e % nc;
      double sum = 0.0;
      for (int m = (c / SB) * SB; m < nc; ++m) sum += L[ib * SB + rr][m] * X[m][c];
      T[rr][c] = sum;
    }
    __syncthreads();
    // X[ib*16 + r][c] = -sum_k X_diag[r][k] T[k][c]
    for (int e = tid; e < SB * nc; e += POTRF_T) {
      const int rr = e / nc, c = e % nc;
      double sum = 0.0;
      for (int k = 0; k <= rr; ++k) sum += X[ib * SB + rr][ib * SB + k] * T[k][c];
      X[ib * SB + rr][c] = -sum;
    }
    __syncthreads();
  }
  double* D = dinv + s.dinv_off + (long long)w.a * TILE_ELEMS;  // column-major TB x TB
  for (int e = tid; e < TB * TB; e += POTRF_T) {
    const int c = e / TB, rr = e % TB;
    D[e] = (rr < b && c < b && rr >= c) ? X[rr][c] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Batched tile GEMM on DMMA (mma.sync m8n8k4 f64), cp.async double-buffered K pipeline.
// C(m x n, <= 64 x 64) = (+/-) A(m x K) B(K x n) (+ C), one tile per CTA,
// 4 warps x (32 x 32) quadrants, K in chunks of 32.
//   A[r][k] = Ab[a_off + k*lda + r]   (column-major, r contiguous)
//   BKC = false: B[k][n] = Bb[b_off + k*ldb + n]  (n contiguous: L^T of a front panel, Dinv^T)
//   BKC = true:  B[k][n] = Bb[b_off + n*ldb + k]  (k contiguous: column-major B)
//   ATR = true:  A[r][k] = Ab[a_off + r*lda + k]  (A given transposed, k contiguous)
// ---------------------------------------------------------------------------
constexpr int KC = 32, GST = 2, KS = 72;  // 2 stages: 74 KB smem, 3 CTAs/SM
constexpr int GEMM_SMEM = GST * 2 * KC * KS * (int)sizeof(double);

__device__ __forceinline__ void cp_async_z16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_z8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}

// load a KC x 64 chunk of a "row-contiguous" operand: dst[k][r] = src[k*ld + r]
__device__ __forceinline__ void load_rc(double* dst, const double* src, long long ld, int kb, int rows, bool al16,
                                        int tid) {
  if (al16) {
    for (int q = tid; q < KC * 32; q += 128) {
      const int k = q >> 5, r = (q & 31) * 2;
      const int nv = (k < kb) ? max(0, min(2, rows - r)) : 0;
      const double* g = src + (nv ? (long long)k * ld + r : 0);
      cp_async_z16(dst + k * KS + r, g, nv * 8);
    }
  } else {
    for (int q = tid; q < KC * 64; q += 128) {
      const int k = q >> 6, r = q & 63;
      const int nv = (k < kb && r < rows) ? 1 : 0;
      const double* g = src + (nv ? (long long)k * ld + r : 0);
      cp_async_z8(dst + k * KS + r, g, nv * 8);
    }
  }
}

template <bool BKC, bool ATR = false>
__global__ void __launch_bounds__(128) k_gemm(const GemmWork* __restrict__ work, const double* __restrict__ Ab,
                                              const double* __restrict__ Bb, double* __restrict__ Cb,
                                              const int* __restrict__ d_rel) {
  extern __shared__ __align__(16) double sm[];
  const GemmWork w = work[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int nch = (w.kdim + KC - 1) / KC;
  const bool a16 = (w.a_off & 1) == 0 && (w.lda & 1) == 0;
  const bool b16 = !BKC && (w.b_off & 1) == 0 && (w.ldb & 1) == 0;
  auto As = [&](int st) { return sm + st * 2 * KC * KS; };
  auto Bs = [&](int st) { return sm + st * 2 * KC * KS + KC * KS; };
  auto load = [&](int st, int ch) {
    const int k0 = ch * KC, kb = min(KC, w.kdim - k0);
    if (!ATR) {
      load_rc(As(st), Ab + w.a_off + (long long)k0 * w.lda, w.lda, kb, w.m, a16, tid);
    } else {  // A[r][k] = Ab[a_off + r*lda + k] (k contiguous)
      double* d = As(st);
      for (int q = tid; q < KC * 64; q += 128) {
        const int r = q >> 5, k = q & 31;
        const int nv = (k < kb && r < w.m) ? 1 : 0;
        const double* gp = Ab + (nv ? w.a_off + (long long)r * w.lda + k0 + k : 0);
        cp_async_z8(d + k * KS + r, gp, nv * 8);
      }
    }
    if (!BKC) {
      load_rc(Bs(st), Bb + w.b_off + (long long)k0 * w.ldb, w.ldb, kb, w.n, b16, tid);
    } else {
      double* d = Bs(st);
      for (int q = tid; q < KC * 64; q += 128) {
        const int n = q >> 5, k = q & 31;  // k fastest: coalesced global reads
        const int nv = (k < kb && n < w.n) ? 1 : 0;
        const double* gp = Bb + (nv ? w.b_off + (long long)n * w.ldb + k0 + k : 0);
        cp_async_z8(d + k * KS + n, gp, nv * 8);
      }
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < GST - 1; ++s) {
    if (s < nch) load(s, s);
    cp_async_commit();
  }
  for (int ch = 0; ch < nch; ++ch) {
    cp_async_wait<GST - 2>();
    __syncthreads();
    if (ch + GST - 1 < nch) load((ch + GST - 1) % GST, ch + GST - 1);
    cp_async_commit();
    const double* a_s = As(ch % GST);
    const double* b_s = Bs(ch % GST);
#pragma unroll
    for (int k0 = 0; k0 < KC; k0 += 4) {
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = a_s[(k0 + t) * KS + wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = b_s[(k0 + t) * KS + wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // C may alias A (in-place TRSM): all reads done before any write
  const double sgn = (w.mode & 1) ? -1.0 : 1.0;
  if (w.mode & 4) {
    // fused multifrontal extend-add: parent[rel_c, rel_r] += C - A B (lower part)
    const int* rr = d_rel + w.rel_r;
    const int* rc = d_rel + w.rel_c;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = wm + i * 8 + g, c = wn + j * 8 + 2 * t + q;
          if (r < w.m && c < w.n && (!w.diag || r >= c)) {
            const double v = Cb[w.c_off + (long long)c * w.ldc + r] + sgn * acc[i][j][q];
            Cb[w.p_off + (long long)rc[c] * w.p_ld + rr[r]] += v;
          }
        }
    return;
  }
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

// Pack the symmetric n_I x n_I matrix held in the lower triangle of a column-major
// block (the r_I root front, or its L11^-1-shaped buffer) into row-major lower
// TB-tiles with full (mirrored) diagonal tiles. One CTA per (entry, block row).
__global__ void __launch_bounds__(256)
    k_pack_sym(const int* __restrict__ list, int maxnt, const SubDev* __restrict__ sub, const SnDev* __restrict__ sn,
               const double* __restrict__ base, int from_front, double* __restrict__ dst) {
  const int e = blockIdx.x / maxnt, i = blockIdx.x % maxnt;
  const int k = list ? list[e] : e;
  const SubDev d = sub[k];
  if (d.nI == 0 || i >= d.nt) return;
  const SnDev s = sn[d.root];
  const double* M = base + (from_front ? s.front_off : s.inv_off);
  const long long ld = from_front ? s.ld : s.ldi;
  for (int j = 0; j <= i; ++j) {
    double* T = dst + d.tile_off + (long long)(i * (i + 1) / 2 + j) * TILE_ELEMS;
    for (int q = threadIdx.x; q < TILE_ELEMS; q += blockDim.x) {
      const int c = q / TB, r = q % TB;
      const int R = i * TB + r, C = j * TB + c;
      double v = 0.0;
      if (R < d.nI && C < d.nI) v = (R >= C) ? M[(long long)C * ld + R] : M[(long long)R * ld + C];
      T[r * TB + c] = v;
    }
  }
}

static void set_smem(const void* f, int bytes) {
  IETI_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void run_factor(ietidp_s* h) {
  cudaStream_t st = h->stream;
  const Plan& P = h->plan;
  static bool attr = false;
  const int sm_potrf = TB * (TB + 1) * sizeof(double);  // A (then X = L^-1); L static
  if (!attr) {
    set_smem((const void*)k_potrf, sm_potrf);
    set_smem((const void*)k_gemm<false>, GEMM_SMEM);
    set_smem((const void*)k_gemm<true>, GEMM_SMEM);
    set_smem((const void*)k_gemm<true, true>, GEMM_SMEM);
    attr = true;
  }
  static const int init_flags[2] = {INT_MAX, 1};  // failing subdomain (min), coarse OK
  IETI_CUDA(cudaMemcpyAsync(h->err_flag.p, init_flags, 2 * sizeof(int), cudaMemcpyHostToDevice, st));
  const Work* W = reinterpret_cast<const Work*>(h->d_work.p);
  const GemmWork* GW = h->d_gwork.p;
  double* pool = h->pool.p;
  // assembly of every front at once: zero the pool, scatter all of K's entries
  IETI_CUDA(cudaMemsetAsync(pool, 0, h->pool.n * sizeof(double), st));
  const long long ne = (long long)h->sc_front_dst.n;
  if (ne > 0) {
    k_scatter<<<grid_for(ne, 256), 256, 0, st>>>(ne, h->sc_front_dst.p, h->sc_front_src.p, h->kval.p, pool);
    IETI_LAUNCHED(h);
  }
  const int* rel = h->d_rel.p;
  int maxnt = 0;
  for (auto& d : h->h_sub) maxnt = std::max(maxnt, d.nt);
  const bool expl = h->opt.loop == IETIDP_LOOP_EXPLICIT;
  for (int L = 0; L <= P.max_level; ++L) {
    const LevelPlan& lp = P.levels[L];
    // explicit loop: S_II is the assembled r_I root front before its factorisation
    if (expl && h->rootlist_range[L].second > 0) {
      k_pack_sym<<<h->rootlist_range[L].second * maxnt, 256, 0, st>>>(h->d_rootlist.p + h->rootlist_range[L].first,
                                                                       maxnt, h->d_sub.p, h->d_sn.p, pool, 1,
                                                                       h->stiles.p);
      IETI_LAUNCHED(h);
    }
    for (auto& pn : lp.panels) {
      if (pn.upd_n) {
        k_gemm<false><<<pn.upd_n, 128, GEMM_SMEM, st>>>(GW + pn.upd_off, pool, pool, pool, rel);
        IETI_LAUNCHED(h);
      }
      if (pn.potrf_n) {
        k_potrf<<<pn.potrf_n, POTRF_T, sm_potrf, st>>>(W + pn.potrf_off, h->d_sn.p, pool, h->dinv.p, h->err_flag.p);
        IETI_LAUNCHED(h);
      }
      if (pn.trsm_n) {
        k_gemm<false><<<pn.trsm_n, 128, GEMM_SMEM, st>>>(GW + pn.trsm_off, pool, h->dinv.p, pool, rel);
        IETI_LAUNCHED(h);
      }
    }
    for (auto& sy : lp.syrk) {
      k_gemm<false><<<sy.second, 128, GEMM_SMEM, st>>>(GW + sy.first, pool, pool, pool, rel);
      IETI_LAUNCHED(h);
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
    k_gemm<true><<<rg.second, 128, GEMM_SMEM, st>>>(GW + rg.first, step1 ? pool : h->ipool.p,
                                                    step1 ? h->ipool.p : h->tpool.p, step1 ? h->tpool.p : h->ipool.p,
                                                    rel);
    IETI_LAUNCHED(h);
  }
  // explicit loop: W_k = L_II^-T L_II^-1 (lower tiles; tpool is free again)
  if (expl && P.w_n) {
    k_gemm<true, true><<<P.w_n, 128, GEMM_SMEM, st>>>(GW + P.w_off, h->ipool.p, h->ipool.p, h->tpool.p, rel);
    IETI_LAUNCHED(h);
    k_pack_sym<<<h->n_sub * maxnt, 256, 0, st>>>(nullptr, maxnt, h->d_sub.p, h->d_sn.p, h->tpool.p, 0, h->wtiles.p);
    IETI_LAUNCHED(h);
  }
  IETI_CHECK_LAUNCH();
}

}  // namespace ieti
