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
#include <cstring>

#include "common.cuh"

namespace ieti {

__global__ void k_scatter(long long n, const long long* __restrict__ dst, const int* __restrict__ src,
                          const double* __restrict__ vals, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[dst[i]] = vals[src[i]];
}

// Scatter-list expansion from per-pattern-class relative entries (analyze.cpp): one
// CTA per segment (subdomain x level, or subdomain loads).
__global__ void __launch_bounds__(256)
    k_expand_scatter(const ExpandSeg* __restrict__ segs, const int* __restrict__ off, const int* __restrict__ sl,
                     const int* __restrict__ src, const SnDev* __restrict__ sn, int nrhs, long long* __restrict__ kdst,
                     int* __restrict__ ksrc, long long* __restrict__ fdst, int* __restrict__ fsrc) {
  const ExpandSeg g = segs[blockIdx.x];
  if (g.kind == 0) {
    for (int q = threadIdx.x; q < g.n; q += blockDim.x) {
      const long long r = g.rel_off + q;
      kdst[g.dst_off + q] = sn[g.sn_base + sl[r]].front_off + off[r];
      ksrc[g.dst_off + q] = (int)(g.base + src[r]);
    }
  } else {
    for (int e = threadIdx.x; e < g.n * nrhs; e += blockDim.x) {
      const int q = e / nrhs, c = e - q * nrhs;
      const long long r = g.rel_off + q;
      fdst[g.dst_off + e] = (g.base + off[r]) * nrhs + c;
      fsrc[g.dst_off + e] = (int)(g.base2 + src[r] + (long long)c * g.nk);
    }
  }
}

void expand_scatter(ietidp_s* h, const std::vector<ExpandSeg>& segs, const std::vector<ClassRel>& cls, long long nrel,
                    long long nK, long long nF) {
  cudaStream_t s = h->stream;
  DevBuf<ExpandSeg> dseg;
  DevBuf<int> doff, dsl, dsrc;
  dseg.upload(segs, s);
  doff.alloc(std::max(nrel, 1LL));
  dsl.alloc(std::max(nrel, 1LL));
  dsrc.alloc(std::max(nrel, 1LL));
  for (const ClassRel& c : cls) {  // each pattern class's entries at their offset
    const size_t n = c.off->size() * sizeof(int);
    if (!n) continue;
    IETI_CUDA(cudaMemcpyAsync(doff.p + c.base, c.off->data(), n, cudaMemcpyHostToDevice, s));
    IETI_CUDA(cudaMemcpyAsync(dsl.p + c.base, c.sl->data(), n, cudaMemcpyHostToDevice, s));
    IETI_CUDA(cudaMemcpyAsync(dsrc.p + c.base, c.src->data(), n, cudaMemcpyHostToDevice, s));
  }
  h->sc_front_dst.alloc(std::max(nK, 1LL));
  h->sc_front_src.alloc(std::max(nK, 1LL));
  h->sc_fx_dst.alloc(std::max(nF, 1LL));
  h->sc_fx_src.alloc(std::max(nF, 1LL));
  h->sc_front_dst.n = nK;
  h->sc_front_src.n = nK;
  h->sc_fx_dst.n = nF;
  h->sc_fx_src.n = nF;
  if (!segs.empty()) {
    k_expand_scatter<<<(unsigned)segs.size(), 256, 0, s>>>(dseg.p, doff.p, dsl.p, dsrc.p, h->d_sn.p, h->nrhs,
                                                           h->sc_front_dst.p, h->sc_front_src.p, h->sc_fx_dst.p,
                                                           h->sc_fx_src.p);
    IETI_LAUNCHED(h);
  }
  IETI_CUDA(cudaStreamSynchronize(s));  // the temporaries are freed on return
}

// ietidp_set_values_lower: a subdomain's full CSR values from its lower-triangle list
// (the mirror's value for an upper entry; the pattern is symmetric, the values are)
__global__ void __launch_bounds__(256) k_expand_lower(long long nnz, const int* __restrict__ map,
                                                     const double* __restrict__ low, double* __restrict__ full) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (long long)gridDim.x * blockDim.x)
    full[e] = low[map[e]];
}
void launch_expand_lower(ietidp_s* h, int k, cudaStream_t st) {
  const long long nnz = (long long)h->in[k].val.size();
  if (!nnz) return;
  k_expand_lower<<<grid_for(nnz, 256), 256, 0, st>>>(nnz, h->low_map.p + h->low_map_off[h->class_rep[k]],
                                                     h->klow.p + h->low_off[k], h->kval.p + h->kval_off[k]);
  IETI_LAUNCHED_SIDE(h);
}

__global__ void k_init_flags(int* err) {
  if (threadIdx.x == 0) {
    err[0] = INT_MAX;
    err[1] = 1;
  }
}

// Zero the lower trapezoid of columns [64 w.a, 64 w.a + 64) of front w.sn (rows c..f-1
// of column c): the only part of a front any kernel reads.
__global__ void __launch_bounds__(256) k_zero_fronts(const Work* __restrict__ work, const SnDev* __restrict__ sn,
                                                     double* __restrict__ pool) {
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const int c0 = w.a * TB, c1 = min(w.b ? s.npiv : s.f, c0 + TB);  // w.b: pivot columns only
  double* F = pool + s.front_off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = c0 + warp; c < c1; c += 8)
    for (int r = c + lane; r < s.f; r += 32) F[(long long)c * s.ld + r] = 0.0;
}

// POTRF of the diagonal block of panel w.a of front w.sn, and its inverse Dinv = L^-1.
// 128 threads; thread (r, h) holds the columns c = 2i + h (i < 32) of row r in registers
// (h is warp-uniform). Elimination step j (64 unrolled steps, one barrier each):
//   s_r = a_r[j] / a_jj,  a_r[c] -= s_r a_c[j]  for c > j,
// with column j read from a double-buffered shared copy. The next pivot column j+1 is
// updated first and published; its owner lanes compute the pivot's reciprocal square
// root (float seed + one third-order correction) while the rest of the row is updated.
// Entries above the diagonal are updated too (never read) so that the step is free of
// per-element predicates; the published column is zero above the diagonal.
// Inverse: 32-blocks X11 = L11^-1, X22 = L22^-1 by forward substitution (lane = column),
// then X21 = -X22 (L21 X11).
constexpr int POTRF_T = 128;
__device__ __forceinline__ double rsqrt_h(double a) {
  if (!(a > 1e-30 && a < 1e30)) return 1.0 / sqrt(a);
  const double r0 = (double)rsqrtf((float)a);
  const double e = fma(-a * r0, r0, 1.0);  // |e| ~ 2^-22
  return fma(r0 * e, fma(0.375, e, 0.5), r0);  // r0 (1 + e/2 + 3e^2/8): error O(e^3)
}
template <int H>
__device__ __forceinline__ void potrf_steps(double (&a)[32], int r, double (*cb)[TB], double* pr, double* dg,
                                            bool& ok) {
#pragma unroll
  for (int j = 0; j < TB; ++j) {
    const double rj = pr[j & 1];
    const double* col = cb[j & 1];
    double* nxt = cb[(j + 1) & 1];
    const double cr = col[r];
    const double s = cr * rj * rj;  // a_r[j] / a_jj
    if ((j & 1) == H) {
      if (r >= j) a[j >> 1] = cr * rj;  // L[r][j]
    }
    if (j + 1 < TB) {
      if (((j + 1) & 1) == H) {
        const int i1 = (j + 1) >> 1;
        a[i1] = fma(-s, col[j + 1], a[i1]);
        const double v = a[i1];
        nxt[r] = (r > j) ? v : 0.0;
        const double rn = rsqrt_h(v);
        if (r == j + 1) {
          pr[(j + 1) & 1] = rn;
          dg[j + 1] = rn;
          ok = ok && (v > 0.0);
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = 2 * i + H;
        if (c >= j + 2) a[i] = fma(-s, col[c], a[i]);
      }
      if (r >= 32) {
#pragma unroll
        for (int i = 16; i < 32; ++i) {
          const int c = 2 * i + H;
          if (c >= j + 2) a[i] = fma(-s, col[c], a[i]);
        }
      }
    }
    __syncthreads();
  }
}
// X = L^-1 from L in Ls (lower, zero upper) into Dinv (column-major TB x TB): 32-blocks
// X11 = L11^-1, X22 = L22^-1 by forward substitution (lane = column), X21 = -X22 (L21 X11).
__device__ __forceinline__ void potrf_inverse(double (*Ls)[TB + 1], double (*Ts)[33], const double* dg, int b,
                                              double* __restrict__ D) {
  const int t = threadIdx.x;
  if (t < 64) {
    const int o = (t >> 5) * 32, c = t & 31;
    double x[32];
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int kk = 0; kk < m; kk += 4) {
        s0 = fma(Ls[o + m][o + kk], x[kk], s0);
        if (kk + 1 < m) s1 = fma(Ls[o + m][o + kk + 1], x[kk + 1], s1);
        if (kk + 2 < m) s2 = fma(Ls[o + m][o + kk + 2], x[kk + 2], s2);
        if (kk + 3 < m) s3 = fma(Ls[o + m][o + kk + 3], x[kk + 3], s3);
      }
      // x[m] = (delta_mc - sum_{k<m} L[m][k] x[k]) / L[m][m]  (0 for m < c)
      x[m] = ((m == c ? 1.0 : 0.0) - ((s0 + s1) + (s2 + s3))) * dg[o + m];
    }
    __syncwarp();
    // X11 over L11; X22 into the unused upper block Ls[m][32 + c]
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      if (o == 0) Ls[m][c] = x[m];
      else Ls[m][32 + c] = x[m];
    }
  }
  __syncthreads();
  const int rr = t >> 2, c0 = (t & 3) * 8;
  double tv[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) tv[q] = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < 32; ++kk) {  // T = L21 X11
    const double l = Ls[32 + rr][kk];
#pragma unroll
    for (int q = 0; q < 8; ++q) tv[q] = fma(l, (kk >= c0 + q) ? Ls[kk][c0 + q] : 0.0, tv[q]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) Ts[rr][c0 + q] = tv[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 8; ++q) tv[q] = 0.0;
  for (int kk = 0; kk <= rr; ++kk) {  // X21 = -X22 T into the L21 block
    const double xk = Ls[rr][32 + kk];
#pragma unroll
    for (int q = 0; q < 8; ++q) tv[q] = fma(xk, Ts[kk][c0 + q], tv[q]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) Ls[32 + rr][c0 + q] = -tv[q];
  __syncthreads();
  for (int e = t; e < TILE_ELEMS; e += POTRF_T) {
    const int c = e >> 6, m = e & 63;
    double v = 0.0;
    if (m >= c && m < b && c < b) v = (c >= 32) ? Ls[m - 32][c] : Ls[m][c];
    D[e] = v;
  }
}

__global__ void __launch_bounds__(POTRF_T) k_potrf(const Work* __restrict__ work, const SnDev* __restrict__ sn,
                                                   double* __restrict__ pool, double* __restrict__ dinv,
                                                   int* __restrict__ err) {
  __shared__ double cb[2][TB];
  __shared__ double pr[2];
  __shared__ double dg[TB];  // 1 / L[j][j]
  __shared__ double Ls[TB][TB + 1];
  __shared__ double Ts[32][33];
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const int p0 = w.a * TB;
  const int b = min(TB, s.npiv - p0);
  double* F = pool + s.front_off + (long long)p0 * s.ld + p0;
  const int t = threadIdx.x, r = t & 63, h = t >> 6;
  double a[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int c = 2 * i + h;
    double v;
    if (r < b && c < b) v = (c <= r) ? F[(long long)c * s.ld + r] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;  // identity padding of a partial block
    a[i] = v;
  }
  bool ok = true;
  if (h == 0) {
    cb[0][r] = a[0];
    if (r == 0) {
      pr[0] = rsqrt_h(a[0]);
      dg[0] = pr[0];
      ok = a[0] > 0.0;
    }
  }
  __syncthreads();
  if (h == 0) potrf_steps<0>(a, r, cb, pr, dg, ok);
  else potrf_steps<1>(a, r, cb, pr, dg, ok);
  if (!ok) atomicMin(err, s.sub);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int c = 2 * i + h;
    if (r < b && c < b && c <= r) F[(long long)c * s.ld + r] = a[i];
    Ls[r][c] = (c <= r) ? a[i] : 0.0;
  }
  __syncthreads();
  potrf_inverse(Ls, Ts, dg, b, dinv + s.dinv_off + (long long)w.a * TILE_ELEMS);
}

// Compact variant (default): the 64 elimination steps as a rolled loop over
// 8-column panels (8 unrolled steps each) with the register window shifted by 4 per panel,
// ~5x less code than k_potrf -- for an instruction cache that is cold at every launch.
template <int H>
__device__ __forceinline__ void potrf_steps_rolled(double (&a)[32], int r, double (*cb)[2 * TB], double* pr,
                                                   double* dg, double (*Ls)[TB + 1], bool& ok) {
#pragma unroll 1
  for (int jb = 0; jb < TB; jb += 8) {
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int j = jb + jj;
      const double rj = pr[jj & 1];
      const double* col = cb[jj & 1];
      double* nxt = cb[(jj + 1) & 1];
      const double cr = col[r];
      const double sc = cr * rj * rj;
      if ((jj & 1) == H) a[jj >> 1] = cr * rj;  // L[r][j] (valid for r >= j; 0 above: col is 0 there)
      if (((jj + 1) & 1) == H && j + 1 < TB) {
        const int i1 = (jj + 1) >> 1;
        a[i1] = fma(-sc, col[j + 1], a[i1]);
        const double v = a[i1];
        nxt[r] = (r > j) ? v : 0.0;
        const double rn = rsqrt_h(v);
        if (r == j + 1) {
          pr[(jj + 1) & 1] = rn;
          dg[j + 1] = rn;
          ok = ok && (v > 0.0);
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int c = 2 * i + H;  // relative to jb
        if (c >= jj + 2) a[i] = fma(-sc, col[jb + c], a[i]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = jb + 2 * i + H;
      Ls[r][c] = (c <= r) ? a[i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 28; ++i) a[i] = a[i + 4];
#pragma unroll
    for (int i = 28; i < 32; ++i) a[i] = 0.0;
  }
}
__global__ void __launch_bounds__(POTRF_T) k_potrf_c(const Work* __restrict__ work, const SnDev* __restrict__ sn,
                                                     double* __restrict__ pool, double* __restrict__ dinv,
                                                     int* __restrict__ err) {
  __shared__ double cb[2][2 * TB];
  __shared__ double pr[2];
  __shared__ double dg[TB];
  __shared__ double Ls[TB][TB + 1];
  __shared__ double Ts[32][33];
  const Work w = work[blockIdx.x];
  const SnDev s = sn[w.sn];
  const int p0 = w.a * TB;
  const int b = min(TB, s.npiv - p0);
  double* F = pool + s.front_off + (long long)p0 * s.ld + p0;
  const int t = threadIdx.x, r = t & 63, h = t >> 6;
  double a[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int c = 2 * i + h;
    double v;
    if (r < b && c < b) v = (c <= r) ? F[(long long)c * s.ld + r] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    a[i] = v;
  }
  cb[0][TB + r] = 0.0;
  cb[1][TB + r] = 0.0;
  bool ok = true;
  if (h == 0) {
    cb[0][r] = a[0];
    if (r == 0) {
      pr[0] = rsqrt_h(a[0]);
      dg[0] = pr[0];
      ok = a[0] > 0.0;
    }
  }
  __syncthreads();
  if (h == 0) potrf_steps_rolled<0>(a, r, cb, pr, dg, Ls, ok);
  else potrf_steps_rolled<1>(a, r, cb, pr, dg, Ls, ok);
  if (!ok) atomicMin(err, s.sub);
  __syncthreads();
  for (int e = t; e < TILE_ELEMS; e += POTRF_T) {
    const int c = e >> 6, m = e & 63;
    if (m >= c && m < b && c < b) F[(long long)c * s.ld + m] = Ls[m][c];
  }
  potrf_inverse(Ls, Ts, dg, b, dinv + s.dinv_off + (long long)w.a * TILE_ELEMS);
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
constexpr int KC = 16, GST = 3, KS = 68;  // 2 stages: 70 KB smem, 3 CTAs/SM; KS = 4 mod 16: conflict-free fragment loads
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
__global__ void __launch_bounds__(128, 4) k_gemm(const GemmWork* __restrict__ work, const double* __restrict__ Ab,
                                              const double* __restrict__ Bb, double* __restrict__ Cb,
                                              const int* __restrict__ d_rel, double* __restrict__ skws = nullptr,
                                              int* __restrict__ skcnt = nullptr) {
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
        const int r = q / KC, k = q % KC;
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
        const int n = q / KC, k = q % KC;  // k fastest: coalesced global reads
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
  // The accumulator tile goes through shared memory (column-major, stride ETS) so that
  // the epilogue walks whole columns: warp w takes the columns c = w (mod 4), lane l the
  // rows 2l, 2l+1 -- every global access of a warp is one contiguous 512-byte column.
  constexpr int ETS = 66;  // 2 ETS = 4 (mod 32): conflict-free fragment stores
  double* Ts = sm;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = wm + i * 8 + g, c = wn + j * 8 + 2 * t;
      Ts[c * ETS + r] = acc[i][j][0];
      Ts[(c + 1) * ETS + r] = acc[i][j][1];
    }
  __syncthreads();
  const double sgn = (w.mode & 1) ? -1.0 : 1.0;
  const int r0 = 2 * lane;
  if (w.mode & 8) {
    // split-K part: store the partial product; the last part to arrive reduces all
    // parts in index order (deterministic) into C
    double* Pp = skws + w.ws_off + (long long)w.ks * TILE_ELEMS;
    for (int c = warp; c < TB; c += 4)
      *reinterpret_cast<double2*>(Pp + c * TB + r0) = *reinterpret_cast<const double2*>(Ts + c * ETS + r0);
    __threadfence();
    __syncthreads();
    __shared__ int last;
    if (tid == 0) last = (atomicAdd(skcnt + w.cnt, 1) == w.nks - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    // each thread reduces 2 x 2 consecutive entries with all SPLITK_MAX loads in flight
    const double* P0 = skws + w.ws_off;
    for (int e0 = 2 * tid; e0 < TILE_ELEMS; e0 += 2 * 256) {
      double2 v[2][SPLITK_MAX];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int q = 0; q < SPLITK_MAX; ++q)
          if (q < w.nks)
            v[u][q] = __ldcg(reinterpret_cast<const double2*>(P0 + (long long)q * TILE_ELEMS + e0 + u * 256));
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        double s0 = v[u][0].x, s1 = v[u][0].y;
#pragma unroll
        for (int q = 1; q < SPLITK_MAX; ++q)
          if (q < w.nks) {
            s0 += v[u][q].x;
            s1 += v[u][q].y;
          }
        const int e = e0 + u * 256;
        const int r = e & (TB - 1), c = e >> 6;  // r even: r, r + 1 in the same column
        if (c < w.n) {
          double* C = Cb + w.c_off + (long long)c * w.ldc + r;
          if (r < w.m) C[0] = (w.mode & 2) ? C[0] + sgn * s0 : sgn * s0;
          if (r + 1 < w.m) C[1] = (w.mode & 2) ? C[1] + sgn * s1 : sgn * s1;
        }
      }
    }
    if (tid == 0) skcnt[w.cnt] = 0;  // ready for the next launch
    return;
  }
  if (w.mode & 16) {
    // row-major TB x TB tile (the loop's symmetric tile layout, stored swizzled:
    // common.cuh swz), zero padded
    for (int r = warp; r < TB; r += 4) {
      const int c = 2 * lane;
      double v[2] = {0.0, 0.0};
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (r < w.m && c + q < w.n)
          v[q] = (w.diag && r < c + q) ? Ts[r * ETS + c + q] : Ts[(c + q) * ETS + r];
      double2* T = reinterpret_cast<double2*>(Cb + w.c_off + swz(r, c));
      if (w.mode & 2) {
        const double2 o = *T;
        v[0] += o.x;
        v[1] += o.y;
      }
      *T = make_double2(v[0], v[1]);
    }
    return;
  }
  const bool ok0 = r0 < w.m, ok1 = r0 + 1 < w.m;
  if (w.mode & 4) {
    // fused multifrontal extend-add: parent[rel_c[c], rel_r[r]] += C - A B (lower part)
    const int* rr = d_rel + w.rel_r;
    const int* rc = d_rel + w.rel_c;
    const int pr0 = ok0 ? __ldg(rr + r0) : 0, pr1 = ok1 ? __ldg(rr + r0 + 1) : 0;
    const double* Cc = Cb + w.c_off + r0;
    double* Pb = Cb + w.p_off;
    const bool noC = (w.mode & 32) != 0;  // the child's update block is zero (no children)
    constexpr int U = 4;  // columns in flight per warp
    for (int c0 = warp; c0 < w.n; c0 += 4 * U) {
      double cv[U][2], pv[U][2];
      long long po[U];
      bool v0[U], v1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 4 * u;
        const bool cok = c < w.n;
        v0[u] = cok && ok0 && (!w.diag || r0 >= c);
        v1[u] = cok && ok1 && (!w.diag || r0 + 1 >= c);
        po[u] = cok ? (long long)__ldg(rc + c) * w.p_ld : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 4 * u;
        cv[u][0] = (v0[u] && !noC) ? Cc[(long long)c * w.ldc] : 0.0;
        cv[u][1] = (v1[u] && !noC) ? Cc[(long long)c * w.ldc + 1] : 0.0;
        pv[u][0] = v0[u] ? Pb[po[u] + pr0] : 0.0;
        pv[u][1] = v1[u] ? Pb[po[u] + pr1] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 4 * u;
        if (v0[u]) Pb[po[u] + pr0] = pv[u][0] + (cv[u][0] + sgn * Ts[c * ETS + r0]);
        if (v1[u]) Pb[po[u] + pr1] = pv[u][1] + (cv[u][1] + sgn * Ts[c * ETS + r0 + 1]);
      }
    }
    return;
  }
  const bool accum = (w.mode & 2) != 0;
  double* Cc = Cb + w.c_off + r0;
  constexpr int U = 4;
  for (int c0 = warp; c0 < w.n; c0 += 4 * U) {
    double cv[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + 4 * u;
      const bool cok = c < w.n && accum;
      cv[u][0] = (cok && ok0) ? Cc[(long long)c * w.ldc] : 0.0;
      cv[u][1] = (cok && ok1) ? Cc[(long long)c * w.ldc + 1] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + 4 * u;
      if (c < w.n) {
        if (ok0) Cc[(long long)c * w.ldc] = cv[u][0] + sgn * Ts[c * ETS + r0];
        if (ok1) Cc[(long long)c * w.ldc + 1] = cv[u][1] + sgn * Ts[c * ETS + r0 + 1];
      }
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
// TB-tiles with full (mirrored) diagonal tiles. One CTA per (entry, block row); each
// tile is transposed through shared memory (coalesced column reads, row writes).
__global__ void __launch_bounds__(256)
    k_pack_sym(const int* __restrict__ list, int maxnt, const SubDev* __restrict__ sub, const SnDev* __restrict__ sn,
               const double* __restrict__ base, int from_front, double* __restrict__ dst) {
  __shared__ double S[TB][TB + 1];
  const int ntl = maxnt * (maxnt + 1) / 2;  // one CTA per lower tile (i, j)
  const int e = blockIdx.x / ntl, t = blockIdx.x % ntl;
  int i = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while (i * (i + 1) / 2 > t) --i;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  const int j = t - i * (i + 1) / 2;
  const int k = list ? list[e] : e;
  const SubDev d = sub[k];
  if (d.nI == 0 || i >= d.nt) return;
  const SnDev s = sn[d.root];
  const double* M = base + (from_front ? s.front_off : s.inv_off);
  const long long ld = from_front ? s.ld : s.ldi;
  // S[c][r] = M(iTB + r, jTB + c), lower entries only (column c contiguous in r)
  for (int q = threadIdx.x; q < TILE_ELEMS; q += blockDim.x) {
    const int c = q >> 6, r = q & (TB - 1);
    const int R = i * TB + r, C = j * TB + c;
    S[c][r] = (R < d.nI && C < d.nI && R >= C) ? M[(long long)C * ld + R] : 0.0;
  }
  __syncthreads();
  double* T = dst + d.tile_off + (long long)t * TILE_ELEMS;
  for (int q = threadIdx.x; q < TILE_ELEMS; q += blockDim.x) {
    const int r = q >> 6, c = q & (TB - 1);
    T[swz(r, c)] = (i == j && r < c) ? S[r][c] : S[c][r];  // diagonal tile: mirror the lower part
  }
}

static void set_smem(const void* f, int bytes) {
  IETI_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void fwd_sweep_lp(ietidp_s* h, double* X, const LevelPlan& lp, cudaStream_t st);

// G_k^T = L_PI L_II^-1 for every subdomain (one DMMA GEMM launch; after k_pack's L_PI)
void launch_form_G(ietidp_s* h) {
  const Plan& P = h->plan;
  if (!P.g_n) return;
  set_smem((const void*)k_gemm<true, true>, GEMM_SMEM);
  k_gemm<true, true><<<P.g_n, 128, GEMM_SMEM, h->stream>>>(h->d_gwork.p + P.g_off, h->lpi.p, h->ipool.p, h->G.p,
                                                           h->d_rel.p);
  IETI_LAUNCHED(h);
}

void run_factor(ietidp_s* h) {
  cudaStream_t st = h->stream;
  const Plan& P = h->plan;
  static bool attr = false;
  if (!attr) {
    set_smem((const void*)k_gemm<false>, GEMM_SMEM);
    set_smem((const void*)k_gemm<true>, GEMM_SMEM);
    set_smem((const void*)k_gemm<true, true>, GEMM_SMEM);
    attr = true;
  }
  k_init_flags<<<1, 32, 0, st>>>(h->err_flag.p);  // failing subdomain (min), coarse OK
  IETI_LAUNCHED(h);
  const Work* W = reinterpret_cast<const Work*>(h->d_work.p);
  const GemmWork* GW = h->d_gwork.p;
  double* pool = h->pool.p;
  // assembly of the fronts, level by level: zero the lower trapezoids, scatter K's
  // entries. Level 0 on the main stream; the levels above on the side stream while
  // level 0 is factored (the main stream waits for them before the first SYRK).
  auto assemble = [&](const LevelPlan& lp, cudaStream_t sx) {
    if (lp.zr_n) {
      k_zero_fronts<<<lp.zr_n, 256, 0, sx>>>(W + lp.zr_off, h->d_sn.p, pool);
      if (sx == st) IETI_LAUNCHED(h); else IETI_LAUNCHED_SIDE(h);
    }
    if (lp.sc_n) {
      k_scatter<<<grid_for(lp.sc_n, 256), 256, 0, sx>>>(lp.sc_n, h->sc_front_dst.p + lp.sc_off,
                                                          h->sc_front_src.p + lp.sc_off, h->kval.p, pool);
      if (sx == st) IETI_LAUNCHED(h); else IETI_LAUNCHED_SIDE(h);
    }
  };
  const int* rel = h->d_rel.p;
  int maxnt = 0;
  for (auto& d : h->h_sub) maxnt = std::max(maxnt, d.nt);
  const bool expl = h->opt.loop == IETIDP_LOOP_EXPLICIT;
  // Streams. The subdomains are split into P.ngroups independent groups; group g runs
  // its panels and SYRKs level after level on its own high-priority stream gst[g]
  // (group 0 on the caller's stream), so that one group's latency-bound panels
  // overlap the other's GEMMs. Each group has a low-priority side stream gside[g] for
  // its partitioned inverse (started as soon as a level's / a panel's factors exist),
  // W_k and the forward sweep of the loads. One more side stream assembles the fronts
  // of levels >= 1 while level 0 is factored. Everything joins the caller's stream at
  // the end.
  const int nlev = P.max_level + 1, G = P.ngroups;
  if (!h->side) {
    IETI_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
    int lo = 0, hi = 0;
    IETI_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    h->gst.assign(G, nullptr);
    h->gside.assign(G, nullptr);
    for (int g = 0; g < G; ++g) {
      if (g > 0) IETI_CUDA(cudaStreamCreateWithPriority(&h->gst[g], cudaStreamNonBlocking, hi));
      IETI_CUDA(cudaStreamCreateWithFlags(&h->gside[g], cudaStreamNonBlocking));
    }
    h->fev.resize(4);
    for (auto& e : h->fev) IETI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->gev.resize((size_t)G * (nlev + 4));
    for (auto& e : h->gev) IETI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    size_t np = 0;
    for (auto& gl : P.glevels)
      for (auto& lv : gl) np += lv.panels.size();
    h->pev.resize(np);
    for (auto& e : h->pev) IETI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  auto gevent = [&](int g, int i) { return h->gev[(size_t)g * (nlev + 4) + i]; };
  // compact POTRF by default (measured faster in the pipeline: the instruction cache is
  // cold at every launch); IETIDP_POTRF=unrolled selects the fully unrolled kernel
  static const bool potrf_compact = !(getenv("IETIDP_POTRF") && !strcmp(getenv("IETIDP_POTRF"), "unrolled"));
  // experiments only (results meaningless): IETIDP_DBG_FACTOR bits skip launches: 1 POTRF,
  // 2 panel updates, 4 TRSM, 8 SYRK / extend-add, 16 side-stream inverse and W_k
  static const int dbgf = getenv("IETIDP_DBG_FACTOR") ? atoi(getenv("IETIDP_DBG_FACTOR")) : 0;
  // the forward sweep of the loads rides on the groups' side streams (one column chunk)
  h->fwd_in_factor = h->nrhs <= 16;
  if (expl) h->wtiles.zero(st);  // W_k is accumulated block row by block row
  if (h->fwd_in_factor) h->Xf.zero(st);
  IETI_CUDA(cudaEventRecord(h->fev[2], st));
  size_t npan = 0;
  for (int g = 0; g < G; ++g) {
    cudaStream_t sg = g == 0 ? st : h->gst[g];
    cudaStream_t s2 = h->gside[g];
    if (g > 0) IETI_CUDA(cudaStreamWaitEvent(sg, h->fev[2], 0));
    // the group's values (ietidp_set_values copies, recorded per subdomain)
    // (inside a graph capture as external wait nodes, so every replay waits for the
    // copies recorded before it)
    if (!h->kev.empty()) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      IETI_CUDA(cudaStreamIsCapturing(sg, &cs));
      const unsigned wflag = cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0;
      for (int k = 0; k < h->n_sub; ++k)
        if (P.sub_group[k] == g) IETI_CUDA(cudaStreamWaitEvent(sg, h->kev[k], wflag));
    }
    // assembly: level 0 here, the levels above on the side stream while level 0 is factored
    assemble(P.glevels[g][0], sg);
    if (h->fwd_in_factor && P.gfx[g].second) {
      k_scatter<<<grid_for(P.gfx[g].second, 256), 256, 0, sg>>>(P.gfx[g].second, h->sc_fx_dst.p + P.gfx[g].first,
                                                                  h->sc_fx_src.p + P.gfx[g].first, h->fval.p,
                                                                  h->Xf.p);
      IETI_LAUNCHED_SIDE(h);
    }
    IETI_CUDA(cudaEventRecord(gevent(g, nlev), sg));
    IETI_CUDA(cudaStreamWaitEvent(s2, gevent(g, nlev), 0));
    for (int L = 1; L < nlev; ++L) assemble(P.glevels[g][L], s2);
    IETI_CUDA(cudaEventRecord(gevent(g, nlev + 1), s2));  // the group's fronts assembled
    const LevelPlan::Panel* wacc_last = nullptr;
    for (int L = 0; L < nlev; ++L) {
      const LevelPlan& lp = P.glevels[g][L];
      // explicit loop: S_II is the assembled r_I root front before its factorisation
      const auto& rr = h->rootlist_range[g][L];
      if (expl && rr.second > 0) {
        k_pack_sym<<<rr.second * (maxnt * (maxnt + 1) / 2), 256, 0, sg>>>(h->d_rootlist.p + rr.first, maxnt,
                                                                          h->d_sub.p, h->d_sn.p, pool, 1,
                                                                          h->stiles.p);
        IETI_LAUNCHED_SIDE(h);
      }
      for (auto& pn : lp.panels) {
        if (pn.upd_n && !(dbgf & 2)) {
          k_gemm<false><<<pn.upd_n, 128, GEMM_SMEM, sg>>>(GW + pn.upd_off, pool, pool, pool, rel, h->skws.p,
                                                           h->skcnt.p);
          IETI_LAUNCHED_SIDE(h);
        }
        if (pn.potrf_n && !(dbgf & 1)) {
          if (potrf_compact)
            k_potrf_c<<<pn.potrf_n, POTRF_T, 0, sg>>>(W + pn.potrf_off, h->d_sn.p, pool, h->dinv.p, h->err_flag.p);
          else
            k_potrf<<<pn.potrf_n, POTRF_T, 0, sg>>>(W + pn.potrf_off, h->d_sn.p, pool, h->dinv.p, h->err_flag.p);
          IETI_LAUNCHED_SIDE(h);
        }
        cudaEvent_t pe = h->pev[npan++];
        IETI_CUDA(cudaEventRecord(pe, sg));
        if (pn.trsm_n && !(dbgf & 4)) {
          k_gemm<false><<<pn.trsm_n, 128, GEMM_SMEM, sg>>>(GW + pn.trsm_off, pool, h->dinv.p, pool, rel);
          IETI_LAUNCHED_SIDE(h);
        }
        // side stream: block row kp of L11^-1 (and of W_k) as soon as Dinv_kp exists
        if (pn.icopy_n || pn.ia_n || pn.ib_n || pn.wacc_n) IETI_CUDA(cudaStreamWaitEvent(s2, pe, 0));
        if (pn.icopy_n && !(dbgf & 16)) {
          k_inv_copy<<<pn.icopy_n, 256, 0, s2>>>(W + pn.icopy_off, h->d_sn.p, h->dinv.p, h->ipool.p);
          IETI_LAUNCHED_SIDE(h);
        }
        if (pn.ia_n && !(dbgf & 16)) {
          k_gemm<true><<<pn.ia_n, 128, GEMM_SMEM, s2>>>(GW + pn.ia_off, pool, h->ipool.p, h->tpool.p, rel);
          IETI_LAUNCHED_SIDE(h);
        }
        if (pn.ib_n && !(dbgf & 16)) {
          k_gemm<true><<<pn.ib_n, 128, GEMM_SMEM, s2>>>(GW + pn.ib_off, h->dinv.p, h->tpool.p, h->ipool.p, rel);
          IETI_LAUNCHED_SIDE(h);
        }
        if (&pn == &lp.panels.back()) {
          wacc_last = pn.wacc_n ? &pn : nullptr;  // after the level's forward sweep (not on the path)
        } else if (pn.wacc_n && !(dbgf & 16)) {
          k_gemm<true, true><<<pn.wacc_n, 128, GEMM_SMEM, s2>>>(GW + pn.wacc_off, h->ipool.p, h->ipool.p,
                                                                h->wtiles.p, rel);
          IETI_LAUNCHED_SIDE(h);
        }
      }
      IETI_CUDA(cudaEventRecord(gevent(g, L), sg));
      if (L == 0) IETI_CUDA(cudaStreamWaitEvent(sg, gevent(g, nlev + 1), 0));  // parents assembled
      for (auto& sy : lp.syrk) {
        if (dbgf & 8) break;
        k_gemm<false><<<sy.second, 128, GEMM_SMEM, sg>>>(GW + sy.first, pool, pool, pool, rel);
        IETI_LAUNCHED_SIDE(h);
      }
      // side stream: recursive-doubling L11^-1 of the level (if not formed per panel)
      IETI_CUDA(cudaStreamWaitEvent(s2, gevent(g, L), 0));  // the level's factors
      if (lp.inv_copy_n) {
        k_inv_copy<<<lp.inv_copy_n, 256, 0, s2>>>(W + lp.inv_copy_off, h->d_sn.p, h->dinv.p, h->ipool.p);
        IETI_LAUNCHED_SIDE(h);
      }
      for (size_t r = 0; r < lp.inv_rounds.size(); ++r) {
        const auto& rg = lp.inv_rounds[r];
        if (!rg.second || (dbgf & 16)) continue;
        const bool step1 = (r % 2) == 0;
        k_gemm<true><<<rg.second, 128, GEMM_SMEM, s2>>>(GW + rg.first, step1 ? pool : h->ipool.p,
                                                        step1 ? h->ipool.p : h->tpool.p,
                                                        step1 ? h->tpool.p : h->ipool.p, rel);
        IETI_LAUNCHED_SIDE(h);
      }
      if (h->fwd_in_factor) fwd_sweep_lp(h, h->Xf.p, lp, s2);
      if (wacc_last && !(dbgf & 16)) {
        k_gemm<true, true><<<wacc_last->wacc_n, 128, GEMM_SMEM, s2>>>(GW + wacc_last->wacc_off, h->ipool.p,
                                                                      h->ipool.p, h->wtiles.p, rel);
        IETI_LAUNCHED_SIDE(h);
        wacc_last = nullptr;
      }
    }
    // join: the group's main and side streams into the caller's stream
    IETI_CUDA(cudaEventRecord(gevent(g, nlev + 2), s2));
    IETI_CUDA(cudaStreamWaitEvent(st, gevent(g, nlev + 2), 0));
    if (g > 0) {
      IETI_CUDA(cudaEventRecord(gevent(g, nlev + 3), sg));
      IETI_CUDA(cudaStreamWaitEvent(st, gevent(g, nlev + 3), 0));
    }
  }
  IETI_CHECK_LAUNCH();
}

}  // namespace ieti
