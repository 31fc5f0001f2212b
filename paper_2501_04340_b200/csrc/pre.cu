// Device pre-processing in front of the solve phase (include/ietidp_pre.h):
// torn per-subdomain assembly K^(k) = C^T M_2(nu) C, j^(k) = C^T t and
// the tree-cotree gauge with the primal selection.
//
// Assembly pipeline of one box subdomain (all stages are kernels of this file):
//   k_basis      spline values at the quadrature points (Cox-de Boor), B and D kinds
//   k_gram       1-D Gram blocks per (2-form component, axis, patch)
//   k_load1d     1-D load integrals per (axis, factor)
//   k_rows<0>    a warp per DOF row walks the candidate columns in ascending order and
//                counts the structural non-zeros of C^T M_2 C
//   k_scan       row pointers
//   k_rows<1>    the same walk; every structural entry's value is the signed sum over
//                the (at most 8) face pairs of sum_patches nu * Gx * Gy * Gz
//   k_loads      j = C^T t, t_f from the separable terms
// Spanning tree: Boruvka rounds (k_bv_*), identical to Kruskal's tree under a total order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "ietidp.h"
#include "ietidp_pre.h"

namespace {

thread_local std::string g_err;

int fail(int st, const std::string& m) {
  g_err = m;
  return st;
}

#define PRE_CUDA(x)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      throw std::make_pair((int)(e_ == cudaErrorMemoryAllocation ? IETIDP_E_NOMEM : IETIDP_E_CUDA), \
                           std::string(#x ": ") + cudaGetErrorString(e_));                   \
  } while (0)

template <class T>
struct Buf {
  T* p = nullptr;
  size_t n = 0;
  Buf() = default;
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  ~Buf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    reset();
    n = count;
    PRE_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  }
  void upload(const T* src, size_t count) {
    alloc(count);
    if (count) PRE_CUDA(cudaMemcpy(p, src, count * sizeof(T), cudaMemcpyHostToDevice));
  }
};

constexpr int MAXP = 3;

// Geometry of one box and the device tables, passed by value to the kernels.
struct Box {
  int p, e, s;      // degree, elements per patch, s = e + p - 1 functions per patch step
  int np[3], m[3];  // patches and control vertices per axis
  int E[3][3];      // edge grids E[d][a]
  int F[3][3];      // face grids F[c][a]
  long long eoff[4];
  int nb[2];          // block sizes of the B and D kinds: s + 1, s
  int goff[3][3];     // offset (doubles) of the Gram blocks of (c, a) in `gram`
  int gtotal;
  const double* gram;
  const double* nu;
  const int* dof_of_edge;
  const int* edge_of_dof;
  int n_dof;
  int R, W;  // column reach p + 1 per axis, W = 2R + 1
  // inputs and scratch of the 1-D stage (device pointers into the batch arena)
  int nq, lq, nrhs, nterms;
  const double* knots[3];
  const double* qx[3];
  const double* qw[3][3];
  const double* lx[3];
  const double* facv[3];
  const int* fac_kind[3];
  int nfac[3];
  double* tabq[3][2];  // spline tables at the Gram points / load points, per axis and kind
  double* tabl[3][2];
  double* v1d[3];      // 1-D load integrals, factor-major with stride m[a]
  double* gram_w;      // = gram (written by the 1-D stage)
  double* ktab;        // value tables of k_entry (diff_tables), ktotal doubles
  int ktotal;
  int* tables;         // k_tables layout
  const int* term_ptr;
  const int* term_fac;
  const double* term_coef;
  // outputs
  int* cnt;
  long long* rowptr;
  long long* nnz_out;
  int* col;
  double* val;
  double* f;
};

// One B-spline of degree `deg` on knots t, index i, at x (Cox-de Boor triangle on the
// functions' own p + 1 spans; x is interior to an element).
__device__ double one_bspline(const double* __restrict__ t, int deg, int i, double x) {
  double N[MAXP + 1];
  for (int j = 0; j <= deg; ++j) N[j] = (x >= t[i + j] && x < t[i + j + 1]) ? 1.0 : 0.0;
  for (int k = 1; k <= deg; ++k)
    for (int j = 0; j <= deg - k; ++j) {
      const double d1 = t[i + j + k] - t[i + j], d2 = t[i + j + k + 1] - t[i + j + 1];
      double v = 0.0;
      if (d1 > 0.0) v += (x - t[i + j]) / d1 * N[j];
      if (d2 > 0.0) v += (t[i + j + k + 1] - x) / d2 * N[j + 1];
      N[j] = v;
    }
  return N[0];
}

// tab[u * nb + l] = value at point u of the l-th function of the point's patch
// (function index q*s + l); kind 0: B_{i,p}; kind 1: D_j = p/(t_{j+p+1}-t_{j+1}) B_{j+1,p-1}.
__device__ void basis_table(const double* __restrict__ t, int p, int s, int kind, int nb, int pts_per_patch, int npts,
                            const double* __restrict__ x, double* __restrict__ tab) {
  for (int idx = threadIdx.x; idx < npts * nb; idx += blockDim.x) {
    const int u = idx / nb, l = idx - u * nb;
    const int q = u / pts_per_patch;
    const int i = q * s + l;
    double v;
    if (kind == 0) {
      v = one_bspline(t, p, i, x[u]);
    } else {
      v = p / (t[i + p + 1] - t[i + 1]) * one_bspline(t, p - 1, i + 1, x[u]);
    }
    tab[idx] = v;
  }
}

// Gram blocks of one (component, axis): G_q[fl + nb*gl] = sum_u (phi_f phi_g) w_u over patch q.
__device__ void gram_blocks(const double* __restrict__ tab, const double* __restrict__ w, int nb, int pts_per_patch, int np,
                            double* __restrict__ out) {
  for (int idx = threadIdx.x; idx < np * nb * nb; idx += blockDim.x) {
    const int q = idx / (nb * nb), r = idx - q * nb * nb;
    const int fl = r % nb, gl = r / nb;
    double acc = 0.0;
    for (int u = q * pts_per_patch; u < (q + 1) * pts_per_patch; ++u) acc += (tab[u * nb + fl] * tab[u * nb + gl]) * w[u];
    out[idx] = acc;
  }
}

// v[i] = sum over the points of the patches carrying function i of fw[u] * phi_i(x_u).
__device__ void load1d(const double* __restrict__ tab, const double* __restrict__ fw, int kind, int nb, int s, int np,
                       int pts_per_patch, int dim, double* __restrict__ v) {
  for (int i = threadIdx.x; i < dim; i += blockDim.x) {
    double acc = 0.0;
    int q0 = i / s, q1 = q0;
    if (kind == 0 && i % s == 0 && i > 0) q0 = q1 - 1;  // shared by two patches
    if (q1 >= np) q1 = np - 1;
    for (int q = q0; q <= q1; ++q) {
      const int l = i - q * s;
      for (int u = q * pts_per_patch; u < (q + 1) * pts_per_patch; ++u) acc += tab[u * nb + l] * fw[u];
    }
    v[i] = acc;
  }
}

struct Edge {
  int d, n[3];
};

__device__ __forceinline__ Edge edge_of(const Box& b, int eid) {
  Edge e;
  e.d = eid >= b.eoff[2] ? 2 : (eid >= b.eoff[1] ? 1 : 0);
  int r = eid - (int)b.eoff[e.d];
  e.n[0] = r % b.E[e.d][0];
  r /= b.E[e.d][0];
  e.n[1] = r % b.E[e.d][1];
  e.n[2] = r / b.E[e.d][1];
  return e;
}

// The patches carrying both 1-D functions fa and ga of the given kind on an axis with np
// patches (0, 1 or 2 of them), with the local indices inside each.
__device__ __forceinline__ int shared_patches(int kind, int s, int np, int fa, int ga, int (&q)[2]) {
  int cnt = 0;
  if (kind == 1) {
    const int qa = fa / s;
    if (qa == ga / s) q[cnt++] = qa;
    return cnt;
  }
  const int hi = min(fa / s, ga / s);
  int lo = max(fa % s == 0 ? fa / s - 1 : fa / s, ga % s == 0 ? ga / s - 1 : ga / s);
  if (lo < 0) lo = 0;
  for (int c = lo; c <= hi && c < np; ++c) q[cnt++] = c;
  return cnt;
}

// ---- 1-D lookup tables (k_tables): the structural test and the patch ranges per axis ----
constexpr int MAXM = 128;  // control vertices per axis of one box
enum { T_CB = 0, T_CD, T_SD, T_SSD, T_PB, T_PD, T_COUNT };
__device__ __forceinline__ int tb_at(int type, int a, int i) { return (type * 3 + a) * MAXM + i; }

// Gram entry (i, j) of the given kind on axis a is structurally non-zero: both functions on
// a common patch and within the band (p for B, p - 1 for D).
__device__ bool compat1d(const Box& b, int a, int kind, int i, int j) {
  const int dim = b.m[a] - kind;
  if (i < 0 || j < 0 || i >= dim || j >= dim) return false;
  const int band = kind == 0 ? b.p : b.p - 1;
  if (i - j > band || j - i > band) return false;
  int q[2];
  return shared_patches(kind, b.s, b.np[a], i, j, q) > 0;
}

// Bit (delta + R) of the masks at coordinate i of axis a, delta in [-R, R]:
//   CB  compat_B(i, i + delta)                 both coordinates index B functions
//   CD  compat_D(i, i + delta)                 both index D functions
//   SD  exists o in {0,1}: compat_D(i - o, i + delta)           i an edge coordinate across its
//                                              direction (its faces sit at i and i - 1)
//   SSD exists o1, o2: compat_D(i - o1, i + delta - o2)
// PB: lowest | highest << 16 patch carrying B function i; PD: the patch of D function i.
__device__ void struct_tables(const Box& b, int* __restrict__ tb) {
  for (int idx = threadIdx.x; idx < 3 * MAXM; idx += blockDim.x) {
    const int a = idx / MAXM, i = idx % MAXM;
    unsigned cb = 0, cd = 0, sd = 0, ssd = 0;
    int pb = 0, pd = 0;
    if (i < b.m[a]) {
      for (int dl = -b.R; dl <= b.R; ++dl) {
        const unsigned bit = 1u << (dl + b.R);
        const int j = i + dl;
        if (compat1d(b, a, 0, i, j)) cb |= bit;
        if (compat1d(b, a, 1, i, j)) cd |= bit;
        if (compat1d(b, a, 1, i, j) || compat1d(b, a, 1, i - 1, j)) sd |= bit;
        if (compat1d(b, a, 1, i, j) || compat1d(b, a, 1, i - 1, j) || compat1d(b, a, 1, i, j - 1) ||
            compat1d(b, a, 1, i - 1, j - 1))
          ssd |= bit;
      }
      const int lo = max(i % b.s == 0 ? i / b.s - 1 : i / b.s, 0), hi = min(i / b.s, b.np[a] - 1);
      pb = lo | (hi << 16);
      pd = min(i / b.s, b.np[a] - 1);
    }
    tb[tb_at(T_CB, a, i)] = (int)cb;
    tb[tb_at(T_CD, a, i)] = (int)cd;
    tb[tb_at(T_SD, a, i)] = (int)sd;
    tb[tb_at(T_SSD, a, i)] = (int)ssd;
    tb[tb_at(T_PB, a, i)] = pb;
    tb[tb_at(T_PD, a, i)] = pd;
  }
}

// ---- value tables: the face shifts folded into 1-D difference tables ----
// Every edge has, per 2-form component c, exactly one axis on which its two faces differ (the
// shift axis), and C's two entries there are +s and -s. With M_2[f, g] = sum_patches nu Gz Gy Gx
// the signed sums over the shifts therefore move inside the per-axis factors:
//   K[e1, e2] = sum_c s1 s2 sum_patches q nu_q prod_a T_a(q_a),
// T_a = the B Gram block G^B_q[n, n'] on a = c, and on the D axes, by which of the two
// coordinates is a shifted (edge-across) one,
//   T00 = Gd(l, l'), T10 = Gd(l, l') - Gd(l-1, l'), T11 = Gd(l, l') - Gd(l-1, l') - Gd(l, l'-1)
//   + Gd(l-1, l'-1)   (T01 = T10 transposed; Gd = G^D_q, zero outside its s x s block),
// in patch-local coordinates l = n - q s in [0, s]. Slot layout per (axis a, patch q), blocks
// of S1 x S1 doubles (S1 = s + 1): slot 0 = G^B of c = a; slots 1 + 3 ci + {0, 1, 2} =
// T00, T10, T11 of the ci-th component other than a.
__device__ __forceinline__ int kt_at(const Box& b, int a, int slot, int q) {
  const int before = a == 0 ? 0 : (a == 1 ? b.np[0] : b.np[0] + b.np[1]);  // patches of the axes before a
  return (7 * before + slot * b.np[a] + q) * (b.s + 1) * (b.s + 1);
}

__device__ void diff_tables(const Box& b) {
  const int S1 = b.s + 1, s = b.s;
  for (int a = 0; a < 3; ++a)
    for (int slot = 0; slot < 7; ++slot) {
      const int ci = (slot - 1) / 3, kind = (slot - 1) % 3;
      int c = a;
      if (slot > 0) c = ci + (ci >= a ? 1 : 0);  // the ci-th component other than a
      const double* G = b.gram + b.goff[c][a];
      const int nb = b.nb[slot == 0 ? 0 : 1];
      for (int idx = threadIdx.x; idx < b.np[a] * S1 * S1; idx += blockDim.x) {
        const int q = idx / (S1 * S1), r = idx - q * S1 * S1;
        const int l = r % S1, l2 = r / S1;
        const double* Gq = G + q * nb * nb;
        auto g = [&](int i, int j) { return (i >= 0 && j >= 0 && i < nb && j < nb) ? Gq[i + nb * j] : 0.0; };
        double v;
        if (slot == 0) v = g(l, l2);
        else if (kind == 0) v = (l < s && l2 < s) ? g(l, l2) : 0.0;
        else if (kind == 1) v = l2 < s ? g(l, l2) - g(l - 1, l2) : 0.0;
        else v = (g(l, l2) - g(l - 1, l2)) - (g(l, l2 - 1) - g(l - 1, l2 - 1));
        b.ktab[kt_at(b, a, slot, q) + l + S1 * l2] = v;
      }
    }
}

// K[e1, e2] from the value tables (kt) and the patch table T_PD (tb), both in shared memory.
__device__ __forceinline__ double k_entry(const Box& b, const double* kt, const int* tb, const Edge& e1, const Edge& e2) {
  const int S1 = b.s + 1;
  double acc = 0.0;
  for (int c = 0; c < 3; ++c) {
    if (c == e1.d || c == e2.d) continue;
    // (c, a, b) cyclic: C[f(n), edge_a(n)] = +1, C[f(n), edge_b(n)] = -1
    const double sg = ((c == (e1.d + 1) % 3) ? -1.0 : 1.0) * ((c == (e2.d + 1) % 3) ? -1.0 : 1.0);
    double t[3][2];
    int q0[3], nq[3];
    bool any = true;
    for (int a = 0; a < 3 && any; ++a) {
      const int n1 = e1.n[a], n2 = e2.n[a];
      const int mn = min(n1, n2), mx = max(n1, n2);
      const int qhi = tb[tb_at(T_PD, a, mn)], qlo = mx ? tb[tb_at(T_PD, a, mx - 1)] : 0;
      q0[a] = qlo;
      nq[a] = qhi - qlo + 1;
      if (nq[a] <= 0) {
        any = false;
        break;
      }
      int slot = 0;
      bool swap = false;
      if (a != c) {
        const bool sh1 = a != e1.d, sh2 = a != e2.d;
        slot = 1 + 3 * (c - (c > a ? 1 : 0)) + (sh1 ? (sh2 ? 2 : 1) : (sh2 ? 1 : 0));
        swap = !sh1 && sh2;
      }
      for (int i = 0; i < 2; ++i) {
        if (i >= nq[a]) break;
        const int q = qlo + i;
        const int l1 = n1 - q * b.s, l2 = n2 - q * b.s;
        t[a][i] = kt[kt_at(b, a, slot, q) + (swap ? l2 + S1 * l1 : l1 + S1 * l2)];
      }
    }
    if (!any) continue;
    double part = 0.0;
    for (int iz = 0; iz < nq[2]; ++iz)
      for (int iy = 0; iy < nq[1]; ++iy)
        for (int ix = 0; ix < nq[0]; ++ix)
          part += b.nu[(q0[0] + ix) + b.np[0] * ((q0[1] + iy) + b.np[1] * (q0[2] + iz))] * (t[2][iz] * (t[1][iy] * t[0][ix]));
    acc += sg * part;
  }
  return acc;
}

// Whether K[e1, e2] has a structurally non-zero face pair. The face shifts act on one axis
// each, so the test factorises into the per-axis masks of k_tables; dl = e2.n - e1.n.
__device__ __forceinline__ bool k_struct(const Box& b, const int* tb, const Edge& e1, const Edge& e2) {
  auto bit = [&](int type, int a, int i, int dl) { return (tb[tb_at(type, a, i)] >> (dl + b.R)) & 1; };
  const int dl[3] = {e2.n[0] - e1.n[0], e2.n[1] - e1.n[1], e2.n[2] - e1.n[2]};
  if (e1.d != e2.d) {
    const int c = 3 - e1.d - e2.d, d1 = e1.d, d2 = e2.d;
    // axis c: B on both; axis d2: e1 across (shifted), e2 along; axis d1: e1 along, e2 across
    return bit(T_CB, c, e1.n[c], dl[c]) && bit(T_SD, d2, e1.n[d2], dl[d2]) && bit(T_SD, d1, e2.n[d1], -dl[d1]);
  }
  const int d = e1.d;
  if (!bit(T_CD, d, e1.n[d], dl[d])) return false;
  for (int c = 0; c < 3; ++c) {
    if (c == d) continue;
    const int r = 3 - c - d;
    if (bit(T_CB, c, e1.n[c], dl[c]) && bit(T_SSD, r, e1.n[r], dl[r])) return true;
  }
  return false;
}

// Candidate column of a row edge e1, packed as direction << 12 | dz << 8 | dy << 4 | dx with
// the offsets dl + R in 0 .. W-1: ascending in the DOF order when compared as integers.
__device__ __forceinline__ Edge unpack_candidate(const Box& b, const Edge& e1, int pk) {
  Edge e2;
  e2.d = pk >> 12;
  e2.n[0] = e1.n[0] + (pk & 15) - b.R;
  e2.n[1] = e1.n[1] + ((pk >> 4) & 15) - b.R;
  e2.n[2] = e1.n[2] + ((pk >> 8) & 15) - b.R;
  return e2;
}
__device__ __forceinline__ int dof_at(const Box& b, const Edge& e) {
  return b.dof_of_edge[b.eoff[e.d] + e.n[0] + (long long)b.E[e.d][0] * (e.n[1] + (long long)b.E[e.d][1] * e.n[2])];
}

// Per-axis mask of the offsets dl (bit dl + R) at which a column edge of direction d2 can
// couple to the row edge e1: inside the edge grid, and the axis' factor of k_struct (for
// d2 = e1.d the union of the two components' factors; k_struct decides).
__device__ __forceinline__ unsigned axis_mask(const Box& b, const int* tb, const Edge& e1, int d2, int a) {
  const int d1 = e1.d, n = e1.n[a];
  unsigned m = 0;
  for (int dl = -b.R; dl <= b.R; ++dl) {
    const int j = n + dl;
    if (j < 0 || j >= b.E[d2][a]) continue;
    const int sh = dl + b.R;
    int ok;
    if (d2 != d1) {
      const int c = 3 - d1 - d2;
      if (a == c) ok = (tb[tb_at(T_CB, a, n)] >> sh) & 1;
      else if (a == d2) ok = (tb[tb_at(T_SD, a, n)] >> sh) & 1;
      else ok = (tb[tb_at(T_SD, a, j)] >> (b.R - dl)) & 1;
    } else if (a == d1) {
      ok = (tb[tb_at(T_CD, a, n)] >> sh) & 1;
    } else {
      ok = ((tb[tb_at(T_CB, a, n)] | tb[tb_at(T_SSD, a, n)]) >> sh) & 1;
    }
    m |= (unsigned)ok << sh;
  }
  return m;
}

constexpr int ROWS_WARPS = 8;

// positions of the set bits of m (at most 16 of them), 4 bits each, ascending
__device__ __forceinline__ unsigned long long pack_bits(unsigned m) {
  unsigned long long p = 0;
  for (int k = 0; m; ++k, m &= m - 1) p |= (unsigned long long)(__ffs(m) - 1) << (4 * k);
  return p;
}

// A warp per DOF row; blockIdx.y = subdomain of the batch. Lanes 0..8 build the row's nine
// per-axis offset masks (column direction x axis); the candidate columns are the products of
// their set bits, walked in ascending DOF order 32 at a time, tested exactly (k_struct,
// Dirichlet mask) and ballot-compacted. FILL = 0: cnt[row] = the number of entries.
// FILL = 1: the compacted candidates go to the warp's shared-memory strip first, then all 32
// lanes evaluate entries (columns and values at rowptr[row], coalesced).
template <int FILL>
__global__ void __launch_bounds__(32 * ROWS_WARPS) k_rows(const Box* __restrict__ boxes) {
  extern __shared__ double sgram[];
  __shared__ int tb[T_COUNT * 3 * MAXM];
  __shared__ Box b;
  if (threadIdx.x == 0) b = boxes[blockIdx.y];
  __syncthreads();
  if (blockIdx.x * ROWS_WARPS >= b.n_dof) return;
  for (int i = threadIdx.x; i < T_COUNT * 3 * MAXM; i += blockDim.x) tb[i] = b.tables[i];
  if (FILL)
    for (int i = threadIdx.x; i < b.ktotal; i += blockDim.x) sgram[i] = b.ktab[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ncand = 3 * b.W * b.W * b.W;
  unsigned short* strip = reinterpret_cast<unsigned short*>(sgram + ((b.ktotal + 1) & ~1)) + (size_t)warp * ((ncand + 7) & ~7);
  for (int row = blockIdx.x * ROWS_WARPS + warp; row < b.n_dof; row += gridDim.x * ROWS_WARPS) {
    const Edge e1 = edge_of(b, b.edge_of_dof[row]);
    const unsigned mine = lane < 9 ? axis_mask(b, tb, e1, lane / 3, lane % 3) : 0u;
    int count = 0;
    for (int d2 = 0; d2 < 3; ++d2) {
      const unsigned mx = __shfl_sync(0xffffffffu, mine, d2 * 3), my = __shfl_sync(0xffffffffu, mine, d2 * 3 + 1),
                     mz = __shfl_sync(0xffffffffu, mine, d2 * 3 + 2);
      const int nx = __popc(mx), nxy = nx * __popc(my);
      if (nxy == 0) continue;
      const unsigned long long px = pack_bits(mx), py = pack_bits(my);  // set-bit positions, 4 bits each
      const int inv = 65536 / nx + 1;                                   // t / nx = (t * inv) >> 16 for t < 128
      for (unsigned mzz = mz; mzz; mzz &= mzz - 1) {                    // z offsets ascending (uniform)
        const int dz = __ffs(mzz) - 1;
        for (int base = 0; base < nxy; base += 32) {
          const int t = base + lane;
          bool ok = t < nxy;
          int pk = 0;
          if (ok) {
            const int iy = (t * inv) >> 16, ix = t - iy * nx;
            pk = (d2 << 12) | (dz << 8) | ((int)((py >> (4 * iy)) & 15) << 4) | (int)((px >> (4 * ix)) & 15);
            const Edge e2 = unpack_candidate(b, e1, pk);
            ok = (d2 != e1.d || k_struct(b, tb, e1, e2)) && dof_at(b, e2) >= 0;
          }
          const unsigned mask = __ballot_sync(0xffffffffu, ok);
          if (FILL && ok) strip[count + __popc(mask & ((1u << lane) - 1u))] = (unsigned short)pk;
          count += __popc(mask);
        }
      }
    }
    if (!FILL) {
      if (lane == 0) b.cnt[row] = count;
      continue;
    }
    __syncwarp();
    const long long pos = b.rowptr[row];
    for (int t = lane; t < count; t += 32) {
      const Edge e2 = unpack_candidate(b, e1, strip[t]);
      const int dof2 = dof_at(b, e2);
      b.col[pos + t] = dof2;
      // exactly symmetric: both (i, j) and (j, i) evaluate the pair (min, max)
      b.val[pos + t] = dof2 < row ? k_entry(b, sgram, tb, e2, e1) : k_entry(b, sgram, tb, e1, e2);
    }
    __syncwarp();
  }
}

// The 1-D stage of a batch: one CTA per subdomain evaluates the spline tables, then the Gram
// blocks, the load integrals and the structural tables.
__global__ void __launch_bounds__(256) k_stage1d(const Box* __restrict__ boxes) {
  __shared__ Box b;
  if (threadIdx.x == 0) b = boxes[blockIdx.x];
  __syncthreads();
  for (int a = 0; a < 3; ++a)
    for (int k = 0; k < 2; ++k) {
      basis_table(b.knots[a], b.p, b.s, k, b.nb[k], b.e * b.nq, b.np[a] * b.e * b.nq, b.qx[a], b.tabq[a][k]);
      if (b.nterms > 0)
        basis_table(b.knots[a], b.p, b.s, k, b.nb[k], b.e * b.lq, b.np[a] * b.e * b.lq, b.lx[a], b.tabl[a][k]);
    }
  __syncthreads();
  for (int c = 0; c < 3; ++c)
    for (int a = 0; a < 3; ++a) {
      const int k = a == c ? 0 : 1;
      gram_blocks(b.tabq[a][k], b.qw[c][a], b.nb[k], b.e * b.nq, b.np[a], b.gram_w + b.goff[c][a]);
    }
  if (b.nterms > 0)
    for (int a = 0; a < 3; ++a) {
      const int lpp = b.e * b.lq, lpts = b.np[a] * lpp;
      for (int fi = 0; fi < b.nfac[a]; ++fi) {
        const int k = b.fac_kind[a][fi];
        load1d(b.tabl[a][k], b.facv[a] + (size_t)fi * lpts, k, b.nb[k], b.s, b.np[a], lpp, b.m[a] - k, b.v1d[a] + (size_t)fi * b.m[a]);
      }
    }
  struct_tables(b, b.tables);
  __syncthreads();  // the Gram blocks are complete (global writes of this CTA)
  diff_tables(b);
}

// rowptr[0..n] = exclusive prefix sums of cnt; one CTA per subdomain (n is a few thousand).
__global__ void __launch_bounds__(1024) k_scan(const Box* __restrict__ boxes) {
  __shared__ long long part[1024];
  const int* cnt = boxes[blockIdx.x].cnt;
  long long* rowptr = boxes[blockIdx.x].rowptr;
  const int n = boxes[blockIdx.x].n_dof;
  const int t = threadIdx.x;
  const int per = (n + 1023) / 1024;
  const int lo = min(t * per, n), hi = min(lo + per, n);
  long long s = 0;
  for (int i = lo; i < hi; ++i) s += cnt[i];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const long long v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  long long run = t ? part[t - 1] : 0;
  for (int i = lo; i < hi; ++i) {
    rowptr[i] = run;
    run += cnt[i];
  }
  if (t == 1023) {
    rowptr[n] = part[1023];
    *boxes[blockIdx.x].nnz_out = part[1023];
  }
}

// j[dof, col] = sum over the (at most 4) faces of the edge of C_f,e * t_f,
// t_f = sum_terms coef * vx[f_x] vy[f_y] vz[f_z]; blockIdx.y = subdomain.
__global__ void __launch_bounds__(256) k_loads(const Box* __restrict__ boxes) {
  __shared__ Box b;
  if (threadIdx.x == 0) b = boxes[blockIdx.y];
  __syncthreads();
  const long long total = (long long)b.n_dof * b.nrhs;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(idx % b.n_dof), colr = (int)(idx / b.n_dof);
    double acc = 0.0;
    if (b.nterms > 0) {
      const Edge e = edge_of(b, b.edge_of_dof[row]);
      for (int c = 0; c < 3; ++c) {
        if (c == e.d) continue;
        const int r = 3 - c - e.d;
        const double sn = (c == (e.d + 1) % 3) ? -1.0 : 1.0;
        const int t0 = b.term_ptr[colr * 3 + c], t1 = b.term_ptr[colr * 3 + c + 1];
        if (t0 == t1) continue;
        for (int o = 0; o < 2; ++o) {
          int f[3] = {e.n[0], e.n[1], e.n[2]};
          f[r] -= o;
          if (f[r] < 0 || f[r] >= b.F[c][r]) continue;
          double tf = 0.0;
          for (int t = t0; t < t1; ++t) {
            const int* fc = b.term_fac + 3 * t;
            tf += b.term_coef[t] * (b.v1d[2][(size_t)fc[2] * b.m[2] + f[2]] *
                                    (b.v1d[1][(size_t)fc[1] * b.m[1] + f[1]] * b.v1d[0][(size_t)fc[0] * b.m[0] + f[0]]));
          }
          acc += (o ? -sn : sn) * tf;
        }
      }
    }
    b.f[idx] = acc;
  }
}

// ---- spanning forest: Boruvka rounds under the total order (w, e) ----
constexpr unsigned long long KEY_NONE = ~0ull;
constexpr int KEY_SHIFT = 40;

__global__ void k_bv_init(long long nv, int* comp) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nv) comp[v] = (int)v;
}
__global__ void k_bv_reset(long long nv, unsigned long long* best) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nv) best[v] = KEY_NONE;
}
__global__ void k_bv_min(long long ne, const int* __restrict__ eu, const int* __restrict__ ev, const int8_t* __restrict__ w,
                         const int* __restrict__ comp, unsigned long long* best) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int cu = comp[eu[e]], cv = comp[ev[e]];
  if (cu == cv) return;
  const unsigned long long key = ((unsigned long long)w[e] << KEY_SHIFT) | (unsigned long long)e;
  atomicMin(&best[cu], key);
  atomicMin(&best[cv], key);
}
// every component root takes its lightest outgoing edge and hooks onto the other side
__global__ void k_bv_pick(long long nv, const int* __restrict__ eu, const int* __restrict__ ev, const int* __restrict__ comp,
                          const unsigned long long* __restrict__ best, int* parent, uint8_t* in_tree, int* changed) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  int par = comp[v];
  if (par == (int)v && best[v] != KEY_NONE) {
    const long long e = (long long)(best[v] & ((1ull << KEY_SHIFT) - 1ull));
    in_tree[e] = 1;
    const int cu = comp[eu[e]], cv = comp[ev[e]];
    par = cu == (int)v ? cv : cu;
    *changed = 1;
  }
  parent[v] = par;
}
// two roots that chose the same edge point at each other: the smaller id stays a root
__global__ void k_bv_break(long long nv, int* parent) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int o = parent[v];
  if (o != (int)v && (int)v < o && parent[o] == (int)v) parent[v] = (int)v;
}
__global__ void k_bv_flatten(long long nv, const int* __restrict__ parent, int* comp) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  int r = parent[v];
  while (parent[r] != r) r = parent[r];
  comp[v] = r;
}
__global__ void k_primal(long long ne, const int8_t* __restrict__ w, const uint8_t* __restrict__ in_tree, uint8_t* primal) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < ne) primal[e] = (!in_tree[e] && w[e] == 2) ? 1 : 0;
}

// One batch of assembled subdomains: a single device arena for the inputs and the 1-D
// scratch, shared outputs, one Box per subdomain.
struct PreBatch {
  int device = 0, n = 0;
  std::vector<Box> boxes;            // host copies (device pointers inside)
  std::vector<long long> nnz;
  Buf<char> arena;
  Buf<Box> d_boxes;
  Buf<long long> rowptr, d_nnz;
  Buf<int> cnt, col;
  Buf<double> val, f;
  double ms = 0.0, ms_fill = 0.0;
  std::vector<size_t> nu_off, nu_cnt;  // arena offsets / counts of every subdomain's nu
  int gx = 1, smem = 0;                // launch shape of k_rows
};

}  // namespace

struct ietidp_pre_s {
  std::shared_ptr<PreBatch> batch;
  int idx = 0;
};

namespace {

// host staging of the arena: 16-byte aligned pieces
struct Stage {
  std::vector<char> host;
  size_t put(const void* src, size_t bytes) {
    const size_t off = (host.size() + 15) & ~size_t(15);
    host.resize(off + bytes);
    if (src && bytes) memcpy(host.data() + off, src, bytes);
    return off;
  }
  size_t reserve(size_t bytes) { return put(nullptr, bytes); }
};

// Validate one descriptor and lay out its Box; offsets (not yet pointers) are recorded in `fix`.
struct Fix {
  size_t knots[3], qx[3], qw[3][3], lx[3], facv[3], fac_kind[3], tabq[3][2], tabl[3][2], v1d[3], gram, ktab, nu, dof_of_edge,
      edge_of_dof, tables, term_ptr, term_fac, term_coef;
};

int layout_box(const ietidp_pre_subdomain* s, Box& b, Fix& fx, Stage& st) {
  if (!s) return fail(IETIDP_E_ARG, "null descriptor");
  if (s->p < 1 || s->p > MAXP || s->e < 1 || s->nq < 1 || s->n_dof < 0 || s->nrhs < 0)
    return fail(IETIDP_E_ARG, "degree must be 1..3, e, nq >= 1");
  for (int a = 0; a < 3; ++a) {
    if (s->npatch[a] < 1 || !s->knots[a] || !s->qx[a]) return fail(IETIDP_E_ARG, "npatch >= 1, knots and qx required");
    for (int c = 0; c < 3; ++c)
      if (!s->qw[c][a]) return fail(IETIDP_E_ARG, "qw[c][a] required");
  }
  if (!s->nu || !s->dof_of_edge) return fail(IETIDP_E_ARG, "nu and dof_of_edge required");
  const bool loads = s->nrhs > 0 && s->nterms > 0;
  if (loads) {
    if (s->lq < 1 || !s->term_col || !s->term_comp || !s->term_fac || !s->term_coef)
      return fail(IETIDP_E_ARG, "load terms incomplete");
    for (int a = 0; a < 3; ++a)
      if (!s->lx[a] || s->nfac[a] < 1 || !s->fac_kind[a] || !s->fac_val[a]) return fail(IETIDP_E_ARG, "load factors incomplete");
  }
  b = Box{};
  b.p = s->p;
  b.e = s->e;
  b.s = s->e + s->p - 1;
  b.nb[0] = b.s + 1;
  b.nb[1] = b.s;
  b.R = s->p + 1;
  b.W = 2 * b.R + 1;
  b.nq = s->nq;
  b.lq = loads ? s->lq : 1;
  b.nrhs = std::max(s->nrhs, 0);
  b.nterms = loads ? s->nterms : 0;
  b.n_dof = s->n_dof;
  long long nedge = 0;
  for (int a = 0; a < 3; ++a) {
    b.np[a] = s->npatch[a];
    b.m[a] = b.np[a] * b.s + 1;
  }
  for (int d = 0; d < 3; ++d) {
    b.eoff[d] = nedge;
    long long sz = 1;
    for (int a = 0; a < 3; ++a) {
      b.E[d][a] = b.m[a] - (a == d ? 1 : 0);
      b.F[d][a] = b.m[a] - (a != d ? 1 : 0);
      sz *= b.E[d][a];
    }
    nedge += sz;
  }
  b.eoff[3] = nedge;
  if (nedge > (1ll << 30) || std::max({b.m[0], b.m[1], b.m[2]}) > MAXM) return fail(IETIDP_E_ARG, "box too large");
  // DOF map: ascending with the edge id
  std::vector<int> edge_of_dof(s->n_dof);
  int next = 0;
  for (long long eid = 0; eid < nedge; ++eid) {
    const int d = s->dof_of_edge[eid];
    if (d < 0) continue;
    if (d != next || d >= s->n_dof) return fail(IETIDP_E_ARG, "dof_of_edge must number the DOFs 0..n_dof-1 in edge order");
    edge_of_dof[next++] = (int)eid;
  }
  if (next != s->n_dof) return fail(IETIDP_E_ARG, "dof_of_edge does not cover n_dof DOFs");
  // load terms grouped by (column, component); factor kinds checked against the component
  std::vector<int> term_ptr((size_t)b.nrhs * 3 + 1, 0), term_fac((size_t)b.nterms * 3);
  std::vector<double> term_coef(b.nterms);
  if (loads) {
    for (int t = 0; t < s->nterms; ++t) {
      const int cl = s->term_col[t], c = s->term_comp[t];
      if (cl < 0 || cl >= s->nrhs || c < 0 || c > 2) return fail(IETIDP_E_ARG, "load term column/component out of range");
      for (int a = 0; a < 3; ++a) {
        const int fi = s->term_fac[3 * t + a];
        if (fi < 0 || fi >= s->nfac[a]) return fail(IETIDP_E_ARG, "load term factor out of range");
        if (s->fac_kind[a][fi] != (a == c ? 0 : 1)) return fail(IETIDP_E_ARG, "load factor kind does not match its component");
      }
      term_ptr[cl * 3 + c + 1]++;
    }
    for (size_t i = 1; i < term_ptr.size(); ++i) term_ptr[i] += term_ptr[i - 1];
    std::vector<int> at(term_ptr.begin(), term_ptr.end() - 1);
    for (int t = 0; t < s->nterms; ++t) {
      const int k = at[s->term_col[t] * 3 + s->term_comp[t]]++;
      for (int a = 0; a < 3; ++a) term_fac[3 * k + a] = s->term_fac[3 * t + a];
      term_coef[k] = s->term_coef[t];
    }
  }
  int gtot = 0;
  for (int c = 0; c < 3; ++c)
    for (int a = 0; a < 3; ++a) {
      b.goff[c][a] = gtot;
      const int nb = b.nb[a == c ? 0 : 1];
      gtot += b.np[a] * nb * nb;
    }
  b.gtotal = gtot;
  b.ktotal = 7 * (b.np[0] + b.np[1] + b.np[2]) * (b.s + 1) * (b.s + 1);
  for (int a = 0; a < 3; ++a) {
    const size_t npts = (size_t)b.np[a] * b.e * b.nq, lpts = (size_t)b.np[a] * b.e * b.lq;
    fx.knots[a] = st.put(s->knots[a], ((size_t)b.m[a] + b.p + 1) * 8);
    fx.qx[a] = st.put(s->qx[a], npts * 8);
    for (int c = 0; c < 3; ++c) fx.qw[c][a] = st.put(s->qw[c][a], npts * 8);
    for (int k = 0; k < 2; ++k) fx.tabq[a][k] = st.reserve(npts * b.nb[k] * 8);
    b.nfac[a] = loads ? s->nfac[a] : 0;
    fx.lx[a] = st.put(loads ? s->lx[a] : nullptr, loads ? lpts * 8 : 0);
    fx.facv[a] = st.put(loads ? s->fac_val[a] : nullptr, loads ? (size_t)s->nfac[a] * lpts * 8 : 0);
    fx.fac_kind[a] = st.put(loads ? s->fac_kind[a] : nullptr, loads ? (size_t)s->nfac[a] * 4 : 0);
    for (int k = 0; k < 2; ++k) fx.tabl[a][k] = st.reserve(loads ? lpts * b.nb[k] * 8 : 0);
    fx.v1d[a] = st.reserve(loads ? (size_t)s->nfac[a] * b.m[a] * 8 : 0);
  }
  fx.gram = st.reserve((size_t)gtot * 8);
  fx.ktab = st.reserve((size_t)b.ktotal * 8);
  fx.nu = st.put(s->nu, (size_t)b.np[0] * b.np[1] * b.np[2] * 8);
  fx.dof_of_edge = st.put(s->dof_of_edge, (size_t)nedge * 4);
  fx.edge_of_dof = st.put(edge_of_dof.data(), edge_of_dof.size() * 4);
  fx.tables = st.reserve((size_t)T_COUNT * 3 * MAXM * 4);
  fx.term_ptr = st.put(term_ptr.data(), term_ptr.size() * 4);
  fx.term_fac = st.put(term_fac.data(), term_fac.size() * 4);
  fx.term_coef = st.put(term_coef.data(), term_coef.size() * 8);
  return IETIDP_OK;
}

void bind_box(Box& b, const Fix& fx, char* base) {
  auto D = [&](size_t off) { return reinterpret_cast<double*>(base + off); };
  auto I = [&](size_t off) { return reinterpret_cast<int*>(base + off); };
  for (int a = 0; a < 3; ++a) {
    b.knots[a] = D(fx.knots[a]);
    b.qx[a] = D(fx.qx[a]);
    for (int c = 0; c < 3; ++c) b.qw[c][a] = D(fx.qw[c][a]);
    b.lx[a] = D(fx.lx[a]);
    b.facv[a] = D(fx.facv[a]);
    b.fac_kind[a] = I(fx.fac_kind[a]);
    for (int k = 0; k < 2; ++k) {
      b.tabq[a][k] = D(fx.tabq[a][k]);
      b.tabl[a][k] = D(fx.tabl[a][k]);
    }
    b.v1d[a] = D(fx.v1d[a]);
  }
  b.gram = b.gram_w = D(fx.gram);
  b.ktab = D(fx.ktab);
  b.nu = D(fx.nu);
  b.dof_of_edge = I(fx.dof_of_edge);
  b.edge_of_dof = I(fx.edge_of_dof);
  b.tables = I(fx.tables);
  b.term_ptr = I(fx.term_ptr);
  b.term_fac = I(fx.term_fac);
  b.term_coef = D(fx.term_coef);
}

}  // namespace

extern "C" {

const char* ietidp_pre_last_error(void) { return g_err.c_str(); }

void ietidp_pre_destroy(ietidp_pre_t a) {
  if (!a) return;
  if (a->batch) cudaSetDevice(a->batch->device);
  delete a;
}

int ietidp_pre_assemble_batch(int device, int n, const ietidp_pre_subdomain* subs, ietidp_pre_t* out) {
  if (n < 1 || !subs || !out) return fail(IETIDP_E_ARG, "null argument or empty batch");
  for (int k = 0; k < n; ++k) out[k] = nullptr;
  std::shared_ptr<PreBatch> B;
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  try {
    B = std::make_shared<PreBatch>();
    B->device = device;
    B->n = n;
    B->boxes.resize(n);
    B->nnz.assign(n, 0);
    std::vector<Fix> fix(n);
    Stage st;
    for (int k = 0; k < n; ++k) {
      const int rc = layout_box(&subs[k], B->boxes[k], fix[k], st);
      if (rc != IETIDP_OK) return rc;
    }
    PRE_CUDA(cudaSetDevice(device));
    for (auto& e : ev) PRE_CUDA(cudaEventCreate(&e));
    B->arena.upload(st.host.data(), st.host.size());
    long long rows = 0, fsz = 0;
    int max_dof = 0, smem = 0;
    std::vector<long long> row_off(n), f_off(n);
    for (int k = 0; k < n; ++k) {
      Box& b = B->boxes[k];
      row_off[k] = rows;
      f_off[k] = fsz;
      rows += b.n_dof + 1;
      fsz += (long long)b.n_dof * b.nrhs;
      max_dof = std::max(max_dof, b.n_dof);
      const int ncand = 3 * b.W * b.W * b.W;
      smem = std::max(smem, ((b.ktotal + 1) & ~1) * (int)sizeof(double) + ROWS_WARPS * ((ncand + 7) & ~7) * (int)sizeof(unsigned short));
    }
    if (smem > 180 * 1024) throw std::make_pair((int)IETIDP_E_ARG, std::string("Gram tables exceed shared memory"));
    B->rowptr.alloc(rows);
    B->cnt.alloc(rows);
    B->d_nnz.alloc(n);
    B->f.alloc(fsz);
    for (int k = 0; k < n; ++k) {
      Box& b = B->boxes[k];
      bind_box(b, fix[k], B->arena.p);
      b.rowptr = B->rowptr.p + row_off[k];
      b.cnt = B->cnt.p + row_off[k];
      b.nnz_out = B->d_nnz.p + k;
      b.f = B->f.p + f_off[k];
    }
    B->d_boxes.upload(B->boxes.data(), n);
    PRE_CUDA(cudaFuncSetAttribute((const void*)k_rows<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int gx = std::max(1, (max_dof + ROWS_WARPS - 1) / ROWS_WARPS);
    B->gx = gx;
    B->smem = smem;
    for (int k = 0; k < n; ++k) {
      B->nu_off.push_back(fix[k].nu);
      B->nu_cnt.push_back((size_t)B->boxes[k].np[0] * B->boxes[k].np[1] * B->boxes[k].np[2]);
    }
    PRE_CUDA(cudaEventRecord(ev[0]));
    k_stage1d<<<n, 256>>>(B->d_boxes.p);
    k_rows<0><<<dim3(gx, n), 32 * ROWS_WARPS>>>(B->d_boxes.p);
    k_scan<<<n, 1024>>>(B->d_boxes.p);
    PRE_CUDA(cudaEventRecord(ev[1]));
    PRE_CUDA(cudaMemcpy(B->nnz.data(), B->d_nnz.p, (size_t)n * sizeof(long long), cudaMemcpyDeviceToHost));
    long long tot = 0;
    std::vector<long long> nz_off(n);
    for (int k = 0; k < n; ++k) {
      nz_off[k] = tot;
      tot += B->nnz[k];
    }
    B->col.alloc((size_t)tot);
    B->val.alloc((size_t)tot);
    for (int k = 0; k < n; ++k) {
      B->boxes[k].col = B->col.p + nz_off[k];
      B->boxes[k].val = B->val.p + nz_off[k];
    }
    PRE_CUDA(cudaMemcpy(B->d_boxes.p, B->boxes.data(), (size_t)n * sizeof(Box), cudaMemcpyHostToDevice));
    PRE_CUDA(cudaEventRecord(ev[2]));
    k_rows<1><<<dim3(gx, n), 32 * ROWS_WARPS, smem>>>(B->d_boxes.p);
    PRE_CUDA(cudaEventRecord(ev[4]));
    if (fsz) k_loads<<<dim3(std::max(1, std::min((max_dof + 255) / 256 * 4, 64)), n), 256>>>(B->d_boxes.p);
    PRE_CUDA(cudaEventRecord(ev[3]));
    PRE_CUDA(cudaEventSynchronize(ev[3]));
    PRE_CUDA(cudaGetLastError());
    float m0 = 0, m1 = 0, m2 = 0;
    PRE_CUDA(cudaEventElapsedTime(&m0, ev[0], ev[1]));
    PRE_CUDA(cudaEventElapsedTime(&m1, ev[2], ev[3]));
    PRE_CUDA(cudaEventElapsedTime(&m2, ev[2], ev[4]));
    B->ms = m0 + m1;
    B->ms_fill = m2;
    for (auto& e : ev) cudaEventDestroy(e);
    for (int k = 0; k < n; ++k) {
      out[k] = new ietidp_pre_s();
      out[k]->batch = B;
      out[k]->idx = k;
    }
    return IETIDP_OK;
  } catch (const std::pair<int, std::string>& ex) {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    return fail(ex.first, ex.second);
  } catch (const std::bad_alloc&) {
    return fail(IETIDP_E_NOMEM, "host allocation failed");
  }
}

int ietidp_pre_assemble(int device, const ietidp_pre_subdomain* s, ietidp_pre_t* out) {
  if (!s || !out) return fail(IETIDP_E_ARG, "null argument");
  return ietidp_pre_assemble_batch(device, 1, s, out);
}

int ietidp_pre_sizes(ietidp_pre_t a, int* n_dof, int64_t* nnz, double* ms, double* ms_fill) {
  if (!a) return fail(IETIDP_E_ARG, "null handle");
  if (n_dof) *n_dof = a->batch->boxes[a->idx].n_dof;
  if (nnz) *nnz = a->batch->nnz[a->idx];
  if (ms) *ms = a->batch->ms;
  if (ms_fill) *ms_fill = a->batch->ms_fill;
  return IETIDP_OK;
}

int ietidp_pre_get(ietidp_pre_t a, int64_t* rowptr, int32_t* col, double* val, double* f) {
  if (!a) return fail(IETIDP_E_ARG, "null handle");
  try {
    const Box& b = a->batch->boxes[a->idx];
    const long long nnz = a->batch->nnz[a->idx];
    PRE_CUDA(cudaSetDevice(a->batch->device));
    static_assert(sizeof(long long) == sizeof(int64_t), "int64");
    if (rowptr) PRE_CUDA(cudaMemcpy(rowptr, b.rowptr, ((size_t)b.n_dof + 1) * 8, cudaMemcpyDeviceToHost));
    if (col && nnz) PRE_CUDA(cudaMemcpy(col, b.col, (size_t)nnz * 4, cudaMemcpyDeviceToHost));
    if (val && nnz) PRE_CUDA(cudaMemcpy(val, b.val, (size_t)nnz * 8, cudaMemcpyDeviceToHost));
    if (f && b.n_dof && b.nrhs) PRE_CUDA(cudaMemcpy(f, b.f, (size_t)b.n_dof * b.nrhs * 8, cudaMemcpyDeviceToHost));
    return IETIDP_OK;
  } catch (const std::pair<int, std::string>& ex) {
    return fail(ex.first, ex.second);
  }
}

int ietidp_pre_refill(ietidp_pre_t a, const double* nu_all, double* ms) {
  if (!a || !nu_all) return fail(IETIDP_E_ARG, "null argument");
  PreBatch& B = *a->batch;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  try {
    PRE_CUDA(cudaSetDevice(B.device));
    size_t at = 0;
    for (int k = 0; k < B.n; ++k) {
      PRE_CUDA(cudaMemcpyAsync(B.arena.p + B.nu_off[k], nu_all + at, B.nu_cnt[k] * sizeof(double), cudaMemcpyHostToDevice, 0));
      at += B.nu_cnt[k];
    }
    PRE_CUDA(cudaEventCreate(&e0));
    PRE_CUDA(cudaEventCreate(&e1));
    PRE_CUDA(cudaEventRecord(e0));
    k_rows<1><<<dim3(B.gx, B.n), 32 * ROWS_WARPS, B.smem>>>(B.d_boxes.p);
    PRE_CUDA(cudaEventRecord(e1));
    PRE_CUDA(cudaEventSynchronize(e1));
    PRE_CUDA(cudaGetLastError());
    float t = 0;
    PRE_CUDA(cudaEventElapsedTime(&t, e0, e1));
    B.ms_fill = t;
    if (ms) *ms = t;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return IETIDP_OK;
  } catch (const std::pair<int, std::string>& ex) {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    return fail(ex.first, ex.second);
  }
}

int ietidp_pre_device_ptrs(ietidp_pre_t a, const double** d_val, const double** d_f) {
  if (!a) return fail(IETIDP_E_ARG, "null handle");
  const Box& b = a->batch->boxes[a->idx];
  if (d_val) *d_val = b.val;
  if (d_f) *d_f = b.f;
  return IETIDP_OK;
}

int ietidp_pre_get_gram(ietidp_pre_t a, int c, int axis, int q, double* block, int* nb_out) {
  if (!a || c < 0 || c > 2 || axis < 0 || axis > 2) return fail(IETIDP_E_ARG, "bad argument");
  const Box& b = a->batch->boxes[a->idx];
  if (q < 0 || q >= b.np[axis]) return fail(IETIDP_E_ARG, "bad argument");
  const int nb = b.nb[axis == c ? 0 : 1];
  if (nb_out) *nb_out = nb;
  if (!block) return IETIDP_OK;
  try {
    PRE_CUDA(cudaSetDevice(a->batch->device));
    PRE_CUDA(cudaMemcpy(block, b.gram + b.goff[c][axis] + (size_t)q * nb * nb, (size_t)nb * nb * 8, cudaMemcpyDeviceToHost));
    return IETIDP_OK;
  } catch (const std::pair<int, std::string>& ex) {
    return fail(ex.first, ex.second);
  }
}

int ietidp_pre_gauge(int device, int64_t nv, int64_t ne, const int32_t* eu, const int32_t* ev, const int8_t* w,
                     uint8_t* in_tree, uint8_t* primal, double* ms) {
  if (nv < 0 || ne < 0 || nv > 0x7fffffffll || ne >= (1ll << KEY_SHIFT) || (ne && (!eu || !ev || !w)) || !in_tree)
    return fail(IETIDP_E_ARG, "bad sizes or null argument");
  for (int64_t e = 0; e < ne; ++e) {
    if (eu[e] < 0 || eu[e] >= nv || ev[e] < 0 || ev[e] >= nv) return fail(IETIDP_E_ARG, "edge endpoint out of range");
    if (w[e] < 1 || w[e] > 5) return fail(IETIDP_E_ARG, "edge weight outside 1..5");
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  try {
    PRE_CUDA(cudaSetDevice(device));
    Buf<int> d_eu, d_ev, comp, parent, changed;
    Buf<int8_t> d_w;
    Buf<uint8_t> d_tree, d_primal;
    Buf<unsigned long long> best;
    d_eu.upload(eu, ne);
    d_ev.upload(ev, ne);
    d_w.upload(w, ne);
    comp.alloc(nv);
    parent.alloc(nv);
    best.alloc(nv);
    changed.alloc(1);
    d_tree.alloc(ne);
    d_primal.alloc(ne);
    PRE_CUDA(cudaEventCreate(&e0));
    PRE_CUDA(cudaEventCreate(&e1));
    PRE_CUDA(cudaEventRecord(e0));
    PRE_CUDA(cudaMemsetAsync(d_tree.p, 0, std::max<size_t>(ne, 1)));
    const unsigned gv = (unsigned)std::max<long long>(1, (nv + 255) / 256), ge = (unsigned)std::max<long long>(1, (ne + 255) / 256);
    k_bv_init<<<gv, 256>>>(nv, comp.p);
    for (int round = 0; round < 64; ++round) {
      k_bv_reset<<<gv, 256>>>(nv, best.p);
      PRE_CUDA(cudaMemsetAsync(changed.p, 0, sizeof(int)));
      k_bv_min<<<ge, 256>>>(ne, d_eu.p, d_ev.p, d_w.p, comp.p, best.p);
      k_bv_pick<<<gv, 256>>>(nv, d_eu.p, d_ev.p, comp.p, best.p, parent.p, d_tree.p, changed.p);
      k_bv_break<<<gv, 256>>>(nv, parent.p);
      k_bv_flatten<<<gv, 256>>>(nv, parent.p, comp.p);
      int ch = 0;
      PRE_CUDA(cudaMemcpy(&ch, changed.p, sizeof(int), cudaMemcpyDeviceToHost));
      if (!ch) break;
    }
    k_primal<<<ge, 256>>>(ne, d_w.p, d_tree.p, d_primal.p);
    PRE_CUDA(cudaEventRecord(e1));
    PRE_CUDA(cudaEventSynchronize(e1));
    PRE_CUDA(cudaGetLastError());
    float t = 0;
    PRE_CUDA(cudaEventElapsedTime(&t, e0, e1));
    if (ms) *ms = t;
    if (ne) PRE_CUDA(cudaMemcpy(in_tree, d_tree.p, ne, cudaMemcpyDeviceToHost));
    if (primal && ne) PRE_CUDA(cudaMemcpy(primal, d_primal.p, ne, cudaMemcpyDeviceToHost));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return IETIDP_OK;
  } catch (const std::pair<int, std::string>& ex) {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    return fail(ex.first, ex.second);
  }
}

}  // extern "C"
