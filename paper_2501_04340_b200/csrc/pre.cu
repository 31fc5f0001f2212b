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
__global__ void k_basis(const double* __restrict__ t, int p, int s, int kind, int nb, int pts_per_patch, int npts,
                        const double* __restrict__ x, double* __restrict__ tab) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= npts * nb) return;
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

// Gram block of one (component, axis, patch): G[fl + nb*gl] = sum_u (phi_f phi_g) w_u.
__global__ void k_gram(const double* __restrict__ tab, const double* __restrict__ w, int nb, int pts_per_patch,
                       double* __restrict__ out) {
  const int q = blockIdx.x;
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int fl = idx % nb, gl = idx / nb;
    double acc = 0.0;
    for (int u = q * pts_per_patch; u < (q + 1) * pts_per_patch; ++u) acc += (tab[u * nb + fl] * tab[u * nb + gl]) * w[u];
    out[(size_t)q * nb * nb + idx] = acc;
  }
}

// v[i] = sum over the points of the patches carrying function i of fw[u] * phi_i(x_u).
__global__ void k_load1d(const double* __restrict__ tab, const double* __restrict__ fw, int kind, int nb, int s, int np,
                         int pts_per_patch, int dim, double* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dim) return;
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
__global__ void k_tables(const Box b, int* __restrict__ tb) {
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

// M_2 entry of component c between faces f and g: sum over the common patches of
// nu * Gz * Gy * Gx (gram and tb in shared memory).
__device__ __forceinline__ double m2_entry(const Box& b, const double* gram, const int* tb, int c, const int (&f)[3],
                                           const int (&g)[3]) {
  int qlo[3], qhi[3];
  for (int a = 0; a < 3; ++a) {
    if (a == c) {
      const int pf = tb[tb_at(T_PB, a, f[a])], pg = tb[tb_at(T_PB, a, g[a])];
      qlo[a] = max(pf & 0xffff, pg & 0xffff);
      qhi[a] = min(pf >> 16, pg >> 16);
    } else {
      qlo[a] = tb[tb_at(T_PD, a, f[a])];
      qhi[a] = qlo[a] == tb[tb_at(T_PD, a, g[a])] ? qlo[a] : qlo[a] - 1;
    }
    if (qhi[a] < qlo[a]) return 0.0;
  }
  double acc = 0.0;
  for (int qz = qlo[2]; qz <= qhi[2]; ++qz)
    for (int qy = qlo[1]; qy <= qhi[1]; ++qy)
      for (int qx = qlo[0]; qx <= qhi[0]; ++qx) {
        const int qq[3] = {qx, qy, qz};
        double v[3];
        for (int a = 0; a < 3; ++a) {
          const int nb = b.nb[a == c ? 0 : 1];
          const double* G = gram + b.goff[c][a] + qq[a] * nb * nb;
          v[a] = G[(f[a] - qq[a] * b.s) + nb * (g[a] - qq[a] * b.s)];
        }
        acc += b.nu[qx + b.np[0] * (qy + b.np[1] * qz)] * (v[2] * (v[1] * v[0]));
      }
  return acc;
}

// K[e1, e2] = sum_c sum_{faces f of e1, g of e2 in component c} C_f,e1 C_g,e2 M_2[f, g].
__device__ __forceinline__ double k_entry(const Box& b, const double* gram, const int* tb, const Edge& e1, const Edge& e2) {
  double acc = 0.0;
  for (int c = 0; c < 3; ++c) {
    if (c == e1.d || c == e2.d) continue;
    const int r1 = 3 - c - e1.d, r2 = 3 - c - e2.d;
    // (c, a, b) cyclic: C[f(n), edge_a(n)] = +1, C[f(n), edge_b(n)] = -1, opposite at n - e_r
    const double s1n = (c == (e1.d + 1) % 3) ? -1.0 : 1.0;
    const double s2n = (c == (e2.d + 1) % 3) ? -1.0 : 1.0;
    for (int o1 = 0; o1 < 2; ++o1) {
      int f[3] = {e1.n[0], e1.n[1], e1.n[2]};
      f[r1] -= o1;
      if (f[r1] < 0 || f[r1] >= b.F[c][r1]) continue;
      for (int o2 = 0; o2 < 2; ++o2) {
        int g[3] = {e2.n[0], e2.n[1], e2.n[2]};
        g[r2] -= o2;
        if (g[r2] < 0 || g[r2] >= b.F[c][r2]) continue;
        const double sg = (o1 ? -s1n : s1n) * (o2 ? -s2n : s2n);
        acc += sg * m2_entry(b, gram, tb, c, f, g);
      }
    }
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

// Candidate column idx of a row edge e1: (direction, dz, dy, dx) over the reach box,
// ascending in the DOF order. Returns false outside the box's edge grid.
__device__ __forceinline__ bool candidate(const Box& b, const Edge& e1, int idx, Edge& e2) {
  const int W = b.W, W3 = W * W * W;
  e2.d = idx / W3;
  int r = idx - e2.d * W3;
  const int dz = r / (W * W);
  r -= dz * W * W;
  const int dy = r / W, dx = r - dy * W;
  e2.n[0] = e1.n[0] + dx - b.R;
  e2.n[1] = e1.n[1] + dy - b.R;
  e2.n[2] = e1.n[2] + dz - b.R;
  bool ok = true;
  for (int a = 0; a < 3; ++a) ok = ok && e2.n[a] >= 0 && e2.n[a] < b.E[e2.d][a];
  return ok;
}
__device__ __forceinline__ int dof_at(const Box& b, const Edge& e) {
  return b.dof_of_edge[b.eoff[e.d] + e.n[0] + (long long)b.E[e.d][0] * (e.n[1] + (long long)b.E[e.d][1] * e.n[2])];
}

constexpr int ROWS_WARPS = 8;

// A warp per DOF row. Candidate columns are walked in ascending DOF order, 32 at a time; a
// ballot compacts the structural entries. FILL = 0: cnt[row] = their number. FILL = 1: the
// compacted candidate list goes to the warp's shared-memory strip first, then all 32 lanes
// evaluate entries (columns and values at rowptr[row], coalesced).
template <int FILL>
__global__ void __launch_bounds__(32 * ROWS_WARPS) k_rows(const Box b, const int* __restrict__ tbg, int* __restrict__ cnt,
                                                          const long long* __restrict__ rowptr, int* __restrict__ col,
                                                          double* __restrict__ val) {
  extern __shared__ double sgram[];
  __shared__ int tb[T_COUNT * 3 * MAXM];
  for (int i = threadIdx.x; i < T_COUNT * 3 * MAXM; i += blockDim.x) tb[i] = tbg[i];
  if (FILL)
    for (int i = threadIdx.x; i < b.gtotal; i += blockDim.x) sgram[i] = b.gram[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ncand = 3 * b.W * b.W * b.W;
  unsigned short* strip = reinterpret_cast<unsigned short*>(sgram + ((b.gtotal + 1) & ~1)) + (size_t)warp * ((ncand + 7) & ~7);
  for (int row = blockIdx.x * ROWS_WARPS + warp; row < b.n_dof; row += gridDim.x * ROWS_WARPS) {
    const Edge e1 = edge_of(b, b.edge_of_dof[row]);
    int count = 0;
    for (int base = 0; base < ncand; base += 32) {
      const int idx = base + lane;
      Edge e2;
      const bool ok = idx < ncand && candidate(b, e1, idx, e2) && k_struct(b, tb, e1, e2) && dof_at(b, e2) >= 0;
      const unsigned mask = __ballot_sync(0xffffffffu, ok);
      if (FILL && ok) strip[count + __popc(mask & ((1u << lane) - 1u))] = (unsigned short)idx;
      count += __popc(mask);
    }
    if (!FILL) {
      if (lane == 0) cnt[row] = count;
      continue;
    }
    __syncwarp();
    const long long pos = rowptr[row];
    for (int t = lane; t < count; t += 32) {
      Edge e2;
      candidate(b, e1, strip[t], e2);
      const int dof2 = dof_at(b, e2);
      col[pos + t] = dof2;
      // exactly symmetric: both (i, j) and (j, i) evaluate the pair (min, max)
      val[pos + t] = dof2 < row ? k_entry(b, sgram, tb, e2, e1) : k_entry(b, sgram, tb, e1, e2);
    }
    __syncwarp();
  }
}

// rowptr[0..n] = exclusive prefix sums of cnt (one CTA; n is a few thousand).
__global__ void __launch_bounds__(1024) k_scan(const int* __restrict__ cnt, int n, long long* __restrict__ rowptr) {
  __shared__ long long part[1024];
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
  if (t == 1023) rowptr[n] = part[1023];
}

struct LoadArgs {
  const double* v[3];     // 1-D integrals per axis, factor-major with stride vstride[a]
  int vstride[3];
  const int* term_ptr;    // (col*3 + comp) -> terms
  const int* term_fac;    // 3 per term
  const double* term_coef;
  int nrhs;
};

// j[dof, col] = sum over the (at most 4) faces of the edge of C_f,e * t_f,
// t_f = sum_terms coef * vx[f_x] vy[f_y] vz[f_z].
__global__ void __launch_bounds__(256) k_loads(const Box b, const LoadArgs L, double* __restrict__ j) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)b.n_dof * L.nrhs) return;
  const int row = (int)(idx % b.n_dof), colr = (int)(idx / b.n_dof);
  const Edge e = edge_of(b, b.edge_of_dof[row]);
  double acc = 0.0;
  for (int c = 0; c < 3; ++c) {
    if (c == e.d) continue;
    const int r = 3 - c - e.d;
    const double sn = (c == (e.d + 1) % 3) ? -1.0 : 1.0;
    const int t0 = L.term_ptr[colr * 3 + c], t1 = L.term_ptr[colr * 3 + c + 1];
    if (t0 == t1) continue;
    for (int o = 0; o < 2; ++o) {
      int f[3] = {e.n[0], e.n[1], e.n[2]};
      f[r] -= o;
      if (f[r] < 0 || f[r] >= b.F[c][r]) continue;
      double tf = 0.0;
      for (int t = t0; t < t1; ++t) {
        const int* fc = L.term_fac + 3 * t;
        tf += L.term_coef[t] * (L.v[2][(size_t)fc[2] * L.vstride[2] + f[2]] *
                                (L.v[1][(size_t)fc[1] * L.vstride[1] + f[1]] * L.v[0][(size_t)fc[0] * L.vstride[0] + f[0]]));
      }
      acc += (o ? -sn : sn) * tf;
    }
  }
  j[idx] = acc;
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

}  // namespace

struct ietidp_pre_s {
  int device = 0, n_dof = 0, nrhs = 0;
  long long nnz = 0;
  double ms = 0.0;
  Box box{};
  Buf<double> gram, nu, val, f;
  Buf<int> dof_of_edge, edge_of_dof, col, cnt, tables;
  double ms_fill = 0.0;
  Buf<long long> rowptr;
};

extern "C" {

const char* ietidp_pre_last_error(void) { return g_err.c_str(); }

void ietidp_pre_destroy(ietidp_pre_t a) {
  if (!a) return;
  cudaSetDevice(a->device);
  delete a;
}

int ietidp_pre_assemble(int device, const ietidp_pre_subdomain* s, ietidp_pre_t* out) {
  if (!s || !out) return fail(IETIDP_E_ARG, "null argument");
  *out = nullptr;
  if (s->p < 1 || s->p > MAXP || s->e < 1 || s->nq < 1 || s->n_dof < 0 || s->nrhs < 0)
    return fail(IETIDP_E_ARG, "degree must be 1..3, e, nq >= 1");
  for (int a = 0; a < 3; ++a) {
    if (s->npatch[a] < 1 || !s->knots[a] || !s->qx[a]) return fail(IETIDP_E_ARG, "npatch >= 1, knots and qx required");
    for (int c = 0; c < 3; ++c)
      if (!s->qw[c][a]) return fail(IETIDP_E_ARG, "qw[c][a] required");
  }
  if (!s->nu || !s->dof_of_edge) return fail(IETIDP_E_ARG, "nu and dof_of_edge required");
  if (s->nrhs > 0 && s->nterms > 0) {
    if (s->lq < 1 || !s->term_col || !s->term_comp || !s->term_fac || !s->term_coef)
      return fail(IETIDP_E_ARG, "load terms incomplete");
    for (int a = 0; a < 3; ++a)
      if (!s->lx[a] || s->nfac[a] < 1 || !s->fac_kind[a] || !s->fac_val[a]) return fail(IETIDP_E_ARG, "load factors incomplete");
  }
  Box b{};
  b.p = s->p;
  b.e = s->e;
  b.s = s->e + s->p - 1;
  b.nb[0] = b.s + 1;
  b.nb[1] = b.s;
  b.R = s->p + 1;
  b.W = 2 * b.R + 1;
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
  if (nedge > (1ll << 30)) return fail(IETIDP_E_ARG, "box too large");
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
  std::vector<int> term_ptr((size_t)std::max(s->nrhs, 0) * 3 + 1, 0), term_fac;
  std::vector<double> term_coef;
  const bool loads = s->nrhs > 0;
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
    term_fac.resize((size_t)s->nterms * 3);
    term_coef.resize(s->nterms);
    for (int t = 0; t < s->nterms; ++t) {
      const int k = at[s->term_col[t] * 3 + s->term_comp[t]]++;
      for (int a = 0; a < 3; ++a) term_fac[3 * k + a] = s->term_fac[3 * t + a];
      term_coef[k] = s->term_coef[t];
    }
  }

  ietidp_pre_s* A = nullptr;
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  try {
    PRE_CUDA(cudaSetDevice(device));
    A = new ietidp_pre_s();
    A->device = device;
    A->n_dof = s->n_dof;
    A->nrhs = std::max(s->nrhs, 0);
    for (auto& e : ev) PRE_CUDA(cudaEventCreate(&e));
    // uploads
    Buf<double> knots[3], qx[3], qw[3][3], lx[3], facv[3], tabq[3][2], tabl[3][2], v1d[3];
    Buf<int> d_term_ptr, d_term_fac;
    Buf<double> d_term_coef;
    int gtot = 0;
    for (int c = 0; c < 3; ++c)
      for (int a = 0; a < 3; ++a) {
        b.goff[c][a] = gtot;
        const int nb = b.nb[a == c ? 0 : 1];
        gtot += b.np[a] * nb * nb;
      }
    b.gtotal = gtot;
    A->gram.alloc(gtot);
    A->nu.upload(s->nu, (size_t)b.np[0] * b.np[1] * b.np[2]);
    A->dof_of_edge.upload(s->dof_of_edge, (size_t)nedge);
    A->edge_of_dof.upload(edge_of_dof.data(), edge_of_dof.size());
    A->cnt.alloc(s->n_dof);
    A->tables.alloc((size_t)T_COUNT * 3 * MAXM);
    A->rowptr.alloc((size_t)s->n_dof + 1);
    A->f.alloc((size_t)s->n_dof * A->nrhs);
    for (int a = 0; a < 3; ++a) {
      const int npts = b.np[a] * b.e * s->nq;
      knots[a].upload(s->knots[a], (size_t)b.m[a] + b.p + 1);
      qx[a].upload(s->qx[a], npts);
      for (int c = 0; c < 3; ++c) qw[c][a].upload(s->qw[c][a], npts);
      for (int k = 0; k < 2; ++k) tabq[a][k].alloc((size_t)npts * b.nb[k]);
      if (loads && s->nterms > 0) {
        const int lpts = b.np[a] * b.e * s->lq;
        lx[a].upload(s->lx[a], lpts);
        facv[a].upload(s->fac_val[a], (size_t)s->nfac[a] * lpts);
        for (int k = 0; k < 2; ++k) tabl[a][k].alloc((size_t)lpts * b.nb[k]);
        v1d[a].alloc((size_t)s->nfac[a] * b.m[a]);
      }
    }
    if (loads) {
      d_term_ptr.upload(term_ptr.data(), term_ptr.size());
      d_term_fac.upload(term_fac.data(), term_fac.size());
      d_term_coef.upload(term_coef.data(), term_coef.size());
    }
    b.gram = A->gram.p;
    b.nu = A->nu.p;
    b.dof_of_edge = A->dof_of_edge.p;
    b.edge_of_dof = A->edge_of_dof.p;
    b.n_dof = s->n_dof;
    A->box = b;

    PRE_CUDA(cudaEventRecord(ev[0]));
    // 1-D stage: spline tables, Gram blocks, load integrals
    for (int a = 0; a < 3; ++a) {
      const int ppp = b.e * s->nq, npts = b.np[a] * ppp;
      for (int k = 0; k < 2; ++k)
        k_basis<<<(npts * b.nb[k] + 127) / 128, 128>>>(knots[a].p, b.p, b.s, k, b.nb[k], ppp, npts, qx[a].p, tabq[a][k].p);
      for (int c = 0; c < 3; ++c) {
        const int k = a == c ? 0 : 1;
        k_gram<<<b.np[a], 128>>>(tabq[a][k].p, qw[c][a].p, b.nb[k], ppp, A->gram.p + b.goff[c][a]);
      }
      if (loads && s->nterms > 0) {
        const int lpp = b.e * s->lq, lpts = b.np[a] * lpp;
        for (int k = 0; k < 2; ++k)
          k_basis<<<(lpts * b.nb[k] + 127) / 128, 128>>>(knots[a].p, b.p, b.s, k, b.nb[k], lpp, lpts, lx[a].p, tabl[a][k].p);
        for (int fi = 0; fi < s->nfac[a]; ++fi) {
          const int k = s->fac_kind[a][fi];
          const int dim = b.m[a] - k;
          k_load1d<<<(dim + 127) / 128, 128>>>(tabl[a][k].p, facv[a].p + (size_t)fi * lpts, k, b.nb[k], b.s, b.np[a], lpp, dim,
                                               v1d[a].p + (size_t)fi * b.m[a]);
        }
      }
    }
    // pattern
    const int ncand = 3 * b.W * b.W * b.W;
    const int smem = ((gtot + 1) & ~1) * (int)sizeof(double) + ROWS_WARPS * ((ncand + 7) & ~7) * (int)sizeof(unsigned short);
    if (smem > 180 * 1024) throw std::make_pair((int)IETIDP_E_ARG, std::string("Gram tables exceed shared memory"));
    PRE_CUDA(cudaFuncSetAttribute((const void*)k_rows<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int grid = std::max(1, std::min((s->n_dof + ROWS_WARPS - 1) / ROWS_WARPS, 148 * 8));
    k_tables<<<1, 128>>>(b, A->tables.p);
    if (s->n_dof) k_rows<0><<<grid, 32 * ROWS_WARPS>>>(b, A->tables.p, A->cnt.p, nullptr, nullptr, nullptr);
    k_scan<<<1, 1024>>>(A->cnt.p, s->n_dof, A->rowptr.p);
    PRE_CUDA(cudaEventRecord(ev[1]));
    PRE_CUDA(cudaMemcpy(&A->nnz, A->rowptr.p + s->n_dof, sizeof(long long), cudaMemcpyDeviceToHost));
    A->col.alloc((size_t)A->nnz);
    A->val.alloc((size_t)A->nnz);
    PRE_CUDA(cudaEventRecord(ev[2]));
    if (s->n_dof) k_rows<1><<<grid, 32 * ROWS_WARPS, smem>>>(b, A->tables.p, nullptr, A->rowptr.p, A->col.p, A->val.p);
    PRE_CUDA(cudaEventRecord(ev[4]));
    if (A->nrhs && s->n_dof) {
      if (s->nterms > 0) {
        LoadArgs L{};
        for (int a = 0; a < 3; ++a) {
          L.v[a] = v1d[a].p;
          L.vstride[a] = b.m[a];
        }
        L.term_ptr = d_term_ptr.p;
        L.term_fac = d_term_fac.p;
        L.term_coef = d_term_coef.p;
        L.nrhs = A->nrhs;
        const long long tot = (long long)s->n_dof * A->nrhs;
        k_loads<<<(unsigned)((tot + 255) / 256), 256>>>(b, L, A->f.p);
      } else {
        PRE_CUDA(cudaMemset(A->f.p, 0, A->f.n * sizeof(double)));
      }
    }
    PRE_CUDA(cudaEventRecord(ev[3]));
    PRE_CUDA(cudaEventSynchronize(ev[3]));
    PRE_CUDA(cudaGetLastError());
    float m0 = 0, m1 = 0;
    PRE_CUDA(cudaEventElapsedTime(&m0, ev[0], ev[1]));
    PRE_CUDA(cudaEventElapsedTime(&m1, ev[2], ev[3]));
    A->ms = m0 + m1;
    PRE_CUDA(cudaEventElapsedTime(&m1, ev[2], ev[4]));
    A->ms_fill = m1;
    for (auto& e : ev) cudaEventDestroy(e);
    *out = A;
    return IETIDP_OK;
  } catch (const std::pair<int, std::string>& ex) {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    delete A;
    return fail(ex.first, ex.second);
  } catch (const std::bad_alloc&) {
    delete A;
    return fail(IETIDP_E_NOMEM, "host allocation failed");
  }
}

int ietidp_pre_sizes(ietidp_pre_t a, int* n_dof, int64_t* nnz, double* ms, double* ms_fill) {
  if (!a) return fail(IETIDP_E_ARG, "null handle");
  if (n_dof) *n_dof = a->n_dof;
  if (nnz) *nnz = a->nnz;
  if (ms) *ms = a->ms;
  if (ms_fill) *ms_fill = a->ms_fill;
  return IETIDP_OK;
}

int ietidp_pre_get(ietidp_pre_t a, int64_t* rowptr, int32_t* col, double* val, double* f) {
  if (!a) return fail(IETIDP_E_ARG, "null handle");
  try {
    PRE_CUDA(cudaSetDevice(a->device));
    static_assert(sizeof(long long) == sizeof(int64_t), "int64");
    if (rowptr) PRE_CUDA(cudaMemcpy(rowptr, a->rowptr.p, ((size_t)a->n_dof + 1) * 8, cudaMemcpyDeviceToHost));
    if (col && a->nnz) PRE_CUDA(cudaMemcpy(col, a->col.p, (size_t)a->nnz * 4, cudaMemcpyDeviceToHost));
    if (val && a->nnz) PRE_CUDA(cudaMemcpy(val, a->val.p, (size_t)a->nnz * 8, cudaMemcpyDeviceToHost));
    if (f && a->f.n) PRE_CUDA(cudaMemcpy(f, a->f.p, a->f.n * 8, cudaMemcpyDeviceToHost));
    return IETIDP_OK;
  } catch (const std::pair<int, std::string>& ex) {
    return fail(ex.first, ex.second);
  }
}

int ietidp_pre_get_gram(ietidp_pre_t a, int c, int axis, int q, double* block, int* nb_out) {
  if (!a || c < 0 || c > 2 || axis < 0 || axis > 2 || q < 0 || q >= a->box.np[axis]) return fail(IETIDP_E_ARG, "bad argument");
  const int nb = a->box.nb[axis == c ? 0 : 1];
  if (nb_out) *nb_out = nb;
  if (!block) return IETIDP_OK;
  try {
    PRE_CUDA(cudaSetDevice(a->device));
    PRE_CUDA(cudaMemcpy(block, a->gram.p + a->box.goff[c][axis] + (size_t)q * nb * nb, (size_t)nb * nb * 8,
                        cudaMemcpyDeviceToHost));
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
