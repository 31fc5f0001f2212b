// Internal structures of libietidp.so (host plan + device-side descriptors).
// Shared by the host C++ (api.cpp, analyze.cpp) and the CUDA translation units.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ietidp.h"

#ifdef __CUDACC__
#define IETI_HD __host__ __device__
#else
#define IETI_HD
#endif

namespace ieti {

constexpr int TB = 64;            // panel width of the supernodal Cholesky = loop tile size
constexpr int TILE_ELEMS = TB * TB;

// ---------------------------------------------------------------------------
// Device descriptors (plain structs, copied to the device as arrays)
// ---------------------------------------------------------------------------

// One supernode (front) of one subdomain's K_rr.
// The front is an f x f column-major block (leading dimension ld) in the fronts
// pool; its first npiv columns hold [L11; L21] after the partial factorisation,
// its trailing (f-npiv)^2 block the update (Schur) matrix passed to the parent.
struct SnDev {
  long long front_off;  // into the fronts pool (doubles)
  long long dinv_off;   // into the Dinv pool: ceil(npiv/TB) tiles of TB x TB (col-major)
  long long vec_off;    // into the sweep vector workspace: f x ncols_max (row-major)
  int f, ld, npiv, c0;  // front size, leading dim, #pivots, first pivot position
  int sub, parent;      // subdomain, parent supernode (-1: root)
  int rows_off;         // rows[rows_off .. +f-npiv): positions (in the subdomain's r order)
  int rel_off;          // rel[rel_off .. +f-npiv): local row index of each update row in the parent front
  int child_off, nchild;// children[child_off .. +nchild)
};

// Per-subdomain descriptor.
struct SubDev {
  int nk, nr, nI, nV, nP;     // local DOFs, remaining, interface-remaining, interior, primal
  int root;                   // supernode holding r_I (-1 if nI == 0)
  long long x_off;            // sweep matrix X: nr x ncx (row-major, ncx = nPmax + nrhs)
  long long rI_off;           // offset in the concatenated r_I slot arrays
  long long kval_off, f_off;  // raw CSR values / raw loads (nk x nrhs col-major)
  long long kpp_off;          // dense K_PP^(k): nP x nP
  long long jp_off;           // j_P^(k): nP x nrhs (row-major)
  long long g_off;            // G_k = X_k[r_I, P]: nI x nP (row-major)
  long long sloc_off;         // local coarse block nP x nP
  long long floc_off;         // local coarse rhs  nP x nrhs
  long long gk_off;           // per-iteration G_k^T b: nP x ncols
  long long tile_off;         // packed L_II tiles (row-block order, TB x TB row-major)
  long long dtile_off;        // packed Dinv_II tiles (TB x TB row-major), one per block row
  int prim_off;               // into prim_gid / prim_dof arrays
  int perm_off;               // perm[perm_off .. +nr): r position -> local DOF
  int nt;                     // ceil(nI / TB)
  int pad_;
};

// One multiplier's two B entries (F3: every row is {+1, -1} in two subdomains).
struct LamDev {
  int slot[2];     // positions in the concatenated r_I storage
  float sign[2];   // +1 / -1
};

// Work item for the tiled factorisation kernels.
struct Work {
  int sn, a, b;
};

// ---------------------------------------------------------------------------
// Host-side input copies and the plan
// ---------------------------------------------------------------------------

struct SubIn {
  bool set = false;
  int n = 0;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> col;
  std::vector<double> val;
  std::vector<double> f;  // n x nrhs col-major
  std::vector<int32_t> B_lambda, B_dof;
  std::vector<int8_t> B_sign;
  std::vector<int32_t> tree, prim, prim_gid;
};

struct SnHost {
  int sub, c0, npiv, f, parent, level;
  std::vector<int> rows;
  std::vector<int> children;
};

struct SubPlan {
  int nr = 0, nI = 0, nV = 0, nP = 0;
  std::vector<int> perm;     // r position -> local DOF
  std::vector<int> pos;      // local DOF -> r position (-1 tree, -1 primal)
  std::vector<int> ploc;     // local DOF -> primal local index (-1 otherwise)
  std::vector<int> sn_begin; // supernode ids of this subdomain [first, last)
  int root = -1;
};

// A launch of the factorisation for one level (host plan, device work lists).
struct LevelPlan {
  long long front_begin = 0, front_end = 0;   // pool range zeroed before assembly
  long long scat_begin = 0, scat_end = 0;     // entries of the K scatter list
  std::vector<std::pair<int, int>> ea;        // extend-add launches: (work offset, count), one per child slot
  struct Panel {
    int potrf_off, potrf_n, trsm_off, trsm_n, upd_off, upd_n;
  };
  std::vector<Panel> panels;
  int sn_off = 0, sn_n = 0;                   // supernodes of this level (in level_sn list)
};

struct Plan {
  std::vector<SubPlan> subs;
  std::vector<SnHost> sn;        // all supernodes, global ids
  std::vector<int> level_sn;     // supernode ids grouped by level
  std::vector<LevelPlan> levels;
  long long pool_doubles = 0, dinv_doubles = 0, vec_doubles = 0;
  int max_level = 0, max_front = 0, max_nI = 0, nPmax = 0, ncx = 0;
  long long nnz_L = 0, flops = 0;
};

}  // namespace ieti
