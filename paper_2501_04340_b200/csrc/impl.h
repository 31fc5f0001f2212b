// Internal structures of libietidp.so (host plan + device-side descriptors).
// Shared by the host C++ (api.cpp, analyze.cpp) and the CUDA translation units.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ietidp.h"

namespace ieti {

constexpr int TB = 64;  // panel width of the supernodal Cholesky = tile size everywhere
constexpr int TILE_ELEMS = TB * TB;
// split-K of the panel updates (long K on few tiles): aim for this many CTAs per launch
// (3 resident GEMM CTAs per SM x 148 SMs), at most SPLITK_MAX parts of >= SPLITK_MIN_K
constexpr int SPLITK_TARGET_CTAS = 444, SPLITK_MAX = 8, SPLITK_MIN_K = 128;

// ---------------------------------------------------------------------------
// Device descriptors (plain structs, copied to the device as arrays)
// ---------------------------------------------------------------------------

// One supernode (front) of one subdomain.
// Local positions of a subdomain: [0, nV) r_V in nested-dissection order,
// [nV, nr) r_I, [nr, ne) the primal DOFs (P).  The front is an f x f
// column-major block (leading dimension ld) in the fronts pool; after the
// partial factorisation its first npiv columns hold [L11; L21] and the trailing
// block the update matrix for the parent. The P supernode ("coarse", one per
// subdomain with primal DOFs) is assembled but never factored: its front ends up
// holding S_loc = K_PP - K_Pr K_rr^-1 K_rP (SPD sign).
struct SnDev {
  long long front_off;  // fronts pool (doubles)
  long long dinv_off;   // inverted diagonal TB-blocks: ceil(npiv/TB) tiles (col-major)
  long long inv_off;    // partitioned inverse L11^-1 (npiv x npiv col-major, ld = ldi)
  long long vec_off;    // sweep vector workspace (rows; x ncols at run time)
  int f, ld, npiv, c0;  // front size, leading dim, #pivots, first pivot position
  int ldi, coarse;      // leading dim of L11^-1; 1 = P supernode (not factored)
  int sub, parent;      // subdomain, parent supernode (-1: root)
  int rows_off;         // rows[rows_off .. +f-npiv): positions of the update rows
  int rel_off;          // rel[rel_off .. +f-npiv): row index of each update row in the parent front
  int child_off, nchild;
  long long bp_off;     // backward sweep: partials of L21^T x per BS_RB-row chunk (chunks x npiv x 16)
};
constexpr int BS_RB = 256;  // rows of L21 per backward-sweep partial item

// Per-subdomain descriptor.
struct SubDev {
  int nk, nr, nI, nV, nP, ne;  // local DOFs, remaining, r_I, r_V, primal, nr + nP
  int root, pnode;             // r_I supernode, P supernode (-1 if absent)
  long long x_off;             // first row of the subdomain in the sweep matrices (ne rows)
  long long rI_off;            // offset in the concatenated r_I slot arrays
  long long kval_off, f_off;   // raw CSR values / raw loads (nk x nrhs col-major)
  long long lpi_off;           // L_PI packed row-major nP x nI (zeros where not coupled)
  long long tile_off;          // packed L_II tiles (row-block order, TB x TB row-major)
  long long itile_off;         // packed L_II^-1 tiles (same layout; also W = S_II^-1 and S_II tiles)
  long long g_off;             // G_k = L_II^-T L_PI^T: nI x nP row-major (explicit loop)
  long long spart_off;         // (unused by the symmetric pass: see SlotRed / pboff)
  int prim_off, perm_off, nt, cta0;  // primal rows, perm, #tile blocks, first loop CTA
  int blk0;             // first (subdomain, block) index: coarse partial rows of the symmetric pass
  long long npart_off;  // (reserved)
};

// One multiplier's two B entries (every row is {+1, -1} in two subdomains).
struct LamDev {
  int slot[2];    // positions in the concatenated r_I storage
  float sign[2];  // +1 / -1
};

// Work item for the factorisation kernels (k_potrf / k_panel_gemm / extend-add).
struct Work {
  int sn, a, b;
};

// Work item of the batched tile GEMM (factor.cu k_gemm):
// C(m x n tile) = (+/-) A(m x K) B(K x n) (+ C), A[r][k] = A_base[a_off + k*lda + r],
// B[k][c] = B_base[b_off + k*ldb + c] (k_gemm<false>) or B_base[b_off + c*ldb + k]
// (k_gemm<true>), C[r][c] = C_base[c_off + c*ldc + r].
struct GemmWork {
  long long c_off, a_off, b_off;
  int lda, ldb, ldc, m, n, kdim;
  int mode;  // bit0: negate, bit1: accumulate into C, bit2: extend-add epilogue (below),
             // bit3: split-K part (below), bit4: C is a row-major TB x TB tile at c_off
             // (zero padded; with diag, the upper part mirrors the lower), bit5: extend-add
             // with C = 0 (a childless front's update block: not read)
  int diag;  // extend-add: the tile is on the diagonal of U (add only r >= c)
  // extend-add epilogue (multifrontal update of the parent, fused into the SYRK):
  //   parent[p_off + rel[rel_c + c] * p_ld + rel[rel_r + r]] += C[r][c] - (A B)[r][c]
  long long p_off;
  int p_ld, rel_r, rel_c;
  // split-K (deterministic): part ks of nks writes its partial product to
  //   ws[ws_off + ks * TILE_ELEMS] (column-major TB x TB); the last part to arrive
  //   (counter cnt) adds sum_{s=0..nks-1} partial_s, in that order, into C.
  int ks, nks, cnt;
  long long ws_off;
};

// The symmetric pass leaves, for every (subdomain, block j), cnt_j = nseg_j + (nt-1-j)
// partial blocks (TB rows x ncols) stored contiguously from pboff[blk0 + j]: first the
// row-segment products of block row j (nseg_j = j / SYM_SEG + 1), then the transposed
// products of the tiles (i, j), i = j+1 .. nt-1. Per r_I slot (row r of block j):
//   y[slot][c] = sum_{p < cnt} spart[(base + p TB) ncols + c],  base = pboff_j TB + r.
struct SlotRed {
  long long base;
  int cnt, pad_;
};

// A work item of the symmetric tile passes (explicit loop): tiles (o, j0..j1) of the
// lower block row o of one subdomain; segment seg of the row.
constexpr int SYM_SEG = 4;  // tiles per segment
struct SymWork {
  int sub, o, j0, j1, seg, cost;
};

// A chunk of the several-RHS symmetric pass (pcg.cu sym_chunks): the tiles
// [t0, t1) of subdomain `sub` in lower row-major order (tile t = (o, j), t = o(o+1)/2 + j),
// the rank-th chunk of that subdomain; its tiles start at global tile index gtile.
// Every chunk writes one partial block (TB rows x ncols) per block j <= its last row:
// block j of the chunk of rank c goes to cpb[blk0 + j] + c - cfirst[blk0 + j] (partial
// blocks of (subdomain, j) contiguous, in chunk order; SlotRed sums them).
struct SymChunk {
  int sub, t0, t1, rank;
  long long gtile;
};

// One multiplier row of the chunk-mode gathers: its two slots' partial-sum lists
// (SlotRed base/count of the chunk partial blocks) and B signs.
struct GatherRec {
  long long base[2];
  int cnt[2];
  float sign[2];
  int slot[2];  // the two r_I slots (the coarse term G_k z_k of the chunk-mode gather)
};

// A CTA of the loop kernels: one subdomain, one or two TB-blocks (i and nt-1-i).
struct LoopWork {
  int sub, nblk, blk0, blk1;
  int cost;  // tiles streamed by the item (for the persistent kernel's balancing)
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
  std::vector<int32_t> B_dof_sorted;  // supp B, sorted (pattern classes)
  uint64_t fp = 0;                    // fingerprint of the pattern (n, CSR pattern, tree, primal, supp B)
};

struct SnHost {
  int sub, c0, npiv, f, parent, level, coarse;
  std::vector<int> rows;
  std::vector<int> children;
};

struct SubPlan {
  int nr = 0, nI = 0, nV = 0, nP = 0;
  std::vector<int> perm;      // position -> local DOF (ne = nr + nP entries)
  std::vector<int> pos;       // local DOF -> position (-1 for tree DOFs)
  std::vector<int> sn_begin;  // supernode ids of this subdomain [first, last)
  int root = -1, pnode = -1;
};

// Launch ranges of one elimination level.
struct LevelPlan {
  // left-looking panels: GemmWork update of the panel columns with all previous
  // panels (k > 0), POTRF (+ inverse) of the diagonal block (Work), GemmWork TRSM
  // of the rows below with Dinv; then one GemmWork SYRK of the update block.
  struct Panel {
    int potrf_off, potrf_n, trsm_off, trsm_n, upd_off, upd_n;
    // progressive L11^-1 (side stream, after this panel's POTRF): block row kp of
    // L11^-1 = [-Dinv (L[kp][0:kp] L11^-1[0:kp][0:kp]), Dinv]  (Work copy + 2 GemmWork),
    // and (explicit loop, r_I roots) W[0:kp+1][0:kp+1] += L11^-1[kp]^T L11^-1[kp]
    int icopy_off, icopy_n, ia_off, ia_n, ib_off, ib_n, wacc_off, wacc_n;
  };
  std::vector<Panel> panels;
  std::vector<std::pair<int, int>> syrk;     // SYRK + extend-add launches (GemmWork offset, count), one per child slot
  int sn_off = 0, sn_n = 0;                  // supernodes of this level (level_sn list)
  int fs_off = 0, fs_n = 0;                  // forward sweep: solve items (sn, row tile)
  int fu_off = 0, fu_n = 0;                  // forward sweep: update items (sn, update-row tile)
  int bt_off = 0, bt_n = 0;                  // backward sweep: partial items (sn, pivot col tile, row chunk)
  int bx_off = 0, bx_n = 0;                  // backward sweep: x partial items (sn, pivot col tile, row chunk)
  int bxr_off = 0, bxr_n = 0;                // backward sweep: x = sum of the partials (sn, pivot col tile)
  // partitioned inverse L11^-1 by recursive doubling (levels without r_I roots; side
  // stream, once the level's panels are factored)
  int inv_copy_off = 0, inv_copy_n = 0;          // Work items (sn, panel) copying Dinv into L11^-1
  std::vector<std::pair<int, int>> inv_rounds;   // GemmWork ranges, 2 per doubling round
  // front assembly of this level: zero the lower trapezoids (Work items (sn, column
  // tile)), then scatter K's entries (range of the scatter list)
  int zr_off = 0, zr_n = 0;
  long long sc_off = 0, sc_n = 0;
};

struct Plan {
  std::vector<SubPlan> subs;
  std::vector<SnHost> sn;     // all supernodes, global ids
  std::vector<int> level_sn;  // supernode ids grouped by level
  std::vector<LevelPlan> levels;                 // all supernodes by level: assembly and sweeps
  int ngroups = 1;                               // subdomain groups of the factorisation
  std::vector<int> sub_group;                    // group of each subdomain (contiguous blocks)
  std::vector<std::pair<long long, long long>> gfx;  // per group: range of the load scatter list
  std::vector<std::vector<LevelPlan>> glevels;   // [group][level]: panels, SYRK, inverse, sweep lists
  int g_off = 0, g_n = 0;                       // GemmWork: G_k^T = L_PI L_II^-1
  std::vector<std::vector<int>> roots_by_level; // subdomains whose r_I root front is at level L
  long long pool_doubles = 0, dinv_doubles = 0, inv_doubles = 0, vec_rows = 0;
  long long splitk_doubles = 0;  // split-K partials workspace (max over launches)
  long long bpart_doubles = 0;   // backward-sweep partials
  int splitk_tiles = 0;          // split-K counters (max tiles per launch)
  int max_level = 0, max_front = 0, max_nI = 0, nPmax = 0;
  long long nnz_L = 0, flops = 0, inv_flops = 0;
};

}  // namespace ieti
