/*
 * ietidp.h — C ABI of the B200 IETI-DP solve phase (libietidp.so).
 *
 * The library solves the dual-primal isogeometric tearing-and-interconnecting
 * system of Mally & Merkel, "On Domain Decomposition for Magnetostatic Problems
 * in 3D" (arXiv 2501.04340; /root/reference/PAPER.md, cited "P:<line>"):
 *
 *   partially assembled saddle system Eq. (5)
 *   local elimination a_r = K_rr^-1(...) Eq. (6)
 *   interface problem Eq. (7), operators F,G,W,d,e
 *   coarse recovery Eq. (8), local recovery Eq. (9)
 *   PCG with Dirichlet preconditioner Eq. (10)
 *
 * in the SPD sign convention (reading R1):
 *   S_PP  = C_p^T (K_pp - K_pr K_rr^-1 K_rp) C_p  (= -F of P:134)
 *   F_DP  = W + G S_PP^-1 G^T                     (= -S of P:128)
 *   d_DP  = e - G S_PP^-1 ftilde,  ftilde = C_p^T (j_p - K_pr K_rr^-1 j_r)
 *
 * Everything numeric runs on the GPU (sm_100a); the host does input validation,
 * DOF classification and the symbolic analysis (ordering, supernodes) only.
 *
 * Conventions (all entry points):
 *  - indices are 0-based; int32 unless stated; values are IEEE FP64;
 *  - pointers are HOST pointers unless the parameter name starts with d_
 *    (device pointers on the handle's device);
 *  - the caller owns every input; inputs are copied during the call and may be
 *    freed on return;
 *  - the handle owns all device memory; handles are not thread-safe, separate
 *    handles are independent;
 *  - no call throws; each returns an ietidp_status and, on failure, leaves a
 *    message for ietidp_last_error(). The handle stays valid for
 *    ietidp_last_error / ietidp_destroy after any failure.
 */
#ifndef IETIDP_H
#define IETIDP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IETIDP_MAX_RHS 64

typedef struct ietidp_s* ietidp_t; /* opaque; owns all device memory */

typedef enum {
  IETIDP_OK = 0,
  IETIDP_E_ARG = 1,            /* null pointer, size/index out of range, unsorted or
                                  non-symmetric CSR pattern, duplicate DOF in a set   */
  IETIDP_E_STATE = 2,          /* call order violated: solve before factor, set twice,
                                  factor with a subdomain missing, solve after a failed
                                  factor                                               */
  IETIDP_E_B_STRUCTURE = 3,    /* a multiplier row is not exactly {+1,-1} in two
                                  distinct subdomains (non-redundant P:116), a DOF
                                  in more than one row, or B touching a tree/primal DOF */
  IETIDP_E_NOT_SPD = 4,        /* K_rr^(k) (report.failed_subdomain = k) or S_PP
                                  (failed_subdomain = -1) has a non-positive pivot:
                                  the gauge did not make the local problem invertible
                                                                     */
  IETIDP_E_NO_CONVERGENCE = 5, /* max_iter reached; lambda/u hold the last iterate     */
  IETIDP_E_CUDA = 6,           /* a CUDA runtime error (message has the details)       */
  IETIDP_E_NOMEM = 7           /* device or host allocation failed                     */
} ietidp_status;

typedef enum {
  IETIDP_SCALE_MULTIPLICITY = 0, /* delta = 1/2 on every multiplier: iterates identical
                                    to the paper's D_s = I (R5)        */
  IETIDP_SCALE_STIFFNESS = 1     /* delta_a^(k) = K^(l)_bb / (K^(k)_aa + K^(l)_bb), b the
                                    partner DOF of a in neighbour l (R5)      */
} ietidp_scaling;

typedef enum {
  IETIDP_LOOP_EXPLICIT = 0,   /* default: the loop applies W_k = S_II^-1 and S_II, each stored once
                                 as a symmetric lower-tile matrix and streamed in one pass per
                                 operator; G_k = L_II^-T L_PI^T explicit       */
  IETIDP_LOOP_TRIANGULAR = 1  /* forward/backward substitutions with L_II^-1 and L_II per iteration
                                 (two passes per operator)                      */
} ietidp_loop;

typedef enum {
  IETIDP_ORDER_NESTED_DISSECTION = 0, /* default: nested dissection of r_V, r_I last     */
  IETIDP_ORDER_DENSE = 1,             /* r_V as one dense supernode (test/oracle aid)    */
  IETIDP_ORDER_MIN_DEGREE = 2         /* approximate minimum degree of r_V, fundamental
                                         supernodes, r_I last                           */
} ietidp_ordering;

typedef enum {
  IETIDP_STOP_RESIDUAL = 0,       /* ||r_k||_2 <= tol ||r_0||_2: the unpreconditioned dual
                                     residual (BASELINE "dual residual <= 1e-10") */
  IETIDP_STOP_PRECONDITIONED = 1  /* sqrt(r_k^T z_k) <= tol sqrt(r_0^T z_0), z = M_D^-1 r: the
                                     preconditioned residual of the paper's experiments
                                     (eta_tol); tested after the
                                     preconditioner apply of each iteration (persistent PCG
                                     kernel only)                                            */
} ietidp_stop;

typedef struct {
  double tol;       /* PCG stop: per column, criterion ietidp_stop below; default ||r_k||_2 <= tol
                       ||r_0||_2, unpreconditioned dual residual, r_0 = d_DP, lambda_0 = 0;
                       default 1e-10                                                         */
  int max_iter;     /* default 500                                                        */
  int scaling;      /* ietidp_scaling; default IETIDP_SCALE_MULTIPLICITY                   */
  int fixed_iters;  /* > 0: run exactly this many iterations, no stop test (parity mode)  */
  int ordering;     /* ietidp_ordering; default nested dissection                         */
  int leaf_size;    /* nested-dissection leaf size (supernode of the leaves); default 96  */
  int loop;         /* ietidp_loop: operators of the PCG loop; default IETIDP_LOOP_EXPLICIT */
  int stop;         /* ietidp_stop: PCG stopping criterion; default IETIDP_STOP_RESIDUAL      */
  int device;       /* CUDA device ordinal; default 0                                     */
  void* stream;     /* cudaStream_t all work is issued on; NULL = library-owned stream    */
} ietidp_options;

typedef struct {
  int n_sub, n_lambda, n_primal, nrhs, failed_subdomain;
  int n_supernodes, n_levels, max_front, max_nI;
  long long sum_nr, sum_nI, nnz_L;
  long long factor_flops;        /* sum over supernode columns of c_j^2 (c_j = column count
                                    of L incl. diagonal), the factorisation's useful flops */
  long long pcg_bytes_per_iter;  /* algorithmic HBM bytes of one PCG iteration */
  long long f_apply_bytes;       /* algorithmic bytes of one F-apply (one column)          */
  int iters[IETIDP_MAX_RHS];     /* F-applies per column in the PCG loop                   */
  int converged[IETIDP_MAX_RHS];
  double rel_residual[IETIDP_MAX_RHS]; /* true ||d - F lambda|| / ||d|| after the loop     */
  double ms_analyze, ms_factor, ms_coarse, ms_pcg, ms_recover; /* CUDA-event / host times:
                                    ms_analyze = host symbolic analysis (validation, pattern
                                    classes, ordering, plan), without the device part     */
  double ms_upload;              /* device allocations, uploads and scatter-list expansion
                                    of ietidp_analyze (host wall time)                     */
  int n_pattern_classes;         /* distinct subdomain patterns (analysed once each)       */
} ietidp_report;

/* Defaults as documented in ietidp_options. */
void ietidp_options_default(ietidp_options* opt);

/* Create a handle for n_sub subdomains, n_lambda multipliers (rows of B_r),
 * n_primal global primal DOFs (columns of C_p) and nrhs right-hand sides
 * (1..IETIDP_MAX_RHS). n_lambda = 0 and n_primal = 0 are legal.
 * Errors: E_ARG (sizes), E_CUDA (device), E_NOMEM. */
ietidp_status ietidp_create(const ietidp_options* opt, int n_sub, int n_lambda,
                            int n_primal, int nrhs, ietidp_t* out);

/* Describe subdomain k: its n_k non-Dirichlet local DOFs.
 *  K_rowptr[n_k+1] (int64), K_col[nnz], K_val[nnz]: the full symmetric local
 *      stiffness K^(k) in CSR, both triangles, columns sorted per row;
 *  f[n_k*nrhs]: local loads j^(k), column-major (n_k x nrhs);
 *  nB, B_lambda[nB], B_dof[nB], B_sign[nB]: the nonzeros of B_r^(k) in COO:
 *      multiplier row, local DOF, sign +1/-1. Every remaining DOF shared with
 *      another subdomain carries exactly one entry (R6);
 *  n_tree, tree_dofs: local DOFs of the tree-cotree gauge's tree, which
 *      are eliminated (value 0);
 *  n_prim, prim_dofs, prim_global: local primal DOFs and their global
 *      primal ids (the nonzeros of C_p).
 * All other DOFs are "remaining" (r). Validation: E_ARG (ranges, CSR sortedness,
 * pattern symmetry, overlapping sets), E_STATE (k set twice or after analysis). */
ietidp_status ietidp_set_subdomain(ietidp_t h, int k, int n_k,
                                   const int64_t* K_rowptr, const int32_t* K_col,
                                   const double* K_val, const double* f,
                                   int nB, const int32_t* B_lambda, const int32_t* B_dof,
                                   const int8_t* B_sign,
                                   int n_tree, const int32_t* tree_dofs,
                                   int n_prim, const int32_t* prim_dofs,
                                   const int32_t* prim_global);

/* Host-side set-up: validate B across subdomains (E_B_STRUCTURE), classify DOFs
 * (tree, primal, r_V, r_I = supp B_r), order r_V by nested dissection with
 * r_I last, symbolic supernodal analysis, device allocation and upload of all
 * values. Called implicitly by ietidp_factor if not called before. */
ietidp_status ietidp_analyze(ietidp_t h);

/* Replace the numeric values (same pattern) of subdomain k after analysis:
 * K_val[nnz] and f[n_k*nrhs] (host; either may be NULL to keep the current values).
 * The copy is asynchronous, on an internal stream ordered after the handle's stream;
 * the caller's buffers must stay unchanged until the next ietidp_factor returns (use
 * page-locked memory for an asynchronous copy). The next ietidp_factor uses the values:
 * each subdomain group of the factorisation starts as soon as its subdomains' copies
 * have arrived, so the transfer overlaps the factorisation of earlier groups. */
ietidp_status ietidp_set_values(ietidp_t h, int k, const double* K_val, const double* f);

/* The same from DEVICE buffers on the handle's device (e.g. the matrix the device assembly
 * of ietidp_pre.h has just produced, ietidp_pre_device_ptrs): d_K_val[nnz] in the CSR order
 * of ietidp_set_subdomain, d_f[n_k*nrhs] column-major; device-to-device copies on the
 * handle's stream, so work the caller has ordered before this call on that stream (or
 * completed) is visible. Either pointer may be NULL.
 * Errors: E_STATE (before analysis, host-only handle), E_ARG (k out of range), E_CUDA. */
ietidp_status ietidp_set_values_device(ietidp_t h, int k, const double* d_K_val, const double* d_f);

/* The same with half the bytes: K_lower_val holds only the values of the stored entries
 * (i, j) with j <= i of subdomain k's CSR pattern, in CSR order (row by row, columns
 * ascending) -- K is symmetric (K = C^T M_2 C), so an upper entry's value is its
 * mirror's. The library expands them on the device into its full CSR value array
 * (k_expand_lower). Copy semantics as for ietidp_set_values: asynchronous on the copy
 * stream, ordered before the next ietidp_factor; the caller's buffers must stay
 * unchanged until that factorisation returns. The first call builds the per-pattern-class
 * maps (host integer work, once per handle). Either pointer may be NULL (keep).
 * Errors: E_STATE (before analysis, host-only handle), E_ARG (k out of range), E_CUDA. */
ietidp_status ietidp_set_values_lower(ietidp_t h, int k, const double* K_lower_val, const double* f);

/* Device numeric phase: batched supernodal Cholesky of every K_rr^(k)
 * (its trailing block is L_II, L_II L_II^T = S_{r_I r_I} of Eq. (10)),
 * coarse basis X_k = K_rr^-1 K_rP, S_PP and its factorisation, G, and d_DP.
 * Errors: E_NOT_SPD (report.failed_subdomain), E_STATE, E_CUDA. */
ietidp_status ietidp_factor(ietidp_t h);

/* PCG on F_DP lambda = d_DP (variant of DESIGN.md) followed by the recovery
 * Eqs. (8)-(9). lambda (host, n_lambda x nrhs column-major) may be NULL.
 * report may be NULL. Returns E_NO_CONVERGENCE if a column hit max_iter. */
ietidp_status ietidp_solve(ietidp_t h, double* lambda, ietidp_report* report);

/* Subdomain solution u^(k) = [a_r; a_p = C_k p; tree = 0] of the last
 * solve, host n_k x nrhs column-major. */
ietidp_status ietidp_get_u(ietidp_t h, int k, double* u);

/* Same as ietidp_get_u / lambda of ietidp_solve, into device buffers (stream-ordered
 * on the handle's stream). */
ietidp_status ietidp_get_u_device(ietidp_t h, int k, double* d_u);
ietidp_status ietidp_get_lambda_device(ietidp_t h, double* d_lambda);

/* Operator access for tests and the F-applies/s benchmark; device pointers,
 * n_lambda x ncols column-major, 1 <= ncols <= nrhs, issued on the handle's stream
 * (asynchronous; synchronise the stream before reading d_y).
 *   y = F_DP x = sum_k B_I L_II^-T L_II^-1 B_I^T x + G S_PP^-1 G^T x   (F2)
 *   y = M_D^-1 x = sum_k B_D L_II L_II^T B_D^T x
 * applied with the handle's loop operators (ietidp_options.loop). */
ietidp_status ietidp_apply_F(ietidp_t h, int ncols, const double* d_x, double* d_y);
ietidp_status ietidp_apply_precond(ietidp_t h, int ncols, const double* d_x, double* d_y);

/* The assembled coarse matrix S_PP (n_primal x n_primal, host, symmetric). */
ietidp_status ietidp_get_coarse(ietidp_t h, double* S_PP);

/* Condition estimate of the preconditioned interface operator M_D^-1 F_DP after a
 * solve (Eq. (11): cond = omega_max / omega_min; SPEC
 * estimate_condition): per column c, the extreme eigenvalues of the
 * Lanczos tridiagonal built from that column's PCG coefficients alpha_j, beta_j
 * (T_jj = 1/alpha_j + beta_{j-1}/alpha_{j-1}, T_{j,j+1} = sqrt(beta_j)/alpha_j),
 * computed on the device by Sturm-count multisection. Outputs are host arrays of
 * nrhs doubles (any may be NULL); a column with 0 iterations reports 0, 0, 0; one
 * iteration gives cond = 1. The Ritz values lie inside the spectrum, so the
 * estimate never exceeds the true condition number.
 * Errors: E_STATE before a solve, E_CUDA. */
ietidp_status ietidp_estimate_condition(ietidp_t h, double* omega_min, double* omega_max, double* cond);

/* The PCG coefficients of the last solve (host, ld x nrhs column-major each,
 * ld >= max iterations): alpha[c*ld + j] for j < iters[c], beta[c*ld + j] for
 * j < iters[c] - 1 (p_{j+1} = z_{j+1} + beta_j p_j); other entries are 0.
 * Errors: E_STATE before a solve, E_ARG (ld smaller than an iteration count). */
ietidp_status ietidp_get_pcg_coefficients(ietidp_t h, int ld, double* alpha, double* beta);

/* d_DP (host, n_lambda x nrhs column-major). */
ietidp_status ietidp_get_rhs(ietidp_t h, double* d);

/* Counters and timings of the last analyze/factor/solve. */
ietidp_status ietidp_get_report(ietidp_t h, ietidp_report* report);

/* Number of this library's kernel launches issued since the handle was created
 * (graph-launched kernel nodes counted per execution). */
long long ietidp_kernel_launches(ietidp_t h);

const char* ietidp_last_error(ietidp_t h);
const char* ietidp_status_string(ietidp_status s);
void ietidp_destroy(ietidp_t h);

#ifdef __cplusplus
}
#endif
#endif /* IETIDP_H */
