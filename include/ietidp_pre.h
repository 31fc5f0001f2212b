/*
 * ietidp_pre.h — C ABI of the device pre-processing in front of the IETI-DP solve
 * phase (libietidp.so). Citations "P:<line>" are lines of
 * /root/reference/PAPER.md (Mally & Merkel, arXiv 2501.04340).
 *
 *   torn per-subdomain assembly of the curl-curl stiffness and the loads
 *       K^(k) = C^T M_2(nu) C  (de Rham factorisation: C the face-edge incidence of
 *       the subdomain's control grid, M_2 the 2-form mass matrix), j^(k) = C^T t,
 *       t_f = int T . v_f (weak-curl load of J = curl T; R3)
 *   tree-cotree gauge on the weighted control graph, primal selection
 *       Kruskal's tree under the order (weight, edge id); primal DOFs =
 *       the cotree edges of weight 2 (edges shared by three or more subdomains)
 *
 * What runs where: the spline evaluation (Cox-de Boor), the Gauss sums of the 1-D Gram
 * matrices and load integrals, the Kronecker sums over patches, the product C^T M_2 C
 * (CSR pattern and values) and the spanning tree run in CUDA kernels. The caller
 * supplies data only: knot vectors, quadrature points, quadrature weights already
 * multiplied by the geometry's separable metric factors and by the source's 1-D
 * factors at those points, reluctivities per patch, and the integer edge
 * classification (Dirichlet mask, graph weights).
 *
 * Subdomains are boxes of patches of a tensor-product multipatch grid whose 2-form
 * mass matrix is, per patch and component, a Kronecker product of 1-D Gram matrices
 * (affine cube patches; the exact-circle tube of DESIGN.md R12). Unions of patches
 * that are not boxes are summed box by box by the caller.
 *
 * Conventions as in ietidp.h: 0-based indices, FP64 values, HOST pointers, inputs
 * copied during the call, no call throws; each returns an ietidp_status (ietidp.h) and
 * leaves a message for ietidp_pre_last_error().
 *
 * Local numbering of a box with m[a] = npatch[a]*(e+p-1)+1 control vertices per axis:
 *   edges of direction d live on the grid E_d[a] = m[a] - (a == d); local edge id =
 *   offset_d + i + E_d[0]*(j + E_d[1]*k) (direction, then x fastest);
 *   faces of component c live on F_c[a] = m[a] - (a != c), numbered the same way;
 *   (curl a)_c(n) = a_b(n + e_a) - a_b(n) - a_a(n + e_b) + a_a(n), (c, a, b) cyclic.
 */
#ifndef IETIDP_PRE_H
#define IETIDP_PRE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ietidp_pre_s* ietidp_pre_t; /* opaque: one assembled subdomain on the device */

typedef struct {
  int p;         /* 0-form degree (1..3); 1-forms are the Curry-Schoenberg-scaled splines
                    D_j = p/(t_{j+p+1}-t_{j+1}) B_{j+1,p-1} (R2)                 */
  int e;         /* elements per patch per direction                                       */
  int npatch[3]; /* patches of the box per parametric axis                                 */
  const double* knots[3]; /* open knot vector of the box per axis, m[a]+p+1 knots, patch
                             boundaries of multiplicity p (C^0 gluing)                      */
  int nq;        /* Gauss points per element of the Gram matrices                           */
  const double* qx[3];    /* points per axis: npatch[a]*e*nq, ascending (patch, element, point) */
  const double* qw[3][3]; /* [c][a]: quadrature weight times the metric factor of 2-form
                             component c along axis a at qx[a] (cube: the plain weights)    */
  const double* nu;       /* reluctivity per patch of the box, x fastest                     */
  const int32_t* dof_of_edge; /* per local edge: its DOF index (ascending with the edge id) or
                                 -1 for a Dirichlet edge (n x A = 0)                   */
  int n_dof;
  /* loads: t_f = sum over terms of coef * vx[f_x] vy[f_y] vz[f_z] on component comp,
     v_a[i] = sum over load points of fac_val[a][u][pt] * phi_i(lx[a][pt]) with phi the
     B-splines when kind = 0, the D-splines when kind = 1 (kind must be 0 on the
     component's own axis and 1 on the other two)                                         */
  int nrhs;
  int lq;                  /* load quadrature points per element                           */
  const double* lx[3];     /* load points per axis: npatch[a]*e*lq                          */
  int nfac[3];             /* distinct 1-D factors per axis                                 */
  const int32_t* fac_kind[3]; /* nfac[a]: 0 = B, 1 = D                                      */
  const double* fac_val[3];   /* nfac[a] x (npatch[a]*e*lq), row-major: weight * f(point)   */
  int nterms;
  const int32_t* term_col;  /* nterms: RHS column                                          */
  const int32_t* term_comp; /* nterms: 2-form component 0..2                                */
  const int32_t* term_fac;  /* nterms x 3: factor index per axis                            */
  const double* term_coef;  /* nterms                                                       */
} ietidp_pre_subdomain;

/* Assemble K^(k) = C^T M_2 C and j^(k) = C^T t of one box subdomain on `device`
 * (P:49-57), Dirichlet rows and columns removed. The result stays on the device
 * inside *out: a CSR matrix with both triangles, columns ascending per row, exactly
 * symmetric (the entry (i, j), j < i, and its mirror are computed by the same sum), on
 * the structural pattern of the product (an entry that cancels to 0.0 is kept), and the
 * loads n_dof x nrhs column-major.
 * Errors: E_ARG (null pointers, sizes, degree outside 1..3, a factor kind that does not
 * match its term, dof_of_edge not ascending), E_CUDA, E_NOMEM. */
int ietidp_pre_assemble(int device, const ietidp_pre_subdomain* s, ietidp_pre_t* out);

/* The same for n subdomains of one workload in one pass: all inputs travel in one upload,
 * and every stage is ONE launch over the whole batch (k_stage1d: a CTA per subdomain;
 * k_rows: grid.y = subdomain), so the value kernel runs at a full-GPU grid. out[0..n)
 * receive one handle per subdomain (each released with ietidp_pre_destroy; they share
 * the batch's device memory, freed with the last of them). Errors as above; on failure no
 * handle is returned. */
int ietidp_pre_assemble_batch(int device, int n, const ietidp_pre_subdomain* subs, ietidp_pre_t* out);

/* n_dof and nnz of the assembled matrix (for a batch, ms and ms_fill are the batch's); ms = device time of the assembly kernels
 * (CUDA events; uploads excluded); ms_fill = of the value kernel alone (the dominant one:
 * 12 bytes written per entry). Any pointer may be NULL. */
int ietidp_pre_sizes(ietidp_pre_t a, int* n_dof, int64_t* nnz, double* ms, double* ms_fill);

/* Copy the assembled CSR matrix and loads to the host: rowptr[n_dof+1] (int64),
 * col[nnz], val[nnz], f[n_dof*nrhs] column-major -- the arguments of
 * ietidp_set_subdomain. Any pointer may be NULL. */
int ietidp_pre_get(ietidp_pre_t a, int64_t* rowptr, int32_t* col, double* val, double* f);

/* New reluctivities, same discretisation: nu_all holds every subdomain's nu array of the
 * handle's batch, concatenated in batch order (host). Only the value kernel reruns; pattern,
 * Gram tables and loads are unchanged (the loads do not depend on nu). ms = its device time.
 * The values are rewritten in place (the device pointers stay valid). */
int ietidp_pre_refill(ietidp_pre_t a, const double* nu_all, double* ms);

/* Device pointers of the assembled values and loads (owned by the handle's batch; valid until
 * its last handle is destroyed; the assembly has completed when ietidp_pre_assemble[_batch]
 * returns): d_val[nnz] in the CSR order of ietidp_pre_get, d_f[n_dof*nrhs] column-major --
 * the arguments of ietidp_set_values_device, which keeps the matrix on the device between
 * assembly and factorisation. Any pointer may be NULL. */
int ietidp_pre_device_ptrs(ietidp_pre_t a, const double** d_val, const double** d_f);

/* The 1-D Gram block of component c, axis a, patch q (host, nb x nb column-major, nb =
 * e+p for the B kind (a == c), e+p-1 for the D kind): test access to the first stage. */
int ietidp_pre_get_gram(ietidp_pre_t a, int c, int axis, int q, double* block, int* nb);

const char* ietidp_pre_last_error(void);
void ietidp_pre_destroy(ietidp_pre_t a);

/* Tree-cotree gauge and primal selection on the device. The control graph
 * has nv vertices and ne edges (eu[e], ev[e]) with integer weights w[e] in 1..5 (Fig. 2:
 * P:160-177). in_tree[e] = 1 for the edges of Kruskal's spanning forest under the total
 * order (w[e], e) (ties by edge id, R4): computed as Boruvka rounds,
 * which give the same forest because the order is total (the minimum spanning forest is
 * unique). primal[e] = 1 for the cotree edges of weight 2. ms = device time.
 * in_tree, primal: host, ne bytes each; primal and ms may be NULL.
 * Errors: E_ARG (null, endpoints out of range, weight outside 1..5), E_CUDA, E_NOMEM. */
int ietidp_pre_gauge(int device, int64_t nv, int64_t ne, const int32_t* eu, const int32_t* ev,
                     const int8_t* w, uint8_t* in_tree, uint8_t* primal, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* IETIDP_PRE_H */
