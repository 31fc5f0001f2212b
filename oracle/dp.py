"""ORACLE — test infrastructure only. Plain, slow CPU FP64 IETI-DP solve phase.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module. It shares no code with the CUDA path (paper_2501_04340_b200/) and
imports nothing from it.

It follows PAPER.md §2.1 step by step, in the SPD sign convention of SURVEY F1
(S_PiPi = -F_paper, F_DP = -S_paper; DESIGN.md "Readings" R1):

  Eq. (5)  partially assembled saddle system;
  Eq. (6)  a_r = K_rr^-1 (j_r - K_rp C_p p - B_r^T lambda);
  Eq. (7)  interface problem, operators of PAPER.md:133-139:
           S_PiPi = C_p^T (K_pp - K_pr K_rr^-1 K_rp) C_p          (= -F)
           G      = B_r K_rr^-1 K_rp C_p
           W      = B_r K_rr^-1 B_r^T
           ftilde = C_p^T (j_p - K_pr K_rr^-1 j_r)                (= -d)
           e      = B_r K_rr^-1 j_r
           F_DP   = W + G S_PiPi^-1 G^T ,  d_DP = e - G S_PiPi^-1 ftilde
  Eq. (8)      p   = S_PiPi^-1 (ftilde + G^T lambda)
  Eq. (9)      a_r = K_rr^-1 (j_r - K_rp C_p p - B_r^T lambda)
  Eq. (10)  M_D^-1 = sum_k B_D S_{r_I r_I} B_D^T with
           S_{r_I r_I} = K_II - K_IV K_VV^-1 K_VI formed explicitly from a
           separate factorisation of K_VV (independent of the CUDA path's reuse
           of the trailing Cholesky block).
  PCG, the variant of SURVEY §8(c): lambda_0 = 0, stop when
  ||r||_2 <= tol ||r_0||_2, one F-apply per iteration; columns independent.

Scaling D_s (R5): "multiplicity" delta = 1/2,
"stiffness" delta_a^(k) = K^(l)_bb / (K^(k)_aa + K^(l)_bb).
"""
import numpy as np
import scipy.linalg as la
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class LocalSingular(Exception):
    def __init__(self, k):
        super().__init__(f"K_rr of subdomain {k} is not SPD")
        self.k = k


def _factor(A, k, check_spd):
    """Direct factorisation of a sparse SPD block (library primitive)."""
    if A.shape[0] == 0:
        return None
    if check_spd:
        try:
            np.linalg.cholesky(A.toarray())
        except np.linalg.LinAlgError:
            raise LocalSingular(k)
    return spla.splu(sp.csc_matrix(A), permc_spec="MMD_AT_PLUS_A",
                     diag_pivot_thresh=0.0, options=dict(SymmetricMode=True))


def _solve(lu, X):
    if lu is None:
        return np.zeros_like(X)
    return lu.solve(np.asarray(X, dtype=np.float64))


class Local:
    """Blocks of one subdomain after the dual-primal split."""

    def __init__(self, k, s, n_lambda, check_spd):
        n = s["n"]
        K = sp.csr_matrix((s["K_data"], s["K_indices"], s["K_indptr"]), shape=(n, n))
        f = np.asarray(s["f"]).reshape(-1, n).T          # n x nrhs
        tree = np.asarray(s["tree"], np.int64)
        prim = np.asarray(s["prim"], np.int64)
        mask = np.ones(n, bool)
        mask[tree] = False
        mask[prim] = False
        r = np.flatnonzero(mask)                          # natural order
        self.k, self.n, self.r, self.prim = k, n, r, prim
        self.prim_gid = np.asarray(s["prim_gid"], np.int64)
        self.K, self.f = K, f
        self.Krr = K[r][:, r].tocsc()
        self.Krp = K[r][:, prim].tocsc()
        self.Kpp = K[prim][:, prim].toarray()
        self.jr, self.jp = f[r], f[prim]
        pos = -np.ones(n, np.int64)
        pos[r] = np.arange(len(r))
        bd = np.asarray(s["B_dof"], np.int64)
        assert np.all(pos[bd] >= 0), "B touches a tree/primal DOF"
        self.B_lambda = np.asarray(s["B_lambda"], np.int64)
        self.B_sign = np.asarray(s["B_sign"], np.float64)
        self.B_dof = bd
        self.B_rpos = pos[bd]
        # B_r^(k): m_r x n_r signed Boolean
        self.Br = sp.csr_matrix((self.B_sign, (self.B_lambda, self.B_rpos)),
                                shape=(n_lambda, len(r)))
        self.lu = _factor(self.Krr, k, check_spd)
        # r_I = remaining DOFs on an interface = supp B; r_V the rest
        isI = np.zeros(len(r), bool)
        isI[self.B_rpos] = True
        self.rI = np.flatnonzero(isI)
        self.rV = np.flatnonzero(~isI)

    def Kinv(self, X):
        return _solve(self.lu, X)

    def schur_II(self, check_spd):
        """S_{r_I r_I} = K_II - K_IV K_VV^-1 K_VI (Eq. 10), dense."""
        KII = self.Krr[self.rI][:, self.rI].toarray()
        if len(self.rV) == 0 or len(self.rI) == 0:
            return KII
        KVV = self.Krr[self.rV][:, self.rV]
        KVI = self.Krr[self.rV][:, self.rI].toarray()
        luV = _factor(KVV, self.k, check_spd)
        return KII - KVI.T @ _solve(luV, KVI)


class DualPrimal:
    """The operators of PAPER.md:133-139 (SPD signs) and the PCG of :142."""

    def __init__(self, bundle, scaling=None, check_spd=False):
        self.nl = int(bundle["n_lambda"])
        self.ng = int(bundle["n_primal"])
        self.nrhs = int(bundle["nrhs"])
        self.scaling = scaling or bundle["scaling"]
        self.loc = [Local(k, s, self.nl, check_spd) for k, s in enumerate(bundle["subs"])]
        nl, ng = self.nl, self.ng
        S = np.zeros((ng, ng))
        G = np.zeros((nl, ng))
        ft = np.zeros((ng, self.nrhs))
        e = np.zeros((nl, self.nrhs))
        for L in self.loc:
            Cp = sp.csr_matrix((np.ones(len(L.prim)), (np.arange(len(L.prim)), L.prim_gid)),
                               shape=(len(L.prim), ng))
            L.Cp = Cp
            X = L.Kinv(L.Krp.toarray()) if len(L.prim) else np.zeros((len(L.r), 0))
            y = L.Kinv(L.jr)
            L.X = X
            L.y = y
            S += Cp.T @ (L.Kpp - L.Krp.T @ X) @ Cp
            G += L.Br @ X @ Cp
            ft += Cp.T @ (L.jp - L.Krp.T @ y)
            e += L.Br @ y
        self.S = (S + S.T) * 0.5 if ng else S
        self.G = G
        self.ftilde = ft
        self.e = e
        if ng:
            self.Sc = la.cho_factor(self.S, lower=True)
            self.d = e - G @ la.cho_solve(self.Sc, ft)
        else:
            self.Sc = None
            self.d = e.copy()
        self._precond_setup(check_spd)

    def Sinv(self, x):
        if self.ng == 0:
            return np.zeros((0,) + x.shape[1:])
        return la.cho_solve(self.Sc, x)

    # ---- F_DP = W + G S^-1 G^T (sign flipped per F1) --------
    def apply_W(self, lam):
        out = np.zeros_like(lam)
        for L in self.loc:
            out += L.Br @ L.Kinv(L.Br.T @ lam)
        return out

    def apply_F(self, lam):
        lam = np.asarray(lam, dtype=np.float64)
        out = self.apply_W(lam)
        if self.ng:
            out += self.G @ self.Sinv(self.G.T @ lam)
        return out

    # ---- Dirichlet preconditioner ----------------------
    def _precond_setup(self, check_spd):
        owner = {}
        for L in self.loc:
            L.SII = L.schur_II(check_spd)
            # B_I^(k): rows lambda, cols positions within r_I
            posI = -np.ones(len(L.r), np.int64)
            posI[L.rI] = np.arange(len(L.rI))
            L.B_Ipos = posI[L.B_rpos]
            diagK = L.Krr.diagonal()
            for lam, rp in zip(L.B_lambda, L.B_rpos):
                owner.setdefault(int(lam), []).append((L.k, float(diagK[rp])))
        for L in self.loc:
            delta = np.empty(len(L.B_lambda))
            for i, lam in enumerate(L.B_lambda):
                pair = owner[int(lam)]
                assert len(pair) == 2
                mine = [kk for kk in pair if kk[0] == L.k][0][1]
                other = [kk for kk in pair if kk[0] != L.k][0][1]
                if self.scaling == "multiplicity":
                    delta[i] = 0.5
                else:
                    delta[i] = other / (mine + other)
            L.delta = delta
            L.BD = sp.csr_matrix((L.B_sign * delta, (L.B_lambda, L.B_Ipos)),
                                 shape=(self.nl, len(L.rI)))

    def apply_M(self, r):
        out = np.zeros_like(r)
        for L in self.loc:
            out += L.BD @ (L.SII @ (L.BD.T @ r))
        return out

    # ---- PCG (SURVEY §8(c) variant) ---------------------------------------
    def pcg(self, tol=1e-10, max_iter=500, fixed_iters=0, d=None, stop="residual"):
        """stop="residual": ||r_k|| <= tol ||r_0|| tested after the r update (SURVEY §8(c)
        variant, BASELINE's dual residual); stop="preconditioned": sqrt(r_k.z_k) <= tol
        sqrt(r_0.z_0) tested after the preconditioner apply (the paper's eta_tol of its
        experiments)."""
        d = self.d if d is None else d
        nl, nc = d.shape
        lam = np.zeros((nl, nc))
        r = d.copy()
        r0 = np.linalg.norm(r, axis=0)
        iters = np.zeros(nc, np.int64)
        active = r0 > 0
        if nl == 0:
            active[:] = False
        z = self.apply_M(r)
        p = z.copy()
        rz = np.sum(r * z, axis=0)
        rz0 = rz.copy()
        alphas = [[] for _ in range(nc)]  # per column: alpha_j, beta_j (Lanczos, cond_lanczos)
        betas = [[] for _ in range(nc)]
        it = 0
        while np.any(active):
            if fixed_iters and it >= fixed_iters:
                break
            if not fixed_iters and it >= max_iter:
                break
            a = np.flatnonzero(active)
            q = self.apply_F(p[:, a])
            pq = np.sum(p[:, a] * q, axis=0)
            alpha = rz[a] / pq
            for c, v in zip(a, alpha):
                alphas[c].append(v)
            lam[:, a] += alpha * p[:, a]
            r[:, a] -= alpha * q
            iters[a] += 1
            it += 1
            rn = np.linalg.norm(r[:, a], axis=0)
            if not fixed_iters and stop == "residual":
                done = rn <= tol * r0[a]
                active[a[done]] = False
                a = np.flatnonzero(active)
                if len(a) == 0:
                    break
            zz = self.apply_M(r[:, a])
            rz_new = np.sum(r[:, a] * zz, axis=0)
            if not fixed_iters and stop == "preconditioned":
                done = np.sqrt(np.maximum(rz_new, 0.0)) <= tol * np.sqrt(rz0[a])
                active[a[done]] = False
                keep = ~done
                a, zz, rz_new = a[keep], zz[:, keep], rz_new[keep]
                if len(a) == 0:
                    break
            beta = rz_new / rz[a]
            for c, v in zip(a, beta):
                betas[c].append(v)
            p[:, a] = zz + beta * p[:, a]
            rz[a] = rz_new
        converged = ~active if not fixed_iters else np.ones(nc, bool)
        true_res = np.linalg.norm(d - self.apply_F(lam), axis=0) / np.where(r0 > 0, r0, 1.0)
        return lam, dict(iters=iters, converged=converged, rel_residual=true_res,
                         alpha=[np.array(x) for x in alphas],
                         beta=[np.array(x[:max(len(y) - 1, 0)]) for x, y in zip(betas, alphas)])

    # ---- recovery, Eqs. (8)-(9) -------------------------------------------
    def recover(self, lam):
        nc = lam.shape[1]
        p = self.Sinv(self.ftilde + self.G.T @ lam) if self.ng else np.zeros((0, nc))
        us = []
        for L in self.loc:
            pk = L.Cp @ p
            ar = L.Kinv(L.jr - L.Krp @ pk - L.Br.T @ lam)
            u = np.zeros((L.n, nc))
            u[L.r] = ar
            u[L.prim] = pk
            us.append(u)
        return us, p


def lanczos_tridiagonal(alpha, beta):
    """The Lanczos matrix T_k of the preconditioned operator M^-1 F from k PCG
    iterations (the CG-Lanczos relation, e.g. Saad, Iterative Methods, §6.7.3;
    SURVEY §8(c) Q25): T_jj = 1/alpha_j + beta_{j-1}/alpha_{j-1} (beta_{-1} = 0),
    T_{j,j+1} = T_{j+1,j} = sqrt(beta_j)/alpha_j, j = 0..k-1."""
    alpha = np.asarray(alpha, float)
    beta = np.asarray(beta, float)
    k = len(alpha)
    T = np.zeros((k, k))
    for j in range(k):
        T[j, j] = 1.0 / alpha[j] + (beta[j - 1] / alpha[j - 1] if j > 0 else 0.0)
        if j + 1 < k:
            T[j, j + 1] = T[j + 1, j] = np.sqrt(beta[j]) / alpha[j]
    return T


def cond_lanczos(alpha, beta):
    """(omega_min, omega_max, cond) of M_D^-1 F_DP estimated from the PCG coefficients:
    the extreme eigenvalues of T_k (cond = omega_max / omega_min).
    0 iterations: (0, 0, 0)."""
    if len(alpha) == 0:
        return 0.0, 0.0, 0.0
    w = np.linalg.eigvalsh(lanczos_tridiagonal(alpha, beta))
    return w[0], w[-1], w[-1] / w[0]


def cond_dense(D):
    """(omega_min, omega_max, cond) of M_D^-1 F_DP from its dense spectrum (small
    cases only): F_DP and M_D^-1 applied to the identity, eigenvalues of the product
    (similar to the symmetric M^1/2 F M^1/2, so real and positive)."""
    E = np.eye(D.nl)
    F = D.apply_F(E)
    M = D.apply_M(E)
    w = np.sort(np.linalg.eigvals(M @ F).real)
    return w[0], w[-1], w[-1] / w[0]


def solve(bundle, tol=None, max_iter=500, fixed_iters=0, scaling=None, check_spd=False, stop="residual"):
    """Full oracle solve: returns dict(lam, u (list n_k x nrhs), iters, ...)."""
    dp = DualPrimal(bundle, scaling=scaling, check_spd=check_spd)
    tol = bundle["tol"] if tol is None else tol
    lam, info = dp.pcg(tol=tol, max_iter=max_iter, fixed_iters=fixed_iters, stop=stop)
    us, p = dp.recover(lam)
    return dict(lam=lam, u=us, p=p, dp=dp, **info)
