"""ORACLE — test infrastructure only. Brute-force references for small inputs.

* `saddle_solve`: one sparse direct solve of the partially assembled system
  Eq. (5) — unknowns [a_r (all subdomains), p, lambda_r].
* `monolithic_solve`: the gauged global Galerkin system K_g a_g = j_g
   restricted to non-Dirichlet, non-tree DOFs,
  assembled from the torn blocks by summation and distributed back to the
  subdomains. For the exact multipliers the IETI-DP solution equals it.
Neither shares any step with oracle/dp.py beyond reading the same bundle.
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def _blocks(s):
    n = s["n"]
    K = sp.csr_matrix((s["K_data"], s["K_indices"], s["K_indptr"]), shape=(n, n))
    f = np.asarray(s["f"]).reshape(-1, n).T
    return n, K, f


def saddle_solve(bundle):
    """Direct solve of Eq. (5); returns (u list, lambda, p)."""
    nl, ng = int(bundle["n_lambda"]), int(bundle["n_primal"])
    rows_K, rows_Bt = [], []
    offs = [0]
    info = []
    for s in bundle["subs"]:
        n, K, f = _blocks(s)
        mask = np.ones(n, bool)
        mask[np.asarray(s["tree"], np.int64)] = False
        mask[np.asarray(s["prim"], np.int64)] = False
        r = np.flatnonzero(mask)
        info.append((n, K, f, r))
        offs.append(offs[-1] + len(r))
    nr = offs[-1]
    N = nr + ng + nl
    I, J, V = [], [], []
    rhs = np.zeros((N, int(bundle["nrhs"])))

    def add(M, ro, co):
        M = sp.coo_matrix(M)
        I.append(M.row + ro)
        J.append(M.col + co)
        V.append(M.data)

    for k, (s, (n, K, f, r)) in enumerate(zip(bundle["subs"], info)):
        prim = np.asarray(s["prim"], np.int64)
        gid = np.asarray(s["prim_gid"], np.int64)
        Cp = sp.csr_matrix((np.ones(len(prim)), (np.arange(len(prim)), gid)), shape=(len(prim), ng))
        Krr = K[r][:, r]
        Krp = K[r][:, prim]
        Kpp = K[prim][:, prim]
        pos = -np.ones(n, np.int64)
        pos[r] = np.arange(len(r))
        Br = sp.csr_matrix((np.asarray(s["B_sign"], np.float64),
                            (np.asarray(s["B_lambda"], np.int64), pos[np.asarray(s["B_dof"], np.int64)])),
                           shape=(nl, len(r)))
        o = offs[k]
        add(Krr, o, o)
        if ng:
            add(Krp @ Cp, o, nr)
            add((Krp @ Cp).T, nr, o)
            add(Cp.T @ Kpp @ Cp, nr, nr)
        add(Br.T, o, nr + ng)
        add(Br, nr + ng, o)
        rhs[o:o + len(r)] = f[r]
        if ng:
            rhs[nr:nr + ng] += Cp.T @ f[prim]
    A = sp.csc_matrix((np.concatenate(V), (np.concatenate(I), np.concatenate(J))), shape=(N, N))
    x = spla.splu(A).solve(rhs)
    lam = x[nr + ng:]
    p = x[nr:nr + ng]
    us = []
    for k, (s, (n, K, f, r)) in enumerate(zip(bundle["subs"], info)):
        u = np.zeros((n, rhs.shape[1]))
        u[r] = x[offs[k]:offs[k + 1]]
        prim = np.asarray(s["prim"], np.int64)
        u[prim] = p[np.asarray(s["prim_gid"], np.int64)]
        us.append(u)
    return us, lam, p


def monolithic_solve(bundle):
    """Gauged global solve; returns (u list per subdomain, a_g)."""
    ngl = int(bundle["n_gauged"])
    I, J, V = [], [], []
    rhs = np.zeros((ngl, int(bundle["nrhs"])))
    for s in bundle["subs"]:
        n, K, f = _blocks(s)
        glob = np.asarray(s["glob"], np.int64)
        Kc = K.tocoo()
        keep = (glob[Kc.row] >= 0) & (glob[Kc.col] >= 0)
        I.append(glob[Kc.row[keep]])
        J.append(glob[Kc.col[keep]])
        V.append(Kc.data[keep])
        m = glob >= 0
        np.add.at(rhs, glob[m], f[m])
    Kg = sp.csc_matrix((np.concatenate(V), (np.concatenate(I), np.concatenate(J))), shape=(ngl, ngl))
    a = spla.splu(Kg).solve(rhs)
    us = []
    for s in bundle["subs"]:
        glob = np.asarray(s["glob"], np.int64)
        u = np.zeros((s["n"], rhs.shape[1]))
        m = glob >= 0
        u[m] = a[glob[m]]
        us.append(u)
    return us, a, Kg, rhs
