"""Discretisation and tree–cotree gauge of one workload: produces the inputs of
the IETI-DP solve phase (the C-ABI's arguments, include/ietidp.h).

This is the problem generator, not the solve phase: torn per-subdomain stiffness
K^(k) and loads j^(k), the global control graph with the
five edge weights of Fig. 2, Kruskal's tree, the primal
selection, the multiplier pairing B.
Nothing here factorises, solves or iterates.

For the device pre-processing (include/ietidp_pre.h) the assembly and the
Kruskal tree of this module are the CPU reference the kernels are compared with
(tests/test_gpu_pre.py): plain SciPy, written from the paper, sharing no code with csrc/pre.cu
and pinned on their own (tests/test_gen.py, tests/test_oracle.py: curl o grad = 0, the DOF counts,
EOC of the manufactured solutions, DD = monolithic). The inputs of those kernels come from
ietigen/predesc.py, which holds no assembly arithmetic.

Index conventions:
* vertices (0-form DOFs) on the global grid m_x x m_y x m_z, x fastest;
* edge (1-form DOF) of direction a at (i,j,k) joins vertex (i,j,k) to (i,j,k)+e_a;
  global edge id = offset[a] + flat(i,j,k) over that direction's edge grid;
* subdomain ids run over the tiling with x fastest; a multiplier is +1 on the
  lower subdomain id.
"""
import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import minimum_spanning_tree, connected_components

from . import configs as cf
from .splines import Space1D, gradient_incidence


def _kron3(Az, Ay, Ax):
    return sp.kron(Az, sp.kron(Ay, Ax, format="csr"), format="csr")


class Grid:
    """Global index space of the glued multipatch control grid."""

    def __init__(self, npatch, s, periodic):
        self.npatch = np.array(npatch)
        self.s = s
        self.periodic = periodic
        self.m = np.array([n * s + (0 if per else 1) for n, per in zip(npatch, periodic)])
        self.nv = int(np.prod(self.m))
        self.eshape = []
        for a in range(3):
            sh = self.m.copy()
            if not periodic[a]:
                sh[a] -= 1
            self.eshape.append(tuple(int(v) for v in sh))
        sizes = [int(np.prod(sh)) for sh in self.eshape]
        self.eoff = np.concatenate([[0], np.cumsum(sizes)])
        self.ne = int(self.eoff[-1])

    def vid(self, i, j, k):
        m = self.m
        return i + m[0] * (j + m[1] * k)

    def eid(self, a, i, j, k):
        sh = self.eshape[a]
        return self.eoff[a] + i + sh[0] * (j + sh[1] * k)

    def edge_coords(self, a):
        sh = self.eshape[a]
        k, j, i = np.meshgrid(np.arange(sh[2]), np.arange(sh[1]), np.arange(sh[0]), indexing="ij")
        return i.ravel(), j.ravel(), k.ravel()

    def endpoints(self):
        u = np.empty(self.ne, np.int64)
        v = np.empty(self.ne, np.int64)
        for a in range(3):
            i, j, k = self.edge_coords(a)
            c = [i, j, k]
            c2 = [i.copy(), j.copy(), k.copy()]
            c2[a] = (c2[a] + 1) % self.m[a]
            sl = slice(self.eoff[a], self.eoff[a + 1])
            u[sl] = self.vid(*c)
            v[sl] = self.vid(*c2)
        return u, v

    def dirichlet_edges(self):
        """Edge has a non-zero tangential trace on the outer boundary: some other
        axis b (non-periodic) has its coordinate at 0 or m_b - 1."""
        d = np.zeros(self.ne, bool)
        for a in range(3):
            coords = self.edge_coords(a)
            sl = slice(self.eoff[a], self.eoff[a + 1])
            for b in range(3):
                if b == a or self.periodic[b]:
                    continue
                d[sl] |= (coords[b] == 0) | (coords[b] == self.m[b] - 1)
        return d

    def dirichlet_vertices(self):
        k, j, i = np.meshgrid(*[np.arange(self.m[a]) for a in (2, 1, 0)], indexing="ij")
        c = [i.ravel(), j.ravel(), k.ravel()]
        d = np.zeros(self.nv, bool)
        for b in range(3):
            if not self.periodic[b]:
                d |= (c[b] == 0) | (c[b] == self.m[b] - 1)
        return d

    def block_edges(self, lo, hi):
        """Global ids of every edge of the local grid of patch block [lo, hi),
        in local order (direction, then x-fastest local flat index)."""
        s = self.s
        ml = [(hi[a] - lo[a]) * s + 1 for a in range(3)]
        out = []
        for a in range(3):
            sh = list(ml)
            sh[a] -= 1
            k, j, i = np.meshgrid(np.arange(sh[2]), np.arange(sh[1]), np.arange(sh[0]), indexing="ij")
            c = [i.ravel() + lo[0] * s, j.ravel() + lo[1] * s, k.ravel() + lo[2] * s]
            for b in range(3):
                c[b] = c[b] % self.m[b]
            out.append(self.eid(a, *c))
        return np.concatenate(out), ml


class Subdomain:
    """A box of patches [lo, hi), or (explicit partitions) a union of unit patch boxes."""

    def __init__(self, idx, lo, hi, boxes=None):
        self.idx, self.lo, self.hi = idx, tuple(lo), tuple(hi)
        self.boxes = boxes if boxes is not None else [(self.lo, self.hi)]


def tiling_subdomains(cfg):
    """Boxes of patches: T[a] parts along axis a, cut at floor(i N[a] / T[a]) (equal
    blocks when T[a] divides N[a]; otherwise sizes differ by one, e.g. 3 patches in 2
    parts -> 1 + 2, for the paper's N_sub in {2..12} on 27 patches).
    With cfg.parts (a part id per patch, x fastest) every subdomain is the union of its
    patches (subdomains are unions of patches, e.g. METIS partitions)."""
    N, T = cfg.npatch, cfg.tiling
    if cfg.parts is not None:
        parts = np.asarray(cfg.parts).reshape(N[2], N[1], N[0])
        subs = []
        for q in range(int(parts.max()) + 1):
            kk, jj, ii = np.nonzero(parts == q)
            boxes = [((int(i), int(j), int(k)), (int(i) + 1, int(j) + 1, int(k) + 1)) for i, j, k in zip(ii, jj, kk)]
            lo = (int(ii.min()), int(jj.min()), int(kk.min()))
            hi = (int(ii.max()) + 1, int(jj.max()) + 1, int(kk.max()) + 1)
            subs.append(Subdomain(q, lo, hi, boxes))
        return subs
    assert all(1 <= T[a] <= N[a] for a in range(3))
    cuts = [[(i * N[a]) // T[a] for i in range(T[a] + 1)] for a in range(3)]
    subs = []
    for tz in range(T[2]):
        for ty in range(T[1]):
            for tx in range(T[0]):
                lo = (cuts[0][tx], cuts[1][ty], cuts[2][tz])
                hi = (cuts[0][tx + 1], cuts[1][ty + 1], cuts[2][tz + 1])
                subs.append(Subdomain(len(subs), lo, hi))
    return subs


# --------------------------------------------------------------------------
# Assembly: K = C^T M2(nu) C (de Rham factorisation)
# --------------------------------------------------------------------------

def local_curl(ml):
    """Face-edge incidence C (curl on coefficient vectors) of a box grid with
    ml vertices per axis; faces ordered (x-faces BDD, y-faces DBD, z-faces DDB),
    edges ordered (x DBB, y BDB, z BBD), each x-fastest."""
    G = [gradient_incidence(m) for m in ml]
    IB = [sp.identity(m, format="csr") for m in ml]
    ID = [sp.identity(m - 1, format="csr") for m in ml]
    Cx_y = -_kron3(G[2], ID[1], IB[0])
    Cx_z = _kron3(ID[2], G[1], IB[0])
    Cy_x = _kron3(G[2], IB[1], ID[0])
    Cy_z = -_kron3(ID[2], IB[1], G[0])
    Cz_x = -_kron3(IB[2], G[1], ID[0])
    Cz_y = _kron3(IB[2], ID[1], G[0])
    return sp.bmat([[None, Cx_y, Cx_z], [Cy_x, None, Cy_z], [Cz_x, Cz_y, None]], format="csr")


def local_grad(ml):
    """Vertex-edge incidence (discrete gradient) of a box grid."""
    G = [gradient_incidence(m) for m in ml]
    IB = [sp.identity(m, format="csr") for m in ml]
    return sp.vstack([_kron3(IB[2], IB[1], G[0]), _kron3(IB[2], G[1], IB[0]),
                      _kron3(G[2], IB[1], IB[0])], format="csr")


def cube_spaces(cfg, sub):
    N = cfg.npatch
    return [Space1D(sub.lo[a] / N[a], sub.hi[a] / N[a], sub.hi[a] - sub.lo[a], cfg.e, cfg.p)
            for a in range(3)]


def cube_mass2(cfg, sub, spaces, nu):
    """2-form mass matrix of the subdomain, sum over its patches of
    nu_patch * kron of 1-D Gram matrices (exact Gauss, p+1 points)."""
    MB = [[spaces[a].mass("B", q) for q in range(spaces[a].npatch)] for a in range(3)]
    MD = [[spaces[a].mass("D", q) for q in range(spaces[a].npatch)] for a in range(3)]
    blocks = [None, None, None]
    for c in range(3):
        acc = None
        for qz in range(spaces[2].npatch):
            for qy in range(spaces[1].npatch):
                for qx in range(spaces[0].npatch):
                    w = nu[sub.lo[0] + qx, sub.lo[1] + qy, sub.lo[2] + qz]
                    mx = MB[0][qx] if c == 0 else MD[0][qx]
                    my = MB[1][qy] if c == 1 else MD[1][qy]
                    mz = MB[2][qz] if c == 2 else MD[2][qz]
                    term = w * _kron3(sp.csr_matrix(mz), sp.csr_matrix(my), sp.csr_matrix(mx))
                    acc = term if acc is None else acc + term
        blocks[c] = acc
    return sp.block_diag(blocks, format="csr")


def cube_face_loads(cfg, sub, spaces):
    """t_f = int_{Omega^(k)} T . v_f for every 2-form basis function (weak-curl
    load); returns (n_faces, nrhs)."""
    terms = cf.source_terms(cfg)
    nq = cfg.p + cfg.load_nq_extra
    cache = {}

    def vec(a, kind, spec):
        if (a, kind, spec) not in cache:
            cache[(a, kind, spec)] = spaces[a].integrals(kind, cf.f1d(spec), nq)
        return cache[(a, kind, spec)]

    cols = []
    for col in terms:
        parts = []
        for c in range(3):
            kinds = ["D", "D", "D"]
            kinds[c] = "B"
            dims = [spaces[a].m - (0 if kinds[a] == "B" else 1) for a in range(3)]
            if not col[c]:
                parts.append(np.zeros(int(np.prod(dims))))
                continue
            # sum_terms coef * kron(vz, vy, vx) as one contraction over the
            # distinct 1-D factors of each axis
            uniq = [sorted({t[1 + a] for t in col[c]}) for a in range(3)]
            V = [np.stack([vec(a, kinds[a], sp_) for sp_ in uniq[a]])
                 for a in range(3)]
            A = np.zeros([len(u) for u in uniq])
            for coef, fx, fy, fz in col[c]:
                A[uniq[0].index(fx), uniq[1].index(fy), uniq[2].index(fz)] += coef
            t = np.einsum("abc,ai,bj,ck->kji", A, V[0], V[1], V[2], optimize=True)
            parts.append(t.ravel())
        cols.append(np.concatenate(parts))
    return np.stack(cols, axis=1)


# --------------------------------------------------------------------------
# The problem
# --------------------------------------------------------------------------

class Problem:
    """Everything the C-ABI consumes for one workload, plus generator-side
    bookkeeping used by the tests (global ids, weights, tree)."""

    def __init__(self, cfg, kruskal="scipy"):
        self.cfg = cfg
        s = cfg.e + cfg.p - 1
        self.grid = Grid(cfg.npatch, s, cfg.periodic)
        self.subs = tiling_subdomains(cfg)
        self.nu = cf.patch_nu(cfg)
        self._classify()
        self._gauge(kruskal)
        self._split()

    # ---- graph classification (Fig. 2) --------------------
    def _classify(self):
        g = self.grid
        ne = g.ne
        self.dir_edge = g.dirichlet_edges()
        self.sub_edges = []
        count = np.zeros(ne, np.int32)
        smin = np.full(ne, 1 << 30, np.int64)
        smax = np.full(ne, -1, np.int64)
        for sd in self.subs:
            if len(sd.boxes) == 1:
                gids, ml = g.block_edges(sd.lo, sd.hi)
                sd.ml = ml
            else:  # union of patch boxes: the distinct global edges, in increasing order
                gids = np.unique(np.concatenate([g.block_edges(lo, hi)[0] for lo, hi in sd.boxes]))
                sd.ml = None
            assert len(np.unique(gids)) == len(gids)
            self.sub_edges.append(gids)
            np.add.at(count, gids, 1)
            np.minimum.at(smin, gids, sd.idx)
            np.maximum.at(smax, gids, sd.idx)
        self.membership, self.smin, self.smax = count, smin, smax

        # facets: one per face-adjacent subdomain pair (interface) and one per
        # boundary patch-facet (Dirichlet). Count, for every edge,
        # the facets whose closure contains it.
        nfacet = np.zeros(ne, np.int32)
        sets = [np.sort(e) for e in self.sub_edges]
        T = self.cfg.tiling
        per = self.cfg.periodic
        pos = {}
        self.iface_pairs = []
        if self.cfg.parts is not None:
            # explicit partitions: an interface per pair of parts with face-adjacent patches
            # (one facet each), its closure = the edges the two share
            N = self.cfg.npatch
            parts = np.asarray(self.cfg.parts).reshape(N[2], N[1], N[0])
            for pz in range(N[2]):
                for py in range(N[1]):
                    for px in range(N[0]):
                        for a in range(3):
                            q = [px, py, pz]
                            q[a] += 1
                            if q[a] >= N[a]:
                                continue
                            k, l = int(parts[pz, py, px]), int(parts[q[2], q[1], q[0]])
                            if k != l and (min(k, l), max(k, l)) not in self.iface_pairs:
                                self.iface_pairs.append((min(k, l), max(k, l)))
            for k, l in self.iface_pairs:
                shared = np.intersect1d(sets[k], sets[l], assume_unique=True)
                nfacet[shared] += 1
        for sd in self.subs if self.cfg.parts is None else []:
            t = (sd.idx % T[0], (sd.idx // T[0]) % T[1], sd.idx // (T[0] * T[1]))
            pos[t] = sd.idx
        for t, k in pos.items():
            for a in range(3):
                t2 = list(t)
                t2[a] += 1
                if per[a]:
                    t2[a] %= T[a]
                t2 = tuple(t2)
                if t2 in pos and pos[t2] != k:
                    l = pos[t2]
                    pair = (min(k, l), max(k, l))
                    if pair in self.iface_pairs:
                        continue
                    self.iface_pairs.append(pair)
                    shared = np.intersect1d(sets[k], sets[l], assume_unique=True)
                    nfacet[shared] += 1
        # Dirichlet patch-facets
        N = self.cfg.npatch
        for pz in range(N[2]):
            for py in range(N[1]):
                for px in range(N[0]):
                    pidx = (px, py, pz)
                    for a in range(3):
                        if per[a]:
                            continue
                        for side in (0, 1):
                            if (side == 0 and pidx[a] != 0) or (side == 1 and pidx[a] != N[a] - 1):
                                continue
                            nfacet[self._patch_face_edges(pidx, a, side)] += 1
        self.nfacet = nfacet
        wire = nfacet >= 2
        w = np.full(ne, 5, np.int8)
        on_iface = count >= 2
        w[(self.dir_edge | on_iface) & (w == 5)] = 4
        w[wire] = 3
        w[(count >= 3)] = 2
        w[self.dir_edge & on_iface] = 1
        self.weight = w

    def _patch_face_edges(self, pidx, a, side):
        """Edges in the closure of face `side` (0: low, 1: high) normal to axis a
        of patch pidx, tangential to it."""
        g, s = self.grid, self.grid.s
        lo = [pidx[b] * s for b in range(3)]
        out = []
        for d in range(3):
            if d == a:
                continue
            sh = [s + 1, s + 1, s + 1]
            sh[d] = s
            sh[a] = 1
            k, j, i = np.meshgrid(np.arange(sh[2]), np.arange(sh[1]), np.arange(sh[0]), indexing="ij")
            c = [i.ravel() + lo[0], j.ravel() + lo[1], k.ravel() + lo[2]]
            c[a] = np.full_like(c[a], lo[a] + side * s)
            for b in range(3):
                c[b] = c[b] % g.m[b]
            out.append(g.eid(d, *c))
        return np.concatenate(out)

    # ---- Kruskal and primal selection -------
    def _gauge(self, kruskal):
        g = self.grid
        u, v = g.endpoints()
        self.eu, self.ev = u, v
        order = np.lexsort((np.arange(g.ne), self.weight))
        if kruskal == "python":
            in_tree = kruskal_unionfind(g.nv, u, v, order)
        else:
            # Distinct keys weight*ne + id make the minimum spanning tree unique,
            # hence equal to Kruskal's tree under this order.
            key = self.weight.astype(np.float64) * g.ne + np.arange(g.ne) + 1.0
            A = sp.csr_matrix((key, (u, v)), shape=(g.nv, g.nv))
            T = minimum_spanning_tree(A).tocoo()
            lut = {}
            in_tree = np.zeros(g.ne, bool)
            eid = np.rint(T.data - 1.0).astype(np.int64) % g.ne
            in_tree[eid] = True
        self.tree = in_tree
        self.primal_edges = np.flatnonzero((~in_tree) & (self.weight == 2))
        self.primal_id = np.full(g.ne, -1, np.int64)
        self.primal_id[self.primal_edges] = np.arange(len(self.primal_edges))

    # ---- per-subdomain DOF classes, B, C_p ---------------------------------
    def _split(self):
        g = self.grid
        keep = ~self.dir_edge
        rem = keep & ~self.tree & (self.primal_id < 0)
        shared = rem & (self.membership >= 2)
        assert np.all(self.membership[shared] == 2), "remaining DOF in >2 subdomains"
        self.lambda_edges = np.flatnonzero(shared)
        self.lambda_id = np.full(g.ne, -1, np.int64)
        self.lambda_id[self.lambda_edges] = np.arange(len(self.lambda_edges))
        unk = keep & ~self.tree
        self.gauged_edges = np.flatnonzero(unk)
        self.gauged_id = np.full(g.ne, -1, np.int64)
        self.gauged_id[self.gauged_edges] = np.arange(len(self.gauged_edges))
        for sd in self.subs:
            gids = self.sub_edges[sd.idx]
            lk = keep[gids]
            sd.local_mask = lk            # which local-grid edges are DOFs
            sd.gid = gids[lk]             # DOF -> global edge id
            n = len(sd.gid)
            sd.n = n
            sd.tree = np.flatnonzero(self.tree[sd.gid]).astype(np.int32)
            pm = self.primal_id[sd.gid] >= 0
            sd.prim = np.flatnonzero(pm).astype(np.int32)
            sd.prim_gid = self.primal_id[sd.gid[pm]].astype(np.int32)
            lm = self.lambda_id[sd.gid] >= 0
            sd.B_dof = np.flatnonzero(lm).astype(np.int32)
            sd.B_lambda = self.lambda_id[sd.gid[lm]].astype(np.int32)
            sd.B_sign = np.where(self.smin[sd.gid[lm]] == sd.idx, 1, -1).astype(np.int8)
            sd.glob = self.gauged_id[sd.gid].astype(np.int64)
        self.n_lambda = len(self.lambda_edges)
        self.n_primal = len(self.primal_edges)

    # ---- assembly (torn, per subdomain) -----------------------------------
    def assemble(self, sd, with_face=False):
        """K^(k) (CSR, Dirichlet rows/cols removed) and j^(k) (n_k x nrhs)."""
        if self.cfg.geometry != "cube":
            from .cylinder import assemble_cylinder
            return assemble_cylinder(self, sd, with_face)
        if len(sd.boxes) > 1:
            # union of patch boxes: every box's K and loads in its own numbering, summed
            # into the subdomain's (global edge ids in increasing order): the integrals
            # over the union (torn assembly)
            assert not with_face
            gid_all = self.sub_edges[sd.idx]
            n_all = len(gid_all)
            K = None
            j = np.zeros((n_all, self.cfg.nrhs))
            for lo, hi in sd.boxes:
                bx = Subdomain(sd.idx, lo, hi)
                gb, mlb = self.grid.block_edges(lo, hi)
                spaces = cube_spaces(self.cfg, bx)
                C = local_curl(mlb)
                Kb = (C.T @ cube_mass2(self.cfg, bx, spaces, self.nu) @ C).tocoo()
                loc = np.searchsorted(gid_all, gb)
                Kb = sp.csr_matrix((Kb.data, (loc[Kb.row], loc[Kb.col])), shape=(n_all, n_all))
                K = Kb if K is None else K + Kb
                np.add.at(j, loc, C.T @ cube_face_loads(self.cfg, bx, spaces))
            m = sd.local_mask
            j = self._lift(sd, K, j)
            K = K[m][:, m].tocsr()
            K = ((K + K.T) * 0.5).tocsr()
            K.sort_indices()
            return K, np.ascontiguousarray(j[m])
        spaces = cube_spaces(self.cfg, sd)
        C = local_curl(sd.ml)
        M2 = cube_mass2(self.cfg, sd, spaces, self.nu)
        K = (C.T @ M2 @ C).tocsr()
        t = cube_face_loads(self.cfg, sd, spaces)
        j = C.T @ t
        m = sd.local_mask
        j = self._lift(sd, K, j)
        K = K[m][:, m].tocsr()
        # C^T M2 C in floating point is symmetric only up to rounding, and SpGEMM
        # drops an entry that cancels to exactly 0.0 on one side only: store the
        # exactly symmetric part on the union pattern (the C-ABI requires a
        # symmetric CSR pattern, include/ietidp.h).
        K = ((K + K.T) * 0.5).tocsr()
        K.sort_indices()
        j = np.ascontiguousarray(j[m])
        if with_face:
            return K, j, C[:, m], M2, t
        return K, j

    # ---- inhomogeneous boundary values (n x A = n x A_ana) ----
    def dirichlet_values(self):
        """Global edge vector: the coefficients of the boundary (Dirichlet) edges of the
        spline interpolant of A_ana, zero elsewhere. Every component of A_ana is a product
        coef * fx(x) fy(y) fz(z), so its tensor-product projection is the Kronecker product
        of three 1-D projections: L2 along the component's own axis (D-splines), L2 with
        the two end coefficients fixed to the exact end values across it (B-splines; open
        knots make them interpolatory there), which makes the tangential trace on each
        boundary face exact in the normal direction and a face-wise projection within it."""
        if getattr(self, "_aD", None) is not None:
            return self._aD
        cfg, g = self.cfg, self.grid
        assert cfg.geometry == "cube" and cfg.rhs == "aana"
        from .splines import Space1D
        nq = cfg.p + cfg.load_nq_extra
        sp1 = [Space1D(0.0, 1.0, cfg.npatch[a], cfg.e, cfg.p) for a in range(3)]

        def proj(a, kind, f):
            S = sp1[a]
            M = sum(S.mass(kind, q, nq) for q in range(S.npatch))
            v = S.integrals(kind, f, nq)
            if kind == "D":
                return np.linalg.solve(M, v)
            c = np.zeros(S.m)
            c[0], c[-1] = f(np.array([0.0]))[0], f(np.array([1.0]))[0]
            I = np.arange(1, S.m - 1)
            c[I] = np.linalg.solve(M[np.ix_(I, I)], v[I] - M[np.ix_(I, [0, S.m - 1])] @ c[[0, -1]])
            return c
        a_all = np.zeros(g.ne)
        for d in range(3):
            coef, *specs = cf.A_ANA[d]
            c1 = [proj(a, "D" if a == d else "B", cf.f1d(specs[a])) for a in range(3)]
            a_all[g.eoff[d]:g.eoff[d + 1]] = coef * np.einsum("i,j,k->kji", c1[0], c1[1], c1[2]).ravel()
        self._a_interp = a_all
        self._aD = np.where(self.dir_edge, a_all, 0.0)
        return self._aD

    def _lift(self, sd, K_full, j_full):
        """j <- j - K[:, Dirichlet] a_D on the subdomain's full (unmasked) edge set."""
        if self.cfg.rhs != "aana":
            return j_full
        aD = self.dirichlet_values()[self.sub_edges[sd.idx]]
        return j_full - (K_full @ aD)[:, None]

    def flux_error(self, us, bnorm2):
        """eps_B of the subdomain solutions us: ||B_h - B||^2 =
        sum over the patches of b^T M2 b - 2 b^T t + ||B||^2, b = C a on the patch, a the
        global edge vector (subdomain solutions + boundary values), t_f = int B . v_f."""
        g, cfg = self.grid, self.cfg
        a = self.dirichlet_values().copy() if cfg.rhs == "aana" else np.zeros(g.ne)
        for sd, u in zip(self.subs, us):
            a[sd.gid] = u[:, 0]
        N = cfg.npatch
        tot = 0.0
        for pz in range(N[2]):
            for py in range(N[1]):
                for px in range(N[0]):
                    bx = Subdomain(0, (px, py, pz), (px + 1, py + 1, pz + 1))
                    gb, ml = g.block_edges(bx.lo, bx.hi)
                    spaces = cube_spaces(cfg, bx)
                    bf = local_curl(ml) @ a[gb]
                    M2 = cube_mass2(cfg, bx, spaces, self.nu)
                    t = cube_face_loads(cfg, bx, spaces)[:, 0]
                    tot += bf @ (M2 @ bf) - 2.0 * bf @ t
        return float(np.sqrt(max(tot + bnorm2, 0.0)))

    def counts(self):
        g = self.grid
        dv = g.dirichlet_vertices()
        E_int = int((~self.dir_edge).sum())
        V_int = int((~dv).sum())
        n_r = [sd.n - len(sd.tree) - len(sd.prim) for sd in self.subs]
        return dict(E_int=E_int, V_int=V_int, n_gp=self.n_primal, m_r=self.n_lambda,
                    sum_nr=int(sum(n_r)), max_nr=int(max(n_r)),
                    sum_nk=int(sum(sd.n for sd in self.subs)),
                    w_counts=[int((self.weight == w).sum()) for w in range(1, 6)])


def kruskal_unionfind(nv, u, v, order):
    """Kruskal's algorithm: scan edges in `order`, keep an edge
    iff it joins two different union-find components."""
    parent = list(range(nv))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    in_tree = np.zeros(len(u), bool)
    uu, vv = u.tolist(), v.tolist()
    for e in order.tolist():
        a, b = find(uu[e]), find(vv[e])
        if a != b:
            parent[a] = b
            in_tree[e] = True
    return in_tree


def build(cfg, kruskal="scipy"):
    if isinstance(cfg, str):
        cfg = cf.get(cfg)
    return Problem(cfg, kruskal=kruskal)
