"""Device pre-processing (include/ietidp_pre.h) against the generator's
plain NumPy/SciPy assembly and gauge (ietigen/problem.py, pinned in tests/test_gen.py and
tests/test_oracle.py by curl o grad = 0, the DOF counts, EOC of the manufactured solutions and
DD = monolithic), which is the reference side here: it shares no code with csrc/pre.cu.

PAPER.md:49-57 (K = C^T M_2 C per subdomain, torn), :83, :150-178 (tree-cotree gauge on the
weighted control graph, primal DOFs).

Tolerances: every K entry is a signed sum of at most 8 x 8 products of three Gram entries, each
a Gauss sum of a few dozen terms; the two sides differ only in summation order, so entries
agree to a few ulp of the largest entry: 1e-12 relative to max|K| with
two orders of margin. Integer results (pattern after dropping exact zeros, tree, primal
set) are compared bit for bit.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from ietigen import predesc
from ietigen.problem import build

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2501_04340_b200 import ietidp
    return ietidp


def _csr(out, n):
    return sp.csr_matrix((out["K_data"], out["K_indices"], out["K_indptr"]), shape=(n, n))


def _subs(P, limit):
    n = len(P.subs)
    if n <= limit:
        return list(range(n))
    return sorted(set(np.linspace(0, n - 1, limit).astype(int).tolist()))


@pytest.mark.parametrize("name", ["C1", "C2r", "C3r", "C4r", "C5r", "E27_221_p3_e2", "E27_311_p1_e3"])
def test_assembly_matches_generator(lib, name):
    P = build(name)
    for k in _subs(P, 6):
        sd = P.subs[k]
        Kref, jref = P.assemble(sd)
        out = lib.pre_assemble(predesc.subdomain_desc(P, sd))
        K = _csr(out, sd.n)
        # CSR invariants of the C ABI (ietidp_set_subdomain): sorted columns, symmetric pattern
        for r in range(0, sd.n, max(1, sd.n // 50)):
            c = out["K_indices"][out["K_indptr"][r]:out["K_indptr"][r + 1]]
            assert np.all(np.diff(c) > 0)
        assert (abs(K - K.T)).max() == 0.0, "exactly symmetric by construction"
        scale = abs(Kref).max()
        assert abs(K - Kref).max() <= 1e-12 * scale, (name, k, abs(K - Kref).max() / scale)
        # structural pattern: a superset of the generator's; the extra entries are exact cancellations
        Kz = K.copy()
        Kz.data[abs(Kz.data) <= 1e-13 * scale] = 0.0
        Kz.eliminate_zeros()
        Rz = Kref.copy()
        Rz.data[abs(Rz.data) <= 1e-13 * scale] = 0.0
        Rz.eliminate_zeros()
        assert (Kz != 0).astype(np.int8).nnz == (Rz != 0).astype(np.int8).nnz
        assert ((Kz != 0) != (Rz != 0)).nnz == 0
        js = abs(jref).max()
        assert abs(out["f"].T - jref).max() <= 1e-12 * max(js, 1e-300), (name, k)


@pytest.mark.parametrize("name", ["C3r", "C4r", "C5r"])
def test_batch_assembly_bitwise_equals_single(lib, name):
    """ietidp_pre_assemble_batch (one launch per stage over all subdomains, the configuration
    bench.py times) gives bit for bit the per-subdomain results, on every subdomain."""
    P = build(name)
    descs = [predesc.subdomain_desc(P, sd) for sd in P.subs]
    outs, info = lib.pre_assemble_batch(descs)
    assert info["nnz"] == sum(len(o["K_data"]) for o in outs)
    for k in _subs(P, 12):
        one = lib.pre_assemble(descs[k])
        for key in ("K_indptr", "K_indices", "K_data", "f"):
            assert np.array_equal(one[key], outs[k][key]), (name, k, key)
    # and against the generator on a subdomain the single-call test does not sample
    k = len(P.subs) // 2 + 1
    Kref, jref = P.assemble(P.subs[k])
    K = _csr(outs[k], P.subs[k].n)
    assert abs(K - Kref).max() <= 1e-12 * abs(Kref).max()
    assert abs(outs[k]["f"].T - jref).max() <= 1e-12 * abs(jref).max()


@pytest.mark.parametrize("name", ["C2r", "C5r", "E27_221_p3_e2"])
def test_assembly_closed_form_energy_and_kernel(lib, name):
    """Pins of the device-assembled K and j that do not involve the generator's assembly
    (PAPER.md:49-57). With no Dirichlet rows removed:
    (1) the field A = (-y/2, x/2, 0) lies in the spline 1-form space (constant along an edge's
        own axis: coefficient (t_{j+p+1}-t_{j+1})/p of the Curry-Schoenberg D_j; linear across:
        the Greville abscissae), curl A = e_z, so a^T K a = int nu |curl A|^2 = sum over the
        patches of nu_q * volume_q -- exactly, for any degree and any per-patch nu;
    (2) K annihilates discrete gradients (curl o grad = 0): K G phi = 0 for a seeded phi;
    (3) the load of a constant T = tau e_z pairs with the same field: a^T j = tau * volume."""
    from ietigen.rng import SplitMix64
    P = build(name)
    sd = P.subs[len(P.subs) // 2]
    d = dict(predesc.subdomain_desc(P, sd))
    p, e, npb = d["p"], d["e"], d["npatch"]
    m = [npb[a] * (e + p - 1) + 1 for a in range(3)]
    E = [[m[a] - (1 if a == dd else 0) for a in range(3)] for dd in range(3)]
    ne = sum(int(np.prod(E[dd])) for dd in range(3))
    d["dof_of_edge"] = np.arange(ne, dtype=np.int32)  # keep the Dirichlet edges
    d["n_dof"] = ne
    # one load column: T = tau e_z (component 2: B along z, D along x and y), factors "one"
    tau = 0.75
    lw = []
    for a in range(3):
        x = d["lx"][a]
        h_el = (d["knots"][a][-1] - d["knots"][a][0]) / (npb[a] * e)
        g, w = np.polynomial.legendre.leggauss(d["lq"])
        lw.append(np.tile(0.5 * h_el * w, npb[a] * e))
        assert len(lw[-1]) == len(x)
    d.update(nrhs=1, fac_kind=[np.array([1], np.int32), np.array([1], np.int32), np.array([0], np.int32)],
             fac_val=[lw[0][None, :], lw[1][None, :], lw[2][None, :]], term_col=np.array([0], np.int32),
             term_comp=np.array([2], np.int32), term_fac=np.array([[0, 0, 0]], np.int32), term_coef=np.array([tau]))
    out = lib.pre_assemble(d)
    K = _csr(out, ne)
    t = d["knots"]
    cD = [np.array([(t[a][j + p + 1] - t[a][j + 1]) / p for j in range(m[a] - 1)]) for a in range(3)]
    gv = [np.array([t[a][i + 1:i + p + 1].sum() / p for i in range(m[a])]) for a in range(3)]
    one = [np.ones(m[a]) for a in range(3)]
    ax = np.einsum("i,j,k->kji", cD[0], -0.5 * gv[1], one[2]).ravel()   # A_x = -y/2 on the x-edges
    ay = np.einsum("i,j,k->kji", 0.5 * gv[0], cD[1], one[2]).ravel()    # A_y = x/2 on the y-edges
    a = np.concatenate([ax, ay, np.zeros(int(np.prod(E[2])))])
    vol_patch = np.prod([(t[a][-1] - t[a][0]) / npb[a] for a in range(3)])
    energy = float(np.sum(d["nu"]) * vol_patch)
    assert abs(a @ (K @ a) - energy) <= 1e-12 * energy, (a @ (K @ a), energy)
    assert abs(a @ out["f"][0] - tau * vol_patch * np.prod(npb)) <= 1e-12 * tau
    # discrete gradient of a seeded vertex function: edge (d; n) = phi(n + e_d) - phi(n)
    g = SplitMix64(5)
    phi = np.array([g.uniform() for _ in range(int(np.prod(m)))]).reshape(m[2], m[1], m[0])
    grad = np.concatenate([np.diff(phi, axis=2).ravel(), np.diff(phi, axis=1).ravel(), np.diff(phi, axis=0).ravel()])
    assert np.abs(K @ grad).max() <= 1e-12 * abs(K).max() * np.abs(grad).max()
    lam_min = np.linalg.eigvalsh(K.toarray())[0] if ne <= 1500 else 0.0
    assert lam_min >= -1e-10 * abs(K).max()


def test_gram_blocks_closed_form(lib):
    """First stage pinned independently of the generator: on one patch with p = 1, e = 2 over
    [0, 1/2] the hat functions' Gram matrix is h/6 [[2,1,0],[1,4,1],[0,1,2]] (h = 1/4) and the
    Curry-Schoenberg D_j = 1/h on element j give diag(1/h)."""
    P = build("C1")
    sd = P.subs[0]
    out = lib.pre_assemble(predesc.subdomain_desc(P, sd), want_gram=True)
    h = 0.25
    GB = h / 6 * np.array([[2, 1, 0], [1, 4, 1], [0, 1, 2.0]])
    GD = np.diag([1 / h, 1 / h])
    # axis 0 of subdomain 0 spans one patch ([0, 1/2]); component 0 is B along x, D along y, z
    assert np.allclose(out["gram"][(0, 0, 0)], GB, rtol=0, atol=1e-15)
    assert np.allclose(out["gram"][(1, 0, 0)], GD, rtol=0, atol=1e-13)
    # partition of unity: the B Gram entries of a patch sum to its length
    for (c, a, q), g in out["gram"].items():
        if c == a:
            assert abs(g.sum() - 0.5) < 1e-14


@pytest.mark.parametrize("name", ["C1", "C2r", "C3r", "C4r", "C5r", "E27_L3_p2_e2", "C5"])
def test_gauge_tree_and_primal_bitwise(lib, name):
    P = build(name)
    g = predesc.gauge_desc(P)
    tree, prim, ms = lib.pre_gauge(g["nv"], g["ne"], g["eu"], g["ev"], g["w"])
    assert np.array_equal(tree, P.tree), (name, int((tree != P.tree).sum()))
    assert np.array_equal(np.flatnonzero(prim), P.primal_edges)


def test_gauge_matches_sequential_kruskal(lib):
    """Against Kruskal's algorithm itself (union-find scan in (weight, id) order)
    on a seeded random multigraph with several components and parallel edges."""
    from ietigen.problem import kruskal_unionfind
    from ietigen.rng import SplitMix64
    g = SplitMix64(7)
    nv, ne = 500, 1800
    eu = np.array([int(g.uniform() * 460) for _ in range(ne)], np.int32)   # vertices 460.. stay isolated
    ev = np.array([int(g.uniform() * 460) for _ in range(ne)], np.int32)
    keep = eu != ev
    eu, ev = eu[keep], ev[keep]
    ne = len(eu)
    w = np.array([1 + int(g.uniform() * 5) for _ in range(ne)], np.int8)
    order = np.lexsort((np.arange(ne), w))
    ref = kruskal_unionfind(nv, eu.astype(np.int64), ev.astype(np.int64), order)
    tree, prim, _ = lib.pre_gauge(nv, ne, eu, ev, w)
    assert np.array_equal(tree, ref)
    assert np.array_equal(prim, (~ref) & (w == 2))


def test_device_assembled_problem_solves(lib):
    """The device-assembled K^(k), j^(k) and the device gauge fed to the solve phase give the
    oracle's solution (u within 1e-8, N_iter within 1)."""
    from ietigen.bundle import make_bundle
    from oracle import dp
    b, P = make_bundle("C3r", with_problem=True)
    ref = dp.solve(b)
    g = predesc.gauge_desc(P)
    tree, prim, _ = lib.pre_gauge(g["nv"], g["ne"], g["eu"], g["ev"], g["w"])
    s = lib.Solver(b["n_sub"], b["n_lambda"], b["n_primal"], b["nrhs"], scaling=b["scaling"], tol=b["tol"])
    for k, sd in enumerate(P.subs):
        out = lib.pre_assemble(predesc.subdomain_desc(P, sd))
        bs = b["subs"][k]
        tr = np.flatnonzero(tree[sd.gid]).astype(np.int32)
        pm = np.flatnonzero(prim[sd.gid]).astype(np.int32)
        assert np.array_equal(tr, bs["tree"]) and np.array_equal(pm, bs["prim"])
        s.set_subdomain(k, out["K_indptr"], out["K_indices"], out["K_data"], out["f"], bs["B_lambda"], bs["B_dof"],
                        bs["B_sign"], tr, pm, bs["prim_gid"])
    s.factor()
    lam, rep = s.solve()
    u = np.concatenate([s.get_u(k) for k in range(b["n_sub"])])
    uref = np.concatenate(ref["u"])
    assert np.linalg.norm(u - uref) <= 1e-8 * np.linalg.norm(uref)
    assert abs(rep["iters"][0] - int(ref["iters"][0])) <= 1


def test_device_assembly_feeds_factorisation_on_device(lib):
    """Assembly -> ietidp_set_values_device -> factor -> solve without the matrix leaving the
    device: the solution is bitwise the one obtained by passing the same device-assembled
    values through the host (ietidp_set_values), and a second assembly with other reluctivities
    re-feeds the same handle."""
    from ietigen.bundle import make_bundle
    b, P = make_bundle("C3r", with_problem=True)
    descs = [predesc.subdomain_desc(P, sd) for sd in P.subs]
    batch = lib.PreBatch(descs)
    host = [batch.fetch(k) for k in range(len(descs))]
    s = lib.Solver(b["n_sub"], b["n_lambda"], b["n_primal"], b["nrhs"], scaling=b["scaling"], tol=b["tol"])
    for k, bs in enumerate(b["subs"]):
        o = host[k]
        s.set_subdomain(k, o["K_indptr"], o["K_indices"], o["K_data"], o["f"], bs["B_lambda"], bs["B_dof"], bs["B_sign"],
                        bs["tree"], bs["prim"], bs["prim_gid"])
    s.factor()
    lam0, _ = s.solve()
    u0 = np.concatenate([s.get_u(k) for k in range(b["n_sub"])])
    # perturbed material: nu scaled per patch; values through the host ...
    descs2 = [dict(d, nu=d["nu"] * (1.0 + 0.25 * ((i % 3) - 1))) for i, d in enumerate(descs)]
    batch2 = lib.PreBatch(descs2)
    for k in range(len(descs)):
        o = batch2.fetch(k)
        s.set_values(k, o["K_data"], o["f"])
    s.factor()
    lam_h, _ = s.solve()
    u_h = np.concatenate([s.get_u(k) for k in range(b["n_sub"])])
    assert np.linalg.norm(u_h - u0) > 1e-3 * np.linalg.norm(u0)  # the material did change the solution
    # ... back to the original values, then the perturbed ones straight from the device
    for k in range(len(descs)):
        s.set_values_device(k, *batch.device_ptrs(k))
    s.factor()
    lam1, _ = s.solve()
    assert np.array_equal(lam1, lam0)
    for k in range(len(descs)):
        s.set_values_device(k, *batch2.device_ptrs(k))
    s.factor()
    lam_d, _ = s.solve()
    u_d = np.concatenate([s.get_u(k) for k in range(b["n_sub"])])
    assert np.array_equal(lam_d, lam_h) and np.array_equal(u_d, u_h)
    # ietidp_pre_refill: the first batch re-assembled in place with the second one's nu
    batch.refill([d["nu"] for d in descs2])
    for k in range(len(descs)):
        assert np.array_equal(batch.fetch(k)["K_data"], batch2.fetch(k)["K_data"])


def test_pre_argument_errors(lib):
    P = build("C1")
    d = predesc.subdomain_desc(P, P.subs[0])
    bad = dict(d)
    bad["p"] = 4
    with pytest.raises(lib.IetiError) as e:
        lib.pre_assemble(bad)
    assert e.value.status == lib.E_ARG
    bad = dict(d)
    bad["fac_kind"] = [1 - k for k in d["fac_kind"]]
    with pytest.raises(lib.IetiError) as e:
        lib.pre_assemble(bad)
    assert e.value.status == lib.E_ARG
    with pytest.raises(lib.IetiError) as e:
        lib.pre_gauge(3, 1, np.array([0], np.int32), np.array([5], np.int32), np.array([1], np.int8))
    assert e.value.status == lib.E_ARG
