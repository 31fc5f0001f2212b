"""Pins of the input generator (ietigen): spline spaces, de Rham assembly,
weights, Kruskal tree, primal selection, multiplier pairing.

Every check is against something other than the generator itself: SPEC/paper
numbers (tests/golden/counts.json), closed forms, exact identities of the de Rham
complex, brute force (pure-Python Kruskal, finite differences).
"""
import json
import os
from dataclasses import replace

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

from ietigen import configs as cf
from ietigen.problem import Problem, local_curl, local_grad, cube_spaces, kruskal_unionfind
from ietigen.splines import Space1D, knot_vector, bspline_values, dspline_values
from ietigen.bundle import make_bundle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "counts.json")))


def cfg_custom(name, npatch, p, e, tiling, **kw):
    return cf.Config(name, npatch, p, e, tiling, **kw)


# ---------------------------------------------------------------- splines ---
@pytest.mark.parametrize("p,e,key", [(1, 1, "p1_e1"), (2, 4, "p2_e4"), (3, 8, "p3_e8")])
def test_single_patch_dims(p, e, key):
    """1-form dimension of one patch."""
    sp1 = Space1D(0.0, 1.0, 1, e, p)
    m = sp1.m
    assert m == e + p
    assert 3 * (m - 1) * m * m == GOLD["space_dims"][key]


@pytest.mark.parametrize("p", [1, 2, 3])
def test_partition_of_unity_and_derivative(p):
    """B-splines sum to 1; B_i' = D_{i-1} - D_i checked by central
    differences; each D_j integrates to 1."""
    s = Space1D(0.0, 1.0, 3, 4, p)
    x = np.random.default_rng(0).uniform(0.01, 0.99, 40)
    B = s.B(x)
    assert np.allclose(B.sum(axis=1), 1.0, atol=1e-14)
    h = 1e-6
    dB = (s.B(x + h) - s.B(x - h)) / (2 * h)
    D = s.D(x)
    Dpad = np.concatenate([np.zeros((len(x), 1)), D, np.zeros((len(x), 1))], axis=1)
    pred = Dpad[:, :-1] - Dpad[:, 1:]
    # away from knots (random points) the derivative is smooth
    assert np.allclose(dB, pred, atol=1e-6)
    xq, wq = s.quad(p + 1)
    assert np.allclose((s.D(xq) * wq[:, None]).sum(axis=0), 1.0, atol=1e-13)


# --------------------------------------------------------------- assembly ---
def test_curl_grad_zero_exact_and_K_kernel():
    """C . G_grad = 0 in integers and K G_grad = 0 to 1e-12 ||K|| (BJ "discrete
    curl o grad = 0")."""
    cfg = cf.get("C2r")
    P = Problem(cfg)
    sd = P.subs[3]
    C = local_curl(sd.ml)
    G = local_grad(sd.ml)
    assert abs(C @ G).max() == 0
    spaces = cube_spaces(cfg, sd)
    from ietigen.problem import cube_mass2
    M2 = cube_mass2(cfg, sd, spaces, P.nu)
    K = C.T @ M2 @ C
    assert abs(K @ G).max() <= 1e-12 * abs(K).max()
    assert abs(K - K.T).max() <= 1e-14 * abs(K).max()
    w = np.linalg.eigvalsh(K.toarray())
    assert w.min() > -1e-12 * w.max()


def test_loads_discretely_divergence_free():
    """G_grad^T j = (C G)^T t = 0: weak-curl loads annihilate gradients."""
    cfg = cf.get("C5r")
    P = Problem(cfg)
    sd = P.subs[5]
    K, j, Cm, M2, t = P.assemble(sd, with_face=True)
    G = local_grad(sd.ml)
    jf = local_curl(sd.ml).T @ t
    assert abs(G.T @ jf).max() <= 1e-13 * abs(jf).max()


def test_manufactured_source_identity():
    """J = curl curl A* = 2 pi^2 A* (SURVEY O3): curl of the generator's T by
    central differences at random points."""
    terms = cf.source_terms(cf.C1)[0]

    def T(x):
        out = np.zeros(3)
        for c in range(3):
            for coef, fx, fy, fz in terms[c]:
                out[c] += coef * cf.f1d(fx)(x[0]) * cf.f1d(fy)(x[1]) * cf.f1d(fz)(x[2])
        return out

    rng = np.random.default_rng(1)
    h = 1e-5
    for _ in range(10):
        x = rng.uniform(0, 1, 3)
        J = np.zeros((3, 3))
        for b in range(3):
            dx = np.zeros(3)
            dx[b] = h
            J[:, b] = (T(x + dx) - T(x - dx)) / (2 * h)
        curlT = np.array([J[2, 1] - J[1, 2], J[0, 2] - J[2, 0], J[1, 0] - J[0, 1]])
        s = np.sin(np.pi * x)
        Astar = np.array([s[1] * s[2], s[2] * s[0], s[0] * s[1]])
        assert np.allclose(curlT, 2 * np.pi ** 2 * Astar, atol=1e-6)


# ------------------------------------------------------------ gauge, counts ---
def test_bar_and_cube27_trees():
    """SPEC.md:127-128, :310-312 graph and tree counts."""
    bar = Problem(cfg_custom("bar", (2, 1, 1), 1, 1, (2, 1, 1)))
    g = GOLD["bar2_p1_e1"]
    assert bar.grid.nv == g["vertices"] and bar.grid.ne == g["edges"]
    assert bar.tree.sum() == g["tree"]
    w1 = bar.weight == 1
    assert w1.sum() == g["weight1"] and (bar.tree & w1).sum() == g["weight1_in_tree"]
    c27 = Problem(cfg_custom("c27", (3, 3, 3), 1, 1, (3, 1, 1)))
    g = GOLD["cube27_p1_e1"]
    assert c27.grid.nv == g["vertices"] and c27.grid.ne == g["edges"] and c27.tree.sum() == g["tree"]


def _closed_form_ngp(T):
    nx, ny, nz = T
    lines = (ny - 1) * (nz - 1) + (nx - 1) * (nz - 1) + (nx - 1) * (ny - 1)
    junctions = (nx - 1) * (ny - 1) * (nz - 1)
    return lines + 2 * junctions


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_global_counts(name):
    """E_int - V_int = (m-2)^2 (2m-1); n_gp closed form F4 (App. B3);
    weight-1/2 counts (App. A); Sum n_r - m_r + n_gp = E_int - V_int."""
    cfg = cf.get(name)
    P = Problem(cfg)
    c = P.counts()
    m = P.grid.m[0]
    assert c["E_int"] - c["V_int"] == (m - 2) ** 2 * (2 * m - 1)
    assert c["n_gp"] == _closed_form_ngp(cfg.tiling)
    w1, w2, ngp = GOLD["weight12_counts"][name]
    assert (c["w_counts"][0], c["w_counts"][1], c["n_gp"]) == (w1, w2, ngp)
    assert c["sum_nr"] - c["m_r"] + c["n_gp"] == c["E_int"] - c["V_int"]
    if name == "C2":
        assert c["m_r"] == GOLD["C2_m_r_hand_count"]["m_r"]


@pytest.mark.parametrize("name", ["C1", "C2r", "C3r", "C5r"])
def test_tree_properties(name):
    """Spanning tree (V-1 edges, connected), pure-Python Kruskal equals the
    unique-key MST, Dirichlet restriction is a spanning tree of the boundary
    graph, classes exhaustive/disjoint, n_gp independent of e
    (PAPER.md:180)."""
    cfg = cf.get(name)
    P = Problem(cfg, kruskal="python")
    Q = Problem(cfg, kruskal="scipy")
    assert np.array_equal(P.tree, Q.tree)
    g = P.grid
    assert P.tree.sum() == g.nv - 1
    A = sp.csr_matrix((np.ones(P.tree.sum()), (P.eu[P.tree], P.ev[P.tree])), shape=(g.nv, g.nv))
    assert connected_components(A, directed=False)[0] == 1
    dv = g.dirichlet_vertices()
    de = P.dir_edge
    nb = dv.sum()
    Ab = sp.csr_matrix((np.ones(de.sum()), (P.eu[de], P.ev[de])), shape=(g.nv, g.nv))
    ncomp_b = connected_components(Ab[dv][:, dv], directed=False)[0]
    assert (P.tree & de).sum() == nb - ncomp_b
    assert set(np.unique(P.weight)) <= {1, 2, 3, 4, 5}
    full = Problem(cf.get(name[:2])) if name != "C1" else P
    assert P.n_primal == full.n_primal


def test_c1_per_subdomain_counts():
    b, P = make_bundle("C1", with_problem=True)
    g = GOLD["C1_per_subdomain"]
    for s in b["subs"]:
        nr = s["n"] - len(s["tree"]) - len(s["prim"])
        assert s["n"] == g["n_k"] and len(s["tree"]) == g["tree"] and nr == g["n_r"]
        assert len(s["B_dof"]) == g["r_I"] and nr - len(s["B_dof"]) == g["r_V"]


@pytest.mark.parametrize("name", ["C2r", "C5r"])
def test_B_structure(name):
    """Each multiplier row has one +1 (lower subdomain) and one -1 (F3);
    each remaining interface DOF in exactly one row; tree consistent across
    interfaces; primal DOFs shared by >= 3 subdomains."""
    b, P = make_bundle(name, with_problem=True)
    rows = {}
    for k, s in enumerate(b["subs"]):
        assert len(np.unique(s["B_dof"])) == len(s["B_dof"])
        for lam, sg in zip(s["B_lambda"], s["B_sign"]):
            rows.setdefault(int(lam), []).append((k, int(sg)))
    assert len(rows) == b["n_lambda"]
    for lam, ent in rows.items():
        assert len(ent) == 2
        (k1, s1), (k2, s2) = sorted(ent)
        assert s1 == 1 and s2 == -1
    for sd in P.subs:
        tr = P.tree[sd.gid]
        assert np.array_equal(np.flatnonzero(tr), sd.tree)
    assert np.all(P.membership[P.primal_edges] >= 3)


# -------------------------------------------------------------- cylinder ---
def test_cylinder_geometry_exact():
    """C4: the rational quadratic arcs lie on the unit circle, the
    angular speed integrates to 2 pi, |det J| integrates to the tube volume."""
    from ietigen import cylinder as cy
    C, dC = cy.arc(np.linspace(0.0, 1.0, 33))
    assert np.abs(np.linalg.norm(C, axis=-1) - 1.0).max() <= 1e-15
    # arc endpoints: angle 0 and 2 pi/16
    assert np.allclose(C[0], [1.0, 0.0]) and np.allclose(C[-1], [np.cos(np.pi / 8), np.sin(np.pi / 8)])
    x, w = np.polynomial.legendre.leggauss(24)
    s, ws = 0.5 * (x + 1), 0.5 * w
    th = sum((ws * cy.theta_s((a + s) / 16)).sum() / 16 for a in range(16))
    assert abs(th - 2 * np.pi) <= 1e-13
    vol = th * (ws * 0.5 * cy.radius(s)).sum() * 1.0
    assert abs(vol - 0.75 * np.pi) <= 1e-13


def test_cylinder_counts():
    """C4 integer pins: E_int = 184,448, V_int = 59,520,
    n_gp = 64 (16 z-lines + 16 r-lines + closed theta ring with 16 junctions),
    m_r = 14,208, sum n_r = 139,072, weight-1/2 edges (2,048, 896); the reduced
    variant keeps n_gp with 14,848 gauged DOFs."""
    P = Problem(cf.get("C4"))
    c = P.counts()
    assert (c["E_int"], c["V_int"]) == (184448, 59520)
    assert (c["n_gp"], c["m_r"], c["sum_nr"]) == (64, 14208, 139072)
    assert (c["w_counts"][0], c["w_counts"][1]) == (2048, 896)
    assert c["sum_nr"] - c["m_r"] + c["n_gp"] == c["E_int"] - c["V_int"]
    r = Problem(cf.get("C4r")).counts()
    assert r["n_gp"] == 64 and r["E_int"] - r["V_int"] == 14848


def test_cylinder_curl_grad_and_loads():
    """Discrete curl o grad = 0 on the curved, periodic patches; K symmetric PSD;
    loads discretely divergence-free (G^T j = 0)."""
    from ietigen import cylinder as cy
    cfg = cf.get("C4r")
    P = Problem(cfg)
    for sd in P.subs[:3]:
        C = local_curl(sd.ml)
        Gd = local_grad(sd.ml)
        assert abs(C @ Gd).max() == 0
        spaces = cy.cylinder_spaces(cfg, sd)
        M2 = cy.cylinder_mass2(cfg, sd, spaces, P.nu)
        t = cy.cylinder_face_loads(cfg, sd, spaces)
        Kf = (C.T @ M2 @ C).tocsr()
        assert abs(Kf @ Gd).max() <= 1e-12 * abs(Kf).max()
        assert abs(Gd.T @ (C.T @ t)).max() <= 1e-12 * abs(t).max()
        K, j = P.assemble(sd)
        ev = np.linalg.eigvalsh(K.toarray())
        assert ev.min() >= -1e-10 * ev.max()


# ---- the paper's 27-patch experiment family (R14) ----

@pytest.mark.parametrize("tiling", ["311", "221", "321", "222", "322", "L3"])
def test_paper_cube_ngp_independent_of_h_and_p(tiling):
    """n_gp depends on the subdomain configuration only, not on h or p (PAPER.md:180,
    :268 "n_gp is independent of h and p")."""
    from ietigen.problem import build
    ngp = {build(cf.get(f"E27_{tiling}_p{p}_e{e}")).counts()["n_gp"] for p in (1, 2, 3) for e in (2, 4)}
    assert len(ngp) == 1, ngp


def test_paper_e1_partition_has_cross_points():
    """E1's partition (three L-shaped 9-patch subdomains, ietigen.configs.PAPER_PARTS):
    all three subdomains meet along one patch line, so the coarse problem is not empty
    (n_gp > 0), unlike a 3 x 1 x 1 slab tiling (n_gp = 0); every subdomain has 9 patches
    and is face-connected to the other two."""
    from ietigen.problem import build
    P = build(cf.get("E27_L3_p1_e2"))
    assert P.counts()["n_gp"] > 0
    assert sorted(len(sd.boxes) for sd in P.subs) == [9, 9, 9]
    assert sorted(P.iface_pairs) == [(0, 1), (0, 2), (1, 2)]
    assert build(cf.get("E27_311_p1_e2")).counts()["n_gp"] == 0


@pytest.mark.parametrize("p", [1, 2])
def test_union_of_patches_assembly_gives_the_same_field(p):
    """The union-of-patches assembly (L-shaped subdomains) against the single-box one: the
    gauged solutions of E27_L3 and of the slab tiling E27_311 differ by a discrete
    gradient (different trees), so their curls C a -- the flux B_h of PAPER.md:255 --
    agree (to the solver's rounding); a wrong torn assembly on the unions would not."""
    from oracle import brute
    from ietigen.problem import build, local_curl
    fields = []
    for t in ("L3", "311"):
        b, P = make_bundle(f"E27_{t}_p{p}_e2", with_problem=True)
        _, a, _, _ = brute.monolithic_solve(b)
        g = P.grid
        x = np.zeros((g.ne, a.shape[1]))
        x[P.gauged_edges] = a
        gids, ml = g.block_edges((0, 0, 0), tuple(P.cfg.npatch))
        fields.append(local_curl(ml) @ x[gids])
    assert np.linalg.norm(fields[0] - fields[1]) <= 1e-9 * np.linalg.norm(fields[1])


@pytest.mark.parametrize("name", ["E27_221_p2_e2", "E27_322_p1_e2", "E27_L3_p1_e2", "E27_L3_p2_e2"])
def test_uneven_tiling_dd_equals_monolithic(name):
    """Uneven box tilings (3 patches cut 1 + 2): every K_rr SPD, the DD solution equals
    the monolithic gauged solve."""
    from oracle import dp, brute
    b = make_bundle(name)
    res = dp.solve(b, tol=1e-12, check_spd=True)
    um, _, _, _ = brute.monolithic_solve(b)
    U, Um = np.concatenate(res["u"]), np.concatenate(um)
    assert np.linalg.norm(U - Um) <= 1e-10 * np.linalg.norm(Um)


# ---- the paper's A_ana with inhomogeneous boundary values ----

def _bana_norm2():
    # ||B_ana||^2 over (0,1)^3, B_ana = (-3 cos x sin y sin z, 0, 3 cos z sin x sin y):
    # 9 (C S S + S S C), C = int cos^2 = 1/2 + sin(2)/4, S = int sin^2 = 1/2 - sin(2)/4
    C, S = 0.5 + np.sin(2.0) / 4, 0.5 - np.sin(2.0) / 4
    return 18.0 * C * S * S


def test_aana_identities():
    """curl curl A_ana = 3 A_ana, div A_ana = 0 and B_ana = curl A_ana,
    checked by central differences at seeded points: the source T = B_ana and the lifted
    boundary data belong to the same closed-form solution."""
    from ietigen import configs as cf
    from ietigen.rng import SplitMix64

    def A(x):
        return np.array([c * cf.f1d(fx)(x[0:1])[0] * cf.f1d(fy)(x[1:2])[0] * cf.f1d(fz)(x[2:3])[0]
                         for c, fx, fy, fz in cf.A_ANA])

    def B(x):
        out = np.zeros(3)
        for s_, col in enumerate(cf.source_terms(cf.get("E27A_311_p1_e1"))[0]):
            for c, fx, fy, fz in col:
                out[s_] += c * cf.f1d(fx)(x[0:1])[0] * cf.f1d(fy)(x[1:2])[0] * cf.f1d(fz)(x[2:3])[0]
        return out

    def curl(F, x, h=1e-5):
        J = np.zeros((3, 3))
        for j in range(3):
            e = np.zeros(3)
            e[j] = h
            J[:, j] = (F(x + e) - F(x - e)) / (2 * h)
        return np.array([J[2, 1] - J[1, 2], J[0, 2] - J[2, 0], J[1, 0] - J[0, 1]]), np.trace(J)
    g = SplitMix64(11)
    for _ in range(5):
        x = np.array([0.1 + 0.8 * g.uniform() for _ in range(3)])
        cA, divA = curl(A, x)
        assert np.allclose(cA, B(x), atol=1e-8) and abs(divA) < 1e-8
        ccA, _ = curl(lambda y: curl(A, y)[0], x, h=1e-3)
        assert np.allclose(ccA, 3 * A(x), atol=1e-5)


@pytest.mark.parametrize("p", [1, 2])
def test_aana_flux_error_order(p):
    """eps_B = O(h^p) for the paper's A_ana with its boundary values lifted (PAPER.md:258,
    Fig. 4b), on a box tiling and on E1's union-of-patches partition (the lifting goes
    through both assembly branches); DD = monolithic."""
    from oracle import brute, dp
    bn2 = _bana_norm2()
    errs = []
    for e in (1, 2, 4):
        b, P = make_bundle(f"E27A_311_p{p}_e{e}", with_problem=True)
        res = dp.solve(b, tol=1e-12)
        errs.append(P.flux_error(res["u"], bn2))
    eoc = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(eoc - p) <= 0.3), (errs, eoc)
    b, P = make_bundle(f"E27A_L3_p{p}_e2", with_problem=True)
    res = dp.solve(b, tol=1e-12)
    assert abs(P.flux_error(res["u"], bn2) - errs[1]) <= 1e-3 * errs[1]  # same field, another partition
    um, _, _, _ = brute.monolithic_solve(b)
    assert abs(P.flux_error(um, bn2) - P.flux_error(res["u"], bn2)) <= 1e-9 * errs[1]
    # without the lifting the boundary data is wrong and the error does not converge
    P._aD = np.zeros_like(P._aD)
    assert P.flux_error(res["u"], bn2) > 10 * errs[1]
