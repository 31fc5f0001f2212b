"""The C-ABI library without a GPU: it builds, loads, exports every entry point
include/ietidp.h declares, and its host-side analysis (validation, DOF
classification, nested dissection, symbolic factorisation) behaves as the header
documents. Handles created with device = -1 run the analysis only."""
import os
import re

import numpy as np
import pytest

from ietigen.bundle import make_bundle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2501_04340_b200 import ietidp
    return ietidp


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "ietidp.h")).read()
    declared = set(re.findall(r"\b(ietidp_[A-Za-z_]+)\s*\(", hdr))
    assert declared == set(lib.SYMBOLS)
    so = lib.load()
    for name in declared:
        assert hasattr(so, name), name
    hdr = open(os.path.join(ROOT, "include", "ietidp_shard.h")).read()
    declared = set(re.findall(r"\b(ietidp_shard_[A-Za-z_]+)\s*\(", hdr))
    assert declared == set(lib.SHARD_SYMBOLS)
    for name in declared:
        assert hasattr(so, name), name
    hdr = open(os.path.join(ROOT, "include", "ietidp_pre.h")).read()
    declared = set(re.findall(r"\b(ietidp_pre_[A-Za-z_]+)\s*\(", hdr))
    assert declared == set(lib.PRE_SYMBOLS)
    for name in declared:
        assert hasattr(so, name), name


def host_solver(lib, b, **kw):
    return lib.from_bundle(b, device=-1, **kw)


@pytest.mark.parametrize("name", ["C1", "C2r", "C3r"])
def test_host_analysis_counts(lib, name):
    b, P = make_bundle(name, with_problem=True)
    s = host_solver(lib, b)
    s.analyze()
    r = s.report()
    c = P.counts()
    assert r["sum_nr"] == c["sum_nr"]
    nI = [len(sd["B_dof"]) for sd in b["subs"]]
    assert r["sum_nI"] == sum(nI) == 2 * b["n_lambda"]  # every multiplier has two entries (F3)
    assert r["max_nI"] == max(nI)
    # the supernodal structure stores at least the lower triangle's diagonal
    assert r["nnz_L"] >= r["sum_nr"]


def test_nested_dissection_beats_dense_ordering(lib):
    b = make_bundle("C2r")
    s1 = host_solver(lib, b)
    s1.analyze()
    s2 = host_solver(lib, b, ordering="dense")
    s2.analyze()
    r1, r2 = s1.report(), s2.report()
    assert r1["factor_flops"] < r2["factor_flops"]
    # dense ordering: one r_V supernode + r_I root + P node per subdomain
    assert r2["n_supernodes"] == sum(1 + (len(sd["B_dof"]) > 0) + (len(sd["prim"]) > 0) for sd in b["subs"])


def test_c1_dense_flops_closed_form(lib):
    """C1 with the dense ordering: each subdomain's K_rr (n_r = 48) is one dense
    front of 48 pivots... split as r_V (33) then r_I (15) plus the P node (none on
    C1): sum_j c_j^2 over columns = sum_{c=1}^{48} c^2 per subdomain."""
    b = make_bundle("C1")
    s = host_solver(lib, b, ordering="dense")
    s.analyze()
    r = s.report()
    per = sum(c * c for c in range(1, 49))
    assert r["factor_flops"] == 2 * per
    assert r["nnz_L"] == 2 * 48 * 49 // 2


def test_b_row_with_three_entries(lib):
    b = make_bundle("C1")
    sd = b["subs"][0]
    # duplicate multiplier 0 onto another remaining DOF of subdomain 1
    sd1 = b["subs"][1]
    free = np.setdiff1d(np.arange(sd1["n"]), np.concatenate([sd1["tree"], sd1["prim"], sd1["B_dof"]]))
    sd1["B_lambda"] = np.append(sd1["B_lambda"], sd["B_lambda"][0]).astype(np.int32)
    sd1["B_dof"] = np.append(sd1["B_dof"], free[0]).astype(np.int32)
    sd1["B_sign"] = np.append(sd1["B_sign"], -1).astype(np.int8)
    s = host_solver(lib, b)
    with pytest.raises(lib.IetiError) as e:
        s.analyze()
    assert e.value.status == lib.E_B_STRUCTURE


def test_b_touching_tree_dof(lib):
    b = make_bundle("C1")
    sd = b["subs"][0]
    sd["B_dof"] = sd["B_dof"].copy()
    sd["B_dof"][0] = sd["tree"][0]
    s = host_solver(lib, b)
    with pytest.raises(lib.IetiError) as e:
        s.analyze()
    assert e.value.status == lib.E_B_STRUCTURE


def test_nonsymmetric_pattern_rejected(lib):
    b = make_bundle("C1")
    sd = b["subs"][0]
    ip, ix = sd["K_indptr"].copy(), sd["K_indices"].copy()
    # drop the last entry of row 0 (its transpose stays)
    row0 = ix[ip[0]:ip[1]]
    keep = np.ones(len(ix), bool)
    keep[ip[1] - 1] = False
    assert row0[-1] != 0
    sd["K_indices"] = ix[keep]
    sd["K_data"] = sd["K_data"][keep]
    sd["K_indptr"] = np.concatenate([[0], ip[1:] - 1])
    with pytest.raises(lib.IetiError) as e:
        host_solver(lib, b)
    assert e.value.status == lib.E_ARG


def test_nonsymmetric_pattern_same_counts_rejected(lib):
    """A pattern whose row and column counts match but which is not symmetric: in a
    symmetric pattern, entry (i, j) is moved to (i, j') with (j, i) left in place -- every
    row keeps its length, the column sets do not mirror."""
    import scipy.sparse as sp
    b = make_bundle("C1")
    sd = b["subs"][0]
    n = len(sd["K_indptr"]) - 1
    A = sp.csr_matrix((sd["K_data"], sd["K_indices"], sd["K_indptr"]), shape=(n, n)).tolil()
    rows, cols = A.nonzero()
    # an upper entry (i, j) and a column j' > i absent from row i
    for i, j in zip(rows, cols):
        if j > i:
            free = [c for c in range(i + 1, n) if A[i, c] == 0]
            if free:
                jp = free[0]
                break
    A[i, jp] = A[i, j]
    A[i, j] = 0
    B = A.tocsr()
    B.eliminate_zeros()
    B.sort_indices()
    assert B.nnz == sp.csr_matrix((sd["K_data"], sd["K_indices"], sd["K_indptr"])).nnz
    sd["K_indptr"], sd["K_indices"], sd["K_data"] = B.indptr.astype(np.int64), B.indices.astype(np.int32), B.data
    with pytest.raises(lib.IetiError) as e:
        host_solver(lib, b)
    assert e.value.status == lib.E_ARG


def test_state_machine(lib):
    b = make_bundle("C1")
    s = host_solver(lib, b)
    with pytest.raises(lib.IetiError) as e:
        s.solve()
    assert e.value.status == lib.E_STATE
    sd = b["subs"][0]
    with pytest.raises(lib.IetiError) as e:
        s.set_subdomain(0, sd["K_indptr"], sd["K_indices"], sd["K_data"], sd["f"], sd["B_lambda"], sd["B_dof"],
                        sd["B_sign"], sd["tree"], sd["prim"], sd["prim_gid"])
    assert e.value.status == lib.E_STATE
    s.analyze()
    with pytest.raises(lib.IetiError) as e:
        s.factor()  # host-only handle: no device work
    assert e.value.status == lib.E_STATE


def test_missing_subdomain(lib):
    b = make_bundle("C1")
    s = lib.Solver(b["n_sub"], b["n_lambda"], b["n_primal"], b["nrhs"], device=-1)
    sd = b["subs"][0]
    s.set_subdomain(0, sd["K_indptr"], sd["K_indices"], sd["K_data"], sd["f"], sd["B_lambda"], sd["B_dof"],
                    sd["B_sign"], sd["tree"], sd["prim"], sd["prim_gid"])
    with pytest.raises(lib.IetiError) as e:
        s.analyze()
    assert e.value.status == lib.E_STATE


# ---- argument validation of the pre-processing and sharding entry points (host side) ----

def test_pre_and_shard_argument_errors_without_gpu(lib):
    """include/ietidp_pre.h / ietidp_shard.h: every documented E_ARG / E_STATE is raised by the
    host-side validation, before any device work (so it can be checked without a GPU)."""
    from ietigen import predesc
    from ietigen.problem import build
    P = build("C1")
    d = predesc.subdomain_desc(P, P.subs[0])
    for key, val in [("p", 4), ("p", 0), ("e", 0), ("nq", 0)]:
        bad = dict(d)
        bad[key] = val
        with pytest.raises(lib.IetiError) as e:
            lib.pre_assemble(bad, device=0)
        assert e.value.status == lib.E_ARG, key
    bad = dict(d)
    bad["fac_kind"] = [1 - k for k in d["fac_kind"]]  # a B factor where the component needs D
    with pytest.raises(lib.IetiError) as e:
        lib.pre_assemble(bad)
    assert e.value.status == lib.E_ARG
    bad = dict(d)
    dof = d["dof_of_edge"].copy()
    i = np.flatnonzero(dof >= 0)[:2]
    dof[i] = dof[i[::-1]]  # DOFs not ascending with the edge id
    bad["dof_of_edge"] = dof
    with pytest.raises(lib.IetiError) as e:
        lib.pre_assemble(bad)
    assert e.value.status == lib.E_ARG
    bad = dict(d)
    bad["term_col"] = d["term_col"] + 7  # RHS column out of range
    with pytest.raises(lib.IetiError) as e:
        lib.pre_assemble(bad)
    assert e.value.status == lib.E_ARG
    # gauge: endpoints and weights
    one = np.array([0], np.int32)
    for eu, ev, w in [(one, np.array([5], np.int32), np.array([1], np.int8)),
                      (one, np.array([1], np.int32), np.array([0], np.int8)),
                      (one, np.array([1], np.int32), np.array([6], np.int8))]:
        with pytest.raises(lib.IetiError) as e:
            lib.pre_gauge(3, 1, eu, ev, w)
        assert e.value.status == lib.E_ARG
    # sharded mode: only before analysis, only the explicit loop with the residual criterion
    b = make_bundle("C1")
    s = host_solver(lib, b)
    s.analyze()
    with pytest.raises(lib.IetiError) as e:
        s.shard_enable(0, 2, lambda ptr, n, stream: 0)
    assert e.value.status == lib.E_STATE
    for kw in (dict(loop="triangular"), dict(stop="preconditioned")):
        s = host_solver(lib, b, **kw)
        with pytest.raises(lib.IetiError) as e:
            s.shard_enable(0, 2, lambda ptr, n, stream: 0)
        assert e.value.status == lib.E_ARG
    s = host_solver(lib, b)
    with pytest.raises(lib.IetiError) as e:
        s.shard_enable(2, 2, lambda ptr, n, stream: 0)  # rank out of range
    assert e.value.status == lib.E_ARG
