"""Sharded solve (include/ietidp_shard.h) against the oracle: the
subdomains split over R "ranks", each a handle of its own driven by its own host thread, all on
the one GPU this pool provides. The all-reduce is a host-side sum (the threads meet at a
barrier; rank 0 adds the R device buffers in rank order and copies the sum back to each), so no
kernel ever waits for another rank's kernel. What is exercised is everything a multi-GPU run
does except the transport: one-sided multiplier rows, the exchanged K diagonals of the
stiffness scaling, the summed S_PP / ftilde / d_DP, the per-iteration sums of g, q and z, the
replicated CG scalars, the recovery with the summed coarse right-hand side.

Parity bar as for the single-handle path: N_iter within 1, u and lambda
within 1e-8, dual residual <= 1e-10.
"""
import threading

import numpy as np
import pytest

from ietigen.bundle import make_bundle
from oracle import dp
from oracle_variants import explicit_inverse_iters
from parity_checks import check_iters, check_solution

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2501_04340_b200 import ietidp
    return ietidp


class HostSumComm:
    """In-process stand-in for NCCL: R threads, one per rank."""

    def __init__(self, lib, nranks):
        import torch
        self.torch, self.lib, self.n = torch, lib, nranks
        self.bar = threading.Barrier(nranks)
        self.views = [None] * nranks
        self.calls = 0
        self.doubles = 0
        self.side = torch.cuda.Stream()  # the sums run here (non-blocking stream)

    def fn(self, rank):
        def allreduce(ptr, n, stream):
            torch = self.torch
            # stream-level waits only: another rank's thread may be capturing its factorisation
            # graph, during which a device-wide synchronisation is not permitted
            torch.cuda.ExternalStream(int(stream)).synchronize()
            self.views[rank] = torch.as_tensor(self.lib.CudaView(ptr, n), device="cuda")
            self.bar.wait()
            if rank == 0:
                assert all(v.numel() == n for v in self.views)
                with torch.cuda.stream(self.side):
                    total = self.views[0].clone()
                    for r in range(1, self.n):
                        total += self.views[r]
                    for r in range(self.n):
                        self.views[r].copy_(total)
                self.side.synchronize()
                self.calls += 1
                self.doubles += n
            self.bar.wait()
            return 0
        return allreduce


def run_sharded(lib, b, nranks, owner=None, **opts):
    if owner is None:
        w = [float(len(sd["K_data"])) for sd in b["subs"]]
        owner = lib.shard_partition(w, nranks)
    comm = HostSumComm(lib, nranks)
    out = [None] * nranks
    err = []

    def work(rank):
        try:
            s = lib.shard_from_bundle(b, owner, rank, nranks, comm.fn(rank), **opts)
            s.factor()
            lam, rep = s.solve()
            us = {k: s.get_u(i) for i, k in enumerate(s.global_ids)}
            out[rank] = (lam, rep, us, s)
        except Exception as e:  # release the other threads
            err.append(e)
            comm.bar.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out, owner, comm


@pytest.mark.parametrize("name,nranks", [("C2r", 2), ("C3r", 2), ("C3r", 3), ("C4r", 2), ("C5r", 2), ("C1", 2)])
def test_sharded_solution_matches_oracle(lib, name, nranks):
    b = make_bundle(name)
    ref = dp.solve(b)
    out, owner, comm = run_sharded(lib, b, nranks)
    assert len(set(owner.tolist())) == nranks
    lam0, rep0 = out[0][0], out[0][1]
    for r in range(1, nranks):  # replicated state: bitwise the same on every rank
        assert np.array_equal(out[r][0], lam0)
        assert out[r][1]["iters"] == rep0["iters"]
    it_gpu, it_ref = np.asarray(rep0["iters"]), np.asarray(ref["iters"])
    it_alt = None
    if not np.all(np.abs(it_gpu - it_ref) <= 1):  # C5r: DESIGN.md R10
        it_alt = explicit_inverse_iters(b)
    check_iters(it_gpu, it_ref, it_alt)
    assert max(rep0["rel_residual"]) <= 1e-10
    us = {}
    for r in range(nranks):
        us.update(out[r][2])
    assert sorted(us) == list(range(b["n_sub"]))
    check_solution(b, lam0, [us[k] for k in range(b["n_sub"])], ref["lam"], ref["u"])
    assert comm.calls > 0


def test_sharded_equals_single_handle_iteration_matched(lib):
    """The same fixed number of iterations on one handle (persistent kernel) and on two shards
    (launch by launch, sums over ranks): lambda and u agree to rounding."""
    b = make_bundle("C3r")
    s = lib.from_bundle(b, fixed_iters=12)
    s.factor()
    lam1, _ = s.solve()
    u1 = np.concatenate([s.get_u(k) for k in range(b["n_sub"])])
    out, owner, _ = run_sharded(lib, b, 2, fixed_iters=12)
    us = {}
    for r in range(2):
        us.update(out[r][2])
    u2 = np.concatenate([us[k] for k in range(b["n_sub"])])
    assert np.linalg.norm(out[0][0] - lam1) <= 1e-10 * np.linalg.norm(lam1)
    assert np.linalg.norm(u2 - u1) <= 1e-10 * np.linalg.norm(u1)


def test_sharded_chunk_loop_equals_stream_loop(lib, monkeypatch):
    """16 RHS: the sharded loop runs the chunk pass and its phases as separate launches
    (IETIDP_SHARD_CHUNK=0: the row-segment stream instead). Same operators, different
    summation layouts: after a fixed number of iterations lambda agrees to the parity bar 1e-8
    (cond(M^-1 F) ~ 800 on C5r amplifies the two layouts' rounding to ~2e-9 by iteration 25)."""
    b = make_bundle("C5r")
    out1, _, _ = run_sharded(lib, b, 2, fixed_iters=25)
    monkeypatch.setenv("IETIDP_SHARD_CHUNK", "0")
    out0, _, _ = run_sharded(lib, b, 2, fixed_iters=25)
    monkeypatch.delenv("IETIDP_SHARD_CHUNK")
    lam1, lam0 = out1[0][0], out0[0][0]
    assert np.all(np.linalg.norm(lam1 - lam0, axis=0) <= 1e-8 * np.linalg.norm(lam0, axis=0))
    assert not np.array_equal(lam1, lam0)  # (they are different code paths)


def test_uneven_partition_and_empty_coarse_rank(lib):
    """A lopsided owner map (one subdomain alone on rank 1): its rank sees only some primal
    DOFs and one-sided multipliers on all its faces."""
    b = make_bundle("C2r")
    owner = np.zeros(b["n_sub"], np.int32)
    owner[-1] = 1
    ref = dp.solve(b)
    out, _, _ = run_sharded(lib, b, 2, owner=owner)
    assert abs(out[0][1]["iters"][0] - int(ref["iters"][0])) <= 1
    us = {}
    for r in range(2):
        us.update(out[r][2])
    u = np.concatenate([us[k] for k in range(b["n_sub"])])
    uref = np.concatenate(ref["u"])
    assert np.linalg.norm(u - uref) <= 1e-8 * np.linalg.norm(uref)


def test_bench_shard_one_rank_native_nccl():
    """`bench.py --shard` on one rank: the library calls ncclAllReduce itself on a one-rank
    communicator created through the binding (ietidp_shard_enable_nccl); one JSON line, the
    oracle's iteration count for C2r, strong scaling declared."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--shard", "--config", "C2r", "--steps", "2", "--warmup", "3"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    if r.returncode != 0 and ("NCCL" in r.stderr or "nccl" in r.stderr or "Address already in use" in r.stderr):
        pytest.skip("NCCL could not initialise in this environment: " + r.stderr[-300:])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    ref = dp.solve(make_bundle("C2r"))
    assert d["scaling"] == "strong" and d["n_gpus"] == 1 and d["value"] > 0
    assert abs(d["iters"][0] - int(ref["iters"][0])) <= 1 and d["rel_residual"] <= 1e-10
    assert d["shard"]["transport"].startswith("ncclAllReduce")
