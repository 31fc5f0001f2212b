"""The N>1 path on CPU (gloo, world size 2): bench.py's rank plumbing -- barrier and
the max-over-ranks timing reduction -- and the reference arm under torchrun, where
rank 0 alone runs the oracle and prints the one JSON line (replicas only,
no data-path collective)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    import torch.distributed as dist

    class A:
        impl = "reference"  # gloo
    r, w, _ = bench.dist_init(A())
    assert (r, w) == (rank, world)
    bench.barrier(w)
    out[rank] = bench.max_over_ranks(1.5 + rank, w)  # per-rank "step time"
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    world = 2
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0] == out[1] == 2.5  # every rank sees the slowest rank's time


def test_reference_arm_torchrun_world2():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
           "--config", "C1", "--steps", "1", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


# ---- sharded solve (include/ietidp_shard.h): host side on CPU ----

def test_shard_partition_properties():
    import numpy as np
    from paper_2501_04340_b200 import ietidp
    import __graft_entry__
    __graft_entry__.build()
    from ietigen.rng import SplitMix64
    g = SplitMix64(3)
    for n_sub, nranks in [(16, 2), (16, 3), (108, 8), (5, 5), (7, 1), (128, 8)]:
        w = np.array([0.5 + 4.0 * g.uniform() for _ in range(n_sub)])
        owner = ietidp.shard_partition(w, nranks)
        assert owner[0] == 0 and owner[-1] == nranks - 1
        assert np.all(np.diff(owner) >= 0) and np.all(np.diff(owner) <= 1)       # contiguous ranges
        load = np.bincount(owner, weights=w, minlength=nranks)
        assert np.all(np.bincount(owner, minlength=nranks) >= 1)
        if n_sub >= 4 * nranks:  # balanced to within one subdomain's weight
            assert load.max() - w.sum() / nranks <= w.max() + 1e-12
    assert list(ietidp.shard_partition([10.0, 1.0, 1.0], 3)) == [0, 1, 2]
    with pytest.raises(ietidp.IetiError):
        ietidp.shard_partition([1.0, -1.0], 2)


def _shard_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist
    from ietigen.bundle import make_bundle
    from paper_2501_04340_b200 import ietidp
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = make_bundle("C3r")
    owner = ietidp.shard_partition([float(len(sd["K_data"])) for sd in b["subs"]], world)
    # host-only handles (device = -1): validation, classification, ordering, symbolic analysis
    s = ietidp.shard_from_bundle(b, owner, rank, world, lambda ptr, n, stream: 0, device=-1)
    s.analyze()
    rep = s.report()
    nB = sum(len(b["subs"][k]["B_lambda"]) for k in s.global_ids)
    t = torch.tensor([rep["sum_nI"], rep["sum_nr"], rep["nnz_L"], rep["factor_flops"], nB, len(s.global_ids)],
                     dtype=torch.float64)
    dist.all_reduce(t)  # the data-path collective of the sharded design, here on its counts
    res = dict(total=t.tolist(), n_lambda=rep["n_lambda"], n_primal=rep["n_primal"])
    if rank == 0:
        full = ietidp.from_bundle(b, device=-1)
        full.analyze()
        res["full"] = full.report()
        # without sharded mode a one-sided multiplier row is a structure error
        part = ietidp.Solver(len(s.global_ids), b["n_lambda"], b["n_primal"], b["nrhs"], device=-1)
        for i, k in enumerate(s.global_ids):
            sd = b["subs"][k]
            part.set_subdomain(i, sd["K_indptr"], sd["K_indices"], sd["K_data"], sd["f"], sd["B_lambda"], sd["B_dof"],
                               sd["B_sign"], sd["tree"], sd["prim"], sd["prim_gid"])
        try:
            part.analyze()
            res["partial_status"] = 0
        except ietidp.IetiError as e:
            res["partial_status"] = e.status
    out[rank] = res
    dist.destroy_process_group()


def test_sharded_host_analysis_gloo_world2():
    """Two ranks analyse their shards of C3r (host-only handles) and all-reduce the counts:
    the shards' r_I slots, remaining DOFs, factor non-zeros and flops add up to the single
    handle's; every multiplier has its two sides somewhere (sum of local B entries = 2 m_r)."""
    import __graft_entry__
    __graft_entry__.build()
    world = 2
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_shard_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0]["total"] == out[1]["total"]
    sum_nI, sum_nr, nnz_L, flops, nB, nsub = out[0]["total"]
    full = out[0]["full"]
    assert sum_nI == full["sum_nI"] and sum_nr == full["sum_nr"]
    assert nnz_L == full["nnz_L"] and flops == full["factor_flops"]
    assert nB == 2 * full["n_lambda"] and nsub == full["n_sub"]
    assert out[0]["partial_status"] == 3  # IETIDP_E_B_STRUCTURE
