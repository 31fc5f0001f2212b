#!/usr/bin/env python
"""Benchmark of the B200 IETI-DP solve phase (BASELINE.json metric).

A step = one pass of the whole hot path on one synthetic
workload resident in HBM: batched multifrontal Cholesky of every K_rr^(k),
coarse set-up (K_rr^-1 K_rP, S_PP, G) and d_DP, the PCG loop on F_DP lambda = d_DP,
and the recovery of every u^(k). Host analysis (ordering/symbolic) and the
one-time upload happen before the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

value = solves per second over all ranks (N independent replicas, weak
scaling: the single-GPU design has no data-path exchange).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IETI-DP solve time, F-applies/s; % of FP64-TC peak (factor) and HBM (PCG)"
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fapply-iters", type=int, default=200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pre", action="store_true", help="skip the device pre-processing (f1) measurement")
    ap.add_argument("--shard-transport", default="nccl", choices=["nccl", "torch"],
                    help="--shard: ncclAllReduce called from the library (default) or torch.distributed through "
                         "the Python callback")
    ap.add_argument("--shard", action="store_true",
                    help="ONE workload split over the ranks by subdomain (include/ietidp_shard.h, NCCL all-reduce; "
                         "strong scaling) instead of one replica per rank")
    return ap.parse_args()


def oracle_flops(config):
    """sum_j c_j^2 of the local factors under the oracle's ordering (committed, offline)."""
    try:
        with open(os.path.join(ROOT, "profiles", "oracle_flops.json")) as f:
            return json.load(f).get(config, {}).get("useful_flops_oracle_ordering")
    except OSError:
        return None


def traffic_from_profiles(config):
    """DRAM traffic per PCG iteration of the persistent kernel, from the committed ncu
    --set full capture (profiles/<run>_raw.txt: dram__bytes_read.sum + write.sum of the
    whole k_pcg launch, divided by its iteration count); only for the captured config."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
    except OSError:
        return {}
    e = t.get(config)
    return e or {}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            out, _ = self.p.communicate(timeout=10)
            self.rows = [r.split(", ") for r in out.strip().splitlines() if r.strip()]
        else:
            self.rows = []

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world, device=None):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU oracle (the reported baseline; the one place bench.py runs oracle/)
# ---------------------------------------------------------------------------
def oracle_iters(config):
    """The oracle's own natural-stopping iteration count at full size (max over the
    columns measured): tests/golden/fullsize_<config>*.npz, written by
    tests/studies/make_fullsize_golden.py (oracle/ and ietigen/ only; C5 on columns 0
    and 7). None if not recorded (C1: the GPU run's own count is used)."""
    import glob
    its = []
    for p in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", f"fullsize_{config}*.npz"))):
        tail = os.path.basename(p)[len(f"fullsize_{config}"):-4]
        if tail and not tail.startswith("c"):
            continue  # fullsize_C2.npz must not match C20 etc.
        its.extend(int(x) for x in np.load(p)["iters"])
    return max(its) if its else None


def oracle_solve_cost(bundle, subs, n_iter, iters_sample=2):
    """Seconds of one full oracle solve (oracle/dp.py as it stands, on this host's
    cores), measured on a bounded sample: every per-subdomain phase is timed on the
    subdomains `subs` and scaled by n_sub / len(subs); every global phase is timed
    at full size. Phases (§2.1 order):
      set-up   per subdomain: Local (sparse LU of K_rr), K_rr^-1 K_rP, K_rr^-1 j_r,
               the explicit S_II = K_II - K_IV K_VV^-1 K_VI (Eq. 10);
               global: cho_factor of S_PP (n_gp x n_gp);
      PCG      `iters_sample` iterations of DualPrimal.pcg (F = W + G S^-1 G^T, M_D^-1,
               dot products and vector updates on the full n_lambda x nrhs vectors)
               over the sampled subdomains, split into the per-subdomain part and the
               global part (the same pcg with no subdomains), scaled to n_iter;
      recovery Eqs. (8)-(9): one K_rr^-1 solve per subdomain (+ the coarse solve).
    Returns (seconds, detail dict)."""
    import scipy.linalg as la
    import threadpoolctl
    from oracle import dp
    nl, ng, nc = int(bundle["n_lambda"]), int(bundle["n_primal"]), int(bundle["nrhs"])
    ns = len(bundle["subs"])
    scale = ns / len(subs)
    rng = np.random.default_rng(0)
    t0 = time.perf_counter()
    loc = []
    for k in subs:
        L = dp.Local(k, bundle["subs"][k], nl, False)
        L.X = L.Kinv(L.Krp.toarray()) if len(L.prim) else np.zeros((len(L.r), 0))
        L.y = L.Kinv(L.jr)
        L.SII = L.schur_II(False)
        loc.append(L)
    t_setup_local = time.perf_counter() - t0
    A = rng.standard_normal((ng, ng))
    Sg = A @ A.T + ng * np.eye(ng)
    t0 = time.perf_counter()
    Sc = la.cho_factor(Sg, lower=True) if ng else None
    t_setup_global = time.perf_counter() - t0

    def make(locs):
        D = dp.DualPrimal.__new__(dp.DualPrimal)
        D.nl, D.ng, D.nrhs, D.scaling = nl, ng, nc, bundle["scaling"]
        D.loc = locs
        D.G = rng.standard_normal((nl, ng))
        D.Sc = Sc
        for L in locs:  # the preconditioner's B_D (scaling weights: any, same cost)
            posI = -np.ones(len(L.r), np.int64)
            posI[L.rI] = np.arange(len(L.rI))
            L.B_Ipos = posI[L.B_rpos]
            L.delta = np.full(len(L.B_lambda), 0.5)
            import scipy.sparse as sp
            L.BD = sp.csr_matrix((L.B_sign * L.delta, (L.B_lambda, L.B_Ipos)), shape=(nl, len(L.rI)))
        return D

    d = rng.standard_normal((nl, nc))
    Ds, Dg = make(loc), make([])
    Dg.apply_M = lambda r: r.copy()  # no subdomains: keep the iteration finite (a copy's cost)

    def per_iter(D):
        # pcg with 1 and with 1 + iters_sample iterations: the difference is iters_sample
        # iterations (the start-up M-apply and the final true-residual F-apply cancel)
        t0 = time.perf_counter()
        D.pcg(tol=0.0, fixed_iters=1, d=d)
        t1 = time.perf_counter()
        D.pcg(tol=0.0, fixed_iters=1 + iters_sample, d=d)
        t2 = time.perf_counter()
        return max((t2 - t1) - (t1 - t0), 0.0) / iters_sample

    t_iter_sample = per_iter(Ds)
    t_iter_global = per_iter(Dg)
    t_iter_local = max(t_iter_sample - t_iter_global, 0.0)
    lam = rng.standard_normal((nl, nc))
    Ds.ftilde = rng.standard_normal((ng, nc))
    for L in loc:
        L.Cp = np.zeros((len(L.prim), ng))
    t0 = time.perf_counter()
    Ds.recover(lam)
    t_recover = time.perf_counter() - t0
    total = (t_setup_local * scale + t_setup_global + n_iter * (t_iter_local * scale + t_iter_global)
             + t_recover * scale)
    threads = max((i.get("num_threads", 1) for i in threadpoolctl.threadpool_info()), default=1)
    detail = {"setup_s": t_setup_local * scale + t_setup_global, "pcg_iter_s": t_iter_local * scale + t_iter_global,
              "recover_s": t_recover * scale, "n_iter": n_iter, "threads": threads,
              "sampled_subdomains": list(map(int, subs)), "scale": scale}
    return total, detail


def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"os_cpu_count": os.cpu_count(), "model": model}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from ietigen.bundle import make_bundle
    b = make_bundle(args.config)
    nsub = b["n_sub"]
    n_iter = oracle_iters(args.config) or 0
    per = 2  # subdomains sampled per step (rotating over the tiling)
    times, walls, det = [], [], None
    for s in range(args.warmup + args.steps):
        subs = [((s * per + i) * 7919) % nsub for i in range(per)]
        w0 = time.perf_counter()
        t, det = oracle_solve_cost(b, sorted(set(subs)), n_iter)
        if s >= args.warmup:
            times.append(t)
            walls.append(time.perf_counter() - w0)
    sec = statistics.mean(times)
    val = 1.0 / sec
    sample = (f"per step: oracle/dp.py on {per} of {nsub} subdomains (set-up: sparse LU of K_rr, K_rr^-1 K_rP, "
              f"explicit S_II; 2 PCG iterations with F, M_D^-1, coarse solve and vector updates; recovery), "
              f"per-subdomain phases scaled x{nsub / per:g}, global phases at full size, PCG scaled to the "
              f"oracle's own {n_iter} iterations (tests/golden/fullsize_*.npz)")
    ci = cpu_info()
    # ms_per_step is the wall time of one bounded sample (what this run actually spent per
    # step); value is the full solve rate the sample extrapolates to (ms_per_solve_extrapolated)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(walls) * 1e3,
            "ms_per_solve_extrapolated": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "n_sub": nsub, "n_lambda": int(b["n_lambda"]),
                       "n_primal": int(b["n_primal"]), "nrhs": int(b["nrhs"]),
                       "l2": "flushed between timed steps (512 MB write)", "replicas": world},
            "cpu_baseline": {"value": val, "unit": "solves/s", "cores": det["threads"], "kind": "oracle",
                             "sample": sample, "cpu": ci, "phases_s": det},
            "e2e": {"value": val, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def measure_dgemm_tflops(torch, dev):
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    best = 1e30
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2 * n ** 3 / (best * 1e-3) / 1e12


def measure_pre(ietidp, prob, device):
    """Device pre-processing (include/ietidp_pre.h) on the same workload,
    outside the timed solve: the tree-cotree gauge of the whole control graph and the batched
    assembly K = C^T M_2 C, j = C^T t of every box subdomain (device times from the library's
    CUDA events, best of three calls; results stay on the device)."""
    from ietigen import predesc
    g = predesc.gauge_desc(prob)
    for _ in range(2):
        tree, prim, g_ms = ietidp.pre_gauge(g["nv"], g["ne"], g["eu"], g["ev"], g["w"], device=device)
    descs = [predesc.subdomain_desc(prob, sd) for sd in prob.subs if len(sd.boxes) == 1]
    asm = None
    if descs:
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            _, info = ietidp.pre_assemble_batch(descs, device=device, fetch=False)
            info["wall_ms"] = (time.perf_counter() - t0) * 1e3
            if best is None or info["ms"] < best["ms"]:
                best = info
        pk = peaks().get("hbm_gbs", 6650.0)
        gbs = best["nnz"] * 12 / (best["ms_fill"] * 1e-3) / 1e9
        asm = {"subdomains": len(descs), "of": len(prob.subs), "nnz": int(best["nnz"]), "device_ms": best["ms"],
               "fill_kernel_ms": best["ms_fill"], "wall_ms_with_upload": best["wall_ms"],
               "roofline": {"kernel": "k_rows<1> (CSR columns and values of C^T M_2 C, all subdomains in one launch)",
                            "bound": "hbm", "achieved": gbs, "peak": pk, "unit": "GB/s", "frac": gbs / pk,
                            "algorithmic_bytes": int(best["nnz"]) * 12,
                            "note": "12 B written per CSR entry (value + column)"}}
    return {"gauge_ms": g_ms, "graph": {"nv": int(g["nv"]), "ne": int(g["ne"])},
            "tree_matches_generator": bool(np.array_equal(tree, prob.tree)), "assembly": asm}


def measure_e2e_device(ietidp, prob, b, local, stream, steps, world, dev):
    """End to end with the matrix never leaving the device (f1 feeding the hot path), the
    parameter-sweep case: per step new reluctivities go to the device (ietidp_pre_refill: nu per
    patch, the value kernel reruns in place), ietidp_set_values_device for every subdomain,
    factor, solve with lambda to the host, ietidp_get_u for every subdomain. The batch and a
    second handle on the device-assembled CSR pattern (the structural pattern of C^T M_2 C) are
    set up once."""
    import ctypes as C
    import torch
    from ietigen import predesc
    if any(len(sd.boxes) != 1 for sd in prob.subs):
        return None
    descs = [predesc.subdomain_desc(prob, sd) for sd in prob.subs]
    batch = ietidp.PreBatch(descs, device=local)
    S2 = ietidp.Solver(b["n_sub"], b["n_lambda"], b["n_primal"], b["nrhs"], scaling=b["scaling"], tol=b["tol"],
                       device=local, stream=stream.cuda_stream)
    for k, bs in enumerate(b["subs"]):
        o = batch.fetch(k)
        S2.set_subdomain(k, o["K_indptr"], o["K_indices"], o["K_data"], o["f"], bs["B_lambda"], bs["B_dof"], bs["B_sign"],
                         bs["tree"], bs["prim"], bs["prim_gid"])
    S2.analyze()
    nus = [d["nu"] for d in descs]
    nc = b["nrhs"]
    uo = [torch.empty((nc, sd["n"]), dtype=torch.float64).pin_memory() for sd in b["subs"]]
    lam_host = torch.empty((nc, b["n_lambda"]), dtype=torch.float64).pin_memory()
    h2d = sum(np.asarray(x).nbytes for x in nus)
    d2h = lam_host.numel() * 8 + sum(t.numel() * 8 for t in uo)
    rep_e = ietidp.Report()
    ets, asm_ms = [], []
    with torch.cuda.stream(stream):
        for it in range(2 + steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fill_ms = batch.refill(nus)
            for k in range(b["n_sub"]):
                S2.set_values_device(k, *batch.device_ptrs(k))
            S2.factor()
            S2._check(S2.lib.ietidp_solve(S2.h, C.c_void_p(lam_host.data_ptr()), C.byref(rep_e)))
            for k in range(b["n_sub"]):
                S2._check(S2.lib.ietidp_get_u(S2.h, k, C.c_void_p(uo[k].data_ptr())))
            dt = time.perf_counter() - t0
            if it >= 2:
                ets.append(dt)
                asm_ms.append(fill_ms)
    batch.close()
    S2.close()
    e2e_s = max_over_ranks(statistics.mean(ets), world, dev)
    return {"value": world / e2e_s, "unit": "solves/s", "ms_per_step": e2e_s * 1e3, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "assembly_kernels_ms": statistics.mean(asm_ms), "iters": max(rep_e.iters[:nc]),
            "note": "per step: new nu per patch to the device (the H2D bytes), the value kernel of the batched device "
                    "assembly (ietidp_pre_refill), ietidp_set_values_device (device to device), factor, solve with "
                    "lambda to the host, ietidp_get_u for every subdomain"}


def run_sharded(args, rank, world, local):
    """ONE workload over all ranks: rank r owns a contiguous, nnz(K)-balanced
    range of subdomains (ietidp_shard_partition) and the ranks exchange g, q, z per iteration
    through torch.distributed (NCCL) on the library's stream. value = solves/s of the whole
    job (max over ranks), scaling strong. With one rank this times the launch-by-launch
    sharded code path (no persistent kernel) with a one-rank all-reduce."""
    import torch
    import torch.distributed as dist
    from ietigen.bundle import make_bundle
    from paper_2501_04340_b200 import ietidp

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world)
    b = make_bundle(args.config)
    owner = ietidp.shard_partition([float(len(sd["K_data"])) for sd in b["subs"]], world)
    stream = torch.cuda.Stream(device=dev)
    comm = ietidp.NcclComm(rank, world, local) if args.shard_transport == "nccl" else ietidp.nccl_allreduce(local)
    S = ietidp.shard_from_bundle(b, owner, rank, world, comm, device=local, stream=stream.cuda_stream)
    S.analyze()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            S.factor()
            S.solve(want_lambda=False)
        torch.cuda.synchronize()
        dist.barrier()
        times = []
        with Clocks(local) as clk:
            for _ in range(args.steps):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                dist.barrier()
                e0, e1 = ev(), ev()
                e0.record(stream)
                S.factor()
                _, rep = S.solve(want_lambda=False)
                e1.record(stream)
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
        dist.barrier()
    ms_step = max_over_ranks(statistics.mean(times), world, dev) if world > 1 else statistics.mean(times)
    if rank != 0:
        return
    it_max = max(rep["iters"])
    line = {
        "metric": METRIC, "value": 1.0 / (ms_step * 1e-3), "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "n_sub": b["n_sub"], "n_lambda": b["n_lambda"],
                   "n_primal": b["n_primal"], "nrhs": b["nrhs"], "l2": "flushed between timed steps (512 MB write)",
                   "parallelism": f"subdomains sharded over {world} rank(s), all-reduce of g, q, z per iteration"},
        "phases_ms": {"factor": rep["ms_factor"], "coarse_rhs": rep["ms_coarse"], "pcg": rep["ms_pcg"],
                      "recover": rep["ms_recover"]},
        "iters": rep["iters"], "rel_residual": max(rep["rel_residual"]),
        "shard": {"subdomains_per_rank": np.bincount(owner, minlength=world).tolist(),
                  "allreduce_doubles_per_iteration": int((2 * b["n_lambda"] + b["n_primal"]) * b["nrhs"]),
                  "us_per_iteration": rep["ms_pcg"] / max(it_max, 1) * 1e3,
                  "transport": "ncclAllReduce from the library, on its stream" if args.shard_transport == "nccl"
                  else "torch.distributed all_reduce through the Python callback",
                  "loop": "host-driven, launch by launch (the persistent kernel's grid barrier cannot span GPUs)"},
        "clocks": clk.summary(), "gpu_launches": int(S.kernel_launches() // max(args.steps + args.warmup, 1)),
        "roofline": None, "e2e": None, "cpu_baseline": None,
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
    import torch
    from ietigen.bundle import make_bundle
    from paper_2501_04340_b200 import ietidp

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    b, prob = make_bundle(args.config, with_problem=True)
    stream = torch.cuda.Stream(device=dev)
    t0 = time.perf_counter()
    S = ietidp.from_bundle(b, device=local, stream=stream.cuda_stream)
    t1 = time.perf_counter()
    S.analyze()
    t2 = time.perf_counter()
    ms_set_sub, ms_analyze = (t1 - t0) * 1e3, (t2 - t1) * 1e3
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def step():
        S.factor()
        return S.solve(want_lambda=False)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        barrier(world)
        launches0 = S.kernel_launches()
        times, reps = [], []
        with Clocks(local) as clk:
            t_wall = time.perf_counter()
            for _ in range(args.steps):
                flush.fill_(1.0)  # L2 flush between timed steps (not timed)
                torch.cuda.synchronize()
                e0, e1 = ev(), ev()
                e0.record(stream)
                _, rep = step()
                e1.record(stream)
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
                reps.append(rep)
            t_wall = time.perf_counter() - t_wall
        torch.cuda.synchronize()
        barrier(world)
        launches = (S.kernel_launches() - launches0) // max(args.steps, 1)
        # condition estimate of M_D^-1 F_DP from the last timed solve's PCG coefficients
        # (untimed, like the paper's own estimate)
        with torch.cuda.stream(stream):
            c_lo, c_hi, c_k = S.estimate_condition()
        ms_step = max_over_ranks(statistics.mean(times), world, dev)
        rep = reps[-1]

        # ---- F-applies/s (operator loop alone, ncols = nrhs) ----
        nc = b["nrhs"]
        x = torch.randn(nc, b["n_lambda"], dtype=torch.float64, device=dev)
        y = torch.empty_like(x)
        for _ in range(5):
            S.apply_F_device(x, y, nc)
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(args.fapply_iters):
            S.apply_F_device(x, y, nc)
        e1.record(stream)
        torch.cuda.synchronize()
        fa_ms = e0.elapsed_time(e1) / args.fapply_iters
        f_apply_per_s = nc / (fa_ms * 1e-3)

        # ---- end-to-end through the C-ABI with host buffers ----
        e2e = None
        if not args.no_e2e:
            # the lower-triangle values (ietidp_set_values_lower: K is symmetric, half the bytes)
            def lower(sd):
                ip, ix = sd["K_indptr"], sd["K_indices"]
                rows = np.repeat(np.arange(len(ip) - 1), np.diff(ip))
                return np.ascontiguousarray(sd["K_data"][ix <= rows])
            kv = [torch.from_numpy(lower(sd)).pin_memory() for sd in b["subs"]]
            fv = [torch.from_numpy(np.ascontiguousarray(sd["f"])).pin_memory() for sd in b["subs"]]
            uo = [torch.empty((nc, sd["n"]), dtype=torch.float64).pin_memory() for sd in b["subs"]]
            lam_host = torch.empty((nc, b["n_lambda"]), dtype=torch.float64).pin_memory()
            import ctypes as C
            h2d = sum(t.numel() * 8 for t in kv) + sum(t.numel() * 8 for t in fv)
            d2h = lam_host.numel() * 8 + sum(t.numel() * 8 for t in uo)
            ets = []
            rep_e = ietidp.Report()
            for it in range(2 + args.steps):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for k in range(b["n_sub"]):
                    S._check(S.lib.ietidp_set_values_lower(S.h, k, C.c_void_p(kv[k].data_ptr()),
                                                           C.c_void_p(fv[k].data_ptr())))
                S.factor()
                S._check(S.lib.ietidp_solve(S.h, C.c_void_p(lam_host.data_ptr()), C.byref(rep_e)))
                for k in range(b["n_sub"]):
                    S._check(S.lib.ietidp_get_u(S.h, k, C.c_void_p(uo[k].data_ptr())))
                dt = time.perf_counter() - t0
                if it >= 2:
                    ets.append(dt)
            e2e_s = max_over_ranks(statistics.mean(ets), world, dev)
            once = (ms_set_sub + ms_analyze) * 1e-3
            e2e = {"value": world / e2e_s, "unit": "solves/s", "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3,
                   "note": "per step: ietidp_set_values_lower (lower-triangle K values + loads, pinned H2D) "
                           "for every subdomain, "
                           "factor, solve with lambda to the host, ietidp_get_u for every subdomain",
                   "with_analysis": {"value": world / (e2e_s + once), "unit": "solves/s",
                                     "ms_set_subdomain": ms_set_sub, "ms_analyze": ms_analyze,
                                     "note": "one solve including the host set-up (ietidp_set_subdomain "
                                             "validation/copies) and the symbolic analysis"}}

        fp64_peak = measure_dgemm_tflops(torch, dev) if rank == 0 else None
        pre = measure_pre(ietidp, prob, local) if (rank == 0 and not args.no_pre) else None
        e2e_dev = None
        if e2e is not None and not args.no_pre:
            e2e_dev = measure_e2e_device(ietidp, prob, b, local, stream, args.steps, world, dev)
            e2e["device_assembly"] = e2e_dev

    if rank != 0:
        return
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    it_max = max(rep["iters"])
    pcg_bytes = rep["pcg_bytes_per_iter"] * 1.0
    pcg_ms_iter = rep["ms_pcg"] / max(it_max, 1)
    pcg_gbs = pcg_bytes / (pcg_ms_iter * 1e-3) / 1e9 if it_max else 0.0
    # useful flops: min(sum c_j^2 under our ordering, the same count under
    # the oracle's reference ordering -- profiles/oracle_flops.json, tools/oracle_flops.py)
    ofl = oracle_flops(args.config)
    useful = min(rep["factor_flops"], ofl) if ofl else rep["factor_flops"]
    fac_tflops = useful / (rep["ms_factor"] * 1e-3) / 1e12
    # one apply streams the W_k tiles once for all nc columns
    fa_gbs = rep["f_apply_bytes"] / (fa_ms * 1e-3) / 1e9
    phases = {"factor": rep["ms_factor"], "coarse_rhs": rep["ms_coarse"], "pcg": rep["ms_pcg"],
              "recover": rep["ms_recover"]}
    dominant = max(phases, key=phases.get)
    tr = traffic_from_profiles(args.config)
    # PCG: two symmetric passes per iteration (W_k = S_II^-1 for F, S_II for M_D^-1), each
    # y = S x on nc columns: 2 |r_I|^2 nc flops per subdomain and pass; the
    # bytes are the stored lower tiles. The binding roofline is the larger floor: HBM for
    # one column, the FP64 tensor pipe (DMMA) for 16 columns.
    sum_nI2 = sum(float(len(np.unique(sd["B_dof"]))) ** 2 for sd in b["subs"])
    pcg_flops = 2 * 2.0 * sum_nI2 * nc
    pcg_tflops = pcg_flops / (pcg_ms_iter * 1e-3) / 1e12 if it_max else 0.0
    t_hbm = pcg_bytes / (hbm * 1e9)
    t_fp = pcg_flops / (fp64_peak * 1e12) if fp64_peak else 0.0
    pcg_kernel = ("persistent PCG kernel k_pcg (W_k and S_II symmetric tile passes, gathers, coarse "
                  "solve, CG updates) per iteration")
    if t_fp > t_hbm:
        roof_pcg = {"kernel": pcg_kernel, "bound": "tensor", "achieved": pcg_tflops, "peak": fp64_peak,
                    "unit": "TFLOP/s", "frac": pcg_tflops / fp64_peak,
                    "algorithmic_flops_per_iter": pcg_flops,
                    "hbm": {"achieved": pcg_gbs, "peak": hbm, "unit": "GB/s", "frac": pcg_gbs / hbm},
                    "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (FP64 tensor pipe, DMMA)"}
    else:
        roof_pcg = {"kernel": pcg_kernel, "bound": "hbm", "achieved": pcg_gbs, "peak": hbm, "unit": "GB/s",
                    "frac": pcg_gbs / hbm,
                    "tensor": {"achieved": pcg_tflops, "peak": fp64_peak, "unit": "TFLOP/s",
                               "frac": pcg_tflops / fp64_peak if fp64_peak else None}}
    roof_pcg.update({"traffic": tr.get("pcg_bytes_per_iter"), "traffic_source": tr.get("pcg_source"),
                     "algorithmic_bytes_per_iter": int(pcg_bytes), "us_per_iter": pcg_ms_iter * 1e3,
                     "floors_us": {"hbm": t_hbm * 1e6, "tensor": t_fp * 1e6}})
    roof_fac = {"kernel": "multifrontal Cholesky phase (k_gemm DMMA panel updates / TRSM / SYRK+extend-add, "
                          "k_potrf, assembly; side stream: L11^-1, W_k, forward sweep)",
                "bound": "tensor", "achieved": fac_tflops, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": fac_tflops / fp64_peak if fp64_peak else None, "traffic": None,
                "useful_flops": useful, "flops_our_ordering": rep["factor_flops"],
                "flops_oracle_ordering": ofl,
                "flops_note": "useful = min(our nested-dissection count, SuperLU MMD count of the oracle); "
                              "ours is higher: the r_I block is ordered last and our separators are thick",
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run"}
    roofline = roof_fac if dominant == "factor" else roof_pcg
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        ns = b["n_sub"]
        nsamp = min(ns, 8)
        subs = sorted(set(int(round(i * (ns - 1) / max(nsamp - 1, 1))) for i in range(nsamp)))
        n_or = oracle_iters(args.config)
        sec, det = oracle_solve_cost(b, subs, n_or or it_max)
        cpu = {"value": 1.0 / sec, "unit": "solves/s", "cores": det["threads"], "kind": "oracle",
               "sample": f"oracle/dp.py on {len(subs)} of {ns} subdomains evenly spaced over the tiling (set-up: "
                         f"sparse LU of K_rr, K_rr^-1 K_rP, K_rr^-1 j, explicit S_II; 2 PCG iterations with F, "
                         f"M_D^-1, coarse solve and vector updates on all {nc} columns; recovery), per-subdomain "
                         f"phases scaled x{ns / len(subs):g}, global phases at full size, PCG scaled to "
                         + (f"the oracle's own {n_or} iterations (tests/golden/fullsize_*.npz)" if n_or else
                            f"the GPU run's {it_max} iterations"),
               "cpu": cpu_info(), "phases_s": det}
    line = {
        "metric": METRIC, "value": world / (ms_step * 1e-3), "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "n_sub": b["n_sub"], "n_lambda": b["n_lambda"],
                   "n_primal": b["n_primal"], "nrhs": nc, "l2": "flushed between timed steps (512 MB write)",
                   "replicas": world},
        "phases_ms": phases, "ms_analyze": rep["ms_analyze"], "ms_upload": rep["ms_upload"],
        "ms_analyze_call": ms_analyze, "ms_set_subdomain": ms_set_sub,
        "analyze_note": "ms_analyze = host symbolic analysis (report); ms_upload = device allocation, "
                        "value upload and scatter-list expansion; ms_analyze_call = wall time of "
                        "ietidp_analyze (both)", "iters": rep["iters"], "rel_residual": max(rep["rel_residual"]),
        "cond_estimate": {"omega_min": float(min(c_lo)), "omega_max": float(max(c_hi)),
                          "cond_max": float(max(c_k)), "method": "Lanczos from the PCG alpha/beta (device)"},
        "f_applies_per_s": f_apply_per_s, "f_apply_us": fa_ms * 1e3, "f_apply_gbs": fa_gbs,
        "f_apply_tflops": 2.0 * sum_nI2 * nc / (fa_ms * 1e-3) / 1e12,
        "f_apply_note": "ietidp_apply_F alone, all %d columns per call (explicit loop: W_k tiles %.0f MB streamed once "
                        "per call; L2 126 MB); f_apply_gbs = tile bytes / call time, f_apply_tflops = 2 sum|r_I|^2 ncols "
                        "/ call time" % (nc, rep["f_apply_bytes"] / 1e6),
        "roofline": roofline, "rooflines": {"factor": roof_fac, "pcg": roof_pcg},
        "fp64_dgemm_tflops": fp64_peak, "clocks": clk.summary(), "gpu_launches": int(launches),
        "e2e": e2e, "cpu_baseline": cpu, "pre": pre,
        "symbolic": {"n_supernodes": rep["n_supernodes"], "n_levels": rep["n_levels"], "max_front": rep["max_front"],
                     "nnz_L": rep["nnz_L"], "factor_flops": rep["factor_flops"]},
        "wall_s": t_wall,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.shard:
        run_sharded(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)
    if world > 1 or args.shard:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
