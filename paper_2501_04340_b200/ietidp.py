"""Thin ctypes binding of libietidp.so (include/ietidp.h): argument marshalling
only — every numeric step runs in the library's CUDA kernels. There is no CPU
fallback: if the library is missing or no CUDA device is present the calls
fail loudly.
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libietidp.so")
# IETIDP_LIB: path of another build of the same library (A/B comparisons in tools/)
LIB_PATH = os.environ.get("IETIDP_LIB", LIB_PATH)

MAX_RHS = 64
STATUS = {0: "IETIDP_OK", 1: "IETIDP_E_ARG", 2: "IETIDP_E_STATE", 3: "IETIDP_E_B_STRUCTURE",
          4: "IETIDP_E_NOT_SPD", 5: "IETIDP_E_NO_CONVERGENCE", 6: "IETIDP_E_CUDA", 7: "IETIDP_E_NOMEM"}
OK, E_ARG, E_STATE, E_B_STRUCTURE, E_NOT_SPD, E_NO_CONVERGENCE, E_CUDA, E_NOMEM = range(8)
SCALING = {"multiplicity": 0, "stiffness": 1}
ORDERING = {"nd": 0, "dense": 1, "md": 2}
LOOP = {"explicit": 0, "triangular": 1}
STOP = {"residual": 0, "preconditioned": 1}

# every entry point include/ietidp.h declares
SYMBOLS = ["ietidp_options_default", "ietidp_create", "ietidp_set_subdomain", "ietidp_analyze",
           "ietidp_set_values", "ietidp_set_values_device", "ietidp_set_values_lower", "ietidp_factor", "ietidp_solve", "ietidp_get_u", "ietidp_get_u_device",
           "ietidp_get_lambda_device", "ietidp_apply_F", "ietidp_apply_precond", "ietidp_get_coarse",
           "ietidp_estimate_condition", "ietidp_get_pcg_coefficients", "ietidp_get_rhs", "ietidp_get_report", "ietidp_kernel_launches", "ietidp_last_error",
           "ietidp_status_string", "ietidp_destroy"]
# every entry point include/ietidp_pre.h declares (device pre-processing)
PRE_SYMBOLS = ["ietidp_pre_assemble", "ietidp_pre_assemble_batch", "ietidp_pre_device_ptrs", "ietidp_pre_refill", "ietidp_pre_sizes", "ietidp_pre_get", "ietidp_pre_get_gram",
               "ietidp_pre_last_error", "ietidp_pre_destroy", "ietidp_pre_gauge"]


class Options(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("scaling", C.c_int), ("fixed_iters", C.c_int),
                ("ordering", C.c_int), ("leaf_size", C.c_int), ("loop", C.c_int), ("stop", C.c_int),
                ("device", C.c_int),
                ("stream", C.c_void_p)]


# every entry point include/ietidp_shard.h declares (sharded multi-GPU solve)
SHARD_SYMBOLS = ["ietidp_shard_enable", "ietidp_shard_enable_nccl", "ietidp_shard_partition"]
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class PreSubdomain(C.Structure):
    """ietidp_pre_subdomain (include/ietidp_pre.h)."""
    _fields_ = [("p", C.c_int), ("e", C.c_int), ("npatch", C.c_int * 3), ("knots", C.c_void_p * 3),
                ("nq", C.c_int), ("qx", C.c_void_p * 3), ("qw", (C.c_void_p * 3) * 3), ("nu", C.c_void_p),
                ("dof_of_edge", C.c_void_p), ("n_dof", C.c_int), ("nrhs", C.c_int), ("lq", C.c_int),
                ("lx", C.c_void_p * 3), ("nfac", C.c_int * 3), ("fac_kind", C.c_void_p * 3),
                ("fac_val", C.c_void_p * 3), ("nterms", C.c_int), ("term_col", C.c_void_p),
                ("term_comp", C.c_void_p), ("term_fac", C.c_void_p), ("term_coef", C.c_void_p)]


class Report(C.Structure):
    _fields_ = [("n_sub", C.c_int), ("n_lambda", C.c_int), ("n_primal", C.c_int), ("nrhs", C.c_int),
                ("failed_subdomain", C.c_int), ("n_supernodes", C.c_int), ("n_levels", C.c_int),
                ("max_front", C.c_int), ("max_nI", C.c_int),
                ("sum_nr", C.c_longlong), ("sum_nI", C.c_longlong), ("nnz_L", C.c_longlong),
                ("factor_flops", C.c_longlong), ("pcg_bytes_per_iter", C.c_longlong),
                ("f_apply_bytes", C.c_longlong),
                ("iters", C.c_int * MAX_RHS), ("converged", C.c_int * MAX_RHS),
                ("rel_residual", C.c_double * MAX_RHS),
                ("ms_analyze", C.c_double), ("ms_factor", C.c_double), ("ms_coarse", C.c_double),
                ("ms_pcg", C.c_double), ("ms_recover", C.c_double), ("ms_upload", C.c_double),
                ("n_pattern_classes", C.c_int)]

    def to_dict(self):
        n = self.nrhs
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("iters", "converged", "rel_residual")}
        d["iters"] = list(self.iters[:n])
        d["converged"] = list(self.converged[:n])
        d["rel_residual"] = list(self.rel_residual[:n])
        return d


_lib = None


def load():
    """Load libietidp.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2501_04340_b200.build`")
    lib = C.CDLL(LIB_PATH)
    P, I, D, LL = C.c_void_p, C.c_int, C.c_double, C.c_longlong
    sig = {
        "ietidp_options_default": (None, [C.POINTER(Options)]),
        "ietidp_create": (I, [C.POINTER(Options), I, I, I, I, C.POINTER(P)]),
        "ietidp_set_subdomain": (I, [P, I, I, P, P, P, P, I, P, P, P, I, P, I, P, P]),
        "ietidp_analyze": (I, [P]),
        "ietidp_set_values": (I, [P, I, P, P]),
        "ietidp_set_values_lower": (I, [P, I, P, P]),
        "ietidp_set_values_device": (I, [P, I, P, P]),
        "ietidp_factor": (I, [P]),
        "ietidp_solve": (I, [P, P, C.POINTER(Report)]),
        "ietidp_get_u": (I, [P, I, P]),
        "ietidp_get_u_device": (I, [P, I, P]),
        "ietidp_get_lambda_device": (I, [P, P]),
        "ietidp_apply_F": (I, [P, I, P, P]),
        "ietidp_apply_precond": (I, [P, I, P, P]),
        "ietidp_get_coarse": (I, [P, P]),
        "ietidp_estimate_condition": (I, [P, P, P, P]),
        "ietidp_get_pcg_coefficients": (I, [P, I, P, P]),
        "ietidp_get_rhs": (I, [P, P]),
        "ietidp_get_report": (I, [P, C.POINTER(Report)]),
        "ietidp_kernel_launches": (LL, [P]),
        "ietidp_last_error": (C.c_char_p, [P]),
        "ietidp_status_string": (C.c_char_p, [I]),
        "ietidp_destroy": (None, [P]),
        "ietidp_shard_enable": (I, [P, I, I, ALLREDUCE_FN, P]),
        "ietidp_shard_enable_nccl": (I, [P, I, I, P, P]),
        "ietidp_shard_partition": (I, [I, P, I, P]),
        "ietidp_pre_assemble": (I, [I, C.POINTER(PreSubdomain), C.POINTER(P)]),
        "ietidp_pre_assemble_batch": (I, [I, I, C.POINTER(PreSubdomain), C.POINTER(P)]),
        "ietidp_pre_device_ptrs": (I, [P, C.POINTER(P), C.POINTER(P)]),
        "ietidp_pre_refill": (I, [P, P, C.POINTER(D)]),
        "ietidp_pre_sizes": (I, [P, C.POINTER(I), C.POINTER(C.c_int64), C.POINTER(D), C.POINTER(D)]),
        "ietidp_pre_get": (I, [P, P, P, P, P]),
        "ietidp_pre_get_gram": (I, [P, I, I, I, P, C.POINTER(I)]),
        "ietidp_pre_last_error": (C.c_char_p, []),
        "ietidp_pre_destroy": (None, [P]),
        "ietidp_pre_gauge": (I, [I, C.c_int64, C.c_int64, P, P, P, P, P, C.POINTER(D)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class IetiError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


class Solver:
    """One IETI-DP handle (include/ietidp.h). Host numpy arrays in, host arrays out;
    the *_device methods take torch CUDA tensors (plumbing only)."""

    def __init__(self, n_sub, n_lambda, n_primal, nrhs=1, tol=1e-10, max_iter=500, scaling="multiplicity",
                 fixed_iters=0, ordering="nd", leaf_size=96, loop="explicit", stop="residual", device=0,
                 stream=None):
        lib = load()
        self.lib = lib
        o = Options()
        lib.ietidp_options_default(C.byref(o))
        o.tol, o.max_iter, o.scaling, o.fixed_iters = tol, max_iter, SCALING[scaling], fixed_iters
        o.ordering, o.leaf_size, o.loop, o.device = ORDERING[ordering], leaf_size, LOOP[loop], device
        o.stop = STOP[stop]
        o.stream = stream
        h = C.c_void_p()
        st = lib.ietidp_create(C.byref(o), n_sub, n_lambda, n_primal, nrhs, C.byref(h))
        self.h = h
        self.n_sub, self.n_lambda, self.n_primal, self.nrhs = n_sub, n_lambda, n_primal, nrhs
        self._n = [0] * n_sub
        self._keep = []
        self._check(st)

    def _check(self, st, allow=()):
        if st != OK and st not in allow:
            msg = self.lib.ietidp_last_error(self.h).decode() if self.h else ""
            raise IetiError(st, msg)
        return st

    def set_subdomain(self, k, K_indptr, K_indices, K_data, f, B_lambda, B_dof, B_sign, tree, prim, prim_gid):
        a = dict(ip=np.ascontiguousarray(K_indptr, np.int64), ix=np.ascontiguousarray(K_indices, np.int32),
                 v=np.ascontiguousarray(K_data, np.float64), f=np.ascontiguousarray(f, np.float64),
                 bl=np.ascontiguousarray(B_lambda, np.int32), bd=np.ascontiguousarray(B_dof, np.int32),
                 bs=np.ascontiguousarray(B_sign, np.int8), tr=np.ascontiguousarray(tree, np.int32),
                 pr=np.ascontiguousarray(prim, np.int32), pg=np.ascontiguousarray(prim_gid, np.int32))
        n = len(a["ip"]) - 1
        self._n[k] = n
        st = self.lib.ietidp_set_subdomain(self.h, k, n, _ptr(a["ip"]), _ptr(a["ix"]), _ptr(a["v"]), _ptr(a["f"]),
                                           len(a["bl"]), _ptr(a["bl"]), _ptr(a["bd"]), _ptr(a["bs"]),
                                           len(a["tr"]), _ptr(a["tr"]), len(a["pr"]), _ptr(a["pr"]), _ptr(a["pg"]))
        self._check(st)

    def shard_enable(self, rank, nranks, allreduce):
        """Sharded mode (include/ietidp_shard.h): this handle holds rank's subdomains only;
        allreduce(ptr, n, stream) sums the device buffer of n doubles at ptr over the ranks in
        place (raise or return non-zero on failure)."""
        def thunk(ctx, ptr, n, stream):
            try:
                rc = allreduce(ptr, n, stream)
                return int(rc or 0)
            except Exception:  # never unwind through the C frames
                import traceback
                traceback.print_exc()
                return 1
        self._allreduce = ALLREDUCE_FN(thunk)  # keep the trampoline alive with the handle
        self._check(self.lib.ietidp_shard_enable(self.h, rank, nranks, self._allreduce, None))

    def shard_enable_nccl(self, rank, nranks, comm):
        """Sharded mode with the native NCCL transport: comm = NcclComm (below)."""
        self._nccl = comm
        self._check(self.lib.ietidp_shard_enable_nccl(self.h, rank, nranks, comm.comm, comm.allreduce_addr))

    def analyze(self):
        self._check(self.lib.ietidp_analyze(self.h))

    def set_values(self, k, K_data=None, f=None):
        v = None if K_data is None else np.ascontiguousarray(K_data, np.float64)
        ff = None if f is None else np.ascontiguousarray(f, np.float64)
        self._check(self.lib.ietidp_set_values(self.h, k, _ptr(v), _ptr(ff)))

    def set_values_lower(self, k, K_lower=None, f=None):
        """Values of the lower-triangle entries (j <= i) of subdomain k's CSR pattern, in
        CSR order (ietidp_set_values_lower: half the bytes of set_values)."""
        v = None if K_lower is None else np.ascontiguousarray(K_lower, np.float64)
        ff = None if f is None else np.ascontiguousarray(f, np.float64)
        self._check(self.lib.ietidp_set_values_lower(self.h, k, _ptr(v), _ptr(ff)))

    def set_values_device(self, k, d_val_ptr=None, d_f_ptr=None):
        """ietidp_set_values_device: raw device pointers (ints), e.g. of a PreBatch."""
        self._check(self.lib.ietidp_set_values_device(self.h, k, C.c_void_p(d_val_ptr) if d_val_ptr else None,
                                                      C.c_void_p(d_f_ptr) if d_f_ptr else None))

    def factor(self):
        self._check(self.lib.ietidp_factor(self.h))

    def solve(self, want_lambda=True, allow_noconv=False):
        lam = np.zeros((self.nrhs, self.n_lambda)) if want_lambda else None
        rep = Report()
        st = self.lib.ietidp_solve(self.h, _ptr(lam), C.byref(rep))
        self._check(st, allow=(E_NO_CONVERGENCE,) if allow_noconv else ())
        return (lam.T.copy() if want_lambda else None), rep.to_dict()

    def get_u(self, k):
        u = np.zeros((self.nrhs, self._n[k]))
        self._check(self.lib.ietidp_get_u(self.h, k, _ptr(u)))
        return u.T.copy()

    def get_coarse(self):
        S = np.zeros((self.n_primal, self.n_primal))
        self._check(self.lib.ietidp_get_coarse(self.h, _ptr(S)))
        return S

    def estimate_condition(self):
        """(omega_min, omega_max, cond) per column of the last solve, from
        the Lanczos tridiagonal of the PCG coefficients, computed on the device."""
        n = self.nrhs
        lo, hi, k = (np.zeros(n) for _ in range(3))
        self._check(self.lib.ietidp_estimate_condition(self.h, _ptr(lo), _ptr(hi), _ptr(k)))
        return lo, hi, k

    def pcg_coefficients(self, ld):
        """alpha, beta of the last solve: arrays (nrhs, ld), zero beyond each column's count."""
        a = np.zeros((self.nrhs, ld))
        b = np.zeros((self.nrhs, ld))
        self._check(self.lib.ietidp_get_pcg_coefficients(self.h, ld, _ptr(a), _ptr(b)))
        return a, b

    def get_rhs(self):
        d = np.zeros((self.nrhs, self.n_lambda))
        self._check(self.lib.ietidp_get_rhs(self.h, _ptr(d)))
        return d.T.copy()

    def report(self):
        rep = Report()
        self._check(self.lib.ietidp_get_report(self.h, C.byref(rep)))
        return rep.to_dict()

    def kernel_launches(self):
        return int(self.lib.ietidp_kernel_launches(self.h))

    # --- device operator access (torch CUDA tensors, n_lambda x ncols column-major) ---
    def apply_F_device(self, x, y, ncols):
        self._check(self.lib.ietidp_apply_F(self.h, ncols, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr())))

    def apply_precond_device(self, x, y, ncols):
        self._check(self.lib.ietidp_apply_precond(self.h, ncols, C.c_void_p(x.data_ptr()),
                                                  C.c_void_p(y.data_ptr())))

    def get_u_device(self, k, out):
        self._check(self.lib.ietidp_get_u_device(self.h, k, C.c_void_p(out.data_ptr())))

    def get_lambda_device(self, out):
        self._check(self.lib.ietidp_get_lambda_device(self.h, C.c_void_p(out.data_ptr())))

    def apply_F(self, X):
        """Host convenience: y = F_DP X for X (n_lambda x ncols), via the device entry point."""
        return self._host_op(X, self.apply_F_device)

    def apply_precond(self, X):
        return self._host_op(X, self.apply_precond_device)

    def _host_op(self, X, fn):
        import torch
        X = np.asarray(X, np.float64)
        if X.ndim == 1:
            X = X[:, None]
        ncols = X.shape[1]
        xt = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
        yt = torch.empty_like(xt)
        fn(xt, yt, ncols)
        torch.cuda.synchronize()
        return yt.cpu().numpy().T.copy()

    def close(self):
        if self.h:
            self.lib.ietidp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def from_bundle(b, **opts):
    """A Solver with every subdomain of a generator bundle (ietigen.bundle) set."""
    opts.setdefault("scaling", b["scaling"])
    opts.setdefault("tol", b["tol"])
    s = Solver(b["n_sub"], b["n_lambda"], b["n_primal"], b["nrhs"], **opts)
    for k, sd in enumerate(b["subs"]):
        s.set_subdomain(k, sd["K_indptr"], sd["K_indices"], sd["K_data"], sd["f"], sd["B_lambda"], sd["B_dof"],
                        sd["B_sign"], sd["tree"], sd["prim"], sd["prim_gid"])
    return s


# ---- device pre-processing (include/ietidp_pre.h): marshalling only ----

def _pre_check(lib, st):
    if st != OK:
        raise IetiError(st, lib.ietidp_pre_last_error().decode())


def _pre_fill(s, desc, keep):
    def arr(a, dt):
        a = np.ascontiguousarray(a, dt)
        keep.append(a)
        return a.ctypes.data if a.size else None

    s.p, s.e, s.nq, s.n_dof, s.nrhs, s.lq = desc["p"], desc["e"], desc["nq"], desc["n_dof"], desc["nrhs"], desc["lq"]
    for a in range(3):
        s.npatch[a] = desc["npatch"][a]
        s.knots[a] = arr(desc["knots"][a], np.float64)
        s.qx[a] = arr(desc["qx"][a], np.float64)
        s.lx[a] = arr(desc["lx"][a], np.float64)
        s.nfac[a] = len(desc["fac_kind"][a])
        s.fac_kind[a] = arr(desc["fac_kind"][a], np.int32)
        s.fac_val[a] = arr(desc["fac_val"][a], np.float64)
        for c in range(3):
            s.qw[c][a] = arr(desc["qw"][c][a], np.float64)
    s.nu = arr(desc["nu"], np.float64)
    s.dof_of_edge = arr(desc["dof_of_edge"], np.int32)
    s.nterms = len(desc["term_coef"])
    s.term_col = arr(desc["term_col"], np.int32)
    s.term_comp = arr(desc["term_comp"], np.int32)
    s.term_fac = arr(desc["term_fac"], np.int32)
    s.term_coef = arr(desc["term_coef"], np.float64)


def _pre_fetch(lib, h, desc, want_gram):
    n, nnz, ms, msf = C.c_int(), C.c_int64(), C.c_double(), C.c_double()
    _pre_check(lib, lib.ietidp_pre_sizes(h, C.byref(n), C.byref(nnz), C.byref(ms), C.byref(msf)))
    ip = np.zeros(n.value + 1, np.int64)
    ix = np.zeros(nnz.value, np.int32)
    v = np.zeros(nnz.value, np.float64)
    f = np.zeros((desc["nrhs"], n.value), np.float64)
    _pre_check(lib, lib.ietidp_pre_get(h, _ptr(ip), _ptr(ix), _ptr(v), _ptr(f)))
    out = dict(K_indptr=ip, K_indices=ix, K_data=v, f=f, ms=ms.value, ms_fill=msf.value)
    if want_gram:
        gram = {}
        for c in range(3):
            for a in range(3):
                for q in range(desc["npatch"][a]):
                    nb = C.c_int()
                    _pre_check(lib, lib.ietidp_pre_get_gram(h, c, a, q, None, C.byref(nb)))
                    g = np.zeros((nb.value, nb.value))
                    _pre_check(lib, lib.ietidp_pre_get_gram(h, c, a, q, _ptr(g), None))
                    gram[(c, a, q)] = g.T.copy()
        out["gram"] = gram
    return out


def pre_assemble(desc, device=0, want_gram=False):
    """ietidp_pre_assemble + ietidp_pre_get for one box subdomain described by plain arrays
    (ietigen.predesc.subdomain_desc). Returns dict(K_indptr, K_indices, K_data, f (nrhs, n),
    ms, ms_fill [, gram])."""
    lib = load()
    keep = []
    s = PreSubdomain()
    _pre_fill(s, desc, keep)
    h = C.c_void_p()
    _pre_check(lib, lib.ietidp_pre_assemble(device, C.byref(s), C.byref(h)))
    try:
        return _pre_fetch(lib, h, desc, want_gram)
    finally:
        lib.ietidp_pre_destroy(h)


class PreBatch:
    """Handles of one ietidp_pre_assemble_batch call kept alive (the matrices stay on the
    device): sizes, device pointers for ietidp_set_values_device, host copies on request."""

    def __init__(self, descs, device=0):
        self.lib = load()
        self.descs = descs
        keep = []
        n = len(descs)
        subs = (PreSubdomain * n)()
        for k, d in enumerate(descs):
            _pre_fill(subs[k], d, keep)
        self.hs = (C.c_void_p * n)()
        _pre_check(self.lib, self.lib.ietidp_pre_assemble_batch(device, n, subs, self.hs))
        ms, msf = C.c_double(), C.c_double()
        _pre_check(self.lib, self.lib.ietidp_pre_sizes(self.hs[0], None, None, C.byref(ms), C.byref(msf)))
        self.ms, self.ms_fill = ms.value, msf.value

    def device_ptrs(self, k):
        v, f = C.c_void_p(), C.c_void_p()
        _pre_check(self.lib, self.lib.ietidp_pre_device_ptrs(self.hs[k], C.byref(v), C.byref(f)))
        return v.value, f.value

    def fetch(self, k):
        return _pre_fetch(self.lib, self.hs[k], self.descs[k], False)

    def refill(self, nus):
        """ietidp_pre_refill: new reluctivities per subdomain (list of arrays, or one concatenated
        array); reruns the value kernel in place. Returns its device time in ms."""
        nu = np.ascontiguousarray(np.concatenate([np.ravel(x) for x in nus]) if isinstance(nus, (list, tuple)) else nus,
                                  np.float64)
        ms = C.c_double()
        _pre_check(self.lib, self.lib.ietidp_pre_refill(self.hs[0], _ptr(nu), C.byref(ms)))
        self.ms_fill = ms.value
        return ms.value

    def close(self):
        for k in range(len(self.hs)):
            if self.hs[k]:
                self.lib.ietidp_pre_destroy(self.hs[k])
                self.hs[k] = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pre_assemble_batch(descs, device=0, fetch=True):
    """ietidp_pre_assemble_batch: every subdomain of a workload in one pass. Returns
    (list of result dicts (or None when fetch is False), dict(ms, ms_fill, nnz))."""
    lib = load()
    keep = []
    n = len(descs)
    subs = (PreSubdomain * n)()
    for k, d in enumerate(descs):
        _pre_fill(subs[k], d, keep)
    hs = (C.c_void_p * n)()
    _pre_check(lib, lib.ietidp_pre_assemble_batch(device, n, subs, hs))
    try:
        outs, nnz_tot = [], 0
        ms, msf = C.c_double(), C.c_double()
        for k in range(n):
            nz = C.c_int64()
            _pre_check(lib, lib.ietidp_pre_sizes(hs[k], None, C.byref(nz), C.byref(ms), C.byref(msf)))
            nnz_tot += nz.value
            outs.append(_pre_fetch(lib, hs[k], descs[k], False) if fetch else None)
        return outs, dict(ms=ms.value, ms_fill=msf.value, nnz=nnz_tot)
    finally:
        for k in range(n):
            lib.ietidp_pre_destroy(hs[k])


def pre_gauge(nv, ne, eu, ev, w, device=0):
    """ietidp_pre_gauge: (in_tree bool[ne], primal bool[ne], ms)."""
    lib = load()
    eu = np.ascontiguousarray(eu, np.int32)
    ev = np.ascontiguousarray(ev, np.int32)
    w = np.ascontiguousarray(w, np.int8)
    tree = np.zeros(ne, np.uint8)
    prim = np.zeros(ne, np.uint8)
    ms = C.c_double()
    _pre_check(lib, lib.ietidp_pre_gauge(device, nv, ne, _ptr(eu), _ptr(ev), _ptr(w), _ptr(tree), _ptr(prim), C.byref(ms)))
    return tree.astype(bool), prim.astype(bool), ms.value


def shard_partition(weights, nranks):
    """ietidp_shard_partition: owner rank per subdomain (contiguous, balanced by weight)."""
    lib = load()
    w = np.ascontiguousarray(weights, np.float64)
    owner = np.zeros(len(w), np.int32)
    st = lib.ietidp_shard_partition(len(w), _ptr(w), nranks, _ptr(owner))
    if st != OK:
        raise IetiError(st, "ietidp_shard_partition")
    return owner


class NcclComm:
    """An ncclComm_t of this process created through ctypes on the NCCL library torch has
    loaded (marshalling only): rank 0 draws the unique id, torch.distributed broadcasts its
    128 bytes, every rank calls ncclCommInitRank. The library then calls ncclAllReduce itself."""

    class _Uid(C.Structure):
        _fields_ = [("internal", C.c_byte * 128)]

    def __init__(self, rank, world, device):
        import glob
        import torch
        import torch.distributed as dist
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "nccl", "lib", "libnccl.so*"))
        self.lib = C.CDLL(cands[0] if cands else "libnccl.so.2")
        uid = self._Uid()
        if rank == 0:
            rc = self.lib.ncclGetUniqueId(C.byref(uid))
            if rc != 0:
                raise RuntimeError(f"ncclGetUniqueId failed ({rc})")
        if world > 1:
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=torch.device("cuda", device))
            dist.broadcast(t, src=0)
            C.memmove(C.byref(uid), bytes(t.cpu().tolist()), 128)
        self.comm = C.c_void_p()
        torch.cuda.set_device(device)
        self.lib.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, self._Uid, C.c_int]
        rc = self.lib.ncclCommInitRank(C.byref(self.comm), world, uid, rank)
        if rc != 0:
            raise RuntimeError(f"ncclCommInitRank failed ({rc})")
        self.allreduce_addr = C.cast(self.lib.ncclAllReduce, C.c_void_p)

    def close(self):
        if self.comm:
            self.lib.ncclCommDestroy.argtypes = [C.c_void_p]
            self.lib.ncclCommDestroy(self.comm)
            self.comm = None


def shard_from_bundle(b, owner, rank, nranks, allreduce, **opts):
    """A sharded Solver holding the subdomains k of a generator bundle with owner[k] == rank
    (local ids in ascending global order; multiplier and primal ids stay global)."""
    opts.setdefault("scaling", b["scaling"])
    opts.setdefault("tol", b["tol"])
    mine = [k for k in range(b["n_sub"]) if owner[k] == rank]
    s = Solver(len(mine), b["n_lambda"], b["n_primal"], b["nrhs"], **opts)
    if isinstance(allreduce, NcclComm):
        s.shard_enable_nccl(rank, nranks, allreduce)
    else:
        s.shard_enable(rank, nranks, allreduce)
    for i, k in enumerate(mine):
        sd = b["subs"][k]
        s.set_subdomain(i, sd["K_indptr"], sd["K_indices"], sd["K_data"], sd["f"], sd["B_lambda"], sd["B_dof"],
                        sd["B_sign"], sd["tree"], sd["prim"], sd["prim_gid"])
    s.global_ids = mine
    return s


class CudaView:
    """Zero-copy view of n doubles at a raw device pointer (for torch.as_tensor)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False), "version": 2}


def nccl_allreduce(device):
    """An all-reduce callback over torch.distributed (backend nccl): sums the buffer in place on
    the library's stream, so it is ordered with the kernels around it without a host sync."""
    import torch
    import torch.distributed as dist

    def fn(ptr, n, stream):
        t = torch.as_tensor(CudaView(ptr, n), device=torch.device("cuda", device))
        with torch.cuda.stream(torch.cuda.ExternalStream(int(stream), device=device)):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return 0
    return fn
