"""Drive every GPU code path once on small workloads, for compute-sanitizer runs:

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/san_run.py C1 C2r C5r

Per workload: analyze, factor (graph capture), solve (persistent PCG), u, the
operator entry points, set_values + refactor (graph replay), the triangular loop,
the per-phase graph PCG driver (IETIDP_PCG=graph) and the condition estimate."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from ietigen.bundle import make_bundle  # noqa: E402
from paper_2501_04340_b200 import ietidp  # noqa: E402


def run(name):
    b = make_bundle(name)
    out = []
    for loop in ("explicit", "triangular"):
        s = ietidp.from_bundle(b, loop=loop)
        s.factor()
        lam, rep = s.solve()
        u = [s.get_u(k) for k in range(b["n_sub"])]
        X = np.random.default_rng(0).standard_normal((b["n_lambda"], b["nrhs"]))
        s.apply_F(X)
        s.apply_precond(X)
        if b["n_primal"]:
            s.get_coarse()
        s.get_rhs()
        s.estimate_condition()
        for k, sd in enumerate(b["subs"]):
            s.set_values(k, sd["K_data"] * 2.0, sd["f"])
        s.factor()
        lam2, rep2 = s.solve()
        out.append((loop, rep["iters"][:2], rep2["iters"][:2], float(np.abs(lam).max()), len(u)))
        s.close()
    os.environ["IETIDP_PCG"] = "graph"
    s = ietidp.from_bundle(b)
    s.factor()
    lam, rep = s.solve()
    out.append(("graph-pcg", rep["iters"][:2]))
    s.close()
    del os.environ["IETIDP_PCG"]
    torch.cuda.synchronize()
    print(name, out, flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["C1", "C2r"]:
        run(n)
    print("san_run OK")
