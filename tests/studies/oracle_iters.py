"""Study (test infrastructure): the CPU oracle's natural-stopping PCG iteration
counts at full size (oracle/dp.py only; C5 on a column subset), written to
profiles/oracle_iters.json. bench.py's reference arm and cpu_baseline extrapolate
their sampled per-iteration oracle cost with these counts.

    python tests/studies/oracle_iters.py C2 C3 C4 C5:0,7
"""
import json
import os
import sys
import time

ROOT = __file__.rsplit("/tests/", 1)[0]
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from ietigen.bundle import make_bundle  # noqa: E402
from oracle import dp  # noqa: E402
from oracle_variants import slice_columns  # noqa: E402


def main():
    path = os.path.join(ROOT, "profiles", "oracle_iters.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for arg in sys.argv[1:]:
        name, _, cols = arg.partition(":")
        b = make_bundle(name)
        if cols:
            b = slice_columns(b, [int(c) for c in cols.split(",")])
        t0 = time.time()
        D = dp.DualPrimal(b)
        t1 = time.time()
        lam, info = D.pcg(tol=b["tol"])
        t2 = time.time()
        D.recover(lam)
        t3 = time.time()
        out[name] = dict(columns=[int(c) for c in cols.split(",")] if cols else "all",
                         iters=[int(x) for x in info["iters"]],
                         rel_residual=[float(x) for x in info["rel_residual"]],
                         seconds=dict(setup=t1 - t0, pcg=t2 - t1, recover=t3 - t2),
                         cpu=f"{os.cpu_count()} cores (this study's host)")
        print(name, out[name], flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
