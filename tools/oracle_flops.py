"""Useful-flop count of the local factorisations under the ORACLE's reference ordering
(factor roofline uses min(GPU-ordering count, oracle-ordering count)).

For every subdomain the oracle factors K_rr with SuperLU (MMD on A^T + A, no pivoting,
symmetric mode, oracle/dp.py::_factor). L's column counts c_j (diagonal included) give
sum_j c_j^2. Writes profiles/oracle_flops.json. Offline tool (CPU): python
tools/oracle_flops.py C2 C3 ..."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from ietigen.bundle import make_bundle  # noqa: E402
from oracle import dp  # noqa: E402

out_path = os.path.join(ROOT, "profiles", "oracle_flops.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
for name in sys.argv[1:] or ["C2"]:
    b = make_bundle(name)
    tot = 0
    nnz = 0
    for k, s in enumerate(b["subs"]):
        L = dp.Local(k, s, int(b["n_lambda"]), False)
        if L.lu is None:
            continue
        cc = np.diff(L.lu.L.tocsc().indptr).astype(np.int64)  # column counts incl. the unit diagonal
        tot += int((cc * cc).sum())
        nnz += int(cc.sum())
    res[name] = {"useful_flops_oracle_ordering": tot, "nnz_L_oracle_ordering": nnz,
                 "ordering": "SuperLU MMD_AT_PLUS_A on K_rr (oracle/dp.py)"}
    print(name, res[name], flush=True)
    json.dump(res, open(out_path, "w"), indent=1)
