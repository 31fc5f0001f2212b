"""A/B check of two builds (IETIDP_LIB selects the library): one factor + solve of a
workload, lambda / u / iteration counts saved to an npz for a bitwise comparison.

    python tools/ab_dump.py C5r out.npz          (then: python tools/ab_dump.py --cmp a.npz b.npz)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        same = np.array_equal(a[k], b[k])
        d = np.abs(a[k] - b[k]).max() / max(np.abs(a[k]).max(), 1e-300) if a[k].shape == b[k].shape else None
        print(f"{k:8s} bitwise {'yes' if same else 'NO '}  max rel diff {d}")
    sys.exit(0)
from ietigen.bundle import make_bundle  # noqa: E402
from paper_2501_04340_b200 import ietidp  # noqa: E402

b = make_bundle(sys.argv[1])
s = ietidp.from_bundle(b)
s.factor()
lam, rep = s.solve()
u = np.concatenate([s.get_u(k) for k in range(b["n_sub"])])
np.savez(sys.argv[2], lam=lam, u=u, iters=np.array(rep["iters"][: b["nrhs"]]))
print(sys.argv[1], "iters", rep["iters"][: b["nrhs"]], "ms_pcg", rep["ms_pcg"], "lib", ietidp.LIB_PATH)
