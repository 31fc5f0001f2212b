"""Factor + solve timing of one workload under each ordering option (device events of
the library's report), for choosing the default. python tools/ordering_compare.py C2"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
orders = sys.argv[2:] or ["nd", "md"]
b = make_bundle(name)
ref = None
for o in orders:
    s = ietidp.from_bundle(b, ordering=o)
    s.analyze()
    for _ in range(2):
        s.factor()
        lam, rep = s.solve()
    fs = []
    for _ in range(5):
        s.factor()
        lam, rep = s.solve()
        fs.append((rep["ms_factor"], rep["ms_coarse"], rep["ms_pcg"], rep["ms_recover"]))
    f = np.median(np.array(fs), axis=0)
    err = 0.0 if ref is None else np.linalg.norm(lam - ref) / np.linalg.norm(ref)
    ref = lam if ref is None else ref
    print(f"{name} {o}: flops {rep['factor_flops']/1e9:.1f} GF nnzL {rep['nnz_L']/1e6:.1f}M levels {rep['n_levels']} "
          f"sn {rep['n_supernodes']} | factor {f[0]:.2f} coarse {f[1]:.2f} pcg {f[2]:.2f} recover {f[3]:.2f} "
          f"total {f.sum():.2f} ms iters {rep['iters'][:2]} rel diff lambda {err:.1e}", flush=True)
