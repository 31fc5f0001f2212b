"""Factorisation experiments (IETIDP_DBG_FACTOR, results meaningless): mean factor time
of 5 factorisations after 2 warm-up ones.  python tools/factor_exp.py C2"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp
b = make_bundle(sys.argv[1] if len(sys.argv) > 1 else "C2")
kw = {}
if os.environ.get("EXP_ORDER"):
    kw["ordering"] = os.environ["EXP_ORDER"]
if os.environ.get("EXP_LEAF"):
    kw["leaf_size"] = int(os.environ["EXP_LEAF"])
s = ietidp.from_bundle(b, **kw)
t = []
for i in range(7):
    s.factor()
    lam, rep = s.solve(want_lambda=False, allow_noconv=True)
    if i >= 2:
        t.append(rep["ms_factor"])
r = s.report()
print(os.environ.get("IETIDP_DBG_FACTOR", "0"), kw, "flops %.1f GF levels %d" % (r["factor_flops"] / 1e9, r["n_levels"]), "factor ms %.3f (min %.3f)" % (statistics.mean(t), min(t)), flush=True)
