"""Pass experiments (IETIDP_DBG_PASS, results meaningless): one C5 solve with 100 fixed
iterations and the per-phase profile.  python tools/pass_exp.py C5"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["IETIDP_PCG_PROF"] = "1"
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp
b = make_bundle(sys.argv[1] if len(sys.argv) > 1 else "C5")
s = ietidp.from_bundle(b, fixed_iters=100)
s.factor()
s.solve(want_lambda=False, allow_noconv=True)
