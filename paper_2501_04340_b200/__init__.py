"""B200-native IETI-DP solve phase (arXiv 2501.04340): libietidp.so + ctypes binding."""
from .ietidp import Solver, from_bundle, load, IetiError  # noqa: F401
