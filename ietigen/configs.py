"""The five synthetic workloads of BASELINE.json `configs` (C1..C5) and their
reduced (e = 2) and EOC variants.

Only recipe data lives here: patch grids, degrees, tilings, materials and source
fields. Random numbers come from `ietigen.rng` (splitmix64, Box–Muller).
"""
import functools
from dataclasses import dataclass, field, replace
import numpy as np

from .rng import SplitMix64


@dataclass(frozen=True)
class Config:
    name: str
    npatch: tuple          # patches per axis (x, y, z); cylinder: (theta, r, z)
    p: int                 # 0-form degree
    e: int                 # elements per direction per patch
    tiling: tuple          # subdomains per axis; each subdomain is a box of patches
    geometry: str = "cube"  # "cube" (unit cube) | "cylinder" (hollow, periodic theta)
    material: str = "one"   # "one" | "c3_block" | "c4_outer" | "c5_random"
    rhs: str = "astar"      # "astar" | "c3" | "c4" | "c5_random" | "aana" (the paper's A_ana, inhomogeneous n x A)
    nrhs: int = 1
    scaling: str = "multiplicity"  # "multiplicity" | "stiffness"
    tol: float = 1e-10
    seed: int = 0
    load_nq_extra: int = 3  # Gauss points per element for loads: p + load_nq_extra
    parts: tuple = None     # explicit partition: a subdomain id per patch (x fastest), else the tiling

    @property
    def n_sub(self):
        return int(np.prod(self.tiling))

    @property
    def periodic(self):
        return (self.geometry == "cylinder", False, False)

    def reduced(self, e=2):
        return replace(self, name=self.name + "r", e=e)


C1 = Config("C1", (2, 2, 2), 1, 2, (2, 1, 1))
C2 = Config("C2", (4, 4, 4), 2, 8, (4, 2, 2))
C3 = Config("C3", (6, 6, 6), 2, 8, (3, 6, 6), material="c3_block", rhs="c3",
            scaling="stiffness")
C4 = Config("C4", (16, 2, 4), 3, 6, (16, 2, 2), geometry="cylinder",
            material="c4_outer", rhs="c4", scaling="stiffness")
C5 = Config("C5", (8, 8, 8), 2, 6, (8, 4, 4), material="c5_random",
            rhs="c5_random", nrhs=16, scaling="stiffness")

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}
# scaling case (not a BASELINE config): C5r's discretisation and data with every patch
# its own subdomain (8 x 8 x 8 = 512 subdomains, n_gp = 833): the coarse problem is
# larger than the one-CTA coarse factorisation (n_gp grows with N_sub)
EXTRA = {"C5s": replace(C5, name="C5s", e=2, tiling=(8, 8, 8))}


def get(name: str) -> Config:
    """'C2' -> full config; 'C2r' -> reduced e=2 variant; 'C1e4' -> C1 with e=4;
    'E27A_...' -> the 27-patch family with the paper's A_ana and its boundary values lifted;
    'C4m<p>e<e>' -> the cylinder with the manufactured A* = sin(2 pi (r - 1/2)) e_z;
    'E27_<tiling or partition>_p<p>_e<e>' -> the paper's 27-patch family."""
    if name in CONFIGS:
        return CONFIGS[name]
    if name in EXTRA:
        return EXTRA[name]
    if name.startswith("E27_"):
        return paper_cube(name)
    if name.startswith("E27A_"):
        return replace(paper_cube("E27_" + name[5:]), name=name, rhs="aana")
    if name.startswith("C4m"):
        p, e = name[3:].split("e")
        return replace(C4, name=name, p=int(p), e=int(e), material="one", rhs="c4_manufactured",
                       scaling="multiplicity")
    if name.endswith("r") and name[:-1] in CONFIGS:
        return CONFIGS[name[:-1]].reduced()
    if "e" in name[1:]:
        base, e = name.split("e", 1)[0], int(name.split("e", 1)[1])
        return replace(CONFIGS[base], name=name, e=e)
    raise KeyError(name)


# E1's three subdomains of 9 patches each (Fig. 1: a METIS-like partition
# of the 27 patches, our reading, R14): part 0 = the patch layer x = 0, part 1
# = (x >= 1, y = 0) + (x = 1, y = 1), part 2 = the rest -- L-shaped cross-sections
# extruded in z. All three meet along the line x = 1/3, y = 2/3: cross edges, n_gp > 0.
def _l3_parts():
    out = []
    for k in range(3):
        for j in range(3):
            for i in range(3):
                out.append(0 if i == 0 else (1 if (j == 0 or (i == 1 and j == 1)) else 2))
    return tuple(out)


PAPER_PARTS = {"L3": _l3_parts()}


def paper_cube(name: str) -> Config:
    """The paper's experiment family: 27 cube patches (3 x 3 x 3),
    nu = 1, homogeneous manufactured A* (our reading, R14), degree p, e elements
    per patch direction (normalised h = 1/(3e)), a box tiling of the patch
    grid: 'E27_<tx><ty><tz>_p<p>_e<e>', e.g. 'E27_311_p2_e4' (N_sub = 3)."""
    _, t, p, e = name.split("_")
    if t in PAPER_PARTS:  # explicit partition ('E27_L3_p<p>_e<e>')
        parts = PAPER_PARTS[t]
        return Config(name, (3, 3, 3), int(p[1:]), int(e[1:]), (max(parts) + 1, 1, 1), tol=1e-6, parts=parts)
    return Config(name, (3, 3, 3), int(p[1:]), int(e[1:]), tuple(int(x) for x in t), tol=1e-6)


def patch_nu(cfg: Config) -> np.ndarray:
    """Reluctivity nu = 1/mu_r per patch, shape npatch."""
    N = cfg.npatch
    nu = np.ones(N)
    if cfg.material == "c3_block":
        nu[2:4, 2:4, 2:4] = 1e-3
    elif cfg.material == "c4_outer":
        nu[:, 1, :] = 1e-3           # outer radial patch layer r in [0.75, 1]
    elif cfg.material == "c5_random":
        g = SplitMix64(cfg.seed)
        for k in range(N[2]):
            for j in range(N[1]):
                for i in range(N[0]):   # patch order: x fastest
                    nu[i, j, k] = 10.0 ** (-3.0 * g.uniform())
    return nu


def c5_coefficients(cfg: Config) -> np.ndarray:
    """a[s, c, k1-1, k2-1, k3-1] ~ N(0,1)/(1+|k|^2), stream splitmix64(seed+1)."""
    g = SplitMix64(cfg.seed + 1)
    a = np.zeros((cfg.nrhs, 3, 3, 3, 3))
    for s in range(cfg.nrhs):
        for c in range(3):
            for k3 in range(1, 4):
                for k2 in range(1, 4):
                    for k1 in range(1, 4):
                        a[s, c, k1 - 1, k2 - 1, k3 - 1] = g.normal() / (
                            1.0 + k1 * k1 + k2 * k2 + k3 * k3)
    return a


@functools.lru_cache(maxsize=8)
def source_terms(cfg: Config):
    """The field T with J = curl T as separable terms, per RHS column and component.

    Returns terms[s][c] = list of (coef, fx, fy, fz) with f = (kind, k), kind in
    {"sin", "cos"}: f(x) = sin(k pi x) or cos(k pi x). Cube configs only.
    C1/C2: T = curl A*, A* = (sin pi y sin pi z, sin pi z sin pi x, sin pi x sin pi y).
    C3: T = (0, 0, sin pi x sin pi y sin pi z). C5: seeded Fourier modes <= 3.
    """
    pi = np.pi
    if cfg.rhs == "astar":
        # T_x = pi sin(pi x)(cos pi y - cos pi z), cyclic.
        Tx = [(pi, ("sin", 1), ("cos", 1), ("one", 0)), (-pi, ("sin", 1), ("one", 0), ("cos", 1))]
        Ty = [(pi, ("one", 0), ("sin", 1), ("cos", 1)), (-pi, ("cos", 1), ("sin", 1), ("one", 0))]
        Tz = [(pi, ("cos", 1), ("one", 0), ("sin", 1)), (-pi, ("one", 0), ("cos", 1), ("sin", 1))]
        return [[Tx, Ty, Tz]]
    if cfg.rhs == "c3":
        return [[[], [], [(1.0, ("sin", 1), ("sin", 1), ("sin", 1))]]]
    if cfg.rhs == "aana":
        # T = nu B_ana = curl A_ana = (-3 cos x sin y sin z, 0, 3 cos z sin x sin y)
        return [[[(-3.0, ("cosx", 0), ("sinx", 0), ("sinx", 0))], [],
                 [(3.0, ("sinx", 0), ("sinx", 0), ("cosx", 0))]]]
    if cfg.rhs == "c5_random":
        a = c5_coefficients(cfg)
        out = []
        for s in range(cfg.nrhs):
            col = []
            for c in range(3):
                terms = []
                for k3 in range(1, 4):
                    for k2 in range(1, 4):
                        for k1 in range(1, 4):
                            terms.append((a[s, c, k1 - 1, k2 - 1, k3 - 1], ("sin", k1),
                                          ("sin", k2), ("sin", k3)))
                col.append(terms)
            out.append(col)
        return out
    raise ValueError(cfg.rhs)


def f1d(spec):
    kind, k = spec
    if kind == "sin":
        return lambda x: np.sin(k * np.pi * x)
    if kind == "cos":
        return lambda x: np.cos(k * np.pi * x)
    if kind == "sinx":
        return lambda x: np.sin(x)
    if kind == "cosx":
        return lambda x: np.cos(x)
    return lambda x: np.ones_like(x)


# The paper's closed-form solution, per component a separable product
# coef * fx(x) fy(y) fz(z): A_ana = (cos y cos z sin x, -2 cos x cos z sin y, cos x cos y sin z).
A_ANA = [(1.0, ("sinx", 0), ("cosx", 0), ("cosx", 0)),
         (-2.0, ("cosx", 0), ("sinx", 0), ("cosx", 0)),
         (1.0, ("cosx", 0), ("cosx", 0), ("sinx", 0))]
