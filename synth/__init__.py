"""Seeded synthetic workloads shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no kernel evaluation, tree,
compression or solve).  It only describes the five BASELINE.json configs and
draws their seeded inputs with numpy's PCG64:

  * points  (N, d) float64, original order   -- SURVEY.md §8(d) "Points"
  * b       (N,)   float64 ~ N(0,1)           -- right-hand side (reading R15)
  * X       (N, k) float64 ~ N(0,1), F-order  -- C5 multi-vectors
  * Omega   (N, w) float64 ~ N(0,1), F-order  -- the sketch of Alg. 2 step 1
                                               (PAPER.md P:823), passed to both
                                               sides for parity runs.

Seeds: points = config index, b = 1000+i, X = 2000+k, Omega = 3000+i.
The paper's own point sets (constant-density ball / sphere) are
replaced by BASELINE.json's unit square / cube / sphere (reading R17) for C1-C5;
the RPY workloads R1/R2 (Table 3) use the paper's
ball of radius (3N/(4 pi))^(1/3) and its right-hand side, uniform on
[-0.5, 0.5].  No public dataset is involved.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
import numpy as np

# kernel ids, same numbering as include/spdhss.h (SPD_K_*)
GAUSSIAN, MATERN32, EXPONENTIAL, IMQ, RPY = 0, 1, 2, 3, 4
KERNEL_NAMES = {GAUSSIAN: "gaussian", MATERN32: "matern32",
                EXPONENTIAL: "exponential", IMQ: "imq", RPY: "rpy"}


@dataclass(frozen=True)
class Config:
    name: str
    index: int          # 1..5, also the points seed
    d: int
    geometry: str       # "square" | "cube" | "sphere"
    n: int
    leaf: int
    kernel: int
    ell: float          # kernel length parameter l of BASELINE.json's formula
    shift: float        # sigma (diagonal shift)
    h2_tol: float = 1e-10
    rank_cap: int = 50
    hss_tol: float = 1e-3
    oversample: int = 10
    pcg_tol: float = 1e-8
    maxit: int = 3000
    n_proxy: int = 0    # 0 = library default (4096 in 2D, 6144 in 3D)
    rhs_kind: str = "normal"   # "normal" (R15) | "uniform" (U[-0.5, 0.5])

    @property
    def dofs(self) -> int:
        """Rows of the operator: n points x (3 for the RPY tensor kernel, else 1)."""
        return self.n * (3 if self.kernel == RPY else 1)

    @property
    def w(self) -> int:
        """Sketch width r + p (Alg. 2)."""
        return self.rank_cap + self.oversample

    def scaled(self, n: int, **kw) -> "Config":
        return replace(self, n=n, **kw)


# BASELINE.json "configs"
C1 = Config("C1", 1, 2, "square", 2048, 64, GAUSSIAN, 0.1, 1e-3, rank_cap=50)
C2 = Config("C2", 2, 3, "cube", 32768, 128, MATERN32, 0.2, 1e-4, rank_cap=100)
C3 = Config("C3", 3, 3, "sphere", 262144, 128, EXPONENTIAL, 0.5, 1e-4, rank_cap=100)
C4 = Config("C4", 4, 3, "cube", 1048576, 256, IMQ, 0.1, 1e-2, rank_cap=150)
# C5: matvec sweep only; Gaussian l=0.2 read as exp(-r^2/0.2^2) (R13), sigma=0 (R14)
C5 = Config("C5", 5, 3, "cube", 1048576, 256, GAUSSIAN, 0.2, 0.0)
# f1: the paper's RPY workloads (Table 3): ball point sets, particle
# radius a = 0.29 / 0.42, no shift, H2 tolerance 1e-8, r = 100, PCG to 1e-4
# with a uniform right-hand side
R1 = Config("R1", 6, 3, "ball", 40000, 128, RPY, 0.29, 0.0, h2_tol=1e-8, rank_cap=100, pcg_tol=1e-4,
            rhs_kind="uniform")
R2 = Config("R2", 7, 3, "ball", 40000, 128, RPY, 0.42, 0.0, h2_tol=1e-8, rank_cap=100, pcg_tol=1e-4,
            rhs_kind="uniform")
CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5, R1, R2)}


def points(cfg: Config, seed: int | None = None) -> np.ndarray:
    """(N, d) float64 points in original order."""
    rng = np.random.default_rng(cfg.index if seed is None else seed)
    if cfg.geometry in ("square", "cube"):
        return rng.random((cfg.n, cfg.d))
    if cfg.geometry == "sphere":
        g = rng.standard_normal((cfg.n, 3))
        return g / np.linalg.norm(g, axis=1, keepdims=True)
    if cfg.geometry == "ball":          # uniform in the ball of radius (3N/(4 pi))^(1/3)
        g = rng.standard_normal((cfg.n, 3))
        g /= np.linalg.norm(g, axis=1, keepdims=True)
        rad = (3.0 * cfg.n / (4.0 * np.pi)) ** (1.0 / 3.0)
        return g * (rad * rng.random((cfg.n, 1)) ** (1.0 / 3.0))
    raise ValueError(cfg.geometry)


def rhs(cfg: Config) -> np.ndarray:
    rng = np.random.default_rng(1000 + cfg.index)
    if cfg.rhs_kind == "uniform":
        return rng.random(cfg.dofs) - 0.5
    return rng.standard_normal(cfg.dofs)


def multivec(n: int, k: int, seed: int | None = None) -> np.ndarray:
    rng = np.random.default_rng(2000 + k if seed is None else seed)
    return np.asfortranarray(rng.standard_normal((n, k)))


def omega(cfg: Config, n: int | None = None, w: int | None = None) -> np.ndarray:
    """Gaussian sketch Omega (N x w), one for all levels (reading R8)."""
    n = cfg.dofs if n is None else n
    w = cfg.w if w is None else w
    rng = np.random.default_rng(3000 + cfg.index)
    return np.asfortranarray(rng.standard_normal((n, w)))
