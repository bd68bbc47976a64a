"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no basis, fit, octree or
evaluation code).  It only draws the point sets and evaluates the benchmark
functions the paper and BASELINE.json name, so that the oracle (``oracle/``)
and the CUDA path (``paper_1511_01353_b200``) read identical arrays.

Citations are PAPER.md lines (``P:<line>``) with their section; the recipe
readings (seeds, Halton details, mixture details) are DESIGN.md §3 / SURVEY.md
§8(c) ledger items G12, G14, G15.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "franke3d", "uniform_points", "halton_points", "mixture_centres",
    "mixture_points", "mixture_values", "Config", "CONFIGS", "make_inputs",
]


def franke3d(x: np.ndarray, chunk: int = 1 << 22) -> np.ndarray:
    """3-D Franke function exactly as printed in PAPER.md:287-288 (§3, Eq. eqF1).

    f = 3/4 [exp(-((9x-2)^2+(9y-2)^2+(9z-2)^2)/4) + exp(-(9x+1)^2/49 - (9y+1)^2/10 - (9z+1)^2/10)]
      + 1/2 exp(-((9x-7)^2+(9y-3)^2+(9z-5)^2)/4) - 1/5 exp(-(9x-4)^2-(9y-7)^2-(9z-5)^2)

    Note (ledger G12): the second term squares (9y+1) and (9z+1), as printed.
    ``x`` is (n, 3) float64; evaluated in chunks to bound temporaries.
    """
    x = np.asarray(x, dtype=np.float64)
    out = np.empty(x.shape[0], dtype=np.float64)
    for s in range(0, x.shape[0], chunk):
        a = 9.0 * x[s:s + chunk, 0]
        b = 9.0 * x[s:s + chunk, 1]
        c = 9.0 * x[s:s + chunk, 2]
        t1 = np.exp(-0.25 * ((a - 2) ** 2 + (b - 2) ** 2 + (c - 2) ** 2))
        t2 = np.exp(-((a + 1) ** 2) / 49.0 - ((b + 1) ** 2) / 10.0 - ((c + 1) ** 2) / 10.0)
        t3 = np.exp(-0.25 * ((a - 7) ** 2 + (b - 3) ** 2 + (c - 5) ** 2))
        t4 = np.exp(-((a - 4) ** 2) - (b - 7) ** 2 - (c - 5) ** 2)
        out[s:s + chunk] = 0.75 * (t1 + t2) + 0.5 * t3 - 0.2 * t4
    return out


def uniform_points(n: int, seed: int) -> np.ndarray:
    """Random grid in [0,1]^3 (§2 'random grid', §3 'p in [0,1]^3').

    numpy PCG64 ``default_rng(seed).random((n, 3))`` (ledger G14)."""
    return np.random.default_rng(seed).random((n, 3))


def _radical_inverse(idx: np.ndarray, base: int) -> np.ndarray:
    """Unscrambled radical inverse of positive integers ``idx`` in ``base``.

    The digit-reversed numerator and ``base**k`` are exact int64; one float64
    division then gives the correctly rounded value (ledger G14)."""
    idx = idx.astype(np.int64)
    num = np.zeros_like(idx)
    den = np.ones_like(idx)
    rem = idx.copy()
    while np.any(rem > 0):
        live = rem > 0
        digit = rem % base
        num = np.where(live, num * base + digit, num)
        den = np.where(live, den * base, den)
        rem = rem // base
    return num.astype(np.float64) / den.astype(np.float64)


def halton_points(n: int, chunk: int = 1 << 22) -> np.ndarray:
    """3-D Halton sequence, bases (2, 3, 5), indices 1..n, unscrambled (BASELINE.json config 3; ledger G14)."""
    out = np.empty((n, 3), dtype=np.float64)
    for s in range(0, n, chunk):
        idx = np.arange(s + 1, min(n, s + chunk) + 1, dtype=np.int64)
        for ax, base in enumerate((2, 3, 5)):
            out[s:s + idx.size, ax] = _radical_inverse(idx, base)
    return out


MIXTURE_K = 8
MIXTURE_SIGMA = 0.05


def mixture_centres(seed: int = 0) -> np.ndarray:
    """Centres of the 8-Gaussian mixture (BASELINE.json config 4): uniform in [0.2,0.8]^3,
    the first draw of ``default_rng(seed)`` (ledger G15)."""
    return np.random.default_rng(seed).uniform(0.2, 0.8, (MIXTURE_K, 3))


def mixture_points(n: int, seed: int, centres: np.ndarray) -> np.ndarray:
    """Clustered points: equal-weight mixture of 8 isotropic Gaussians (sigma 0.05) clipped to [0,1]^3.

    For seed 0 the generator first draws the centres (so the points use the same
    stream as ``mixture_centres(0)``); other seeds draw only components and offsets."""
    rng = np.random.default_rng(seed)
    if seed == 0:
        rng.uniform(0.2, 0.8, (MIXTURE_K, 3))  # the centres' draw (ledger G15)
    comp = rng.integers(0, MIXTURE_K, n)
    x = centres[comp] + MIXTURE_SIGMA * rng.standard_normal((n, 3))
    np.clip(x, 0.0, 1.0, out=x)
    return x


def mixture_values(x: np.ndarray, centres: np.ndarray, chunk: int = 1 << 22) -> np.ndarray:
    """f(x) = sum_k exp(-|x - c_k|^2 / 0.02) at the (clipped) points (BASELINE.json config 4)."""
    out = np.zeros(x.shape[0], dtype=np.float64)
    for s in range(0, x.shape[0], chunk):
        xs = x[s:s + chunk]
        acc = np.zeros(xs.shape[0])
        for c in centres:
            d2 = (xs[:, 0] - c[0]) ** 2 + (xs[:, 1] - c[1]) ** 2 + (xs[:, 2] - c[2]) ** 2
            acc += np.exp(-d2 / 0.02)
        out[s:s + chunk] = acc
    return out


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json workload (configs[i-1])."""
    cfg: int
    n: int
    m: int
    degree: int
    max_depth: int
    tol: float
    points: str   # "uniform" | "halton" | "mixture"
    values: str   # "franke" | "mixture"

    @property
    def name(self) -> str:
        return f"cfg{self.cfg}"

    def scaled(self, n: int | None = None, m: int | None = None) -> "Config":
        return dataclasses.replace(self, n=self.n if n is None else n, m=self.m if m is None else m)


CONFIGS = {
    1: Config(1, 2_000, 10_000, 4, 2, 1e-6, "uniform", "franke"),
    2: Config(2, 100_000, 1_000_000, 6, 5, 1e-8, "uniform", "franke"),
    3: Config(3, 2_000_000, 10_000_000, 8, 8, 1e-10, "halton", "franke"),
    4: Config(4, 20_000_000, 10_000_000, 6, 12, 1e-9, "mixture", "mixture"),
    5: Config(5, 200_000_000, 100_000_000, 10, 10, 1e-11, "uniform", "franke"),
}


def make_inputs(cfg: Config):
    """Return (pts (N,3), f (N,), q (M,3)) float64, C-contiguous, for a config.

    Points: seed 0; queries: seed 1 (uniform for configs 1, 2, 3, 5; the same
    mixture for config 4).  Values: the analytic function at the points."""
    if cfg.points == "uniform":
        pts = uniform_points(cfg.n, 0)
    elif cfg.points == "halton":
        pts = halton_points(cfg.n)
    elif cfg.points == "mixture":
        centres = mixture_centres(0)
        pts = mixture_points(cfg.n, 0, centres)
    else:
        raise ValueError(cfg.points)
    if cfg.points == "mixture":
        q = mixture_points(cfg.m, 1, centres)
        f = mixture_values(pts, centres)
    else:
        q = uniform_points(cfg.m, 1)
        f = franke3d(pts)
    return np.ascontiguousarray(pts), np.ascontiguousarray(f), np.ascontiguousarray(q)


def exact_values(cfg: Config, x: np.ndarray) -> np.ndarray:
    """The analytic function of a config at arbitrary points (for E_rms / E_inf)."""
    if cfg.values == "franke":
        return franke3d(x)
    return mixture_values(x, mixture_centres(0))


def rms_and_max(err: np.ndarray) -> tuple[float, float]:
    """E_rms and E_inf of an error vector (§4)."""
    err = np.asarray(err, dtype=np.float64)
    return float(math.sqrt(np.mean(err * err))) if err.size else 0.0, float(np.max(np.abs(err))) if err.size else 0.0


def cell_queries(depth: int, cell, n: int, seed: int) -> np.ndarray:
    """Uniform query points inside the octree cell ``cell`` = (i, j, k) at ``depth`` of the unit root
    cube: (cell + U[0,1)^3) / 2^depth, ``default_rng(seed)``.  Used for the parity queries inside the
    sampled subtrees of the full-size configs (tests/golden/oracle_cfg*.npz)."""
    r = np.random.default_rng(seed).random((n, 3))
    return (np.asarray(cell, dtype=np.float64) + r) / float(2 ** depth)


def cell_of(points: np.ndarray, depth: int) -> np.ndarray:
    """Integer cell (i, j, k) of unit-cube points at ``depth``: min(floor(x 2^depth), 2^depth - 1)
    (selection of a subtree's points for the harness)."""
    return np.minimum(np.floor(np.asarray(points) * float(2 ** depth)), 2 ** depth - 1).astype(np.int64)
