"""The BASELINE.json workloads as seeded synthetic problems (host setup).

SURVEY.md §8(d) fixes the RNG protocol that BASELINE.json leaves open; the
oracle, the golden generator, the GPU tests and bench.py all build their
inputs through these functions so that every arm sees identical data.

  config 1: N=16,  k=2, nu=1,    Dirichlet left/top/bottom, Gamma_N outlet x=1
  config 2: N=128, k=4, nu=1e-2, same boundary, interior vertices jittered by
            U(-0.2h, 0.2h) from default_rng(1)
  config 3: N=256, k=6, nu=1,    outlet is Gamma_Ntilde (u_t = 0)
  config 5: synthetic SPD Schur microbench (n_s=60, n_c=36), see
            `microbench_batch`.
Body force (seed s): 4 modes sin(a x + b y), (a, b) integers in [1, 4],
2-vector amplitudes N(0, 1).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import build_structured, classify_boundary, jittered_structured

EPS = 1e-12


class FourierForce:
    """f(x) = amp^T sin(ab[:,0] x + ab[:,1] y); callable on one point (the
    reference signature) and `vectorized` on an (n, 2) array."""

    def __init__(self, seed: int, modes: int = 4):
        rng = np.random.default_rng(seed)
        self.ab = rng.integers(1, 5, size=(modes, 2))
        self.amp = rng.standard_normal((modes, 2))

    def __call__(self, x):
        return self.amp.T @ np.sin(self.ab[:, 0] * x[0] + self.ab[:, 1] * x[1])

    def vectorized(self, X):
        X = np.asarray(X, dtype=float)
        return np.sin(X[:, :1] * self.ab[:, 0] + X[:, 1:2] * self.ab[:, 1]) @ self.amp


@dataclass
class MCSProblem:
    name: str
    mesh: object
    regions: object
    k: int
    nu: float
    body_force: object


def outlet_regions(mesh, tilde: bool):
    """Dirichlet (u = 0) on x < 1, natural (Gamma_N) or tangential-Dirichlet
    (Gamma_Ntilde) outlet on x = 1."""
    out = {"tilde_neumann" if tilde else "neumann": lambda x: x[0] >= 1 - EPS}
    return classify_boundary(mesh, dirichlet=lambda x: x[0] < 1 - EPS, **out)


def baseline_config(cfg: int, n: int = None) -> MCSProblem:
    """BASELINE config 1-3 (optionally on a smaller n x n grid, same k/nu/BC
    and seeds, for parity tests)."""
    if cfg == 1:
        n = n or 16
        mesh = build_structured(n, n)
        return MCSProblem("cfg1", mesh, outlet_regions(mesh, False), 2, 1.0,
                          FourierForce(0))
    if cfg == 2:
        n = n or 128
        mesh = jittered_structured(n, 0.2, seed=1)
        return MCSProblem("cfg2", mesh, outlet_regions(mesh, False), 4, 1e-2,
                          FourierForce(0))
    if cfg == 3:
        n = n or 256
        mesh = build_structured(n, n)
        return MCSProblem("cfg3", mesh, outlet_regions(mesh, True), 6, 1.0,
                          FourierForce(2))
    raise ValueError(f"no 2D MCS problem for config {cfg}")


MICRO_N, MICRO_M = 60, 36


def microbench_host(count: int, seed: int = 3, n: int = MICRO_N, m: int = MICRO_M):
    """Host generator of the config-5 distribution for small parity samples:
    G ~ N(0,1)^(count,n,n), B ~ N(0,1)^(count,n,m), A = G G^T + n I."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((count, n, n))
    B = rng.standard_normal((count, n, m))
    return G @ np.swapaxes(G, 1, 2) + n * np.eye(n), B
