"""Seeded synthetic workload generators (inputs only -- none of the method's arithmetic).

Shared by tests/, bench.py and the oracle harness.  Everything here is an
*input* to the ADI step: element-wise material maps (the nested-ellipsoid head
phantom standing in for the paper's MRI head), random coefficient
fields, source positions and source time signals sampled at (n+1/2)tau (D9).
Nothing here evaluates B-splines, matrices or the scheme: the oracle and the
CUDA library each turn these inputs into their own discrete objects.

Recipes follow SURVEY.md §8(d) (proposals where the paper is silent; recorded
in DESIGN.md):
  c1: n=8,   p=2, eps=mu=1, tau=1e-2, 10 steps, E0 = u_A (oracle projection) or random
  c2: n=32,  p=2, eps=mu=1, tau in {1e-2, 5e-3, 2.5e-3}, 100 steps
  c3: n=64,  p=3, phantom (air 1 / tissue 50 / skull 12) x (1 + 0.05 U(-1,1)), seed 3,
      Gaussian-pulse dipole on E3 just outside the scalp top, 200 steps
  c4: n=128, p=2, phantom with tissue eps_r ~ U[30,70] per voxel (seed 4), skull 12, air 1,
      Gaussian-modulated sinusoid dipole, 500 steps
  c5: n=512, p=2, inside the scalp ellipsoid eps_r ~ U[1,80] per voxel (seed 5), 1 outside,
      no source, 100 steps
"""
from __future__ import annotations

import math

import numpy as np

# Nested ellipsoids centred at (1/2,1/2,1/2).
S0 = np.array([0.36, 0.44, 0.40])  # scalp
S1 = S0 - 0.03  # skull outer
S2 = S1 - 0.04  # skull inner

CONFIGS = {
    "c1": dict(n=8, p=2, tau=1e-2, steps=10, material="uniform", source=None),
    "c2": dict(n=32, p=2, tau=1e-2, steps=100, material="uniform", source=None),
    "c3": dict(n=64, p=3, tau=1e-2, steps=200, material="phantom3", source="pulse"),
    "c4": dict(n=128, p=2, tau=1e-2, steps=500, material="phantom4", source="modsine"),
    "c5": dict(n=512, p=2, tau=1e-2, steps=100, material="phantom5", source=None),
}


def _centres(n: int):
    c = (np.arange(n) + 0.5) / n
    # element (a,b,c) -> a + n(b + n c): arrays indexed [c, b, a] in C order
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    return x, y, z


def _inside(x, y, z, S):
    return ((x - 0.5) / S[0]) ** 2 + ((y - 0.5) / S[1]) ** 2 + ((z - 0.5) / S[2]) ** 2 <= 1.0


def element_eps(n: int, kind: str, seed: int | None = None) -> np.ndarray:
    """Element-wise relative permittivity, flat, element index a + n(b + n c)."""
    if kind == "uniform":
        return np.ones(n ** 3)
    x, y, z = _centres(n)
    in0, in1, in2 = _inside(x, y, z, S0), _inside(x, y, z, S1), _inside(x, y, z, S2)
    skull = in1 & ~in2
    tissue = (in0 & ~in1) | in2
    eps = np.ones((n, n, n))
    if kind == "phantom3":
        rng = np.random.default_rng(3 if seed is None else seed)
        eps[tissue] = 50.0
        eps[skull] = 12.0
        eps *= 1.0 + 0.05 * rng.uniform(-1.0, 1.0, size=eps.shape)
    elif kind == "phantom4":
        rng = np.random.default_rng(4 if seed is None else seed)
        vals = rng.uniform(30.0, 70.0, size=eps.shape)
        eps[tissue] = vals[tissue]
        eps[skull] = 12.0
    elif kind == "phantom5":
        rng = np.random.default_rng(5 if seed is None else seed)
        vals = rng.uniform(1.0, 80.0, size=eps.shape)
        eps[in0] = vals[in0]
    elif kind == "random":
        rng = np.random.default_rng(0 if seed is None else seed)
        eps = rng.uniform(1.0, 80.0, size=eps.shape)
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(eps.reshape(-1))


def random_fields(N: int, seed: int, scale: float = 1.0):
    """Six seeded coefficient arrays (E1,E2,E3,H1,H2,H3), uniform in [-scale, scale]."""
    rng = np.random.default_rng(seed)
    return [scale * rng.uniform(-1.0, 1.0, size=N ** 3) for _ in range(6)]


def random_tf(N: int, seed: int, lo: float = 1e-3, hi: float = 1e3):
    """Per-test-function values, log-uniform in [lo, hi]."""
    rng = np.random.default_rng(seed)
    return np.exp(rng.uniform(math.log(lo), math.log(hi), size=N ** 3))


def dipole_position(n: int):
    """Point dipole just outside the scalp top."""
    h = 1.0 / n
    return (0.5 + 0.25 * h, 0.5 + 0.25 * h, 0.5 + 0.40 + 0.5 * h)


def signal(kind: str | None, tau: float, nsteps: int) -> np.ndarray:
    """s((m + 1/2) tau), m = 0..nsteps-1 (D9)."""
    t = (np.arange(nsteps) + 0.5) * tau
    if kind is None:
        return np.zeros(nsteps)
    if kind == "pulse":
        return np.exp(-(((t - 0.3) / 0.08) ** 2))
    if kind == "modsine":
        return np.sin(2 * np.pi * 2.0 * (t - 1.0)) * np.exp(-(((t - 1.0) / 0.4) ** 2))
    raise ValueError(kind)
