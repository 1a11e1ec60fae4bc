"""Seeded random fields and manufactured solutions / right-hand sides.

Manufactured pairs:
  * sin3:  u = sin x sin y sin z on [0,2pi]^3, -Lap u = 3u.
  * TGV pressure (Taylor-Green vortex):
        p = (cos2x + cos2y)(cos2z + 2)/16,
        -Lap p = (cos2x + cos2y)(1 + cos2z)/2.
  * cylinder (R = 0.5, H = 1): u = (1 - 4 r^2) sin(pi z) vanishes on all walls,
        -Lap u = [16 + pi^2 (1 - 4 r^2)] sin(pi z).
These are pointwise function evaluations at node coordinates -- no SEM
arithmetic.
"""
from __future__ import annotations

import math

import numpy as np

PARITY_SEED = 20240509


def random_field(shape, seed=PARITY_SEED, low=-1.0, high=1.0):
    """u ~ U(low, high), numpy default_rng(seed), float64."""
    return np.random.default_rng(seed).uniform(low, high, size=shape)


def positive_field(shape, seed, low=0.5, high=1.5):
    """Strictly positive coefficient field (variable h1/h2 parity cases)."""
    return np.random.default_rng(seed).uniform(low, high, size=shape)


def sin3(coords):
    x, y, z = coords
    return np.sin(x) * np.sin(y) * np.sin(z)


def sin3_source(coords):
    return 3.0 * sin3(coords)


def tgv_pressure(coords):
    x, y, z = coords
    return (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2.0) / 16.0


def tgv_source(coords):
    x, y, z = coords
    return 0.5 * (np.cos(2 * x) + np.cos(2 * y)) * (1.0 + np.cos(2 * z))


def cyl_exact(coords):
    """u = (1 - 4 r^2) sin(pi z) on the R = 0.5, H = 1 cylinder."""
    x, y, z = coords
    r2 = x * x + y * y
    return (1.0 - 4.0 * r2) * np.sin(math.pi * z)


def cyl_source(coords, h1=1.0, h2=0.0):
    """f = h1 (-Lap u) + h2 u for u = cyl_exact (R = 0.5, H = 1)."""
    x, y, z = coords
    r2 = x * x + y * y
    u = (1.0 - 4.0 * r2) * np.sin(math.pi * z)
    lap = (16.0 + math.pi ** 2 * (1.0 - 4.0 * r2)) * np.sin(math.pi * z)
    return h1 * lap + h2 * u


def tgv_velocity(coords):
    """Taylor-Green vortex initial velocity (unit amplitude,
    [0, 2pi]^3): u = sin x cos y cos z, v = -cos x sin y cos z, w = 0."""
    x, y, z = coords
    return np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z), 0.0 * z])
