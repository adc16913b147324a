"""Seeded synthetic inputs for the BASELINE.json configurations (numpy, host).

The paper/reference measure on uniformly refined coarse meshes; BASELINE.json
names them (2-triangle unit square, 6-triangle L-shape, the L12 "stress" mesh
with jitter / permutation / rotation / flips).  None of these meshes ships with
the reference except the 4-triangle crisscross square (proj/data/unit-square,
proj/tests/support.hpp:13-20), so they are generated here with fixed seeds.
Randomness is a counter-based splitmix64 stream: value_i = mix(seed + (i+1) *
0x9E3779B97F4A7C15), U[-1,1] = ((value >> 11) * 2^-53) * 2 - 1.
"""
from __future__ import annotations

import math

import numpy as np

from .capi import (COEFF_CENTROID_POLY, FIELD_EXP_SINSIN, FIELD_SINSIN, FIELD_ZERO, FLUX_GRAD_SINSIN,
                   FLUX_ZERO, TWO_PI2, TWO_PI2_M1, HostMesh, coeffs_centroid_poly, coeffs_const,
                   field)

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(seed: int, n: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (np.arange(1, n + 1, dtype=np.uint64) * _GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform_pm1(seed: int, n: int) -> np.ndarray:
    z = splitmix64(seed, n)
    return ((z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)) * 2.0 - 1.0


# ---- coarse meshes ------------------------------------------------------------
def crisscross_square() -> HostMesh:
    """The reference fixture (support.hpp:13-20 / proj/data/unit-square)."""
    return HostMesh(np.array([[0, 0], [1, 0], [0, 1], [1, 1], [0.5, 0.5]], dtype=np.float64),
                    np.array([[4, 0, 1], [4, 2, 0], [4, 3, 2], [4, 1, 3]]),
                    np.array([[0, 1], [1, 3]]), np.array([[3, 2], [2, 0]]))


def unit_right_triangle() -> HostMesh:
    """support.hpp:23-28."""
    return HostMesh(np.array([[0, 0], [1, 0], [0, 1]], dtype=np.float64), np.array([[0, 1, 2]]),
                    np.zeros((0, 2)), np.zeros((0, 2)))


def square_2tri() -> HostMesh:
    """Config 1/3/4/5 coarse mesh: unit square, diagonal (0,0)-(1,1); Dirichlet on
    x=0 and y=0, Neumann on x=1 and y=1 (pairs CCW w.r.t. their element)."""
    return HostMesh(np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=np.float64),
                    np.array([[0, 1, 2], [0, 2, 3]]),
                    np.array([[0, 1], [3, 0]]), np.array([[1, 2], [2, 3]]))


def lshape_6tri() -> HostMesh:
    """Config 2 coarse mesh: [-1,1]^2 minus [0,1]x[-1,0]; three squares, each
    split along its (min,min)-(max,max) diagonal.  Dirichlet on x=-1, y=-1 and
    the two re-entrant sides; Neumann on x=1 and y=1 (fixed in-repo: the
    BASELINE leaves the sides unspecified)."""
    coords = np.array([[-1, -1], [0, -1], [-1, 0], [0, 0], [1, 0], [-1, 1], [0, 1], [1, 1]],
                      dtype=np.float64)
    elems = np.array([[0, 1, 3], [0, 3, 2], [2, 3, 6], [2, 6, 5], [3, 4, 7], [3, 7, 6]])
    dirichlet = np.array([[2, 0], [5, 2], [0, 1], [1, 3], [3, 4]])
    neumann = np.array([[4, 7], [7, 6], [6, 5]])
    return HostMesh(coords, elems, dirichlet, neumann)


def fan(k: int, center_last: bool = True) -> HostMesh:
    """A disc fan: one centre node of valence k (tests the high-valence
    fallbacks of the edge-generation tile kernel).  Ring edges are Dirichlet."""
    ang = 2.0 * math.pi * np.arange(k) / k
    ring = np.stack([np.cos(ang), np.sin(ang)], axis=1)
    if center_last:
        coords = np.vstack([ring, [[0.0, 0.0]]])
        c, r = k, np.arange(k)
    else:
        coords = np.vstack([[[0.0, 0.0]], ring])
        c, r = 0, np.arange(1, k + 1)
    elems = np.stack([np.full(k, c), r, np.roll(r, -1)], axis=1)
    dirichlet = np.stack([r, np.roll(r, -1)], axis=1)
    return HostMesh(coords, elems, dirichlet, np.zeros((0, 2)))


# ---- config-4 stress transformation --------------------------------------------
def stress_transform(hm: HostMesh, level: int, seeds=(1, 2, 3, 4)) -> HostMesh:
    """Jitter interior nodes by U[-0.2h, 0.2h] (h = 2^-level, the leg length),
    permute elements, rotate each vertex triple and flip half of them to CW.
    The result is NOT a valid reference input until orientation-normalised
    (phfem_orient_ccw / oracle orient_ccw)."""
    coords = hm.coords.copy()
    h = 2.0 ** (-level)
    x, y = coords[:, 0], coords[:, 1]
    interior = (x > 0.0) & (x < 1.0) & (y > 0.0) & (y < 1.0)
    n = coords.shape[0]
    jx = uniform_pm1(seeds[0], 2 * n)
    coords[interior, 0] += 0.2 * h * jx[0::2][interior]
    coords[interior, 1] += 0.2 * h * jx[1::2][interior]
    nE = hm.nE
    perm = np.argsort(splitmix64(seeds[1], nE), kind="stable")
    elems = hm.elements[perm].copy()
    rot = (splitmix64(seeds[2], nE) % np.uint64(3)).astype(np.int64)
    idx = (np.arange(3)[None, :] + rot[:, None]) % 3
    elems = np.take_along_axis(elems, idx, axis=1)
    flip = (splitmix64(seeds[3], nE) >> np.uint64(63)).astype(bool)
    elems[flip, 1], elems[flip, 2] = elems[flip, 2].copy(), elems[flip, 1].copy()
    return HostMesh(coords, elems, hm.dirichlet.copy(), hm.neumann.copy())


def signed_area2(hm: HostMesh) -> np.ndarray:
    a, b, c = (hm.coords[hm.elements[:, k]] for k in range(3))
    return (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0])


# ---- configuration presets -------------------------------------------------------
def config_fields(cfg: int):
    """(coeffs, f, g, uD) of BASELINE.json configs[cfg-1] (fields fixed in-repo
    where the BASELINE leaves them open)."""
    if cfg == 1:
        return (coeffs_const(), field(FIELD_SINSIN, TWO_PI2), field(FLUX_GRAD_SINSIN, 1.0),
                field(FIELD_ZERO))
    if cfg in (2, 4, 5):
        return (coeffs_centroid_poly((0.1, -0.1)), field(FIELD_SINSIN, TWO_PI2), field(FLUX_ZERO),
                field(FIELD_ZERO))
    if cfg == 3:
        return (coeffs_const(), field(FIELD_EXP_SINSIN, TWO_PI2_M1), field(FLUX_ZERO),
                field(FIELD_ZERO))
    raise ValueError(cfg)


CONFIG_COARSE = {1: square_2tri, 2: lshape_6tri, 3: square_2tri, 4: square_2tri, 5: square_2tri}
CONFIG_LEVELS = {1: 6, 2: 10, 3: 11, 4: 12, 5: 13}
