"""Configuration-5 synthetic inputs: the per-slab
divergence-free advection fields of the scalar advection-diffusion
micro-benchmark.

For each slab k, in order, from one ``np.random.default_rng(seed)``:
``kx, ky = rng.integers(1, 9, size=(8, 2))`` and ``a = rng.standard_normal(8)``;
psi_k = sum_m a_m sin(pi kx_m (x+1)/2) sin(pi ky_m (y+1)/2),
u_k = (d psi/dy, -d psi/dx) at the P1 nodes, scaled so max_node |u_k| = 1.
The same function feeds the GPU run, the CPU oracle and the golden fixture.
"""

from __future__ import annotations

import numpy as np


def c5_velocity_fields(coords: np.ndarray, nt: int, seed: int = 0) -> np.ndarray:
    """(nt, n_nodes, 2) nodal velocities for the slabs 0..nt-1."""
    rng = np.random.default_rng(seed)
    x = coords[:, 0] + 1.0
    y = coords[:, 1] + 1.0
    out = np.empty((nt, len(coords), 2))
    for k in range(nt):
        kk = rng.integers(1, 9, size=(8, 2))
        amp = rng.standard_normal(8)
        ux = np.zeros(len(coords))
        uy = np.zeros(len(coords))
        for (kx, ky), a in zip(kk, amp):
            sx, cx = np.sin(0.5 * np.pi * kx * x), np.cos(0.5 * np.pi * kx * x)
            sy, cy = np.sin(0.5 * np.pi * ky * y), np.cos(0.5 * np.pi * ky * y)
            ux += a * sx * (0.5 * np.pi * ky) * cy
            uy -= a * (0.5 * np.pi * kx) * cx * sy
        scale = np.sqrt(ux * ux + uy * uy).max()
        out[k, :, 0] = ux / scale
        out[k, :, 1] = uy / scale
    return out
