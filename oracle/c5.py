"""Configuration-5 scalar advection-diffusion operator (TEST INFRASTRUCTURE
ONLY).  SURVEY.md 8(d): per slab F_k = M/dt + 1e-3 K + W(u_k) on a P1 space,
W from reference fem.py:430-462 (lin_a with a P1 vector velocity), Dirichlet
rows on top/bottom via bc_identity (fem.py:593-600), sub-diagonal -M/dt with
BC rows/cols zeroed (fem.py:603-610).  The "preconditioner application" is the
exact inverse by sequential block forward substitution with per-slab SuperLU
(reference solve_potential, precond.py:173-180)."""

from __future__ import annotations

import numpy as np

from . import fe
from .model import LU


class C5:
    def __init__(self, n, nt, ufields, dt=1e-2, eps=1e-3):
        self.mesh = fe.Mesh(-1.0, 1.0, -1.0, 1.0, n, n)
        self.p1 = fe.Space(self.mesh, 1)
        self.v1 = fe.Space(self.mesh, 1, 2)
        p1 = self.p1
        self.bc = np.unique(np.concatenate([p1.side_nodes["top"], p1.side_nodes["bottom"]]))
        m, k = fe.mass(p1), fe.stiffness(p1)
        self.coupling = fe.bc_zero((m / dt).tocsr(), rows=self.bc, cols=self.bc)
        self.nt, self.n = nt, p1.ndof
        self.F = []
        for kk in range(nt):
            u = np.concatenate([ufields[kk, :, 0], ufields[kk, :, 1]])
            _, lin_a, _ = fe.potential_advection(p1, self.v1, u, np.zeros(p1.ndof))
            self.F.append(fe.bc_identity((m / dt + eps * k + lin_a).tocsr(), self.bc))
        self._lu = None

    def apply(self, x):
        x = x.reshape(self.nt, self.n)
        y = np.empty_like(x)
        for k in range(self.nt):
            y[k] = self.F[k] @ x[k]
            if k:
                y[k] -= self.coupling @ x[k - 1]
        return y

    def factor(self):
        self._lu = [LU(f) for f in self.F]

    def solve(self, r):
        if self._lu is None:
            self.factor()
        r = r.reshape(self.nt, self.n)
        x = np.empty_like(r)
        for k in range(self.nt):
            x[k] = self._lu[k].solve(r[k] if k == 0 else r[k] + self.coupling @ x[k - 1])
        return x
