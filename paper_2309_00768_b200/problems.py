"""Model problems: the reference's built-ins and the BASELINE configurations.

``ProblemSpec`` is the reference record (``problems.py:25-47``) field for field --
``a_eq_normal_flux_top`` and ``bcs: BCSpec`` included, with the reference's
``BCSpec`` / ``Condition`` / ``dirichlet`` / ``slip`` / ``natural`` / ``Side``
vocabulary (``fem.py:478-529``, ``mesh.py`` sides) -- so a problem written for the
reference (or the reference's own ``ProblemSpec`` object) can be passed to
``discretize``.  Three optional adapter fields follow for the BASELINE
configurations: ``vel_degree`` (P2/P1 instead of the reference's
P3/P2), ``a_flux`` (natural-flux terms of the current equation on sides other than
the top) and ``a_dirichlet`` (legacy side list, used only when ``bcs`` is None).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from typing import Callable

import numpy as np

from .errors import ConfigurationError


class Side(Enum):
    """Rectangle sides (reference mesh.py Side)."""

    LEFT = "left"
    RIGHT = "right"
    BOTTOM = "bottom"
    TOP = "top"


class BCKind(Enum):
    DIRICHLET = "dirichlet"
    SLIP = "slip"
    NATURAL = "natural"


@dataclass(frozen=True)
class Condition:
    kind: BCKind
    value: Callable | None = None


def dirichlet(fn) -> Condition:
    return Condition(BCKind.DIRICHLET, fn)


def slip() -> Condition:
    return Condition(BCKind.SLIP)


def natural() -> Condition:
    return Condition(BCKind.NATURAL)


FIELDS = ("u", "p", "j", "A")


@dataclass(frozen=True)
class BCSpec:
    """Per-field, per-side boundary conditions (reference fem.py:508-529; same
    validation and error messages)."""

    conditions: dict

    def for_field(self, field_name: str) -> dict:
        if field_name not in FIELDS:
            raise ConfigurationError(f"unknown field '{field_name}'")
        per_side = self.conditions.get(field_name)
        if per_side is None:
            raise ConfigurationError(f"no boundary conditions given for field '{field_name}'")
        for side in Side:
            if side not in per_side:
                raise ConfigurationError(f"field '{field_name}' missing condition on {side.value}")
        for side in per_side:
            if not isinstance(side, Side):
                raise ConfigurationError(f"unknown boundary tag {side!r}")
        return per_side


@dataclass(frozen=True)
class ProblemSpec:
    name: str
    domain: tuple
    mu: float
    eta: float
    mu0: float
    eps: float
    a_eq: Callable
    e_eq: Callable
    p_eq: Callable
    a_perturbation: Callable
    a_eq_normal_flux_top: Callable | None = None
    bcs: BCSpec | None = None
    # adapter fields, absent from the reference record
    vel_degree: int = 3
    # outward normal derivative of A_eq per side name; when empty the top side
    # carries a_eq_normal_flux_top (the reference's only flux term)
    a_flux: dict = field(default_factory=dict)
    a_dirichlet: tuple = ("top",)


def enclosed_bcs(a_eq, a_dirichlet_sides=(Side.TOP,)) -> BCSpec:
    """Slip velocity on every side, natural p and j, Dirichlet potential (= a_eq)
    on `a_dirichlet_sides`, natural elsewhere (reference problems.py:50-63 with
    the top side only)."""
    sym = {s: slip() for s in Side}
    a_conditions = {s: natural() for s in Side}
    for s in a_dirichlet_sides:
        a_conditions[s] = dirichlet(a_eq)
    return BCSpec(conditions={"u": sym, "p": {s: natural() for s in Side},
                              "j": {s: natural() for s in Side}, "A": a_conditions})


# -- boundary data of a problem (reference fem.py:532-568, problems.py:173-180) ----

def _side_name(side) -> str:
    """Side key -> 'left'|'right'|'bottom'|'top' (this module's Side, the
    reference's Side enum, or a plain string)."""
    name = getattr(side, "value", side)
    if name not in ("left", "right", "bottom", "top"):
        raise ConfigurationError(f"unknown boundary tag {side!r}")
    return name


def _kind(cond) -> str:
    k = getattr(cond, "kind", None)
    k = getattr(k, "value", k)
    if k not in ("dirichlet", "slip", "natural"):
        raise ConfigurationError(f"unknown boundary condition {cond!r}")
    return k


def field_conditions(problem, field_name: str) -> dict | None:
    """{side name: condition} for one field from ``problem.bcs`` (validated by its
    own ``for_field``), or None when the problem carries no BCSpec."""
    bcs = getattr(problem, "bcs", None)
    if bcs is None:
        return None
    per_side = bcs.for_field(field_name) if hasattr(bcs, "for_field") else bcs.conditions[field_name]
    return {_side_name(s): c for s, c in per_side.items()}


def constrained_dofs(space, problem, field_name: str):
    """Constrained DOF indices and prescribed values of one field (reference
    ``constrained_dofs``, fem.py:532-568): slip fixes the normal component of a
    vector field to zero and is a no-op for scalar fields; Dirichlet takes the
    condition's value (a callable, or an (fx, fy) pair for a vector field).
    Without a BCSpec: slip on every side for u, Dirichlet a_eq on
    ``problem.a_dirichlet`` for A (the legacy adapter fields)."""
    from . import fem

    conds = field_conditions(problem, field_name)
    ncomp = 2 if field_name == "u" else 1
    if conds is None:
        if field_name == "u":
            conds = {s: slip() for s in fem.SIDES}
        elif field_name == "A":
            sides = tuple(_side_name(s) for s in getattr(problem, "a_dirichlet", ("top",)))
            conds = {s: (dirichlet(problem.a_eq) if s in sides else natural()) for s in fem.SIDES}
        else:
            conds = {s: natural() for s in fem.SIDES}
    idx_parts, val_parts = [], []
    for side in fem.SIDES:  # reference order: Side enum order left, right, bottom, top
        cond = conds[side]
        kind = _kind(cond)
        nodes = space.side_nodes[side]
        if kind == "natural":
            continue
        if kind == "slip":
            if ncomp == 1:
                continue
            idx_parts.append(nodes + fem.NORMAL_COMP[side] * space.n_nodes)
            val_parts.append(np.zeros(len(nodes)))
        else:
            x, y = space.coords[nodes, 0], space.coords[nodes, 1]
            if ncomp == 1:
                idx_parts.append(nodes)
                val_parts.append(np.asarray(cond.value(x, y), dtype=float) + np.zeros(len(nodes)))
            else:
                for comp, f in enumerate(cond.value):
                    idx_parts.append(nodes + comp * space.n_nodes)
                    val_parts.append(np.asarray(f(x, y), dtype=float) + np.zeros(len(nodes)))
    if not idx_parts:
        return np.empty(0, dtype=np.int64), np.empty(0)
    idx, first = np.unique(np.concatenate(idx_parts), return_index=True)
    return idx, np.concatenate(val_parts)[first]


def flux_terms(problem) -> dict:
    """{side name: outward normal derivative of A_eq} for the natural-flux term of
    the current equation: the adapter's ``a_flux`` when given, else the
    reference's single top-side term ``a_eq_normal_flux_top`` (problems.py:173-177)."""
    a_flux = getattr(problem, "a_flux", None)
    if a_flux:
        return {_side_name(s): f for s, f in a_flux.items()}
    top = getattr(problem, "a_eq_normal_flux_top", None)
    return {"top": top} if top is not None else {}


def _island_closures(beta, eta, mu0):
    tp = 2.0 * np.pi

    def sheet(x, y):
        return np.cosh(tp * y) + beta * np.cos(tp * x)

    return (lambda x, y: np.log(sheet(x, y)) / tp,
            lambda x, y: (eta / mu0) * tp * (1.0 - beta**2) / sheet(x, y) ** 2,
            lambda x, y: (1.0 - beta**2) / (2.0 * mu0 * sheet(x, y) ** 2),
            lambda x, y: np.sinh(tp * y) / sheet(x, y))


def _harris_closures(s, eta, mu0):
    """A = ln(cosh(s y))/s."""
    return (lambda x, y: np.log(np.cosh(s * y)) / s + 0.0 * x,
            lambda x, y: (s * eta / mu0) * np.cosh(s * y) ** -2 + 0.0 * x,
            lambda x, y: np.cosh(s * y) ** -2 / (2.0 * mu0) + 0.0 * x,
            lambda x, y: np.tanh(s * y) + 0.0 * x)


def island_coalescence(eps=1e-3, beta=0.2, mu=1.0, eta=1.0, mu0=1.0) -> ProblemSpec:
    """Reference built-in (problems.py:96-127): [0,1]^2, Dirichlet A on top, P3/P2."""
    a, e, p, dady = _island_closures(beta, eta, mu0)
    return ProblemSpec("island_coalescence", (0.0, 1.0, 0.0, 1.0), mu, eta, mu0, eps, a, e, p,
                       lambda x, y: eps * np.cos(0.5 * np.pi * y) * np.cos(np.pi * x),
                       dady, enclosed_bcs(a))


def tearing_mode(eps=1e-3, lam=5.0, length=3.0, mu=1.0, eta=1.0, mu0=1.0) -> ProblemSpec:
    """Reference built-in (problems.py:66-93): [0,L]x[0,1/2], Dirichlet A on top, P3/P2."""
    a, e, p, dady = _harris_closures(lam, eta, mu0)
    return ProblemSpec("tearing_mode", (0.0, length, 0.0, 0.5), mu, eta, mu0, eps, a, e, p,
                       lambda x, y: -eps * np.cos(np.pi * y) * np.cos(2.0 * np.pi * x / length),
                       dady, enclosed_bcs(a))


PROBLEMS = {"tearing_mode": tearing_mode, "island_coalescence": island_coalescence}


def by_name(name: str, **kw) -> ProblemSpec:
    try:
        return PROBLEMS[name](**kw)
    except KeyError:
        raise ConfigurationError(f"unknown problem '{name}'") from None


def baseline_island(visc=1e-2, vel_degree=2) -> ProblemSpec:
    """BASELINE island coalescence on [-1,1]^2 (lambda = 1/(2 pi), eps(beta)=0.2,
    perturbation 1e-3 cos(pi x/2) cos(pi y/2))."""
    a, e, p, dady = _island_closures(0.2, visc, 1.0)
    return ProblemSpec("island_coalescence", (-1.0, 1.0, -1.0, 1.0), visc, visc, 1.0, 1e-3, a, e, p,
                       lambda x, y: 1e-3 * np.cos(0.5 * np.pi * x) * np.cos(0.5 * np.pi * y),
                       dady, enclosed_bcs(a, (Side.TOP, Side.BOTTOM)), vel_degree,
                       {"top": dady, "bottom": lambda x, y: -dady(x, y)}, ("top", "bottom"))


def baseline_tearing(visc=1e-3, vel_degree=2) -> ProblemSpec:
    """BASELINE tearing mode on [-1,1]^2: A0 = 0.5 ln cosh(2y), perturbation
    1e-3 cos(pi x) cos(pi y/2)."""
    a, e, p, dady = _harris_closures(2.0, visc, 1.0)
    return ProblemSpec("tearing_mode", (-1.0, 1.0, -1.0, 1.0), visc, visc, 1.0, 1e-3, a, e, p,
                       lambda x, y: 1e-3 * np.cos(np.pi * x) * np.cos(0.5 * np.pi * y),
                       dady, enclosed_bcs(a, (Side.TOP, Side.BOTTOM)), vel_degree,
                       {"top": dady, "bottom": lambda x, y: -dady(x, y)}, ("top", "bottom"))


# BASELINE.json configurations (SURVEY.md section 8 notation).
CONFIGS = {
    "C1": dict(problem="island", n=16, dt=0.1, nt=8, visc=1e-2, newton_rel=None),
    "C2": dict(problem="island", n=32, dt=0.05, nt=64, visc=1e-2, newton_rel=1e-6),
    "C3": dict(problem="tearing", n=64, dt=0.02, nt=128, visc=1e-3, newton_rel=1e-6),
    "C4_64": dict(problem="island", n=64, dt=1.0 / 64, nt=64, visc=1e-2, newton_rel=1e-6),
    "C4_128": dict(problem="island", n=64, dt=1.0 / 128, nt=128, visc=1e-2, newton_rel=1e-6),
    "C4_256": dict(problem="island", n=64, dt=1.0 / 256, nt=256, visc=1e-2, newton_rel=1e-6),
    "C4_512": dict(problem="island", n=64, dt=1.0 / 512, nt=512, visc=1e-2, newton_rel=1e-6),
}


def config_problem(name: str) -> tuple:
    """(ProblemSpec, n, dt, nt, newton_rel) of a BASELINE configuration."""
    c = CONFIGS[name]
    prob = baseline_island(c["visc"]) if c["problem"] == "island" else baseline_tearing(c["visc"])
    return prob, c["n"], c["dt"], c["nt"], c["newton_rel"]
