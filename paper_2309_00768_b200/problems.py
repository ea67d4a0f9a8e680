"""Model problems: the reference's built-ins and the BASELINE configurations.

``ProblemSpec`` keeps the field names of the reference record
(``problems.py:25-47``) and adds the adapter knobs SURVEY.md 0.1 fixes for
the BASELINE configs: the velocity degree (P2/P1 instead of P3/P2), the
sides carrying a Dirichlet potential and the matching natural-flux sides of
the current equation.  The choice "Dirichlet A on top and bottom, flux on
both" is frozen here and is the one the CPU oracle's fixtures were made with.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .errors import ConfigurationError


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
    # outward normal derivative of A_eq per side (natural flux of the j equation)
    a_flux: dict = field(default_factory=dict)
    a_dirichlet: tuple = ("top",)
    vel_degree: int = 3


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
                       {"top": dady}, ("top",), 3)


def tearing_mode(eps=1e-3, lam=5.0, length=3.0, mu=1.0, eta=1.0, mu0=1.0) -> ProblemSpec:
    """Reference built-in (problems.py:66-93): [0,L]x[0,1/2], Dirichlet A on top, P3/P2."""
    a, e, p, dady = _harris_closures(lam, eta, mu0)
    return ProblemSpec("tearing_mode", (0.0, length, 0.0, 0.5), mu, eta, mu0, eps, a, e, p,
                       lambda x, y: -eps * np.cos(np.pi * y) * np.cos(2.0 * np.pi * x / length),
                       {"top": dady}, ("top",), 3)


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
                       {"top": dady, "bottom": lambda x, y: -dady(x, y)}, ("top", "bottom"),
                       vel_degree)


def baseline_tearing(visc=1e-3, vel_degree=2) -> ProblemSpec:
    """BASELINE tearing mode on [-1,1]^2: A0 = 0.5 ln cosh(2y), perturbation
    1e-3 cos(pi x) cos(pi y/2)."""
    a, e, p, dady = _harris_closures(2.0, visc, 1.0)
    return ProblemSpec("tearing_mode", (-1.0, 1.0, -1.0, 1.0), visc, visc, 1.0, 1e-3, a, e, p,
                       lambda x, y: 1e-3 * np.cos(np.pi * x) * np.cos(0.5 * np.pi * y),
                       {"top": dady, "bottom": lambda x, y: -dady(x, y)}, ("top", "bottom"),
                       vel_degree)


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
