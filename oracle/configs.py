"""Problem definitions for the oracle (TEST INFRASTRUCTURE ONLY).

Two families:

* ``reference_problem(name)`` -- the reference's built-in problems exactly as
  ``pkg/src/stmhd/problems.py:66-127`` defines them (tearing mode on
  [0,3]x[0,1/2], island coalescence on [0,1]^2, Dirichlet A on top only,
  P3/P2 velocity/pressure).
* ``baseline_problem(cfg)`` -- the BASELINE.json configurations through the
  SURVEY.md section 0.1 adapter: [-1,1]^2, P2/P1, Dirichlet A on top *and*
  bottom with the bottom edge flux added to the current equation.

A problem is a plain record of closures; the discretisation lives in
``oracle.model``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np


@dataclass(frozen=True)
class ProblemSpec:
    """Closures and parameters of one model problem (mirrors the fields of
    ``ProblemSpec``, reference ``problems.py:25-47``)."""

    name: str
    domain: tuple
    mu: float
    eta: float
    mu0: float
    a_eq: Callable
    e_eq: Callable
    p_eq: Callable
    a_pert: Callable
    # side -> outward normal derivative of A_eq on that side (flux of j eq.)
    flux: dict
    # sides carrying a Dirichlet condition for A (u is slip everywhere)
    a_dirichlet: tuple
    vel_degree: int = 2


def _island(beta, mu, eta, mu0, amp, pert, domain, dirichlet, flux_sides, deg):
    """Fadeev equilibrium, reference ``problems.py:96-127``."""
    tp = 2.0 * np.pi

    def sheet(x, y):
        return np.cosh(tp * y) + beta * np.cos(tp * x)

    def a_eq(x, y):
        return np.log(sheet(x, y)) / tp

    def e_eq(x, y):
        return (eta / mu0) * tp * (1.0 - beta**2) / sheet(x, y) ** 2

    def p_eq(x, y):
        return (1.0 - beta**2) / (2.0 * mu0 * sheet(x, y) ** 2)

    def dady(x, y):
        return np.sinh(tp * y) / sheet(x, y)

    flux = {}
    if "top" in flux_sides:
        flux["top"] = dady
    if "bottom" in flux_sides:
        flux["bottom"] = lambda x, y: -dady(x, y)
    return ProblemSpec("island_coalescence", domain, mu, eta, mu0, a_eq, e_eq, p_eq,
                       lambda x, y: amp * pert(x, y), flux, dirichlet, deg)


def _harris(lam_mode, lam, mu, eta, mu0, amp, pert, domain, dirichlet, flux_sides, deg):
    """Harris sheet.  ``lam_mode='inv'`` is the reference form
    ln(cosh(lam y))/lam (``problems.py:71-84``); ``'mul'`` is the BASELINE
    form lam*ln(cosh(y/lam))."""
    s = lam if lam_mode == "inv" else 1.0 / lam

    def a_eq(x, y):
        return np.log(np.cosh(s * y)) / s + 0.0 * x

    def e_eq(x, y):
        return (s * eta / mu0) * np.cosh(s * y) ** -2 + 0.0 * x

    def p_eq(x, y):
        return np.cosh(s * y) ** -2 / (2.0 * mu0) + 0.0 * x

    def dady(x, y):
        return np.tanh(s * y) + 0.0 * x

    flux = {}
    if "top" in flux_sides:
        flux["top"] = dady
    if "bottom" in flux_sides:
        flux["bottom"] = lambda x, y: -dady(x, y)
    return ProblemSpec("tearing_mode", domain, mu, eta, mu0, a_eq, e_eq, p_eq,
                       lambda x, y: amp * pert(x, y), flux, dirichlet, deg)


def reference_problem(name: str, **kw) -> ProblemSpec:
    """Built-in problems of the reference with its default parameters."""
    if name == "island_coalescence":
        eps = kw.get("eps", 1e-3)
        return _island(kw.get("beta", 0.2), kw.get("mu", 1.0), kw.get("eta", 1.0),
                       kw.get("mu0", 1.0), eps,
                       lambda x, y: np.cos(0.5 * np.pi * y) * np.cos(np.pi * x),
                       (0.0, 1.0, 0.0, 1.0), ("top",), ("top",), 3)
    if name == "tearing_mode":
        eps = kw.get("eps", 1e-3)
        length = kw.get("length", 3.0)
        return _harris("inv", kw.get("lam", 5.0), kw.get("mu", 1.0), kw.get("eta", 1.0),
                       kw.get("mu0", 1.0), -eps,
                       lambda x, y: np.cos(np.pi * y) * np.cos(2.0 * np.pi * x / length),
                       (0.0, length, 0.0, 0.5), ("top",), ("top",), 3)
    raise KeyError(name)


# BASELINE.json configurations (SURVEY.md section 8 notation C1..C5).
CONFIGS = {
    "C1": dict(problem="island", n=16, dt=0.1, nt=8, visc=1e-2, newton="one_step"),
    "C2": dict(problem="island", n=32, dt=0.05, nt=64, visc=1e-2, newton="rel1e-6"),
    "C3": dict(problem="tearing", n=64, dt=0.02, nt=128, visc=1e-3, newton="rel1e-6"),
    "C4_64": dict(problem="island", n=64, dt=1.0 / 64, nt=64, visc=1e-2, newton="rel1e-6"),
    "C4_128": dict(problem="island", n=64, dt=1.0 / 128, nt=128, visc=1e-2, newton="rel1e-6"),
    "C4_256": dict(problem="island", n=64, dt=1.0 / 256, nt=256, visc=1e-2, newton="rel1e-6"),
    "C4_512": dict(problem="island", n=64, dt=1.0 / 512, nt=512, visc=1e-2, newton="rel1e-6"),
}


def baseline_problem(kind: str, visc: float, vel_degree: int = 2) -> ProblemSpec:
    """BASELINE physics on [-1,1]^2 through the SURVEY 0.1 adapter."""
    dom = (-1.0, 1.0, -1.0, 1.0)
    sides = ("top", "bottom")
    if kind == "island":
        return _island(0.2, visc, visc, 1.0, 1e-3,
                       lambda x, y: np.cos(0.5 * np.pi * x) * np.cos(0.5 * np.pi * y),
                       dom, sides, sides, vel_degree)
    if kind == "tearing":
        return _harris("mul", 0.5, visc, visc, 1.0, 1e-3,
                       lambda x, y: np.cos(np.pi * x) * np.cos(0.5 * np.pi * y),
                       dom, sides, sides, vel_degree)
    raise KeyError(kind)
