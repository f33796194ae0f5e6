"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no semi-Lagrangian step, no
interpolation, no spectral operator of the method).  It only draws seeded
parameters and evaluates closed-form fields: analytic phantoms, analytic
velocity fields, and the exact transport of an analytic phantom along the
analytic characteristics of v* (classical RK4 on the ODE dX/dt = v*(X)).
Recipes: DESIGN.md §5 (after SURVEY.md §8(d), BASELINE.json configs).
"""
from .phantoms import CONFIGS, make_problem, sample_sinusoid_field  # noqa: F401
