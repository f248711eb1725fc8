"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This package holds NONE of the method's arithmetic: it only draws the
inputs a user would hand to ``de_setup``/``de_solve`` (mesh sizes, the
Dirichlet mask, element densities, the nodal load vector).  Recipes follow
BASELINE.json ``configs`` with the readings listed in DESIGN.md §3.
"""
from .configs import Problem, make_config, config_names, density_sequence_step, paper_problem  # noqa: F401
