"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO sorting arithmetic: only the counter-based generators
that stand in for the paper's input distributions (§5) and
BASELINE.json's five configs.  See generators.py.
"""
from .generators import *  # noqa: F401,F403
