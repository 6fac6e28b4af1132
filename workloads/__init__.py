"""Seeded synthetic input generators (no method arithmetic); see workloads/gen.py."""
from .gen import *  # noqa: F401,F403
